// sm_100a primitives: mbarrier, TMA, tcgen05 (TMEM alloc / MMA / commit / ld),
// UMMA shared-memory and instruction descriptors.  Inline PTX only — no
// CUTLASS types; the descriptor bit layouts follow the PTX ISA "matrix
// descriptor" / "instruction descriptor" tables for tcgen05.
#pragma once
#include <cstdint>
#include <cuda.h>

namespace mxp {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// NVLS multicast store: one 16-byte store to a multicast address is written
// by the NVSwitch into every bound copy (every rank's buffer)
__device__ __forceinline__ void multimem_st_v4(void* mc_addr, uint32_t a, uint32_t b, uint32_t c,
                                               uint32_t d) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_addr),
                 "f"(__uint_as_float(a)), "f"(__uint_as_float(b)), "f"(__uint_as_float(c)),
                 "f"(__uint_as_float(d))
                 : "memory");
}

// the GPU-wide nanosecond timer (pairs with clock64 to measure the SM clock)
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// No memory ordering: only for publishing completed tcgen05.ld drains.
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MXP_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MXP_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Same, but a waiting thread is suspended in hardware (up to `ns`) instead of
// spinning, so waiting warps leave the issue slots of their SM sub-partition to
// the warps that work (the MMA issuer above all).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns = 1000000) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MXP_WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra MXP_WAITS_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(ns)
        : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// TMA tensor store shared -> global (bulk-group completion), and the group waits.
// (shared addresses as 32-bit shared-window offsets)
__device__ __forceinline__ void tma_store_2d_s(const CUtensorMap* map, uint32_t src, int32_t c0,
                                               int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(src), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_s(uint32_t dst, const CUtensorMap* map, uint64_t* bar,
                                              int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_commit_group() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the shared-memory sources of all committed bulk stores have been read
__device__ __forceinline__ void bulk_wait_group_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_group0() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// 1-D bulk copy global -> shared (size and addresses 16-byte aligned).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// generic-proxy shared writes -> visible to the async proxy (tensor core / TMA)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::tf32, issued by ONE thread.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem] (A from tensor memory: lane = row m,
// column = k, one 32-bit tf32 per column), kind::tf32, issued by ONE thread.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// kind::f16 (bf16 operands here), SS and TS (A from TMEM: lane = row m, two
// 16-bit k-consecutive values per 32-bit column, the lower k in the low half —
// measured with tools/bf16_probe.cu).
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Offset forms: the constant offsets are added INSIDE the asm, so the
// compiler cannot hoist 48 precomputed descriptors into registers (each then
// needs an R2UR per MMA); ptxas adds them on the uniform datapath instead.
template <uint32_t kD, uint32_t kA, uint32_t kB>
__device__ __forceinline__ void mma_f16_ts_off(uint32_t tbase, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 dt, at;\n\t.reg .b64 bd;\n\t"
        "add.u32 dt, %0, %4;\n\t"
        "add.u32 at, %0, %5;\n\t"
        "add.s64 bd, %1, %6;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [dt], [at], bd, %2, p;\n}" ::"r"(tbase),
        "l"(bdesc), "r"(idesc), "r"(accumulate), "n"(kD), "n"(kA), "n"(kB)
        : "memory");
}
template <uint32_t kD, uint32_t kA, uint32_t kB>
__device__ __forceinline__ void mma_f16_ss_off(uint32_t tbase, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 dt;\n\t.reg .b64 ad, bd;\n\t"
        "add.u32 dt, %0, %5;\n\t"
        "add.s64 ad, %1, %6;\n\t"
        "add.s64 bd, %2, %7;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [dt], ad, bd, %3, p;\n}" ::"r"(tbase),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "n"(kD), "n"(kA), "n"(kB)
        : "memory");
}
// Eight K=16 steps of one term in ONE asm block (one elect/waterfall wrapper
// for all eight MMAs instead of one per MMA): A from TMEM columns
// tbase + kA + 8j, B descriptor bdesc + kB + j * kBStep, all accumulating.
template <uint32_t kD, uint32_t kA, uint32_t kB, uint32_t kBStep, bool kFirst = false>
__device__ __forceinline__ void mma_f16_ts_x8(uint32_t tbase, uint64_t bdesc, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p, p0, e;\n\t.reg .b32 dt, a0, a1, a2, a3, a4, a5, a6, a7;\n\t"
        ".reg .b64 b0, b1, b2, b3, b4, b5, b6, b7;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.eq.u32 p, 1, 1;\n\t"
        "setp.eq.u32 p0, %7, 0;\n\t"
        "add.u32 dt, %0, %3;\n\t"
        "add.u32 a0, %0, %4;\n\tadd.u32 a1, a0, 8;\n\tadd.u32 a2, a0, 16;\n\tadd.u32 a3, a0, 24;\n\t"
        "add.u32 a4, a0, 32;\n\tadd.u32 a5, a0, 40;\n\tadd.u32 a6, a0, 48;\n\tadd.u32 a7, a0, 56;\n\t"
        "add.s64 b0, %1, %5;\n\tadd.s64 b1, b0, %6;\n\tadd.s64 b2, b1, %6;\n\tadd.s64 b3, b2, %6;\n\t"
        "add.s64 b4, b3, %6;\n\tadd.s64 b5, b4, %6;\n\tadd.s64 b6, b5, %6;\n\tadd.s64 b7, b6, %6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a0], b0, %2, p0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a1], b1, %2, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a2], b2, %2, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a3], b3, %2, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a4], b4, %2, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a5], b5, %2, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a6], b6, %2, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], [a7], b7, %2, p;\n}" ::"r"(tbase),
        "l"(bdesc), "r"(idesc), "n"(kD), "n"(kA), "n"(kB), "n"(kBStep), "n"(kFirst ? 1 : 0)
        : "memory");
}
// SS: A descriptor adesc + (j/4) * kAChunk + (j%4) * 2 (K-major SW128, 32 B per
// K=16 step inside the atom), B as above; the first MMA overwrites D when
// kFirst (accumulate = 0).
template <uint32_t kD, uint32_t kB, uint32_t kBStep, uint32_t kAChunk, bool kFirst>
__device__ __forceinline__ void mma_f16_ss_x8(uint32_t tbase, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p, p0, e;\n\t.reg .b32 dt;\n\t"
        ".reg .b64 a0, a1, a2, a3, a4, a5, a6, a7, b0, b1, b2, b3, b4, b5, b6, b7;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.eq.u32 p, 1, 1;\n\t"
        "setp.eq.u32 p0, %7, 0;\n\t"
        "add.u32 dt, %0, %4;\n\t"
        "mov.b64 a0, %1;\n\tadd.s64 a1, a0, 2;\n\tadd.s64 a2, a0, 4;\n\tadd.s64 a3, a0, 6;\n\t"
        "add.s64 a4, a0, %6;\n\tadd.s64 a5, a4, 2;\n\tadd.s64 a6, a4, 4;\n\tadd.s64 a7, a4, 6;\n\t"
        "add.s64 b0, %2, %5;\n\tadd.s64 b1, b0, %8;\n\tadd.s64 b2, b1, %8;\n\tadd.s64 b3, b2, %8;\n\t"
        "add.s64 b4, b3, %8;\n\tadd.s64 b5, b4, %8;\n\tadd.s64 b6, b5, %8;\n\tadd.s64 b7, b6, %8;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a0, b0, %3, p0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a1, b1, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a2, b2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a3, b3, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a4, b4, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a5, b5, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a6, b6, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [dt], a7, b7, %3, p;\n}" ::"r"(tbase),
        "l"(adesc), "l"(bdesc), "r"(idesc), "n"(kD), "n"(kB), "n"(kAChunk), "n"(kFirst ? 1 : 0),
        "n"(kBStep)
        : "memory");
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {  // warp-collective
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
            smem_u32(bar))
        : "memory");
}
// Arrive on an mbarrier once every previously issued tcgen05 op of this
// thread has completed (implicitly fence::before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp receives
// lane (taddr.lane + t), columns [taddr.col, taddr.col + 32).  The wait is
// fused into the same asm statement so no consumer of r[] can be scheduled
// before the asynchronous load has landed.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
// Store 32 consecutive columns of this thread's lane (32x32b.x32), then wait.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
// 16-column variants (32x32b.x16).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
// Two 16-column loads (e.g. two accumulators) under a single wait.
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, uint32_t (&a)[16],
                                            uint32_t (&b)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
          "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]),
          "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]),
          "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]), "=r"(b[8]), "=r"(b[9]), "=r"(b[10]),
          "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15])
        : "r"(ta), "r"(tb)
        : "memory");
}
// Four 16-column loads under a single wait.
__device__ __forceinline__ void tmem_ld16x4(uint32_t ta, uint32_t tb, uint32_t tc, uint32_t td,
                                            uint32_t (&a)[16], uint32_t (&b)[16],
                                            uint32_t (&c)[16], uint32_t (&d)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%64];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%65];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47}, [%66];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%67];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
          "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]),
          "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]),
          "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]), "=r"(b[8]), "=r"(b[9]), "=r"(b[10]),
          "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15]), "=r"(c[0]),
          "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7]),
          "=r"(c[8]), "=r"(c[9]), "=r"(c[10]), "=r"(c[11]), "=r"(c[12]), "=r"(c[13]),
          "=r"(c[14]), "=r"(c[15]), "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]),
          "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]),
          "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(ta), "r"(tb), "r"(tc), "r"(td)
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                 "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}
// Split form: issue the load, do other work, then wait.  The wait takes the
// destination registers as in/out operands so no use of them can be
// scheduled before it.
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld_wait_dep(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                   "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                   "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- named barriers
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- clusters / CTA pairs
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}
// shared::cluster address of the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}
// 16 bytes from a shared::cluster address (distributed shared memory).  No
// "memory" clobber, so independent loads overlap (~0.5 us round trip each);
// the caller orders them after the cluster barrier that publishes the data.
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t cluster_addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(cluster_addr));
    return v;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
// Relaxed remote arrive: no memory ordering (the .release.cluster form costs a
// MEMBAR.ALL.GPU).  Valid when the only thing the arrive publishes is the
// completion of this thread's tcgen05.ld (already waited on with wait::ld).
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
// Pair (cta_group::2) variants.  The peer's TMA completes bytes on the
// leader's barrier: clear the peer bit (bit 24) of the shared address.
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
        "r"(smem_u32(bar) & kPeerBitMask)
        : "memory");
}
// the same box written into every CTA of `mask` (same SMEM offset); each
// destination's bytes complete on its pair leader's barrier at `bar`'s offset
__device__ __forceinline__ void tma_load_2d_pair_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                    int32_t c0, int32_t c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
        "r"(smem_u32(bar) & kPeerBitMask), "h"(mask)
        : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot) {  // one warp in EACH CTA
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// commit the pair's MMAs to the barrier at this offset in both CTAs
// arrive on `bar` (same offset) in every CTA of `mask` once the issued MMAs
// complete (0x3: both CTAs of the pair at cluster ranks 0/1)
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask = 0x3) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// ---------------------------------------------------------------- descriptors
// Shared-memory matrix descriptor, sm_100 version 1.
//   bits [0,14)  start address >> 4
//   bits [16,30) leading-dimension byte offset >> 4
//   bits [32,46) stride-dimension byte offset >> 4
//   bits [46,48) version (1 on sm_100)
//   bits [49,52) base offset (0: atoms are 1024-byte aligned)
//   bits [61,64) layout: 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
// K-major SW128 (left operand): rows of 128 B (32 fp32 of K), 16-byte units
//   XOR-swizzled by row % 8, 8-row atoms 1024 B apart (SBO); advancing K by 8
//   fp32 inside the atom adds 32 B to the start address.
// MN-major SW128_BASE32B (right operand; the ONLY MN-major layout the tf32
//   datapath accepts — plain SWIZZLE_128B MN-major silently yields zeros,
//   measured with tools/tc_probe3.cu): rows of 128 B (32 fp32 of N) indexed
//   by K, 32-byte units XOR-swizzled by K % 4, 4-row groups 512 B apart (SBO),
//   32-wide N chunks LBO bytes apart.  Matches TMA SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(layout & 7u) << 61;
    return d;
}
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr) {
    return smem_desc(saddr, 16, 1024, 2);
}
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t saddr, uint32_t chunk_stride) {
    return smem_desc(saddr, chunk_stride, 512, 1);
}
// Instruction descriptor, kind::tf32, fp32 accumulate, A K-major, B MN-major.
//   [4,6) c_format=1 (F32)  [7,10) a_format=2 (TF32)  [10,13) b_format=2 (TF32)
//   [15] a_major=0 (K)  [16] b_major=1 (MN)  [17,23) N>>3  [24,29) M>>4
template <int M, int N>
__host__ __device__ constexpr uint32_t idesc_tf32_kmaj_mnmaj() {
    static_assert(M == 64 || M == 128 || M == 256, "M (256: cta_group::2)");
    static_assert(N % 16 == 0 && N >= 16 && N <= 256, "N");
    return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// Instruction descriptor, kind::f16 with bf16 A/B, fp32 accumulate, A K-major,
// B MN-major:  [4,6) c_format=1  [7,10) a_format=1 (BF16)  [10,13) b_format=1
template <int M, int N>
__host__ __device__ constexpr uint32_t idesc_bf16_kmaj_mnmaj() {
    static_assert(M == 64 || M == 128, "M");
    static_assert(N % 16 == 0 && N >= 16 && N <= 256, "N");
    return (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// L2 prefetch of a global range (bulk async, no completion tracking).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)),
                 "r"(bytes)
                 : "memory");
}

// ---------------------------------------------------------------- 3xTF32 split
// hi = rna_tf32(x), lo = rna_tf32(x - hi).  The tensor core reads only the
// top 19 bits of each 32-bit operand, so both halves are pre-rounded.
// rna (round to nearest, ties away from zero) on the bit pattern: add half an
// ulp of the 10-bit mantissa (0x1000) and clear the 13 dropped bits.  Exact
// for finite values (carry into the exponent is the correct rounding, and
// overflow rounds to inf); inf stays inf.  NaNs are clamped to the quiet NaN
// 0x7FC00000 first: the GPU's arithmetic NaN is 0x7FFFFFFF, whose +0x1000
// would carry into the sign bit and turn it into -0 (a NaN in a chain's
// product vanished that way — test_one_launch_chain_zero_nan_identity).
// Four integer ops instead of the ~5-instruction cvt.rna.tf32.f32 lowering.
__device__ __forceinline__ uint32_t cvt_tf32(float x) {
    const uint32_t b = __float_as_uint(x);
    const uint32_t r = min(b & 0x7FFFFFFFu, 0x7FC00000u) + 0x1000u;
    return (r & 0xFFFFE000u) | (b & 0x80000000u);
}
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = cvt_tf32(x);
    lo = cvt_tf32(__fsub_rn(x, __uint_as_float(hi)));
}

// ---------------------------------------------------------------- shared memory
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}
template <uint32_t kOff>  // [addr + kOff]: the offset rides in the instruction
__device__ __forceinline__ void sts128_imm(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                           uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0+%5], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
                 "r"(d), "n"(kOff)
                 : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

// byte offset of element (r, c) inside a [c/32][r][32] fp32 tile whose column
// chunks are `chunk_bytes` apart: K-major SW128 (16-byte units ^ r%8) ...
__device__ __forceinline__ uint32_t sw128_offset(uint32_t r, uint32_t c, uint32_t chunk_bytes) {
    return (c >> 5) * chunk_bytes + r * 128u + ((((c & 31u) >> 2) ^ (r & 7u)) << 4) + (c & 3u) * 4u;
}
// ... and MN-major SW128_BASE32B (32-byte units ^ r%4).
__device__ __forceinline__ uint32_t sw32b_offset(uint32_t r, uint32_t c, uint32_t chunk_bytes) {
    return (c >> 5) * chunk_bytes + r * 128u + ((((c & 31u) >> 3) ^ (r & 3u)) << 5) + (c & 7u) * 4u;
}

}  // namespace mxp
