// K3B — persistent batched A^k for n <= 128 with TWO independent chains per
// SM, split-FP32 as three bf16 planes (kind::f16 tcgen05, fp32 accumulate).
//
// Why: a 128x128 chain step is 48 tensor-core MMAs (~3100 cycles) followed by
// an epilogue (drain D, split, write the next operands) of the same order.
// One chain per SM serialises the two (K3, kernels_tf32.cu: tensor pipe ~50%
// busy).  Two chains per SM overlap chain X's MMAs with chain Y's epilogue,
// which needs two resident powers per SM.  3xTF32 operands cost 128 KB of
// SMEM + 256 TMEM columns per chain and do not fit twice; bf16x3 planes do:
//
//   x = b0 + b1 + b2,  b0 = rn_bf16(x), b1 = rn_bf16(x - b0), b2 = rn_bf16(x - b0 - b1)
//   (24 significant bits: the representation error is <= 2^-26 |x|, vs
//   2^-22 for the tf32 hi/lo pair), and
//   X*Y ~= x2*y0 + x0*y2 + x1*y1 + x0*y1 + x1*y0 + x0*y0
//   (dropped terms x1*y2, x2*y1, x2*y2 are <= 2^-24 relative).
//   Six bf16 MMAs run in the time of three tf32 MMAs (kind::f16 K=16 vs
//   kind::tf32 K=8 at the same 64 cycles per M=N=128 instruction).
//
// One row-major bf16 plane, stored as [c/64][r][128 B] with 16-byte units
// XOR-swizzled by r % 8, is at the same time a K-major SWIZZLE_128B LEFT
// operand and an MN-major SWIZZLE_128B RIGHT operand (measured:
// tools/bf16_probe.cu), so the power needs ONE copy per plane in SMEM.
//
//   SMEM (224 KB):  chain c: y0, y1, y2 planes of the resident power P (96 KB)
//                   S: b2 plane of the base for a MULTIPLY_BASE step (32 KB,
//                   shared by the chains, handed over with an mbarrier)
//   TMEM (512 col): chain c at 256c: D (fp32 accumulator, 128 cols),
//                   x0, x1 left-operand planes (2 bf16 per column, 64 cols each)
//
// Per step of chain c the issue warp runs 48 MMAs (M=N=128, K=16):
//   x2*y0 (SS; x2 = the y2 plane itself, or S) then x0*y2, x1*y1, x0*y1,
//   x1*y0 (TS, A from TMEM) and x0*y0 last — small terms first because the
//   tensor core truncates its fp32 accumulator on every MMA.
// One dedicated warp issues them (an issuing thread stalls while the MMA
// queue is full, so it must not also be an epilogue worker).  The 16 epilogue
// warps alternate between the chains: while the tensor pipe
// runs chain X's MMAs they drain chain Y's D, split it and publish Y's next
// operands (named barrier per chain), so the pipe always has the next
// chain's 48 MMAs queued.
//
// MULTIPLY_BASE computes base * acc (the base is the left operand), as K3
// does: equal to the reference's acc * base (expo.py:135-136) because acc is
// a power of the base.  Parity with the reference (linalg.py:151-164 chain,
// expo.py:121-139) is by the relative-Frobenius tolerance of SURVEY §8(d).
#include <cstring>

#include "mxp_internal.h"
#include "ptx.cuh"

namespace mxp {
namespace {

constexpr int kWorkers = 16;                   // epilogue warps: 4 TMEM lane quarters x 4
constexpr int kIssueWarp = kWorkers;           //   column groups, + one MMA-issue warp
constexpr int kIOWarp = kWorkers + 1;          //   + one TMA IO warp
constexpr int kThreads = (kWorkers + 2) * 32;  // 576 (<= 96 registers per thread)
constexpr uint32_t kPlane = 128u * 128u * 2u;     // one bf16 plane: 32 KB
constexpr uint32_t kChainSmem = 3u * kPlane;      // y0, y1, y2 of one chain
constexpr uint32_t kSOff = 2u * kChainSmem;       // base-b2 scratch
constexpr uint32_t kBarOff = kSOff + kPlane;      // mbarriers + TMEM slot
constexpr size_t kSmem = kBarOff + 256 + 1024;    // + alignment slack
constexpr uint32_t kIdesc = idesc_bf16_kmaj_mnmaj<128, 128>();
// plane 1 holds -b1 (split3): x1*y0 negates A, x0*y1 negates B
constexpr uint32_t kIdescNegA = kIdesc | (1u << 13);
constexpr uint32_t kIdescNegB = kIdesc | (1u << 14);
// descriptor address-field advance (16-byte units) per K=16 step
//   right operand (MN-major): 16 rows of 128 B;  left (K-major): 32 B inside
//   the 128-byte atom row, next 64-column chunk every 4 steps
constexpr uint32_t kBStep = (16u * 128u) >> 4;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023u) & ~uintptr_t(1023));
}

// Split the pair (a = column 2j, b = column 2j+1) into three packed bf16x2
// words p0 = b0, p1 = -b1, p2 = b2 (x = b0 + b1 + b2); every subtraction is
// exact.  The residuals come from mixed bf16-fp32 subtractions that read the
// bf16 half in place (FHADD.BF16): n1 = b0 - x = -r1, p1 = rn(n1) = -b1,
// r2 = p1 - n1 = r1 - b1 — 7 instructions per pair instead of 11 (unpacking
// each bf16 half first).  The MMAs that read p1 against a positive plane set
// the instruction descriptor's negate bit; x1*y1 needs none.
__device__ __forceinline__ void split3(float a, float b, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
    asm("{\n\t.reg .b16 l0, h0, l1, h1;\n\t.reg .f32 a1, b1, a2, b2;\n\t"
        "cvt.rn.bf16x2.f32 %0, %4, %3;\n\t"
        "mov.b32 {l0, h0}, %0;\n\t"
        "sub.f32.bf16 a1, l0, %3;\n\t"
        "sub.f32.bf16 b1, h0, %4;\n\t"
        "cvt.rn.bf16x2.f32 %1, b1, a1;\n\t"
        "mov.b32 {l1, h1}, %1;\n\t"
        "sub.f32.bf16 a2, l1, a1;\n\t"
        "sub.f32.bf16 b2, h1, b1;\n\t"
        "cvt.rn.bf16x2.f32 %2, b2, a2;\n\t}"
        : "=r"(p0), "=r"(p1), "=r"(p2)
        : "f"(a), "f"(b));
}

// Row `row`, columns [32g + 16h, +16) of a plane: two 16-byte units, unit
// index XOR row % 8 (a quarter-warp = 8 consecutive rows hits 8 distinct bank
// groups).
__device__ __forceinline__ void put_half(uint32_t plane, uint32_t row, uint32_t g, uint32_t h,
                                         const uint32_t (&p)[8]) {
    const uint32_t base = plane + (g >> 1) * 16384u + row * 128u;
    const uint32_t u0 = (g & 1u) * 4u + 2u * h;
    sts128(base + ((u0 ^ (row & 7u)) << 4), p[0], p[1], p[2], p[3]);
    sts128(base + (((u0 + 1u) ^ (row & 7u)) << 4), p[4], p[5], p[6], p[7]);
}

// 32 values of one row of an n x n fp32 matrix, zero padded to 128.
__device__ __forceinline__ void load_row(const float* __restrict__ src, int n, int vec,
                                         uint32_t row, uint32_t col0, float (&x)[32]) {
    if (vec) {  // n == 128, 16-byte aligned
        const float4* p = reinterpret_cast<const float4*>(src + row * 128u + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float4 v = __ldg(p + i);
            x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const uint32_t c = col0 + i;
            x[i] = (row < static_cast<uint32_t>(n) && c < static_cast<uint32_t>(n))
                       ? __ldg(src + static_cast<size_t>(row) * n + c)
                       : 0.f;
        }
    }
}

__device__ __forceinline__ void store_row(float* __restrict__ dst, int n, int vec, uint32_t row,
                                          uint32_t col0, const uint32_t (&v)[32]) {
    if (vec) {
        float4* p = reinterpret_cast<float4*>(dst + row * 128u + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            __stcs(p + i, make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                      __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])));
    } else if (row < static_cast<uint32_t>(n)) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (col0 + i < static_cast<uint32_t>(n))
                dst[static_cast<size_t>(row) * n + col0 + i] = __uint_as_float(v[i]);
    }
}

// One chain step: 48 MMAs (M=N=128, K=16) into D of chain C, small terms
// first; issued by ONE thread.  x2 (left b2 plane) is the chain's own y2 plane
// for a SQUARE and the scratch S (the base's b2) for a MULTIPLY_BASE step.
// The issue rate decides the kernel's speed (the tensor pipe must never wait
// for the issuer), so every operand is a compile-time offset from uniform
// values: chain and step kind are template parameters and TMEM is addressed
// from column 0 (the CTA owns the SM's whole TMEM, see k3b_batched_power).
template <uint32_t C, bool kMult>
__device__ __forceinline__ void k3b_issue(uint32_t tbase, uint32_t s0, uint64_t* mma_bar,
                                          uint64_t* s_free) {
    // descriptor bases: the chain's y0 plane, and the x2 plane (own y2 or S)
    const uint64_t y0 = smem_desc(s0 + C * kChainSmem, 16384, 1024, 2);
    const uint64_t x2 = kMult ? smem_desc(s0 + kSOff, 16, 1024, 2)
                              : smem_desc(s0 + C * kChainSmem + 2 * kPlane, 16, 1024, 2);
    constexpr uint32_t D = C * 256u, X0 = D + 128u, X1 = D + 192u;
    constexpr uint32_t Y1 = kPlane >> 4, Y2 = 2 * kPlane >> 4;
    mma_f16_ss_x8<D, 0, kBStep, (16384u >> 4), true>(tbase, x2, y0, kIdesc);  // x2*y0
    if (kMult) mma_commit_warp(s_free);
    mma_f16_ts_x8<D, X0, Y2, kBStep>(tbase, y0, kIdesc);  // x0*y2
    mma_f16_ts_x8<D, X1, Y1, kBStep>(tbase, y0, kIdesc);      // x1*y1 ((-b1)(-b1))
    mma_f16_ts_x8<D, X0, Y1, kBStep>(tbase, y0, kIdescNegB);  // x0*y1
    mma_f16_ts_x8<D, X1, 0, kBStep>(tbase, y0, kIdescNegA);   // x1*y0
    mma_f16_ts_x8<D, X0, 0, kBStep>(tbase, y0, kIdesc);   // x0*y0
    mma_commit_warp(mma_bar + C);
}

// Global IO (n == 128) through a warp-private 4 KB SMEM tile: the warp's 32
// rows x 32 columns, row r at r * 128 B with its 16-byte units XOR r % 8 —
// the TMA SWIZZLE_128B box layout, and conflict-free for thread-per-row
// access (the TMEM lane layout).  TMA moves whole tiles between HBM and SMEM
// asynchronously, off the epilogue warps' instruction stream.
__device__ __forceinline__ void tile_put_rows(uint32_t tile, uint32_t lane, const uint32_t (&v)[32]) {
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u)
        sts128(tile + lane * 128u + ((u ^ (lane & 7u)) << 4), v[4 * u], v[4 * u + 1], v[4 * u + 2],
               v[4 * u + 3]);
}
__device__ __forceinline__ void tile_get_rows(uint32_t tile, uint32_t lane, float (&x)[32]) {
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u) {
        const uint4 w = lds128(tile + lane * 128u + ((u ^ (lane & 7u)) << 4));
        x[4 * u] = __uint_as_float(w.x); x[4 * u + 1] = __uint_as_float(w.y);
        x[4 * u + 2] = __uint_as_float(w.z); x[4 * u + 3] = __uint_as_float(w.w);
    }
}
}  // namespace

size_t k3b_smem_bytes() { return kSmem; }

#ifdef K3B_TRACE  // tools/k3b_trace.cu: per-phase cycle totals of CTA 0 (warp 0 / issuer lane 0)
__device__ long long* g_k3b_trace;
__shared__ long long k3b_acc[16];
#define K3B_MARK(k)                                                          \
    do {                                                                     \
        if (blockIdx.x == 0 && (warp == 0 || warp == kIssueWarp || warp == kIOWarp) && lane == 0) { \
            const long long t_ = clock64();                                  \
            k3b_acc[k] += t_ - k3b_tprev;                                    \
            k3b_tprev = t_;                                                  \
        }                                                                    \
    } while (0)
#define K3B_COUNT(k)                                                         \
    do {                                                                     \
        if (blockIdx.x == 0 && (warp == 0 || warp == kIssueWarp || warp == kIOWarp) && lane == 0) k3b_acc[k] += 1; \
    } while (0)
#else
#define K3B_MARK(k) \
    do {            \
    } while (0)
#define K3B_COUNT(k) \
    do {             \
    } while (0)
#endif

// Matrices of CTA b are b, b + G, b + 2G, ... (G = gridDim.x); chain c takes
// every other one starting at b + cG.  Three roles run the same deterministic
// (chain, matrix, step) state machine, so they agree on every hand-off
// without exchanging state:
//   warps 0-15  epilogue: drain D, split, write the next operands, publish;
//   warp 16     MMA issue (one elected lane);
//   warp 17     IO: TMA stores of finished results and TMA loads of the next
//               inputs (n == 128), L2 prefetch one matrix ahead.
// A chain's matrix boundary takes two of its slots: OUT (drain the last
// product into the warp tiles, hand them to the IO warp) and, one slot later,
// IN (convert the freshly loaded input into operands, publish step 0).  In
// between, the epilogue warps serve the other chain, so the HBM round trip
// overlaps that chain's MMAs instead of stalling the epilogue.
__global__ void __launch_bounds__(kThreads, 1)
    k3b_batched_power(const __grid_constant__ CUtensorMap in_map,
                      const __grid_constant__ CUtensorMap out_map, const float* __restrict__ in,
                      float* __restrict__ out, int n, long long batch, PlanBits plan, int vec,
                      const int* __restrict__ idx, const int* __restrict__ count) {
    // idx != nullptr: recompute only the matrices listed in idx[0 .. *count)
    // (K3H's dynamic-range fixup, kernels_k3h.cu); matrix m of this launch is
    // matrix idx[m] of the caller's stack
    if (idx != nullptr) {
        // launched as K3H's programmatic dependent: wait for K3H's list
        asm volatile("griddepcontrol.wait;" ::: "memory");
        batch = *count;
        if (batch == 0) return;  // nothing listed: leave before any setup
    }
    auto mat = [&](long long m) -> long long { return idx != nullptr ? idx[m] : m; };
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint64_t* mma_bar = bars;        // [2] a chain's step MMAs completed
    uint64_t* s_free = bars + 2;     // the SS MMAs reading S completed
    uint64_t* out_ready = bars + 3;  // [2] a chain's result is in its warp tiles (16 arrivals)
    uint64_t* in_ready = bars + 5;   // [2] a chain's next input landed in its warp tiles (TMA)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        mbar_init(mma_bar, 1);
        mbar_init(mma_bar + 1, 1);
        mbar_init(s_free, 1);
        mbar_init(out_ready, kWorkers);
        mbar_init(out_ready + 1, kWorkers);
        mbar_init(in_ready, 1);
        mbar_init(in_ready + 1, 1);
        fence_mbar_init();
    }
    if (warp == kIssueWarp) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t s0 = smem_u32(smem);
    const long long G = gridDim.x;
    const size_t n2 = static_cast<size_t>(n) * n;
    const int last = plan.len - 1;
    constexpr int kIn = -2;  // s value: the next input is being loaded / converted

    // state of the current chain (c) and of the other one, swapped every slot
    // (runtime-indexed arrays would live in local memory)
    long long m_c = blockIdx.x, m_o = static_cast<long long>(blockIdx.x) + G;
    int s_c = kIn, s_o = kIn;
    bool act_c = m_c < batch, act_o = m_o < batch;
    // Start-phase skew: chain c of CTA b sits out its first dly slots, so the
    // chains' matrix boundaries (64 KB in + 64 KB out each) are spread over
    // the plan instead of hitting HBM from all 296 chains at once.
    int dly_c = 0, dly_o = 0;
    if (batch >= 4 * G && plan.len > 1) {
        dly_c = (2 * static_cast<int>(blockIdx.x)) % plan.len;
        dly_o = (2 * static_cast<int>(blockIdx.x) + 1) % plan.len;
    }
    uint32_t c = 0;
    uint32_t ph_c = 0, ph_o = 0;  // per-chain mbarrier parities of this role
#ifdef K3B_TRACE
    if (tid < 16) k3b_acc[tid] = 0;
    __syncthreads();
    long long k3b_tprev = clock64();
#endif
    auto swap_chains = [&]() {
        const long long tm = m_c;
        m_c = m_o;
        m_o = tm;
        const int ts = s_c;
        s_c = s_o;
        s_o = ts;
        const bool ta = act_c;
        act_c = act_o;
        act_o = ta;
        const int td = dly_c;
        dly_c = dly_o;
        dly_o = td;
        const uint32_t tp = ph_c;
        ph_c = ph_o;
        ph_o = tp;
        c ^= 1u;
    };
    // the 16 warp tiles of chain cc <-> matrix mm (TMA boxes of 32 x 32)
    auto tiles_load = [&](uint32_t cc, long long mm) {
        mbar_expect_tx(in_ready + cc, 16 * 4096);
        for (uint32_t w = 0; w < kWorkers; ++w)
            tma_load_2d_s(s0 + cc * kChainSmem + w * 4096u, &in_map, in_ready + cc,
                          static_cast<int32_t>((w >> 2) * 32), static_cast<int32_t>(mat(mm) * 128 + (w & 3) * 32));
        if (mm + 2 * G < batch)
            prefetch_l2(in + static_cast<size_t>(mat(mm + 2 * G)) * n2, static_cast<uint32_t>(n2 * 4));
    };

    if (warp == kIssueWarp) {
        // ------------------------------------------------------------ MMA issue
        while (act_c || act_o) {
            if (act_c && dly_c > 0) {
                --dly_c;
            } else if (act_c) {
                if (s_c == last) {  // OUT slot: nothing to issue
                    m_c += 2 * G;
                    act_c = m_c < batch;
                    s_c = kIn;
                } else {
                    s_c = (s_c == kIn) ? 0 : s_c + 1;
                    K3B_MARK(10);
                    named_bar_sync(1 + c, kWorkers * 32 + 32);
                    K3B_MARK(8);
                    tc_fence_after();  // the whole warp: the MMA blocks elect one lane
                    const bool mult = plan_is_mult(plan, s_c);
                    if (c == 0) {
                        if (mult) k3b_issue<0, true>(tmem, s0, mma_bar, s_free);
                        else k3b_issue<0, false>(tmem, s0, mma_bar, s_free);
                    } else {
                        if (mult) k3b_issue<1, true>(tmem, s0, mma_bar, s_free);
                        else k3b_issue<1, false>(tmem, s0, mma_bar, s_free);
                    }
                    __syncwarp();
                    K3B_MARK(9);
                }
            }
            swap_chains();
        }
    } else if (warp == kIOWarp) {
        // ------------------------------------------------------------ IO (TMA)
        if (vec && lane == 0) {
            if (act_c) tiles_load(0, m_c);
            if (act_o) tiles_load(1, m_o);
        }
        while (act_c || act_o) {
            if (act_c && dly_c > 0) {
                --dly_c;
            } else if (act_c) {
                if (s_c == last) {
                    const long long m_prev = m_c;
                    m_c += 2 * G;
                    act_c = m_c < batch;
                    s_c = kIn;
                    if (vec) {
                        K3B_MARK(10);
                        mbar_wait_sleep(out_ready + c, ph_c);
                        ph_c ^= 1;
                        K3B_MARK(8);
                        if (lane == 0) {
                            for (uint32_t w = 0; w < kWorkers; ++w)
                                tma_store_2d_s(&out_map, s0 + c * kChainSmem + w * 4096u,
                                               static_cast<int32_t>((w >> 2) * 32),
                                               static_cast<int32_t>(mat(m_prev) * 128 + (w & 3) * 32));
                            bulk_commit_group();
                            bulk_wait_group_read0();  // tiles read: reuse them for the input
                            if (act_c) tiles_load(c, m_c);
                        }
                        __syncwarp();
                        K3B_MARK(9);
                    }
                } else {
                    s_c = (s_c == kIn) ? 0 : s_c + 1;
                }
            }
            swap_chains();
        }
        if (vec && lane == 0) bulk_wait_group0();  // results written before exit
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t q = warp & 3, g = warp >> 2;
        const uint32_t row = q * 32 + lane;
        const uint32_t col0 = g * 32;
        const uint32_t lane_base = tmem + ((q * 32) << 16);
        const uint32_t tile_off = warp * 4096u;  // the warp's tile inside a chain's plane region
        uint32_t inph_c = 0, inph_o = 0;         // in_ready parities (swapped with the chains)
        uint32_t s_uses = 0;

        // 16 values (columns col0 + 16h ...) -> the chain's y planes and,
        // when `left`, its x0/x1 TMEM planes; !right: only the b2 plane, into S.
        auto emit = [&](uint32_t cc, uint32_t h, const float* x, bool right, bool left) {
            uint32_t p0[8], p1[8], p2[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) split3(x[2 * j], x[2 * j + 1], p0[j], p1[j], p2[j]);
            // opaque copies: recompute the swizzled addresses here instead of
            // letting the compiler hoist ~20 of them out of the loop (and spill)
            uint32_t r_ = row, b_ = s0;
            asm volatile("" : "+r"(r_), "+r"(b_));
            if (right) {
                const uint32_t pb = b_ + cc * kChainSmem;
                put_half(pb, r_, g, h, p0);
                put_half(pb + kPlane, r_, g, h, p1);
                put_half(pb + 2 * kPlane, r_, g, h, p2);
            } else {
                put_half(b_ + kSOff, r_, g, h, p2);
            }
            if (left) {
                uint32_t lb_ = lane_base;
                asm volatile("" : "+r"(lb_));
                const uint32_t tl = lb_ + cc * 256u + 128u + g * 16u + h * 8u;
                tmem_st8(tl, p0);
                tmem_st8(tl + 64u, p1);
            }
        };
        // matrix m_c straight from global (n != 128, and the base of a MULTIPLY_BASE step)
        auto emit_global = [&](uint32_t cc, bool right, bool left) {
            float x[32];
            load_row(in + static_cast<size_t>(mat(m_c)) * n2, n, vec, row, col0, x);
            emit(cc, 0, x, right, left);
            emit(cc, 1, x + 16, right, left);
        };

        while (act_c || act_o) {
            if (act_c && dly_c > 0) {
                --dly_c;
            } else if (act_c) {
                bool publish = true;
                if (s_c == kIn) {
                    // ---- IN: the new matrix -> operands of step 0
                    if (vec) {
                        K3B_MARK(7);
                        mbar_wait_sleep(in_ready + c, inph_c);
                        inph_c ^= 1;
                        K3B_MARK(3);
                        float x[32];
                        tile_get_rows(s0 + c * kChainSmem + tile_off, lane, x);
                        named_bar_sync(3, kWorkers * 32);  // all tiles read before planes overwrite them
                        K3B_MARK(4);
                        emit(c, 0, x, true, true);
                        emit(c, 1, x + 16, true, true);
                        K3B_MARK(5);
                    } else {
                        emit_global(c, true, true);
                    }
                    s_c = 0;
                } else {
                    K3B_MARK(7);
                    mbar_wait_sleep(mma_bar + c, ph_c);
                    K3B_MARK(0);
                    ph_c ^= 1;
                    tc_fence_after();
                    uint32_t v[32];
                    tmem_ld32(lane_base + c * 256u + col0, v);
                    K3B_MARK(1);
                    if (s_c == last) {
                        // ---- OUT: the result -> the warp tile (IO warp stores it)
                        if (vec) {
                            tile_put_rows(s0 + c * kChainSmem + tile_off, lane, v);
                            fence_proxy_async_smem();
                            tc_fence_before();  // D reads done before the next MMAs into D
                            __syncwarp();
                            if (lane == 0) mbar_arrive(out_ready + c);
                            K3B_MARK(2);
                            K3B_COUNT(13);
                        } else {
                            store_row(out + static_cast<size_t>(mat(m_c)) * n2, n, vec, row, col0, v);
                            tc_fence_before();
                        }
                        m_c += 2 * G;
                        act_c = m_c < batch;
                        s_c = kIn;
                        publish = false;
                    } else {
                        s_c += 1;
                        const bool mult = plan_is_mult(plan, s_c);
                        emit(c, 0, reinterpret_cast<const float*>(v), true, !mult);
                        emit(c, 1, reinterpret_cast<const float*>(v) + 16, true, !mult);
                        K3B_MARK(6);
                        K3B_COUNT(14);
                        if (mult) {  // left operand = the base: x0, x1 to TMEM, x2 to S
                            if (s_uses > 0) mbar_wait_sleep(s_free, (s_uses - 1) & 1u);
                            emit_global(c, false, true);
                            ++s_uses;
                        }
                    }
                }
                if (publish) {
                    // workers arrive; the issue warp waits for all of them (the
                    // hardware barrier also drains pending st.shared) and issues
                    tmem_st_wait();
                    fence_proxy_async_smem();
                    tc_fence_before();
                    named_bar_arrive(1 + c, kWorkers * 32 + 32);
                }
            }
            swap_chains();
            const uint32_t tp = inph_c;
            inph_c = inph_o;
            inph_o = tp;
        }
    }
    tc_fence_before();
    __syncthreads();
#ifdef K3B_TRACE
    if (blockIdx.x == 0 && tid < 16) g_k3b_trace[tid] = k3b_acc[tid];
#endif
    if (warp == kIssueWarp) tmem_dealloc<512>(tmem);
}

cudaError_t prepare_k3b_kernel() {
    return cudaFuncSetAttribute(k3b_batched_power, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmem));
}

cudaError_t launch_k3b_batched(const float* in, float* out, int n, int64_t batch,
                               const PlanBits& plan, int grid, cudaStream_t s, const int* idx,
                               const int* count) {
    if (plan.len < 1 || n < 1 || n > kSmallMax) return cudaErrorInvalidValue;
    if (grid > batch) grid = static_cast<int>(batch);
    CUtensorMap in_map, out_map;
    std::memset(&in_map, 0, sizeof in_map);
    std::memset(&out_map, 0, sizeof out_map);
    int vec = (n == 128 && batch * 128 < (int64_t(1) << 31) &&
               (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
               (reinterpret_cast<uintptr_t>(out) & 15) == 0)
                  ? 1
                  : 0;
    if (vec && !(encode_tile_map(&in_map, in, batch * 128) && encode_tile_map(&out_map, out, batch * 128)))
        vec = 0;
    if (idx == nullptr) {
        k3b_batched_power<<<grid, kThreads, kSmem, s>>>(in_map, out_map, in, out, n, batch, plan, vec,
                                                        idx, count);
        return cudaGetLastError();
    }
    // the fixup pass: a programmatic dependent launch, so its launch latency
    // overlaps K3H's tail (it waits for K3H with griddepcontrol.wait)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k3b_batched_power, in_map, out_map, in, out, n,
                              static_cast<long long>(batch), plan, vec, idx, count);
}

}  // namespace mxp
