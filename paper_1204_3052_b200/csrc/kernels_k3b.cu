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
constexpr int kThreads = (kWorkers + 1) * 32;  // 544 (<= 96 registers per thread)
constexpr uint32_t kPlane = 128u * 128u * 2u;     // one bf16 plane: 32 KB
constexpr uint32_t kChainSmem = 3u * kPlane;      // y0, y1, y2 of one chain
constexpr uint32_t kSOff = 2u * kChainSmem;       // base-b2 scratch
constexpr uint32_t kBarOff = kSOff + kPlane;      // mbarriers + TMEM slot
constexpr size_t kSmem = kBarOff + 256 + 1024;    // + alignment slack
constexpr uint32_t kIdesc = idesc_bf16_kmaj_mnmaj<128, 128>();
// descriptor address-field advance (16-byte units) per K=16 step
//   right operand (MN-major): 16 rows of 128 B;  left (K-major): 32 B inside
//   the 128-byte atom row, next 64-column chunk every 4 steps
constexpr uint32_t kBStep = (16u * 128u) >> 4;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023u) & ~uintptr_t(1023));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float bf_lo(uint32_t p) { return __uint_as_float(p << 16); }
__device__ __forceinline__ float bf_hi(uint32_t p) { return __uint_as_float(p & 0xFFFF0000u); }

// Split the pair (a = column 2j, b = column 2j+1) into three packed bf16x2
// words; every subtraction is exact.
__device__ __forceinline__ void split3(float a, float b, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
    p0 = pack_bf16x2(a, b);
    const float a1 = __fsub_rn(a, bf_lo(p0)), b1 = __fsub_rn(b, bf_hi(p0));
    p1 = pack_bf16x2(a1, b1);
    const float a2 = __fsub_rn(a1, bf_lo(p1)), b2 = __fsub_rn(b1, bf_hi(p1));
    p2 = pack_bf16x2(a2, b2);
}

// Row `row`, columns [32g + 16h, +16) of a plane: two 16-byte units, unit
// index XOR row % 8 (a quarter-warp = 8 consecutive rows hits 8 distinct bank
// groups).
__device__ __forceinline__ void put_half(uint32_t plane, uint32_t row, uint32_t g, uint32_t h,
                                         const uint32_t (&p)[8]) {
    const uint32_t base = plane + (g >> 1) * 16384u + row * 128u;
    const uint32_t u0 = (g & 1u) * 4u + 2u * h;
#ifndef K3B_X_NOSTS
    sts128(base + ((u0 ^ (row & 7u)) << 4), p[0], p[1], p[2], p[3]);
    sts128(base + (((u0 + 1u) ^ (row & 7u)) << 4), p[4], p[5], p[6], p[7]);
#endif
}

// 32 values of one row of an n x n fp32 matrix, zero padded to 128.
__device__ __forceinline__ void load_row(const float* __restrict__ src, int n, int vec,
                                         uint32_t row, uint32_t col0, float (&x)[32]) {
#ifdef K3B_X_NOLDG
    for (int i = 0; i < 32; ++i) x[i] = (row + i) * 1e-3f;
    return;
#endif
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
#ifdef K3B_X_NOSTG
    if (v[0] == 0x7fc00001u) dst[row] = 0.f;
    return;
#endif
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
    mma_f16_ts_x8<D, X1, Y1, kBStep>(tbase, y0, kIdesc);  // x1*y1
    mma_f16_ts_x8<D, X0, Y1, kBStep>(tbase, y0, kIdesc);  // x0*y1
    mma_f16_ts_x8<D, X1, 0, kBStep>(tbase, y0, kIdesc);   // x1*y0
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
        if (blockIdx.x == 0 && (warp == 0 || warp == kIssueWarp) && lane == 0) { \
            const long long t_ = clock64();                                  \
            k3b_acc[k] += t_ - k3b_tprev;                                    \
            k3b_tprev = t_;                                                  \
        }                                                                    \
    } while (0)
#define K3B_COUNT(k)                                                         \
    do {                                                                     \
        if (blockIdx.x == 0 && (warp == 0 || warp == kIssueWarp) && lane == 0) k3b_acc[k] += 1; \
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
// every other one starting at b + cG.  The issue warp and the epilogue warps
// run the same deterministic (chain, matrix, step) state machine, so they
// agree on every publish without exchanging state.
__global__ void __launch_bounds__(kThreads, 1)
    k3b_batched_power(const __grid_constant__ CUtensorMap in_map,
                      const __grid_constant__ CUtensorMap out_map, const float* __restrict__ in,
                      float* __restrict__ out, int n, long long batch, PlanBits plan, int vec) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint64_t* mma_bar = bars;     // [2] a chain's step MMAs completed
    uint64_t* s_free = bars + 2;  // the SS MMAs reading S completed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
    uint64_t* io_bar = bars + 8;  // [16] per epilogue warp: its input tile landed (TMA)

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        mbar_init(mma_bar, 1);
        mbar_init(mma_bar + 1, 1);
        mbar_init(s_free, 1);
        for (int w = 0; w < kWorkers; ++w) mbar_init(io_bar + w, 1);
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

    // state of the current chain (c) and of the other one, swapped every slot
    // (runtime-indexed arrays would live in local memory)
    long long m_c = blockIdx.x, m_o = static_cast<long long>(blockIdx.x) + G;
    int s_c = -1, s_o = -1;
    bool act_c = m_c < batch, act_o = m_o < batch;
    // Start-phase skew: chain c of CTA b sits out its first dly slots, so the
    // chains' input/output steps (64 KB in + 64 KB out each) are spread over
    // the plan instead of hitting HBM from all 296 chains at once.
    int dly_c = 0, dly_o = 0;
    if (batch >= 4 * G && plan.len > 1) {
        dly_c = (2 * static_cast<int>(blockIdx.x)) % plan.len;
        dly_o = (2 * static_cast<int>(blockIdx.x) + 1) % plan.len;
    }
    uint32_t c = 0;
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
        c ^= 1u;
    };

    if (warp == kIssueWarp) {
        // ------------------------------------------------------------ MMA issue
        while (act_c || act_o) {
            if (act_c && dly_c > 0) {
                --dly_c;
            } else if (act_c) {
                if (s_c == last) {
                    m_c += 2 * G;
                    s_c = -1;
                    act_c = m_c < batch;
                }
                if (act_c) {
                    s_c += 1;
                    K3B_MARK(10);
                    named_bar_sync(1 + c, kThreads);
                    K3B_MARK(8);
                    {  // the whole warp: the MMA blocks elect one lane themselves
                        tc_fence_after();
                        const bool mult = plan_is_mult(plan, s_c);
                        if (c == 0) {
                            if (mult) k3b_issue<0, true>(tmem, s0, mma_bar, s_free);
                            else k3b_issue<0, false>(tmem, s0, mma_bar, s_free);
                        } else {
                            if (mult) k3b_issue<1, true>(tmem, s0, mma_bar, s_free);
                            else k3b_issue<1, false>(tmem, s0, mma_bar, s_free);
                        }
#ifndef K3B_X_NOPF
                        if (lane == 0 && vec && s_c == 0 && m_c + 2 * G < batch)
#else
                        if (false)
#endif
                            prefetch_l2(in + static_cast<size_t>(m_c + 2 * G) * n2,
                                        static_cast<uint32_t>(n2 * 4));
                    }
                    __syncwarp();
                    K3B_MARK(9);
                }
            }
            swap_chains();
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t q = warp & 3, g = warp >> 2;
        const uint32_t row = q * 32 + lane;
        const uint32_t col0 = g * 32;
        const uint32_t lane_base = tmem + ((q * 32) << 16);
        uint32_t ph_c = 0, ph_o = 0;  // mma_bar parities (swapped with the state)
        uint32_t s_uses = 0;

        // 16 values (columns col0 + 16h ...) -> the chain's y planes and,
        // when `left`, its x0/x1 TMEM planes; `sonly`: the base's b2 into S.
        auto emit = [&](uint32_t cc, uint32_t h, const float* x, bool right, bool left) {
#ifdef K3B_X_NOEPI
            return;
#endif
            uint32_t p0[8], p1[8], p2[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) split3(x[2 * j], x[2 * j + 1], p0[j], p1[j], p2[j]);
            if (right) {
                const uint32_t pb = s0 + cc * kChainSmem;
                put_half(pb, row, g, h, p0);
                put_half(pb + kPlane, row, g, h, p1);
                put_half(pb + 2 * kPlane, row, g, h, p2);
            } else {
                put_half(s0 + kSOff, row, g, h, p2);
            }
            if (left) {
                const uint32_t tl = lane_base + cc * 256u + 128u + g * 16u + h * 8u;
#ifndef K3B_X_NOTMEM
                tmem_st8(tl, p0);
                tmem_st8(tl + 64u, p1);
#endif
            }
        };
        // new matrix m_c of chain cc: all three planes + x0/x1.  For n == 128
        // the rows come in coalesced through the warp's tile in the chain's
        // (dead) plane region; `pre` holds loads already in flight.
        auto emit_input = [&](uint32_t cc, bool right, bool left) {
            const float* src = in + static_cast<size_t>(m_c) * n2;
            float x[32];
            load_row(src, n, vec, row, col0, x);
            emit(cc, 0, x, right, left);
            emit(cc, 1, x + 16, right, left);
        };
        const uint32_t tile_off = warp * 4096u;  // inside the chain's plane region
        uint32_t io_ph = 0;
        // (TMA) the warp's 32 x 32 box of matrix mm into its tile; lane 0 issues
        auto tile_load = [&](uint32_t tile, long long mm) {
            if (lane == 0) {
                mbar_expect_tx(io_bar + warp, 4096);
                tma_load_2d_s(tile, &in_map, io_bar + warp, static_cast<int32_t>(col0),
                              static_cast<int32_t>(mm * 128 + q * 32));
            }
        };
        auto emit_input_tiled = [&](uint32_t cc) {
            const uint32_t tile = s0 + cc * kChainSmem + tile_off;
            float x[32];
            mbar_wait_sleep(io_bar + warp, io_ph);
            io_ph ^= 1;
            K3B_MARK(3);
            tile_get_rows(tile, lane, x);
            named_bar_sync(3, kWorkers * 32);  // every tile read before planes overwrite them
            K3B_MARK(4);
            emit(cc, 0, x, true, true);
            emit(cc, 1, x + 16, true, true);
            K3B_MARK(5);
        };

        while (act_c || act_o) {
            if (act_c && dly_c > 0) {
                --dly_c;
            } else if (act_c) {
                bool publish = true;
                if (s_c < 0) {
                    if (vec) {
                        tile_load(s0 + c * kChainSmem + tile_off, m_c);
                        emit_input_tiled(c);
                    } else {
                        emit_input(c, true, true);
                    }
                    s_c = 0;
                } else {
                    K3B_MARK(7);
                    mbar_wait_sleep(mma_bar + c, ph_c);
                    K3B_MARK(0);
                    ph_c ^= 1;
                    tc_fence_after();
                    uint32_t v[32];
#if defined(K3B_X_NOTMEM) || defined(K3B_X_NOEPI)
                    for (int i = 0; i < 32; ++i) v[i] = row + i;
#else
                    tmem_ld32(lane_base + c * 256u + col0, v);
#endif
                    K3B_MARK(1);
                    if (s_c == last) {
                        const long long m_prev = m_c;
                        m_c += 2 * G;
                        act_c = m_c < batch;
                        if (vec) {
                            // result -> the warp's tile -> TMA store; once the store
                            // has read the tile, TMA loads the next input into it
                            const uint32_t tile = s0 + c * kChainSmem + tile_off;
                            tile_put_rows(tile, lane, v);
                            fence_proxy_async_smem();
                            __syncwarp();
                            if (lane == 0) {
                                tma_store_2d_s(&out_map, tile, static_cast<int32_t>(col0),
                                               static_cast<int32_t>(m_prev * 128 + q * 32));
                                bulk_commit_group();
                                bulk_wait_group_read0();
                            }
                            __syncwarp();
                            K3B_MARK(2);
                            K3B_COUNT(11);
                            if (act_c) {  // (prefetched into L2 one matrix ahead)
                                tile_load(tile, m_c);
                                emit_input_tiled(c);
                            }
                        } else {
                            store_row(out + static_cast<size_t>(m_prev) * n2, n, vec, row, col0, v);
                            if (act_c) emit_input(c, true, true);
                        }
                        if (act_c) s_c = 0;
                        else publish = false;
                    } else {
                        s_c += 1;
                        const bool mult = plan_is_mult(plan, s_c);
                        emit(c, 0, reinterpret_cast<const float*>(v), true, !mult);
                        emit(c, 1, reinterpret_cast<const float*>(v) + 16, true, !mult);
                        K3B_MARK(6);
                        K3B_COUNT(12);
                        if (mult) {  // left operand = the base: x0, x1 to TMEM, x2 to S
                            if (s_uses > 0) mbar_wait_sleep(s_free, (s_uses - 1) & 1u);
                            emit_input(c, false, true);
                            ++s_uses;
                        }
                    }
                }
                if (publish) {
                    tmem_st_wait();
                    fence_proxy_async_smem();
                    tc_fence_before();
                    named_bar_arrive(1 + c, kThreads);
                }
            }
            swap_chains();
            const uint32_t tp = ph_c;
            ph_c = ph_o;
            ph_o = tp;
        }
    }
    if (vec && warp < kWorkers && lane == 0) bulk_wait_group0();  // output stores done
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
                               const PlanBits& plan, int grid, cudaStream_t s) {
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
    k3b_batched_power<<<grid, kThreads, kSmem, s>>>(in_map, out_map, in, out, n, batch, plan, vec);
    return cudaGetLastError();
}

}  // namespace mxp
