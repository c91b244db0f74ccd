// K3H — persistent batched A^k for n <= 128: two independent chains per SM,
// split-FP32 as two scaled fp16 planes (tcgen05 kind::f16, fp32 accumulate).
//
// A 128x128 chain step is a run of tensor-core MMAs followed by an epilogue
// (drain the accumulator, split, write the next operands).  One chain per SM
// serialises the two; two chains per SM overlap chain X's MMAs with chain Y's
// epilogue.  That needs two resident powers per SM, which the 3xTF32 operands
// of K3 (kernels_tf32.cu) cannot provide (128 KB SMEM + 256 TMEM columns each).
//
// Split (the fp16 analogue of 3xTF32, same 22-bit operand precision):
//   P = 2^e * P',  max|P'| in [2^13, 2^14)   (power-of-two scale: exact)
//   h0 = rn_fp16(x'),  h1 = rn_fp16(x' - h0)  (x' - h0 exact; |x' - h0 - h1| <= 2^-22 |x'|)
//   X * Y = 2^(ex + ey) * (x1*y0 + x0*y1 + x0*y0)   (dropped x1*y1 ~ 2^-22)
// fp16 shares tf32's 11-bit significand; the per-step scale replaces tf32's
// 8-bit exponent (each step rescales from the max |element| of its product,
// so powers that grow or shrink by orders of magnitude stay in range).  fp16
// MMAs run K=16 per 64 cycles where tf32 runs K=8: a 3-term split costs 24
// MMAs per 128^3 step instead of 48.
//
// One row-major 16-bit plane, stored as [c/64][r][128 B] with 16-byte units
// XOR-swizzled by r % 8, is a K-major SWIZZLE_128B left operand and an
// MN-major SWIZZLE_128B right operand at once (tools/bf16_probe.cu).
//
//   SMEM:  three 64 KB regions: each chain's home (y0, y1 planes of its
//          resident power P') and a spare (the next input, pre-loaded)
//   TMEM:  chain c at column 256c: D (fp32 accumulator, 128 columns),
//          x0, x1 left-operand planes (2 fp16 per column, 64 columns each)
//
// Per step of chain c one elected lane of the issue warp runs 24 MMAs
// (M=N=128, K=16, A from TMEM): x1*y0, x0*y1, then x0*y0 — small terms first
// because the tensor core truncates its fp32 accumulator on every MMA
// (DESIGN.md §3).  The 8 epilogue warps alternate between the chains.
//
// MULTIPLY_BASE computes base * acc (the base is the left operand), as K3
// does: equal to the reference's acc * base (expo.py:135-136) because acc is
// a power of the base.  Parity with the reference chain (linalg.py:151-164,
// expo.py:121-139) is by the relative-Frobenius tolerance of SURVEY §8(d).
#include <cstring>
#include <type_traits>

#include "mxp_internal.h"
#include "ptx.cuh"
#include "split16.cuh"

namespace mxp {
namespace {

constexpr int kWorkers = 8;                    // epilogue warps: 4 TMEM lane quarters x 2
constexpr int kIssueWarp = kWorkers + 1;       //   column halves, + one MMA-issue warp
constexpr int kIOWarp = kWorkers;              //   + one TMA IO warp
constexpr int kThreads = (kWorkers + 2) * 32;  // 320 (<= 168 registers per thread)
constexpr uint32_t kPlane = 128u * 128u * 2u;  // one fp16 plane: 32 KB
constexpr uint32_t kChainSmem = 2u * kPlane;   // y0, y1 of one chain
constexpr uint32_t kMaxOff = 3u * kChainSmem;  // after 3 regions: [chain][buffer][8] max slots
constexpr uint32_t kBarOff = kMaxOff + 256;    // mbarriers + TMEM slot
constexpr size_t kSmem = kBarOff + 128 + 1024; // + alignment slack
// kind::f16 with fp16 A/B (formats 0), fp32 D, A K-major, B MN-major, M = N = 128
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | (1u << 16) | ((128u >> 3) << 17) |
                            ((128u >> 4) << 24);
constexpr uint32_t kBStep = (16u * 128u) >> 4;  // right-operand descriptor advance per K=16
// the planes hold -h1 (split2): x1*y0 negates A, x0*y1 negates B
constexpr uint32_t kIdescNegA = kIdesc | (1u << 13);
constexpr uint32_t kIdescNegB = kIdesc | (1u << 14);

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023u) & ~uintptr_t(1023));
}

// 32 values of one row of an n x n fp32 matrix, zero padded to 128.
__device__ __forceinline__ void load_row(const float* __restrict__ src, int n, uint32_t row,
                                         uint32_t col0, float (&x)[32]) {
    if (n == 128 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
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
__device__ __forceinline__ void store_row(float* __restrict__ dst, int n, uint32_t row,
                                          uint32_t col0, const float* v) {
    if (row < static_cast<uint32_t>(n)) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (col0 + i < static_cast<uint32_t>(n))
                dst[static_cast<size_t>(row) * n + col0 + i] = v[i];
    }
}

// Global IO (n == 128) through a warp-private 4 KB SMEM tile: the warp's 32
// rows x 32 columns, row r at r * 128 B with its 16-byte units XOR r % 8 —
// the TMA SWIZZLE_128B box layout, and conflict-free for thread-per-row
// access (the TMEM lane layout).
__device__ __forceinline__ void tile_put_rows(uint32_t tile, uint32_t lane, const float* v) {
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u)
        sts128(tile + lane * 128u + ((u ^ (lane & 7u)) << 4), __float_as_uint(v[4 * u]),
               __float_as_uint(v[4 * u + 1]), __float_as_uint(v[4 * u + 2]),
               __float_as_uint(v[4 * u + 3]));
}
__device__ __forceinline__ void tile_get_rows(uint32_t tile, uint32_t lane, float (&x)[32]) {
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u) {
        const uint4 w = lds128(tile + lane * 128u + ((u ^ (lane & 7u)) << 4));
        x[4 * u] = __uint_as_float(w.x); x[4 * u + 1] = __uint_as_float(w.y);
        x[4 * u + 2] = __uint_as_float(w.z); x[4 * u + 3] = __uint_as_float(w.w);
    }
}

// One chain step: 24 MMAs into D of chain C; the whole issue warp calls it
// (the asm blocks elect one lane) so descriptors and TMEM addresses stay on
// the uniform datapath — the issue rate bounds the kernel.
template <uint32_t C>
__device__ __forceinline__ void k3h_issue(uint32_t tbase, uint32_t region, uint64_t* mma_bar) {
    const uint64_t y0 = smem_desc(region, 16384, 1024, 2);
    constexpr uint32_t D = C * 256u, X0 = D + 128u, X1 = D + 192u;
    constexpr uint32_t Y1 = kPlane >> 4;
    mma_f16_ts_x8<D, X1, 0, kBStep, true>(tbase, y0, kIdescNegA);  // x1*y0 (first: D =)
    mma_f16_ts_x8<D, X0, Y1, kBStep>(tbase, y0, kIdescNegB);                // x0*y1
    mma_f16_ts_x8<D, X0, 0, kBStep>(tbase, y0, kIdesc);                 // x0*y0
    mma_commit_warp(mma_bar + C);
}

}  // namespace

size_t k3h_smem_bytes() { return kSmem; }

#ifdef K3H_TRACE  // tools/k3h_trace.cu: per-phase cycle totals of CTA 0 (lane 0 of one
                  // epilogue warp, the issue warp and the IO warp)
#ifndef K3H_TRACE_WARP
#define K3H_TRACE_WARP 0
#endif
__device__ long long* g_k3h_trace;
__shared__ long long k3h_acc[16];
#define K3H_MARK(k)                                                                      \
    do {                                                                                 \
        if (blockIdx.x == 0 && (warp == K3H_TRACE_WARP || warp == kIssueWarp || warp == kIOWarp) && \
            lane == 0) {                                                                 \
            const long long t_ = clock64();                                              \
            k3h_acc[k] += t_ - k3h_tprev;                                                \
            k3h_tprev = t_;                                                              \
        }                                                                                \
    } while (0)
#define K3H_COUNT(k)                                                                     \
    do {                                                                                 \
        if (blockIdx.x == 0 && warp == K3H_TRACE_WARP && lane == 0) k3h_acc[k] += 1;                  \
    } while (0)
#elif defined(K3H_EVT)
__device__ long long* g_k3h_evt;  // [role slot][8] stamps of CTA 0
#define K3H_MARK(k) \
    do {            \
    } while (0)
#define K3H_COUNT(k) \
    do {             \
    } while (0)
#define K3H_EV(slot, k)                                                        \
    do {                                                                       \
        if (blockIdx.x == 0 && lane == 0 && (slot) < 4096) evt[(slot) * 8 + (k)] = clock64(); \
    } while (0)
#else
#define K3H_MARK(k) \
    do {            \
    } while (0)
#define K3H_COUNT(k) \
    do {             \
    } while (0)
#endif

// Per-chain state of one role.  Two named instances, and the slot code is
// instantiated per chain (template parameter), so nothing is swapped or
// indexed at run time.
struct Chain {
    long long m;    // current matrix
    int s;          // step whose MMAs are in flight, or kIn
    int dly;        // start-phase skew slots still to sit out
    uint32_t ph;    // mbarrier parity (mma_bar for the epilogue, out_ready for IO)
    uint32_t inph;  // in_ready parity (epilogue)
    int e, eb;      // P = 2^e P', base = 2^eb base' (epilogue)
    int t_prev;     // scale exponent applied at this chain's previous epilogue
    int bmax_e;     // floor(log2 max |base'|)
    uint32_t sb;    // max-slot buffer the next epilogue reads (0/1)
    uint32_t mph;   // max_bar parities, bit b for buffer b; bit 31: a step of the
                    // current matrix lost range (listed for K3B at its boundary)
    uint32_t home;  // SMEM region (0..2) holding the chain's operand planes
    bool act;
};
constexpr uint32_t kLost = 1u << 31;  // Chain::mph: range lost in this matrix
constexpr int kIn = -2;  // Chain::s: the next input is being loaded / converted

// Matrices of CTA b are b, b + G, b + 2G, ... (G = gridDim.x); chain c takes
// every other one starting at b + cG.  Three roles run the same deterministic
// (chain, matrix, step) state machine, so they agree on every hand-off
// without exchanging state:
//   warps 0-7   epilogue: drain D, rescale, split, write the next operands
//               (a thread owns one row x 64 columns: 8 warps with 168
//               registers each beat 16 with 96 — the per-step control and
//               synchronisation cost is paid once per 64 values, not 32);
//   warp 8      IO: TMA stores of finished results and TMA loads of the next
//               inputs (n == 128), L2 prefetch one matrix ahead;
//   warp 9      MMA issue (one elected lane).
// SMEM holds three 64 KB regions: each chain's operand planes (its home) and
// a spare that the IO warp fills, ahead of time, with the next input of
// whichever chain reaches a matrix boundary next.  A boundary is one slot:
// the last product goes out through the old home (fp32 tiles, TMA store),
// the next input is converted in place in the spare, which becomes the new
// home, and step 0 is published — the chain's MMAs resume one slot later,
// never waiting for HBM.
// kMults: the plan has MULTIPLY_BASE steps.  Square-only plans (k a power
// of two) run the kMults = false instance, which drops every base-operand
// path from the epilogue.
template <bool kMults>
__global__ void __launch_bounds__(kThreads, 1)
    k3h_batched_power(const __grid_constant__ CUtensorMap in_map,
                      const __grid_constant__ CUtensorMap out_map, const float* __restrict__ in,
                      float* __restrict__ out, int n, long long batch, PlanBits plan, int vec,
                      unsigned long long* stamps, int* __restrict__ fix_idx,
                      int* __restrict__ fix_count) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint64_t* mma_bar = bars;        // [2] a chain's step MMAs completed
    uint64_t* out_ready = bars + 2;  // [2] a chain's result is in its old home (8 arrivals)
    uint64_t* in_ready = bars + 4;   // [3] an input landed in region r (TMA)
    uint64_t* max_bar = bars + 7;    // [chain][buffer] the 8 per-warp maxima are written
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        mbar_init(mma_bar, 1);
        mbar_init(mma_bar + 1, 1);
        mbar_init(out_ready, kWorkers);
        mbar_init(out_ready + 1, kWorkers);
        for (int i = 0; i < 3; ++i) mbar_init(in_ready + i, 1);
        for (int i = 0; i < 4; ++i) mbar_init(max_bar + i, kWorkers);
        fence_mbar_init();
    }
    if (warp == kIssueWarp) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t s0 = smem_u32(smem);
    const long long G = gridDim.x;
    if (fix_count != nullptr && gridDim.x == 1 && tid == 0) *fix_count = 0;  // (one CTA: no race)
    // let the K3B fixup pass (a programmatic dependent) launch now: it only
    // waits for this grid's completion (griddepcontrol.wait), so its launch
    // latency hides under this kernel instead of adding to a short chain
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (stamps != nullptr && blockIdx.x == 0 && tid == 0) {
        stamps[0] = clock64();
        stamps[1] = globaltimer_ns();
    }
    const size_t n2 = static_cast<size_t>(n) * n;
    const int last = plan.len - 1;
    auto is_mult = [&](int step) { return kMults && plan_is_mult(plan, step); };

    Chain ch0{}, ch1{};
    ch0.m = blockIdx.x;
    ch1.m = static_cast<long long>(blockIdx.x) + G;
    ch0.s = ch1.s = kIn;
    ch0.act = ch0.m < batch;
    ch1.act = ch1.m < batch;
    ch0.home = 0;
    ch1.home = 1;
    uint32_t spare = 2;  // every role tracks the region rotation identically
    // Start-phase skew: chain c of CTA b sits out its first dly slots, so the
    // CTAs' matrix boundaries are spread over the plan (HBM bursts), and the
    // two chains of a CTA are half a plan apart (the spare is refilled
    // between their boundaries).
    if (batch >= 4 * G && plan.len > 1) {
        ch0.dly = (2 * static_cast<int>(blockIdx.x)) % plan.len;
        ch1.dly = ch0.dly + plan.len / 2;
    }
    auto has_next = [&](const Chain& st) { return st.m + 2 * G < batch; };
#ifdef K3H_TRACE
    if (tid < 16) k3h_acc[tid] = 0;
    __syncthreads();
    long long k3h_tprev = clock64();
#endif
#ifdef K3H_EVT
    long long* evt = g_k3h_evt;
    int evs = 0;  // this role's slot counter
#else
#define K3H_EV(slot, k) \
    do {                \
    } while (0)
#endif
    // the 16 warp tiles of region rg <-> matrix mm (TMA boxes of 32 x 32)
    auto tiles_load = [&](uint32_t rg, long long mm) {
        mbar_expect_tx(in_ready + rg, 16 * 4096);
        for (uint32_t w = 0; w < 16; ++w)
            tma_load_2d_s(s0 + rg * kChainSmem + w * 4096u, &in_map, in_ready + rg,
                          static_cast<int32_t>((w >> 2) * 32),
                          static_cast<int32_t>(mm * 128 + (w & 3) * 32));
        if (mm + 2 * G < batch)
            prefetch_l2(in + static_cast<size_t>(mm + 2 * G) * n2, static_cast<uint32_t>(n2 * 4));
    };

    if (warp == kIssueWarp) {
        // ------------------------------------------------------------ MMA issue
        auto slot = [&](Chain& st, auto cc) {
            constexpr uint32_t C = decltype(cc)::value;
            if (!st.act) return;
            if (st.dly > 0) {
                --st.dly;
                return;
            }
            if (st.s == last) {  // boundary: step 0 of the next matrix, in the spare
                const bool more = has_next(st);
                st.m += 2 * G;
                st.act = more;
                if (!more) return;
                const uint32_t h = st.home;
                st.home = spare;
                spare = h;
                st.s = 0;
            } else {
                st.s = (st.s == kIn) ? 0 : st.s + 1;
            }
            K3H_MARK(10);
            K3H_EV(evs, 0);
            named_bar_sync(1 + C, kWorkers * 32 + 32);
            K3H_MARK(8);
            K3H_EV(evs, 1);
            tc_fence_after();
            k3h_issue<C>(tmem, s0 + st.home * kChainSmem, mma_bar);
            __syncwarp();
            K3H_EV(evs, 2);
#ifdef K3H_EVT
            ++evs;
#endif
            K3H_MARK(9);
        };
        while (ch0.act || ch1.act) {
            slot(ch0, std::integral_constant<uint32_t, 0>{});
            slot(ch1, std::integral_constant<uint32_t, 1>{});
        }
    } else if (warp == kIOWarp) {
        // ------------------------------------------------------------ IO (TMA)
        // Which chain reaches its next boundary first with a matrix after it,
        // and that matrix: replays the shared state machine from the slot
        // after chain `from`'s.
        auto next_boundary = [&](uint32_t from, long long& mm) -> int {
            Chain a = ch0, b = ch1;
            for (int it = 0; it < 4 * (plan.len + 2) + 8; ++it) {
                for (uint32_t k = 0; k < 2; ++k) {
                    const uint32_t c = (from + 1 + k) & 1u;
                    Chain& st = c == 0 ? a : b;
                    if (!st.act) continue;
                    if (st.dly > 0) {
                        --st.dly;
                        continue;
                    }
                    if (st.s == last) {
                        if (has_next(st)) {
                            mm = st.m + 2 * G;
                            return static_cast<int>(c);
                        }
                        st.act = false;
                        continue;
                    }
                    st.s = (st.s == kIn) ? 0 : st.s + 1;
                }
                if (!a.act && !b.act) break;
            }
            return -1;
        };
        if (vec && lane == 0) {
            if (ch0.act) tiles_load(ch0.home, ch0.m);
            if (ch1.act) tiles_load(ch1.home, ch1.m);
            long long mm = 0;
            if (next_boundary(1, mm) >= 0) tiles_load(spare, mm);
        }
        // Boundary of chain C: its result is in the old home once the
        // epilogue says so; store it, and when the store has read the region,
        // fill it (the new spare) with the input of the next boundary.
        auto slot = [&](Chain& st, auto cc) {
            constexpr uint32_t C = decltype(cc)::value;
            if (!st.act) return;
            if (st.dly > 0) {
                --st.dly;
                return;
            }
            if (st.s != last) {
                st.s = (st.s == kIn) ? 0 : st.s + 1;
                return;
            }
            const long long m_prev = st.m;
            const bool more = has_next(st);
            const uint32_t old_home = st.home;
            st.m += 2 * G;
            st.act = more;
            if (more) {
                st.home = spare;
                spare = old_home;
                st.s = 0;
            }
            if (!vec) return;
            mbar_wait_sleep(out_ready + C, st.ph);
            st.ph ^= 1;
            if (lane == 0) {
                for (uint32_t w = 0; w < 16; ++w)
                    tma_store_2d_s(&out_map, s0 + old_home * kChainSmem + w * 4096u,
                                   static_cast<int32_t>((w >> 2) * 32),
                                   static_cast<int32_t>(m_prev * 128 + (w & 3) * 32));
                bulk_commit_group();
                if (more) {
                    bulk_wait_group_read0();  // the old home is the new spare
                    long long mm = 0;
                    if (next_boundary(C, mm) >= 0) tiles_load(spare, mm);
                }
            }
            __syncwarp();
        };
        while (ch0.act || ch1.act) {
            slot(ch0, std::integral_constant<uint32_t, 0>{});
            slot(ch1, std::integral_constant<uint32_t, 1>{});
        }
        if (vec && lane == 0) bulk_wait_group0();  // results written before exit
    } else {
        // ------------------------------------------------------------ epilogue
        // 8 warps: 4 TMEM lane quarters x 2 column halves; a thread owns row
        // `row`, columns 64g .. 64g + 63 (four 16-column chunks)
        const uint32_t q = warp & 3, g = warp >> 2;
        const uint32_t row = q * 32 + lane;
        const uint32_t col0 = g * 64;
        const uint32_t lane_base = tmem + ((q * 32) << 16);
        // its two 32 x 32 IO tiles (TMA boxes 8g + q and 8g + 4 + q of a region)
        const uint32_t tile0 = (8u * g + q) * 4096u, tile1 = tile0 + 4u * 4096u;
        uint32_t rph = 0;   // in_ready parities, bit r for region r
        bool out_pending = false;  // a result in the old home awaits the IO warp

        const uint32_t lg_n = 32u - __clz(static_cast<int>(n - 1));  // ceil(log2 n), n >= 2
        // max of the 8 per-warp slots at `slots` (lane i < 8 reads slot i)
        auto max8 = [&](uint32_t slots) -> uint32_t {
            uint32_t v = 0;
            if (lane < kWorkers) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(slots + lane * 4u) : "memory");
            return __reduce_max_sync(0xFFFFFFFFu, v);
        };
        // max |x_i| (3-input FMNMX with |.| operands; a NaN is skipped, which is
        // harmless: it propagates through the products anyway)
        auto absmax64 = [](const float* x) {
            float m = 0.f;
#pragma unroll
            for (int i = 0; i < 64; i += 2) m = fmaxf(fmaxf(m, fabsf(x[i])), fabsf(x[i + 1]));
            return __float_as_uint(m);
        };
        // Per-warp maxima of a chain live in SMEM slots [cc][buffer][warp].
        // IN: exact max of the new input (one barrier among the epilogue
        // warps, which also orders every warp's tile reads before the plane
        // writes); the slots then hold max |A| for the first step's bound.
        auto block_max_in = [&](uint32_t cc, uint32_t buf, const float* x) -> uint32_t {
            const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, absmax64(x));
            const uint32_t slots = s0 + kMaxOff + cc * 64u + buf * 32u;
            if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(slots + warp * 4u), "r"(m) : "memory");
            named_bar_sync(3, kWorkers * 32);
            if (lane == 0) mbar_arrive(max_bar + cc * 2 + buf);  // uniform hand-off to the next step
            return max8(slots);
        };
        // max over the slots written at this chain's previous epilogue (the
        // mbarrier wait is the acquire that makes them visible)
        auto slots_max = [&](uint32_t cc, Chain& st) -> uint32_t {
            mbar_wait_sleep(max_bar + cc * 2 + st.sb, (st.mph >> st.sb) & 1u);
            st.mph ^= 1u << st.sb;
            return max8(s0 + kMaxOff + cc * 64u + st.sb * 32u);
        };
        // Dynamic range: the planes carry one exponent for the whole matrix,
        // so entries more than ~2^38 below its max are lost.  A product that
        // came out more than 2^12 below its bound (strong cancellation — the
        // same test that selects the exact scale path below) is the sign that
        // such entries may matter to a later product: the matrix goes on the
        // fixup list and K3B (an exponent per element) recomputes it after
        // this launch.  Random inputs never trigger it.  The steps only OR
        // the test into st.mph's kLost bit; the list append happens once, at the
        // matrix boundary (an atomic inside the per-step epilogue cost 4%).
        auto range_lost = [](int pmax_e, uint32_t mprev) {
            return pmax_e < kCeil - 12 || mprev == 0u || mprev >= 0x7F800000u;
        };
        // Plane addresses: row `row` of panel g, 16-byte unit u at
        // (u ^ (row & 7)) << 4.  Chunk k (units 2k, 2k+1): unit 2k + i sits at
        // pa_i ^ (k << 5); chain and plane are immediate offsets.
        const uint32_t pa0 = g * 16384u + row * 128u + ((row & 6u) << 4) + ((row & 1u) << 4);
        // chunk k (16 values, columns col0 + 16k ...), scaled by sc2 -> planes
        // y0/y1 in the region whose row base is ra = region + pa0 (right
        // operand) and, if `left`, x0/x1 of chain CC in TMEM
        auto emit_chunk = [&](auto cc, auto kk, uint32_t ra, const float* x, uint64_t sc2, bool left) {
            constexpr uint32_t CC = decltype(cc)::value, K = decltype(kk)::value;
            uint32_t p0[8], p1[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) split2(x[2 * j], x[2 * j + 1], sc2, p0[j], p1[j]);
            const uint32_t a0 = ra ^ (K << 5), a1 = (ra ^ 16u) ^ (K << 5);
            sts128_imm<0>(a0, p0[0], p0[1], p0[2], p0[3]);
            sts128_imm<0>(a1, p0[4], p0[5], p0[6], p0[7]);
            sts128_imm<kPlane>(a0, p1[0], p1[1], p1[2], p1[3]);
            sts128_imm<kPlane>(a1, p1[4], p1[5], p1[6], p1[7]);
            if (left) {
                const uint32_t tl = lane_base + CC * 256u + 128u + g * 32u + K * 8u;
                tmem_st8(tl, p0);
                tmem_st8(tl + 64u, p1);
            }
        };
        auto emit64 = [&](auto cc, uint32_t ra, const float* x, uint64_t sc2, bool left) {
            emit_chunk(cc, std::integral_constant<uint32_t, 0>{}, ra, x, sc2, left);
            emit_chunk(cc, std::integral_constant<uint32_t, 1>{}, ra, x + 16, sc2, left);
            emit_chunk(cc, std::integral_constant<uint32_t, 2>{}, ra, x + 32, sc2, left);
            emit_chunk(cc, std::integral_constant<uint32_t, 3>{}, ra, x + 48, sc2, left);
        };
        // the base of a MULTIPLY_BASE step: x0/x1 (TMEM) only
        auto emit_left = [&](uint32_t cc, const float* x, float sc) {
            const uint64_t sc2 = splat2(sc);
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                uint32_t p0[8], p1[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) split2(x[16 * k + 2 * j], x[16 * k + 2 * j + 1], sc2, p0[j], p1[j]);
                const uint32_t tl = lane_base + cc * 256u + 128u + g * 32u + k * 8u;
                tmem_st8(tl, p0);
                tmem_st8(tl + 64u, p1);
            }
        };
        auto load_row64 = [&](long long m, float (&x)[64]) {
            const float* src = in + static_cast<size_t>(m) * n2;
            load_row(src, n, row, col0, *reinterpret_cast<float(*)[32]>(x));
            load_row(src, n, row, col0 + 32u, *reinterpret_cast<float(*)[32]>(x + 32));
        };

        // a new matrix (in the chain's home region) -> exact scale, operands
        // of step 0
        auto convert_input = [&](auto cc, Chain& st) {
            constexpr uint32_t C = decltype(cc)::value;
            float x[64];
            const uint32_t rg = st.home;
            if (vec) {
                mbar_wait_sleep(in_ready + rg, (rph >> rg) & 1u);
                rph ^= 1u << rg;
                K3H_MARK(3);
                tile_get_rows(s0 + rg * kChainSmem + tile0, lane, *reinterpret_cast<float(*)[32]>(x));
                tile_get_rows(s0 + rg * kChainSmem + tile1, lane, *reinterpret_cast<float(*)[32]>(x + 32));
            } else {
                load_row64(st.m, x);
            }
            st.sb ^= 1u;  // (the other buffer: the current one was read at the boundary)
            st.mph &= ~kLost;
            const uint32_t mA = block_max_in(C, st.sb, x);  // (also orders tile reads before plane writes)
            const int t = scale_exp(mA);
            K3H_MARK(4);
            st.e = -t;
            st.eb = -t;
            st.t_prev = t;
            st.bmax_e = ilogb_bits(mA) + t;
            emit64(cc, s0 + rg * kChainSmem + pa0, x, splat2(exp2i(t)), true);
            K3H_MARK(5);
            K3H_COUNT(13);
            st.s = 0;
        };

        auto slot = [&](Chain& st, auto cc) {
            constexpr uint32_t C = decltype(cc)::value;
            if (!st.act) return;
            if (st.dly > 0) {
                --st.dly;
                return;
            }
            if (st.s == kIn) {
                // ---- the chain's first matrix, converted in its home region
                K3H_MARK(7);
                convert_input(cc, st);
            } else {
                K3H_MARK(7);
                mbar_wait_sleep(mma_bar + C, st.ph);
                K3H_MARK(0);
                if (warp == 2) K3H_EV(evs, 3);
                st.ph ^= 1;
                tc_fence_after();
                // exponent of this step's product: 2^(ex + ey) * D
                const int pe = (is_mult(st.s) ? st.eb : st.e) + st.e;
                if (st.s == last) {
                    // ---- boundary: 2^pe * D -> the old home's tiles (its planes
                    // are dead; the IO warp stores them), then the next input,
                    // already in the spare, -> step 0 there
                    {  // the last step's maxima: did the product feeding this one cancel?
                        const uint32_t mlast = slots_max(C, st);
                        const bool lost = (st.mph & kLost) || range_lost(ilogb_bits(mlast) + st.t_prev, mlast);
                        if (lost && fix_idx != nullptr && warp == 0 && lane == 0)
                            fix_idx[atomicAdd(fix_count, 1)] = static_cast<int>(st.m);
                    }
                    const uint64_t g1 = splat2(exp2i(pe / 2)), g2 = splat2(exp2i(pe - pe / 2));
                    const uint32_t old_region = s0 + st.home * kChainSmem;
#pragma unroll
                    for (uint32_t h = 0; h < 2; ++h) {
                        float v[32];
                        tmem_ld32(lane_base + C * 256u + col0 + 32u * h, reinterpret_cast<uint32_t(&)[32]>(v));
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {  // two exact-range steps, packed
                            uint64_t w;
                            asm("mov.b64 %0, {%1, %2};" : "=l"(w) : "f"(v[i]), "f"(v[i + 1]));
                            asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(w) : "l"(g1));
                            asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(w) : "l"(g2));
                            asm("mov.b64 {%0, %1}, %2;" : "=f"(v[i]), "=f"(v[i + 1]) : "l"(w));
                        }
                        if (vec) tile_put_rows(old_region + (h ? tile1 : tile0), lane, v);
                        else store_row(out + static_cast<size_t>(st.m) * n2, n, row, col0 + 32u * h, v);
                    }
                    const bool more = has_next(st);
                    st.m += 2 * G;
                    st.act = more;
                    if (!more) {  // the chain is done: hand the result over, nothing to publish
                        if (vec) fence_proxy_async_smem();
                        tc_fence_before();
                        __syncwarp();
                        if (vec && lane == 0) mbar_arrive(out_ready + C);
                        return;
                    }
                    const uint32_t h = st.home;
                    st.home = spare;
                    spare = h;
                    convert_input(cc, st);
                    // the result tiles are handed to the IO warp together with
                    // the publish below (one proxy fence for both)
                    out_pending = vec != 0;
                } else {
                // ---- step: D -> operands of the next step.  All four 16-column
                // TMEM loads are issued at once; the scale is settled under them.
                // Scale for the split, from a bound instead of a barrier:
                // |D| <= n max|X'| max|Y'|, with max|P'| known exactly one step
                // late (the previous epilogue's maxima).  The scaled max stays
                // < 2^14 (no fp16 overflow).  A product that cancels strongly
                // against its bound would land low in fp16's range and lose
                // bits of h1, so the exact path (block max, one barrier) runs
                // whenever the previous product came out more than 2^12 below
                // its bound (the input's exact max feeds the first step's bound).
                const uint32_t ra = s0 + st.home * kChainSmem + pa0;
                uint32_t d0[16], d1[16], d2[16], d3[16];
                tmem_ld16_async(lane_base + C * 256u + col0, d0);
                tmem_ld16_async(lane_base + C * 256u + col0 + 16u, d1);
                const bool was_mult = is_mult(st.s);
                const uint32_t mprev = slots_max(C, st);
                const int pmax_e = ilogb_bits(mprev) + st.t_prev;  // floor(log2 max|P'_s|)
                const bool exact = pmax_e < kCeil - 12;
                if (range_lost(pmax_e, mprev)) st.mph |= kLost;
                const int xmax_e = was_mult ? st.bmax_e : pmax_e;
                int t = kCeil - static_cast<int>(lg_n) - (xmax_e + 1) - (pmax_e + 1);
                if (mprev == 0u || mprev >= 0x7F800000u) t = 0;  // zero / non-finite operand
                st.s += 1;
                const bool mult = is_mult(st.s);
                const uint32_t nb = st.sb ^ 1u;  // this step's maxima -> slots [nb]
                const uint32_t slots = s0 + kMaxOff + C * 64u + nb * 32u;
                const float* f0 = reinterpret_cast<const float*>(d0);
                const float* f1 = reinterpret_cast<const float*>(d1);
                const float* f2 = reinterpret_cast<const float*>(d2);
                const float* f3 = reinterpret_cast<const float*>(d3);
                auto absmax32 = [](const float* x, const float* y, float m) {
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        m = fmaxf(fmaxf(m, fabsf(x[i])), fabsf(x[i + 1]));
                        m = fmaxf(fmaxf(m, fabsf(y[i])), fabsf(y[i + 1]));
                    }
                    return m;
                };
                // columns 0-31 land, columns 32-63 are loaded while they are split
                tmem_ld_wait_dep(d0);
                tmem_ld_wait_dep(d1);
                tmem_ld16_async(lane_base + C * 256u + col0 + 32u, d2);
                tmem_ld16_async(lane_base + C * 256u + col0 + 48u, d3);
                float m = absmax32(f0, f1, 0.f);
                K3H_MARK(1);
                if (!exact) {
                    t = max(-126, min(126, t));
                    const uint64_t sc2 = splat2(exp2i(t));
                    emit_chunk(cc, std::integral_constant<uint32_t, 0>{}, ra, f0, sc2, !mult);
                    emit_chunk(cc, std::integral_constant<uint32_t, 1>{}, ra, f1, sc2, !mult);
                    tmem_ld_wait_dep(d2);
                    tmem_ld_wait_dep(d3);
                    m = absmax32(f2, f3, m);
                    const uint32_t mw = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(m));
                    if (lane == 0) {
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(slots + warp * 4u), "r"(mw) : "memory");
                        mbar_arrive(max_bar + C * 2 + nb);
                    }
                    emit_chunk(cc, std::integral_constant<uint32_t, 2>{}, ra, f2, sc2, !mult);
                    emit_chunk(cc, std::integral_constant<uint32_t, 3>{}, ra, f3, sc2, !mult);
                } else {
                    tmem_ld_wait_dep(d2);
                    tmem_ld_wait_dep(d3);
                    m = absmax32(f2, f3, m);
                    const uint32_t mw = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(m));
                    if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(slots + warp * 4u), "r"(mw) : "memory");
                    named_bar_sync(3, kWorkers * 32);
                    if (lane == 0) mbar_arrive(max_bar + C * 2 + nb);
                    t = scale_exp(max8(slots));
                    const uint64_t sc2 = splat2(exp2i(t));
                    emit_chunk(cc, std::integral_constant<uint32_t, 0>{}, ra, f0, sc2, !mult);
                    emit_chunk(cc, std::integral_constant<uint32_t, 1>{}, ra, f1, sc2, !mult);
                    emit_chunk(cc, std::integral_constant<uint32_t, 2>{}, ra, f2, sc2, !mult);
                    emit_chunk(cc, std::integral_constant<uint32_t, 3>{}, ra, f3, sc2, !mult);
                }
                st.sb = nb;
                st.t_prev = t;
                st.e = pe - t;
                K3H_MARK(6);
                K3H_COUNT(14);
                if (mult) {  // left operand = the base, rescaled by its input exponent
                    float x[64];
                    load_row64(st.m, x);
                    emit_left(C, x, exp2i(-st.eb));
                }
                }
            }
            // workers arrive; the issue warp waits for all of them (the hardware
            // barrier also drains pending st.shared) and issues the step
            tmem_st_wait();
            fence_proxy_async_smem();
            tc_fence_before();
            if (out_pending) {
                __syncwarp();
                if (lane == 0) mbar_arrive(out_ready + C);
                out_pending = false;
            }
            if (warp == 2) K3H_EV(evs, 4);
            if (warp == 0) K3H_EV(evs, 5);
            if (warp == 7) K3H_EV(evs, 6);
#ifdef K3H_EVT
            ++evs;
#endif
            named_bar_arrive(1 + C, kWorkers * 32 + 32);
        };
        while (ch0.act || ch1.act) {
            slot(ch0, std::integral_constant<uint32_t, 0>{});
            slot(ch1, std::integral_constant<uint32_t, 1>{});
        }
    }
    tc_fence_before();
    __syncthreads();
    if (stamps != nullptr && blockIdx.x == 0 && tid == 0) {
        stamps[2] = clock64();
        stamps[3] = globaltimer_ns();
    }
#ifdef K3H_TRACE
    if (blockIdx.x == 0 && tid < 16) g_k3h_trace[tid] = k3h_acc[tid];
#endif
    if (warp == kIssueWarp) tmem_dealloc<512>(tmem);
}

cudaError_t prepare_k3h_kernel() {
    cudaError_t e = cudaFuncSetAttribute(k3h_batched_power<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmem));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k3h_batched_power<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmem));
    return e;
}

cudaError_t launch_k3h_batched(const float* in, float* out, int n, int64_t batch,
                               const PlanBits& plan, int grid, unsigned long long* stamps,
                               int* fix_idx, int* fix_count,
                               cudaStream_t s) {
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
    if (plan.mult[0] | plan.mult[1])
        k3h_batched_power<true><<<grid, kThreads, kSmem, s>>>(in_map, out_map, in, out, n, batch, plan, vec,
                                                               stamps, fix_idx, fix_count);
    else
        k3h_batched_power<false><<<grid, kThreads, kSmem, s>>>(in_map, out_map, in, out, n, batch, plan,
                                                                vec, stamps, fix_idx, fix_count);
    return cudaGetLastError();
}

}  // namespace mxp
