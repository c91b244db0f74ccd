// REJECTED EXPERIMENT (round 2, not built): see DESIGN.md §3 K1C.  C2 100.4 us vs
// 107.5 for K1C, but the scaled-fp16 planes lose entries far below the
// matrix max that a later product depends on (profiles/r02_cancellation_probe.txt).
// K1H — a whole FP32 chain A^k in ONE launch for 256 <= n_pad <= 768 (C2's
// 512^2 A^1000), with the operands as scaled fp16x2 planes (K3H's split)
// instead of K1C's tf32 hi/lo planes.
//
// Same grid and pipeline shape as K1C's 64-column variant (kernels_tf32.cu):
// 128 x 64 output tiles, split-K over a cluster of S CTAs reduced through
// DSMEM, a grid barrier per plan step.  What changes is the bytes per step:
// an fp16 plane is half a tf32 plane, and kind::f16 runs K = 16 per MMA where
// kind::tf32 runs K = 8, so each step streams half the operand bytes from L2
// into half the shared memory and issues half the MMAs — the mainloop of this
// latency-bound chain was L2/SMEM-bandwidth-bound.
//
// Scaling (as K3H): P = 2^e P', max|P'| kept near 2^13..2^14 so
// fp16 planes hold P' = h0 + h1 with 22 significant bits; X*Y = 2^(ex+ey) *
// (x1 y0 + x0 y1 + x0 y0), small terms first, each 64-deep k-block in its own
// TMEM chunk accumulator drained into fp32 registers with round-to-nearest
// adds (the tensor core truncates its accumulator on every MMA).  The scale
// of a product is chosen from the bound n max|X'| max|Y'| with the exact
// maxima one step late: every CTA folds max |D| of the values it writes into
// a global word (red.max) before the step's grid barrier.  If the product
// came out more than 2^12 below its bound (strong cancellation: the planes'
// low halves would go subnormal) every CTA re-splits the values it still
// holds in registers at the exact scale and the step pays one more grid
// barrier; otherwise the lag costs nothing.  All CTAs derive the same
// exponents from the same global words.
//
// MULTIPLY_BASE computes acc * base (accumulator on the left, expo.py:135-136).
#include <cstring>

#include "mxp_internal.h"
#include "ptx.cuh"
#include "split16.cuh"

namespace mxp {
namespace {

constexpr int kBN = 64;
constexpr int kKB = 64;  // k per pipeline stage: one 128-byte fp16 row
constexpr int kStages = 4;
constexpr uint32_t kAPlane = 128u * kKB * 2u;  // 16 KB: 128 rows x 64 k
constexpr uint32_t kBPlane = kKB * kBN * 2u;   // 8 KB: 64 k-rows x 64 n
constexpr uint32_t kStageBytes = 2 * kAPlane + 2 * kBPlane;  // 48 KB
constexpr size_t kSmem = kStages * kStageBytes + 1024 + 256;
constexpr int kThreads = 384;
constexpr uint32_t kUnits = kBN / 4;  // 16-byte units per partial row
// kind::f16, fp16 A/B (format 0), fp32 D, A K-major, B MN-major, M = 128, N = 64;
// the -h1 planes are read with the negate bits (A: bit 13, B: bit 14)
constexpr uint32_t kIdesc = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescNegA = kIdesc | (1u << 13);
constexpr uint32_t kIdescNegB = kIdesc | (1u << 14);
constexpr int kMaxItems = 3;  // reduce groups per thread: 128/S rows x 16 units over 384 threads

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023u) & ~uintptr_t(1023));
}

__device__ __forceinline__ void grid_sync(unsigned int* ctr, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= target) break;
            __nanosleep(64);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_max(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// max |x| over a float4 as non-negative float bits (orderable as uint); NaN skipped
__device__ __forceinline__ float absmax4(float4 a, float m) {
    return fmaxf(fmaxf(m, fmaxf(fabsf(a.x), fabsf(a.y))), fmaxf(fabsf(a.z), fabsf(a.w)));
}

// the exponents of the chain, identical in every CTA (derived from the
// shared maxima in the same order)
struct Scale {
    int e, eb;     // P = 2^e P', base = 2^eb base'
    int t_prev;    // scale applied to the last written planes (P'_s = 2^t_prev D_{s-1})
    int bmax_e;    // floor(log2 max|base'|)
};

}  // namespace

struct K1HMaps {
    CUtensorMap a[6];  // plane pairs 0 base, 1 ping, 2 pong: [2p] h0, [2p + 1] -h1; K-major view
    CUtensorMap b[6];  // the same planes as MN-major right operands
};
struct K1HPlanes {
    uint16_t* p[6];
};

__global__ void __launch_bounds__(kThreads, 1)
    k1h_chain_f16(const __grid_constant__ K1HMaps maps, const __grid_constant__ K1HPlanes pl,
                  PlanBits plan, const float* __restrict__ in, int n, int n_pad,
                  float* __restrict__ out_f32, uint32_t* __restrict__ ws, uint32_t* progress,
                  int fault_step) {
    // ws[0]: grid barrier counter; ws[32]: max|A|; ws[33 + s]: max|D_s| (unscaled)
    unsigned int* bar_ctr = ws;
    uint32_t* maxw = ws + 32;
    constexpr int S_ = kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S_ * kStageBytes);
    uint64_t* empty = full + S_;
    uint64_t* cfull = empty + S_;
    uint64_t* cempty = cfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    constexpr int kGroupM = 16;
    const int num_m = n_pad / 128, num_n = n_pad / kBN;
    const int pid = blockIdx.x;
    const int per_group = kGroupM * num_n;
    const int first_m = (pid / per_group) * kGroupM;
    const int gm = min(num_m - first_m, kGroupM);
    const int m0 = (first_m + (pid % per_group) % gm) * 128;
    const int n0 = ((pid % per_group) / gm) * kBN;
    const int splits = static_cast<int>(gridDim.y);
    const int kb_per = (n_pad / kKB) / splits;
    const int kb0 = static_cast<int>(blockIdx.y) * kb_per;
    const unsigned int nctas = gridDim.x * gridDim.y;
    unsigned int barriers = 0;
    const int lg_n = 32 - __clz(n_pad - 1);  // ceil(log2 n_pad)

    if (threadIdx.x == 0) {
        for (int i = 0; i < S_; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&cfull[i], 1);
            mbar_init(&cempty[i], 8);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<2 * kBN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t s0 = smem_u32(smem);

    // ---------------------------------------------------------------- input
    // A (n x n fp32, zero padded to n_pad) -> base planes at the exact scale
    // (max|A| was folded into maxw[0] by mod_prep / k1h_prep before this launch)
    Scale sc;
    {
        const uint32_t mA = ld_acquire(maxw);
        const int t0 = scale_exp(mA);
        sc.e = sc.eb = -t0;
        sc.t_prev = t0;
        sc.bmax_e = ilogb_bits(mA) + t0;
        const uint64_t s2 = splat2(exp2i(t0));
        const size_t quads = static_cast<size_t>(n_pad) * n_pad / 4;
        const size_t cta = static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x;
        for (size_t i = cta * kThreads + threadIdx.x; i < quads; i += static_cast<size_t>(nctas) * kThreads) {
            const size_t e = i * 4;
            const int r = static_cast<int>(e / n_pad), c = static_cast<int>(e % n_pad);
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (r < n) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c + k < n) v[k] = __ldg(in + static_cast<size_t>(r) * n + c + k);
            }
            uint32_t h[2], l[2];
            split2(v[0], v[1], s2, h[0], l[0]);
            split2(v[2], v[3], s2, h[1], l[1]);
            *reinterpret_cast<uint2*>(pl.p[0] + e) = make_uint2(h[0], h[1]);
            *reinterpret_cast<uint2*>(pl.p[1] + e) = make_uint2(l[0], l[1]);
        }
    }
    grid_sync(bar_ctr, nctas * ++barriers);

    int acc = 0;  // plane pair holding the running power: 0 base, 1 ping, 2 pong
    uint32_t mprev = 0;  // max|D_{s-1}| (unscaled), read after the previous barrier
    for (int step = 0; step < plan.len; ++step) {
        const bool mult = plan_is_mult(plan, step);
        const bool last = step == plan.len - 1;
        const int dst = (acc == 1) ? 2 : 1;
        const int rhs = mult ? 0 : acc;
        const int g0 = step * kb_per;  // pipeline position of this step's first k-block
        if (threadIdx.x == 0 && progress != nullptr) {
            *reinterpret_cast<volatile uint32_t*>(progress) = static_cast<uint32_t>(step + 1);
            if (step == fault_step && blockIdx.x == 0 && blockIdx.y == 0) {
                __threadfence_system();
                __trap();
            }
        }
        // this step's exponents: product D = X'Y', X' = P'_s, Y' = P'_s or base'
        const int pmax_e = step == 0 ? sc.bmax_e : ilogb_bits(mprev) + sc.t_prev;
        const int ymax_e = mult ? sc.bmax_e : pmax_e;
        const int pe = sc.e + (mult ? sc.eb : sc.e);  // P_{s+1} = 2^pe D
        const bool degenerate = step > 0 && (mprev == 0u || mprev >= 0x7F800000u);
        int t = kCeil - lg_n - (pmax_e + 1) - (ymax_e + 1);
        if (degenerate) t = 0;
        t = max(-126, min(126, t));

        if (warp == 0 && lane == 0) {
            // the planes this step reads were written by other CTAs' generic
            // stores before the grid barrier: order them before TMA (async proxy)
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const CUtensorMap* a0m = &maps.a[2 * acc];
            const CUtensorMap* a1m = &maps.a[2 * acc + 1];
            const CUtensorMap* b0m = &maps.b[2 * rhs];
            const CUtensorMap* b1m = &maps.b[2 * rhs + 1];
            for (int kb = 0; kb < kb_per; ++kb) {
                const int g = g0 + kb;
                const int st = g % S_;
                mbar_wait(&empty[st], ((g / S_) & 1) ^ 1);
                uint8_t* base = smem + st * kStageBytes;
                mbar_expect_tx(&full[st], kStageBytes);
                const int kg = (kb0 + kb) * kKB;
                tma_load_2d(base, a0m, &full[st], kg, m0);
                tma_load_2d(base + kAPlane, a1m, &full[st], kg, m0);
                tma_load_2d(base + 2 * kAPlane, b0m, &full[st], n0, kg);
                tma_load_2d(base + 2 * kAPlane + kBPlane, b1m, &full[st], n0, kg);
            }
        } else if (warp == 1 && lane == 0) {
            const uint64_t da0 = smem_desc(s0, 16, 1024, 2);                   // x0 (h0), K-major
            const uint64_t da1 = smem_desc(s0 + kAPlane, 16, 1024, 2);         // x1 (-h1)
            const uint64_t db0 = smem_desc(s0 + 2 * kAPlane, 8192, 1024, 2);   // y0, MN-major
            const uint64_t db1 = smem_desc(s0 + 2 * kAPlane + kBPlane, 8192, 1024, 2);  // y1
            for (int kb = 0; kb < kb_per; ++kb) {
                const int g = g0 + kb;
                const int st = g % S_;
                const int c = g & 1;
                mbar_wait(&cempty[c], ((g >> 1) & 1) ^ 1);
                mbar_wait(&full[st], (g / S_) & 1);
                tc_fence_after();
                const uint64_t so = static_cast<uint64_t>((st * kStageBytes) >> 4);
                const uint32_t d = tmem + c * kBN;
                // small cross terms first (x1 y0, x0 y1), then x0 y0; K = 16 per
                // MMA: +32 B along A's rows, +16 rows (2048 B) of B
#pragma unroll
                for (int k = 0; k < kKB / 16; ++k) {
                    const uint64_t ao = so + ((32 * k) >> 4), bo = so + ((2048 * k) >> 4);
                    mma_f16_ss(d, da1 + ao, db0 + bo, kIdescNegA, k > 0 ? 1u : 0u);
                    mma_f16_ss(d, da0 + ao, db1 + bo, kIdescNegB, 1u);
                }
#pragma unroll
                for (int k = 0; k < kKB / 16; ++k) {
                    const uint64_t ao = so + ((32 * k) >> 4), bo = so + ((2048 * k) >> 4);
                    mma_f16_ss(d, da0 + ao, db0 + bo, kIdesc, 1u);
                }
                mma_commit(&empty[st]);
                mma_commit(&cfull[c]);
            }
        } else if (warp >= 4) {
            constexpr int kCols = kBN / 2;  // columns per epilogue warp
            const int q = warp & 3;
            const int ch = ((warp - 4) >> 2) * kCols;
            const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
            float sum[kCols];
#pragma unroll
            for (int i = 0; i < kCols; ++i) sum[i] = 0.f;
            for (int kb = 0; kb < kb_per; ++kb) {
                const int g = g0 + kb;
                const int c = g & 1;
                mbar_wait(&cfull[c], (g >> 1) & 1);
                tc_fence_after();
                uint32_t v[32];
                tmem_ld32(lane_base + c * kBN + ch, v);
#pragma unroll
                for (int i = 0; i < 32; ++i) sum[i] = __fadd_rn(sum[i], __uint_as_float(v[i]));
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_relaxed(&cempty[c]);
            }
            // partial -> SMEM (every MMA of the step has completed: stages free)
            const uint32_t rr = static_cast<uint32_t>(q * 32 + lane);
            const uint32_t base = s0 + rr * (kUnits * 16u);
#pragma unroll
            for (int u = 0; u < kCols / 4; ++u) {
                const uint32_t uu = static_cast<uint32_t>(ch / 4 + u);
                sts128(base + ((uu ^ (rr & 7u)) << 4), __float_as_uint(sum[4 * u]),
                       __float_as_uint(sum[4 * u + 1]), __float_as_uint(sum[4 * u + 2]),
                       __float_as_uint(sum[4 * u + 3]));
            }
        }
        tc_fence_before();
        __syncwarp();
        cluster_sync_all();  // every partial of the tile is in SMEM

        // ---- split-K reduction over the cluster: CTA r sums rows [r R, (r+1) R)
        // of the S partials in split order (round-to-nearest adds)
        const uint32_t R = 128u / static_cast<uint32_t>(splits);
        const uint32_t items = R * kUnits;
        const uint32_t rank = cluster_ctarank();
        float4 val[kMaxItems];
        // group it of this thread: row rank R + i / 16, 16-byte unit i % 16
        auto row_of = [&](int it) { return rank * R + (threadIdx.x + it * kThreads) / kUnits; };
        auto unit_of = [&](int it) { return (threadIdx.x + it * kThreads) % kUnits; };
        float m = 0.f;
#pragma unroll
        for (int it = 0; it < kMaxItems; ++it) {
            const uint32_t i = threadIdx.x + it * kThreads;
            if (i < items) {
                const uint32_t rr = row_of(it), uu = unit_of(it);
                const uint32_t la = s0 + rr * (kUnits * 16u) + ((uu ^ (rr & 7u)) << 4);
                float4 a = ld_dsmem_f4(mapa_shared(la, 0));
                for (int p = 1; p < splits; ++p) {
                    const float4 b = ld_dsmem_f4(mapa_shared(la, static_cast<uint32_t>(p)));
                    a.x = __fadd_rn(a.x, b.x);
                    a.y = __fadd_rn(a.y, b.y);
                    a.z = __fadd_rn(a.z, b.z);
                    a.w = __fadd_rn(a.w, b.w);
                }
                val[it] = a;
                m = absmax4(a, m);
            }
        }
        if (!last) {
            uint16_t* o0 = pl.p[2 * dst];
            uint16_t* o1 = pl.p[2 * dst + 1];
            auto store_planes = [&](int tt) {
                const uint64_t s2 = splat2(exp2i(tt));
#pragma unroll
                for (int it = 0; it < kMaxItems; ++it) {
                    if (threadIdx.x + it * kThreads < items) {
                        const size_t off =
                            static_cast<size_t>(m0 + row_of(it)) * n_pad + n0 + 4 * unit_of(it);
                        uint32_t h[2], l[2];
                        split2(val[it].x, val[it].y, s2, h[0], l[0]);
                        split2(val[it].z, val[it].w, s2, h[1], l[1]);
                        *reinterpret_cast<uint2*>(o0 + off) = make_uint2(h[0], h[1]);
                        *reinterpret_cast<uint2*>(o1 + off) = make_uint2(l[0], l[1]);
                    }
                }
            };
            // max |D| of this CTA's values -> the step's global word
            const uint32_t mw = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(m));
            if (lane == 0 && mw != 0u) red_max(maxw + step + 1, mw);
            store_planes(t);
            grid_sync(bar_ctr, nctas * ++barriers);
            mprev = ld_acquire(maxw + step + 1);
            if (mprev != 0u && mprev < 0x7F800000u && ilogb_bits(mprev) + t < kCeil - 12) {
                // strong cancellation: the product is far below its bound —
                // re-split at the exact scale (the same decision in every CTA)
                t = max(-126, min(126, scale_exp(mprev)));
                store_planes(t);
                grid_sync(bar_ctr, nctas * ++barriers);
            }
        } else {
            // 2^pe D in two exact-range multiplies
            const float g1 = exp2i(pe / 2), g2 = exp2i(pe - pe / 2);
#pragma unroll
            for (int it = 0; it < kMaxItems; ++it) {
                const int grow = m0 + static_cast<int>(row_of(it));
                const int col = n0 + 4 * static_cast<int>(unit_of(it));
                if (threadIdx.x + it * kThreads < items && grow < n) {
                    const float vv[4] = {val[it].x, val[it].y, val[it].z, val[it].w};
                    float* d = out_f32 + static_cast<size_t>(grow) * n;
                    for (int k = 0; k < 4; ++k)
                        if (col + k < n) d[col + k] = __fmul_rn(__fmul_rn(vv[k], g1), g2);
                }
            }
        }
        // the barrier also tells every CTA that its peers have finished reading
        // its SMEM partial (their reduce precedes their arrival)
        if (last) {
            cluster_sync_all();
        } else {
            sc.e = pe - t;
            sc.t_prev = t;
        }
        acc = dst;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc<2 * kBN>(tmem);
}

// max |A| over the n x n input, folded into ws[32] (ws zeroed before)
__global__ void k1h_prep(const float* __restrict__ in, size_t count, uint32_t* ws) {
    float m = 0.f;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        m = fmaxf(m, fabsf(__ldg(in + i)));
    const uint32_t mw = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(m));
    if ((threadIdx.x & 31) == 0 && mw != 0u) red_max(ws + 32, mw);
}

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (fn == nullptr) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}
bool encode_f16(CUtensorMap* m, const void* plane, int n_pad, bool right) {
    EncodeFn fn = encode_fn();
    if (fn == nullptr) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(n_pad), static_cast<cuuint64_t>(n_pad)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(n_pad) * 2};
    cuuint32_t box[2] = {64u, right ? static_cast<cuuint32_t>(kKB) : 128u};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(plane), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t prepare_k1h_kernel() {
    return cudaFuncSetAttribute(k1h_chain_f16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmem));
}

bool k1h_supported(int n_pad, int splits, bool narrow) {
#ifdef K1H_DISABLE
    return false;
#endif
    return narrow && (splits == 2 || splits == 4) && n_pad >= 256 && n_pad % 128 == 0 &&
           (n_pad / kKB) % splits == 0;
}

cudaError_t launch_k1h_chain(const float* in, int n, int n_pad, int splits, int tiles,
                             const PlanBits& plan, uint16_t* const* planes, float* out,
                             uint32_t* ws, uint32_t* progress, int fault_step, cudaStream_t s) {
#ifdef K1H_FORCE_SPLITS
    splits = K1H_FORCE_SPLITS;
#endif
    if (!k1h_supported(n_pad, splits, true) || plan.len < 1 || plan.len > 126)
        return cudaErrorNotSupported;
    K1HMaps maps;
    K1HPlanes pl;
    for (int i = 0; i < 6; ++i) {
        pl.p[i] = planes[i];
        if (!encode_f16(&maps.a[i], planes[i], n_pad, false) || !encode_f16(&maps.b[i], planes[i], n_pad, true))
            return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaMemsetAsync(ws, 0, 256 * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    k1h_prep<<<148, 256, 0, s>>>(in, static_cast<size_t>(n) * n, ws);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * tiles, splits);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = static_cast<unsigned>(splits);
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k1h_chain_f16, maps, pl, plan, in, n, n_pad, out, ws, progress,
                              fault_step);
}

}  // namespace mxp
