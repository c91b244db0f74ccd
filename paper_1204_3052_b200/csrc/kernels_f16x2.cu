// K1PH — the large-n FP32 chain on the 16-bit tensor datapath (sm_100a).
//
// The same split-FP32 idea K3H uses for n <= 128, at CTA-pair GEMM scale
// (C5: 8192^2 A^1024).  Every power P of the chain is held as two fp16
// planes with ONE power-of-two exponent for the whole matrix:
//   P = 2^-t P',  max|P'| in [2^13, 2^14),  h0 = rn_fp16(P'),  h1 = rn_fp16(P' - h0)
// (P' - h0 is exact in fp32; |P' - h0 - h1| <= 2^-22 |P'| while h1 is a
// normal fp16, the operand precision of tf32 hi/lo), and a product is
//   X Y = 2^-(tx + ty) (x1 y0 + x0 y1 + x0 y0)       (x1 y1 ~ 2^-22 dropped)
// — three kind::f16 MMAs per K=16 where 3xTF32 needs three kind::tf32 MMAs
// per K=8: half the tensor work, half the operand bytes.  The reference's
// product is the ascending-k fp32 loop (linalg.py:151-164); parity is by the
// relative-Frobenius tolerance.
//
// One exponent per matrix loses entries more than ~2^38 below the matrix max
// (h1 underflows first, below ~2^-17 of the max).  As in K3H, the tell-tale is
// a product that came out more than 2^12 below its bound n max|X| max|Y|
// (strong cancellation), or a zero / non-finite product: the split of that
// product raises the chain's flag, and the 3xTF32 chain (an exponent per
// element), enqueued behind this one with every launch gated on the flag,
// recomputes the whole power.  Random inputs never raise it.
//
// Per step: k1ph_gemm_f16x2 (persistent CTA pairs, M = N = 256, K = 64 per
// stage, the accumulator drained per stage into fp32 register sums as in
// K1P) writes the unscaled fp32 product and its max |.| (atomicMax on the bit
// patterns); split16_kernel turns it into the next step's planes at the
// exact scale of that max.
#include <cuda_fp16.h>

#include <cmath>

#include "mxp_internal.h"
#include "ptx.cuh"
#include "split16.cuh"

namespace mxp {
namespace {

__device__ __forceinline__ uint8_t* align1024h(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023u) & ~uintptr_t(1023));
}

struct K1HCfg {
    static constexpr int kStages = 3;
    static constexpr int kBK = 64;                               // fp16 K per stage (128 B rows)
    static constexpr uint32_t kABytes = 128u * 128u;             // one plane: 128 rows x 64 fp16
    static constexpr uint32_t kBBytes = 64u * 128u * 2u;         // one plane: 2 panels x 64 k-rows x 128 B
    static constexpr uint32_t kStageBytes = 2 * kABytes + 2 * kBBytes;  // 64 KB per CTA
    static constexpr size_t kSmem = kStages * kStageBytes + 1024 + 256;
    static constexpr int kThreads = 384;
#ifndef MXP_K1PH_CHUNK_STAGES
#define MXP_K1PH_CHUNK_STAGES 1
#endif
    // stages accumulated in one TMEM chunk before the drain (bias control)
    static constexpr int kChunkStages = MXP_K1PH_CHUNK_STAGES;
};

// kind::f16, fp16 A/B (formats 0), fp32 D, A K-major, B MN-major, M = N = 256 (pair)
constexpr uint32_t kIdescPair = (1u << 4) | (1u << 16) | ((256u >> 3) << 17) | ((256u >> 4) << 24);

__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 2^-(tx + ty) as two factors (each in the normal range)
__device__ __forceinline__ void product_scale(uint32_t xmax, uint32_t ymax, float& g1, float& g2) {
    const int pe = -(scale_exp(xmax) + scale_exp(ymax));
    g1 = exp2i(pe / 2);
    g2 = exp2i(pe - pe / 2);
}

}  // namespace

// Per-chain state (device memory, zeroed before the chain): index 0 is the
// base A, index s + 1 the product of plan step s.
//   maxw[i]  max |P_i| (fp32 bit pattern, atomicMax by the producing GEMM)
//   texp[i]  the planes of P_i hold P_i * 2^texp[i] (set by its split)
//   flag     a product lost dynamic range (-> the gated 3xTF32 recomputation)
struct F16Chain {
    uint32_t maxw[kF16MaxSteps + 1];
    int texp[kF16MaxSteps + 1];
    int flag;
};

// C = X Y over scaled fp16 planes, persistent: one CTA pair per two SMs
// walks the 256 x 256 tiles (grouped raster), so a tile's epilogue overlaps
// the next tile's first MMAs (the two 256-column chunk accumulators run
// ahead of the drain).
//   warp 0 : TMA producer (both CTAs; bytes complete on the leader's barrier)
//   warp 1 : MMA issuer (leader only)     warp 2 : TMEM allocator (both)
//   warps 4-11 : epilogue (both CTAs; lane quarter = warp % 4, 128-column half)
// out (fp32, leading dim ld_out; entries of global row >= n_out or column >=
// n_out are not written) = 2^-(texp[xi] + texp[yi]) * sums; oi >= 0: max |out| -> maxw[oi] (atomicMax of the bit patterns), which
// the split of the next planes turns into their exact scale.
//
// (Measured and rejected, DESIGN.md §3 K1PH: writing the next planes straight
// from the epilogue at a bound scale instead of this split pass — at the
// bound n max|X| max|Y| a signed permutation power with 2^13 of dynamic range
// lost its exactness at n = 1024; at the tighter row-norm bound it stayed
// exact but ran no faster than the split under the board's power cap.)
__global__ void __launch_bounds__(K1HCfg::kThreads, 1)
    k1ph_gemm_f16x2(const __grid_constant__ CUtensorMap ma0, const __grid_constant__ CUtensorMap ma1,
                    const __grid_constant__ CUtensorMap mb0, const __grid_constant__ CUtensorMap mb1,
                    int n_pad, int m_rows, int row0, float* __restrict__ out, int n_out,
                    int ld_out, F16Chain* __restrict__ st, int xi, int yi, int oi) {
    using Cfg = K1HCfg;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024h(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* cfull = empty + S;   // [2] chunk accumulator ready (multicast by the leader)
    uint64_t* cempty = cfull + 2;  // [2] chunk drained (leader's copy counts both CTAs)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank() & 1;  // half of the pair (A rows, B columns)
    const bool leader = (rank == 0);

    // grouped tile raster (as K1P); pair p takes tiles p, p + P, p + 2P, ...
    constexpr int kGroupM = 8;
    // row block [row0, row0 + m_rows) of the product (the whole matrix:
    // m_rows = n_pad, row0 = 0); out row r holds global row row0 + r
    const int num_m = m_rows / 256, num_n = n_pad / 256;
    const int num_tiles = num_m * num_n;
    const int per_group = kGroupM * num_n;
    const int num_kb = n_pad / Cfg::kBK;
    const int pairs = gridDim.x / 2;
    auto tile_origin = [&](int tile, int& m0, int& n0) {
        const int first_m = (tile / per_group) * kGroupM;
        const int gm = min(num_m - first_m, kGroupM);
        m0 = (first_m + (tile % per_group) % gm) * 256 + static_cast<int>(rank) * 128;
        n0 = ((tile % per_group) / gm) * 256;
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&cfull[i], 1);
            mbar_init(&cempty[i], 16);  // 8 epilogue warps x 2 CTAs
        }
        fence_mbar_init();
        tma_prefetch(&ma0);
        tma_prefetch(&ma1);
        tma_prefetch(&mb0);
        tma_prefetch(&mb1);
    }
    if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA traffic
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        uint32_t g = 0;  // k-blocks issued by this CTA over all its tiles
        for (int tile = blockIdx.x / 2; tile < num_tiles; tile += pairs) {
            int m0, n0;
            tile_origin(tile, m0, n0);
            const int nb = n0 + static_cast<int>(rank) * 128;
            for (int kb = 0; kb < num_kb; ++kb, ++g) {
                const uint32_t stg = g % S;
                const uint32_t ph = (g / S) & 1;
                mbar_wait(&empty[stg], ph ^ 1);
                uint8_t* base = smem + stg * Cfg::kStageBytes;
                if (leader) mbar_expect_tx(&full[stg], 2 * Cfg::kStageBytes);
                const int kk = kb * Cfg::kBK;
                tma_load_2d_pair(base, &ma0, &full[stg], kk, row0 + m0);
                tma_load_2d_pair(base + Cfg::kABytes, &ma1, &full[stg], kk, row0 + m0);
                uint8_t* b0 = base + 2 * Cfg::kABytes;
                uint8_t* b1 = b0 + Cfg::kBBytes;
#pragma unroll
                for (int j = 0; j < 2; ++j) {  // two 64-column panels of this CTA's 128 columns
                    tma_load_2d_pair(b0 + j * 8192, &mb0, &full[stg], nb + 64 * j, kk);
                    tma_load_2d_pair(b1 + j * 8192, &mb1, &full[stg], nb + 64 * j, kk);
                }
            }
        }
    } else if (warp == 1 && lane == 0 && leader) {
        const uint32_t s0 = smem_u32(smem);
        const uint64_t da0 = kmajor_desc(s0), da1 = kmajor_desc(s0 + Cfg::kABytes);
        // MN-major SW128: 64-column panels 8 KB apart (LBO), 8 k-rows per 1 KB atom (SBO)
        const uint64_t db0 = smem_desc(s0 + 2 * Cfg::kABytes, 8192, 1024, 2);
        const uint64_t db1 = smem_desc(s0 + 2 * Cfg::kABytes + Cfg::kBBytes, 8192, 1024, 2);
        uint32_t g = 0;
        for (int tile = blockIdx.x / 2; tile < num_tiles; tile += pairs) {
            for (int kb = 0; kb < num_kb; ++kb, ++g) {
                const uint32_t stg = g % S;
                const uint32_t ph = (g / S) & 1;
                constexpr uint32_t CS = Cfg::kChunkStages;
                const uint32_t hc = g / CS;  // chunk counter
                const uint32_t c = hc & 1;
                const bool first = (g % CS) == 0, lastc = (g % CS) == CS - 1;
                if (first) mbar_wait(&cempty[c], ((hc >> 1) & 1) ^ 1);
                mbar_wait(&full[stg], ph);
                tc_fence_after();
                const uint64_t so = static_cast<uint64_t>((stg * Cfg::kStageBytes) >> 4);
                const uint32_t d = tmem + c * 256;
                // small cross terms first (the accumulator truncates), then x0 y0
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t ao = so + ((32 * k) >> 4), bo = so + ((2048 * k) >> 4);
                    mma_f16_pair(d, da1 + ao, db0 + bo, kIdescPair, (k > 0 || !first) ? 1u : 0u);
                    mma_f16_pair(d, da0 + ao, db1 + bo, kIdescPair, 1u);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t ao = so + ((32 * k) >> 4), bo = so + ((2048 * k) >> 4);
                    mma_f16_pair(d, da0 + ao, db0 + bo, kIdescPair, 1u);
                }
                mma_commit_pair(&empty[stg], 0x3);
                if (lastc) mma_commit_pair(&cfull[c], 0x3);
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        const int ch = ((warp - 4) >> 2) * 128;  // column half of the 256
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        const uint32_t cempty_leader0 = mapa_shared(smem_u32(&cempty[0]), 0);
        const int pe = -(st->texp[xi] + st->texp[yi]);  // P = 2^pe sums
        const float g1 = exp2i(pe / 2), g2 = exp2i(pe - pe / 2);
        uint32_t g = 0;
        for (int tile = blockIdx.x / 2; tile < num_tiles; tile += pairs) {
            int m0, n0;
            tile_origin(tile, m0, n0);
            float sum[128];
#pragma unroll
            for (int i = 0; i < 128; ++i) sum[i] = 0.f;
            for (int kb = 0; kb < num_kb; kb += Cfg::kChunkStages, ++g) {
                const uint32_t c = g & 1;  // (g counts chunks here)
                mbar_wait(&cfull[c], (g >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int gg = 0; gg < 8; ++gg) {
                    uint32_t v[16];
                    tmem_ld16(lane_base + c * 256 + ch + 16 * gg, v);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        sum[16 * gg + i] = __fadd_rn(sum[16 * gg + i], __uint_as_float(v[i]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster_relaxed(cempty_leader0 + 8 * c);
            }
            const int row = m0 + q * 32 + lane;  // local row of out
            uint32_t mbits = 0;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int col = n0 + ch + 32 * h;
                float* v = sum + 32 * h;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    v[i] = __fmul_rn(__fmul_rn(v[i], g1), g2);
                    mbits = max(mbits, __float_as_uint(v[i]) & 0x7FFFFFFFu);
                }
                if (row0 + row < n_out && col < n_out) {
                    float* d = out + static_cast<size_t>(row) * ld_out + col;
                    if ((ld_out & 3) == 0 && col + 32 <= n_out) {
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            reinterpret_cast<float4*>(d)[u] =
                                make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                    } else {
                        for (int i = 0; i < 32; ++i)
                            if (col + i < n_out) d[i] = v[i];
                    }
                }
            }
            if (oi >= 0) {
                mbits = __reduce_max_sync(0xFFFFFFFFu, mbits);
                if (lane == 0) atomicMax(&st->maxw[oi], mbits);
            }
        }
    }
    // both CTAs done with the pair's TMEM before the paired dealloc
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) tmem_dealloc_pair<512>(tmem);
}

namespace {

// max |x| over an n x n fp32 matrix (leading dim ld) -> atomicMax of the bits
__global__ void absmax_kernel(const float* __restrict__ in, int n, int ld, uint32_t* __restrict__ omax) {
    uint32_t m = 0;
    if ((ld & 3) == 0 && (n & 3) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
        const size_t quads = static_cast<size_t>(n) * n / 4;
        const int qpr = n / 4;  // quads per row
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < quads;
             i += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const size_t r = i / qpr, c = (i - r * qpr) * 4;
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(in + r * ld + c));
            m = max(max(m, w.x & 0x7FFFFFFFu), max(w.y & 0x7FFFFFFFu, max(w.z & 0x7FFFFFFFu, w.w & 0x7FFFFFFFu)));
        }
    } else {
        const size_t total = static_cast<size_t>(n) * n;
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
             i += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const size_t r = i / n, c = i - r * n;
            m = max(m, __float_as_uint(__ldg(in + r * ld + c)) & 0x7FFFFFFFu);
        }
    }
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(omax, m);
}

// fp32 P_i (n x n, leading dim ld) -> scaled fp16 planes h0, h1 (n_pad x
// n_pad, zero padded) at the exact scale of st->maxw[i] (block 0 records it
// in st->texp[i]).  A product (xi >= 0: P_i = P_xi P_yi) is also tested for
// lost dynamic range: zero, non-finite, or more than 2^12 below its bound
// n max|P_xi| max|P_yi| raises st->flag.
__global__ void split16_kernel(const float* __restrict__ in, int n, int ld,
                               __half* __restrict__ h0, __half* __restrict__ h1, int n_pad,
                               F16Chain* __restrict__ st, int i, int xi, int yi, int lg_n) {
    const uint32_t mb = st->maxw[i];
    const int t = max(-126, min(126, scale_exp(mb)));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->texp[i] = t;
        if (xi >= 0) {
            const uint32_t xb = st->maxw[xi], yb = st->maxw[yi];
            bool lost = mb == 0u || mb >= 0x7F800000u || xb >= 0x7F800000u || yb >= 0x7F800000u;
            if (!lost && xb != 0u && yb != 0u) {
                const int bound_e = (ilogb_bits(xb) + 1) + (ilogb_bits(yb) + 1) + lg_n;
                lost = ilogb_bits(mb) < bound_e - 12;
            }
            if (lost) st->flag = 1;
        } else if (mb >= 0x7F800000u) {
            // a non-finite base: the 3xTF32 recomputation gives the reference's
            // inf / NaN pattern (an inf split into fp16 halves becomes inf + NaN)
            st->flag = 1;
        }
    }
    const float sc = exp2i(t);
    const size_t groups = static_cast<size_t>(n_pad) * n_pad / 8;
    for (size_t g = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; g < groups;
         g += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t e = g * 8;
        const int r = static_cast<int>(e / n_pad);
        const int c = static_cast<int>(e - static_cast<size_t>(r) * n_pad);
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.f;
        if (r < n) {
            const float* p = in + static_cast<size_t>(r) * ld + c;
            if ((ld & 3) == 0 && c + 7 < n && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(p));
                const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
                v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
                v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (c + k < n) v[k] = __ldg(p + k);
            }
        }
        __align__(16) __half a0[8], a1[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float x = __fmul_rn(v[k], sc);
            a0[k] = __float2half_rn(x);
            a1[k] = __float2half_rn(__fsub_rn(x, __half2float(a0[k])));
        }
        reinterpret_cast<uint4*>(h0)[g] = *reinterpret_cast<const uint4*>(a0);
        reinterpret_cast<uint4*>(h1)[g] = *reinterpret_cast<const uint4*>(a1);
    }
}

// Row-sharded chains (mxp_power_multi): max |P_i| of this device's rows ->
// every device's maxw[i] (system-scope atomics over peer access), so each
// device then holds the global max.
struct PeerStates {
    F16Chain* st[kF16MaxPeers];
    int n;
};
__global__ void max_to_peers_kernel(const F16Chain* __restrict__ mine, int i, PeerStates ps) {
    const uint32_t v = mine->maxw[i];
    for (int p = 0; p < ps.n; ++p) atomicMax_system(&ps.st[p]->maxw[i], v);
}

// This device's fp32 rows of P_i (m_rows x n_pad, global rows row0 ..) ->
// the h0 / h1 rows of P_i in EVERY device's planes (peer stores), at the
// exact scale of the global max st->maxw[i]; texp[i] and the dynamic-range
// test as split16_kernel (every device derives the same values).
struct PeerPlanes {
    __half* h0[kF16MaxPeers];
    __half* h1[kF16MaxPeers];
    int n;
};
__global__ void split16_rows_peers_kernel(const float* __restrict__ in, int m_rows, int row0,
                                          int n_pad, F16Chain* __restrict__ st, int i, int xi,
                                          int yi, int lg_n, PeerPlanes pp) {
    const uint32_t mb = st->maxw[i];
    const int t = max(-126, min(126, scale_exp(mb)));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->texp[i] = t;
        const uint32_t xb = st->maxw[xi], yb = st->maxw[yi];
        bool lost = mb == 0u || mb >= 0x7F800000u || xb >= 0x7F800000u || yb >= 0x7F800000u;
        if (!lost && xb != 0u && yb != 0u) {
            const int bound_e = (ilogb_bits(xb) + 1) + (ilogb_bits(yb) + 1) + lg_n;
            lost = ilogb_bits(mb) < bound_e - 12;
        }
        if (lost) st->flag = 1;
    }
    const float sc = exp2i(t);
    const size_t groups = static_cast<size_t>(m_rows) * n_pad / 8;
    const size_t off = static_cast<size_t>(row0) * n_pad / 8;  // in 16-byte units
    for (size_t g = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; g < groups;
         g += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(in) + 2 * g);
        const float4 b = __ldg(reinterpret_cast<const float4*>(in) + 2 * g + 1);
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        __align__(16) __half a0[8], a1[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float x = __fmul_rn(v[k], sc);
            a0[k] = __float2half_rn(x);
            a1[k] = __float2half_rn(__fsub_rn(x, __half2float(a0[k])));
        }
        const uint4 w0 = *reinterpret_cast<const uint4*>(a0), w1 = *reinterpret_cast<const uint4*>(a1);
        for (int p = 0; p < pp.n; ++p) {
            reinterpret_cast<uint4*>(pp.h0[p])[off + g] = w0;
            reinterpret_cast<uint4*>(pp.h1[p])[off + g] = w1;
        }
    }
}

}  // namespace

cudaError_t prepare_f16x2_kernels() {
    return cudaFuncSetAttribute(k1ph_gemm_f16x2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(K1HCfg::kSmem));
}

bool k1ph_eligible(int64_t n_pad) { return n_pad % 256 == 0 && n_pad >= 1024; }

// fp16 plane map: box {64 columns (128 B), box_rows}, SWIZZLE_128B — the
// K-major left-operand box (128 rows) and the MN-major right-operand panel
// (64 k-rows) over the same row-major plane.
bool encode_plane16_map(CUtensorMap* map, const void* plane, int n_pad, int box_rows) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = nullptr;
    if (fn == nullptr) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        fn = reinterpret_cast<EncodeFn>(p);
    }
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(n_pad), static_cast<cuuint64_t>(n_pad)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(n_pad) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(plane), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t f16_chain_state_bytes() { return sizeof(F16Chain); }
int* f16_chain_flag(void* state) { return &static_cast<F16Chain*>(state)->flag; }

cudaError_t launch_k1ph_gemm(const F16Maps& x, const F16Maps& y, int n_pad, float* out, int n_out,
                             int ld_out, void* state, int xi, int yi, int oi, int num_sms,
                             cudaStream_t s, int m_rows, int row0) {
    if (m_rows <= 0) m_rows = n_pad;
    if (!k1ph_eligible(n_pad) || xi < 0 || yi < 0 || xi > kF16MaxSteps || yi > kF16MaxSteps ||
        oi > kF16MaxSteps || m_rows % 256 != 0 || row0 < 0 || row0 + m_rows > n_pad)
        return cudaErrorInvalidValue;
    const int tiles = (m_rows / 256) * (n_pad / 256);
    const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(K1HCfg::kThreads);
    cfg.dynamicSmemBytes = K1HCfg::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k1ph_gemm_f16x2, x.a0, x.a1, y.b0, y.b1, n_pad, m_rows, row0, out,
                              n_out, ld_out, static_cast<F16Chain*>(state), xi, yi, oi);
}

cudaError_t launch_split16(const float* in, int n, int ld, void* h0, void* h1, int n_pad,
                           void* state, int i, int xi, int yi, cudaStream_t s) {
    F16Chain* st = static_cast<F16Chain*>(state);
    int blocks;
    if (xi < 0) {  // the base: its max first
        const size_t total = static_cast<size_t>(n) * n;
        blocks = static_cast<int>((total / 4 + 255) / 256);
        if (blocks > 148 * 8) blocks = 148 * 8;
        if (blocks < 1) blocks = 1;
        absmax_kernel<<<blocks, 256, 0, s>>>(in, n, ld, &st->maxw[i]);
    }
    int lg_n = 0;
    while ((1ll << lg_n) < n) ++lg_n;
    const size_t groups = static_cast<size_t>(n_pad) * n_pad / 8;
    blocks = static_cast<int>((groups + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    split16_kernel<<<blocks, 256, 0, s>>>(in, n, ld, static_cast<__half*>(h0), static_cast<__half*>(h1),
                                          n_pad, st, i, xi, yi, lg_n);
    return cudaGetLastError();
}

cudaError_t launch_max_to_peers(const void* state, int i, void* const* peer_states, int npeers,
                                cudaStream_t s) {
    if (npeers < 1 || npeers > kF16MaxPeers || i < 0 || i > kF16MaxSteps) return cudaErrorInvalidValue;
    PeerStates ps{};
    for (int p = 0; p < npeers; ++p) ps.st[p] = static_cast<F16Chain*>(peer_states[p]);
    ps.n = npeers;
    max_to_peers_kernel<<<1, 1, 0, s>>>(static_cast<const F16Chain*>(state), i, ps);
    return cudaGetLastError();
}

cudaError_t launch_split16_rows_peers(const float* in, int m_rows, int row0, int n_pad, int n,
                                      void* state, int i, int xi, int yi, void* const* h0,
                                      void* const* h1, int npeers, cudaStream_t s) {
    if (npeers < 1 || npeers > kF16MaxPeers || n_pad % 8 != 0) return cudaErrorInvalidValue;
    PeerPlanes pp{};
    for (int p = 0; p < npeers; ++p) {
        pp.h0[p] = static_cast<__half*>(h0[p]);
        pp.h1[p] = static_cast<__half*>(h1[p]);
    }
    pp.n = npeers;
    int lg_n = 0;
    while ((1ll << lg_n) < n) ++lg_n;
    const size_t groups = static_cast<size_t>(m_rows) * n_pad / 8;
    int blocks = static_cast<int>((groups + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    split16_rows_peers_kernel<<<blocks, 256, 0, s>>>(in, m_rows, row0, n_pad,
                                                     static_cast<F16Chain*>(state), i, xi, yi, lg_n, pp);
    return cudaGetLastError();
}

}  // namespace mxp
