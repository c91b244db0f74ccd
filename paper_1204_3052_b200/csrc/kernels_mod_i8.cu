// K5I — exact modular product C = A*B mod p on the INT8 tensor cores
// (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM).  The fast datapath of the
// exact modular mode (no reference counterpart: the reference rejects integer
// dtypes, dtypes.py:37-42); bit-exact by construction, checked against the
// oracle's exact restatement (oracle/matexpo_oracle.c mxo_exponentiate_mod).
//
// Residues x < p < 2^31 are four byte limbs x = sum_a x_a 2^(8a).  Then
//   A*B = sum_s 2^(8s) D_s,   D_s = sum_{a+b=s} A_a B_b   (s = 0..6)
// and every D_s entry is an exact integer < 4 n 255^2 < 2^31 for n <= 8192, so
// the s32 accumulators never wrap.  A 128 x 64 output tile keeps its seven
// D_s accumulators in TMEM (7 x 64 = 448 columns) for the whole K loop; per
// 64-deep k-block (four pipeline stages of 48 KB) the issue thread runs the
// 16 limb pairs x 2 K=32 MMAs into them.  The epilogue folds the diagonals
// exactly in uint64,
//   lo = D0 + D1 2^8 + D2 2^16 + D3 2^24 < 2^56,  hi = D4 + D5 2^8 + D6 2^16,
//   C = (lo mod p + (hi mod p) (2^32 mod p)) mod p      (Barrett reductions)
// and writes the next step's byte planes (or the final uint32 matrix).
//
// Operands straight from the row-major byte planes: A K-major (TMA
// SWIZZLE_64B, 64 k per row), B MN-major (TMA SWIZZLE_64B, 64 n per k-row);
// operand layouts and the 49-cycle M128 N64 K32 rate measured with
// tools/i8_probe.cu (profiles/r02_i8_probe.txt; reading A from TMEM instead
// only gets it to 44.5 cycles).
#include <cstring>

#include "mxp_internal.h"
#include "ptx.cuh"

namespace mxp {
namespace {

constexpr int kStages = 4;
constexpr int kKB = 64;                     // k per pipeline stage
constexpr uint32_t kAPlane = 128u * kKB;    // 128 rows x 64 k (bytes), K-major SW64
constexpr uint32_t kBPlane = kKB * 64u;     // 64 k-rows x 64 n, MN-major SW64
constexpr uint32_t kStageBytes = 4u * kAPlane + 4u * kBPlane;  // 48 KB
constexpr size_t kSmem = kStages * kStageBytes + 1024 + 256;
constexpr int kThreads = 384;
constexpr int kBN = 64;
// kind::i8: [4,6) c_format = 2 (S32), [7,10) / [10,13) a/b_format = 0 (u8),
// [15] a_major = 0 (K), [16] b_major = 1 (MN), [17,23) N >> 3, [24,29) M >> 4
constexpr uint32_t kIdesc = (2u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023u) & ~uintptr_t(1023));
}

// One K=32 step of all 16 limb pairs (a, b) into the diagonal accumulators
// D_{a+b} (TMEM columns tmem + 64 (a+b)), in ONE asm block issued by an
// elected lane of the whole warp: descriptors and TMEM addresses are formed
// with immediate offsets on the uniform datapath, so the 49-cycle MMAs are
// issued back to back (per-MMA calls spent more cycles issuing than the
// tensor pipe spent executing).  kFirst: the first MMA into each diagonal
// overwrites it (the first K step of the tile).
template <bool kFirst>
__device__ __forceinline__ void mma_i8_x16(uint32_t tmem, uint64_t da, uint64_t db) {
    asm volatile(
        "{\n\t.reg .pred p, f, e;\n\t"
        ".reg .b32 d0, d1, d2, d3, d4, d5, d6;\n\t"
        ".reg .b64 a0, a1, a2, a3, b0, b1, b2, b3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.eq.u32 p, 1, 1;\n\t"
        "setp.eq.u32 f, %3, 0;\n\t"
        "mov.b32 d0, %0;\n\tadd.u32 d1, d0, 64;\n\tadd.u32 d2, d0, 128;\n\tadd.u32 d3, d0, 192;\n\t"
        "add.u32 d4, d0, 256;\n\tadd.u32 d5, d0, 320;\n\tadd.u32 d6, d0, 384;\n\t"
        "mov.b64 a0, %1;\n\tadd.s64 a1, a0, %4;\n\tadd.s64 a2, a1, %4;\n\tadd.s64 a3, a2, %4;\n\t"
        "mov.b64 b0, %2;\n\tadd.s64 b1, b0, %5;\n\tadd.s64 b2, b1, %5;\n\tadd.s64 b3, b2, %5;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d0], a0, b0, %6, f;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d1], a0, b1, %6, f;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d2], a0, b2, %6, f;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d3], a0, b3, %6, f;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d1], a1, b0, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d2], a1, b1, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d3], a1, b2, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d4], a1, b3, %6, f;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d2], a2, b0, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d3], a2, b1, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d4], a2, b2, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d5], a2, b3, %6, f;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d3], a3, b0, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d4], a3, b1, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d5], a3, b2, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [d6], a3, b3, %6, f;\n}" ::"r"(tmem),
        "l"(da), "l"(db), "n"(kFirst ? 1 : 0), "n"(kAPlane >> 4), "n"(kBPlane >> 4), "n"(kIdesc)
        : "memory");
}

// x mod p for x < 2^64, p < 2^31, m = floor((2^64 - 1) / p): the quotient
// estimate is at most two short
__device__ __forceinline__ uint32_t barrett(uint64_t x, uint32_t p, uint64_t m) {
    const uint64_t q = __umul64hi(x, m);
    uint64_t r = x - q * p;
    if (r >= p) r -= p;
    if (r >= p) r -= p;
    return static_cast<uint32_t>(r);
}

}  // namespace

struct I8Maps {
    CUtensorMap a[4];  // left-operand limb planes, box {64 k, 128 rows}, SWIZZLE_64B
    CUtensorMap b[4];  // right-operand limb planes, box {64 n, 64 k}, SWIZZLE_64B
};
struct I8Out {
    uint8_t* limb[4];  // next step's limb planes (n_pad x n_pad), or
    uint32_t* out;     // the final n x n residues (leading dim n)
    int n, n_pad;
    uint32_t p, r32;  // r32 = 2^32 mod p
    unsigned long long bm;  // floor((2^64 - 1) / p)
};

__global__ void __launch_bounds__(kThreads, 1)
    k5i_modmul(const __grid_constant__ I8Maps maps, const __grid_constant__ I8Out o) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // grouped raster (as K1): CTAs resident together share A row slabs and
    // B column slabs in L2
    constexpr int kGroupM = 16;
    const int num_m = o.n_pad / 128, num_n = o.n_pad / kBN;
    const int pid = blockIdx.x;
    const int per_group = kGroupM * num_n;
    const int first_m = (pid / per_group) * kGroupM;
    const int gm = min(num_m - first_m, kGroupM);
    const int m0 = (first_m + (pid % per_group) % gm) * 128;
    const int n0 = ((pid % per_group) / gm) * kBN;
    const int num_kb = o.n_pad / kKB;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
        for (int j = 0; j < 4; ++j) {
            tma_prefetch(&maps.a[j]);
            tma_prefetch(&maps.b[j]);
        }
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---------------------------------------------------------- TMA producer
        for (int kb = 0; kb < num_kb; ++kb) {
            const int st = kb % kStages;
            mbar_wait(&empty[st], ((kb / kStages) & 1) ^ 1);
            uint8_t* base = smem + st * kStageBytes;
            mbar_expect_tx(&full[st], kStageBytes);
            for (int j = 0; j < 4; ++j) {
                tma_load_2d(base + j * kAPlane, &maps.a[j], &full[st], kb * kKB, m0);
                tma_load_2d(base + 4 * kAPlane + j * kBPlane, &maps.b[j], &full[st], n0, kb * kKB);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA issue (whole warp)
        const uint32_t s0 = smem_u32(smem);
        const uint64_t da = smem_desc(s0, 16, 512, 4);                 // K-major SW64
        const uint64_t db = smem_desc(s0 + 4 * kAPlane, 8192, 512, 4);  // MN-major SW64
        for (int kb = 0; kb < num_kb; ++kb) {
            const int st = kb % kStages;
            mbar_wait(&full[st], (kb / kStages) & 1);
            tc_fence_after();
            const uint64_t so = static_cast<uint64_t>((st * kStageBytes) >> 4);
            // K step 0 (+32 B of A, +2048 B of B per further step)
            if (kb == 0) mma_i8_x16<true>(tmem, da + so, db + so);
            else mma_i8_x16<false>(tmem, da + so, db + so);
            mma_i8_x16<false>(tmem, da + so + (32 >> 4), db + so + (2048 >> 4));
            __syncwarp();
            if (lane == 0) mma_commit(&empty[st]);
            __syncwarp();
        }
        if (lane == 0) mma_commit(done);
        __syncwarp();
    } else if (warp >= 4) {
        // ---------------------------------------------------------- epilogue
        mbar_wait(done, 0);
        tc_fence_after();
        const int q = warp & 3, g = (warp - 4) >> 2;
        const int row = m0 + q * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int col_l = g * 32 + h * 16;
            uint64_t lo[16], hi[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) lo[i] = hi[i] = 0;
#pragma unroll
            for (int s = 0; s < 7; ++s) {
                uint32_t d[16];
                tmem_ld16(lane_base + static_cast<uint32_t>(s * kBN + col_l), d);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (s <= 3) lo[i] += static_cast<uint64_t>(d[i]) << (8 * s);
                    else hi[i] += static_cast<uint64_t>(d[i]) << (8 * (s - 4));
                }
            }
            uint32_t c[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t l = barrett(lo[i], o.p, o.bm);
                const uint32_t hm = barrett(hi[i], o.p, o.bm);
                uint32_t v = l + barrett(static_cast<uint64_t>(hm) * o.r32, o.p, o.bm);
                c[i] = v >= o.p ? v - o.p : v;
            }
            const int col = n0 + col_l;
            if (o.out != nullptr) {
                if (row < o.n) {
                    uint32_t* dst = o.out + static_cast<size_t>(row) * o.n;
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (col + i < o.n) dst[col + i] = c[i];
                }
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t w[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        w[u] = ((c[4 * u] >> (8 * j)) & 0xFFu) | (((c[4 * u + 1] >> (8 * j)) & 0xFFu) << 8) |
                               (((c[4 * u + 2] >> (8 * j)) & 0xFFu) << 16) |
                               (((c[4 * u + 3] >> (8 * j)) & 0xFFu) << 24);
                    *reinterpret_cast<uint4*>(o.limb[j] + static_cast<size_t>(row) * o.n_pad + col) =
                        make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// uint32 n x n residues -> reduced (mod p) byte limb planes, n_pad x n_pad, zero padded
__global__ void mod_split_u8_kernel(const uint32_t* __restrict__ in, int n, uint32_t p,
                                    uint8_t* __restrict__ l0, uint8_t* __restrict__ l1,
                                    uint8_t* __restrict__ l2, uint8_t* __restrict__ l3, int n_pad) {
    const size_t quads = static_cast<size_t>(n_pad) * n_pad / 4;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < quads;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t e = i * 4;
        const int r = static_cast<int>(e / n_pad), c = static_cast<int>(e % n_pad);
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = (r < n && c + k < n) ? in[static_cast<size_t>(r) * n + c + k] % p : 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] |= ((x >> (8 * j)) & 0xFFu) << (8 * k);
        }
        reinterpret_cast<uint32_t*>(l0)[i] = w[0];
        reinterpret_cast<uint32_t*>(l1)[i] = w[1];
        reinterpret_cast<uint32_t*>(l2)[i] = w[2];
        reinterpret_cast<uint32_t*>(l3)[i] = w[3];
    }
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
bool encode_u8(CUtensorMap* m, const void* plane, int n_pad, bool right) {
    EncodeFn fn = encode_fn();
    if (fn == nullptr) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(n_pad), static_cast<cuuint64_t>(n_pad)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(n_pad)};
    cuuint32_t box[2] = {64u, right ? static_cast<cuuint32_t>(kKB) : 128u};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(plane), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t prepare_mod_i8_kernel() {
    return cudaFuncSetAttribute(k5i_modmul, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmem));
}

cudaError_t launch_mod_split_u8(const uint32_t* in, int n, uint32_t p, uint8_t* const* limb,
                                int n_pad, cudaStream_t s) {
    mod_split_u8_kernel<<<148 * 8, 256, 0, s>>>(in, n, p, limb[0], limb[1], limb[2], limb[3], n_pad);
    return cudaGetLastError();
}

cudaError_t launch_mod_i8_gemm(uint8_t* const* a_limb, uint8_t* const* b_limb, int n_pad, uint32_t p,
                               uint8_t* const* out_limb, uint32_t* out, int n, cudaStream_t s) {
    if (n_pad % 128 != 0 || n_pad > kModI8MaxN || p < 2 || p >= (1u << 31)) return cudaErrorInvalidValue;
    I8Maps maps;
    for (int j = 0; j < 4; ++j)
        if (!encode_u8(&maps.a[j], a_limb[j], n_pad, false) || !encode_u8(&maps.b[j], b_limb[j], n_pad, true))
            return cudaErrorInvalidValue;
    I8Out o;
    std::memset(&o, 0, sizeof o);
    for (int j = 0; j < 4; ++j) o.limb[j] = out_limb ? out_limb[j] : nullptr;
    o.out = out;
    o.n = n;
    o.n_pad = n_pad;
    o.p = p;
    o.r32 = static_cast<uint32_t>((1ull << 32) % p);
    o.bm = ~0ull / p;
    const int grid = (n_pad / 128) * (n_pad / kBN);
    k5i_modmul<<<grid, kThreads, kSmem, s>>>(maps, o);
    return cudaGetLastError();
}

}  // namespace mxp
