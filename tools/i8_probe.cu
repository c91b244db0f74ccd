// Probe: tcgen05.mma kind::i8 (u8 x u8 -> s32) operand layouts and rate on
// sm_100a, for the exact-modular int8 limb GEMM (kernels_mod.cu K5I).
//   V1: A K-major SWIZZLE_128B, B MN-major SWIZZLE_64B (N = 64)
//   V2: A K-major SWIZZLE_128B, B K-major SWIZZLE_128B (B^T rows, N = 64)
//   V3: A K-major SWIZZLE_128B, B MN-major SWIZZLE_128B (N = 128)
//   V4: as V1 with A copied into TMEM (tcgen05.cp 128x256b) and read from there (TS)
// Each: D = A[128 x 128] * B[128 x N] (4 MMAs of K = 32) vs a host int matmul.
// Then the issue rate of 256 back-to-back MMAs (N = 64 and N = 128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include \
//        tools/i8_probe.cu -o tools/i8_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1204_3052_b200/csrc/ptx.cuh"

using namespace mxp;

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

template <int N, bool kBMN>
__host__ __device__ constexpr uint32_t idesc_i8() {
    // [4,6) c_format = 2 (S32), a/b_format = 0 (u8), [15] a_major = 0 (K),
    // [16] b_major, [17,23) N >> 3, [24,29) M >> 4 (M = 128)
    return (2u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | ((kBMN ? 1u : 0u) << 16) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

struct Maps {
    CUtensorMap a, b;
};

// variant: 1, 2, 3 (see above); out: 128 x N int32
template <int N, int V>
__global__ void probe_kernel(const __grid_constant__ Maps m, int* out, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;               // 128 x 128 B = 16 KB
    uint8_t* sb = smem + 16384;       // up to 16 KB
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        const uint32_t bbytes = (V == 2) ? N * 128 : 128 * N;
        mbar_expect_tx(bar, 16384 + bbytes);
        tma_load_2d(sa, &m.a, bar, 0, 0);
        if (V == 1 || V == 4) {
            tma_load_2d(sb, &m.b, bar, 0, 0);           // box {64 N, 128 K}
        } else if (V == 2) {
            tma_load_2d(sb, &m.b, bar, 0, 0);           // box {128 K, 64 N}
        } else {
            tma_load_2d(sb, &m.b, bar, 0, 0);           // box {128 N, 128 K}
        }
        mbar_wait(bar, 0);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
        constexpr uint32_t idesc = idesc_i8<N, V != 2>();
        if (V == 4) {
            // A -> TMEM columns 256 + 8 ks (128 lanes x 32 bytes per K=32 step)
            for (int k = 0; k < 4; ++k) tmem_cp_128x256b(tmem + 256 + 8 * k, smem_desc(a0 + 32 * k, 16, 1024, 2));
            for (int k = 0; k < 4; ++k)
                mma_i8_ts(tmem, tmem + 256 + 8 * k, smem_desc(b0 + 2048 * k, 8192, 512, 4), idesc, k > 0);
            mma_commit(bar + 1);
            mbar_wait(bar + 1, 0);
            const long long t0 = clock64();
            for (int r = 0; r < 64; ++r)
                for (int k = 0; k < 4; ++k)
                    mma_i8_ts(tmem, tmem + 256 + 8 * k, smem_desc(b0 + 2048 * k, 8192, 512, 4), idesc, 1);
            mma_commit(bar + 1);
            mbar_wait(bar + 1, 1);
            cycles[0] = clock64() - t0;
        } else {
        for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc(a0 + 32 * k, 16, 1024, 2);
            uint64_t bd;
            if (V == 1) bd = smem_desc(b0 + 2048 * k, 8192, 512, 4);       // MN SW64
            else if (V == 2) bd = smem_desc(b0 + 32 * k, 16, 1024, 2);     // K-major SW128
            else bd = smem_desc(b0 + 4096 * k, 16384, 1024, 2);            // MN SW128
            mma_i8(tmem, ad, bd, idesc, k > 0);
        }
        mma_commit(bar + 1);
        // rate: 256 MMAs into a scratch accumulator, timed
        mbar_wait(bar + 1, 0);
        const long long t0 = clock64();
        for (int r = 0; r < 64; ++r)
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad = smem_desc(a0 + 32 * k, 16, 1024, 2);
                const uint64_t bd = (V == 2) ? smem_desc(b0 + 32 * k, 16, 1024, 2)
                                             : (V == 1 ? smem_desc(b0 + 2048 * k, 8192, 512, 4)
                                                       : smem_desc(b0 + 4096 * k, 16384, 1024, 2));
                mma_i8(tmem + 0, ad, bd, idesc, 1);
            }
        mma_commit(bar + 1);
        mbar_wait(bar + 1, 1);
        cycles[0] = clock64() - t0;
        }
    }
    __syncthreads();
    tc_fence_after();
    // the accumulated result after the first 4 MMAs was overwritten by the
    // rate loop (it kept accumulating): recompute expected = 65 * A*B on host
    if (warp < 4) {
        for (int c = 0; c < N; c += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
            for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * N + c + i] = static_cast<int>(v[i]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
static EncodeFn enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<EncodeFn>(p);
}
static void map2d(CUtensorMap* m, void* p, int cols, int rows, int bc, int br, CUtensorMapSwizzle sw) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)cols};
    cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, str, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
}

template <int N, int V>
static void run(const std::vector<uint8_t>& A, const std::vector<uint8_t>& B) {
    // A: 128 x 128 (K); B: 128 (K) x N row-major; Bt: N x 128
    std::vector<uint8_t> Bt(N * 128);
    for (int k = 0; k < 128; ++k)
        for (int j = 0; j < N; ++j) Bt[j * 128 + k] = B[k * N + j];
    uint8_t *dA, *dB;
    int* dO;
    long long* dC;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, 128 * N);
    cudaMalloc(&dO, 128 * N * 4);
    cudaMalloc(&dC, 8);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, V == 2 ? Bt.data() : B.data(), 128 * N, cudaMemcpyHostToDevice);
    Maps m;
    map2d(&m.a, dA, 128, 128, 128, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (V == 1 || V == 4) map2d(&m.b, dB, N, 128, N, 128, CU_TENSOR_MAP_SWIZZLE_64B);
    else if (V == 2) map2d(&m.b, dB, 128, N, 128, N, CU_TENSOR_MAP_SWIZZLE_128B);
    else map2d(&m.b, dB, N, 128, N, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    cudaFuncSetAttribute(probe_kernel<N, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    probe_kernel<N, V><<<1, 128, 40000>>>(m, dO, dC);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> out(128 * N);
    long long cyc = 0;
    cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dC, 8, cudaMemcpyDeviceToHost);
    long long bad = 0, first = -1;
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
            long long s = 0;
            for (int k = 0; k < 128; ++k) s += (long long)A[i * 128 + k] * B[k * N + j];
            s *= 65;  // 1 + 64 rate rounds of the same 4 MMAs
            if ((long long)(unsigned)out[i * N + j] != s) {
                if (first < 0) first = i * N + j;
                ++bad;
            }
        }
    printf("V%d N=%d: err=%s mismatches=%lld/%d%s  rate: 256 MMAs in %lld cycles = %.1f cyc/MMA\n", V,
           N, cudaGetErrorString(e), bad, 128 * N,
           first >= 0 ? " (first at row/col shown below)" : "", cyc, cyc / 256.0);
    if (first >= 0) {
        int i = first / N, j = first % N;
        long long s = 0;
        for (int k = 0; k < 128; ++k) s += (long long)A[i * 128 + k] * B[k * N + j];
        printf("   row %d col %d: got %u want %lld\n", i, j, (unsigned)out[first], s * 65);
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
    cudaFree(dC);
}

int main() {
    std::vector<uint8_t> A(128 * 128), B64(128 * 64), B128(128 * 128);
    unsigned s = 12345;
    auto rnd = [&] { s = s * 1103515245u + 12345u; return static_cast<uint8_t>((s >> 16) & 0xFF); };
    for (auto& x : A) x = rnd();
    for (auto& x : B64) x = rnd();
    for (auto& x : B128) x = rnd();
    run<64, 1>(A, B64);
    run<64, 2>(A, B64);
    run<128, 3>(A, B128);
    run<64, 4>(A, B64);
    return 0;
}
