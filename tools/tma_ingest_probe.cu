// TMA ingest from L2: how fast can N CTAs (one per SM) each pull B bytes
// of 16 KB boxes (32 fp32 columns x 128 rows, SWIZZLE_128B — K1C's A boxes)
// from an L2-resident tensor, with `share` CTAs loading the same boxes?
// Distinguishes a per-SM ingest limit from a chip-wide L2 limit (K1C's
// mainloop streams 192 KB per CTA per step at ~37 B/cycle).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_ingest_probe tools/tma_ingest_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(128, 1) ingest(const __grid_constant__ CUtensorMap map, int nbox,
                                                 int share, int iters, unsigned* ctr,
                                                 long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar;
    const int cta = blockIdx.x;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int group = cta / share;
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) {
            long long t0 = clock64();
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                         "r"(nbox * 16384));
            for (int b = 0; b < nbox; ++b) {
                const int id = group * nbox + b;  // box id: 16 column blocks per row block
                const int x = (id % 16) * 32, y = (id / 16) * 128;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem + b * 16384)),
                    "l"(&map), "r"(x), "r"(y), "r"(smem_u32(&bar))
                    : "memory");
            }
            asm volatile(
                "{\n\t.reg .pred p;\nW_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra W_%=;\n}" ::"r"(smem_u32(&bar)), "r"(it & 1) : "memory");
            long long t1 = clock64();
            cyc[it * gridDim.x + cta] = t1 - t0;
            // grid barrier before the next round
            atomicAdd(ctr, 1u);
            while (atomicAdd(ctr, 0u) < gridDim.x * (it + 1)) {
            }
        }
        __syncthreads();
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int rows = 32768, cols = 512;  // 64 MB fp32: L2-resident after a warm pass
    float* buf;
    cudaMalloc(&buf, (size_t)rows * cols * 4);
    cudaMemset(buf, 0, (size_t)rows * cols * 4);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
    }
    const size_t smem = 12 * 16384 + 1024;
    cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned* ctr;
    long long* cyc;
    cudaMalloc(&ctr, 4);
    cudaMalloc(&cyc, 148 * 16 * 8);
    const int iters = 8;
    struct Case { int ctas, nbox, share; };
    const Case cases[] = {{128, 12, 1}, {128, 12, 8}, {128, 12, 4}, {128, 12, 128}, {64, 12, 1},
                          {32, 12, 1}, {16, 12, 1}, {1, 12, 1}, {128, 6, 1}, {148, 12, 1}};
    for (const Case& c : cases) {
        cudaMemset(ctr, 0, 4);
        ingest<<<c.ctas, 128, smem>>>(map, c.nbox, c.share, iters, ctr, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        std::vector<long long> h(c.ctas * iters);
        cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
        double mean = 0, mx = 0;
        int cnt = 0;
        for (int it = 2; it < iters; ++it) {
            long long m = 0;
            for (int i = 0; i < c.ctas; ++i) {
                mean += h[it * c.ctas + i];
                ++cnt;
                if (h[it * c.ctas + i] > m) m = h[it * c.ctas + i];
            }
            mx += m;
        }
        mean /= cnt;
        mx /= (iters - 2);
        const double bytes = c.nbox * 16384.0;
        printf("ctas %3d  %3d KB/CTA  share %3d: mean %6.0f cyc (%5.1f B/cyc/SM), max %6.0f cyc; "
               "chip %6.0f B/cyc at the max\n",
               c.ctas, c.nbox * 16, c.share, mean, bytes / mean, mx, bytes * c.ctas / mx);
    }
    return 0;
}
