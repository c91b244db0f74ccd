// TMEM store (tcgen05.st 32x32b.x16) and st.shared.v4 throughput, 16 warps.
#include <cstdio>
#include "ptx.cuh"
using namespace mxp;

__global__ void bench(long long* cyc, int mode, int iters) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 131072);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tmem_alloc<512>(slot);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t q = warp & 3, g = warp >> 2;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = tid * 16 + i;
    const uint32_t s0 = smem_u32(smem);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {  // 128 KB of TMEM stores per iteration (each warp 8 KB: 4 x16 stores x 2 cols... )
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_st16(tmem + ((q * 32) << 16) + 256 + g * 64 + c * 16, v);
            tmem_st_wait();
        } else if (mode == 1) {  // 128 KB of st.shared.v4 per iteration, conflict-free
            const uint32_t row = q * 32 + lane;
#pragma unroll
            for (int c = 0; c < 16; ++c)
                sts128(s0 + ((g * 16 + c) & 31) * 4096 + (row & 31) * 128 + (((c ^ row) & 7) << 4), v[0], v[1], v[2], v[3]);
        } else {  // TMEM loads, 128 KB per iteration
            uint32_t a[16], b[16];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                tmem_ld16x2(tmem + ((q * 32) << 16) + g * 32 + c * 16, tmem + ((q * 32) << 16) + 128 + g * 32 + c * 16, a, b);
                for (int i = 0; i < 16; ++i) v[i] += a[i] + b[i];
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) cyc[0] = t1 - t0;
    if (v[0] == 12345) cyc[1] = v[1];
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    long long* dc; long long h;
    cudaMalloc(&dc, 16);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    const char* names[] = {"tcgen05.st 128KB/iter", "st.shared 128KB/iter", "tcgen05.ld 128KB/iter"};
    for (int mode = 0; mode < 3; ++mode) {
        bench<<<1, 512, 140000>>>(dc, mode, 256);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
        printf("%-26s err=%s %.1f cyc/iter -> %.1f B/cyc\n", names[mode], cudaGetErrorString(e), h / 256.0, 131072.0 / (h / 256.0));
    }
    return 0;
}
