// Microbenchmarks on one SM: tcgen05.ld bandwidth and tcgen05.mma (tf32) rate.
#include <cstdio>
#include "ptx.cuh"
using namespace mxp;

__global__ void bench(long long* cyc, float* sink, int mode, int iters) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 131072);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 131072 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i & 255);
    if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t q = warp & 3, half = warp >> 2;
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {  // every warp drains its 32 lanes x 64 columns, `iters` times
        for (int it = 0; it < iters; ++it) {
            uint32_t v[32];
            tmem_ld32(tmem + (q * 32 << 16) + half * 64, v);
            for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
            tmem_ld32(tmem + (q * 32 << 16) + half * 64 + 32, v);
            for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
        }
    } else if (tid == 0) {  // mode 1: SS MMAs N=128; mode 2: TS MMAs N=128; mode 3: SS N=256
        const uint32_t s = smem_u32(smem);
        const uint32_t id128 = idesc_tf32_kmaj_mnmaj<128, 128>();
        const uint32_t id256 = idesc_tf32_kmaj_mnmaj<128, 256>();
        for (int it = 0; it < iters; ++it) {
            const int k = it & 15;
            if (mode == 1)
                mma_tf32(tmem, kmajor_desc(s + (k >> 2) * 16384 + (k & 3) * 32), mnmajor_desc(s + 65536 + k * 1024, 16384), id128, it > 0);
            else if (mode == 2)
                mma_tf32_ts(tmem, tmem + 256 + 8 * k, mnmajor_desc(s + 65536 + k * 1024, 16384), id128, it > 0);
            else if (mode == 3)
                mma_tf32(tmem, kmajor_desc(s + (k >> 2) * 16384 + (k & 3) * 32), mnmajor_desc(s + k * 1024, 8192), id256, it > 0);
            else if (mode == 4)  // TS N=128 alternating 2 accumulators
                mma_tf32_ts(tmem + 128 * (it & 1), tmem + 256 + 8 * k, mnmajor_desc(s + 65536 + k * 1024, 16384), id128, it > 1);
            else if (mode == 5)  // SS N=128 alternating 2 accumulators
                mma_tf32(tmem + 128 * (it & 1), kmajor_desc(s + (k >> 2) * 16384 + (k & 3) * 32), mnmajor_desc(s + 65536 + k * 1024, 16384), id128, it > 1);
            else if (mode == 6)  // SS N=256 alternating 2 accumulators
                mma_tf32(tmem + 256 * (it & 1), kmajor_desc(s + (k >> 2) * 16384 + (k & 3) * 32), mnmajor_desc(s + k * 1024, 8192), id256, it > 1);
            else if (mode == 7)  // TS N=128 4 accumulators (cols 0..255 only 2 fit with A at 256) -> use 2
                mma_tf32_ts(tmem + 64 * (it & 3), tmem + 256 + 8 * k, mnmajor_desc(s + 65536 + k * 1024, 16384), idesc_tf32_kmaj_mnmaj<128, 64>(), it > 3);
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
    }
    long long t1 = clock64();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) cyc[0] = t1 - t0;
    sink[tid] = acc;
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    long long* dc; float* ds; long long h;
    cudaMalloc(&dc, 8); cudaMalloc(&ds, 4096);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    const char* names[] = {"tmem ld 64KB per iter (8 warps)", "mma SS M128 N128 K8", "mma TS M128 N128 K8", "mma SS M128 N256 K8",
                           "mma TS N128 2 accumulators", "mma SS N128 2 accumulators", "mma SS N256 2 accumulators", "mma TS N64 4 accumulators"};
    for (int mode = 0; mode < 8; ++mode) {
        for (int iters : {64, 1024}) {
            bench<<<1, 256, 140000>>>(dc, ds, mode, iters);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
            double per = double(h) / iters;
            if (mode == 0) printf("%-34s iters=%5d err=%s: %.1f cyc/iter -> %.1f B/cyc\n", names[mode], iters, cudaGetErrorString(e), per, 65536.0 / per);
            else printf("%-34s iters=%5d err=%s: %.1f cyc/mma\n", names[mode], iters, cudaGetErrorString(e), per);
        }
    }
    return 0;
}
