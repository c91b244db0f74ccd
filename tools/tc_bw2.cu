// MMA rate with fully unrolled issue (precomputed descriptors, constant offsets).
#include <cstdio>
#include "ptx.cuh"
using namespace mxp;

template <int MODE>
__device__ __forceinline__ void issue16(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t a_t, uint32_t first) {
    constexpr uint32_t id128 = idesc_tf32_kmaj_mnmaj<128, 128>();
    constexpr uint32_t id256 = idesc_tf32_kmaj_mnmaj<128, 256>();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        // descriptor start address field is in 16-byte units (bits 0..13)
        const uint64_t a = adesc + (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
        const uint64_t b = bdesc + (uint64_t)((k * 1024) >> 4);
        const uint32_t acc = (k > 0) ? 1u : first;
        if (MODE == 1) mma_tf32(tmem, a, b, id128, acc);
        if (MODE == 2) mma_tf32_ts(tmem, a_t + 8 * k, b, id128, acc);
        if (MODE == 3) mma_tf32(tmem, a, b, id256, acc);
        if (MODE == 4) mma_tf32_ts(tmem + 128 * (k & 1), a_t + 8 * k, b, id128, k > 1 ? 1u : first);
        if (MODE == 5) mma_tf32(tmem + 256 * (k & 1), a, b, id256, k > 1 ? 1u : first);
        if (MODE == 6) mma_tf32_ts(tmem + 64 * (k & 1), a_t + 8 * k, b, idesc_tf32_kmaj_mnmaj<128, 64>(), k > 1 ? 1u : first);
        if (MODE == 7) mma_tf32_ts(tmem + 32 * (k & 1), a_t + 8 * k, b, idesc_tf32_kmaj_mnmaj<128, 32>(), k > 1 ? 1u : first);
        if (MODE == 8) mma_tf32(tmem + 64 * (k & 1), a, b, idesc_tf32_kmaj_mnmaj<128, 64>(), k > 1 ? 1u : first);
    }
}

template <int MODE>
__global__ void bench(long long* cyc, int reps) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 196608);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 196608 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i & 255);
    if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot;
    if (tid == 0) {
        const uint32_t s = smem_u32(smem);
        const uint64_t adesc = kmajor_desc(s);
        const uint64_t bdesc = (MODE == 3 || MODE == 5) ? mnmajor_desc(s + 65536, 16384) : mnmajor_desc(s + 65536, 16384);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) issue16<MODE>(tmem, adesc, bdesc, tmem + 256, r > 0);
        long long t1 = clock64();
        mma_commit(bar);
        mbar_wait(bar, 0);
        long long t2 = clock64();
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name) {
    long long* dc; long long h[2];
    cudaMalloc(&dc, 16);
    cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    for (int reps : {4, 64}) {
        bench<MODE><<<1, 128, 200000>>>(dc, reps);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, dc, 16, cudaMemcpyDeviceToHost);
        const int n = reps * 16;
        printf("%-36s mmas=%5d err=%s issue %.1f cyc/mma, complete %.1f cyc/mma\n", name, n, cudaGetErrorString(e),
               double(h[0]) / n, double(h[1]) / n);
    }
}

int main() {
    run<1>("SS M128 N128 K8 (1 acc)");
    run<2>("TS M128 N128 K8 (1 acc)");
    run<3>("SS M128 N256 K8 (1 acc)");
    run<4>("TS M128 N128 K8 (2 accs)");
    run<5>("SS M128 N256 K8 (2 accs)");
    run<6>("TS M128 N64 K8 (2 accs)");
    run<7>("TS M128 N32 K8 (2 accs)");
    run<8>("SS M128 N64 K8 (2 accs)");
    return 0;
}
