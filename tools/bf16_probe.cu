// Layout + rate probe for the bf16x3 dual-chain K3 design (kind::f16, bf16
// operands, fp32 accumulate):
//   * one row-major 128x128 bf16 plane stored as [c/64][r][128 B, 16-byte
//     units XOR r%8] serves as the K-major SW128 LEFT operand (SS) AND as the
//     MN-major SW128 RIGHT operand;
//   * the TS form (A in TMEM, two bf16 per 32-bit column) — which half is
//     the lower k;
//   * the issue rate of 48 M=N=128 K=16 MMAs (40 TS + 8 SS) per "step".
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2
//        -I paper_1204_3052_b200/csrc tools/bf16_probe.cu -o tools/bf16_probe -lcuda
#include <cuda_bf16.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "ptx.cuh"
using namespace mxp;

// bf16 A/B, f32 D, A K-major, B MN-major (bit 16), N>>3 at 17, M>>4 at 24
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((128u >> 3) << 17) |
                            ((128u >> 4) << 24);

__host__ __device__ inline uint32_t plane_off(int r, int c) {
    return (c / 64) * 16384 + r * 128 + ((((c % 64) / 8) ^ (r % 8)) * 16) + (c % 8) * 2;
}

// mode 0: SS, mode 1: TS (lo half = even k), mode 2: TS (hi half = even k)
// bswap: 0 -> LBO = 16384 (N chunk), SBO = 1024 (K group); 1 -> swapped
__global__ void probe(const uint16_t* plane_img, int mode, int bswap, int reps, float* out,
                      long long* cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 32768 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = reinterpret_cast<const uint4*>(plane_img)[i];
    if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t s = smem_u32(smem);
    if (mode >= 1 && warp < 4) {
        // A in TMEM columns [256, 320): row m = warp*32+lane, 2 bf16 per column
        const int m = warp * 32 + lane;
        for (int c0 = 0; c0 < 64; c0 += 16) {
            uint32_t v[16];
            for (int j = 0; j < 16; ++j) {
                const int k = 2 * (c0 + j);
                const uint16_t e0 = *reinterpret_cast<const uint16_t*>(smem + plane_off(m, k));
                const uint16_t e1 = *reinterpret_cast<const uint16_t*>(smem + plane_off(m, k + 1));
                v[j] = (mode == 1) ? (uint32_t(e1) << 16 | e0) : (uint32_t(e0) << 16 | e1);
            }
            tmem_st16(tmem + ((warp * 32) << 16) + 256 + c0, v);
        }
        tmem_st_wait();
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    long long t0 = clock64();
    if (tid == 0) {
        const uint32_t lbo = bswap ? 1024 : 16384, sbo = bswap ? 16384 : 1024;
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t bd = smem_desc(s + kk * 2048, lbo, sbo, 2);
                const uint64_t ad = smem_desc(s + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, 2);
                const uint32_t acc = (kk > 0 || r > 0) ? 1u : 0u;
                if (mode == 0) mma_f16_ss(tmem, ad, bd, kIdesc, acc);
                else mma_f16_ts(tmem, tmem + 256 + 8 * kk, bd, kIdesc, acc);
                if (reps > 1) {  // rate test: 6 MMAs per k-step (5 TS + 1 SS)
                    mma_f16_ts(tmem + 128, tmem + 256 + 8 * kk, bd, kIdesc, 1);
                    mma_f16_ts(tmem + 128, tmem + 256 + 8 * kk, bd, kIdesc, 1);
                    mma_f16_ts(tmem + 128, tmem + 256 + 8 * kk, bd, kIdesc, 1);
                    mma_f16_ts(tmem + 128, tmem + 256 + 8 * kk, bd, kIdesc, 1);
                    mma_f16_ss(tmem + 128, ad, bd, kIdesc, 1);
                }
            }
        }
        mma_commit(bar);
    }
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (tid == 0) *cycles = t1 - t0;
    tc_fence_after();
    if (warp < 4) {
        for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld32(tmem + ((warp * 32) << 16) + 32 * c, v);
            for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 128 + 32 * c + i] = __uint_as_float(v[i]);
        }
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int mode>
__global__ void rate(const uint16_t* plane_img, int reps, long long* cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 32768 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = reinterpret_cast<const uint4*>(plane_img)[i];
    if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t s = smem_u32(smem);
    long long t0 = clock64();
    if (tid == 0) {
        const uint64_t bd0 = smem_desc(s, 16384, 1024, 2);
        const uint64_t ad0 = smem_desc(s, 16, 1024, 2);
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int t = 0; t < 6; ++t)
#pragma unroll
                for (uint32_t kk = 0; kk < 8; ++kk) {
                    const bool alt = (mode & 1);
                    const uint32_t d = tmem + ((alt && (kk & 1)) ? 128u : 0u);
                    const uint64_t bd = bd0 + kk * 128u;
                    const uint64_t ad = ad0 + (kk >> 2) * 1024u + (kk & 3u) * 2u;
                    const bool ss = (mode == 2 || mode == 3) || ((mode == 4 || mode == 5) && t == 0);
                    if (ss) mma_f16_ss(d, ad, bd, kIdesc, 1u);
                    else mma_f16_ts(d, tmem + 256 + 8 * kk, bd, kIdesc, 1u);
                }
        }
        mma_commit(bar);
    }
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (tid == 0 && blockIdx.x == 0) *cycles = t1 - t0;
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

static uint16_t bf(float x) {
    uint32_t u; memcpy(&u, &x, 4);
    return uint16_t(u >> 16);  // exact for the small integers used here
}

int main() {
    const int n = 128;
    std::vector<float> P(n * n);
    unsigned st = 12345;
    for (auto& x : P) { st = st * 1103515245u + 12345u; x = float(int((st >> 16) % 5) - 2); }
    std::vector<uint16_t> img(16384, 0);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) img[plane_off(r, c) / 2] = bf(P[r * n + c]);
    std::vector<double> ref(n * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j) ref[i * n + j] += double(P[i * n + k]) * P[k * n + j];
    uint16_t* dimg; float* dout; long long* dcyc;
    cudaMalloc(&dimg, 32768); cudaMalloc(&dout, n * n * 4); cudaMalloc(&dcyc, 8);
    cudaMemcpy(dimg, img.data(), 32768, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaFuncSetAttribute(rate<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaFuncSetAttribute(rate<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaFuncSetAttribute(rate<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaFuncSetAttribute(rate<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    const char* names[3] = {"SS", "TS lo=even", "TS hi=even"};
    std::vector<float> h(n * n);
    for (int mode = 0; mode < 3; ++mode)
        for (int bswap = 0; bswap < 2; ++bswap) {
            cudaMemset(dout, 0xFF, n * n * 4);
            probe<<<1, 128, 40000>>>(dimg, mode, bswap, 1, dout, dcyc);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h.data(), dout, n * n * 4, cudaMemcpyDeviceToHost);
            int bad = 0, first = -1;
            for (int i = 0; i < n * n; ++i)
                if (double(h[i]) != ref[i]) { if (first < 0) first = i; ++bad; }
            printf("%-12s bswap=%d err=%s bad=%d", names[mode], bswap, cudaGetErrorString(e), bad);
            if (first >= 0) printf(" first(%d,%d) got %g want %g", first / n, first % n, h[first], ref[first]);
            printf("\n");
            if (e != cudaSuccess) return 1;
        }
    // rate: 48 MMAs per rep, accumulator patterns
    const char* rn[] = {"TS same D", "TS alt D0/D1", "SS same D", "SS alt D0/D1", "8SS+40TS same D", "8SS+40TS alt"};
    for (int rm = 0; rm < 6; ++rm) {
        long long cyc = 0;
        switch (rm) {
            case 0: rate<0><<<1, 128, 40000>>>(dimg, 128, dcyc); break;
            case 1: rate<1><<<1, 128, 40000>>>(dimg, 128, dcyc); break;
            case 2: rate<2><<<1, 128, 40000>>>(dimg, 128, dcyc); break;
            case 3: rate<3><<<1, 128, 40000>>>(dimg, 128, dcyc); break;
            case 4: rate<4><<<1, 128, 40000>>>(dimg, 128, dcyc); break;
            default: rate<5><<<1, 128, 40000>>>(dimg, 128, dcyc); break;
        }
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
        printf("rate %-18s err=%s %.1f cycles/MMA\n", rn[rm], cudaGetErrorString(e), double(cyc) / (48.0 * 128));
    }
    // chip-wide: 148 CTAs (one per SM), SS/TS mix, longer run
    for (int reps : {128, 1024}) {
        long long cyc = 0;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        rate<4><<<148, 128, 40000>>>(dimg, reps, dcyc);
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, a, b);
        cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
        printf("rate 148 CTAs reps=%d err=%s %.1f cycles/MMA, %.3f ms -> %.0f MHz effective, %.1f dense bf16 TFLOP/s\n", reps,
               cudaGetErrorString(e), double(cyc) / (48.0 * reps), ms, cyc / (ms * 1e3),
               148.0 * 48 * reps * 2.0 * 128 * 128 * 16 / (ms * 1e-3) / 1e12);
    }
    return 0;
}
