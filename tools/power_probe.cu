// Power-capped tensor throughput: the same logical 128^3 step (a product at
// ~22-24 significant bits) as
//   F16: K3H's step — 24 fp16 MMAs (M128 N128 K16), A from TMEM (TS), the
//        scaled fp16x2 planes (h0 ~ U(-2^14, 2^14), h1 ~ U(-4, 4));
//   I8 : 24 int8 MMAs (M128 N128 K32, s8 x s8 -> s32), both operands from
//        SMEM (SS): three byte limbs per value, the 6 limb products of weight
//        >= 2^16 (4 K-chunks x 6), uniform random bytes;
//   Z16: F16 with all-zero h1 planes (what a "free" residual would cost).
// One CTA per SM, ~0.6 s per run: ns per step from globaltimer and the SM
// clock from clock64, i.e. what the board's power limit lets each datapath do.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I paper_1204_3052_b200/csrc
//   tools/power_probe.cu paper_1204_3052_b200/csrc/kernels_tf32.cu paper_1204_3052_b200/csrc/kernels_k3b.cu -o tools/power_probe -lcuda
#include <cstdio>
#include <cuda_fp16.h>
#include "../paper_1204_3052_b200/csrc/kernels_k3h.cu"
using namespace mxp;

// s8 x s8 -> s32, A K-major, B MN-major, N = 128, M = 128
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((128u >> 3) << 17) |
                              ((128u >> 4) << 24);

// one K=32 chunk: the six limb products (a, b) with a + b >= 2 into three
// weight groups (TMEM columns 0 / 128 / 256), descriptors advanced in-asm
__device__ __forceinline__ void i8_chunk6(uint32_t tmem, uint64_t a0, uint64_t b0, uint64_t lstride,
                                          uint32_t first) {
    asm volatile(
        "{\n\t.reg .pred p, f, e;\n\t.reg .b32 g0, g1, g2;\n\t.reg .b64 a1, a2, b1, b2;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.eq.u32 p, 1, 1;\n\tsetp.eq.u32 f, %4, 0;\n\t"
        "mov.b32 g0, %0;\n\tadd.u32 g1, g0, 128;\n\tadd.u32 g2, g0, 256;\n\t"
        "add.s64 a1, %1, %3;\n\tadd.s64 a2, a1, %3;\n\t"
        "add.s64 b1, %2, %3;\n\tadd.s64 b2, b1, %3;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [g0], a2, b2, %5, f;\n\t"   // 2^32
        "@e tcgen05.mma.cta_group::1.kind::i8 [g1], a2, b1, %5, f;\n\t"   // 2^24
        "@e tcgen05.mma.cta_group::1.kind::i8 [g1], a1, b2, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [g2], a2, %2, %5, f;\n\t"   // 2^16
        "@e tcgen05.mma.cta_group::1.kind::i8 [g2], a1, b1, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [g2], %1, b2, %5, p;\n\t}" ::"r"(tmem),
        "l"(a0), "l"(b0), "l"(lstride), "r"(first), "r"(kIdescI8)
        : "memory");
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t f16bits(float v) {
    return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v)));
}
// two fp16 of U(-r, r) packed
__device__ __forceinline__ uint32_t rnd_f16x2(uint32_t h, float r) {
    const float a = ((h & 0xFFFFu) / 65536.0f * 2.0f - 1.0f) * r;
    const float b = ((h >> 16) / 65536.0f * 2.0f - 1.0f) * r;
    return f16bits(a) | (f16bits(b) << 16);
}

__global__ void __launch_bounds__(kThreads, 1) probe(int variant, int steps, long long* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
    const int tid = threadIdx.x, warp = tid >> 5;
    // SMEM: F16 -> y0 plane h0-like, y1 plane h1-like for both chains; I8 -> random bytes
    for (uint32_t i = tid; i < kMaxOff / 4; i += blockDim.x) {
        const uint32_t h = hash32(i * 2654435761u + blockIdx.x * 0x9E3779B9u);
        uint32_t v;
        if (variant == 1) {
            v = h;
        } else {
            const bool lo_plane = ((i * 4) / kPlane) & 1;  // y1 planes
            v = lo_plane ? (variant == 2 ? 0u : rnd_f16x2(h, 4.0f)) : rnd_f16x2(h, 16384.0f);
        }
        reinterpret_cast<uint32_t*>(smem)[i] = v;
    }
    if (tid == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        mbar_init(bars + 2, 1);
        fence_mbar_init();
    }
    if (warp == kIssueWarp) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot, s0 = smem_u32(smem);
    if (variant != 1 && warp < 4) {  // TMEM x planes (x0 h0-like at D+128, x1 h1-like at D+192)
        for (uint32_t c = 0; c < 512; c += 8) {
            uint32_t p[8];
            const bool x1 = (c & 255u) >= 192u;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t h = hash32((c + i) * 0x85EBCA6Bu ^ (tid * 0xC2B2AE35u) ^ blockIdx.x);
                p[i] = x1 ? (variant == 2 ? 0u : rnd_f16x2(h, 4.0f)) : rnd_f16x2(h, 16384.0f);
            }
            tmem_st8(tmem + ((warp * 32) << 16) + c, p);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kIssueWarp) {
        long long c0 = clock64();
        unsigned long long g0 = globaltimer_ns();
        for (int s = 0; s < steps; ++s) {
            if (variant == 1) {
                // limb planes: 3 x 16 KB (128 rows x 128 bytes), chunk c = 32 bytes of K
                const uint64_t a = kmajor_desc(s0), b = smem_desc(s0, 8192, 1024, 2);
                const uint64_t lstride = (16384u >> 4);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    i8_chunk6(tmem, a + ((32u * c) >> 4), b + ((4096u * c) >> 4), lstride, c);
                mma_commit_warp(bars + (s & 1));
            } else {
                if (s & 1) k3h_issue<1>(tmem, s0 + kChainSmem, bars);
                else k3h_issue<0>(tmem, s0, bars);
            }
        }
        mma_commit_warp(bars + 2);
        mbar_wait_sleep(bars + 2, 0);
        if ((tid & 31) == 0) {
            out[blockIdx.x * 2] = clock64() - c0;
            out[blockIdx.x * 2 + 1] = static_cast<long long>(globaltimer_ns() - g0);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kIssueWarp) tmem_dealloc<512>(tmem);
}

int main() {
    long long* out;
    cudaMalloc(&out, 148 * 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    const char* names[3] = {"F16 (K3H step, TS, realistic planes)", "I8  (6 limb products, SS, random bytes)",
                            "Z16 (F16 with zero h1 planes)"};
    const int steps = 400000;
    for (int rep = 0; rep < 2; ++rep)
        for (int v : {0, 1, 2, 0}) {
            probe<<<148, kThreads, kSmem>>>(v, steps, out);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[296];
            cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
            double cyc = 0, ns = 0;
            for (int i = 0; i < 148; ++i) {
                cyc += h[2 * i];
                ns += h[2 * i + 1];
            }
            cyc /= 148;
            ns /= 148;
            printf("%-44s err=%s: %.1f ns/step, %.1f cycles/step (%.1f per MMA), %.0f MHz, %.3f s\n",
                   names[v], cudaGetErrorString(e), ns / steps, cyc / steps, cyc / steps / 24,
                   cyc / ns * 1e3, ns * 1e-9);
        }
    return 0;
}
