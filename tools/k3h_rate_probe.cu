// Tensor-pipe rate of the K3H step (k3h_issue: 24 TS-mode fp16 MMAs, N = 128)
// alone and under the epilogue's kinds of traffic, one CTA per SM.  The issue
// warp alternates chains 0/1 back to back; the 16 other warps run, until the
// issuer is done, a loop of (mode bits): 1 tcgen05.ld 32 columns (+wait) of
// chain 0's D, 2 st.shared 128-bit into the planes, 4 tcgen05.st 8 columns
// into chain 1's x planes.  Prints cycles per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I paper_1204_3052_b200/csrc
//   tools/k3h_rate_probe.cu paper_1204_3052_b200/csrc/kernels_tf32.cu paper_1204_3052_b200/csrc/kernels_k3b.cu -lcuda
#include <cstdio>
#include "../paper_1204_3052_b200/csrc/kernels_k3h.cu"
using namespace mxp;
// the same step with both operands from SMEM (SS): the plane is the K-major
// left operand and the MN-major right operand at once
template <uint32_t C>
__device__ __forceinline__ void k3h_issue_ss(uint32_t tbase, uint32_t s0, uint64_t* mma_bar) {
    const uint32_t pl = s0 + C * kChainSmem;
    const uint64_t y0 = smem_desc(pl, 16384, 1024, 2), y1 = smem_desc(pl + kPlane, 16384, 1024, 2);
    const uint64_t x0 = smem_desc(pl, 16, 1024, 2), x1 = smem_desc(pl + kPlane, 16, 1024, 2);
    constexpr uint32_t D = C * 256u;
    mma_f16_ss_x8<D, 0, kBStep, (16384u >> 4), true>(tbase, x1, y0, kIdescNegA);
    mma_f16_ss_x8<D, 0, kBStep, (16384u >> 4), false>(tbase, x0, y1, kIdescNegB);
    mma_f16_ss_x8<D, 0, kBStep, (16384u >> 4), false>(tbase, x0, y0, kIdesc);
    mma_commit_warp(mma_bar + C);
}
__global__ void __launch_bounds__(kThreads, 1) rate(int steps, int mode, int fill, int ss, long long* cyc, uint32_t* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
    volatile uint32_t* done = reinterpret_cast<volatile uint32_t*>(bars + 5);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < static_cast<int>(kMaxOff / 16); i += blockDim.x) {
        uint32_t x = (i * 2654435761u) ^ 0x9E3779B9u;
        x ^= x >> 13;
        x *= 0x85EBCA6Bu;
        // fill 0: fp16 in +-[0.5, 1); 1: random fp16 over the full finite range; 2: zeros
        x = fill == 0 ? ((x & 0x83FF83FFu) | 0x38003800u) : (fill == 1 ? (x & 0xBBFFBBFFu) : 0u);
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(x, x ^ 0x01230123u, x ^ 0x00450045u, x ^ 0x02000200u);
    }
    if (tid == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        mbar_init(bars + 2, 1);
        *done = 0;
        fence_mbar_init();
    }
    if (warp == kIssueWarp) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot, s0 = smem_u32(smem);
    uint32_t acc = 0;
    if (warp < 4) {  // x planes of both chains: the same kind of data as the SMEM operands
        for (uint32_t c = 0; c < 512; c += 8) {
            uint32_t p[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t x = ((c + i) * 2654435761u) ^ (tid * 0x9E3779B9u);
                x ^= x >> 15;
                x *= 0x2C1B3C6Du;
                p[i] = fill == 0 ? ((x & 0x83FF83FFu) | 0x38003800u) : (fill == 1 ? (x & 0xBBFFBBFFu) : 0u);
            }
            tmem_st8(tmem + ((warp * 32) << 16) + c, p);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    long long t0 = clock64();
    if (warp == kIssueWarp) {
        for (int s = 0; s < steps; ++s) {
            if (ss) {
                if (s & 1) k3h_issue_ss<1>(tmem, s0, bars);
                else k3h_issue_ss<0>(tmem, s0, bars);
            } else {
                if (s & 1) k3h_issue<1>(tmem, s0, bars);
                else k3h_issue<0>(tmem, s0, bars);
            }
        }
        mma_commit_warp(bars + 2);
        mbar_wait_sleep(bars + 2, 0);
        if (lane == 0) {
            cyc[blockIdx.x] = clock64() - t0;
            *done = 1;
        }
    } else if (warp < kWorkers) {
        const uint32_t q = warp & 3, g = warp >> 2;
        const uint32_t lb = tmem + ((q * 32) << 16);
        uint32_t it = 0;
        while (!*done) {
            if (mode & 1) {
                uint32_t r[32];
                tmem_ld32(lb + g * 32u, r);
#pragma unroll
                for (int i = 0; i < 32; ++i) acc ^= r[i];
            }
            if (mode & 2) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t a = s0 + ((warp * 512u + lane * 16u + (it & 7u) * 8192u + i * 16384u) & 0x1FFF0u);
                    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(0x3C003C00u + (acc & 1u)) : "memory");
                }
            }
            if (mode & 4) {
                uint32_t p[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) p[i] = 0x3C003C00u ^ (acc & 1u);
                tmem_st8(lb + 256u + 128u + g * 16u + (it & 1u) * 8u, p);
                tmem_st8(lb + 256u + 192u + g * 16u + (it & 1u) * 8u, p);
            }
            ++it;
            if (mode == 0) __nanosleep(200);
            if (mode & 8) __nanosleep(1000);  // ~64 KB of st.shared per ~2000 cycles (the epilogue's rate)
        }
        tmem_st_wait();
    }
    if (acc == 0x12345678u) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == kIssueWarp) tmem_dealloc<512>(tmem);
}
int main() {
    long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 64);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    const int steps = 2000;
    for (int ss = 0; ss < 2; ++ss)
    for (int fill = 1; fill < 2; ++fill)
    for (int mode : {0, 2, 10, 7, 15}) {
        for (int grid : {148}) {
            rate<<<grid, kThreads, kSmem>>>(steps, mode, fill, ss, cyc, sink);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; ++i) avg += h[i];
            avg /= grid;
            printf("%s fill %d mode %d (ld %d sts %d st %d) grid %3d err=%s: %.1f cycles/step = %.1f per MMA\n", ss ? "SS" : "TS", fill, mode, mode & 1,
                   (mode >> 1) & 1, (mode >> 2) & 1, grid, cudaGetErrorString(e), avg / steps, avg / steps / 24);
        }
    }
    return 0;
}
