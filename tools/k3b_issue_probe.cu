// Rate of the exact K3B step issue sequence (k3b_issue<C, MULT>) with no
// epilogue: one CTA per SM, `steps` back-to-back steps per CTA.
#include <cstdio>
#include "../paper_1204_3052_b200/csrc/kernels_k3b.cu"
using namespace mxp;
template <int kMode>
__global__ void __launch_bounds__(128, 1) issue_rate(int steps, long long* cyc, int fill) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (int)(kBarOff / 16); i += blockDim.x) {
        uint32_t x = (i * 2654435761u) ^ 0x9E3779B9u; x ^= x >> 13; x *= 0x85EBCA6Bu; x ^= x >> 16;
        // fill 0: zeros; 1: random bf16 in [-1, 1) (exponent kept sane); 2: raw random bits
        uint32_t w = fill == 0 ? 0u : (fill == 1 ? ((x & 0x807F807Fu) | 0x3F003F00u) : x);
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(w, w * 3u + 1u, w ^ 0x12345678u, w + 7u);
        if (fill == 1) { uint4& q = reinterpret_cast<uint4*>(smem)[i]; q.y = (q.y & 0x807F807Fu) | 0x3F003F00u; q.z = (q.z & 0x807F807Fu) | 0x3F003F00u; q.w = (q.w & 0x807F807Fu) | 0x3F003F00u; }
    }
    if (tid == 0) { mbar_init(bars, 1); mbar_init(bars + 1, 1); mbar_init(bars + 2, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot, s0 = smem_u32(smem);
    long long t0 = clock64();
    if (warp == 0) {
        for (int s = 0; s < steps; ++s) {
            if (threadIdx.x == 0) {
                if (kMode == 0) k3b_issue<0, false>(tmem, s0, bars, bars + 2);
                else { if (s & 1) k3b_issue<1, false>(tmem, s0, bars, bars + 2); else k3b_issue<0, false>(tmem, s0, bars, bars + 2); }
            }
            __syncwarp();
        }
        if (threadIdx.x == 0) mma_commit(bars + 2);
        mbar_wait(bars + 2, 0);
        if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = clock64() - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
int main() {
    long long* d; cudaMalloc(&d, 8);
    cudaFuncSetAttribute(issue_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    cudaFuncSetAttribute(issue_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    for (int fill = 0; fill < 2; ++fill)
    for (int mode = 0; mode < 2; ++mode)
        for (int grid : {1, 148}) {
            long long h = 0;
            printf("fill %d ", fill);
            if (mode == 0) issue_rate<0><<<grid, 128, kSmem>>>(2000, d, fill); else issue_rate<1><<<grid, 128, kSmem>>>(2000, d, fill);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("mode %d grid %3d err=%s: %.1f cycles/step (48 MMAs) = %.1f per MMA\n", mode, grid, cudaGetErrorString(e), h / 2000.0, h / 2000.0 / 48);
        }
    return 0;
}
