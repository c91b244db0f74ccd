// Grid-barrier latency among K1C's CTA geometry (128 CTAs of 384 threads,
// clusters of 4, one CTA per SM): ns per barrier for several designs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridbar_probe tools/gridbar_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// 0: every CTA red.release on one counter, thread 0 polls (nanosleep 64)   [product]
// 1: same, no nanosleep
// 2: cluster barrier, leader red on one counter, leader polls, cluster barrier
// 3: per-CTA flags (st.release, no atomics), warp 0 polls all flags
// 4: cluster barrier, leader st.release to its cluster flag, warp 0 of leader polls
//    the cluster flags, cluster barrier
// 5: per-CTA flags, every CTA's warp 0 polls; flags 128 B apart
template <int V>
__global__ void __launch_bounds__(384, 1) bar_kernel(unsigned* ctr, unsigned* flags, int iters,
                                                     unsigned long long* out) {
    const unsigned nctas = gridDim.x * gridDim.y;
    const unsigned cta = blockIdx.x * gridDim.y + blockIdx.y;
    const unsigned nclus = nctas / 4;
    unsigned long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int it = 1; it <= iters; ++it) {
        if (V == 0 || V == 1) {
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                for (;;) {
                    if (ld_acq(ctr) >= nctas * it) break;
                    if (V == 0) __nanosleep(64);
                }
            }
            __syncthreads();
        } else if (V == 2) {
            cluster_sync_all();
            if (cluster_ctarank() == 0 && threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                while (ld_acq(ctr) < nclus * it) {
                }
            }
            cluster_sync_all();
        } else if (V == 3 || V == 5) {
            const int stride = V == 5 ? 32 : 1;
            __syncthreads();
            if (threadIdx.x == 0)
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + cta * stride), "r"((unsigned)it) : "memory");
            if (threadIdx.x < 32) {
                for (;;) {
                    bool ok = true;
                    for (unsigned c = threadIdx.x; c < nctas; c += 32) ok &= ld_acq(flags + c * stride) >= (unsigned)it;
                    if (__all_sync(0xffffffffu, ok)) break;
                }
            }
            __syncthreads();
        } else if (V == 6 || V == 7 || V == 9) {
            // arrival counter + a separate release flag written by the last arriver
            // (6: pollers ld.acquire; 7: ld.relaxed + fence after; 9: as 6 with
            // 16 KB of plane stores per CTA before the barrier, like K1C's reduce)
            if (V == 9) {
                float4* dst = reinterpret_cast<float4*>(flags + 65536) + cta * 1024;
                for (int i = threadIdx.x; i < 1024; i += blockDim.x) dst[i] = make_float4(it, 0, 0, 0);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned old;
                asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
                if (old == nctas * it - 1) {
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags), "r"((unsigned)it) : "memory");
                } else if (V == 7) {
                    unsigned v;
                    do {
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags) : "memory");
                    } while (v < (unsigned)it);
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                } else {
                    while (ld_acq(flags) < (unsigned)it) {
                    }
                }
            }
            __syncthreads();
        } else if (V == 8) {
            // 0 with 16 KB of plane stores per CTA before the barrier
            float4* dst = reinterpret_cast<float4*>(flags + 65536) + cta * 1024;
            for (int i = threadIdx.x; i < 1024; i += blockDim.x) dst[i] = make_float4(it, 0, 0, 0);
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                for (;;) {
                    if (ld_acq(ctr) >= nctas * it) break;
                    __nanosleep(64);
                }
            }
            __syncthreads();
        } else if (V == 4) {
            cluster_sync_all();
            if (cluster_ctarank() == 0 && threadIdx.x < 32) {
                const unsigned clus = cta / 4;
                if (threadIdx.x == 0)
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + clus * 32), "r"((unsigned)it) : "memory");
                for (;;) {
                    bool ok = true;
                    for (unsigned c = threadIdx.x; c < nclus; c += 32) ok &= ld_acq(flags + c * 32) >= (unsigned)it;
                    if (__all_sync(0xffffffffu, ok)) break;
                }
            }
            cluster_sync_all();
        }
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0 && cta == 0) out[0] = t1 - t0;
}

template <int V>
void run(int nx, int iters) {
    unsigned *ctr, *flags;
    unsigned long long* out;
    cudaMalloc(&ctr, 4);
    cudaMalloc(&flags, 65536 * 4 + 256 * 1024 * 16);
    cudaMalloc(&out, 8);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(ctr, 0, 4);
        cudaMemset(flags, 0, 65536 * 4);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nx, 4);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 1;
        a[0].val.clusterDim.y = 4;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, bar_kernel<V>, ctr, flags, iters, out);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("V%d error %s\n", V, cudaGetErrorString(e));
            return;
        }
        unsigned long long ns;
        cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
        best = fminf(best, (float)ns / iters);
    }
    printf("variant %d  ctas %d: %.0f ns per barrier\n", V, nx * 4, best);
    cudaFree(ctr);
    cudaFree(flags);
    cudaFree(out);
}

int main() {
    cudaFuncSetAttribute(bar_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(bar_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(bar_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(bar_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(bar_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(bar_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int v = 6; v <= 9; ++v) {
        void* f = v == 6 ? (void*)bar_kernel<6> : v == 7 ? (void*)bar_kernel<7> : v == 8 ? (void*)bar_kernel<8> : (void*)bar_kernel<9>;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    for (int nx : {8, 32}) {
        run<0>(nx, 2000);
        run<1>(nx, 2000);
        run<2>(nx, 2000);
        run<3>(nx, 2000);
        run<4>(nx, 2000);
        run<5>(nx, 2000);
        run<6>(nx, 2000);
        run<7>(nx, 2000);
        run<8>(nx, 2000);
        run<9>(nx, 2000);
    }
    return 0;
}
