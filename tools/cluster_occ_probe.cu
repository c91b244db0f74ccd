// How many clusters of 2 / 4 / 8 CTAs (K1P's 193 KB SMEM, 384 threads, 1 CTA per SM)
// the B200 can hold at once: cudaOccupancyMaxActiveClusters.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* p) { extern __shared__ int s[]; if (p) p[0] = s[threadIdx.x]; }
int main() {
    const int smem = 3 * 65536 + 1024 + 256;
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(c * 64);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d SMs busy (%s)\n", c, n, n * c,
               cudaGetErrorString(e));
    }
}
