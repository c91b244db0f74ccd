// Standalone tcgen05 probe: TMEM st/ld round trip and single-MMA checks.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1204_3052_b200/csrc tools/tc_probe.cu -o tools/tc_probe
#include <cstdio>
#include <cstring>
#include <vector>
#include "ptx.cuh"

using namespace mxp;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// mode 0: TMEM st/ld round trip.  mode 1: A=ones, B=ones, one MMA (K=8).
// mode 2: A[r][k] = r (row id), B = ones -> D[r][j] = 8r.  mode 3: A = ones,
// B[k][j] = j -> D[r][j] = 8j.   Out: 128 x 32 floats (columns 0..31).
__global__ void probe(int mode, float* out, uint32_t idesc, uint32_t lbo_b, uint32_t sbo) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;            // 128 rows x 128 B
    uint8_t* B = smem + 16384;    // 4 chunks x 32 K-rows x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 16384);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 32; i += blockDim.x) {
        const int r = i / 32, c = i % 32;
        float a = (mode == 2) ? float(r) : 1.f;
        *reinterpret_cast<float*>(A + sw128_offset(r, c, 16384)) = a;
    }
    for (int i = tid; i < 32 * 128; i += blockDim.x) {
        const int k = i / 128, j = i % 128;  // B[k][j], MN-major: chunk j/32, row k
        float b = (mode == 3) ? float(j) : 1.f;
        *reinterpret_cast<float*>(B + (j >> 5) * 4096 + k * 128 +
                                  ((((j & 31) >> 2) ^ (k & 7)) << 4) + (j & 3) * 4) = b;
    }
    if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<128>(slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (mode == 0) {
        if (warp < 4) {
            uint32_t v[32];
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(float((warp * 32 + lane) * 1000 + i));
            tmem_st32(tmem + ((warp * 32) << 16), v);
        }
    } else if (tid == 0) {
        tc_fence_after();
        mma_tf32(tmem, sw128_desc(smem_u32(A), 16, sbo), sw128_desc(smem_u32(B), lbo_b, sbo), idesc, 0);
        mma_commit(bar);
    }
    if (mode != 0) mbar_wait(bar, 0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp < 4) {
        uint32_t v[32];
        tmem_ld32(tmem + ((warp * 32) << 16), v);
        for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 32 + i] = __uint_as_float(v[i]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tmem);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 32 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    std::vector<float> h(128 * 32);
    const uint32_t idesc = idesc_tf32_kmaj_mnmaj<128, 128>();
    printf("idesc=0x%08x\n", idesc);
    for (int mode = 0; mode < 4; ++mode) {
        cudaMemset(d, 0xFF, 128 * 32 * 4);
        probe<<<1, 256, 40000>>>(mode, d, idesc, 4096, 1024);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        printf("mode %d err=%s\n", mode, cudaGetErrorString(e));
        for (int r : {0, 1, 2, 33, 127}) {
            printf("  row %3d:", r);
            for (int c : {0, 1, 2, 7, 8, 31}) printf(" %9.1f", h[r * 32 + c]);
            printf("\n");
        }
    }
    return 0;
}
