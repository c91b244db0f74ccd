// Probe variants of a single tcgen05.mma with all-ones operands.
#include <cstdio>
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
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_tf32_mask(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5,%5,%5,%5}, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0) : "memory");
}

__global__ void probe(int kind, uint32_t fill, uint64_t adesc_hi, uint64_t bdesc_hi, uint32_t lbo_a, uint32_t lbo_b,
                      uint32_t idesc, int prestore, int acc, float* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = fill;
    if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<256>(slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot;
    if (prestore && warp < 4) {
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(100.f);
        tmem_st32(tmem + ((warp * 32) << 16), v);
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (tid == 0) {
        uint64_t a = (uint64_t(smem_u32(smem)) >> 4) | (uint64_t(lbo_a >> 4) << 16) | adesc_hi;
        uint64_t b = (uint64_t(smem_u32(smem + 32768)) >> 4) | (uint64_t(lbo_b >> 4) << 16) | bdesc_hi;
        if (kind == 0) mma_tf32(tmem, a, b, idesc, acc);
        else if (kind == 1) mma_f16(tmem, a, b, idesc, acc);
        else mma_tf32_mask(tmem, a, b, idesc, acc);
        mma_commit(bar);
    }
    mbar_wait(bar, 0);
    tc_fence_after();
    if (warp < 4) {
        uint32_t v[32];
        tmem_ld32(tmem + ((warp * 32) << 16), v);
        for (int i = 0; i < 4; ++i) out[(warp * 32 + lane) * 4 + i] = __uint_as_float(v[i * 8]);
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tmem);
}

int main() {
    float* d; cudaMalloc(&d, 128 * 4 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    std::vector<float> h(128 * 4);
    auto hi = [](uint64_t sbo, uint64_t ver, uint64_t layout) {
        return ((sbo >> 4) << 32) | (ver << 46) | (layout << 61);
    };
    const uint32_t tf32_mn = idesc_tf32_kmaj_mnmaj<128, 128>();
    const uint32_t tf32_kk = tf32_mn & ~(1u << 16);
    const uint32_t bf16_kk = (1u << 4) | (1u << 7) | (1u << 10) | (16u << 17) | (8u << 24);
    struct V { const char* name; int kind; uint32_t fill; uint64_t ah, bh; uint32_t la, lb, idesc; int pre, acc; };
    V vs[] = {
        {"tf32 sw128 mn acc0", 0, 0x3F800000u, hi(1024,1,2), hi(1024,1,2), 16, 4096, tf32_mn, 0, 0},
        {"tf32 sw128 mn pre acc1", 0, 0x3F800000u, hi(1024,1,2), hi(1024,1,2), 16, 4096, tf32_mn, 1, 1},
        {"tf32 sw128 kk acc0", 0, 0x3F800000u, hi(1024,1,2), hi(1024,1,2), 16, 16, tf32_kk, 0, 0},
        {"tf32 none kk acc0", 0, 0x3F800000u, hi(256,1,0), hi(256,1,0), 128, 128, tf32_kk, 0, 0},
        {"tf32 none kk ver0", 0, 0x3F800000u, hi(256,0,0), hi(256,0,0), 128, 128, tf32_kk, 0, 0},
        {"tf32 mask sw128 mn", 2, 0x3F800000u, hi(1024,1,2), hi(1024,1,2), 16, 4096, tf32_mn, 0, 0},
        {"bf16 sw128 kk acc0", 1, 0x3F803F80u, hi(1024,1,2), hi(1024,1,2), 16, 16, bf16_kk, 0, 0},
        {"bf16 none kk acc0", 1, 0x3F803F80u, hi(256,1,0), hi(256,1,0), 128, 128, bf16_kk, 0, 0},
        {"bf16 sw128 kk pre acc1", 1, 0x3F803F80u, hi(1024,1,2), hi(1024,1,2), 16, 16, bf16_kk, 1, 1},
    };
    for (auto& v : vs) {
        cudaMemset(d, 0xFF, 128 * 16);
        probe<<<1, 256, 70000>>>(v.kind, v.fill, v.ah, v.bh, v.la, v.lb, v.idesc, v.pre, v.acc, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        printf("%-26s idesc=%08x err=%s | r0: %g %g %g %g | r1 %g r64 %g r127 %g\n", v.name, v.idesc,
               cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[64 * 4], h[127 * 4]);
    }
    return 0;
}
