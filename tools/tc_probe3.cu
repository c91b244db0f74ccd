// Layout probe: host-built shared-memory images, one tcgen05.mma (K=8 tf32),
// D (128 x 128) compared with the host-expected product.
#include <cstdio>
#include <cstring>
#include <functional>
#include <vector>
#include "ptx.cuh"
using namespace mxp;

__device__ __forceinline__ void probe_tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
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
__device__ __forceinline__ void probe_mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// img: 64 KB smem image (A at 0, B at 16384).  atm: A for TMEM, [128][32] words (used if ts).
__global__ void probe(const uint4* img, const uint32_t* atm, int ts, uint64_t adesc_rest, uint64_t bdesc_rest,
                      uint32_t idesc, float* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = img[i];
    if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<512>(slot);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *slot;
    if (ts && warp < 4) {
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = atm[(warp * 32 + lane) * 32 + i];
        probe_tmem_st32(tmem + ((warp * 32) << 16) + 256, v);
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (tid == 0) {
        uint64_t a = (uint64_t(smem_u32(smem)) >> 4) | adesc_rest;
        uint64_t b = (uint64_t(smem_u32(smem + 16384)) >> 4) | bdesc_rest;
        if (ts) probe_mma_tf32_ts(tmem, tmem + 256, b, idesc, 0);
        else mma_tf32(tmem, a, b, idesc, 0);
        mma_commit(bar);
    }
    mbar_wait(bar, 0);
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

static uint64_t rest(uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) | (1ull << 46) | (uint64_t(layout) << 61);
}
static void putf(std::vector<uint8_t>& img, size_t off, float v) { memcpy(&img[off], &v, 4); }

int main() {
    uint4* dimg; uint32_t* datm; float* dout;
    cudaMalloc(&dimg, 65536); cudaMalloc(&datm, 128 * 32 * 4); cudaMalloc(&dout, 128 * 128 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    const uint32_t id_mn = idesc_tf32_kmaj_mnmaj<128, 128>();
    const uint32_t id_kk = id_mn & ~(1u << 16);
    // A (128 x 8 used), K-major SW128: A[m][k] at m*128 + ((k/4) ^ (m%8))*16 + (k%4)*4
    auto aval = [](int m, int k) { return (m == k) ? 1.f : 0.f; };  // identity in rows 0..7
    auto bval = [](int k, int n) { return float(1000 * k + n); };
    auto expect = [&](int m, int n) { float s = 0; for (int k = 0; k < 8; ++k) s += aval(m, k) * bval(k, n); return s; };

    struct Case { const char* name; std::function<size_t(int k, int n)> boff; uint64_t brest; uint32_t idesc; int ts; };
    // B MN-major: element (k, n) in chunk n/32 (stride LBO) ...
    const uint32_t LBO = 4096;
    std::vector<Case> cases = {
        {"MN sw128_32B swz(k%4) sbo512", [&](int k, int n) { return size_t((n / 32) * LBO + k * 128 + ((((n % 32) / 8) ^ (k % 4)) * 32) + (n % 8) * 4); },
         rest(LBO, 512, 1), id_mn, 0},
        {"MN sw128_32B swz((k%8)/2) sbo512", [&](int k, int n) { return size_t((n / 32) * LBO + k * 128 + ((((n % 32) / 8) ^ ((k % 8) / 2)) * 32) + (n % 8) * 4); },
         rest(LBO, 512, 1), id_mn, 0},
        {"MN sw128_32B swz(k%4) sbo1024", [&](int k, int n) { return size_t((n / 32) * LBO + k * 128 + ((((n % 32) / 8) ^ (k % 4)) * 32) + (n % 8) * 4); },
         rest(LBO, 1024, 1), id_mn, 0},
        {"MN none", [&](int k, int n) { return size_t((n / 4) * 128 + k * 16 + (n % 4) * 4); },  // ((T,1,m),(8,k)):((1,T,SBO),(1T,LBO)) guess
         rest(128, 128, 0), id_mn, 0},
        {"KK sw128 (B^T)", [&](int k, int n) { return size_t((n) * 128 + (((k / 4) ^ (n % 8)) * 16) + (k % 4) * 4); },
         rest(16, 1024, 2), id_kk, 0},
        {"TS: A tmem, B KK sw128", [&](int k, int n) { return size_t((n) * 128 + (((k / 4) ^ (n % 8)) * 16) + (k % 4) * 4); },
         rest(16, 1024, 2), id_kk, 1},
        {"TS: A tmem, B MN sw128_32B swz(k%4)", [&](int k, int n) { return size_t((n / 32) * LBO + k * 128 + ((((n % 32) / 8) ^ (k % 4)) * 32) + (n % 8) * 4); },
         rest(LBO, 512, 1), id_mn, 1},
    };
    std::vector<float> h(128 * 128);
    std::vector<uint32_t> atm(128 * 32, 0);
    for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) { float v = aval(m, k); memcpy(&atm[m * 32 + k], &v, 4); }
    cudaMemcpy(datm, atm.data(), atm.size() * 4, cudaMemcpyHostToDevice);
    for (auto& c : cases) {
        std::vector<uint8_t> img(65536, 0);
        for (int m = 0; m < 128; ++m)
            for (int k = 0; k < 8; ++k) putf(img, m * 128 + (((k / 4) ^ (m % 8)) * 16) + (k % 4) * 4, aval(m, k));
        for (int k = 0; k < 8; ++k)
            for (int n = 0; n < 128; ++n) putf(img, 16384 + c.boff(k, n), bval(k, n));
        cudaMemcpy(dimg, img.data(), 65536, cudaMemcpyHostToDevice);
        cudaMemset(dout, 0xFF, 128 * 128 * 4);
        probe<<<1, 256, 70000>>>(dimg, datm, c.ts, rest(16, 1024, 2), c.brest, c.idesc, dout);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h.data(), dout, h.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0; int first = -1;
        for (int m = 0; m < 128; ++m) for (int n = 0; n < 128; ++n)
            if (h[m * 128 + n] != expect(m, n)) { if (first < 0) first = m * 128 + n; ++bad; }
        printf("%-40s err=%s bad=%d", c.name, cudaGetErrorString(e), bad);
        if (first >= 0) printf(" first (m=%d,n=%d) got %g want %g | row1: %g %g %g %g %g", first / 128, first % 128, h[first], expect(first / 128, first % 128),
                               h[128], h[129], h[130], h[131], h[132]);
        printf("\n");
    }
    return 0;
}
