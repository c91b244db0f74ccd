// K1C per-step phase timeline of CTA (0, 0), epilogue warp 4 (cycles):
//   0 step start, 1 last chunk drained, 2 partial in SMEM, 3 after cluster
//   sync, 4 reduce written, 5 after cluster sync, 6 after the grid barrier's
//   (non-blocking, deferred) BAR.SYNC, 7 end of the step: 6 -> 7 is where the
//   grid barrier's wait actually lands.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DK1C_TRACE
//   -I paper_1204_3052_b200/csrc tools/k1c_trace.cu paper_1204_3052_b200/csrc/kernels_k3b.cu
//   paper_1204_3052_b200/csrc/kernels_k3h.cu -o k1c_trace -lcuda
#include <cstdio>
#include <vector>
#include <algorithm>
#include <climits>
#include "../paper_1204_3052_b200/csrc/kernels_tf32.cu"
using namespace mxp;
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 512, np = (n + 127) / 128 * 128;
    PlanBits plan{};
    plan.len = 14; plan.squares = 9;  // k = 1000: S M S M S M S M S S M S S S
    const char* pat = "SMSMSMSMSSMSSS";
    for (int i = 0; i < 14; ++i) if (pat[i] == 'M') plan.mult[0] |= 1ull << i;
    prepare_tf32_kernels();
    float *a, *out; uint32_t* planes[6]; unsigned int* ctr; long long* tr;
    cudaMalloc(&a, n * n * 4); cudaMalloc(&out, n * n * 4); cudaMalloc(&ctr, 256); cudaMemset(ctr, 0, 256);
    cudaMalloc(&tr, 64 * 16 * 8); cudaMemset(tr, 0, 64 * 16 * 8);
    cudaMemcpyToSymbol(g_k1c_trace, &tr, sizeof(tr));
    long long* gtr;
    cudaMalloc(&gtr, 64 * 256 * 4 * 8);
    cudaMemset(gtr, 0, 64 * 256 * 4 * 8);
    cudaMemcpyToSymbol(g_k1c_gtrace, &gtr, sizeof(gtr));
    std::vector<float> h(n * n);
    uint32_t x = 1;
    for (auto& v : h) { x = x * 1664525u + 1013904223u; v = ((x >> 8) / 16777216.0f - 0.5f) * 0.153f; }
    cudaMemcpy(a, h.data(), n * n * 4, cudaMemcpyHostToDevice);
    CUtensorMap ma[6], mb[6];
    for (int i = 0; i < 6; ++i) {
        cudaMalloc(&planes[i], (size_t)np * np * 4);
        encode_plane_map(&ma[i], planes[i], np, 32, 128, false);
        encode_plane_map(&mb[i], planes[i], np, 32, 32, true);
    }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int splits = k1_split_k(np, np, sms);
    for (int r = 0; r < 3; ++r) {
        launch_split(a, n, n, planes[0], planes[1], np, 0);
        cudaError_t e = launch_k1c_chain(ma, mb, planes, plan, np, splits, out, n, ctr, nullptr, -1, 0);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch_k1c_chain(ma, mb, planes, plan, np, splits, out, n, ctr, nullptr, -1, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("n=%d splits=%d err=%s chain %.1f us (%.2f us/step)\n", n, splits, cudaGetErrorString(e), ms * 1e3, ms * 1e3 / 14);
    std::vector<long long> t(64 * 16);
    cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
    printf("step: mainloop | partial | csync1 | reduce | csync2 | grid bar | (6->7) (7->next 0) | total || tma issue, kb0..3 landed (from step start)\n");
    for (int s = 0; s < 14; ++s) {
        const long long* r = &t[s * 16];
        printf("%2d %c: %6lld %6lld %6lld %6lld %6lld %6lld | %6lld %6lld | %6lld || %6lld %6lld %6lld %6lld %6lld\n", s, pat[s], r[1] - r[0], r[2] - r[1], r[3] - r[2],
               r[4] - r[3], r[5] - r[4], s < 13 ? r[6] - r[5] : 0, r[7] - r[6], s < 13 ? t[(s + 1) * 16] - r[7] : 0,
               s < 13 ? t[(s + 1) * 16] - r[0] : r[5] - r[0], r[8] - r[0], r[9] - r[0], r[10] - r[0], r[11] - r[0], r[12] - r[0]);
    }
    // every CTA (globaltimer, ns): spread of the step phases across the grid
    const int nctas = 2 * (np / 128) * (np / 128) * splits;  // 64-column K1C tiles
    std::vector<long long> g(64 * 256 * 4);
    cudaMemcpy(g.data(), gtr, g.size() * 8, cudaMemcpyDeviceToHost);
    printf("\nall %d CTAs (ns from the earliest step start): start min/max | mainloop done min/med/max | reduce done min/max | after barrier min/max   [slowest mainloop CTA]\n", nctas);
    for (int s = 0; s < 14; ++s) {
        std::vector<long long> v[4];
        long long t0 = LLONG_MAX;
        int slow = 0; long long slowv = 0;
        for (int c = 0; c < nctas; ++c) {
            for (int k = 0; k < 4; ++k) v[k].push_back(g[(s * nctas + c) * 4 + k]);
            t0 = std::min(t0, g[(s * nctas + c) * 4 + 0]);
            if (g[(s * nctas + c) * 4 + 1] > slowv) { slowv = g[(s * nctas + c) * 4 + 1]; slow = c; }
        }
        for (auto& x : v) std::sort(x.begin(), x.end());
        auto r = [&](int k, int i) { return v[k][i] - t0; };
        printf("%2d: %5lld %5lld | %5lld %5lld %5lld | %5lld %5lld | %5lld %5lld   [cta %d]\n", s, r(0, 0), r(0, nctas - 1),
               r(1, 0), r(1, nctas / 2), r(1, nctas - 1), r(2, 0), r(2, nctas - 1), r(3, 0), r(3, nctas - 1), slow);
    }
    return 0;
}
