// K3H event timeline (CTA 0): per publish i of the issuer / epilogue:
//   issuer: bar-sync start, sync done, issue done; epilogue: MMA-done (warp 2),
//   publish time of warps 2, 0, 15.
// Build: nvcc ... -DK3H_EVT tools/k3h_evt.cu kernels_tf32.cu kernels_k3b.cu
#include <cstdio>
#include <vector>
#include "../paper_1204_3052_b200/csrc/kernels_k3h.cu"
using namespace mxp;
int main() {
    const int n = 128; const long long B = 65536;
    PlanBits plan{}; plan.len = 6; plan.squares = 6;
    float *din, *dout; long long* ev;
    cudaMalloc(&din, B * n * n * 4); cudaMalloc(&dout, B * n * n * 4);
    {  // random inputs (zeros would take the exact-scale path every step)
        std::vector<float> hbuf(static_cast<size_t>(B) * n * n);
        uint32_t x = 12345u;
        for (auto& v : hbuf) { x = x * 1664525u + 1013904223u; v = (static_cast<float>(x >> 8) / 16777216.0f - 0.5f) * 0.306f; }
        cudaMemcpy(din, hbuf.data(), hbuf.size() * 4, cudaMemcpyHostToDevice);
    }
    cudaMalloc(&ev, 4096 * 8 * 8); cudaMemset(ev, 0, 4096 * 8 * 8);
    cudaMemcpyToSymbol(g_k3h_evt, &ev, sizeof(ev));
    prepare_k3h_kernel();
    for (int r = 0; r < 3; ++r) launch_k3h_batched(din, dout, n, B, plan, 148, nullptr, 0);
    cudaDeviceSynchronize();
    std::vector<long long> h(4096 * 8);
    cudaMemcpy(h.data(), ev, h.size() * 8, cudaMemcpyDeviceToHost);
    // Note: issuer slots count publishes; epilogue slots count publishes too (same order).
    long long base = h[100 * 8 + 1];
    double gsum = 0, isum = 0, esum = 0, wsum = 0, skew = 0; int cnt = 0;
    for (int i = 100; i < 140; ++i) {
        const long long* r = &h[i * 8];
        const long long* nx = &h[(i + 1) * 8];
        printf("pub %3d: sync-start %7lld done %7lld issued %7lld | mma-done(w2) %7lld publish w2 %7lld w0 %7lld w15 %7lld\n", i,
               r[0] - base, r[1] - base, r[2] - base, r[3] - base, r[4] - base, r[5] - base, r[6] - base);
    }
    for (int i = 100; i < 2000; ++i) {
        const long long* r = &h[i * 8];
        const long long* nx = &h[(i + 1) * 8];
        if (!r[1] || !nx[1] || !r[3]) continue;
        gsum += nx[1] - r[1]; isum += r[2] - r[1]; esum += r[4] - r[3];
        long long mx = std::max(r[4], std::max(r[5], r[6])), mn = std::min(r[4], std::min(r[5], r[6]));
        skew += mx - mn; ++cnt;
    }
    printf("avg over %d publishes: sync->sync %.0f, issue %.0f, epilogue (w2 mma-done -> publish) %.0f, publish skew w0/w2/w15 %.0f\n",
           cnt, gsum / cnt, isum / cnt, esum / cnt, skew / cnt);
    return 0;
}
