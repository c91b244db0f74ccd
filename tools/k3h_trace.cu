// K3H phase profile (CTA 0): cycle totals of epilogue warp 0 / the issue warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DK3H_TRACE
//   -I paper_1204_3052_b200/csrc tools/k3h_trace.cu -o tools/k3h_trace -lcuda
#include <cstdio>
#include <vector>
#include "../paper_1204_3052_b200/csrc/kernels_k3h.cu"
using namespace mxp;
int main(int argc, char** argv) {
    const int n = 128;
    const long long B = argc > 1 ? atoll(argv[1]) : 65536;
    PlanBits plan{};
    plan.len = 6; plan.squares = 6;  // k = 64
    float *din, *dout; long long* tr;
    cudaMalloc(&din, B * n * n * 4); cudaMalloc(&dout, B * n * n * 4);
    cudaMalloc(&tr, 16 * 8); cudaMemset(tr, 0, 16 * 8);
    {  // random inputs (zeros would take the exact-scale path every step)
        std::vector<float> hbuf(static_cast<size_t>(B) * n * n);
        uint32_t x = 12345u;
        for (auto& v : hbuf) { x = x * 1664525u + 1013904223u; v = (static_cast<float>(x >> 8) / 16777216.0f - 0.5f) * 0.306f; }
        cudaMemcpy(din, hbuf.data(), hbuf.size() * 4, cudaMemcpyHostToDevice);
    }
    cudaMemcpyToSymbol(g_k3h_trace, &tr, sizeof(tr));
    prepare_k3h_kernel();
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int r = 0; r < 2; ++r) launch_k3h_batched(din, dout, n, B, plan, sms, nullptr, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch_k3h_batched(din, dout, n, B, plan, sms, nullptr, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[16];
    cudaMemcpy(h, tr, sizeof h, cudaMemcpyDeviceToHost);
    printf("err=%s  %.3f ms\n", cudaGetErrorString(e), ms);
    const char* nm[12] = {"E wait mma", "E tmem drain", "E OUT scale+tile", "E IN wait input", "E IN get+max+bar",
                          "E IN emit", "E step emit", "E publish+loop", "I bar.sync wait", "I issue", "I loop", "E step max+bar"};
    long long tot_e = 0, tot_i = 0;
    for (int i = 0; i < 8; ++i) tot_e += h[i];
    tot_e += h[11];
    for (int i = 8; i < 11; ++i) tot_i += h[i];
    for (int i = 0; i < 12; ++i)
        printf("%-20s %10lld cycles  %5.1f%%\n", nm[i], h[i], 100.0 * h[i] / ((i < 8 || i == 11) ? tot_e : tot_i));
    printf("IN steps %lld, normal steps %lld; per normal step: wait %.0f drain %.0f max+bar %.0f emit %.0f publish %.0f; issue per step %.0f (%.1f/MMA) bar wait %.0f loop %.0f\n",
           h[13], h[14], double(h[0]) / (h[13] + h[14]), double(h[1]) / (h[13] + h[14]), double(h[11]) / h[14], double(h[6]) / h[14],
           double(h[7]) / (h[13] + h[14]), double(h[9]) / (h[13] + h[14]), double(h[9]) / (h[13] + h[14]) / 24.0,
           double(h[8]) / (h[13] + h[14]), double(h[10]) / (h[13] + h[14]));
    printf("per IN step: wait input %.0f, get+max+bar %.0f, emit %.0f; OUT scale+tile %.0f\n", double(h[3]) / h[13], double(h[4]) / h[13], double(h[5]) / h[13], double(h[2]) / h[13]);
    return 0;
}
