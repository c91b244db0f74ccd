// K3B phase profile (CTA 0): cycle totals of epilogue warp 0 / the issue warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DK3B_TRACE
//   -I paper_1204_3052_b200/csrc tools/k3b_trace.cu -o tools/k3b_trace -lcuda
#include <cstdio>
#include <vector>
#include "../paper_1204_3052_b200/csrc/kernels_k3b.cu"
using namespace mxp;
int main(int argc, char** argv) {
    const int n = 128;
    const long long B = argc > 1 ? atoll(argv[1]) : 65536;
    PlanBits plan{};
    plan.len = 6; plan.squares = 6;  // k = 64
    float *din, *dout; long long* tr;
    cudaMalloc(&din, B * n * n * 4); cudaMalloc(&dout, B * n * n * 4);
    cudaMalloc(&tr, 16 * 8); cudaMemset(tr, 0, 16 * 8);
    cudaMemset(din, 0, B * n * n * 4);
    cudaMemcpyToSymbol(g_k3b_trace, &tr, sizeof(tr));
    prepare_k3b_kernel();
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int r = 0; r < 2; ++r) launch_k3b_batched(din, dout, n, B, plan, sms, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch_k3b_batched(din, dout, n, B, plan, sms, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[16];
    cudaMemcpy(h, tr, sizeof h, cudaMemcpyDeviceToHost);
    printf("err=%s  %.3f ms\n", cudaGetErrorString(e), ms);
    const char* nm[11] = {"E wait mma", "E tmem drain", "E IO out tile+STG", "E IO LDG+tile put", "E IO tile get+bar",
                          "E IO emit", "E step emit", "E publish+loop", "I bar.sync wait", "I issue", "I loop"};
    long long tot_e = 0, tot_i = 0;
    for (int i = 0; i < 8; ++i) tot_e += h[i];
    for (int i = 8; i < 11; ++i) tot_i += h[i];
    for (int i = 0; i < 11; ++i)
        printf("%-20s %10lld cycles  %5.1f%%\n", nm[i], h[i], 100.0 * h[i] / (i < 8 ? tot_e : tot_i));
    printf("IO steps %lld, normal steps %lld; per IO step: out %.0f ldg %.0f bar %.0f emit %.0f; per normal step emit %.0f\n",
           h[11], h[12], double(h[2]) / h[11], double(h[3]) / h[11], double(h[4]) / h[11], double(h[5]) / h[11], double(h[6]) / h[12]);
    printf("IO out split: tile st.shared %.0f, fence+syncwarp %.0f, TMA store+wait read %.0f\n", double(h[13]) / h[11], double(h[14]) / h[11], double(h[2]) / h[11]);
    printf("per slot (E total / slots) %.0f, issue per step %.0f\n", double(tot_e) / (h[11] + h[12]), double(h[9]) / (h[11] + h[12]));
    return 0;
}
