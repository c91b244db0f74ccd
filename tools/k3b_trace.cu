// K3B slot timeline (CTA 0): per slot, each epilogue warp's MMA-wait start /
// end and publish time, the issue warp's barrier-release and issue-done time.
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
    const size_t slots = 1 << 14;
    cudaMalloc(&tr, slots * 64 * 8); cudaMemset(tr, 0, slots * 64 * 8);
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
    std::vector<long long> h(slots * 64);
    cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
    printf("err=%s  %.3f ms\n", cudaGetErrorString(e), ms);
    int ns = 0;
    while (ns < (int)slots && h[ns * 64 + 48] != 0) ++ns;
    printf("slots %d\n", ns);
    // per-slot: issue(i) -> next issue; epilogue span: max wait-done -> max arrive
    double sum_gap = 0, sum_epi = 0, sum_issue = 0, sum_spread = 0, sum_wait_first = 0; int cnt = 0;
    for (int i = 8; i + 1 < ns && i < 8 + 400; ++i) {
        const long long* r = &h[i * 64];
        long long wd_min = 1LL << 62, wd_max = 0, ar_max = 0, ar_min = 1LL << 62;
        for (int w = 0; w < 16; ++w) {
            if (r[16 + w]) { wd_min = std::min(wd_min, r[16 + w]); wd_max = std::max(wd_max, r[16 + w]); }
            ar_max = std::max(ar_max, r[32 + w]); ar_min = std::min(ar_min, r[32 + w]);
        }
        sum_gap += h[(i + 1) * 64 + 48] - r[48];
        sum_issue += r[49] - r[48];
        if (wd_max) { sum_epi += ar_max - wd_max; sum_spread += ar_max - ar_min; sum_wait_first += wd_max - wd_min; }
        ++cnt;
        if (i < 20)
            printf("slot %3d: sync %lld issue %lld | wait-done spread %lld | epi(max wd->max arrive) %lld | arrive spread %lld | gap to next sync %lld\n",
                   i, r[48] - h[8 * 64 + 48], r[49] - r[48], wd_max ? wd_max - wd_min : -1,
                   wd_max ? ar_max - wd_max : -1, ar_max - ar_min, h[(i + 1) * 64 + 48] - r[48]);
    }
    // raw timeline, slots 40..64: publish i's epilogue saw its MMA completion at wd(i)
    long long base = h[40 * 64 + 48];
    for (int i = 40; i < 64 && i < ns; ++i) {
        const long long* r = &h[i * 64];
        long long wd = 1LL << 62, wdx = 0, ar = 0, ws = 1LL << 62;
        for (int w = 0; w < 16; ++w) {
            if (r[16 + w]) { wd = std::min(wd, r[16 + w]); wdx = std::max(wdx, r[16 + w]); }
            if (r[w]) ws = std::min(ws, r[w]);
            ar = std::max(ar, r[32 + w]);
        }
        printf("pub %2d: wait-start %7lld  mma-done(seen) %7lld..%7lld  arrive-max %7lld  sync %7lld  issued %7lld\n", i,
               ws == (1LL << 62) ? -1 : ws - base, wd == (1LL << 62) ? -1 : wd - base, wdx - base, ar - base, r[48] - base, r[49] - base);
    }
    printf("avg over %d slots: sync->sync %.0f  issue %.0f  epilogue %.0f  arrive spread %.0f  wait-done spread %.0f\n",
           cnt, sum_gap / cnt, sum_issue / cnt, sum_epi / cnt, sum_spread / cnt, sum_wait_first / cnt);
    return 0;
}
