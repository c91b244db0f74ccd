// Run K3 on the C3 workload with the phase-timer hook and print the split.
#include <cstdio>
#include <cmath>
#include "mxp_internal.h"
#include "../../include/matexpo_b200.h"
int main() {
    mxp_handle h; if (mxp_create(0, &h)) { printf("create failed\n"); return 1; }
    const int n = 128; const long long B = 65536;
    void *din, *dout; long long* prof;
    mxp_alloc(h, B * n * n * 4, &din); mxp_alloc(h, B * n * n * 4, &dout);
    cudaMalloc(&prof, 64); cudaMemset(prof, 0, 64);
    mxp_random_device(h, 0, n, B, 42, -0.5, 0.5, std::sqrt(12.0 / n), din);
    mxp_stats st;
    mxp_power_batched_device(h, 0, n, B, 64, din, dout, &st);
    mxp::k3_set_profile(prof);
    mxp_power_batched_device(h, 0, n, B, 64, din, dout, &st);
    mxp_synchronize(h);
    long long p[3]; cudaMemcpy(p, prof, 24, cudaMemcpyDeviceToHost);
    const double per = 65536.0 / 148;  // matrices per CTA
    printf("CTA0 cycles: load %lld mma %lld epi %lld total %lld\n", p[0], p[1], p[2], p[0] + p[1] + p[2]);
    printf("per matrix: load %.0f  per step: mma %.0f epi %.0f\n", p[0] / per, p[1] / per / 6, p[2] / per / 6);
    return 0;
}
