// FP64 GEMM on the sm_100a DMMA tensor pipe (mma.sync .f64 -> DMMA.8x8x4).
//
// tcgen05 has no kind::f64, so the FP64 mode uses warp-level DMMA fed by a
// cp.async double-buffered shared-memory pipeline.  Replaces the reference's
// F64 matmul_naive (linalg.py:151-164) on the hot path; parity is by the
// relative-Frobenius tolerance (FMA + tensor-core order differ from the
// reference's separately rounded ascending-k loop).
//
// Block tile 128 x 64, BK = 32 (16 was 3% slower: twice the barriers), 8 warps
// as 4 (M) x 2 (N), warp tile 32 x 32
// = 2 x 4 m16n8k4 fragments.  Operands are zero-padded to a multiple of 128.
#include "mxp_internal.h"

namespace mxp {

namespace {
constexpr int BM = 128, BN = 64, BK = 32;
constexpr int A_LD = BK + 4;   // 36 doubles: 288 B row stride -> conflict-free fragment loads
constexpr int B_LD = BN + 8;   // 72 doubles: 576 B row stride
constexpr int kThreads = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}
}  // namespace

__global__ void __launch_bounds__(kThreads, 2)
    f64_gemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                    double* __restrict__ C, int n) {
    extern __shared__ __align__(16) double f64_smem[];
    double (*sA)[BM * A_LD] = reinterpret_cast<double (*)[BM * A_LD]>(f64_smem);
    double (*sB)[BK * B_LD] = reinterpret_cast<double (*)[BK * B_LD]>(f64_smem + 2 * BM * A_LD);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp >> 1, wn = warp & 1;  // 4 x 2 warps
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

    auto load_stage = [&](int stage, int k0) {
        // A: 128 x BK doubles = 128 * BK / 2 x 16 B
#pragma unroll
        for (int i = 0; i < BM * BK / 2 / kThreads; ++i) {
            const int idx = tid + i * kThreads;
            const int r = idx / (BK / 2), c2 = (idx % (BK / 2)) * 2;
            cp_async16(&sA[stage][r * A_LD + c2], A + static_cast<size_t>(m0 + r) * n + k0 + c2);
        }
        // B: BK x 64 doubles = BK * 32 x 16 B
#pragma unroll
        for (int i = 0; i < BK * 32 / kThreads; ++i) {
            const int idx = tid + i * kThreads;
            const int r = idx >> 5, c2 = (idx & 31) * 2;
            cp_async16(&sB[stage][r * B_LD + c2], B + static_cast<size_t>(k0 + r) * n + n0 + c2);
        }
        cp_async_commit();
    };

    double acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

    const int nk = n / BK;
    load_stage(0, 0);
    for (int kt = 0; kt < nk; ++kt) {
        const int st = kt & 1;
        if (kt + 1 < nk) {
            load_stage(st ^ 1, (kt + 1) * BK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* a = sA[st];
        const double* b = sB[st];
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[2][2], bf[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int r = wm * 32 + i * 16 + (lane >> 2);
                af[i][0] = a[r * A_LD + kk + (lane & 3)];
                af[i][1] = a[(r + 8) * A_LD + kk + (lane & 3)];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                bf[j] = b[(kk + (lane & 3)) * B_LD + wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_16x8x4(acc[i][j], af[i][0], af[i][1], bf[j]);
        }
        __syncthreads();
    }
    // c0,c1: row lane/4, cols 2*(lane%4)+{0,1}; c2,c3: row +8
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = m0 + wm * 32 + i * 16 + (lane >> 2);
            const int c = n0 + wn * 32 + j * 8 + 2 * (lane & 3);
            *reinterpret_cast<double2*>(C + static_cast<size_t>(r) * n + c) =
                make_double2(acc[i][j][0], acc[i][j][1]);
            *reinterpret_cast<double2*>(C + static_cast<size_t>(r + 8) * n + c) =
                make_double2(acc[i][j][2], acc[i][j][3]);
        }
}

int f64_pad(int n) { return (n + 127) / 128 * 128; }

namespace {
constexpr int kF64Smem = (2 * BM * A_LD + 2 * BK * B_LD) * sizeof(double);
}

cudaError_t prepare_f64_kernels() {
    return cudaFuncSetAttribute(f64_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kF64Smem);
}

cudaError_t launch_f64_gemm(const double* a, const double* b, double* c, int n, cudaStream_t s) {
    return launch_f64_gemm_rows(a, b, c, n, n, s);
}

cudaError_t launch_f64_gemm_rows(const double* a, const double* b, double* c, int n, int m,
                                 cudaStream_t s) {
    constexpr int kSmem = kF64Smem;
    dim3 grid(n / BN, m / BM);
    f64_gemm_kernel<<<grid, kThreads, kSmem, s>>>(a, b, c, n);
    return cudaGetLastError();
}

__global__ void f64_pad_kernel(const double* __restrict__ in, int n, int rows,
                               double* __restrict__ out, int n_pad, int rows_pad) {
    const size_t total = static_cast<size_t>(rows_pad) * n_pad;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / n_pad), c = static_cast<int>(i % n_pad);
        out[i] = (r < rows && c < n) ? in[static_cast<size_t>(r) * n + c] : 0.0;
    }
}
__global__ void f64_unpad_kernel(const double* __restrict__ in, int n_pad, double* __restrict__ out,
                                 int n, int rows) {
    const size_t total = static_cast<size_t>(rows) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / n), c = static_cast<int>(i % n);
        out[i] = in[static_cast<size_t>(r) * n_pad + c];
    }
}
cudaError_t launch_f64_pad(const double* in, int n, double* out, int n_pad, cudaStream_t s) {
    return launch_f64_pad_rows(in, n, n, out, n_pad, n_pad, s);
}
cudaError_t launch_f64_unpad(const double* in, int n_pad, double* out, int n, cudaStream_t s) {
    return launch_f64_unpad_rows(in, n_pad, out, n, n, s);
}
cudaError_t launch_f64_pad_rows(const double* in, int n, int rows, double* out, int n_pad,
                                int rows_pad, cudaStream_t s) {
    f64_pad_kernel<<<148 * 8, 256, 0, s>>>(in, n, rows, out, n_pad, rows_pad);
    return cudaGetLastError();
}
cudaError_t launch_f64_unpad_rows(const double* in, int n_pad, double* out, int n, int rows,
                                  cudaStream_t s) {
    f64_unpad_kernel<<<148 * 8, 256, 0, s>>>(in, n_pad, out, n, rows);
    return cudaGetLastError();
}

}  // namespace mxp
