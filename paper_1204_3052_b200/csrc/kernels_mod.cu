// Exact modular mode: (A^k) mod p for uint32 residues, p < 2^31.
//
// No reference counterpart (the reference rejects integer dtypes,
// dtypes.py:37-42); parity is bit-exact by construction and pinned by KATs
// (Pisano periods, permutation orders) and by the oracle's exact restatement
// (oracle/matexpo_oracle.c: mxo_exponentiate_mod).
//
// Each residue x < 2^31 is split into 16-bit limbs x = x1*2^16 + x0.  One
// product C = A*B mod p is three FP64 DMMA GEMMs (Karatsuba):
//   T1 = A1 B1,  T0 = A0 B0,  T2 = (A0 + A1)(B0 + B1)
//   C  = T1 * 2^32 + (T2 - T1 - T0) * 2^16 + T0   (mod p)
// Every operand is an integer < 2^17 and every partial sum of a GEMM is an
// integer < n * 2^34 <= 2^53 (n <= 2^19), so the FP64 tensor-core FMAs are
// exact and so is the result.  The combine kernel reduces mod p in uint64 and
// directly emits the next step's limb planes (or the final uint32 matrix).
#include "mxp_internal.h"

namespace mxp {

__device__ __forceinline__ void limbs(uint32_t x, double& l0, double& l1, double& ls) {
    const uint32_t a0 = x & 0xFFFFu, a1 = x >> 16;
    l0 = static_cast<double>(a0);
    l1 = static_cast<double>(a1);
    ls = static_cast<double>(a0 + a1);
}

// uint32 n x n (leading dim n) -> reduced residues' limb planes (n_pad, zero pad)
__global__ void mod_split_kernel(const uint32_t* __restrict__ in, int n, uint32_t p,
                                 double* __restrict__ l0, double* __restrict__ l1,
                                 double* __restrict__ ls, int n_pad) {
    const size_t total = static_cast<size_t>(n_pad) * n_pad;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / n_pad), c = static_cast<int>(i % n_pad);
        const uint32_t x = (r < n && c < n) ? in[static_cast<size_t>(r) * n + c] % p : 0u;
        limbs(x, l0[i], l1[i], ls[i]);
    }
}

// T0, T1, T2 (n_pad^2 exact integers in fp64) -> C mod p; either the next limb
// planes (out_u32 == nullptr) or the final n x n uint32 matrix.
__global__ void mod_combine_kernel(const double* __restrict__ t0, const double* __restrict__ t1,
                                   const double* __restrict__ t2, uint32_t p, uint64_t r16,
                                   uint64_t r32, int n_pad, double* __restrict__ l0,
                                   double* __restrict__ l1, double* __restrict__ ls,
                                   uint32_t* __restrict__ out_u32, int n) {
    const size_t total = static_cast<size_t>(n_pad) * n_pad;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint64_t a = static_cast<uint64_t>(t0[i]);
        const uint64_t b = static_cast<uint64_t>(t1[i]);
        const uint64_t s = static_cast<uint64_t>(t2[i]);
        const uint64_t mid = s - a - b;  // exact, non-negative
        uint64_t c = (b % p) * r32 % p;
        c = (c + (mid % p) * r16) % p;
        c = (c + a % p) % p;
        if (out_u32 != nullptr) {
            const int r = static_cast<int>(i / n_pad), col = static_cast<int>(i % n_pad);
            if (r < n && col < n) out_u32[static_cast<size_t>(r) * n + col] = static_cast<uint32_t>(c);
        } else {
            limbs(static_cast<uint32_t>(c), l0[i], l1[i], ls[i]);
        }
    }
}

cudaError_t launch_mod_split(const uint32_t* in, int n, uint32_t p, double* l0, double* l1,
                             double* ls, int n_pad, cudaStream_t s) {
    mod_split_kernel<<<148 * 8, 256, 0, s>>>(in, n, p, l0, l1, ls, n_pad);
    return cudaGetLastError();
}

cudaError_t launch_mod_combine(const double* t0, const double* t1, const double* t2, uint32_t p,
                               int n_pad, double* l0, double* l1, double* ls, uint32_t* out,
                               int n, cudaStream_t s) {
    const uint64_t r16 = (1ull << 16) % p;
    const uint64_t r32 = (1ull << 32) % p;
    mod_combine_kernel<<<148 * 8, 256, 0, s>>>(t0, t1, t2, p, r16, r32, n_pad, l0, l1, ls, out, n);
    return cudaGetLastError();
}

__global__ void mod_identity_kernel(uint32_t* __restrict__ out, const uint32_t* __restrict__ a,
                                    int n, uint32_t p, int copy) {
    const size_t total = static_cast<size_t>(n) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = copy ? a[i] % p : ((i / n == i % n) ? 1u % p : 0u);
}

// k = 0 -> I, k = 1 -> A mod p
cudaError_t launch_mod_trivial(uint32_t* out, const uint32_t* a, int n, uint32_t p, int copy,
                               cudaStream_t s) {
    mod_identity_kernel<<<148 * 4, 256, 0, s>>>(out, a, n, p, copy);
    return cudaGetLastError();
}

}  // namespace mxp
