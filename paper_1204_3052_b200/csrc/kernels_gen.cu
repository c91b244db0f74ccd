// Device-side SplitMix64 input generation, bit-identical to the reference's
// random_matrix (linalg.py:109-148) and to the SURVEY §8(d) scaled recipe
// fl(random_matrix(n, F64, seed) * s).  Removes host generation and makes the
// batched config's inputs reproducible on any device (next-row f3).
#include "mxp_internal.h"

namespace mxp {

__device__ __forceinline__ uint64_t sm64(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// f64 path: lo + u*(hi-lo) with two roundings (no FMA), clamp onto
// nextafter(hi, lo), optional scale, then cast.
template <typename T>
__global__ void random_kernel(T* __restrict__ out, int64_t n2, int64_t batch, uint64_t seed0,
                              double lo, double span, double hi, double below64, double scale,
                              float fhi, float below32) {
    const int64_t total = n2 * batch;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = i / n2, e = i - b * n2;
        const uint64_t z = sm64(seed0 + static_cast<uint64_t>(b), static_cast<uint64_t>(e));
        const double u = __dmul_rn(__ull2double_rn(z >> 11), 0x1p-53);
        double v = __dadd_rn(lo, __dmul_rn(u, span));
        if (scale != 0.0) {
            if (v >= hi) v = below64;
            v = __dmul_rn(v, scale);
            out[i] = static_cast<T>(v);
        } else if (sizeof(T) == 8) {
            if (v >= hi) v = below64;
            out[i] = static_cast<T>(v);
        } else {
            float f = __double2float_rn(v);
            if (f >= fhi) f = below32;
            out[i] = static_cast<T>(f);
        }
    }
}

// The raw stream (linalg.py:117-124: splitmix64(seed, count)), draw k at out[k].
__global__ void splitmix64_kernel(uint64_t* __restrict__ out, int64_t count, uint64_t seed) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = sm64(seed, static_cast<uint64_t>(i));
}

cudaError_t launch_splitmix64(uint64_t seed, int64_t count, uint64_t* out, cudaStream_t s) {
    int blocks = static_cast<int>((count + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks < 1) blocks = 1;
    splitmix64_kernel<<<blocks, 256, 0, s>>>(out, count, seed);
    return cudaGetLastError();
}

cudaError_t launch_random(int mode, int64_t n, int64_t batch, uint64_t seed0, double lo, double hi,
                          double scale, void* out, cudaStream_t s) {
    const double span = hi - lo;
    const double below64 = nextafter(hi, lo);
    const float fhi = static_cast<float>(hi);
    const float below32 = nextafterf(fhi, static_cast<float>(lo));
    const int64_t total = n * n * batch;
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (mode == 1)
        random_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double*>(out), n * n, batch, seed0,
                                                     lo, span, hi, below64, scale, fhi, below32);
    else
        random_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float*>(out), n * n, batch, seed0,
                                                    lo, span, hi, below64, scale, fhi, below32);
    return cudaGetLastError();
}

}  // namespace mxp
