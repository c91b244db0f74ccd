// Scaled fp16x2 split of fp32 values (K3H): P = 2^e P', the planes hold
// h0 = rn_fp16(x') and -h1 = -rn_fp16(x' - h0); the MMAs that read the -h1
// plane set the instruction descriptor's negate bit.  See kernels_k3h.cu.
#pragma once

#include <cstdint>

namespace mxp {
namespace {

constexpr int kTarget = 13;  // input: scaled max |A'| in [2^13, 2^14)
constexpr int kCeil = 14;    // products: scaled max |D'| < 2^14 guaranteed

// (a, b) = columns 2j, 2j+1 (unscaled), sc2 = the scale in both halves:
// two packed fp16x2 words p0 = h0 = rn(a', b') and p1 = -h1.
__device__ __forceinline__ void split2(float a, float b, uint64_t sc2, uint32_t& p0, uint32_t& p1) {
    // p1 = rn(p0 - x') = -rn(x' - p0) (the residual is exact in fp32).  Per
    // pair: FMUL2, F2FP, two mixed fp16-fp32 subtractions (FHADD, the fp16
    // half read in place), F2FP — one instruction fewer than unpacking h0
    // (2 HADD2.F32) for an FADD2.  The MMAs that read p1 negate it back
    // (instruction-descriptor negate bits), so the products are those of
    // h1 = rn(x' - h0) bit for bit (measured: identical outputs, -4% time).
    uint64_t ab, s2;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ab) : "f"(a), "f"(b));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(s2) : "l"(ab), "l"(sc2));
    asm("{\n\t.reg .f32 sa, sb, ra, rb;\n\t.reg .b16 l, h;\n\t"
        "mov.b64 {sa, sb}, %2;\n\t"
        "cvt.rn.f16x2.f32 %0, sb, sa;\n\t"
        "mov.b32 {l, h}, %0;\n\t"
        "sub.f32.f16 ra, l, sa;\n\t"
        "sub.f32.f16 rb, h, sb;\n\t"
        "cvt.rn.f16x2.f32 %1, rb, ra;\n\t}"
        : "=r"(p0), "=r"(p1)
        : "l"(s2));
}
__device__ __forceinline__ uint64_t splat2(float x) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
    return r;
}
// 2^t as a float, t clamped to the normal range
__device__ __forceinline__ float exp2i(int t) {
    t = max(-126, min(127, t));
    return __int_as_float((t + 127) << 23);
}
// scale exponent for a block whose max |element| has bit pattern mbits:
// returns t with max * 2^t in [2^13, 2^14) (0 for zero, inf or NaN maxima)
__device__ __forceinline__ int scale_exp(uint32_t mbits) {
    if (mbits == 0u || mbits >= 0x7F800000u) return 0;
    const int k = mbits >= 0x00800000u ? static_cast<int>(mbits >> 23) - 127
                                       : -127 + (31 - __clz(static_cast<int>(mbits))) - 22;
    return kTarget - k;
}
// floor(log2(x)) from the bits of |x| (x finite, > 0); -1000 for 0
__device__ __forceinline__ int ilogb_bits(uint32_t mbits) {
    if (mbits == 0u) return -1000;
    return mbits >= 0x00800000u ? static_cast<int>(mbits >> 23) - 127
                                : (31 - __clz(static_cast<int>(mbits))) - 149;
}

}  // namespace
}  // namespace mxp
