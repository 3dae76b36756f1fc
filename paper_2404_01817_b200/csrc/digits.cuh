// Exact tensor-core dot products for the fp32 forward's input layer.
//
// The input-sourced part of every step's aggregation, sum_i w_ij * x_i, is a
// (samples x I) . (I x steps) product.  The tensor cores' fp32 accumulation is
// not round-to-nearest (a tf32 hi/lo split measured ~4e-6 error per MMA,
// tools/micro/tc_precision.cu), so the product is computed in integers:
//
//   * every sample row x (and every weight column w) is block-scaled by a
//     power of two so that max |.| lies in [2^27, 2^28), then written as three
//     balanced base-1024 digits  X = d2 2^20 + d1 2^10 + d0,  |d| <= 512
//     (|d2| <= 256).  The digits are small integers, exact in fp16.
//   * products of digits are integers <= 2^18; a K = 32 sum of them stays an
//     integer <= 2^24, which fp32 represents exactly whatever the tensor
//     core's internal rounding (kind::f16 MMAs with fp32 accumulation).
//   * D4  = sum d2 e2                                   (exact, <= 2^21)
//     D32 = sum (d2 e1 + d1 e2) + 2^-10 sum (d2 e0 + d1 e1 + d0 e2)
//           (class 2 accumulated first, exact <= 2^24; then scaled by 2^-10
//            with the MMA's scale-input-d and class 3 added: error <= 2^-23
//            of a term that is itself 2^-10 of the result's scale)
//   * sum x w = 2^(ex + ew - 24) * (1024 D4 + D32): one FFMA and two exact
//     power-of-two multiplies per step and sample.
// Dropped classes (d1 e0 + d0 e1, d0 e0) and the digit quantisation (|y - X|
// <= 1/2) are below 2^-27 of max|x| * max|w| * K; the result carries one fp32
// rounding of T = 1024 D4 + D32 -- the accuracy of an fp32 FMA chain.
//
// Rows / columns whose max |.| is not finite or outside [2^-62, 2^62] (or is
// 0: all digits 0) cannot be scaled this way; rows take an exact CUDA-core
// path (forward.cu), columns make the transform emit a standard program.
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda_fp16.h>

namespace tneat {

constexpr int TC_K = 32;            // input digits per plane (I <= 32, zero padded)
constexpr int TC_ROWB = 3 * TC_K * 2;  // bytes of one operand row: 3 planes x 32 fp16 = 192
// K-major, no-swizzle UMMA operand layout for rows of 96 fp16 (3 planes x 32):
// core matrices of 8 rows x 16 bytes; K-adjacent core matrices 128 B apart
// (LBO), 8-row groups 12 * 128 = 1536 B apart (SBO)
constexpr uint32_t TC_LBO = 128, TC_SBO = 12 * 128;
constexpr int TC_EMAX = 62;         // block exponents in [-62, 62]

__host__ __device__ inline uint32_t tc_offset(int row, int k) {  // k in [0, 96)
  return (uint32_t)(row >> 3) * TC_SBO + (uint32_t)(k >> 3) * TC_LBO + (uint32_t)(row & 7) * 16 +
         (uint32_t)(k & 7) * 2;
}

// instruction descriptor: kind::f16, D = F32, A = B = F16, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// floor(log2 m) for a positive normal float m
__device__ __forceinline__ int float_exponent(float m) { return (int)((__float_as_uint(m) >> 23) & 0xFF) - 127; }

// 2^e as a float, e in [-126, 127]
__host__ __device__ inline float pow2f(int e) {
#ifdef __CUDA_ARCH__
  return __uint_as_float((uint32_t)(e + 127) << 23);
#else
  uint32_t b = (uint32_t)(e + 127) << 23;
  float f;
  memcpy(&f, &b, 4);
  return f;
#endif
}

// y in (-2^28, 2^28) -> balanced digits (exact integers, |d2| <= 256,
// |d1|, |d0| <= 512) with |y - (d2 2^20 + d1 2^10 + d0)| <= 1/2.  The magic
// constant 1.5 * 2^23 rounds to the nearest integer; the _rn intrinsics keep
// the compiler from folding (t + M) - M.
__device__ __forceinline__ void digits3(float y, float& d2, float& d1, float& d0) {
  constexpr float M = 12582912.0f;
  d2 = __fsub_rn(__fmaf_rn(y, 0x1p-20f, M), M);
  const float r1 = __fmaf_rn(d2, -0x1p20f, y);  // exact
  d1 = __fsub_rn(__fmaf_rn(r1, 0x1p-10f, M), M);
  const float r0 = __fmaf_rn(d1, -1024.0f, r1);  // exact
  d0 = __fsub_rn(__fadd_rn(r0, M), M);
}

// Two elements at once in the row's unscaled space (packed fp32: FFMA2 /
// FADD2), with y = x * sc folded into the constants s20 = sc 2^-20,
// i20 = 2^20 / sc, s10 = sc 2^-10, i10 = 2^10 / sc, s0 = sc (all powers of two,
// so every residual is exact as above): 5 FFMA2 + 3 FADD2 per pair.
// Constants all 0 give zero digits (finite x).
__device__ __forceinline__ void digits3x2(float2 x, float s20, float i20, float s10, float i10, float s0, float2& d2,
                                          float2& d1, float2& d0) {
  const float2 M = make_float2(12582912.0f, 12582912.0f), nM = make_float2(-12582912.0f, -12582912.0f);
  d2 = __fadd2_rn(__ffma2_rn(x, make_float2(s20, s20), M), nM);
  const float2 r1 = __ffma2_rn(d2, make_float2(-i20, -i20), x);
  d1 = __fadd2_rn(__ffma2_rn(r1, make_float2(s10, s10), M), nM);
  const float2 r0 = __ffma2_rn(d1, make_float2(-i10, -i10), r1);
  d0 = __fadd2_rn(__ffma2_rn(r0, make_float2(s0, s0), M), nM);
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// the same digits from a double (the transform's weights, exact integers in
// double arithmetic)
__host__ __device__ inline void digits3_d(double y, double& d2, double& d1, double& d0) {
  d2 = rint(y * 0x1p-20);
  const double r1 = y - d2 * 0x1p20;
  d1 = rint(r1 * 0x1p-10);
  d0 = rint(r1 - d1 * 1024.0);
}

}  // namespace tneat
