// Microbenchmark: exactness of the digit-split tensor-core input layer
// (csrc/digits.cuh) on sm_100a.  D = X W for X (128 x 32), W (32 x 64) sparse,
// rows/columns of very different magnitudes; prints the max error relative to
// sum |x w| (and absolute) against fp64, next to an fp32 FMA chain's.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2404_01817_b200/csrc tc_digits.cu
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "digits.cuh"
#include "tc.cuh"

using namespace tneat;
constexpr int M = 128, K = 32, N = 64;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_f16_s10(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, 10;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}

__global__ void kern(const float* X, const float* W, float* out) {
  __shared__ __align__(1024) uint8_t a_s[M * TC_ROWB];
  __shared__ __align__(1024) uint8_t b_s[N * TC_ROWB];
  __shared__ float cf[N];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { tmem_alloc(smem_u32(&tbase), 128); tmem_relinquish(); }
  if (tid == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  // A: row tid
  float x[K];
  float m = 0.f;
  for (int k = 0; k < K; ++k) { x[k] = X[tid * K + k]; m = fmaxf(m, fabsf(x[k])); }
  const int ex = m > 0.f ? float_exponent(m) : 0;
  const float sc = pow2f(27 - ex);
  for (int k = 0; k < K; k += 2) {
    float a2, a1, a0, b2, b1, b0;
    digits3(x[k] * sc, a2, a1, a0);
    digits3(x[k + 1] * sc, b2, b1, b0);
    *reinterpret_cast<__half2*>(a_s + tc_offset(tid, k)) = __floats2half2_rn(a2, b2);
    *reinterpret_cast<__half2*>(a_s + tc_offset(tid, 32 + k)) = __floats2half2_rn(a1, b1);
    *reinterpret_cast<__half2*>(a_s + tc_offset(tid, 64 + k)) = __floats2half2_rn(a0, b0);
  }
  if (tid < N) {  // B: column tid (the transform does this in double)
    double mw = 0.0;
    for (int k = 0; k < K; ++k) mw = fmax(mw, fabs((double)W[k * N + tid]));
    int ew = 0;
    if (mw > 0) { frexp(mw, &ew); ew -= 1; }
    const double s = ldexp(1.0, 27 - ew);
    for (int k = 0; k < K; ++k) {
      double d2, d1, d0;
      digits3_d((double)W[k * N + tid] * s, d2, d1, d0);
      *reinterpret_cast<__half*>(b_s + tc_offset(tid, k)) = __double2half(d2);
      *reinterpret_cast<__half*>(b_s + tc_offset(tid, 32 + k)) = __double2half(d1);
      *reinterpret_cast<__half*>(b_s + tc_offset(tid, 64 + k)) = __double2half(d0);
    }
    cf[tid] = pow2f(ew - 12);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t a = smem_u32(a_s), b = smem_u32(b_s), id = idesc_f16(M, N);
    auto A = [&](int k0) { return smem_desc(a + (k0 >> 3) * TC_LBO, TC_SBO, TC_LBO); };
    auto B = [&](int k0) { return smem_desc(b + (k0 >> 3) * TC_LBO, TC_SBO, TC_LBO); };
    // D4 = A2 . B2 (cols 0..63)
    mma_f16(tm, A(0), B(0), id, 0);
    mma_f16(tm, A(16), B(16), id, 1);
    // D32 (cols 64..127): class 2 = A2 B0 + A1 B1 + A0 B2
    const uint32_t d32 = tm + N;
    mma_f16(d32, A(0), B(64), id, 0);
    mma_f16(d32, A(16), B(80), id, 1);
    mma_f16(d32, A(32), B(32), id, 1);
    mma_f16(d32, A(48), B(48), id, 1);
    mma_f16(d32, A(64), B(0), id, 1);
    mma_f16(d32, A(80), B(16), id, 1);
    // * 2^-10, + class 3 = A2 B1 + A1 B2
    mma_f16_s10(d32, A(0), B(32), id);
    mma_f16(d32, A(16), B(48), id, 1);
    mma_f16(d32, A(32), B(0), id, 1);
    mma_f16(d32, A(48), B(16), id, 1);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const float rf = pow2f(ex - 12);
  const uint32_t lane_base = tm + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < N; c += 16) {
    uint32_t r4[16], r3[16];
    TMEM_LD16(lane_base + c, r4);
    TMEM_LD16(lane_base + N + c, r3);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) {
      const float t = __fmaf_rn(__uint_as_float(r4[i]), 1024.0f, __uint_as_float(r3[i]));
      out[tid * N + c + i] = t * rf * cf[c + i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 128); }
}

int main() {
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud;
  std::vector<float> X(M * K), W(K * N), out(M * N);
  for (int r = 0; r < M; ++r) {
    double s = 1.0;
    if (r % 8 == 1) s = 1e-3;
    if (r % 8 == 2) s = 1e3;
    if (r % 8 == 3) s = 0.0;
    for (int k = 0; k < K; ++k) {
      double v = nd(rng) * s;
      if (r % 8 == 4 && k % 5 == 0) v *= 1e-6;  // wide dynamic range inside a row
      X[r * K + k] = (float)v;
    }
  }
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) W[k * N + n] = ud(rng) < 0.2 ? (float)std::max(-30.0, std::min(30.0, nd(rng))) : 0.f;
  W[0 * N + 5] = 30.f;  // one large weight beside small ones
  W[1 * N + 5] = 1e-4f;
  float *dX, *dW, *dO;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dW, W.size() * 4); cudaMalloc(&dO, out.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  kern<<<1, 128>>>(dX, dW, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost);
  double max_rel = 0, max_abs = 0, max_rel32 = 0, max_abs32 = 0;
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      double ref = 0, mag = 0;
      float f32 = 0.f;
      for (int k = 0; k < K; ++k) {
        ref += (double)X[r * K + k] * W[k * N + n];
        mag += fabs((double)X[r * K + k] * W[k * N + n]);
        f32 = fmaf(X[r * K + k], W[k * N + n], f32);
      }
      if (mag == 0) { if (out[r * N + n] != 0.f) max_rel = 1e9; continue; }
      max_rel = fmax(max_rel, fabs(out[r * N + n] - ref) / mag);
      max_abs = fmax(max_abs, fabs(out[r * N + n] - ref));
      max_rel32 = fmax(max_rel32, fabs(f32 - ref) / mag);
      max_abs32 = fmax(max_abs32, fabs(f32 - ref));
    }
  printf("digit-split tcgen05: max |err|/sum|xw| = %.3e  max abs = %.3e\n", max_rel, max_abs);
  printf("fp32 FMA chain     : max |err|/sum|xw| = %.3e  max abs = %.3e\n", max_rel32, max_abs32);
  printf("sample out[0][0..3] = %.8f %.8f %.8f %.8f\n", out[0], out[1], out[2], out[3]);
  return (max_abs <= 2 * max_abs32 && max_rel < 2e-6) ? 0 : 2;
}
