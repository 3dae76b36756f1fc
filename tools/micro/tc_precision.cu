// Microbenchmark: accuracy of tf32 tensor-core split products on sm_100a.
// D = X W^T for X (128 x 32) ~ N(0,1), W (32 x 32) sparse N(0,1) rows, under
// several hi/lo split / accumulation orders; prints max |err| vs fp64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2404_01817_b200/csrc tc_precision.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <random>
#include <vector>

#include "tc.cuh"

using namespace tneat;
constexpr int M = 128, K = 32, NC = 32;
constexpr uint32_t SBO = K * 32;

__device__ float hi_of(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// mode 0: hi*hi, hi*lo, lo*hi interleaved per kk, one accumulator
// mode 1: cross terms first, then hi*hi (one accumulator)
// mode 2: hi*hi -> D0, cross -> D1 (two accumulators, summed in fp32)
// mode 3: per-kk hi*hi accumulators D0..D3 + cross D4 (summed in fp32)
// mode 4: raw fp32 operands (hardware tf32 conversion), single pass
__global__ void kern(const float* X, const float* W, float* out, int mode) {
  __shared__ __align__(1024) uint8_t sm[M * K * 4 + 2 * NC * K * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase[2];
  uint8_t* ahi = sm;
  uint8_t* bhi = sm + M * K * 4;
  uint8_t* blo = bhi + NC * K * 4;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) { tmem_alloc(smem_u32(&tbase[0]), 256); tmem_alloc(smem_u32(&tbase[1]), 32); tmem_relinquish(); }
  if (tid == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  for (int k = 0; k < K; ++k) {
    float x = X[tid * K + k];
    *reinterpret_cast<float*>(ahi + kmajor_offset(tid, k, SBO)) = mode == 4 ? x : hi_of(x);
  }
  if (tid < NC)
    for (int k = 0; k < K; ++k) {
      float w = W[tid * K + k];
      *reinterpret_cast<float*>(bhi + kmajor_offset(tid, k, SBO)) = mode == 4 ? w : hi_of(w);
      *reinterpret_cast<float*>(blo + kmajor_offset(tid, k, SBO)) = w - hi_of(w);
    }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t td = tbase[0], ta = tbase[1];
  const uint32_t lb = (uint32_t)(warp * 32) << 16;
  float lo[K];
  for (int k = 0; k < K; ++k) { float x = X[tid * K + k]; lo[k] = x - hi_of(x); }
  for (int q = 0; q < K / 8; ++q) tmem_st8(ta + lb + 8 * q, lo + 8 * q);
  tmem_wait_st();
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  const uint32_t idesc = idesc_tf32(M, NC);
  const uint32_t xs = smem_u32(ahi), bh = smem_u32(bhi), bl = smem_u32(blo);
  if (tid == 0) {
    tc_fence_after();
    auto A = [&](int kk) { return smem_desc(xs + kk * 256, SBO); };
    auto BH = [&](int kk) { return smem_desc(bh + kk * 256, SBO); };
    auto BL = [&](int kk) { return smem_desc(bl + kk * 256, SBO); };
    if (mode == 0) {
      for (int kk = 0; kk < K / 8; ++kk) {
        mma_tf32(td, A(kk), BH(kk), idesc, kk > 0);
        mma_tf32(td, A(kk), BL(kk), idesc, 1);
        mma_tf32_ts(td, ta + 8 * kk, BH(kk), idesc, 1);
      }
    } else if (mode == 1) {
      for (int kk = 0; kk < K / 8; ++kk) {
        mma_tf32(td, A(kk), BL(kk), idesc, kk > 0);
        mma_tf32_ts(td, ta + 8 * kk, BH(kk), idesc, 1);
      }
      for (int kk = 0; kk < K / 8; ++kk) mma_tf32(td, A(kk), BH(kk), idesc, 1);
    } else if (mode == 2) {
      for (int kk = 0; kk < K / 8; ++kk) mma_tf32(td, A(kk), BH(kk), idesc, kk > 0);
      for (int kk = 0; kk < K / 8; ++kk) {
        mma_tf32(td + NC, A(kk), BL(kk), idesc, kk > 0);
        mma_tf32_ts(td + NC, ta + 8 * kk, BH(kk), idesc, 1);
      }
    } else if (mode == 3) {
      for (int kk = 0; kk < K / 8; ++kk) mma_tf32(td + NC * kk, A(kk), BH(kk), idesc, 0);
      for (int kk = 0; kk < K / 8; ++kk) {
        mma_tf32(td + 4 * NC, A(kk), BL(kk), idesc, kk > 0);
        mma_tf32_ts(td + 4 * NC, ta + 8 * kk, BH(kk), idesc, 1);
      }
    } else {
      for (int kk = 0; kk < K / 8; ++kk) mma_tf32(td, A(kk), BH(kk), idesc, kk > 0);
    }
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const int nacc = mode == 2 ? 2 : (mode == 3 ? 5 : 1);
  for (int n = 0; n < NC; ++n) {
    float acc = 0.f;
    for (int a = 0; a < nacc; ++a) {
      float v[1] = {tmem_ld1(td + lb + a * NC + n)};
      tmem_wait_ld(v);
      acc += v[0];
    }
    out[tid * NC + n] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(td, 256); tmem_dealloc(ta, 32); }
}

int main() {
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  std::uniform_real_distribution<float> ud;
  std::vector<float> X(M * K), W(NC * K, 0.f), out(M * NC);
  double worst[5] = {0, 0, 0, 0, 0}, mean[5] = {0, 0, 0, 0, 0};
  float *dX, *dW, *dO;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dW, W.size() * 4); cudaMalloc(&dO, out.size() * 4);
  const int trials = 50;
  for (int t = 0; t < trials; ++t) {
    for (auto& v : X) v = nd(rng);
    for (auto& v : W) v = ud(rng) < 0.18f ? nd(rng) : 0.f;
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 5; ++mode) {
      kern<<<1, 128>>>(dX, dW, dO, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost);
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < NC; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)X[m * K + k] * W[n * K + k];
          const double err = fabs(out[m * NC + n] - ref) / fmax(1.0, fabs(ref));
          worst[mode] = fmax(worst[mode], err);
          mean[mode] += err / (M * NC * trials);
        }
    }
  }
  const char* names[5] = {"interleaved", "cross-first", "hihi|cross", "per-kk hihi", "raw 1-pass"};
  for (int mode = 0; mode < 5; ++mode) printf("%-12s max %.3e mean %.3e\n", names[mode], worst[mode], mean[mode]);
  // fp32 sequential FMA for comparison
  double w32 = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NC; ++n) {
      float acc = 0.f; double ref = 0;
      for (int k = 0; k < K; ++k) { acc = fmaf(X[m * K + k], W[n * K + k], acc); ref += (double)X[m * K + k] * W[n * K + k]; }
      w32 = fmax(w32, fabs(acc - ref) / fmax(1.0, fabs(ref)));
    }
  printf("fp32 fma     max %.3e (last trial)\n", w32);
  return 0;
}
