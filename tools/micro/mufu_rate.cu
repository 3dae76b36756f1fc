// MUFU throughput on this GPU: tanh.approx.f32 vs ex2.approx.f32 vs rcp.approx
// (independent chains, all SMs busy).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      else if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      else asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      x[i] = y;
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  const int iters = 4096;
  const char* names[3] = {"tanh.approx.f32", "ex2.approx.f32", "rcp.approx.f32"};
  for (int op = 0; op < 3; ++op) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<sms * 8, 1024 / 8 * 8 / 8 * 8 > 0 ? 256 : 256>>>(out, iters);
      if (op == 1) k<1><<<sms * 8, 256>>>(out, iters);
      if (op == 2) k<2><<<sms * 8, 256>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)sms * 8 * 256 * iters * 8;
    printf("%s: %.3g ops/s = %.2f per SM per clock (at %.0f MHz max)\n", names[op], ops / (ms * 1e-3),
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
  }
  return 0;
}
