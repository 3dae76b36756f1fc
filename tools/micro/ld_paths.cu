// Micro-benchmark: the load paths a forward sweep can take per edge entry.
//   tmem   : tcgen05.ld 32x32b.x2 (two samples of the thread's lane), dynamic column
//   lds    : per-thread LDS.64 from a [slot][thread] float2 tile
//   mix    : one TMEM load and two LDS.64 per three entries (both paths at once)
//   uni32/64/128 : warp-uniform shared loads (program words), per-warp loads/s
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ld_paths ld_paths.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE, int BATCH>
__global__ void __launch_bounds__(128) bench(const uint32_t* __restrict__ cols, int iters, float* out, long long* cyc) {
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float2 vals[32 * 128];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 32 * 128; i += 128) vals[i] = make_float2(1.0f, 2.0f);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase + ((uint32_t)(warp * 32) << 16);
  float acc0 = 0.f, acc1 = 0.f;
  const float* vf = reinterpret_cast<const float*>(vals);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[2 * BATCH];
#pragma unroll
    for (int b = 0; b < BATCH; ++b) {
      const uint32_t c = (uint32_t)(it * 5 + b * 7 + threadIdx.x / 32) & 31u;
      if (MODE == 0 || (MODE == 2 && b % 3 == 0)) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[2 * b]), "=r"(r[2 * b + 1]) : "r"(tm + 2 * c));
      } else if (MODE <= 2) {
        const float2 v = vals[c * 128 + threadIdx.x];
        r[2 * b] = __float_as_uint(v.x); r[2 * b + 1] = __float_as_uint(v.y);
      } else if (MODE == 3) {  // uniform 32-bit
        r[2 * b] = __float_as_uint(vf[c * 4]); r[2 * b + 1] = 0;
      } else if (MODE == 4) {  // uniform 64-bit
        const float2 v = vals[c * 2];
        r[2 * b] = __float_as_uint(v.x); r[2 * b + 1] = __float_as_uint(v.y);
      } else {  // uniform 128-bit
        const float4 v = reinterpret_cast<const float4*>(vals)[c];
        r[2 * b] = __float_as_uint(v.x + v.z); r[2 * b + 1] = __float_as_uint(v.y + v.w);
      }
    }
    if (MODE == 0 || MODE == 2) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int b = 0; b < BATCH; ++b) { acc0 += __uint_as_float(r[2 * b]); acc1 += __uint_as_float(r[2 * b + 1]); }
  }
  long long t1 = clock64();
  out[blockIdx.x * 128 + threadIdx.x] = acc0 + acc1;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tbase) : "memory");
}

template <int MODE, int BATCH>
void run(const char* name, int blocks, const uint32_t* cols, float* out, long long* cyc, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  bench<MODE, BATCH><<<blocks, 128>>>(cols, 10, out, cyc);
  cudaEventRecord(a);
  bench<MODE, BATCH><<<blocks, 128>>>(cols, iters, out, cyc);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double loads = (double)blocks * 4 * iters * BATCH;  // warp-level loads
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double sm_cycles = ms * 1e-3 * clk * 1e3;
  printf("%-6s batch=%d warps/SM=%2d  %.3f ms  %.3f warp-loads/clk/SM  err=%s\n", name, BATCH, blocks / 148 * 4, ms,
         loads / 148 / sm_cycles, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint32_t h[256]; for (int i = 0; i < 256; ++i) h[i] = (i * 37) % 32;
  uint32_t* cols; float* out; long long* cyc;
  cudaMalloc(&cols, sizeof(h)); cudaMemcpy(cols, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&out, 148 * 8 * 128 * 4); cudaMalloc(&cyc, 148 * 8 * 8);
  for (int occ : {2, 4, 6}) {
    run<0, 4>("tmem", 148 * occ, cols, out, cyc, 8000);
    run<1, 4>("lds", 148 * occ, cols, out, cyc, 8000);
    run<0, 8>("tmem", 148 * occ, cols, out, cyc, 4000);
    run<1, 8>("lds", 148 * occ, cols, out, cyc, 4000);
    run<2, 6>("mix", 148 * occ, cols, out, cyc, 5000);
    run<3, 8>("uni32", 148 * occ, cols, out, cyc, 4000);
    run<4, 8>("uni64", 148 * occ, cols, out, cyc, 4000);
    run<5, 8>("uni128", 148 * occ, cols, out, cyc, 4000);
  }
  return 0;
}
