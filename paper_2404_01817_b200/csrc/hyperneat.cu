// K9: HyperNEAT substrate evaluation on the 5th-generation tensor cores.
//
// No reference implementation exists; semantics are
// builder-defined and documented in DESIGN.md:
//   * each genome's CPPN is queried on the 64 x 64 (output node, input node)
//     grid of an 8x8 -> 8x8 substrate (forward kernel, shared inputs) giving
//     W_p (64 x 64, row = output node k, column = input node j);
//   * substrate batch X (S x 64, S = multiple of 128) is shared by all genomes;
//     Y_p = tanh(X W_p^T), fitness_p = -mean_{s,k} (Y_p[s,k] - t[s])^2.
//
// This is the only dense contraction of the system, so it is the one kernel on
// tcgen05: each CTA owns 4 genomes (N = 4 x 64 = 256 accumulator columns),
// their W rows are the B operand (K-major, loaded once by TMA); the CTA streams
// 128-row tiles of X as the A operand through two shared-memory buffers
// (TMA 2-D tensor copies completing on mbarriers), one elected thread issues `tcgen05.mma.kind::tf32` (M=128,
// N=256, K=8 per instruction, 8 per tile) into one of two TMEM accumulators
// (2 x 256 columns), and the four warps run the fused epilogue (tcgen05.ld ->
// tanh -> squared error -> running sum) of tile t-1 while the tensor core
// works on tile t.  Y is never written to memory.

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace tneat {

constexpr int HN_K = 64;           // substrate inputs
constexpr int HN_N1 = 64;          // substrate outputs per genome
#ifndef TNEAT_HN_G
#define TNEAT_HN_G 4
#endif
constexpr int HN_G = TNEAT_HN_G;   // genomes per CTA (2 = two CTAs per SM: 1.41 vs 1.17 ms, slower)
constexpr int HN_N = HN_N1 * HN_G; // MMA N
constexpr int HN_M = 128;          // rows per tile (MMA M)
constexpr int HN_THREADS = 512;        // 16 warps: warp w reads TMEM lanes 32*(w%4).. of
constexpr int HN_SETS = HN_THREADS / 128; // column sets: warp w reads columns (w/4)*HN_CW.. in the epilogue
constexpr int HN_CW = HN_N / HN_SETS;     // columns per warp (one genome: HN_CW <= HN_N1)
constexpr int HN_TMEM_COLS = 2 * HN_N;    // two accumulator stages
static_assert(HN_CW <= HN_N1 && HN_N1 % HN_CW == 0 && HN_CW % 32 == 0, "epilogue mapping");

// K-major, no-swizzle operands laid out as K-chunk slabs: element (row, k) at
// (k / 4) * LBO + row * 16 + (k % 4) * 4, i.e. core matrices 8 rows x 16 B with
// SBO = 128 B between 8-row blocks and LBO = rows * 16 B between K chunks.  A
// slab (all rows of one 4-float K chunk) is one TMA box {4, rows}.
constexpr uint32_t HN_SBO = 128;
constexpr uint32_t HN_LBO_A = HN_M * 16;   // 2 KB
constexpr uint32_t HN_LBO_B = HN_N * 16;   // 4 KB

constexpr uint32_t HN_IDESC = idesc_tf32(HN_M, HN_N);

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct __align__(1024) HnSmem {
  float b[HN_N * HN_K];          // 64 KB: 4 genomes' W rows, 16 K-chunk slabs of 256 rows
  float a[2][HN_M * HN_K];       // 2 x 32 KB: X tiles, 16 K-chunk slabs of 128 rows
  float part[HN_THREADS / 32][HN_G];
  uint64_t mma_bar[2];
  uint64_t load_bar[2];          // TMA completion of A[stage] (and of B with stage 0's first use)
  uint32_t tmem_base;
};

// one 128 x 64 tile of X (rows r0..) by TMA: 16 slab copies of 2 KB
__device__ __forceinline__ void tma_a_tile(float* a, const void* tx, int r0, uint32_t bar, bool arrive = true) {
  if (arrive) mbar_expect_tx(bar, HN_M * HN_K * 4);
  const uint32_t base = smem_u32(a);
#pragma unroll
  for (int kc = 0; kc < HN_K / 4; ++kc) tma_load_2d(base + kc * HN_LBO_A, tx, kc * 4, r0, bar);
}

__global__ void __launch_bounds__(HN_THREADS, 512 / HN_TMEM_COLS)
substrate_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x, int64_t P,
                 const float* __restrict__ target, int S, double* __restrict__ fitness) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  HnSmem& sm = *reinterpret_cast<HnSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t g0 = (int64_t)blockIdx.x * HN_G;
  const int ng = (int)(P - g0 < HN_G ? P - g0 : HN_G);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)), "n"(HN_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&sm.mma_bar[0]), 1);
    mbar_init(smem_u32(&sm.mma_bar[1]), 1);
    mbar_init(smem_u32(&sm.load_bar[0]), 1);
    mbar_init(smem_u32(&sm.load_bar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // B operand: rows n = g*64 + k (output node k of genome g) = rows g0*64.. of
    // W viewed as (P*64, 64); rows past P*64 come back as zeros (TMA bounds)
    // B and the first A tile complete one phase of load_bar[0]: one arrival
    // carrying both transaction counts
    const uint32_t bar = smem_u32(&sm.load_bar[0]);
    mbar_expect_tx(bar, (HN_N + HN_M) * HN_K * 4);
    const uint32_t base = smem_u32(sm.b);
#pragma unroll
    for (int kc = 0; kc < HN_K / 4; ++kc) tma_load_2d(base + kc * HN_LBO_B, &tmap_w, kc * 4, (int)(g0 * HN_N1), bar);
    tma_a_tile(sm.a[0], &tmap_x, 0, bar, false);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;
  const int tiles = S / HN_M;
  float acc_err = 0.f;  // this warp's genome
  uint32_t phase[2] = {0u, 0u};

  auto epilogue = [&](int tile, int stage) {
    // tile row = TMEM lane = 32 * (warp % 4) + lane; warp / 4 picks the genome set
    const int row = (warp & 3) * 32 + lane;
    const float tv = target[(int64_t)tile * HN_M + row];
    const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(stage * HN_N) +
                           (uint32_t)((warp >> 2) * HN_CW);
#pragma unroll 1
    for (int q = 0; q < HN_CW / 16; q += 2) {  // two 16-column loads per wait
      uint32_t r[16], r2[16];
      TMEM_LD16(taddr + q * 16, r);
      TMEM_LD16(taddr + (q + 1) * 16, r2);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float d = tanh_approx(__uint_as_float(r[i])) - tv;
        const float d2 = tanh_approx(__uint_as_float(r2[i])) - tv;
        acc_err = fmaf(d, d, acc_err);
        acc_err = fmaf(d2, d2, acc_err);
      }
    }
  };

  uint32_t lphase[2] = {0u, 0u};
  for (int t = 0; t < tiles; ++t) {
    const int stage = t & 1;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // epilogue(t-2) is done with accumulator `stage`
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
      mbar_wait(smem_u32(&sm.load_bar[stage]), lphase[stage]);  // A[t] (and B) landed
      const uint32_t a0 = smem_u32(sm.a[stage]), b0 = smem_u32(sm.b);
#pragma unroll
      for (int kk = 0; kk < HN_K / 8; ++kk)  // K = 8 tf32 per instruction = 2 K-chunk slabs
        mma_tf32(tmem + (uint32_t)(stage * HN_N), smem_desc(a0 + kk * 2 * HN_LBO_A, HN_SBO, HN_LBO_A),
                 smem_desc(b0 + kk * 2 * HN_LBO_B, HN_SBO, HN_LBO_B), HN_IDESC, kk > 0 ? 1u : 0u);
      mma_commit(smem_u32(&sm.mma_bar[stage]));
    }
    lphase[stage] ^= 1u;
    if (t >= 1) {
      // MMA t-1 finished -> its A buffer (the other one) is free and its accumulator ready
      mbar_wait(smem_u32(&sm.mma_bar[stage ^ 1]), phase[stage ^ 1]);
      phase[stage ^ 1] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (tid == 0 && t + 1 < tiles) tma_a_tile(sm.a[stage ^ 1], &tmap_x, (t + 1) * HN_M, smem_u32(&sm.load_bar[stage ^ 1]));
      epilogue(t - 1, stage ^ 1);
    } else if (tid == 0 && t + 1 < tiles) {
      // the other A buffer has never been used
      tma_a_tile(sm.a[stage ^ 1], &tmap_x, (t + 1) * HN_M, smem_u32(&sm.load_bar[stage ^ 1]));
    }
  }
  {
    const int last = tiles - 1, stage = last & 1;
    mbar_wait(smem_u32(&sm.mma_bar[stage]), phase[stage]);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    epilogue(last, stage);
  }
  // reduce squared errors over the CTA's 128 rows (each warp holds one genome's columns)
  {
    if (lane < HN_G) sm.part[warp][lane] = 0.f;
    __syncwarp();
    float v = acc_err;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0) sm.part[warp][(warp >> 2) * HN_CW / HN_N1] = v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < ng) {
    double s = 0.0;
    for (int w = 0; w < HN_THREADS / 32; ++w) s += (double)sm.part[w][tid];
    fitness[g0 + tid] = -s / ((double)S * HN_N1);
  }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(HN_TMEM_COLS) : "memory");
  }
}

}  // namespace tneat

using namespace tneat;

extern "C" {

// HyperNEAT substrate fitness (builder-defined): W (P,64,64) fp32
// CPPN weights (row = output node), X (S,64) fp32 shared substrate inputs
// (S a multiple of 128), target (S,) fp32; fitness (P,) float64 =
// -mean((tanh(X W_p^T) - target[:,None])^2).  tcgen05 kind::tf32 MMAs.
int an_substrate_fitness(const float* W, int64_t P, const float* X, const float* target, int S, double* fitness,
                         void* stream) {
  if (P < 0 || S <= 0 || S % HN_M != 0) return -1;
  if (P == 0) return 0;
  if (!W || !X || !target || !fitness) return -2;
  if (((uintptr_t)W | (uintptr_t)X) & 15) return -2;
  // TMA descriptors: W as a (P*64, 64) and X as an (S, 64) row-major fp32 matrix,
  // boxes of one 4-float K chunk x all tile rows
  const PFN_cuTensorMapEncodeTiled_v12000 encode = tmap_encoder();
  if (!encode) return -9;
  CUtensorMap tw, tx;
  const cuuint32_t estr[2] = {1, 1};
  {
    const cuuint64_t dims[2] = {HN_K, (cuuint64_t)P * HN_N1}, strides[1] = {HN_K * 4};
    const cuuint32_t box[2] = {4, HN_N};
    if (encode(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(W), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -9;
  }
  {
    const cuuint64_t dims[2] = {HN_K, (cuuint64_t)S}, strides[1] = {HN_K * 4};
    const cuuint32_t box[2] = {4, HN_M};
    if (encode(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -9;
  }
  const int smem = (int)sizeof(HnSmem) + 1024;
  cudaFuncSetAttribute(substrate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int64_t blocks = (P + HN_G - 1) / HN_G;
  substrate_kernel<<<(unsigned)blocks, HN_THREADS, smem, (cudaStream_t)stream>>>(tw, tx, P, target, S, fitness);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
