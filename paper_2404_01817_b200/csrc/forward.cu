// K2: population forward -- executes transform programs over input batches.
//
// Replaces arrayneat inference.forward_arrays (inference.py:185-262).
//
// Two kernels:
//   * fwd_tile: one CTA per (genome, tile of NT*S inputs).  Each thread owns S
//     consecutive inputs; node values live in shared memory as [slot][tile]
//     (inputs first, staged from HBM with 16-byte loads), so a thread only ever
//     reads values it wrote itself -- no barrier inside the node sweep.  Edge
//     descriptors are warp-uniform broadcast reads, value reads are S-wide
//     vector loads.  For large per-genome batches (config 2: B = 4096).
//   * fwd_warp: one warp per genome; lanes split a node's incoming edges and
//     combine with warp-shuffle reductions (sum/product/max/min/mean).  For
//     small batches (XOR B=4, regression B=64, cart-pole B=1) where a
//     thread-per-input mapping would idle most lanes.  Optionally fuses the
//     XOR / regression fitness epilogue (problems.py:54-61).
//
// Semantics: input rows hold raw inputs and are never
// activated; node = act(bias + response * agg(w * v)); empty aggregation = 0;
// mean divides by the incoming count; outputs read at the rows of keys I..I+O-1.

#include "common.cuh"

namespace tneat {

template <typename T, int S> struct __align__(sizeof(T) * S) Pack { T v[S]; };

template <typename T, int S, int NT>
__global__ void __launch_bounds__(NT) fwd_tile_kernel(const uint8_t* __restrict__ prog, ProgLayout L,
                                                      const T* __restrict__ in, int64_t in_gstride,
                                                      int B, int I, int O, int tiles,
                                                      T* __restrict__ out, int64_t out_gstride) {
  constexpr int TT = NT * S;
  using PackT = Pack<T, S>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int64_t gi = blockIdx.x / tiles;
  const int tile = (int)(blockIdx.x - gi * tiles);
  const uint8_t* gp = prog + gi * L.stride;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const int n_steps = hdr.n_steps, n_edges = hdr.n_edges;
  const int tid = threadIdx.x;

  StepT<T>* st_s = reinterpret_cast<StepT<T>*>(smem);
  const int64_t off_e = align_up((int64_t)n_steps * sizeof(StepT<T>), 16);
  EdgeT<T>* ed_s = reinterpret_cast<EdgeT<T>*>(smem + off_e);
  const int64_t off_v = align_up(off_e + (int64_t)n_edges * sizeof(EdgeT<T>), 16);
  T* vals = reinterpret_cast<T*>(smem + off_v);

  // program -> shared memory (edge sources become byte offsets of the slot row)
  {
    const int4* src = reinterpret_cast<const int4*>(gp + L.off_steps);
    int4* dst = reinterpret_cast<int4*>(st_s);
    const int n16 = (int)((int64_t)n_steps * sizeof(StepT<T>) / 16);
    for (int i = tid; i < n16; i += NT) dst[i] = __ldg(src + i);
    const EdgeT<T>* esrc = reinterpret_cast<const EdgeT<T>*>(gp + L.off_edges);
    for (int e = tid; e < n_edges; e += NT) {
      EdgeT<T> x = esrc[e];
      x.src = x.src * (uint32_t)(TT * sizeof(T));
      ed_s[e] = x;
    }
  }

  // inputs -> value slots 0..I-1 (input key i lives in slot i)
  const int s0 = tile * TT + tid * S;
  const T* gin = in + gi * in_gstride;
  if (sizeof(T) == 4 && (I & 3) == 0) {
    for (int i4 = 0; i4 < I; i4 += 4) {
      float4 x[S];
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const int s = s0 + j;
        x[j] = s < B ? __ldg(reinterpret_cast<const float4*>(gin + (int64_t)s * I + i4))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      PackT p0, p1, p2, p3;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        p0.v[j] = (T)x[j].x; p1.v[j] = (T)x[j].y; p2.v[j] = (T)x[j].z; p3.v[j] = (T)x[j].w;
      }
      *reinterpret_cast<PackT*>(vals + (int64_t)(i4 + 0) * TT + tid * S) = p0;
      *reinterpret_cast<PackT*>(vals + (int64_t)(i4 + 1) * TT + tid * S) = p1;
      *reinterpret_cast<PackT*>(vals + (int64_t)(i4 + 2) * TT + tid * S) = p2;
      *reinterpret_cast<PackT*>(vals + (int64_t)(i4 + 3) * TT + tid * S) = p3;
    }
  } else {
    for (int i = 0; i < I; ++i) {
      PackT p;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const int s = s0 + j;
        p.v[j] = s < B ? gin[(int64_t)s * I + i] : T(0);
      }
      *reinterpret_cast<PackT*>(vals + (int64_t)i * TT + tid * S) = p;
    }
  }
  __syncthreads();

  // node sweep in program (topological) order
  const char* vb = reinterpret_cast<const char*>(vals) + tid * S * sizeof(T);
  for (int k = 0; k < n_steps; ++k) {
    const StepT<T> st = st_s[k];
    const EdgeT<T>* ep = ed_s + st.e_begin;
    const int ne = st.e_count;
    const int agg = st.agg;
    T acc[S];
    if (agg == AGG_SUM || agg == AGG_MEAN) {
      T a0[S], a1[S];
#pragma unroll
      for (int j = 0; j < S; ++j) { a0[j] = T(0); a1[j] = T(0); }
      int e = 0;
      for (; e + 2 <= ne; e += 2) {
        const EdgeT<T> x0 = ep[e], x1 = ep[e + 1];
        const PackT v0 = *reinterpret_cast<const PackT*>(vb + x0.src);
        const PackT v1 = *reinterpret_cast<const PackT*>(vb + x1.src);
#pragma unroll
        for (int j = 0; j < S; ++j) {
          a0[j] = fma(x0.w, v0.v[j], a0[j]);
          a1[j] = fma(x1.w, v1.v[j], a1[j]);
        }
      }
      if (e < ne) {
        const EdgeT<T> x0 = ep[e];
        const PackT v0 = *reinterpret_cast<const PackT*>(vb + x0.src);
#pragma unroll
        for (int j = 0; j < S; ++j) a0[j] = fma(x0.w, v0.v[j], a0[j]);
      }
#pragma unroll
      for (int j = 0; j < S; ++j) acc[j] = a0[j] + a1[j];
    } else {
      const T neutral = agg_neutral<T>(agg);
#pragma unroll
      for (int j = 0; j < S; ++j) acc[j] = neutral;
      for (int e = 0; e < ne; ++e) {
        const EdgeT<T> x0 = ep[e];
        const PackT v0 = *reinterpret_cast<const PackT*>(vb + x0.src);
#pragma unroll
        for (int j = 0; j < S; ++j) acc[j] = agg_combine<T>(agg, acc[j], x0.w * v0.v[j]);
      }
    }
    PackT y;
#pragma unroll
    for (int j = 0; j < S; ++j)
      y.v[j] = apply_act(st.act, fma(st.resp, agg_finish<T>(agg, acc[j], ne), st.bias));
    if (st.slot != NO_SLOT)
      *reinterpret_cast<PackT*>(vals + (int64_t)st.slot * TT + tid * S) = y;
  }

  // outputs (P, B, O)
  const uint16_t* os = reinterpret_cast<const uint16_t*>(gp + L.off_out);
  T* go = out + gi * out_gstride;
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int s = s0 + j;
    if (s >= B) break;
    T* row = go + (int64_t)s * O;
    for (int o = 0; o < O; ++o) {
      const uint16_t sl = __ldg(os + o);
      row[o] = sl != NO_SLOT ? vals[(int64_t)sl * TT + tid * S + j] : T(NAN);
    }
  }
}

// ---------------------------------------------------------------------------
// warp-per-genome kernel for small batches
// ---------------------------------------------------------------------------

template <typename T> __device__ __forceinline__ T warp_allreduce(int agg, T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = agg_combine<T>(agg, v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

enum : int { FIT_NONE = 0, FIT_XOR = 1, FIT_REGRESSION = 2 };

template <typename T>
__global__ void fwd_warp_kernel(const uint8_t* __restrict__ prog, ProgLayout L, int64_t P,
                                const T* __restrict__ in, int64_t in_gstride, int B, int I, int O,
                                int max_slots, T* __restrict__ out, int64_t out_gstride,
                                int fit_kind, const double* __restrict__ targets,
                                double* __restrict__ fitness) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t gi = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (gi >= P) return;
  T* vals = reinterpret_cast<T*>(smem) + (int64_t)warp * max_slots * B;  // [slot][B]
  const uint8_t* gp = prog + gi * L.stride;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const StepT<T>* steps = reinterpret_cast<const StepT<T>*>(gp + L.off_steps);
  const EdgeT<T>* edges = reinterpret_cast<const EdgeT<T>*>(gp + L.off_edges);
  const T* gin = in + gi * in_gstride;
  for (int idx = lane; idx < B * I; idx += 32) {
    const int b = idx / I, i = idx - b * I;
    vals[i * B + b] = gin[idx];
  }
  __syncwarp();
  for (int k = 0; k < hdr.n_steps; ++k) {
    const StepT<T> st = steps[k];
    const int agg = st.agg, ne = st.e_count;
    for (int b = 0; b < B; ++b) {
      T part = agg_neutral<T>(agg);
      for (int e = lane; e < ne; e += 32) {
        const EdgeT<T> x = edges[st.e_begin + e];
        part = agg_combine<T>(agg, part, x.w * vals[(int64_t)x.src * B + b]);
      }
      const T a = warp_allreduce<T>(agg, part);
      if (lane == 0 && st.slot != NO_SLOT)
        vals[(int64_t)st.slot * B + b] = apply_act(st.act, fma(st.resp, agg_finish<T>(agg, a, ne), st.bias));
    }
    __syncwarp();
  }
  const uint16_t* os = reinterpret_cast<const uint16_t*>(gp + L.off_out);
  if (fit_kind == FIT_NONE) {
    T* go = out + gi * out_gstride;
    for (int idx = lane; idx < B * O; idx += 32) {
      const int b = idx / O, o = idx - b * O;
      const uint16_t sl = os[o];
      go[idx] = sl != NO_SLOT ? vals[(int64_t)sl * B + b] : T(NAN);
    }
  } else if (lane == 0) {
    // fitness in float64 (problems.py:54-61), summation order of numpy for n < 8
    // (sequential) and 8-way pairwise blocks for 8 <= n <= 128
    const uint16_t sl = os[0];
    double r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    double acc = 0.0;
    const bool blocked = B >= 8;
    for (int b = 0; b < B; ++b) {
      const double y = (double)vals[(int64_t)sl * B + b];
      const double t = fit_kind == FIT_XOR ? (double)(((b >> 1) ^ b) & 1) : targets[b];
      const double d = (y - t) * (y - t);
      if (blocked) {
        if (b < (B & ~7)) r[b & 7] += d; else acc += d;
      } else {
        acc += d;
      }
    }
    double total = acc;
    if (blocked) total = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7])) + acc;
    fitness[gi] = fit_kind == FIT_XOR ? 4.0 - total : -(total / (double)B);
  }
}

template <typename T, int S, int NT>
int launch_tile(const uint8_t* prog, const ProgLayout& L, const T* in, int64_t in_gstride, int64_t P,
                int B, int I, int O, const int32_t* maxdims_host, T* out, int64_t out_gstride,
                cudaStream_t st) {
  constexpr int TT = NT * S;
  const int tiles = (B + TT - 1) / TT;
  const int64_t grid = P * tiles;
  if (grid > 0x7FFFFFFFll) return -5;
  const int64_t smem = align_up((int64_t)maxdims_host[1] * sizeof(StepT<T>), 16) +
                       align_up((int64_t)maxdims_host[2] * sizeof(EdgeT<T>), 16) +
                       (int64_t)maxdims_host[0] * TT * sizeof(T);
  if (smem > 227 * 1024) return -6;
  cudaFuncSetAttribute(fwd_tile_kernel<T, S, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fwd_tile_kernel<T, S, NT><<<(unsigned)grid, NT, smem, st>>>(prog, L, in, in_gstride, B, I, O, tiles,
                                                              out, out_gstride);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // namespace tneat

using namespace tneat;

extern "C" {

// Replaces inference.forward_arrays (inference.py:185-262).  See include/tneat.h.
int an_forward(const void* program, int64_t program_stride, int N, int C, int precision,
               const int32_t* maxdims_host, const void* inputs, int64_t input_genome_stride,
               int64_t P, int B, int I, int O, void* outputs, int variant, void* stream) {
  if (P < 0 || B < 0 || I < 1 || O < 1 || !maxdims_host) return -1;
  if (P == 0 || B == 0) return 0;
  if (!program || !inputs || !outputs) return -2;
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (L.stride != program_stride) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* pg = (const uint8_t*)program;
  const int64_t ogs = (int64_t)B * O;
  // variant: 0 = auto, 1 = tile S=1, 2 = tile S=2, 4 = tile S=4, 8 = warp kernel
  if (variant == 0) variant = B >= 96 ? 2 : 8;
  if (variant == 8) {
    const int wpb = 4;
    const int64_t smem = (int64_t)wpb * maxdims_host[0] * B * (precision ? 8 : 4);
    if (smem > 227 * 1024) return -6;
    const int64_t blocks = (P + wpb - 1) / wpb;
    if (precision) {
      cudaFuncSetAttribute(fwd_warp_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      fwd_warp_kernel<double><<<(unsigned)blocks, 32 * wpb, smem, st>>>(
          pg, L, P, (const double*)inputs, input_genome_stride, B, I, O, maxdims_host[0],
          (double*)outputs, ogs, FIT_NONE, nullptr, nullptr);
    } else {
      cudaFuncSetAttribute(fwd_warp_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      fwd_warp_kernel<float><<<(unsigned)blocks, 32 * wpb, smem, st>>>(
          pg, L, P, (const float*)inputs, input_genome_stride, B, I, O, maxdims_host[0],
          (float*)outputs, ogs, FIT_NONE, nullptr, nullptr);
    }
    TNEAT_CHECK_LAUNCH();
    return 0;
  }
  if (precision) {
    const double* in = (const double*)inputs;
    double* out = (double*)outputs;
    if (variant == 1) return launch_tile<double, 1, 128>(pg, L, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, st);
    return launch_tile<double, 2, 64>(pg, L, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, st);
  }
  const float* in = (const float*)inputs;
  float* out = (float*)outputs;
  switch (variant) {
    case 1: return launch_tile<float, 1, 128>(pg, L, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, st);
    case 4: return launch_tile<float, 4, 64>(pg, L, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, st);
    default: return launch_tile<float, 2, 64>(pg, L, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, st);
  }
}

// Fused forward + fitness for the built-in problems (problems.py:221-254):
// kind 1 = XOR (B=4, inputs = XOR table), kind 2 = regression (targets[B]).
int an_forward_fitness(const void* program, int64_t program_stride, int N, int C, int precision,
                       const int32_t* maxdims_host, const void* inputs, int64_t input_genome_stride,
                       int64_t P, int B, int I, int O, int kind, const double* targets,
                       double* fitness, void* stream) {
  if (P < 0 || B < 1 || I < 1 || O != 1 || !maxdims_host || (kind != 1 && kind != 2)) return -1;
  if (kind == 1 && B != 4) return -1;
  if (kind == 2 && !targets) return -2;
  if (P == 0) return 0;
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (L.stride != program_stride) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  const int wpb = 4;
  const int64_t smem = (int64_t)wpb * maxdims_host[0] * B * (precision ? 8 : 4);
  if (smem > 227 * 1024) return -6;
  const int64_t blocks = (P + wpb - 1) / wpb;
  if (precision) {
    cudaFuncSetAttribute(fwd_warp_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fwd_warp_kernel<double><<<(unsigned)blocks, 32 * wpb, smem, st>>>(
        (const uint8_t*)program, L, P, (const double*)inputs, input_genome_stride, B, I, O,
        maxdims_host[0], nullptr, 0, kind, targets, fitness);
  } else {
    cudaFuncSetAttribute(fwd_warp_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fwd_warp_kernel<float><<<(unsigned)blocks, 32 * wpb, smem, st>>>(
        (const uint8_t*)program, L, P, (const float*)inputs, input_genome_stride, B, I, O,
        maxdims_host[0], nullptr, 0, kind, targets, fitness);
  }
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
