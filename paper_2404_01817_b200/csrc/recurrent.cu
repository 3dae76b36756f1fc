// K10: recurrent NEAT rollouts -- fixed-step synchronous activation inside a
// synthetic Ant-shaped environment, one warp per genome, state on chip.
//
// No reference implementation (the reference rejects recurrent genomes at
// transform time, SPEC.md:360 / inference.py:143).  Builder-
// defined semantics:
//   * the genome is compiled in recurrent mode (transform mode 1): every live
//     non-input node is a step with its own value slot, cycles allowed;
//   * per environment step the inputs are clamped to the observation and K
//     synchronous sweeps run: v'[n] = act(bias + resp * agg_j(w_j * v[src_j]))
//     computed from the previous sweep's values (double-buffered), node
//     values start at 0 and persist across environment steps;
//   * environment: s_{t+1} = tanh(A s_t + M a_t),
//     A (D x D), M (D x O) shared; observation = s_t, action a_t = outputs
//     after the K sweeps, reward = s_t[0]; fitness = sum over T steps.
// Lanes own nodes (a sweep is max-in-degree deep, not node-count deep) and
// environment rows; the warp needs no block barrier.

#include "common.cuh"

namespace tneat {

template <typename T>
__device__ __forceinline__ T node_value(const StepT<T>& st, T acc, int count);
template <>
__device__ __forceinline__ float node_value<float>(const StepT<float>& st, float acc, int count) {
  const float a = agg_finish<float>(st.agg, acc, count);
  return apply_act(st.act, fmaf(st.resp, a, st.bias));
}
template <>
__device__ __forceinline__ double node_value<double>(const StepT<double>& st, double acc, int count) {
  return apply_act(st.act, fma(st.resp, agg_finish<double>(st.agg, acc, count), st.bias));
}

// shared memory of one warp: value buffers, environment vectors, then the
// genome's step records and its edges compacted to the steps' real counts
template <typename T>
__host__ __device__ inline int64_t rollout_warp_bytes(int slots, int D, int O, int max_n, int max_e) {
  return align_up((2ll * slots + 2ll * D + O) * (int64_t)sizeof(T), 16) + (int64_t)max_n * sizeof(StepT<T>) +
         align_up((int64_t)max_e * sizeof(T), 16) + align_up(2ll * max_e, 16);
}

template <typename T>
__global__ void rollout_kernel(const uint8_t* __restrict__ prog, ProgLayout L, int64_t P, int slots, int I, int O,
                               const T* __restrict__ A, const T* __restrict__ M, const T* __restrict__ s0, int D,
                               int steps, int sweeps, int max_n, int max_e, double* __restrict__ fitness) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gi = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  // environment matrices once per CTA
  T* Am = reinterpret_cast<T*>(smem);
  T* Mm = Am + D * D;
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) Am[i] = A[i];
  for (int i = threadIdx.x; i < D * O; i += blockDim.x) Mm[i] = M[i];
  __syncthreads();
  if (gi >= P) return;
  uint8_t* wbase = smem + align_up((int64_t)(D * D + D * O) * sizeof(T), 16) +
                   (int64_t)warp * rollout_warp_bytes<T>(slots, D, O, max_n, max_e);
  T* buf0 = reinterpret_cast<T*>(wbase);
  T* buf1 = buf0 + slots;
  T* s = buf1 + slots;        // environment state (D)
  T* s_next = s + D;          // (D)
  T* act = s_next + D;        // actions (O)
  StepT<T>* rec = reinterpret_cast<StepT<T>*>(wbase + align_up((2ll * slots + 2ll * D + O) * (int64_t)sizeof(T), 16));
  T* wt = reinterpret_cast<T*>(rec + max_n);
  uint16_t* srcs = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(wt) + align_up((int64_t)max_e * sizeof(T), 16));
  const uint8_t* gp = prog + gi * L.stride;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const StepT<T>* stp = reinterpret_cast<const StepT<T>*>(gp + L.off_steps);
  const GroupRec* grp = reinterpret_cast<const GroupRec*>(gp + L.off_groups);
  const uint16_t* esrc = reinterpret_cast<const uint16_t*>(gp + L.off_src);
  const float* ew = reinterpret_cast<const float*>(gp + L.off_w);
  const EdgeD* ed = reinterpret_cast<const EdgeD*>(gp + L.off_w);
  const uint16_t* out_slot = reinterpret_cast<const uint16_t*>(gp + L.off_out);
  const int n_steps = hdr.n_steps;
  // stage the program: step records (pad = compact first edge) and the edges
  // of every step back to back (recurrent programs: singleton groups, step j =
  // group j)
  int carry = 0;
  for (int base = 0; base < n_steps; base += 32) {
    const int j = base + lane;
    StepT<T> st;
    int c = 0;
    if (j < n_steps) { st = stp[j]; c = st.count; }
    int x = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (j < n_steps) {
      const int c0 = carry + x - c;
      st.pad = (uint16_t)c0;
      rec[j] = st;
      const int g0 = grp[j].e_begin;
      for (int e = 0; e < c; ++e) {
        if constexpr (sizeof(T) == 8) { srcs[c0 + e] = (uint16_t)ed[g0 + e].src; wt[c0 + e] = (T)ed[g0 + e].w; }
        else { srcs[c0 + e] = esrc[g0 + e]; wt[c0 + e] = (T)ew[g0 + e]; }
      }
    }
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  for (int i = lane; i < slots; i += 32) { buf0[i] = T(0); buf1[i] = T(0); }
  for (int i = lane; i < D; i += 32) s[i] = s0[i];
  __syncwarp();
  T* cur = buf0;
  T* nxt = buf1;
  double reward = 0.0;
  for (int t = 0; t < steps; ++t) {
    reward += (double)s[0];
    for (int i = lane; i < I; i += 32) {  // observation -> input slots of both buffers
      const T v = i < D ? s[i] : T(0);
      cur[i] = v;
      nxt[i] = v;
    }
    __syncwarp();
    for (int k = 0; k < sweeps; ++k) {
      for (int j = lane; j < n_steps; j += 32) {
        const StepT<T> st = rec[j];
        const int e0 = st.pad;
        T acc;
        if (st.agg == AGG_SUM || st.agg == AGG_MEAN) {  // (mean divides in node_value)
          acc = T(0);
          for (int e = 0; e < st.count; ++e) acc = acc + wt[e0 + e] * cur[srcs[e0 + e]];
        } else {
          acc = agg_neutral<T>(st.agg);
          for (int e = 0; e < st.count; ++e) acc = agg_combine<T>(st.agg, acc, wt[e0 + e] * cur[srcs[e0 + e]]);
        }
        if (st.slot != NO_SLOT) nxt[st.slot] = node_value<T>(st, acc, st.count);
      }
      __syncwarp();
      T* tmp = cur; cur = nxt; nxt = tmp;
    }
    for (int o = lane; o < O; o += 32) {
      const uint16_t sl = out_slot[o];
      act[o] = sl != NO_SLOT ? cur[sl] : T(0);
    }
    __syncwarp();
    // s <- tanh(A s + M a)
    for (int r = lane; r < D; r += 32) {
      T z = T(0);
      for (int c = 0; c < D; ++c) z = fma(Am[r * D + c], s[c], z);
      for (int c = 0; c < O; ++c) z = fma(Mm[r * O + c], act[c], z);
      s_next[r] = tanh(z);
    }
    __syncwarp();
    for (int r = lane; r < D; r += 32) s[r] = s_next[r];
    __syncwarp();
  }
  if (lane == 0) fitness[gi] = reward;
}

}  // namespace tneat

using namespace tneat;

extern "C" {

// Recurrent rollouts (builder-defined, see file header): program compiled with
// an_transform mode 1; A (D,D), M (D,O), s0 (D,) in the program's precision;
// fitness (P,) float64 = sum_t s_t[0] over `steps` environment steps with
// `sweeps` synchronous activation sweeps per step.
int an_rollout(const void* program, int64_t program_stride, int N, int C, int precision,
               const int32_t* maxdims_host, int64_t P, int I, int O, const void* A, const void* M, const void* s0,
               int D, int steps, int sweeps, double* fitness, void* stream) {
  if (P < 0 || !maxdims_host || D < 1 || steps < 0 || sweeps < 1 || I < 1 || O < 1) return -1;
  if (P == 0) return 0;
  if (precision & FMT_TC) return -7;  // standard programs only
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (L.stride != program_stride) return -3;
  const int slots = max(maxdims_host[0], I);
  const int max_n = max(maxdims_host[1], 1), max_e = max(C, 1);  // compact edges: at most one per connection
  const int wpb = 4;
  const int64_t esz = precision ? 8 : 4;
  const int64_t per = precision ? rollout_warp_bytes<double>(slots, D, O, max_n, max_e)
                                : rollout_warp_bytes<float>(slots, D, O, max_n, max_e);
  const int64_t smem = align_up((int64_t)(D * D + D * O) * esz, 16) + per * wpb;
  if (smem > 200 * 1024) return -6;
  const int64_t blocks = (P + wpb - 1) / wpb;
  cudaStream_t st = (cudaStream_t)stream;
  if (precision) {
    cudaFuncSetAttribute(rollout_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rollout_kernel<double><<<(unsigned)blocks, 32 * wpb, smem, st>>>((const uint8_t*)program, L, P, slots, I, O,
                                                                     (const double*)A, (const double*)M,
                                                                     (const double*)s0, D, steps, sweeps, max_n,
                                                                     max_e, fitness);
  } else {
    cudaFuncSetAttribute(rollout_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rollout_kernel<float><<<(unsigned)blocks, 32 * wpb, smem, st>>>((const uint8_t*)program, L, P, slots, I, O,
                                                                    (const float*)A, (const float*)M,
                                                                    (const float*)s0, D, steps, sweeps, max_n, max_e,
                                                                    fitness);
  }
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
