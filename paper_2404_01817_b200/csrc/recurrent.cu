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

template <typename T>
__global__ void rollout_kernel(const uint8_t* __restrict__ prog, ProgLayout L, int64_t P, int slots, int I, int O,
                               const T* __restrict__ A, const T* __restrict__ M, const T* __restrict__ s0, int D,
                               int steps, int sweeps, double* __restrict__ fitness) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gi = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (gi >= P) return;
  const int per = 2 * slots + 2 * D + O;
  T* buf0 = reinterpret_cast<T*>(smem) + (int64_t)warp * per;
  T* buf1 = buf0 + slots;
  T* s = buf1 + slots;        // environment state (D)
  T* s_next = s + D;          // (D)
  T* act = s_next + D;        // actions (O)
  const uint8_t* gp = prog + gi * L.stride;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const StepT<T>* stp = reinterpret_cast<const StepT<T>*>(gp + L.off_steps);
  const GroupRec* grp = reinterpret_cast<const GroupRec*>(gp + L.off_groups);
  const uint16_t* esrc = reinterpret_cast<const uint16_t*>(gp + L.off_src);
  const float* ew = reinterpret_cast<const float*>(gp + L.off_w);
  const EdgeD* ed = reinterpret_cast<const EdgeD*>(gp + L.off_w);
  const uint16_t* out_slot = reinterpret_cast<const uint16_t*>(gp + L.off_out);
  for (int i = lane; i < slots; i += 32) { buf0[i] = T(0); buf1[i] = T(0); }
  for (int i = lane; i < D; i += 32) s[i] = s0[i];
  __syncwarp();
  T* cur = buf0;
  T* nxt = buf1;
  double reward = 0.0;
  const int n_steps = hdr.n_steps;
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
        const StepT<T> st = stp[j];
        const int e0 = grp[j].e_begin;  // recurrent programs: singleton groups, step j = group j
        T acc = agg_neutral<T>(st.agg);
        for (int e = 0; e < st.count; ++e) {
          uint32_t src;
          T w;
          if constexpr (sizeof(T) == 8) { src = ed[e0 + e].src; w = (T)ed[e0 + e].w; }
          else { src = esrc[e0 + e]; w = (T)ew[e0 + e]; }
          acc = agg_combine<T>(st.agg, acc, w * cur[src]);
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
      for (int c = 0; c < D; ++c) z = fma(A[r * D + c], s[c], z);
      for (int c = 0; c < O; ++c) z = fma(M[r * O + c], act[c], z);
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
  if (precision & FMT_SPLIT) return -7;
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (L.stride != program_stride) return -3;
  const int slots = max(maxdims_host[0], I);
  const int wpb = 4;
  const int64_t per = (2ll * slots + 2ll * D + O) * (precision ? 8 : 4);
  const int64_t smem = per * wpb;
  if (smem > 200 * 1024) return -6;
  const int64_t blocks = (P + wpb - 1) / wpb;
  cudaStream_t st = (cudaStream_t)stream;
  if (precision) {
    cudaFuncSetAttribute(rollout_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rollout_kernel<double><<<(unsigned)blocks, 32 * wpb, smem, st>>>((const uint8_t*)program, L, P, slots, I, O,
                                                                     (const double*)A, (const double*)M,
                                                                     (const double*)s0, D, steps, sweeps, fitness);
  } else {
    cudaFuncSetAttribute(rollout_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rollout_kernel<float><<<(unsigned)blocks, 32 * wpb, smem, st>>>((const uint8_t*)program, L, P, slots, I, O,
                                                                    (const float*)A, (const float*)M,
                                                                    (const float*)s0, D, steps, sweeps, fitness);
  }
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
