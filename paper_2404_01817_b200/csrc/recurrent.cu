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
// Lanes own nodes (a sweep is max-in-degree deep, not node-count deep; nodes
// sorted by in-degree so the 32 deepest share one iteration) and environment
// rows; the warp needs no block barrier.

#include "common.cuh"

namespace tneat {

// shared memory of one warp: value buffers, environment vectors, then the
// genome's nodes in descending in-degree order and their edges as packed
// (source byte offset, weight) pairs
template <typename T>
struct __align__(8) RecEdge {
  uint32_t off;  // source slot * sizeof(T)
  T w;
};
template <typename T>
struct __align__(16) RecNode {
  uint16_t slot, count, e_begin;
  uint8_t act, agg;
  T bias, resp;
};
// environment rows padded to whole 16-byte vectors (zeros past D)
template <typename T>
__host__ __device__ inline int rollout_dp(int D) {
  constexpr int VW = 16 / (int)sizeof(T);
  return (D + VW - 1) / VW * VW;
}
// per warp: [s (Dp) | s_next (Dp) | actions (O) | values (slots) | values (slots)],
// then the node records and the edge records
template <typename T>
__host__ __device__ inline int64_t rollout_warp_bytes(int slots, int D, int O, int max_n, int max_e) {
  return align_up((2ll * slots + 2ll * rollout_dp<T>(D) + O) * (int64_t)sizeof(T), 16) +
         (int64_t)max_n * sizeof(RecNode<T>) + align_up((int64_t)max_e * sizeof(RecEdge<T>), 16);
}

template <typename T>
__device__ __forceinline__ T node_sum_act(const RecNode<T>& nd, T acc);
template <>
__device__ __forceinline__ float node_sum_act<float>(const RecNode<float>& nd, float acc) {
  return tanh_fast(fmaf(nd.resp, acc, nd.bias));
}
template <>
__device__ __forceinline__ double node_sum_act<double>(const RecNode<double>& nd, double acc) {
  return tanh(fma(nd.resp, acc, nd.bias));
}

template <typename T>
__global__ void rollout_kernel(const uint8_t* __restrict__ prog, ProgLayout L, int64_t P, int slots, int I, int O,
                               const T* __restrict__ A, const T* __restrict__ M, const T* __restrict__ s0, int D,
                               int steps, int sweeps, int max_n, int max_e, double* __restrict__ fitness) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gi = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  // environment matrices once per CTA (A rows padded to Dp with zeros)
  const int Dp = rollout_dp<T>(D);
  T* Am = reinterpret_cast<T*>(smem);
  T* Mm = Am + D * Dp;
  for (int i = threadIdx.x; i < D * Dp; i += blockDim.x) {
    const int r = i / Dp, c = i - r * Dp;
    Am[i] = c < D ? A[r * D + c] : T(0);
  }
  for (int i = threadIdx.x; i < D * O; i += blockDim.x) Mm[i] = M[i];
  __syncthreads();
  if (gi >= P) return;
  uint8_t* wbase = smem + align_up((int64_t)(D * Dp + D * O) * sizeof(T), 16) +
                   (int64_t)warp * rollout_warp_bytes<T>(slots, D, O, max_n, max_e);
  T* s = reinterpret_cast<T*>(wbase);  // environment state (Dp, zeros past D; 16-byte aligned)
  T* s_next = s + Dp;                   // (Dp)
  T* act = s_next + Dp;                 // actions (O)
  T* buf0 = act + O;
  T* buf1 = buf0 + slots;
  RecNode<T>* nodes =
      reinterpret_cast<RecNode<T>*>(wbase + align_up((2ll * slots + 2ll * Dp + O) * (int64_t)sizeof(T), 16));
  RecEdge<T>* edges = reinterpret_cast<RecEdge<T>*>(nodes + max_n);
  const uint8_t* gp = prog + gi * L.stride;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const StepT<T>* stp = reinterpret_cast<const StepT<T>*>(gp + L.off_steps);
  const GroupRec* grp = reinterpret_cast<const GroupRec*>(gp + L.off_groups);
  const uint16_t* esrc = reinterpret_cast<const uint16_t*>(gp + L.off_src);
  const float* ew = reinterpret_cast<const float*>(gp + L.off_w);
  const EdgeD* ed = reinterpret_cast<const EdgeD*>(gp + L.off_w);
  const uint16_t* out_slot = reinterpret_cast<const uint16_t*>(gp + L.off_out);
  const int n_steps = hdr.n_steps;
  // stage the program (recurrent programs: singleton groups, step j = group j):
  // position of step j = its rank by (in-degree descending, j) -- lanes take
  // positions lane, lane + 32, ...: the warp's edge rounds per sweep are the
  // sum over those iterations of the largest degree, which this order
  // minimises.  A node's edges keep their program order (the sum's order).
  for (int j = lane; j < n_steps; j += 32) {
    const int cj = stp[j].count;
    int rank = 0;
    for (int k = 0; k < n_steps; ++k) {
      const int ck = stp[k].count;
      rank += (ck > cj || (ck == cj && k < j)) ? 1 : 0;
    }
    buf0[j] = (T)rank;  // scratch: the value buffers are cleared below
  }
  __syncwarp();
  // edge offsets: exclusive scan of the counts in position order, each list
  // starting at an even record (two records = one 16-byte load for fp32)
  int carry = 0;
  for (int base = 0; base < n_steps; base += 32) {
    const int p = base + lane;
    int j = -1;
    for (int k = 0; k < n_steps && p < n_steps; ++k)
      if ((int)buf0[k] == p) { j = k; break; }
    const int c = j >= 0 ? ((int)stp[j].count + 1) & ~1 : 0;
    int x = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (j >= 0) {
      const StepT<T> st = stp[j];
      const int c0 = carry + x - c;
      RecNode<T> nd;
      nd.slot = st.slot;
      nd.count = st.count;
      nd.e_begin = (uint16_t)c0;
      nd.act = st.act;
      nd.agg = st.agg;
      nd.bias = st.bias;
      nd.resp = st.resp;
      nodes[p] = nd;
      const int g0 = grp[j].e_begin;
      for (int e = 0; e < (int)st.count; ++e) {
        RecEdge<T> r;
        if constexpr (sizeof(T) == 8) { r.off = ed[g0 + e].src * (uint32_t)sizeof(T); r.w = (T)ed[g0 + e].w; }
        else { r.off = (uint32_t)esrc[g0 + e] * (uint32_t)sizeof(T); r.w = (T)ew[g0 + e]; }
        edges[c0 + e] = r;
      }
    }
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  __syncwarp();
  for (int i = lane; i < slots; i += 32) { buf0[i] = T(0); buf1[i] = T(0); }
  for (int i = lane; i < Dp; i += 32) {
    s[i] = i < D ? s0[i] : T(0);
    s_next[i] = T(0);
  }
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
      const char* cb = reinterpret_cast<const char*>(cur);
      for (int p = lane; p < n_steps; p += 32) {
        const RecNode<T> nd = nodes[p];
        const RecEdge<T>* er = edges + nd.e_begin;
        const int cnt = nd.count;
        T v;
        if (nd.agg == AGG_SUM && nd.act == ACT_TANH) {  // the common node: inline, edges two at a time
          T acc = T(0);
          int e = 0;
          // four edges per iteration: the record and value loads of the four are
          // in flight together; the sum keeps the edge order
          for (; e + 4 <= cnt; e += 4) {
            RecEdge<T> r[4];
            if constexpr (sizeof(T) == 4) {
              const uint4 a = *reinterpret_cast<const uint4*>(er + e), b = *reinterpret_cast<const uint4*>(er + e + 2);
              r[0].off = a.x; r[0].w = __uint_as_float(a.y); r[1].off = a.z; r[1].w = __uint_as_float(a.w);
              r[2].off = b.x; r[2].w = __uint_as_float(b.y); r[3].off = b.z; r[3].w = __uint_as_float(b.w);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) r[u] = er[e + u];
            }
            T x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = *reinterpret_cast<const T*>(cb + r[u].off);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = acc + r[u].w * x[u];
          }
          for (; e < cnt; ++e) {
            const RecEdge<T> r0 = er[e];
            acc = acc + r0.w * *reinterpret_cast<const T*>(cb + r0.off);
          }
          v = node_sum_act<T>(nd, acc);
        } else {
          T acc;
          if (nd.agg == AGG_SUM || nd.agg == AGG_MEAN) {  // (mean divides in agg_finish)
            acc = T(0);
            for (int e = 0; e < cnt; ++e) acc = acc + er[e].w * *reinterpret_cast<const T*>(cb + er[e].off);
          } else {
            acc = agg_neutral<T>(nd.agg);
            for (int e = 0; e < cnt; ++e)
              acc = agg_combine<T>(nd.agg, acc, er[e].w * *reinterpret_cast<const T*>(cb + er[e].off));
          }
          const T a = agg_finish<T>(nd.agg, acc, cnt);
          if constexpr (sizeof(T) == 8) v = apply_act(nd.act, fma(nd.resp, a, nd.bias));
          else v = apply_act(nd.act, fmaf(nd.resp, a, nd.bias));
        }
        if (nd.slot != NO_SLOT) nxt[nd.slot] = v;
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
      // 16-byte loads of the row and the state, FMAs in column order (the padding adds 0 * 0)
      T z = T(0);
      const T* ar = Am + r * Dp;
      for (int c = 0; c < Dp; c += 16 / (int)sizeof(T)) {
        if constexpr (sizeof(T) == 4) {
          const float4 a = *reinterpret_cast<const float4*>(ar + c), v = *reinterpret_cast<const float4*>(s + c);
          z = fmaf(a.x, v.x, z); z = fmaf(a.y, v.y, z); z = fmaf(a.z, v.z, z); z = fmaf(a.w, v.w, z);
        } else {
          const double2 a = *reinterpret_cast<const double2*>(ar + c), v = *reinterpret_cast<const double2*>(s + c);
          z = fma(a.x, v.x, z); z = fma(a.y, v.y, z);
        }
      }
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
  // compact edges: at most one per connection, plus one pad record per node;
  // maxdims[2] (edge entries: every recurrent step its own group, padded to 8)
  // bounds the padded lists as well and is usually tighter
  const int max_n = max(maxdims_host[1], 1), max_e = max(min(C + max_n, maxdims_host[2]), 1);
  const int wpb = 4;
  const int64_t esz = precision ? 8 : 4;
  const int64_t per = precision ? rollout_warp_bytes<double>(slots, D, O, max_n, max_e)
                                : rollout_warp_bytes<float>(slots, D, O, max_n, max_e);
  const int64_t Dp = precision ? rollout_dp<double>(D) : rollout_dp<float>(D);
  const int64_t smem = align_up((int64_t)(D * Dp + D * O) * esz, 16) + per * wpb;
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
