// K2: population forward -- executes transform programs over input batches.
//
// Replaces arrayneat inference.forward_arrays (inference.py:185-262).
//
// Kernels:
//   * fwd_tile (default for large batches, config 2: B = 4096): one CTA per
//     (genome, run of tiles of NT*S inputs).  Each thread owns S consecutive
//     inputs; node values live in shared memory as [slot][tile] (inputs staged
//     from HBM with coalesced 16-byte loads, the next tile prefetched into L2 by
//     the TMA engine), so a thread only ever reads values it wrote itself -- no
//     barrier inside the node sweep.  Steps run a group at a time (<= 4
//     independent same-level nodes with interleaved edge lists): the group's
//     nodes accumulate in lock-step as independent FFMA2 chains (two samples
//     per instruction); padding entries read a zero slot so every round is
//     unpredicated; program words are warp-uniform 16-byte loads, prefetched
//     one group ahead.
//   * fwd_warp: one warp per (genome, input chunk); lanes split a node's incoming
//     edges and combine with warp-shuffle reductions (sum/product/max/min/mean).
//     For small batches (XOR B=4, regression B=64, cart-pole B=1) where a
//     thread-per-input mapping would idle most lanes.  Optionally fuses the
//     XOR / regression fitness epilogue (problems.py:54-61).
//   * fwd_tc (FMT_TC programs, config 2's default): the input-sourced edges
//     of every step as one exact digit-split tcgen05 MMA per 128-sample tile
//     (csrc/digits.cuh), the hidden-sourced edges swept on CUDA cores.
//
// Semantics: input rows hold raw inputs and are never
// activated; node = act(bias + response * agg(w * v)); empty aggregation = 0;
// mean divides by the incoming count; outputs read at the rows of keys I..I+O-1.

#include "common.cuh"
#include "tc.cuh"
#include "digits.cuh"
#include "tmap.cuh"
#include <cuda_fp16.h>

namespace tneat {

template <typename T, int S> struct __align__(sizeof(T) * S) Pack { T v[S]; };

// TMA-engine prefetch of a contiguous block into L2 (bytes: multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// finish one step: aggregate -> bias + response * agg -> activation -> slot
template <int S, int RB>
__device__ __forceinline__ void finish_step(const StepT<float>& st, const float (&acc)[S], char* vb) {
  Pack<float, S> y;
  const int act = st.act;
  const float kx = act == ACT_TANH ? -2.8853900817779268f : (act == ACT_SIGMOID ? -1.4426950408889634f : 0.0f);
  const float ca = act == ACT_TANH ? 2.0f : 1.0f;
  const float cb = act == ACT_TANH ? -1.0f : 0.0f;
#pragma unroll
  for (int j = 0; j < S; ++j) {
    float a = acc[j];
    if (st.agg == AGG_MEAN) a = st.count ? __fdividef(a, (float)st.count) : 0.0f;
    y.v[j] = step_act(kx, ca, cb, act == ACT_RELU, fmaf(st.resp, a, st.bias));
  }
  if (st.slot != NO_SLOT) *reinterpret_cast<Pack<float, S>*>(vb + st.slot * RB) = y;
}
template <int S, int RB>
__device__ __forceinline__ void finish_step(const StepT<double>& st, const double (&acc)[S], char* vb) {
  Pack<double, S> y;
#pragma unroll
  for (int j = 0; j < S; ++j)
    y.v[j] = apply_act(st.act, fma(st.resp, agg_finish<double>(st.agg, acc[j], st.count), st.bias));
  if (st.slot != NO_SLOT) *reinterpret_cast<Pack<double, S>*>(vb + st.slot * RB) = y;
}

template <int N> struct U16Vec;
template <> struct U16Vec<2> { using type = uint32_t; };
template <> struct U16Vec<4> { using type = uint2; };
template <> struct U16Vec<8> { using type = uint4; };
template <int N> struct F32Vec;
template <> struct F32Vec<2> { using type = float2; };
template <> struct F32Vec<4> { using type = float4; };

template <int N>
__device__ __forceinline__ void load_u16(const uint16_t* p, uint32_t (&out)[N]) {
  using V = typename U16Vec<N>::type;
  const V v = *reinterpret_cast<const V*>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) { out[2 * i] = w[i] & 0xFFFFu; out[2 * i + 1] = w[i] >> 16; }
}
template <int N>
__device__ __forceinline__ void load_f32(const float* p, float (&out)[N]) {
  if constexpr (N == 2) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    out[0] = v.x; out[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      const float4 v = reinterpret_cast<const float4*>(p)[i];
      out[4 * i] = v.x; out[4 * i + 1] = v.y; out[4 * i + 2] = v.z; out[4 * i + 3] = v.w;
    }
  }
}

template <int N>
__device__ __forceinline__ void load_u32(const uint32_t* p, uint32_t (&out)[N]) {
  if constexpr (N == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    out[0] = v.x; out[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[i];
      out[4 * i] = v.x; out[4 * i + 1] = v.y; out[4 * i + 2] = v.z; out[4 * i + 3] = v.w;
    }
  }
}

// the first two rounds' program words of a group (<= 8 entries for GW <= 4),
// loaded one group ahead by the sweep loop
struct Words {
  uint32_t o[8];
  float w[8];
};
__device__ __forceinline__ void load_words(Words& d, const uint32_t* off_s, const float* w_s, int e) {
  load_u32<8>(off_s + e, d.o);
  load_f32<8>(w_s + e, d.w);
}

// two rounds of a sum group: 2*GW value loads (byte offsets into the thread's
// value column), then one FFMA2 (or FFMA for S = 1) per edge and sample pair
template <int S, int G, int GW, typename OffA, typename WA>
__device__ __forceinline__ void sum_rounds(float2 (&acc)[G][(S + 1) / 2], const OffA& off, const WA& w,
                                           const char* vb) {
  using PackT = Pack<float, S>;
  PackT v[2 * GW];
#pragma unroll
  for (int q = 0; q < 2 * GW; ++q)
    if (q % GW < G) {
#ifdef TNEAT_DIAG_NOLDS  // diagnostic builds only: value loads replaced by the offset
      for (int s = 0; s < S; ++s) v[q].v[s] = __uint_as_float(off[q]);
#else
      v[q] = *reinterpret_cast<const PackT*>(vb + off[q]);
#endif
    }
#pragma unroll
  for (int q = 0; q < 2 * GW; ++q)
    if (q % GW < G) {
      if constexpr (S == 1) {
        acc[q % GW][0].x = fmaf(w[q], v[q].v[0], acc[q % GW][0].x);
      } else {
#pragma unroll
        for (int p = 0; p < S / 2; ++p)  // one FFMA2 per edge and sample pair (exact fp32 FMA per lane)
          acc[q % GW][p] = __ffma2_rn(make_float2(w[q], w[q]), make_float2(v[q].v[2 * p], v[q].v[2 * p + 1]),
                                      acc[q % GW][p]);
      }
    }
}

// one round (the first GW entries of a two-round buffer)
template <int S, int G, int GW, typename OffA, typename WA>
__device__ __forceinline__ void sum_round1(float2 (&acc)[G][(S + 1) / 2], const OffA& off, const WA& w,
                                           const char* vb) {
  using PackT = Pack<float, S>;
  PackT v[GW];
#pragma unroll
  for (int q = 0; q < G; ++q) v[q] = *reinterpret_cast<const PackT*>(vb + off[q]);
#pragma unroll
  for (int q = 0; q < G; ++q) {
    if constexpr (S == 1) {
      acc[q][0].x = fmaf(w[q], v[q].v[0], acc[q][0].x);
    } else {
#pragma unroll
      for (int p = 0; p < S / 2; ++p)
        acc[q][p] = __ffma2_rn(make_float2(w[q], w[q]), make_float2(v[q].v[2 * p], v[q].v[2 * p + 1]), acc[q][p]);
    }
  }
}

// One sum/mean group of G steps (fp32 program): edge block of width GW = G|4,
// two rounds per step of the pipeline (2*GW byte offsets in <= two 16-byte
// loads, weights likewise) and up to 2G independent value loads / FMA chains,
// all unpredicated (holes are zero-slot entries).  Program words are
// double-buffered: the next two rounds' words load while this pair's values
// are in flight (the look-ahead past the block's end stays inside shared
// memory: weights and value slots follow the offsets).  TANH: every step is
// tanh/sum (short epilogue).
// MERGE (GRP_SPLIT0 groups of 3 steps): G = 4 columns, column 3 continues
// step 0 and is added into it before the epilogue
// INIT (TC programs): every step owns slot step_begin + j, which holds the
// step's input-layer partial sum on entry (the accumulator's initial value)
template <int S, int G, int RB, bool TANH, bool MERGE = false, bool INIT = false>
__device__ __forceinline__ void run_sum_group(const GroupRec& gr, const uint32_t* __restrict__ off_s,
                                              const float* __restrict__ w_s,
                                              const StepT<float>* __restrict__ st, char* vb, Words& wd,
                                              int next_e) {
  constexpr int GW = G == 3 ? 4 : G;
  constexpr int NS = MERGE ? G - 1 : G;  // steps
  constexpr int SP = (S + 1) / 2;  // sample pairs: Blackwell packed fp32 (FFMA2 / FADD2)
  using PackT = Pack<float, S>;
  float2 acc[G][SP];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int p = 0; p < SP; ++p) acc[j][p] = make_float2(0.0f, 0.0f);
  if constexpr (INIT) {
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const PackT v = *reinterpret_cast<const PackT*>(vb + (uint32_t)(gr.step_begin + j) * RB);
#pragma unroll
      for (int p = 0; p < SP; ++p) acc[j][p] = make_float2(v.v[2 * p], S > 2 * p + 1 ? v.v[(2 * p + 1) % S] : 0.0f);
    }
  }
  // step records are read up front so the epilogue does not wait on them
  uint32_t slot_j[G];
  float rk_j[G], bk_j[G];
  if constexpr (TANH) {
    constexpr float K = -2.8853900817779268f;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const StepT<float> sj = st[j];
      slot_j[j] = INIT ? (uint32_t)(gr.step_begin + j) : sj.slot;
      rk_j[j] = INIT ? sj.resp : sj.resp * K;  // TC programs store them pre-scaled (common.cuh GroupTC)
      bk_j[j] = INIT ? sj.bias : sj.bias * K;
    }
  }
  const uint32_t* op = off_s + gr.e_begin;
  const float* wp = w_s + gr.e_begin;
  const int rounds = gr.rounds;  // holes read the zero slot with weight 0
  uint32_t oa[2 * GW], ob[2 * GW];
  float wa[2 * GW], wb[2 * GW];
  // rounds 0-1 come from `wd` (prefetched by the previous group); after the
  // last round `wd` takes the next group's first words in place (no copies)
  bool more = false;
  if (rounds < 2) {
    if (rounds == 1) sum_round1<S, G, GW>(acc, wd.o, wd.w, vb);
  } else {
    load_u32<2 * GW>(op + 2 * GW, ob);
    load_f32<2 * GW>(wp + 2 * GW, wb);
    sum_rounds<S, G, GW>(acc, wd.o, wd.w, vb);
    if (rounds < 4) {
      if (rounds == 3) sum_round1<S, G, GW>(acc, ob, wb, vb);
    } else {
      load_u32<2 * GW>(op + 4 * GW, oa);
      load_f32<2 * GW>(wp + 4 * GW, wa);
      sum_rounds<S, G, GW>(acc, ob, wb, vb);
      more = true;
    }
  }
  // round pairs from alternating buffers (loads one pair ahead; `oa` holds
  // rounds r, r+1 on entry), a single exit so the accumulators keep their
  // registers across iterations; then the last 0-3 rounds
  if (more) {
    int r = 4;
#pragma unroll 1
    for (; r + 4 <= rounds; r += 4) {
      load_u32<2 * GW>(op + (r + 2) * GW, ob);
      load_f32<2 * GW>(wp + (r + 2) * GW, wb);
      sum_rounds<S, G, GW>(acc, oa, wa, vb);
      load_u32<2 * GW>(op + (r + 4) * GW, oa);
      load_f32<2 * GW>(wp + (r + 4) * GW, wa);
      sum_rounds<S, G, GW>(acc, ob, wb, vb);
    }
    const int rem = rounds - r;
    if (rem >= 2) {
      if (rem == 3) {
        load_u32<2 * GW>(op + (r + 2) * GW, ob);
        load_f32<2 * GW>(wp + (r + 2) * GW, wb);
      }
      sum_rounds<S, G, GW>(acc, oa, wa, vb);
      if (rem == 3) sum_round1<S, G, GW>(acc, ob, wb, vb);
    } else if (rem == 1) {
      sum_round1<S, G, GW>(acc, oa, wa, vb);
    }
  }
  load_words(wd, off_s, w_s, next_e);  // in flight during the epilogue
  if constexpr (MERGE) {
#pragma unroll
    for (int p = 0; p < SP; ++p) acc[0][p] = __fadd2_rn(acc[0][p], acc[G - 1][p]);
  }
  if constexpr (TANH) {
    const uint32_t vbs = (uint32_t)__cvta_generic_to_shared(vb);
    // tanh(b + r*a) = 2 / (1 + 2^(k (b + r*a))) - 1, k = -2 log2(e): one FFMA into
    // EX2 (k folded into b and r once per step), FADD, RCP, FFMA -- |err| <~ 2e-7
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const float rk = rk_j[j], bk = bk_j[j];
      PackT y;
      if constexpr (S == 1) {
        y.v[0] = fmaf(2.0f, rcp_approx(1.0f + ex2_approx(fmaf(rk, acc[j][0].x, bk))), -1.0f);
      } else {
#pragma unroll
        for (int p = 0; p < SP; ++p) {
          const float2 t = __ffma2_rn(make_float2(rk, rk), acc[j][p], make_float2(bk, bk));
#ifdef TNEAT_DIAG_NOACT  // diagnostic builds only: no MUFU in the epilogue
          const float2 yy = t;
#else
          const float2 d = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(ex2_approx(t.x), ex2_approx(t.y)));
          const float2 yy = __ffma2_rn(make_float2(2.0f, 2.0f), make_float2(rcp_approx(d.x), rcp_approx(d.y)),
                                       make_float2(-1.0f, -1.0f));
#endif
          y.v[2 * p] = yy.x;
          y.v[2 * p + 1] = yy.y;
        }
      }
      // every step has a slot (the transform gives unread steps a scratch slot)
      if constexpr (S == 2) {  // explicit shared store: the window base is computed once per group
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(vbs + slot_j[j] * RB), "f"(y.v[0]), "f"(y.v[1])
                     : "memory");
      } else {
        *reinterpret_cast<PackT*>(vb + slot_j[j] * RB) = y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      float a[S];
#pragma unroll
      for (int s = 0; s < S; ++s) a[s] = (s & 1) ? acc[j][s / 2].y : acc[j][s / 2].x;
      finish_step<S, RB>(st[j], a, vb);
    }
  }
}

// fp64 program group (parity mode): same structure, (src, w) pairs
template <int S, int G, int RB>
__device__ __forceinline__ void run_sum_group_f64(const GroupRec& gr, const EdgeD* __restrict__ ed_s,
                                                  const StepT<double>* __restrict__ st, char* vb) {
  constexpr int GW = G == 3 ? 4 : G;
  double acc[G][S];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int s = 0; s < S; ++s) acc[j][s] = 0.0;
  const EdgeD* ep = ed_s + gr.e_begin;
  for (int r = 0; r < gr.rounds; ++r) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (r < gr.cnt[j]) {
        const EdgeD d = ep[r * GW + j];
        const Pack<double, S> v = *reinterpret_cast<const Pack<double, S>*>(vb + d.src * RB);
#pragma unroll
        for (int s = 0; s < S; ++s) acc[j][s] = fma(d.w, v.v[s], acc[j][s]);
      }
    }
  }
  if constexpr (G == 3) {
    if (gr.cls & GRP_SPLIT0) {  // step 0's second half (column 3), after its first: the list order
      for (int r = 0; r < gr.cnt[3]; ++r) {
        const EdgeD d = ep[r * GW + 3];
        const Pack<double, S> v = *reinterpret_cast<const Pack<double, S>*>(vb + d.src * RB);
#pragma unroll
        for (int s = 0; s < S; ++s) acc[0][s] = fma(d.w, v.v[s], acc[0][s]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) finish_step<S, RB>(st[j], acc[j], vb);
}

// singleton group with a non-sum aggregation (product / max / min), exact
// count; the aggregation is a template parameter (no per-edge dispatch) and the
// edges go two at a time (both value loads in flight before the combines)
template <typename T, int AGG>
__device__ __forceinline__ T agg_step(T acc, T x) {
  if constexpr (AGG == AGG_PRODUCT) return acc * x;
  // numpy's maximum / minimum (the reference's max reduction): a NaN on either
  // side wins, ties keep the accumulator
  else if constexpr (AGG == AGG_MAX) return (acc >= x || acc != acc) ? acc : x;
  else if constexpr (AGG == AGG_MIN) return (acc <= x || acc != acc) ? acc : x;
  else return acc + x;
}

template <typename T, int S, int RB, int AGG>
__device__ __forceinline__ void generic_edges(T (&acc)[S], int e_begin, int count, const uint32_t* __restrict__ off_s,
                                              const float* __restrict__ w_s, const EdgeD* __restrict__ ed_s,
                                              const char* vb) {
  auto edge = [&](int e, uint32_t& off, T& w) {
    if constexpr (sizeof(T) == 8) { off = ed_s[e_begin + e].src * RB; w = ed_s[e_begin + e].w; }
    else { off = off_s[e_begin + e]; w = w_s[e_begin + e]; }
  };
  int e = 0;
  for (; e + 2 <= count; e += 2) {
    uint32_t o0, o1;
    T w0, w1;
    edge(e, o0, w0);
    edge(e + 1, o1, w1);
    const Pack<T, S> v0 = *reinterpret_cast<const Pack<T, S>*>(vb + o0);
    const Pack<T, S> v1 = *reinterpret_cast<const Pack<T, S>*>(vb + o1);
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = agg_step<T, AGG>(agg_step<T, AGG>(acc[s], w0 * v0.v[s]), w1 * v1.v[s]);
  }
  if (e < count) {
    uint32_t o0;
    T w0;
    edge(e, o0, w0);
    const Pack<T, S> v0 = *reinterpret_cast<const Pack<T, S>*>(vb + o0);
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = agg_step<T, AGG>(acc[s], w0 * v0.v[s]);
  }
}

template <typename T, int S, int RB>
__device__ __forceinline__ void run_generic_step(const GroupRec& gr, const uint32_t* __restrict__ off_s,
                                                 const float* __restrict__ w_s, const EdgeD* __restrict__ ed_s,
                                                 const StepT<T>& st, char* vb) {
  T acc[S];
  const T neutral = agg_neutral<T>(st.agg);
#pragma unroll
  for (int s = 0; s < S; ++s) acc[s] = neutral;
  switch (st.agg) {
    case AGG_PRODUCT: generic_edges<T, S, RB, AGG_PRODUCT>(acc, gr.e_begin, st.count, off_s, w_s, ed_s, vb); break;
    case AGG_MAX: generic_edges<T, S, RB, AGG_MAX>(acc, gr.e_begin, st.count, off_s, w_s, ed_s, vb); break;
    case AGG_MIN: generic_edges<T, S, RB, AGG_MIN>(acc, gr.e_begin, st.count, off_s, w_s, ed_s, vb); break;
    default: generic_edges<T, S, RB, AGG_SUM>(acc, gr.e_begin, st.count, off_s, w_s, ed_s, vb); break;
  }
  if (st.count == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = T(0);
  }
  StepT<T> sum_like = st;
  sum_like.agg = AGG_SUM;  // acc already aggregated
  finish_step<S, RB>(sum_like, acc, vb);
}

template <typename T, int S, int RB>
__device__ __forceinline__ void run_group(const GroupRec& gr, const uint32_t* src_s, const float* w_s,
                                          const EdgeD* ed_s, const StepT<T>* st, char* vb, Words& wd,
                                          int next_e) {
  if (!(gr.cls & GRP_GENERIC)) {
    if constexpr (sizeof(T) == 4) {
      if (gr.cls & GRP_TANH_SUM) {
        switch (gr.n) {
          case 1: run_sum_group<S, 1, RB, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
          case 2: run_sum_group<S, 2, RB, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
          case 3:
            if (gr.cls & GRP_SPLIT0) run_sum_group<S, 4, RB, true, true>(gr, src_s, w_s, st, vb, wd, next_e);
            else run_sum_group<S, 3, RB, true>(gr, src_s, w_s, st, vb, wd, next_e);
            break;
          default: run_sum_group<S, 4, RB, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
        }
      } else {
        switch (gr.n) {
          case 1: run_sum_group<S, 1, RB, false>(gr, src_s, w_s, st, vb, wd, next_e); break;
          case 2: run_sum_group<S, 2, RB, false>(gr, src_s, w_s, st, vb, wd, next_e); break;
          case 3:
            if (gr.cls & GRP_SPLIT0) run_sum_group<S, 4, RB, false, true>(gr, src_s, w_s, st, vb, wd, next_e);
            else run_sum_group<S, 3, RB, false>(gr, src_s, w_s, st, vb, wd, next_e);
            break;
          default: run_sum_group<S, 4, RB, false>(gr, src_s, w_s, st, vb, wd, next_e); break;
        }
      }
    } else {
      switch (gr.n) {
        case 1: run_sum_group_f64<S, 1, RB>(gr, ed_s, st, vb); break;
        case 2: run_sum_group_f64<S, 2, RB>(gr, ed_s, st, vb); break;
        case 3: run_sum_group_f64<S, 3, RB>(gr, ed_s, st, vb); break;
        default: run_sum_group_f64<S, 4, RB>(gr, ed_s, st, vb); break;
      }
    }
  } else {
    if constexpr (sizeof(T) == 4) load_words(wd, src_s, w_s, next_e);
    run_generic_step<T, S, RB>(gr, src_s, w_s, ed_s, st[0], vb);
  }
}

// register cap: at least TNEAT_TILE_WARPS resident warps per SM (shared memory
// permitting), i.e. <= 64K / (32 * warps) registers per thread
#ifndef TNEAT_TILE_WARPS
#define TNEAT_TILE_WARPS 16
#endif
#define TNEAT_TILE_MINB(nt) (TNEAT_TILE_WARPS * 32 / (nt) > 0 ? TNEAT_TILE_WARPS * 32 / (nt) : 1)

// grid: one CTA per (genome, run of `tpc` consecutive tiles); the genome's
// program is staged in shared memory once and reused for every tile
template <typename T, int S, int NT>
__device__ __forceinline__ void tile_task(const uint8_t* __restrict__ prog, const ProgLayout& L,
                                          const int32_t* __restrict__ genome_ids, const T* __restrict__ in,
                                          int64_t in_gstride, int B, int I, int O, int64_t task, int run, int tpc,
                                          T* __restrict__ out, int64_t out_gstride, float* __restrict__ gsq) {
  constexpr int TT = NT * S;
  constexpr int RB = (TT + S) * sizeof(T);  // bytes of one value slot row (padded by S)
  using PackT = Pack<T, S>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int64_t gi = genome_ids ? (int64_t)__ldg(genome_ids + task) : task;
  const uint8_t* gp = prog + gi * L.stride;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const int n_steps = hdr.n_steps, n_edges = hdr.n_edges, n_groups = hdr.n_groups;
  const int tid = threadIdx.x;

  // shared memory: groups | steps | edge sources | edge weights | values [slot][TT]
  GroupRec* gr_s = reinterpret_cast<GroupRec*>(smem);
  const int64_t off_st = (int64_t)n_groups * sizeof(GroupRec);
  StepT<T>* st_s = reinterpret_cast<StepT<T>*>(smem + off_st);
  const int64_t off_src = off_st + (int64_t)n_steps * sizeof(StepT<T>);
  // fp32: u16 source slots are expanded to u32 byte offsets (slot * RB) in shared memory
  const int64_t src_bytes = sizeof(T) == 8 ? 0 : align_up(4ll * n_edges, 16);
  const int64_t off_w = off_src + src_bytes;
  const int64_t w_bytes = sizeof(T) == 8 ? 16ll * n_edges : 4ll * n_edges;
  uint32_t* src_s = reinterpret_cast<uint32_t*>(smem + off_src);
  float* w_s = reinterpret_cast<float*>(smem + off_w);
  EdgeD* ed_s = reinterpret_cast<EdgeD*>(smem + off_w);
  T* vals = reinterpret_cast<T*>(smem + align_up(off_w + w_bytes, 16));
  TNEAT_DCHECK(align_up(off_w + w_bytes, 16) + (int64_t)hdr.n_slots * RB <= (int64_t)dynamic_smem_bytes(),
               "tile program + value slots fit shared memory", hdr.n_slots, dynamic_smem_bytes());
#ifdef TNEAT_CHECKS
  if (sizeof(T) == 4) {  // every entry a sum group sweeps reads a value slot
    const uint16_t* gsrc = reinterpret_cast<const uint16_t*>(gp + L.off_src);
    const GroupRec* grs = reinterpret_cast<const GroupRec*>(gp + L.off_groups);
    for (int g = threadIdx.x; g < n_groups; g += blockDim.x) {
      const GroupRec r = grs[g];
      const int gw = group_width(r.n);
      if (r.cls & GRP_GENERIC) continue;
      TNEAT_DCHECK(r.e_begin + gw * r.rounds <= n_edges, "tile group record", r.e_begin + gw * r.rounds, n_edges);
      for (int e = r.e_begin; e < r.e_begin + gw * r.rounds; ++e)
        TNEAT_DCHECK(gsrc[e] < hdr.n_slots, "tile edge source slot", gsrc[e], hdr.n_slots);
    }
  }
#endif
  if (sizeof(T) == 4 && tid == 0 && (((uintptr_t)in | (uint32_t)(I * 4) | (uint64_t)in_gstride * 4) & 15) == 0) {
    const int t0 = run * tpc * TT;  // first tile of this CTA: in flight while the program is staged
    if (t0 < B) prefetch_l2(in + gi * in_gstride + (int64_t)t0 * I, (uint32_t)(min(TT, B - t0) * I * 4));
  }
  {
    auto copy16 = [&](void* dst, const void* src, int64_t bytes) {
      const int n16 = (int)(bytes / 16);
      for (int i = tid; i < n16; i += NT)
        reinterpret_cast<int4*>(dst)[i] = __ldg(reinterpret_cast<const int4*>(src) + i);
    };
    copy16(gr_s, gp + L.off_groups, off_st);
    copy16(st_s, gp + L.off_steps, (int64_t)n_steps * sizeof(StepT<T>));
    if (sizeof(T) == 4) {
      const uint32_t* gs = reinterpret_cast<const uint32_t*>(gp + L.off_src);  // u16 pairs
      for (int i = tid; i < n_edges / 2; i += NT) {
        const uint32_t pr = __ldg(gs + i);
        reinterpret_cast<uint2*>(src_s)[i] = make_uint2((pr & 0xFFFFu) * RB, (pr >> 16) * RB);
      }
    }
    copy16(reinterpret_cast<void*>(smem + off_w), gp + L.off_w, w_bytes);
  }
  // output slots of this genome (first 8 staged in shared memory)
  const uint16_t* os = reinterpret_cast<const uint16_t*>(gp + L.off_out);
  __shared__ uint16_t oslot[8];
  if (tid < 8) oslot[tid] = tid < O ? __ldg(os + tid) : NO_SLOT;
  // zero slot (last slot): read by padding entries, never written
  if (hdr.n_slots > 0)
    for (int i = tid; i < TT + S; i += NT) vals[(int64_t)(hdr.n_slots - 1) * (RB / sizeof(T)) + i] = T(0);
  __syncthreads();

  const T* gin = in + gi * in_gstride;
  T* go = out + gi * out_gstride;
  char* vb = reinterpret_cast<char*>(vals) + tid * S * sizeof(T);
  bool fast_out = sizeof(T) == 4 && O == 8;
#pragma unroll
  for (int o = 0; o < 8; ++o) fast_out = fast_out && oslot[o] != NO_SLOT;
  const int tile_end = min((run + 1) * tpc, (B + TT - 1) / TT);
  const bool vec_in = sizeof(T) == 4 && (I & 3) == 0 && (in_gstride & 3) == 0;
  const int step_s = (4 * NT) / I, step_i = (4 * NT) - step_s * I;  // chunk stride in (sample, input)
  const int step_s1 = NT / I, step_i1 = NT - step_s1 * I;
  const int cps = I >> 2;
  const int cps_shift = (cps & (cps - 1)) == 0 ? __ffs(cps) - 1 : -1;
  const int cps_mask = cps - 1;
  // inputs -> value slots 0..I-1 (input key i lives in slot i).  A tile's
  // (samples x I) block is contiguous in HBM: it is read with coalesced 16-byte
  // loads and scattered into the [slot][sample] layout (rows padded by S
  // elements, so a warp's scattered stores hit distinct banks).  The next
  // tile's block is prefetched into L2 by the TMA engine while this tile
  // computes, so the tile-start loads are L2 hits.
  const bool pf_l2 = sizeof(T) == 4 && (((uintptr_t)gin | (uint32_t)(I * 4)) & 15) == 0;
  float* const vf = reinterpret_cast<float*>(vals);
#define TNEAT_SCATTER4(sm_, i_, x_)                 \
  {                                                 \
    float* base_ = vf + (sm_) + (i_) * (RB / 4);    \
    base_[0] = (x_).x;                              \
    base_[RB / 4] = (x_).y;                         \
    base_[2 * (RB / 4)] = (x_).z;                   \
    base_[3 * (RB / 4)] = (x_).w;                   \
  }
  float sq = 0.0f;  // fused fitness: sum of squared outputs of this thread's samples
  for (int tile = run * tpc; tile < tile_end; ++tile) {
    const int t0 = tile * TT;
    const int nt = min(TT, B - t0);
    if (tile != run * tpc) __syncthreads();  // previous tile fully consumed
    if (pf_l2 && tid == 0 && tile + 1 < tile_end) {
      const int t1 = t0 + TT;
      prefetch_l2(gin + (int64_t)t1 * I, (uint32_t)(min(TT, B - t1) * I * 4));
    }
#ifdef TNEAT_DIAG_NOSTAGE  // diagnostic builds only: sweep over stale inputs
    if (tile == run * tpc && vec_in && cps_shift >= 0) {
#else
    if (vec_in && cps_shift >= 0) {  // I/4 chunks per input row is a power of two
#endif
      const float4* src = reinterpret_cast<const float4*>(gin + (int64_t)t0 * I);
      const int n4 = nt * I / 4;
      if (cps == 8 && (RB / 4) % 32 == 2) {
        // I = 32 with a row stride of 2 banks: a warp's 32 lanes hold 4 samples x
        // 8 input chunks; storing component k of every chunk would hit rows
        // {0,4,..,28}+k, i.e. every bank twice.  Lanes of the upper 4 chunks
        // store their components in the order 2,0,3,1 (lower: 0,2,1,3), so the
        // 8 rows of each store have distinct even residues mod 16 and the
        // store is conflict-free.
        // c & 7 == tid & 7 (NT is a multiple of 8): the lane's swizzle is fixed
        // (hoisted out of the loop; batching several loads per thread before
        // the stores measured slower)
        const bool hi = (tid & 4) != 0;
        const int o2 = hi ? 0 : 2 * (RB / 4), o0 = hi ? 2 * (RB / 4) : 0;
        float* const cbase = vf + ((tid & 7) << 2) * (RB / 4);
        for (int c = tid; c < n4; c += NT) {
          const float4 x = __ldg(src + c);
          float* base = cbase + (c >> 3);
          base[o0] = hi ? x.z : x.x;
          base[o2] = hi ? x.x : x.z;
          base[o0 + (RB / 4)] = hi ? x.w : x.y;
          base[o2 + (RB / 4)] = hi ? x.y : x.w;
        }
      } else {
        for (int c = tid; c < n4; c += NT) {
          const float4 x = __ldg(src + c);
          TNEAT_SCATTER4(c >> cps_shift, (c & cps_mask) << 2, x);
        }
      }
    } else if (vec_in) {
      const float4* src = reinterpret_cast<const float4*>(gin + (int64_t)t0 * I);
      const int n4 = nt * I / 4;
      int sm = (4 * tid) / I, i = 4 * tid - sm * I;  // (sample, input) of chunk c, stepped
      for (int c = tid; c < n4; c += NT) {           // incrementally (no division)
        const float4 x = __ldg(src + c);
        TNEAT_SCATTER4(sm, i, x);
        i += step_i;
        sm += step_s;
        if (i >= I) { i -= I; ++sm; }
      }
    } else {
      const T* src = gin + (int64_t)t0 * I;
      int sm = tid / I, i = tid - sm * I;
      for (int c = tid; c < nt * I; c += NT) {
        reinterpret_cast<T*>(reinterpret_cast<char*>(vals) + i * RB)[sm] = src[c];
        i += step_i1;
        sm += step_s1;
        if (i >= I) { i -= I; ++sm; }
      }
    }
    __syncthreads();
    const int s0 = t0 + tid * S;

    // node sweep, one group of independent same-level nodes at a time
#ifdef TNEAT_DIAG_NOSWEEP  // diagnostic builds only: staging and outputs alone
    if (n_groups < 0)
#endif
    // the next group's record is loaded while this group runs (look-ahead past
    // the last record reads the step table: still shared memory)
    // (two records ahead), and -- fp32 -- the next group's first program words
    uint4 raw_next = reinterpret_cast<const uint4*>(gr_s)[0];
    uint4 raw_next2 = reinterpret_cast<const uint4*>(gr_s)[1];
    Words wd;  // the current group's first words; refilled in place with the next group's
    if constexpr (sizeof(T) == 4) {
      if (n_groups > 0) load_words(wd, src_s, w_s, (int)(raw_next.y & 0xFFFF));
    }
#pragma unroll 1
    for (int g = 0; g < n_groups; ++g) {
      const uint4 raw = raw_next;
      raw_next = raw_next2;
      raw_next2 = reinterpret_cast<const uint4*>(gr_s)[g + 2];
      const int next_e = g + 1 < n_groups ? (int)(raw_next.y & 0xFFFF) : 0;
      GroupRec gr;
      gr.n = (uint8_t)(raw.x & 0xFF);
      gr.cls = (uint8_t)((raw.x >> 8) & 0xFF);
      gr.rounds = (uint16_t)(raw.x >> 16);
      gr.e_begin = (uint16_t)(raw.y & 0xFFFF);
      gr.step_begin = (uint16_t)(raw.y >> 16);
      gr.cnt[0] = (uint16_t)(raw.z & 0xFFFF);
      gr.cnt[1] = (uint16_t)(raw.z >> 16);
      gr.cnt[2] = (uint16_t)(raw.w & 0xFFFF);
      gr.cnt[3] = (uint16_t)(raw.w >> 16);
      run_group<T, S, RB>(gr, src_s, w_s, ed_s, st_s + gr.step_begin, vb, wd, next_e);
    }

    // outputs (P, B, O): one S-wide load per output slot, 16-byte stores per input
    if (fast_out) {
      PackT v[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) v[o] = *reinterpret_cast<const PackT*>(vb + (uint32_t)oslot[o] * RB);
#pragma unroll
      for (int j = 0; j < S; ++j) {
        if (s0 + j >= B) break;
        float4* row = reinterpret_cast<float4*>(go + (int64_t)(s0 + j) * 8);
        row[0] = make_float4(v[0].v[j], v[1].v[j], v[2].v[j], v[3].v[j]);
        row[1] = make_float4(v[4].v[j], v[5].v[j], v[6].v[j], v[7].v[j]);
        if (gsq)
#pragma unroll
          for (int o = 0; o < 8; ++o) sq += (float)(v[o].v[j] * v[o].v[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const int s = s0 + j;
        if (s >= B) break;
        T* row = go + (int64_t)s * O;
        for (int o = 0; o < O; ++o) {
          const uint16_t sl = __ldg(os + o);
          const T y = sl != NO_SLOT ? *reinterpret_cast<const T*>(vb + sl * RB + j * sizeof(T)) : T(NAN);
          row[o] = y;
          sq += (float)(y * y);
        }
      }
    }
  }
  if (gsq) {  // fused fitness (device-planned forward): one atomic per warp and task
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, d);
    if ((tid & 31) == 0) atomicAdd(gsq + gi, sq);
  }
}

// grid: (genome, run of `tpc` consecutive tiles) tasks; with a device-side
// genome count (count_dev, the device launch plan) the grid strides over the
// tasks of the first *count_dev genome ids
template <typename T, int S, int NT>
__global__ void __launch_bounds__(NT, TNEAT_TILE_MINB(NT)) fwd_tile_kernel(const uint8_t* __restrict__ prog, ProgLayout L,
                                                      const int32_t* __restrict__ genome_ids,
                                                      const int32_t* __restrict__ count_dev,
                                                      const T* __restrict__ in, int64_t in_gstride,
                                                      int B, int I, int O, int runs, int tpc,
                                                      T* __restrict__ out, int64_t out_gstride,
                                                      float* __restrict__ gsq) {
  if (!count_dev) {
    const int64_t task = blockIdx.x / runs;
    tile_task<T, S, NT>(prog, L, genome_ids, in, in_gstride, B, I, O, task, (int)(blockIdx.x - task * runs), tpc,
                        out, out_gstride, gsq);
    return;
  }
  const int64_t n = (int64_t)__ldg(count_dev) * runs;
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (t != blockIdx.x) __syncthreads();  // the previous task's shared memory is consumed
    const int64_t task = t / runs;
    tile_task<T, S, NT>(prog, L, genome_ids, in, in_gstride, B, I, O, task, (int)(t - task * runs), tpc, out,
                        out_gstride, gsq);
  }
}

// ---------------------------------------------------------------------------
// tensor-core forward (FMT_TC programs): input layer on tcgen05, hidden
// edges on CUDA cores
// ---------------------------------------------------------------------------
//
// Persistent: one CTA per SM with W warpgroups (4 warps each, W <= 4 as shared
// memory allows).  The CTA walks its genomes (blockIdx.x, + gridDim.x, ...);
// each genome's staged block (B operand, column factors, group / step records,
// hidden edges: common.cuh tc_block) arrives by one bulk copy into one of two
// buffers -- the next genome's copy is in flight while the current one runs --
// and the warpgroups share it, warpgroup w taking tiles w, w + W, ... of 256
// samples.  Thread r of a warpgroup owns samples r and r + 128 of its tile
// (TMEM lane r of the two MMA halves; warp w%4 reads lanes 32(w%4)..), two
// samples per thread so the sweep's warp-uniform work (program words, group
// records, dispatch) and its packed FFMA2 arithmetic cover 64 samples.  Per
// tile, within the warpgroup (named barrier 1 + w):
//   1. the (256 x 32) fp32 input block lands by TMA (3-D tensor map, 128-byte
//      swizzle, zero fill past B and past I) in the warpgroup's area;
//   2. each thread reads its two rows into registers, block-scales them by a
//      power of two and writes three fp16 digit planes over the same area
//      (A operand, two 128-row halves, K-major core matrices;
//      csrc/digits.cuh);
//   3. one thread takes a TMEM column slot (2 halves x D4 / D32 x nb columns;
//      the CTA's 512 columns are shared by its warpgroups through a bitmask)
//      and issues 2 x 12 kind::f16 MMAs against the genome's B operand;
//   4. each thread reads its TMEM lane and writes every step's input partial
//      sums (both samples) into the step's value slot ([slot][128][2] fp32,
//      over the consumed A area), then the slot is released;
//   5. the hidden-edge sweep (the tile kernel's group records) starts each
//      step's accumulator from its slot, and the outputs are stored.
// Rows whose scale is out of range (non-finite inputs, |x| >= 2^62 or a
// nonzero max < 2^-62) get zero digits and an exact fp32 partial from the
// program's input edge lists instead.
constexpr int TC_NT = 128;                   // threads per warpgroup = rows per MMA half
constexpr int TC_TT = TC_SAMPLES;            // samples per tile
constexpr int TC_RB = TC_SLOT_BYTES;         // bytes of one value slot row
constexpr int TC_IN_BYTES = TC_TT * 128;     // fp32 input tile, 256 rows x 128 B
constexpr int TC_A_HALF = TC_NT * TC_ROWB;   // A operand of one 128-row half: 24 KB
constexpr int TC_MAX_WG = 4;
static_assert(TC_TT == 2 * TC_NT, "two samples per thread");

// per-warpgroup area: A operand / value slots from the start, the input tile
// at the end (>= 48 KB, 1024-aligned: TMA 128-byte swizzle)
__host__ __device__ inline uint32_t tc_wg_bytes(int nb) {
  int64_t u = (int64_t)(nb + 1) * TC_RB;
  if (u < 2 * TC_A_HALF) u = 2 * TC_A_HALF;
  if (u < TC_IN_BYTES) u = TC_IN_BYTES;
  return (uint32_t)align_up(u, 1024);
}

__device__ __forceinline__ void run_group_tc(const uint4 rec, const uint32_t* src_s, const float* w_s,
                                             const StepT<float>* st_all, char* vb, Words& wd, int next_e) {
  constexpr int S = 2, RB = TC_RB;
  GroupRec gr;  // the fields run_sum_group reads (TC group records are pre-decoded: common.cuh GroupTC)
  gr.rounds = (uint16_t)rec.y;
  gr.e_begin = (uint16_t)rec.z;
  gr.step_begin = (uint16_t)rec.w;
  const StepT<float>* st = st_all + rec.w;
  switch (rec.x) {
    case 0: run_sum_group<S, 1, RB, false, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 1: run_sum_group<S, 2, RB, false, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 2: run_sum_group<S, 3, RB, false, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 3: run_sum_group<S, 4, RB, false, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 4: run_sum_group<S, 1, RB, true, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 5: run_sum_group<S, 2, RB, true, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 6: run_sum_group<S, 3, RB, true, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 7: run_sum_group<S, 4, RB, true, false, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    case 10: run_sum_group<S, 4, RB, false, true, true>(gr, src_s, w_s, st, vb, wd, next_e); break;
    default: run_sum_group<S, 4, RB, true, true, true>(gr, src_s, w_s, st, vb, wd, next_e); break;  // 14
  }
}

// the 2 x 12 MMAs of a tile, from one elected lane of a converged warp whose
// operands are warp-uniform (shuffled from lane 0): the compiler keeps them in
// uniform registers (no per-MMA broadcast loop)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 %%rx;\n.reg .pred %%px;\nelect.sync %%rx|%%px, %1;\n@%%px mov.s32 %0, 1;\n}\n"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

__device__ __forceinline__ void tc_issue_mmas(uint32_t a_addr, uint32_t b_addr, uint32_t dcol, int nb,
                                              uint32_t bar) {
  const uint32_t idesc = idesc_f16(TC_NT, nb);
  if (elect_one()) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t ah = a_addr + (uint32_t)(h * TC_A_HALF);
      auto A = [&](int k0) { return smem_desc(ah + (uint32_t)(k0 >> 3) * TC_LBO, TC_SBO, TC_LBO); };
      auto Bd = [&](int k0) { return smem_desc(b_addr + (uint32_t)(k0 >> 3) * TC_LBO, TC_SBO, TC_LBO); };
      const uint32_t d4 = dcol + (uint32_t)(2 * h * nb), d32 = d4 + (uint32_t)nb;
#ifndef TNEAT_DIAG_TC_NOMMA  // diagnostic builds only: commit without MMAs
      mma_f16(d4, A(0), Bd(0), idesc, 0u);  // D4 = A2 B2
      mma_f16(d4, A(16), Bd(16), idesc, 1u);
      mma_f16(d32, A(0), Bd(64), idesc, 0u);  // class 2 = A2 B0 + A1 B1 + A0 B2
      mma_f16(d32, A(16), Bd(80), idesc, 1u);
      mma_f16(d32, A(32), Bd(32), idesc, 1u);
      mma_f16(d32, A(48), Bd(48), idesc, 1u);
      mma_f16(d32, A(64), Bd(0), idesc, 1u);
      mma_f16(d32, A(80), Bd(16), idesc, 1u);
      mma_f16_scale10(d32, A(0), Bd(32), idesc);  // * 2^-10, + class 3 = A2 B1 + A1 B2
      mma_f16(d32, A(16), Bd(48), idesc, 1u);
      mma_f16(d32, A(32), Bd(0), idesc, 1u);
      mma_f16(d32, A(48), Bd(16), idesc, 1u);
#endif
    }
    mma_commit(bar);
  }
  __syncwarp();
}

// one input row -> registers (128-byte swizzle: chunk c of row r at c ^ (r & 7))
__device__ __forceinline__ void tc_load_row(const uint8_t* rowp, int r, float (&x)[TC_K]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 v = *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
    x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
  }
}

__device__ __forceinline__ float max3_nan(float a, float b, float c) {  // NaN-propagating
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// block exponent of a row; returns whether the row takes the exact path (a
// non-finite input makes the NaN-propagating max non-finite)
__device__ __forceinline__ bool tc_row_scale(const float (&x)[TC_K], int& ex) {
  float m = 0.0f;
#pragma unroll
  for (int k = 0; k < TC_K; k += 2) m = max3_nan(m, fabsf(x[k]), fabsf(x[k + 1]));
  const bool exact = !(m < 0x1p62f) || (m != 0.0f && m < 0x1p-62f);
  ex = (m > 0.0f && !exact) ? float_exponent(m) : 0;
  return exact;
}

// digit planes of one row into A row r (exact rows: zero digits).  d0 is left
// unrounded (r0 * sc, |.| <= 512): the fp16 conversion keeps it to 1/4 and it
// only enters the 2^-20-weighted class 2
__device__ __forceinline__ void tc_store_digits(const float (&x)[TC_K], int ex, bool exact, int r, uint8_t* a_half) {
  const float s20 = exact ? 0.0f : pow2f(7 - ex), i20 = exact ? 0.0f : pow2f(ex - 7);
  const float s10 = exact ? 0.0f : pow2f(17 - ex), i10 = exact ? 0.0f : pow2f(ex - 17);
  const float s0 = exact ? 0.0f : pow2f(27 - ex);
  const float2 M = make_float2(12582912.0f, 12582912.0f), nM = make_float2(-12582912.0f, -12582912.0f);
  const float2 S20 = make_float2(s20, s20), NI20 = make_float2(-i20, -i20), S10 = make_float2(s10, s10),
               NI10 = make_float2(-i10, -i10), S0 = make_float2(s0, s0);
#pragma unroll
  for (int q = 0; q < TC_K / 8; ++q) {  // 8 inputs = one 16-byte chunk per plane
    uint32_t w2[4], w1[4], w0[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 xv = make_float2(x[8 * q + 2 * h], x[8 * q + 2 * h + 1]);
#ifdef TNEAT_DIAG_TC_NOCONV  // diagnostic builds only: no digit arithmetic
      w2[h] = w1[h] = w0[h] = pack_half2(xv.x, xv.y);
      continue;
#endif
      const float2 d2 = __fadd2_rn(__ffma2_rn(xv, S20, M), nM);
      const float2 r1 = __ffma2_rn(d2, NI20, xv);
      const float2 d1 = __fadd2_rn(__ffma2_rn(r1, S10, M), nM);
      const float2 d0 = __fmul2_rn(__ffma2_rn(d1, NI10, r1), S0);
      w2[h] = pack_half2(d2.x, d2.y);
      w1[h] = pack_half2(d1.x, d1.y);
      w0[h] = pack_half2(d0.x, d0.y);
    }
    *reinterpret_cast<uint4*>(a_half + tc_offset(r, 8 * q)) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
    *reinterpret_cast<uint4*>(a_half + tc_offset(r, TC_K + 8 * q)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
    *reinterpret_cast<uint4*>(a_half + tc_offset(r, 2 * TC_K + 8 * q)) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
  }
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

struct TcShared {
  uint64_t gbar[2];                 // genome block staged in buffer b
  uint64_t tma_bar[TC_MAX_WG];      // input tile of warpgroup w
  uint64_t mma_bar[TC_MAX_WG];      // MMAs of warpgroup w done
  uint32_t tmem_base;
  uint32_t tmem_mask;               // TMEM column slots in use
  uint32_t slot_col[TC_MAX_WG];     // column offset of warpgroup w's slot
  int32_t hdr[2][4];                // n_steps, n_edges, n_groups, genome of buffer b
  uint16_t oslot[2][8];
  int64_t next_task[2];             // task after task k: next_task[k & 1] (thread 0 writes)
};

__global__ void __launch_bounds__(TC_NT* TC_MAX_WG, 1)
fwd_tc_kernel(const __grid_constant__ CUtensorMap tmap_in, const uint8_t* __restrict__ prog, ProgLayout L,
              const int32_t* __restrict__ genome_ids, const int32_t* __restrict__ count_dev, int64_t P,
              const float* __restrict__ in, int64_t in_gstride,
              int B, int I, int O, int nwg, uint32_t wg_bytes, uint32_t gbuf_bytes, int nbuf, int nb_max,
              float* __restrict__ gsq, float* __restrict__ out,
              int64_t out_gstride, int32_t* __restrict__ task_ctr) {
  // no static shared memory: the dynamic area starts the CTA's shared window,
  // 1024-aligned for the swizzled TMA tiles; the control block is at its end
  extern __shared__ __align__(1024) uint8_t smem[];
  TcShared& sh = *reinterpret_cast<TcShared*>(smem + (uint32_t)nwg * wg_bytes + (uint32_t)nbuf * gbuf_bytes);
  const int tid = threadIdx.x, warp = tid >> 5, wg = tid >> 7, wt = tid & (TC_NT - 1);
  const int bar_id = 1 + wg;
  uint8_t* const wg_area = smem + (uint32_t)wg * wg_bytes;
  uint8_t* const gbuf0 = smem + (uint32_t)nwg * wg_bytes;
  // the next class launch of a device plan may take SMs as this grid's CTAs
  // exit (programmatic dependent launch; a no-op otherwise)
  asm volatile("griddepcontrol.launch_dependents;");
  if (count_dev) P = __ldg(count_dev);  // device launch plan: this class's genome count
  const uint32_t slot_cols = 4u * (uint32_t)nb_max;
  const uint32_t n_slots = 512u / slot_cols;
  const int tiles = (B + TC_TT - 1) / TC_TT;
  // tasks: (genome, run of tiles).  A genome is one run unless the launch has
  // fewer genomes than CTAs (small classes): then its tiles are split into up
  // to gridDim / P runs (each of >= nwg tiles) so every SM gets work
  int runs = 1;
  if (P > 0 && P < (int64_t)gridDim.x) {
    const int64_t want = ((int64_t)gridDim.x + P - 1) / P, cap = tiles / nwg > 1 ? tiles / nwg : 1;
    runs = (int)(want < cap ? want : cap);
  }
  const int run_tiles = (tiles + runs - 1) / runs;
  const int64_t n_tasks = P * runs;

  auto issue_stage = [&](int64_t task, int buf) {  // one thread: header + block of task's genome
    const int64_t gi = genome_ids ? (int64_t)__ldg(genome_ids + task / runs) : task / runs;
    const uint8_t* gp = prog + gi * L.stride;
    const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
    const int ns = hdr.mode == MODE_TC ? hdr.n_steps : 0, ng = hdr.mode == MODE_TC ? hdr.n_groups : 0;
    const int ne = hdr.mode == MODE_TC ? hdr.n_edges : 0;
    sh.hdr[buf][0] = ns; sh.hdr[buf][1] = ne; sh.hdr[buf][2] = ng; sh.hdr[buf][3] = (int)gi;
    const uint16_t* os = reinterpret_cast<const uint16_t*>(gp + L.off_out);
    for (int o = 0; o < 8; ++o) sh.oslot[buf][o] = (o < O && hdr.mode == MODE_TC) ? __ldg(os + o) : NO_SLOT;
    const TcBlock tb = tc_block(ns, ng, ne);
    const uint32_t bar = smem_u32(&sh.gbar[buf]);
    mbar_expect_tx(bar, tb.bytes);
    if (tb.bytes) bulk_g2s(smem_u32(gbuf0 + (uint32_t)buf * gbuf_bytes), gp + L.off_tc, tb.bytes, bar);
  };

  if (warp == 0) {
    tmem_alloc(smem_u32(&sh.tmem_base), 512);
    tmem_relinquish();
  }
  if (tid == 0) {
    mbar_init(smem_u32(&sh.gbar[0]), 1);
    mbar_init(smem_u32(&sh.gbar[1]), 1);
    for (int w = 0; w < TC_MAX_WG; ++w) {
      mbar_init(smem_u32(&sh.tma_bar[w]), 1);
      mbar_init(smem_u32(&sh.mma_bar[w]), 1);
    }
    sh.tmem_mask = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (blockIdx.x < n_tasks) issue_stage(blockIdx.x, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem_base;
  const uint32_t bar_tma = smem_u32(&sh.tma_bar[wg]), bar_mma = smem_u32(&sh.mma_bar[wg]);
  uint8_t* const in_area = wg_area + wg_bytes - TC_IN_BYTES;  // input tile: end of the area
  const uint32_t in_addr = smem_u32(in_area);
  char* const vb = reinterpret_cast<char*>(wg_area) + wt * 8;
  const uint32_t a_addr = smem_u32(wg_area);
  uint32_t tphase = 0, mphase = 0, gphase[2] = {0u, 0u};

  // tasks: the CTA's first is blockIdx.x; later ones come from the launch's
  // task counter (dynamic: a CTA that drew small genomes takes more of them)
  // or, without one, every gridDim.x-th
  int k = 0;
  for (int64_t task = blockIdx.x; task < n_tasks; ++k) {
    // two buffers: the next task's genome block is in flight during this one;
    // one buffer (when a second would cost a warpgroup): staged after the barrier
    const int buf = nbuf == 2 ? (k & 1) : 0;
    mbar_wait(smem_u32(&sh.gbar[buf]), gphase[buf]);
    gphase[buf] ^= 1u;
    if (tid == 0) {
      const int64_t nx = task_ctr ? (int64_t)gridDim.x + atomicAdd(task_ctr, 1) : task + gridDim.x;
      sh.next_task[k & 1] = nx;
      if (nbuf == 2 && nx < n_tasks) issue_stage(nx, buf ^ 1);
    }
    const int run = (int)(task % runs);
    const int t_begin = run * run_tiles, t_end = min(tiles, t_begin + run_tiles);
    const int n_steps = sh.hdr[buf][0], n_edges = sh.hdr[buf][1], n_groups = sh.hdr[buf][2];
    const int64_t gi = sh.hdr[buf][3];
    const int nb = tc_rows(n_steps);
    const TcBlock tb = tc_block(n_steps, n_groups, n_edges);
    uint8_t* const gb = gbuf0 + (uint32_t)buf * gbuf_bytes;
    const GroupRec* gr_s = reinterpret_cast<const GroupRec*>(gb + tb.gr);
    const StepT<float>* st_s = reinterpret_cast<const StepT<float>*>(gb + tb.st);
    const uint32_t* src_s = reinterpret_cast<const uint32_t*>(gb + tb.src);
    const float* w_s = reinterpret_cast<const float*>(gb + tb.w);
    const float* cf_s = reinterpret_cast<const float*>(gb + tb.cf);
    const uint32_t b_addr = smem_u32(gb + tb.b);
    const uint16_t* oslot = sh.oslot[buf];
    bool fast_out = O == 8 && n_steps > 0;
#pragma unroll
    for (int o = 0; o < 8; ++o) fast_out = fast_out && oslot[o] != NO_SLOT;
    const uint8_t* gp = prog + gi * L.stride;
    const float* gin = in + gi * in_gstride;
    float* go = out + gi * out_gstride;
    const int zc = in_gstride ? (int)gi : 0;  // input tensor map: (I, B, genomes)
    TNEAT_DCHECK(n_steps == 0 || (tb.bytes + 64 <= gbuf_bytes), "tc genome block fits its buffer", tb.bytes, gbuf_bytes);
    TNEAT_DCHECK(nb <= nb_max, "tc MMA width within the class", nb, nb_max);
    TNEAT_DCHECK((uint32_t)(n_steps + 1) * TC_RB <= wg_bytes, "tc value slots fit the warpgroup area", n_steps, wg_bytes);
#ifdef TNEAT_CHECKS
    for (int g = tid; g < n_groups; g += blockDim.x) {  // every entry a group sweeps reads a value slot
      const uint4 r = reinterpret_cast<const uint4*>(gr_s)[g];
      const uint32_t n = (r.x & 3) + 1, gw = n == 3 ? 4 : n;
      TNEAT_DCHECK(r.z + gw * r.y <= (uint32_t)n_edges && r.w + n <= (uint32_t)n_steps, "tc group record",
                   r.z + gw * r.y, n_edges);
      for (uint32_t e = r.z; e < r.z + gw * r.y; ++e)
        TNEAT_DCHECK(src_s[e] <= (uint32_t)n_steps * TC_RB && (src_s[e] % TC_RB) == 0, "tc hidden source slot",
                     src_s[e], n_steps);
    }
    TNEAT_DCHECK(smem_u32(gb) + tb.bytes + 64 <= smem_u32(smem) + dynamic_smem_bytes(), "tc block in smem",
                 tb.bytes, dynamic_smem_bytes());
#endif
    const bool pf_l2 = ((uintptr_t)gin & 15) == 0;
    const uint16_t* in_start = reinterpret_cast<const uint16_t*>(gp + L.off_in);
    const uint16_t* isrc = reinterpret_cast<const uint16_t*>(gp + L.off_isrc);
    const float* iw = reinterpret_cast<const float*>(gp + L.off_iw);

    float sq = 0.0f;  // fused fitness: sum of squared outputs of this thread's samples
    if (n_steps > 0 && wt == 0 && t_begin + wg < t_end) {  // this warpgroup's first tile
      mbar_expect_tx(bar_tma, TC_IN_BYTES);
      tma_load_3d(in_addr, &tmap_in, 0, (t_begin + wg) * TC_TT, zc, bar_tma);
    }
    for (int tile = t_begin + wg; tile < t_end && n_steps > 0; tile += nwg) {
      const int s0 = tile * TC_TT + wt, s1 = s0 + TC_NT;  // this thread's samples
      const int next = tile + nwg;
      // ---- 1-2: input rows -> block scales -> digit planes (A rows wt of both halves)
      mbar_wait_sleep(bar_tma, tphase);
      tphase ^= 1u;
      if (wt == 0 && next < t_end && pf_l2)  // next tile: HBM -> L2 while this one computes
        prefetch_l2(gin + (int64_t)next * TC_TT * I, (uint32_t)(min(TC_TT, B - next * TC_TT) * I * 4));
      // the input tile sits at the end of the area: A half 0 ([0, 24K)) only
      // overlaps input rows of half 0, so each half is read (into registers),
      // then its digits are written
      int ex0, ex1;
      bool exact0, exact1;
      {
        float x[TC_K];
        tc_load_row(in_area + wt * 128, wt, x);
        exact0 = tc_row_scale(x, ex0);
        named_barrier_sync(bar_id, TC_NT);
        tc_store_digits(x, ex0, exact0, wt, wg_area);
      }
      {
        float x[TC_K];
        tc_load_row(in_area + (TC_NT + wt) * 128, wt, x);
        exact1 = tc_row_scale(x, ex1);
        named_barrier_sync(bar_id, TC_NT);
        tc_store_digits(x, ex1, exact1, wt, wg_area + TC_A_HALF);
      }
      fence_proxy_async_smem();
      // ---- 3: a TMEM column slot, MMAs (one thread) -------------------------------------
      if (wt == 0) {
        uint32_t slot = (uint32_t)wg;
        if (n_slots < (uint32_t)nwg) {  // fewer slots than warpgroups: take a free one
          for (;;) {
            const uint32_t m = *reinterpret_cast<volatile uint32_t*>(&sh.tmem_mask);
            slot = __ffs(~m) - 1;
            if (slot < n_slots && atomicCAS(&sh.tmem_mask, m, m | (1u << slot)) == m) break;
            __nanosleep(32);
          }
        }
        TNEAT_DCHECK(slot < n_slots && (slot + 1) * slot_cols <= 512u, "tc TMEM slot", slot, n_slots);
        sh.slot_col[wg] = slot * slot_cols;
      }
      tc_fence_before();
      named_barrier_sync(bar_id, TC_NT);  // A complete, column slot taken
      tc_fence_after();
      const uint32_t dcol = tmem + sh.slot_col[wg];
      if (wt < 32)
        tc_issue_mmas(__shfl_sync(0xffffffffu, a_addr, 0), __shfl_sync(0xffffffffu, b_addr, 0),
                      __shfl_sync(0xffffffffu, dcol, 0), __shfl_sync(0xffffffffu, nb, 0), bar_mma);
      // ---- 4: TMEM -> input partials in the step slots ------------------------------------
      mbar_wait_sleep(bar_mma, mphase);
      mphase ^= 1u;
      tc_fence_after();
      {
        // warp-uniform TMEM address (uniform registers for tcgen05.ld)
        const uint32_t t_lane = __shfl_sync(0xffffffffu, dcol + ((uint32_t)((warp & 3) * 32) << 16), 0);
        // partial / cf = T * 2^(ex - 12): the column factor cf lives in the step
        // (response and hidden weights, transform.cu)
        const float2 rf0 = make_float2(pow2f(ex0 - 12), pow2f(ex0 - 12));
        const float2 rf1 = make_float2(pow2f(ex1 - 12), pow2f(ex1 - 12));
        const float2 k1024 = make_float2(1024.0f, 1024.0f);
#pragma unroll 1
#ifdef TNEAT_DIAG_TC_NOEPI  // diagnostic builds only: no TMEM -> slot epilogue
        for (int c = 0; c < 0; c += 8) {
#else
        for (int c = 0; c < n_steps; c += 8) {  // columns past the last step are not read
#endif
          uint32_t a4[8], a3[8], b4[8], b3[8];
          TMEM_LD8(t_lane + (uint32_t)c, a4);
          TMEM_LD8(t_lane + (uint32_t)(nb + c), a3);
          TMEM_LD8(t_lane + (uint32_t)(2 * nb + c), b4);
          TMEM_LD8(t_lane + (uint32_t)(3 * nb + c), b3);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; i += 2) {  // steps c+i, c+i+1: packed over adjacent columns
            const float2 p0 =
                __fmul2_rn(__ffma2_rn(make_float2(__uint_as_float(a4[i]), __uint_as_float(a4[i + 1])), k1024,
                                      make_float2(__uint_as_float(a3[i]), __uint_as_float(a3[i + 1]))),
                           rf0);
            const float2 p1 =
                __fmul2_rn(__ffma2_rn(make_float2(__uint_as_float(b4[i]), __uint_as_float(b4[i + 1])), k1024,
                                      make_float2(__uint_as_float(b3[i]), __uint_as_float(b3[i + 1]))),
                           rf1);
            *reinterpret_cast<float2*>(vb + (uint32_t)(c + i) * TC_RB) = make_float2(p0.x, p1.x);
            *reinterpret_cast<float2*>(vb + (uint32_t)(c + i + 1) * TC_RB) = make_float2(p0.y, p1.y);
          }
        }
        tc_fence_before();
        named_barrier_sync(bar_id, TC_NT);  // every warp has read its lanes: release the slot
        if (wt == 0 && n_slots < (uint32_t)nwg) atomicAnd(&sh.tmem_mask, ~(1u << (sh.slot_col[wg] / slot_cols)));
        *reinterpret_cast<float2*>(vb + (uint32_t)n_steps * TC_RB) = make_float2(0.0f, 0.0f);  // zero slot
        if (exact0 || exact1) {  // exact fp32 partials (program order of each step's input edges)
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            const int s = h ? s1 : s0;
            if (!(h ? exact1 : exact0) || s >= B) continue;
            const float* xr = gin + (int64_t)s * I;
            for (int kk = 0; kk < n_steps; ++kk) {
              float p = 0.0f;
              for (int e = __ldg(in_start + kk); e < __ldg(in_start + kk + 1); ++e)
                p = fmaf(__ldg(iw + e), __ldg(xr + __ldg(isrc + e)), p);
              reinterpret_cast<float*>(vb + (uint32_t)kk * TC_RB)[h] = p * cf_s[kk];  // cf_s: 1 / cf
            }
          }
        }
      }
#ifdef TNEAT_DIAG_TC_EARLYTMA  // diagnostic builds only (wrong results): next tile's TMA before the sweep
      if (wt == 0 && next < t_end) {
        mbar_expect_tx(bar_tma, TC_IN_BYTES);
        tma_load_3d(in_addr, &tmap_in, 0, next * TC_TT, zc, bar_tma);
      }
#endif
      // ---- 5: hidden-edge sweep ---------------------------------------------------------
      {
        Words wd;
        if (n_groups > 0) load_words(wd, src_s, w_s, (int)reinterpret_cast<const uint4*>(gr_s)[0].z);
#ifdef TNEAT_DIAG_TC_NOSWEEP  // diagnostic builds only: no hidden-edge sweep
        const int n_groups_run = 0;
#else
        const int n_groups_run = n_groups;
#endif
#pragma unroll 1
        for (int g = 0; g < n_groups_run; ++g) {
          // the record and the next group's first entry (its words are loaded
          // at the end of this group; past the last group: the step table)
          const uint4 raw = reinterpret_cast<const uint4*>(gr_s)[g];
          const int next_e = (int)reinterpret_cast<const uint4*>(gr_s)[g + 1].z;
          run_group_tc(raw, src_s, w_s, st_s, vb, wd, g + 1 < n_groups ? next_e : 0);
        }
      }
      // ---- outputs (P, B, O) ------------------------------------------------------------
      if (fast_out) {
        float2 v[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) v[o] = *reinterpret_cast<const float2*>(vb + (uint32_t)oslot[o] * TC_RB);
        if (s0 < B) {
          float4* row = reinterpret_cast<float4*>(go + (int64_t)s0 * 8);
          row[0] = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
          row[1] = make_float4(v[4].x, v[5].x, v[6].x, v[7].x);
        }
        if (s1 < B) {
          float4* row = reinterpret_cast<float4*>(go + (int64_t)s1 * 8);
          row[0] = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
          row[1] = make_float4(v[4].y, v[5].y, v[6].y, v[7].y);
        }
        if (gsq) {
          const float m0 = s0 < B ? 1.0f : 0.0f, m1 = s1 < B ? 1.0f : 0.0f;
#pragma unroll
          for (int o = 0; o < 8; ++o) sq = fmaf(m0 * v[o].x, v[o].x, fmaf(m1 * v[o].y, v[o].y, sq));
        }
      } else {
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const int s = h ? s1 : s0;
          if (s >= B) continue;
          float* row = go + (int64_t)s * O;
          const uint16_t* os = reinterpret_cast<const uint16_t*>(gp + L.off_out);
          for (int o = 0; o < O; ++o) {
            const uint16_t sl = __ldg(os + o);
            const float y = sl != NO_SLOT ? reinterpret_cast<const float*>(vb + (uint32_t)sl * TC_RB)[h] : NAN;
            row[o] = y;
            sq = fmaf(y, y, sq);
          }
        }
      }
      named_barrier_sync(bar_id, TC_NT);  // slots dead: the next tile's inputs may land
#ifndef TNEAT_DIAG_TC_EARLYTMA
      if (wt == 0 && next < t_end) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar_tma, TC_IN_BYTES);
        tma_load_3d(in_addr, &tmap_in, 0, next * TC_TT, zc, bar_tma);
      }
#endif
    }
    if (gsq && n_steps > 0) {  // one atomic per warp and genome
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, d);
      if ((tid & 31) == 0) atomicAdd(gsq + gi, sq);
    }
    __syncthreads();  // every warpgroup is done with buffer `buf` before it is restaged
    const int64_t nx = sh.next_task[k & 1];
    if (nbuf == 1 && tid == 0 && nx < n_tasks) issue_stage(nx, 0);
    task = nx;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  // launched early behind the previous class launch: complete only after it
  // (so every later stream operation follows the whole chain); immediate for
  // a normal launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------

template <typename T> __device__ __forceinline__ T warp_allreduce(int agg, T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = agg_combine<T>(agg, v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

template <typename T> __device__ __forceinline__ T eval_node(const StepT<T>& st, T a);
template <> __device__ __forceinline__ float eval_node<float>(const StepT<float>& st, float a) {
  a = agg_finish<float>(st.agg, a, st.count);
  const int act = st.act;
  const float kx = act == ACT_TANH ? -2.8853900817779268f : (act == ACT_SIGMOID ? -1.4426950408889634f : 0.0f);
  return step_act(kx, act == ACT_TANH ? 2.0f : 1.0f, act == ACT_TANH ? -1.0f : 0.0f, act == ACT_RELU,
                  fmaf(st.resp, a, st.bias));
}
template <> __device__ __forceinline__ double eval_node<double>(const StepT<double>& st, double a) {
  return apply_act(st.act, fma(st.resp, agg_finish<double>(st.agg, a, st.count), st.bias));
}

enum : int { FIT_NONE = 0, FIT_XOR = 1, FIT_REGRESSION = 2 };

template <typename T>
__global__ void fwd_warp_kernel(const uint8_t* __restrict__ prog, ProgLayout L, int64_t P,
                                const T* __restrict__ in, int64_t in_gstride, int B, int I, int O,
                                int bchunk, int max_slots, T* __restrict__ out, int64_t out_gstride,
                                int fit_kind, const double* __restrict__ targets,
                                double* __restrict__ fitness) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int chunks = (B + bchunk - 1) / bchunk;
  const int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t gi = task / chunks;
  if (gi >= P) return;
  const int b0 = (int)(task - gi * chunks) * bchunk;
  const int nb = min(bchunk, B - b0);
  T* vals = reinterpret_cast<T*>(smem) + (int64_t)warp * max_slots * bchunk;  // [slot][bchunk]
  const uint8_t* gp = prog + gi * L.stride;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const GroupRec* groups = reinterpret_cast<const GroupRec*>(gp + L.off_groups);
  const StepT<T>* steps = reinterpret_cast<const StepT<T>*>(gp + L.off_steps);
  const uint16_t* esrc = reinterpret_cast<const uint16_t*>(gp + L.off_src);
  const float* ew = reinterpret_cast<const float*>(gp + L.off_w);
  const EdgeD* ed = reinterpret_cast<const EdgeD*>(gp + L.off_w);
  const T* gin = in + gi * in_gstride + (int64_t)b0 * I;
  for (int idx = lane; idx < nb * I; idx += 32) {
    const int b = idx / I, i = idx - b * I;
    vals[i * bchunk + b] = gin[idx];
  }
  __syncwarp();
  for (int g = 0; g < hdr.n_groups; ++g) {
    const GroupRec gr = groups[g];
    const int gw = group_width(gr.n);
    for (int b = 0; b < nb; ++b) {
      T y[4];
      for (int j = 0; j < gr.n; ++j) {  // all reads of the group precede its writes
        const StepT<T> st = steps[gr.step_begin + j];
        const int agg = st.agg;
        const int stride = (gr.cls & GRP_GENERIC) ? 1 : gw;
        T part = agg_neutral<T>(agg);
        const int h0 = (j == 0 && (gr.cls & GRP_SPLIT0)) ? gr.cnt[0] : 0x7FFFFFFF;  // split step 0
        for (int e = lane; e < st.count; e += 32) {
          const int idx = e < h0 ? gr.e_begin + e * stride + j : gr.e_begin + (e - h0) * stride + 3;
          uint32_t src;
          T w;
          if constexpr (sizeof(T) == 8) { src = ed[idx].src; w = ed[idx].w; }
          else { src = esrc[idx]; w = ew[idx]; }
          part = agg_combine<T>(agg, part, w * vals[(int64_t)src * bchunk + b]);
        }
        y[j & 3] = eval_node<T>(st, warp_allreduce<T>(agg, part));
      }
      __syncwarp();
      if (lane == 0) {
        for (int j = 0; j < gr.n; ++j) {
          const uint16_t sl = steps[gr.step_begin + j].slot;
          if (sl != NO_SLOT) vals[(int64_t)sl * bchunk + b] = y[j & 3];
        }
      }
      __syncwarp();
    }
  }
  const uint16_t* os = reinterpret_cast<const uint16_t*>(gp + L.off_out);
  if (fit_kind == FIT_NONE) {
    T* go = out + gi * out_gstride + (int64_t)b0 * O;
    for (int idx = lane; idx < nb * O; idx += 32) {
      const int b = idx / O, o = idx - b * O;
      const uint16_t sl = os[o];
      go[idx] = sl != NO_SLOT ? vals[(int64_t)sl * bchunk + b] : T(NAN);
    }
  } else if (lane == 0) {
    // fitness in float64 (problems.py:54-61) with numpy's summation order:
    // sequential below 8 terms, else 8 strided partial sums combined pairwise,
    // then the remainder added one by one
    const uint16_t sl = os[0];
    auto term = [&](int b) {
      // (an errored genome's program has no output slot: NaN; the host raises)
      const double y = sl != NO_SLOT ? (double)vals[(int64_t)sl * bchunk + b] : __longlong_as_double(0x7ff8000000000000ll);
      const double t = fit_kind == FIT_XOR ? (double)(((b >> 1) ^ b) & 1) : targets[b];
      return (y - t) * (y - t);
    };
    double total = 0.0;
    int b = 0;
    if (B >= 8) {
      double r[8];
      for (int j = 0; j < 8; ++j) r[j] = term(j);
      for (b = 8; b + 8 <= B; b += 8)
        for (int j = 0; j < 8; ++j) r[j] += term(b + j);
      total = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    }
    for (; b < B; ++b) total += term(b);
    fitness[gi] = fit_kind == FIT_XOR ? 4.0 - total : -(total / (double)B);
  }
}

// ---------------------------------------------------------------------------
// cart-pole lockstep episodes (problems.py:153-177), warp per genome, B = 1
// ---------------------------------------------------------------------------

// one synchronous pass over the program for a single input vector held in vals[slot]
template <typename T>
__device__ void warp_eval_single(const uint8_t* gp, const ProgLayout& L, T* vals) {
  const int lane = threadIdx.x & 31;
  const ProgHeader hdr = *reinterpret_cast<const ProgHeader*>(gp);
  const GroupRec* groups = reinterpret_cast<const GroupRec*>(gp + L.off_groups);
  const StepT<T>* steps = reinterpret_cast<const StepT<T>*>(gp + L.off_steps);
  const uint16_t* esrc = reinterpret_cast<const uint16_t*>(gp + L.off_src);
  const float* ew = reinterpret_cast<const float*>(gp + L.off_w);
  const EdgeD* ed = reinterpret_cast<const EdgeD*>(gp + L.off_w);
  for (int g = 0; g < hdr.n_groups; ++g) {
    const GroupRec gr = groups[g];
    const int stride = (gr.cls & GRP_GENERIC) ? 1 : group_width(gr.n);
    T y[4];
    for (int j = 0; j < gr.n; ++j) {
      const StepT<T> st = steps[gr.step_begin + j];
      T part = agg_neutral<T>(st.agg);
      const int h0 = (j == 0 && (gr.cls & GRP_SPLIT0)) ? gr.cnt[0] : 0x7FFFFFFF;  // split step 0
      for (int e = lane; e < st.count; e += 32) {
        const int idx = e < h0 ? gr.e_begin + e * stride + j : gr.e_begin + (e - h0) * stride + 3;
        uint32_t src;
        T w;
        if constexpr (sizeof(T) == 8) { src = ed[idx].src; w = ed[idx].w; }
        else { src = esrc[idx]; w = ew[idx]; }
        part = agg_combine<T>(st.agg, part, w * vals[src]);
      }
      y[j & 3] = eval_node<T>(st, warp_allreduce<T>(st.agg, part));
    }
    __syncwarp();
    if (lane == 0)
      for (int j = 0; j < gr.n; ++j) {
        const uint16_t sl = steps[gr.step_begin + j].slot;
        if (sl != NO_SLOT) vals[sl] = y[j & 3];
      }
    __syncwarp();
  }
}

// cos / sin of the pole angle, correctly rounded for |x| <= 0.5 (double-double
// Taylor sums; the cart-pole angle stays within ~0.21 rad).  numpy's float64
// cos/sin agree with glibc's correctly rounded results on this range, so the
// episode's float64 states follow the reference bit for bit (the CUDA libm
// versions are within 1-2 ulp and let chaotic episodes drift apart).
struct DD { double hi, lo; };
__device__ __forceinline__ DD dd_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = dd_two_sum(a.hi, b.hi);
  s.lo = __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo));
  return dd_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  const double p = __dmul_rn(a.hi, b.hi);
  const double e = fma(a.hi, b.hi, -p);
  return dd_two_sum(p, __dadd_rn(e, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi))));
}
// sum_{k=0..K} c_k * y^k (Horner, y = x^2) with double-double coefficients
// c_k = s * 1 / (j0 + 2k)! alternating; (hi, lo) pairs of 1/n! below
__device__ DD dd_series(DD y, bool is_sin) {
  // 1/n! for n = 0..19 as double-double (hi = RN(1/n!), lo = RN(1/n! - hi))
  const double fh[20] = {1.0, 1.0, 0.5, 1.6666666666666666e-01, 4.1666666666666664e-02, 8.3333333333333332e-03,
                         1.3888888888888889e-03, 1.9841269841269841e-04, 2.4801587301587302e-05,
                         2.7557319223985893e-06, 2.7557319223985888e-07, 2.5052108385441720e-08,
                         2.0876756987868100e-09, 1.6059043836821613e-10, 1.1470745597729725e-11,
                         7.6471637318198164e-13, 4.7794773323873853e-14, 2.8114572543455206e-15,
                         1.5619206968586225e-16, 8.2206352466243295e-18};
  const double fl[20] = {0.0, 0.0, 0.0, 9.2518585385429707e-18, 2.3129646346357427e-18, 1.1564823173178714e-19,
                         -5.3005439543735771e-20, 1.7209558293420705e-22, 2.1511947866775882e-23,
                         -1.8583932740464721e-22, 2.3767714622250297e-23, -1.4488140709359119e-24,
                         -1.2073450591132599e-25, 1.2585294588752098e-26, 2.0655512752830745e-28,
                         7.0387287773345300e-30, 4.3992054858340813e-31, 1.6508842730861433e-31,
                         1.1910679660273754e-32, 2.2141894119604265e-34};
  const int j0 = is_sin ? 1 : 0;
  DD acc = {0.0, 0.0};
  for (int k = 8; k >= 0; --k) {
    const int n = j0 + 2 * k;
    DD c = {(k & 1) ? -fh[n] : fh[n], (k & 1) ? -fl[n] : fl[n]};
    acc = dd_add(dd_mul(acc, y), c);
  }
  return acc;
}
__device__ __forceinline__ void cos_sin_cr(double x, double& c, double& s) {
  const double x2h = __dmul_rn(x, x);
  const DD y = {x2h, fma(x, x, -x2h)};
  const DD cs = dd_series(y, false);
  const DD sn = dd_mul(dd_series(y, true), DD{x, 0.0});
  c = __dadd_rn(cs.hi, cs.lo);
  s = __dadd_rn(sn.hi, sn.lo);
}

template <typename T>
__global__ void cartpole_kernel(const uint8_t* __restrict__ prog, ProgLayout L, int64_t P, int max_slots,
                                const double* __restrict__ start, int max_steps, double* __restrict__ fitness) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gi = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (gi >= P) return;
  T* vals = reinterpret_cast<T*>(smem) + (int64_t)warp * max_slots;
  const uint8_t* gp = prog + gi * L.stride;
  const uint16_t out0 = *reinterpret_cast<const uint16_t*>(gp + L.off_out);
  // classic constants (problems.py:37-47), evaluated as numpy does
  const double G = 9.8, PM = 0.1, TM = 1.0 + 0.1, HL = 0.5, PL = 0.1 * 0.5, FM = 10.0, TS = 0.02;
  const double XL = 2.4, THL = 12.0 * 2.0 * 3.141592653589793 / 360.0;
  double x = start[gi * 4 + 0], xd = start[gi * 4 + 1], th = start[gi * 4 + 2], thd = start[gi * 4 + 3];
  int steps = 0;
  for (int t = 0; t < max_steps; ++t) {
    if (lane == 0) { vals[0] = (T)x; vals[1] = (T)xd; vals[2] = (T)th; vals[3] = (T)thd; }
    __syncwarp();
    warp_eval_single<T>(gp, L, vals);
    const double out = out0 != NO_SLOT ? (double)vals[out0] : __longlong_as_double(0x7ff8000000000000ll);
    const double force = out > 0.0 ? FM : -FM;
    double ct, st;
    if (fabs(th) <= 0.5) cos_sin_cr(th, ct, st);
    else { ct = cos(th); st = sin(th); }
    const double tmp = __ddiv_rn(__dadd_rn(force, __dmul_rn(__dmul_rn(PL, __dmul_rn(thd, thd)), st)), TM);
    const double tacc = __ddiv_rn(__dsub_rn(__dmul_rn(G, st), __dmul_rn(ct, tmp)),
                                  __dmul_rn(HL, __dsub_rn(4.0 / 3.0, __ddiv_rn(__dmul_rn(PM, __dmul_rn(ct, ct)), TM))));
    const double xacc = __dsub_rn(tmp, __ddiv_rn(__dmul_rn(__dmul_rn(PL, tacc), ct), TM));
    x = __dadd_rn(x, __dmul_rn(TS, xd));
    xd = __dadd_rn(xd, __dmul_rn(TS, xacc));
    th = __dadd_rn(th, __dmul_rn(TS, thd));
    thd = __dadd_rn(thd, __dmul_rn(TS, tacc));
    ++steps;
    if (fabs(x) > XL || fabs(th) > THL) break;
  }
  if (lane == 0) fitness[gi] = (double)steps;
}

template <typename T>
int launch_warp(const uint8_t* prog, const ProgLayout& L, int64_t P, const T* in, int64_t in_gstride,
                int B, int I, int O, const int32_t* maxdims_host, T* out, int64_t out_gstride,
                int fit_kind, const double* targets, double* fitness, cudaStream_t st) {
  const int slots = maxdims_host[0] > 0 ? maxdims_host[0] : I + 1;
  int bchunk = B;
  if (fit_kind == FIT_NONE) {
    const int cap = (int)((48 * 1024) / ((int64_t)slots * sizeof(T)));
    bchunk = max(1, min(B, cap));
  }
  const int64_t per_warp = (int64_t)slots * bchunk * sizeof(T);
  int wpb = 4;
  while (wpb > 1 && per_warp * wpb > 200 * 1024) wpb >>= 1;
  if (per_warp * wpb > 227 * 1024) return -6;
  const int64_t tasks = P * ((B + bchunk - 1) / bchunk);
  const int64_t blocks = (tasks + wpb - 1) / wpb;
  const int64_t smem = per_warp * wpb;
  cudaFuncSetAttribute(fwd_warp_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fwd_warp_kernel<T><<<(unsigned)blocks, 32 * wpb, smem, st>>>(prog, L, P, in, in_gstride, B, I, O, bchunk,
                                                               slots, out, out_gstride, fit_kind, targets,
                                                               fitness);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

template <typename T, int S, int NT>
int launch_tile(const uint8_t* prog, const ProgLayout& L, const int32_t* ids, const T* in, int64_t in_gstride,
                int64_t P, int B, int I, int O, const int32_t* maxdims_host, T* out, int64_t out_gstride,
                int tpc, cudaStream_t st, const int32_t* count_dev = nullptr, float* gsq = nullptr) {
  constexpr int TT = NT * S;
  const int tiles = (B + TT - 1) / TT;
  tpc = max(1, min(tpc, tiles));
  const int runs = (tiles + tpc - 1) / tpc;
  int64_t grid = P * runs;
  if (count_dev) {  // device plan: a grid-striding launch of a few waves
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = min(grid, (int64_t)sms * 8);
  }
  if (grid > 0x7FFFFFFFll) return -5;
  if (grid == 0) return 0;
  const int64_t ms = maxdims_host[1], me = maxdims_host[2];
  const int64_t prog_bytes = ms * sizeof(GroupRec) + ms * sizeof(StepT<T>) +
                             (sizeof(T) == 8 ? 16 * me : align_up(4 * me, 16) + 4 * me);
  int64_t smem = align_up(prog_bytes, 16) + (int64_t)max(maxdims_host[0], I) * (TT + S) * sizeof(T);
  if (smem > 227 * 1024) return -6;
  cudaFuncSetAttribute(fwd_tile_kernel<T, S, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fwd_tile_kernel<T, S, NT><<<(unsigned)grid, NT, smem, st>>>(prog, L, ids, count_dev, in, in_gstride, B, I, O, runs, tpc,
                                                              out, out_gstride, gsq);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

// shared-memory configuration of a tensor-core launch whose genomes have at
// most ms steps and me edge entries: warpgroup areas, genome buffers (two
// unless a single one buys another warpgroup or is the only way one fits)
struct TcConfig {
  uint32_t wg_bytes, gbuf;
  int nbuf, nwg;
  int64_t smem;
  bool ok;
};
inline TcConfig tc_config(int ms, int me, int max_wg) {
  TcConfig c;
  const int nb = tc_rows(ms);
  c.wg_bytes = tc_wg_bytes(nb);
  c.gbuf = (uint32_t)align_up(tc_block(ms, ms, me).bytes + 64, 128);  // + look-ahead slack
  const int64_t budget = 227 * 1024, ctl = (int64_t)align_up(sizeof(TcShared), 16);
  auto fit = [&](int nbuf) {
    int w = max_wg > 0 ? min(max_wg, TC_MAX_WG) : TC_MAX_WG;
    while (w > 1 && ctl + nbuf * (int64_t)c.gbuf + (int64_t)w * c.wg_bytes > budget) --w;
    return w;
  };
  const bool two_fit = ctl + 2ll * c.gbuf + (int64_t)c.wg_bytes <= budget;
  c.nbuf = (!two_fit || fit(1) > fit(2)) ? 1 : 2;
  c.nwg = fit(c.nbuf);
  c.smem = ctl + c.nbuf * (int64_t)c.gbuf + (int64_t)c.nwg * c.wg_bytes;
  c.ok = c.smem <= budget && 4 * nb <= 512;
  return c;
}

// TC programs: maxdims_host = (slots, steps, edge entries) maxima over the
// launched genomes (all MODE_TC).  Persistent grid: one CTA per SM (or fewer
// for small launches) with as many warpgroups as shared memory allows.
int launch_tc(const uint8_t* prog, const ProgLayout& L, const int32_t* ids, const float* in, int64_t in_gstride,
              int64_t P, int B, int I, int O, const int32_t* maxdims_host, float* out, int64_t out_gstride,
              int max_wg, cudaStream_t st, const int32_t* count_dev = nullptr, float* gsq = nullptr,
              int32_t* task_ctr = nullptr, bool pdl = false) {
  if (I > TC_K || (I & 3) || (((uintptr_t)in) & 15)) return -8;
  const int ms = max(maxdims_host[1], 1), me = maxdims_host[2];
  const int nb = tc_rows(ms);
  if (4 * nb > 512) return -8;
  const TcConfig cfg = tc_config(ms, me, max_wg);
  if (!cfg.ok) return -6;
  const uint32_t wg_bytes = cfg.wg_bytes, gbuf = cfg.gbuf;
  const int nbuf = cfg.nbuf, nwg = cfg.nwg;
  const int64_t smem = cfg.smem;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = P < sms ? P : sms;
  const PFN_cuTensorMapEncodeTiled_v12000 encode = tmap_encoder();
  if (!encode) return -9;
  // inputs as an (I, B, genomes) fp32 tensor; boxes of 32 inputs x 256 rows
  // (zero fill past I and B), 128-byte swizzle (conflict-free row reads)
  CUtensorMap tmap;
  const cuuint64_t dims[3] = {(cuuint64_t)I, (cuuint64_t)B, in_gstride ? (cuuint64_t)1 << 30 : 1};
  const cuuint64_t strides[2] = {(cuuint64_t)I * 4, (cuuint64_t)(in_gstride ? in_gstride : (int64_t)B * I) * 4};
  const cuuint32_t box[3] = {TC_K, TC_TT, 1}, estr[3] = {1, 1, 1};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -9;
  cudaFuncSetAttribute(fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (grid == 0) return 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3((unsigned)(TC_NT * nwg));
  lc.dynamicSmemBytes = (size_t)smem;
  lc.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = la;
  lc.numAttrs = pdl ? 1 : 0;
  const cudaError_t le = cudaLaunchKernelEx(&lc, fwd_tc_kernel, tmap, prog, L, ids, count_dev, P, in, in_gstride, B, I,
                                            O, nwg, wg_bytes, gbuf, nbuf, nb, gsq, out, out_gstride, task_ctr);
  if (le != cudaSuccess) return -100 - (int)le;
  TNEAT_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// device-side launch plan of an FMT_TC population (no host read-back)
// ---------------------------------------------------------------------------
// Class of a genome (plan_tc_kernel): 0..4 tensor-core programs by MMA width (round16(steps) <=
// 32, 48, 64, 96, 128: 4, 4, 3, 2, 1 warpgroups per CTA) whose hidden-edge
// entries fit the class buffer; 5 tensor-core programs with more entries
// (buffer sized by the capacity); 6 standard
// programs (the tile kernel with capacity-sized shared memory).  A thread per
// genome, positions claimed per warp with one atomic per class: ids[c * P + i]
// = the class's genomes (in no particular order), counts[c].
constexpr int TC_NCLASS = 7;
constexpr int TC_CLASS_EDGES = 512;
__host__ __device__ inline int tc_class_nb(int c) { return c == 0 ? 32 : c == 1 ? 48 : c == 2 ? 64 : c == 3 ? 96 : 128; }

__global__ void __launch_bounds__(1024) plan_tc_kernel(const uint8_t* __restrict__ prog, int64_t stride, int64_t P,
                                                       int32_t* __restrict__ ids, int32_t* __restrict__ counts) {
  // one genome per thread over as many CTAs as needed; each warp claims its
  // positions per class with one atomic (counts zeroed on the stream first).
  // The order inside a class is the order the warps reach the counters: the
  // class launches hand tasks out dynamically, so no order is needed.
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int cls = -1;
  if (g < P) {
    const ProgHeader h = *reinterpret_cast<const ProgHeader*>(prog + g * stride);
    if (h.mode != MODE_TC) {
      cls = 6;
    } else {
      const int nb = tc_rows(h.n_steps);
      cls = h.n_edges > TC_CLASS_EDGES ? 5 : nb <= 32 ? 0 : nb <= 48 ? 1 : nb <= 64 ? 2 : nb <= 96 ? 3 : 4;
    }
  }
#pragma unroll
  for (int c = 0; c < TC_NCLASS; ++c) {
    const unsigned m = __ballot_sync(0xffffffffu, cls == c);
    if (!m) continue;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counts + c, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (cls == c) ids[(int64_t)c * P + base + __popc(m & ((1u << lane) - 1))] = (int32_t)g;
  }
}

// forward of a whole FMT_TC population from the device plan: the plan kernel,
// then one persistent launch per tensor-core class and a grid-striding tile
// launch for standard programs, every launch sized from class bounds (no
// host-side counts or extents)
int launch_planned(const uint8_t* prog, const ProgLayout& L, int N, int C, int32_t* ids, int32_t* counts,
                   const float* in, int64_t in_gstride, int64_t P, int B, int I, int O, float* out,
                   int64_t out_gstride, float* gsq, cudaStream_t st) {
  const int steps_cap = N < 128 ? N : 128;
  {  // every class launch must fit before anything is enqueued (-6: the caller
     // plans on the host instead -- very large genome capacities)
    if (!tc_config(steps_cap, (int)edge_capacity(N, C), 0).ok) return -6;
    const int64_t tile_smem = align_up(32ll * N + 8ll * edge_capacity(N, C) + 16, 16) + (int64_t)(N + 2) * 130 * 4;
    if (tile_smem > 227 * 1024) return -6;
  }
  // class counts and the class launches' task counters start at zero
  if (cudaMemsetAsync(counts, 0, 2 * TC_NCLASS * sizeof(int32_t), st) != cudaSuccess) return -100 - (int)cudaGetLastError();
  plan_tc_kernel<<<(unsigned)((P + 1023) / 1024), 1024, 0, st>>>(prog, L.stride, P, ids, counts);
  TNEAT_CHECK_LAUNCH();
  // class launches after the first are programmatic dependent launches: each
  // one's CTAs start on SMs the previous launch's drain frees (the launches are
  // independent: disjoint genomes, their own task counters; the plan they
  // read completed before the first one started)
  bool first = true;
  for (int c = 0; c < TC_NCLASS - 1; ++c) {
    const int nb = c < 5 ? tc_class_nb(c) : tc_rows(steps_cap);
    if (c < 5 && nb > tc_rows(steps_cap) && c > 0 && tc_class_nb(c - 1) >= tc_rows(steps_cap)) continue;  // empty by construction
    const int32_t md[3] = {nb + 1, nb, c < 5 ? TC_CLASS_EDGES : (int)edge_capacity(N, C)};
    const int r = launch_tc(prog, L, ids + (int64_t)c * P, in, in_gstride, P, B, I, O, md, out, out_gstride, 0, st,
                            counts + c, gsq, counts + TC_NCLASS + c, !first);
    if (r) return r;
    first = false;
  }
  // standard programs (genomes the tensor-core format cannot take, cyclic or
  // invalid genomes): capacity-sized tile launch
  const int32_t md[3] = {N + 2, N, (int)edge_capacity(N, C)};
  return launch_tile<float, 2, 64>(prog, L, ids + 6 * P, in, in_gstride, P, B, I, O, md, out, out_gstride, 4, st,
                                   counts + 6, gsq);
}

}  // namespace tneat

using namespace tneat;

extern "C" {

// Replaces inference.forward_arrays (inference.py:185-262).  See include/tneat.h.
int an_forward(const void* program, int64_t program_stride, int N, int C, int precision,
               const int32_t* maxdims_host, const int32_t* genome_ids, const void* inputs,
               int64_t input_genome_stride, int64_t P, int B, int I, int O, void* outputs, int variant,
               void* stream) {
  if (P < 0 || B < 0 || I < 1 || O < 1 || !maxdims_host) return -1;
  if (P == 0 || B == 0) return 0;
  if (!program || !inputs || !outputs) return -2;
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (L.stride != program_stride) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* pg = (const uint8_t*)program;
  const int64_t ogs = (int64_t)B * O;
  // variant (low 4 bits): 0 = auto, 1 = tile S=1 (128 thr), 2 = tile S=2 (128 thr),
  // 3 = tile S=1 (64 thr), 4 = tile S=4 (64 thr), 5 = tile S=2 (64 thr), 6 = tile S=4 (32 thr),
  // 8 = warp kernel, 11 = tensor-core kernel (FMT_TC programs whose header
  // mode is MODE_TC; the other genomes of an FMT_TC population are standard
  // programs for the variants above); bits 8..15 = tiles per CTA (0 = default
  // 4; tensor-core kernel: maximum warpgroups per CTA, 0 = as many as fit)
  int tpc = (variant >> 8) & 0xFF;
  variant &= 0xF;
  if (variant == 11) {
    if (!(precision & FMT_TC)) return -7;
    return launch_tc(pg, L, genome_ids, (const float*)inputs, input_genome_stride, P, B, I, O, maxdims_host,
                     (float*)outputs, ogs, tpc & 0xF, st);
  }
  if (tpc == 0) tpc = 4;
  // an FMT_TC population holds tensor-core programs the standard kernels cannot
  // read: they take explicitly listed standard-program genomes only
  if ((precision & FMT_TC) && !genome_ids) return -7;
  if (variant == 0) variant = B >= 192 ? ((precision & FMT_F64) ? 1 : 5) : (B >= 96 ? 3 : 8);  // fp64: one sample per thread
  if (variant == 8) {
    if (genome_ids) return -7;
    if (precision & FMT_F64)
      return launch_warp<double>(pg, L, P, (const double*)inputs, input_genome_stride, B, I, O, maxdims_host,
                                 (double*)outputs, ogs, FIT_NONE, nullptr, nullptr, st);
    return launch_warp<float>(pg, L, P, (const float*)inputs, input_genome_stride, B, I, O, maxdims_host,
                              (float*)outputs, ogs, FIT_NONE, nullptr, nullptr, st);
  }
  const int32_t* ids = genome_ids;
  if (precision & FMT_F64) {
    const double* in = (const double*)inputs;
    double* out = (double*)outputs;
    if (variant == 2 || variant == 5)
      return launch_tile<double, 2, 64>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
    if (variant == 3)  // half the samples per CTA: fp64 value rows are twice as wide
      return launch_tile<double, 1, 64>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
    return launch_tile<double, 1, 128>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
  }
  const float* in = (const float*)inputs;
  float* out = (float*)outputs;
  switch (variant) {
    case 2: return launch_tile<float, 2, 128>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
    case 3: return launch_tile<float, 1, 64>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
    case 4: return launch_tile<float, 4, 64>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
    case 5: return launch_tile<float, 2, 64>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
    case 6: return launch_tile<float, 4, 32>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
    default: return launch_tile<float, 1, 128>(pg, L, ids, in, input_genome_stride, P, B, I, O, maxdims_host, out, ogs, tpc, st);
  }
}

// FMT_TC populations: forward from a device-side launch plan (no host-known
// launch sizes; see include/tneat.h).  plan_ids: int32[7 * P] and
// plan_counts: int32[14] scratch owned by the caller ([7..13]: task counters).
int an_forward_planned(const void* program, int64_t program_stride, int N, int C, int precision, int32_t* plan_ids,
                       int32_t* plan_counts, const void* inputs, int64_t input_genome_stride, int64_t P, int B, int I,
                       int O, void* outputs, float* genome_sq, void* stream) {
  if (P < 0 || B < 0 || I < 1 || O < 1) return -1;
  if (!(precision & FMT_TC) || (precision & FMT_F64)) return -7;
  if (P == 0 || B == 0) return 0;
  if (!program || !inputs || !outputs || !plan_ids || !plan_counts) return -2;
  if (P > 0x7FFFFFFF / TC_NCLASS) return -5;
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (L.stride != program_stride) return -3;
  return launch_planned((const uint8_t*)program, L, N, C, plan_ids, plan_counts, (const float*)inputs,
                        input_genome_stride, P, B, I, O, (float*)outputs, (int64_t)B * O, genome_sq,
                        (cudaStream_t)stream);
}

int an_plan_tc(const void* program, int64_t program_stride, int64_t P, int32_t* plan_ids, int32_t* plan_counts,
               void* stream) {
  if (P < 0) return -1;
  if (!program || !plan_ids || !plan_counts) return -2;
  if (P > 0x7FFFFFFF / TC_NCLASS) return -5;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(plan_counts, 0, 2 * TC_NCLASS * sizeof(int32_t), st) != cudaSuccess)
    return -100 - (int)cudaGetLastError();
  if (P == 0) return 0;
  plan_tc_kernel<<<(unsigned)((P + 1023) / 1024), 1024, 0, st>>>((const uint8_t*)program, program_stride, P,
                                                                  plan_ids, plan_counts);
  TNEAT_CHECK_LAUNCH();
  return 0;
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
  if (precision & FMT_TC) return -7;  // standard programs only
  if (P == 0) return 0;
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (L.stride != program_stride) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  if (precision & FMT_F64)
    return launch_warp<double>((const uint8_t*)program, L, P, (const double*)inputs, input_genome_stride, B, I,
                               O, maxdims_host, nullptr, 0, kind, targets, fitness, st);
  return launch_warp<float>((const uint8_t*)program, L, P, (const float*)inputs, input_genome_stride, B, I, O,
                            maxdims_host, nullptr, 0, kind, targets, fitness, st);
}

// Cart-pole lockstep fitness (problems.py:153-177, 257-271): start (P,4) float64
// states, episodes of at most max_steps, fitness = steps survived.
int an_cartpole(const void* program, int64_t program_stride, int N, int C, int precision,
                const int32_t* maxdims_host, int64_t P, const double* start, int max_steps, double* fitness,
                void* stream) {
  if (P < 0 || !maxdims_host || max_steps < 0) return -1;
  if (precision & FMT_TC) return -7;  // standard programs only
  if (P == 0) return 0;
  const ProgLayout L = prog_layout(N, C, 1, precision);
  if (L.stride != program_stride) return -3;
  const int slots = max(maxdims_host[0], 4);
  const int wpb = 4;
  const int64_t smem = (int64_t)wpb * slots * (precision ? 8 : 4);
  const int64_t blocks = (P + wpb - 1) / wpb;
  cudaStream_t st = (cudaStream_t)stream;
  if (precision)
    cartpole_kernel<double><<<(unsigned)blocks, 32 * wpb, smem, st>>>((const uint8_t*)program, L, P, slots,
                                                                      start, max_steps, fitness);
  else
    cartpole_kernel<float><<<(unsigned)blocks, 32 * wpb, smem, st>>>((const uint8_t*)program, L, P, slots,
                                                                     start, max_steps, fitness);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
