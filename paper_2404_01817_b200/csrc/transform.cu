// K1: genome transform -- endpoint key lookup, enabled mask, Kahn order,
// ancestor-cone pruning and program emission, one warp per genome.
//
// Replaces arrayneat inference.transform_arrays (inference.py:82-147):
//   * key -> row resolution (search.py:103-124) by a warp bitonic sort of the
//     live (key,row) pairs and binary search -- exact integer work;
//   * enabled = live & enabled==1.0 (inference.py:93-95);
//   * Kahn with the smallest ready ROW first, one node per step
//     (inference.py:127-141): the ready set is a bitset in shared memory, the
//     minimum is a warp __reduce_min over per-lane first-nonzero words, the
//     successor decrements run lane-parallel;
//   * cyclic genomes flagged (inference.py:143).
// The dense (P,N,N) `incoming` tensor of the reference is NOT materialised;
// the kernel compiles each genome into a program (common.cuh): level-sorted,
// grouped steps with per-step edge lists and liveness-recycled value slots.

#include "common.cuh"
#include "digits.cuh"
#include <cuda_fp16.h>

namespace tneat {

constexpr uint64_t U64_MAX = ~0ull;
// group join rule: a step joins if DEN * count >= NUM * (longest count); 1/2
// bounds the padded entries (edge_capacity) -- tighter rules only shrink them
#ifndef TNEAT_JOIN_NUM
#define TNEAT_JOIN_NUM 1
#define TNEAT_JOIN_DEN 2
#endif
constexpr int32_t NEVER = 0x7FFFFFFF;
constexpr uint8_t F_LIVE = 1, F_INPUT = 2, F_OUTPUT = 4, F_FREED = 8, F_TANH_SUM = 16;

// Edge keys (dst, src, connection row) and step sort keys (level, class,
// -count, position), packed so that integer order is the sort order.  Genomes
// with N <= 256 and C <= 16383 use 32-bit keys and byte successor lists: a
// genome-warp then needs 10.7 instead of 13.7 KB of shared memory at 128/512
// (more resident warps -- the transform is latency-bound).
template <bool SMALL> struct KeyTraits;
template <> struct KeyTraits<false> {
  using E = uint64_t;
  using G = uint64_t;
  using Succ = uint16_t;
  using Idx = int32_t;  // CSR starts (<= C)
  static constexpr int DSH = 48, SSH = 32;
  static constexpr uint32_t FM = 0xFFFF;
  static constexpr G GMAX = ~0ull;
  __device__ static E make(int d, int s, int c) { return ((uint64_t)d << 48) | ((uint64_t)s << 32) | (uint64_t)c; }
  __device__ static int dst(E k) { return (int)((k >> 48) & 0xFFFF); }
  __device__ static int src(E k) { return (int)((k >> 32) & 0xFFFF); }
  __device__ static int64_t row(E k) { return (int64_t)(k & 0xFFFFFFFFu); }
  __device__ static bool same_pair(E a, E b) { return ((a ^ b) >> 32) == 0; }
  __device__ static G gmake(uint32_t lv, uint32_t cls, uint32_t cnt, uint32_t pos) {
    return ((uint64_t)lv << 48) | ((uint64_t)cls << 47) | ((uint64_t)(0xFFFF - cnt) << 16) | (uint64_t)pos;
  }
  __device__ static int gpos(G k) { return (int)(k & 0xFFFF); }
  __device__ static int gcnt(G k) { return 0xFFFF - (int)((k >> 16) & 0xFFFF); }
  __device__ static int gcls(G k) { return (int)((k >> 47) & 1); }
  __device__ static int glv(G k) { return (int)(k >> 48); }
};
template <> struct KeyTraits<true> {
  using E = uint32_t;
  using G = uint32_t;
  using Succ = uint8_t;
  using Idx = int16_t;  // CSR starts (<= C <= 16383)
  static constexpr int DSH = 24, SSH = 16;
  static constexpr uint32_t FM = 0xFF;
  static constexpr G GMAX = ~0u;
  __device__ static E make(int d, int s, int c) { return ((uint32_t)d << 24) | ((uint32_t)s << 16) | (uint32_t)c; }
  __device__ static int dst(E k) { return (int)((k >> 24) & 0xFF); }
  __device__ static int src(E k) { return (int)((k >> 16) & 0xFF); }
  __device__ static int64_t row(E k) { return (int64_t)(k & 0xFFFFu); }
  __device__ static bool same_pair(E a, E b) { return ((a ^ b) >> 16) == 0; }
  __device__ static G gmake(uint32_t lv, uint32_t cls, uint32_t cnt, uint32_t pos) {
    return (lv << 24) | (cls << 23) | ((0x3FFFu - cnt) << 9) | pos;
  }
  __device__ static int gpos(G k) { return (int)(k & 0x1FF); }
  __device__ static int gcnt(G k) { return 0x3FFF - (int)((k >> 9) & 0x3FFF); }
  __device__ static int gcls(G k) { return (int)((k >> 23) & 1); }
  __device__ static int glv(G k) { return (int)(k >> 24); }
};
__host__ __device__ inline bool small_keys(int N, int C) { return N <= 256 && C <= 16383; }

template <typename KT>
struct WarpSmem {
  using E = typename KT::E;
  using G = typename KT::G;
  uint64_t* skey;     // [Npad]   (key << 16 | row), sorted; dead from Kahn on
  E* ekey;            // [Cpad]   edge keys, sorted (CSR by destination)
  E* ekey2;           // [C]      unsorted staging for the counting sort
  G* gkey;            // [pow2(N - I)] step sort keys
  int32_t* indeg;     // [N]
  int32_t* outdeg;    // [N]
  typename KT::Idx* in_start;  // [N+1]    CSR by destination into ekey
  typename KT::Idx* su_start;  // [N+1]    CSR by source into succ (TC programs: the step's weight exponent)
  int32_t* lvl;       // [N]      topological level
  int32_t* last_grp;  // [N+1]    last group that reads the node (level starts during Kahn)
  typename KT::Succ* succ;  // [C] destination rows, CSR by source
  uint16_t* order;    // [N]
  uint16_t* slot_of;  // [N]
  uint16_t* step_row; // [N - I]
  uint16_t* grp_of;   // [N - I]
  GroupRec* grp;      // [N - I]  (steps are non-input nodes)
  uint8_t* flags;     // [N]
  uint8_t* needed;    // [N]
  uint8_t* used;      // [N]
  uint32_t* ready;    // [W]
  uint32_t* freemask; // [WS]
};

__host__ __device__ inline int next_pow2(int x) {
  int p = 32;
  while (p < x) p <<= 1;
  return p;
}

template <bool kCarve, typename KT>
__host__ __device__ inline int64_t layout_warp(uint8_t* base, int N, int C, int I, WarpSmem<KT>* s) {
  using E = typename KT::E;
  using G = typename KT::G;
  using Idx = typename KT::Idx;
  const int Npad = next_pow2(N), Cpad = next_pow2(C);
  const int S = N - I > 1 ? N - I : 1, Spad = next_pow2(S);  // steps are non-input nodes
  const int W = (N + 31) / 32, WS = (N + 2 + 31) / 32;
  int64_t o = 0;
  auto take = [&](int64_t bytes, int64_t al) {
    o = align_up(o, al);
    const int64_t at = o;
    o += bytes;
    return at;
  };
  const int64_t a_ekey = take((int64_t)sizeof(E) * Cpad, 8);
  // union: the key table and ekey2 (edge staging), both dead once the CSR is
  // built (the io rows are looked up before Kahn), share memory with the
  // arrays first written by Kahn and after it (gkey, grp, last_grp, step_row,
  // grp_of)
  const int64_t a_union = take(0, 16);
  const int64_t a_gkey = take((int64_t)sizeof(G) * Spad, 8), a_grp = take(16ll * S, 16);
  const int64_t a_last = take(4ll * (N + 1), 4);  // also the level starts of the level-synchronous Kahn
  const int64_t a_srow = take(2ll * S, 2), a_grpof = take(2ll * S, 2);
  const int64_t a_skey = a_union, a_ekey2 = align_up(a_union + 8ll * Npad, 8);
  const int64_t front = a_ekey2 + (int64_t)sizeof(E) * (C > 0 ? C : 1) - a_union;
  o = a_union + (o - a_union > front ? o - a_union : front);
  const int64_t a_indeg = take(4ll * N, 4), a_outdeg = take(4ll * N, 4);
  const int64_t a_in = take((int64_t)sizeof(Idx) * (N + 1), 4), a_su = take((int64_t)sizeof(Idx) * (N + 1), 4);
  const int64_t a_lvl = take(4ll * N, 4);
  const int64_t a_succ = take((int64_t)sizeof(typename KT::Succ) * C, 2), a_order = take(2ll * N, 2),
                a_slot = take(2ll * N, 2);
  const int64_t a_flags = take(N, 1), a_needed = take(N, 1), a_used = take(N, 1);
  const int64_t a_ready = take(4ll * W, 4), a_free = take(4ll * WS, 4);
  if (kCarve) {
    s->skey = (uint64_t*)(base + a_skey);
    s->ekey = (E*)(base + a_ekey);
    s->ekey2 = (E*)(base + a_ekey2);
    s->gkey = (G*)(base + a_gkey);
    s->indeg = (int32_t*)(base + a_indeg);
    s->outdeg = (int32_t*)(base + a_outdeg);
    s->in_start = (Idx*)(base + a_in);
    s->su_start = (Idx*)(base + a_su);
    s->lvl = (int32_t*)(base + a_lvl);
    s->last_grp = (int32_t*)(base + a_last);
    s->grp = (GroupRec*)(base + a_grp);
    s->succ = (typename KT::Succ*)(base + a_succ);
    s->order = (uint16_t*)(base + a_order);
    s->slot_of = (uint16_t*)(base + a_slot);
    s->step_row = (uint16_t*)(base + a_srow);
    s->grp_of = (uint16_t*)(base + a_grpof);
    s->flags = base + a_flags;
    s->needed = base + a_needed;
    s->used = base + a_used;
    s->ready = (uint32_t*)(base + a_ready);
    s->freemask = (uint32_t*)(base + a_free);
  }
  return align_up(o, 16);
}

__host__ inline int64_t warp_smem_bytes(int N, int C, int I) {
  if (small_keys(N, C)) return layout_warp<false, KeyTraits<true>>(nullptr, N, C, I, nullptr);
  return layout_warp<false, KeyTraits<false>>(nullptr, N, C, I, nullptr);
}

// ascending bitonic sort of n (power of two, >= 32) values, one warp
template <typename K>
__device__ void warp_bitonic_sort(K* a, int n) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < (n >> 1); t += 32) {  // compare-exchange pair t: (i, i + j)
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int l = i + j;
        const K x = a[i], y = a[l];
        const bool up = (i & k) == 0;
        if ((x > y) == up) { a[i] = y; a[l] = x; }
      }
      __syncwarp();
    }
  }
}

// exclusive scan of cnt[0..n) into out[0..n]; out[n] = total. One warp.
template <typename OutT>
__device__ void warp_exclusive_scan(const int32_t* cnt, OutT* out, int n) {
  const int lane = threadIdx.x & 31;
  int32_t carry = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int32_t v = i < n ? cnt[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (i < n) out[i] = (OutT)(carry + x - v);
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) out[n] = (OutT)carry;
  __syncwarp();
}

// Stable scatter of n edge keys into buckets by the 16-bit field at `shift`
// (bucket b starts at start[b]; cursor[] zeroed by the caller).  Chunks of 32
// keep the input order: lanes with equal buckets rank themselves with
// __match_any_sync and the lowest of them advances the bucket cursor.  With
// `succ`, also writes the destination row (bits 48..63) of each key at its
// position (the CSR by source).
template <typename KT>
__device__ void stable_scatter(const typename KT::E* in, typename KT::E* out, int n, int shift,
                               const typename KT::Idx* start, int32_t* cursor, typename KT::Succ* succ) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const bool valid = i < n;
    const typename KT::E k = valid ? in[i] : 0;
    const uint32_t b = valid ? (uint32_t)((k >> shift) & KT::FM) : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(peers) - 1;
    int old = 0;
    if (valid && lane == leader) {
      old = cursor[b];
      cursor[b] = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    if (valid) {
      const int pos = start[b] + old + __popc(peers & ((1u << lane) - 1));
      out[pos] = k;
      if (succ) succ[pos] = (typename KT::Succ)KT::dst(k);
    }
    __syncwarp();
  }
}

// row of `key` among the sorted live (key<<16|row) pairs, or -1: branchless
// search over the power-of-two table (packed entries compare against key<<16
// directly, keys < 2^47); the smallest row wins for a repeated key
__device__ inline int lookup_row(const uint64_t* skey, int Npad, uint64_t key) {
  const uint64_t kk = key << 16;
  int pos = 0;
  for (int step = Npad >> 1; step > 0; step >>= 1) pos = skey[pos + step - 1] < kk ? pos + step : pos;
  const uint64_t e = skey[pos];
  return (e != U64_MAX && (e >> 16) == key) ? (int)(e & 0xFFFF) : -1;
}

// both endpoints of a connection at once: two independent search chains
__device__ inline void lookup_rows2(const uint64_t* skey, int Npad, uint64_t ka, uint64_t kb, int& ra, int& rb) {
  const uint64_t sa = ka << 16, sb = kb << 16;
  int pa = 0, pb = 0;
  for (int step = Npad >> 1; step > 0; step >>= 1) {
    pa = skey[pa + step - 1] < sa ? pa + step : pa;
    pb = skey[pb + step - 1] < sb ? pb + step : pb;
  }
  const uint64_t ea = skey[pa], eb = skey[pb];
  ra = (ea != U64_MAX && (ea >> 16) == ka) ? (int)(ea & 0xFFFF) : -1;
  rb = (eb != U64_MAX && (eb >> 16) == kb) ? (int)(eb & 0xFFFF) : -1;
}

// one connection row's in key, out key and enabled flag (16-byte key load
// when the population is 16-byte aligned; rows are 32 bytes)
__device__ __forceinline__ void load_conn(const double* gc, int c, bool vec, double& ik, double& ok, double& en) {
  if (vec) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(gc + (int64_t)c * 4));
    ik = a.x;
    ok = a.y;
  } else {
    ik = __ldg(gc + (int64_t)c * 4);
    ok = __ldg(gc + (int64_t)c * 4 + 1);
  }
  en = __ldg(gc + (int64_t)c * 4 + 2);
}

__device__ inline bool key_ok(double k) {
  return k >= 0.0 && k < 140737488355328.0 /* 2^47 */ && k == floor(k);
}

// lowest set bit over words[0..nw) (lane-strided ownership); -1 if none
__device__ inline int warp_first_set(const uint32_t* words, int nw) {
  const int lane = threadIdx.x & 31;
  unsigned mine = 0xFFFFFFFFu;
  for (int w = lane; w < nw; w += 32)
    if (words[w]) { mine = (unsigned)w; break; }
  const unsigned wmin = __reduce_min_sync(0xffffffffu, mine);
  if (wmin == 0xFFFFFFFFu) return -1;
  return (int)wmin * 32 + __ffs(words[wmin]) - 1;
}

// TNEAT_DIAG_TR_STOP=k (diagnostic builds, tools/build_variant.py): the kernel
// returns before phase k's successor (6 entry, 7 nodes, 1 connections, 2 CSR
// and repeated pairs, 3 io rows + Kahn, 4 pruning + TC eligibility, 5 steps /
// groups / slots; the full kernel adds the program writes) --
// tools/time_transform.py times the cumulative phases
#ifndef TNEAT_TR_WPB
#define TNEAT_TR_WPB 1  // one genome-warp per CTA: its shared memory is released as soon as it finishes
#endif
// register bounds: fp32 small-key genomes are shared-memory-limited at 24 per
// SM (80 registers); fp64 ones (small genomes, evolution) fit 32 at 62
template <typename T, bool SMALL>
__global__ void __launch_bounds__(32 * TNEAT_TR_WPB, SMALL ? (sizeof(T) == 8 ? 32 : 24) / TNEAT_TR_WPB : 1) transform_kernel(const double* __restrict__ nodes, const double* __restrict__ conns,
                                 int64_t P, int N, int C, int I, int O, int mode, int prune, bool tc,
                                 int64_t wsmem, uint8_t* __restrict__ prog, ProgLayout L,
                                 int16_t* __restrict__ order_out, int16_t* __restrict__ conn_rows,
                                 int32_t* __restrict__ io_rows, int32_t* __restrict__ status_out,
                                 int32_t* __restrict__ maxdims) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= P) return;
  using KT = KeyTraits<SMALL>;
  WarpSmem<KT> s;
  layout_warp<true, KT>(smem + warp * wsmem, N, C, I, &s);
  const int Npad = next_pow2(N);
  const double* gn = nodes + g * (int64_t)N * 5;
  const double* gc = conns + g * (int64_t)C * 4;
  const int io = I + O;
  const bool recurrent = mode == 1;
  int status = 0;

#if defined(TNEAT_DIAG_TR_STOP) && TNEAT_DIAG_TR_STOP == 6  // diagnostic builds only: phase split
  return;
#endif
  // ---- nodes: live mask, key table ------------------------------------------
  int n_live = 0;
  for (int r = lane; r < Npad; r += 32) {
    uint64_t packed = U64_MAX;
    if (r < N) {
      uint8_t f = 0;
      // the three fields in flight together: one round trip per row
      const double k = __ldg(gn + (int64_t)r * 5), gv = __ldg(gn + (int64_t)r * 5 + 3),
                   av = __ldg(gn + (int64_t)r * 5 + 4);
      if (!isnan(k)) {
        if (!key_ok(k)) status |= ST_BAD_KEY;
        const uint64_t ki = (uint64_t)k;
        packed = (ki << 16) | (uint64_t)r;
        f = F_LIVE | (ki < (uint64_t)I ? F_INPUT : 0) | (ki >= (uint64_t)I && ki < (uint64_t)io ? F_OUTPUT : 0);
        ++n_live;
        if (ki >= (uint64_t)I) {  // the reference evaluates every live non-input node (pruned ones too)
          if (!(av >= 0.0 && av < ACT_COUNT && av == floor(av))) status |= ST_BAD_ACT;
          if (!(gv >= 0.0 && gv < AGG_COUNT && gv == floor(gv))) status |= ST_BAD_AGG;
          if (av == (double)ACT_TANH && gv == (double)AGG_SUM) f |= F_TANH_SUM;  // read by the group pass
        }
      }
      s.flags[r] = f;
      s.needed[r] = 0;
      s.used[r] = 0;
      s.indeg[r] = 0;
      s.outdeg[r] = 0;
      s.lvl[r] = 0;
      s.slot_of[r] = NO_SLOT;
    }
    s.skey[r] = packed;
  }
  n_live = __reduce_add_sync(0xffffffffu, n_live);
  // io fast path (search.py:112-114): io keys 0..I+O-1 at rows 0..I+O-1 resolve
  // without a search (the sorted table gives the same rows)
  bool io_fast = true;
  for (int r = lane; r < io; r += 32) io_fast = io_fast && gn[(int64_t)r * 5] == (double)r;
  io_fast = __all_sync(0xffffffffu, io_fast);
  __syncwarp();
  warp_bitonic_sort(s.skey, Npad);

#if defined(TNEAT_DIAG_TR_STOP) && TNEAT_DIAG_TR_STOP == 7  // diagnostic builds only: phase split
  return;
#endif
  // ---- conns: endpoint rows, enabled mask, compacted edge keys ----------------
  int n_en = 0;
  // rows software-pipelined: the next iteration's row is in flight during this
  // one's searches (a genome's transform is latency-bound when few genomes
  // share an SM, e.g. one GPU's shard of a multi-GPU population)
  const bool vec = ((uint64_t)gc & 15) == 0;
  double nik = 0.0, nok = 0.0, nen = 0.0;
  if (lane < C) load_conn(gc, lane, vec, nik, nok, nen);
  for (int base = 0; base < C; base += 32) {
    const int c = base + lane;
    bool en = false;
    int sr = -1, dr = -1;
    const double ik = nik, ok = nok, env = nen;
    if (c + 32 < C) load_conn(gc, c + 32, vec, nik, nok, nen);
    if (c < C) {
      if (!isnan(ik)) {
        if (!key_ok(ik) || !key_ok(ok)) {
          status |= ST_BAD_KEY;
        } else {
          const bool fs = io_fast && ik < (double)io, fd = io_fast && ok < (double)io;
          if (fs && fd) {
            sr = (int)ik;
            dr = (int)ok;
          } else {
            lookup_rows2(s.skey, Npad, (uint64_t)ik, (uint64_t)ok, sr, dr);
            if (fs) sr = (int)ik;
            if (fd) dr = (int)ok;
          }
          if (sr < 0 || dr < 0) status |= ST_DANGLING;
          else en = env == 1.0;
        }
      }
      if (conn_rows) {
        conn_rows[(g * C + c) * 2 + 0] = en ? (int16_t)sr : (int16_t)-1;
        conn_rows[(g * C + c) * 2 + 1] = en ? (int16_t)dr : (int16_t)-1;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, en);
    if (en) {
      const int pos = n_en + __popc(m & ((1u << lane) - 1));
      s.ekey2[pos] = KT::make(dr, sr, c);
    }
    n_en += __popc(m);
  }
  __syncwarp();

#if defined(TNEAT_DIAG_TR_STOP) && TNEAT_DIAG_TR_STOP == 1  // diagnostic builds only: phase split
  return;
#endif
  // ---- counting sort by destination, then by source inside each bucket; CSR by
  // destination (in_start) and by source (su_start/succ) ------------------------
  for (int e = lane; e < n_en; e += 32) {
    const typename KT::E k = s.ekey2[e];
    atomicAdd(&s.indeg[KT::dst(k)], 1);
    atomicAdd(&s.outdeg[KT::src(k)], 1);
  }
  __syncwarp();
  warp_exclusive_scan(s.indeg, s.in_start, N);
  warp_exclusive_scan(s.outdeg, s.su_start, N);
  for (int r = lane; r < N; r += 32) { s.outdeg[r] = 0; s.lvl[r] = 0; }  // cursors
  __syncwarp();
  // two stable, order-preserving scatters (LSD radix by source, then by
  // destination): the edges start in connection-row order, so every
  // destination bucket ends up sorted by (source row, connection row)
  stable_scatter<KT>(s.ekey2, s.ekey, n_en, KT::SSH, s.su_start, s.outdeg, s.succ);
  stable_scatter<KT>(s.ekey, s.ekey2, n_en, KT::DSH, s.in_start, s.lvl, nullptr);
  for (int e = lane; e < n_en; e += 32) s.ekey[e] = s.ekey2[e];
  __syncwarp();
  int shadowed_any = 0;
  for (int r = lane; r < N; r += 32) {
    const int b0 = s.in_start[r], b1 = s.in_start[r + 1];
    // repeated enabled (src, dst) pairs: the reference's dense incoming keeps
    // the last connection row (inference.py:108-112); the earlier ones are
    // shadowed -- counted here, removed below
    int kept = 0;
    for (int i = b0; i < b1; ++i) {
      const bool shadow = i + 1 < b1 && KT::same_pair(s.ekey[i], s.ekey[i + 1]);
      if (shadow) {
        ++shadowed_any;
        if (conn_rows) conn_rows[(g * C + KT::row(s.ekey[i])) * 2 + 0] = -1,
                       conn_rows[(g * C + KT::row(s.ekey[i])) * 2 + 1] = -1;
      } else {
        ++kept;
      }
    }
    s.lvl[r] = kept;
  }
  shadowed_any = __reduce_add_sync(0xffffffffu, shadowed_any);
  __syncwarp();
  if (shadowed_any) {
    if (N <= 64) {
      // the reference's Kahn for N <= 64 decrements through successor bitmasks
      // (one per pair) while the indegree counts every connection: the
      // destination never becomes ready and the genome reads as cyclic
      for (int r = lane; r < N; r += 32) s.indeg[r] += (s.in_start[r + 1] - s.in_start[r]) - s.lvl[r];
    } else {
      // N > 64: the Kahn decrements per connection (no effect); the programs
      // see each pair once, with the last row's weight: compact the buckets
      // new bucket starts in outdeg (free between the CSR fill and the split
      // input counts), staging in ekey2 (free since the CSR fill)
      int carry = 0;
      for (int base = 0; base < N; base += 32) {
        const int r = base + lane;
        const int v = r < N ? s.lvl[r] : 0;
        int x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        if (r < N) s.outdeg[r] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      __syncwarp();
      for (int r = lane; r < N; r += 32) {
        int at = s.outdeg[r];
        for (int i = s.in_start[r]; i < s.in_start[r + 1]; ++i)
          if (!(i + 1 < s.in_start[r + 1] && KT::same_pair(s.ekey[i], s.ekey[i + 1]))) s.ekey2[at++] = s.ekey[i];
      }
      __syncwarp();
      for (int i = lane; i < carry; i += 32) s.ekey[i] = s.ekey2[i];
      for (int r = lane; r < N; r += 32) s.in_start[r] = (typename KT::Idx)s.outdeg[r];
      if (lane == 0) s.in_start[N] = (typename KT::Idx)carry;
    }
  }
  for (int r = lane; r < N; r += 32) s.lvl[r] = 0;
  __syncwarp();

#if defined(TNEAT_DIAG_TR_STOP) && TNEAT_DIAG_TR_STOP == 2  // diagnostic builds only: phase split
  return;
#endif
  // ---- io rows (the key table is dead from Kahn on: its memory is reused) ----
  // output rows park in the program's output-slot area; they become slots at the end
  uint8_t* gp = prog + g * L.stride;
  uint16_t* out_slot = (uint16_t*)(gp + L.off_out);
  for (int k = lane; k < io; k += 32) {
    const int r = lookup_row(s.skey, Npad, (uint64_t)k);
    if (r < 0) status |= ST_MISSING_IO;
    if (io_rows) io_rows[g * io + k] = r;
    if (k >= I) out_slot[k - I] = r >= 0 ? (uint16_t)r : NO_SLOT;
  }
  __syncwarp();

  // ---- Kahn, smallest ready row first (inference.py:127-141) + levels ---------
  const int W = (N + 31) / 32;
  for (int w = 0; w < W; ++w) {
    const int r = w * 32 + lane;
    const bool rdy = r < N && (s.flags[r] & F_LIVE) && s.indeg[r] == 0;
    const unsigned m = __ballot_sync(0xffffffffu, rdy);
    if (lane == 0) s.ready[w] = m;
  }
  __syncwarp();
  int n_order = 0, n_levels = 0;
  const bool exact_order = order_out != nullptr;
  if (exact_order) {
    // the reference's order: one node per step, smallest ready row first
    for (; n_order < n_live; ++n_order) {
      const int pick = warp_first_set(s.ready, W);
      if (pick < 0) break;
      __syncwarp();
      if (lane == 0) {
        s.ready[pick >> 5] &= ~(1u << (pick & 31));
        s.order[n_order] = (uint16_t)pick;
      }
      __syncwarp();
      const int nl = s.lvl[pick] + 1;
      const int e1 = s.su_start[pick + 1];
      for (int e = s.su_start[pick] + lane; e < e1; e += 32) {
        const int d = s.succ[e];
        atomicMax(&s.lvl[d], nl);
        if (atomicSub(&s.indeg[d], 1) == 1) atomicOr(&s.ready[d >> 5], 1u << (d & 31));
      }
      __syncwarp();
    }
  } else {
    // programs only need levels and cycle detection: level-synchronous Kahn,
    // the whole ready set per round (depth rounds instead of one per node).
    // s.order gets the nodes level by level; level k starts at last_grp[k].
    for (;;) {
      int cnt = 0;
      uint32_t bits = 0;
      for (int base = 0; base < W; base += 32) {  // compact the ready set into s.order
        const int w = base + lane;
        bits = w < W ? s.ready[w] : 0u;
        const int c = __popc(bits);
        int x = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        int at = n_order + cnt + x - c;
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          s.order[at++] = (uint16_t)(w * 32 + b);
        }
        if (w < W) s.ready[w] = 0u;
        cnt += __shfl_sync(0xffffffffu, x, 31);
      }
      if (cnt == 0) break;
      if (lane == 0) s.last_grp[n_levels] = n_order;
      __syncwarp();
      for (int i = n_order + lane; i < n_order + cnt; i += 32) {
        const int u = s.order[i];
        s.lvl[u] = n_levels;
        for (int e = s.su_start[u]; e < s.su_start[u + 1]; ++e) {
          const int d = s.succ[e];
          if (atomicSub(&s.indeg[d], 1) == 1) atomicOr(&s.ready[d >> 5], 1u << (d & 31));
        }
      }
      __syncwarp();
      n_order += cnt;
      ++n_levels;
    }
    if (lane == 0) s.last_grp[n_levels] = n_order;
    __syncwarp();
  }
  if (n_order < n_live) status |= ST_CYCLIC;

#if defined(TNEAT_DIAG_TR_STOP) && TNEAT_DIAG_TR_STOP == 3  // diagnostic builds only: phase split
  return;
#endif
  // ---- order / io rows outputs -----------------------------------------------
  if (order_out) {
    for (int i = lane; i < N; i += 32)
      order_out[g * N + i] = i < n_order ? (int16_t)s.order[i] : (int16_t)-1;
  }
  status = __reduce_or_sync(0xffffffffu, status);

  ProgHeader* hdr = (ProgHeader*)gp;
  if ((status & ~ST_CYCLIC) || ((status & ST_CYCLIC) && !recurrent)) {
    for (int o = lane; o < O; o += 32) out_slot[o] = NO_SLOT;
    if (lane == 0) {
      ProgHeader h{0, 0, I, n_order, status, n_live, mode, 0};
      *hdr = h;
      if (status_out) status_out[g] = status;
    }
    return;
  }

  // ---- which nodes matter (ancestor cone of the outputs) and which are read ----
  if (!recurrent && prune && !exact_order) {
    // levels in descending order; the nodes of one level are independent
    for (int r = lane; r < N; r += 32)
      if (s.flags[r] & F_OUTPUT) s.needed[r] = 1;
    __syncwarp();
    for (int lv = n_levels - 1; lv >= 1; --lv) {
      for (int i = s.last_grp[lv] + lane; i < s.last_grp[lv + 1]; i += 32) {
        const int r = s.order[i];
        if (!s.needed[r] || (s.flags[r] & F_INPUT)) continue;
        for (int e = s.in_start[r]; e < s.in_start[r + 1]; ++e) {
          const int sr = KT::src(s.ekey[e]);
          s.needed[sr] = 1;
          s.used[sr] = 1;
        }
      }
      __syncwarp();
    }
  } else if (!recurrent && prune) {
    for (int r = lane; r < N; r += 32)
      if (s.flags[r] & F_OUTPUT) s.needed[r] = 1;
    __syncwarp();
    for (int i = n_order - 1; i >= 0; --i) {
      const int r = s.order[i];
      if (!s.needed[r] || (s.flags[r] & F_INPUT)) continue;
      for (int e = s.in_start[r] + lane; e < s.in_start[r + 1]; e += 32) {
        const int sr = KT::src(s.ekey[e]);
        s.needed[sr] = 1;
        s.used[sr] = 1;
      }
      __syncwarp();
    }
  } else {
    for (int r = lane; r < N; r += 32) {
      s.needed[r] = (s.flags[r] & F_LIVE) ? 1 : 0;
      s.used[r] = (recurrent || s.su_start[r + 1] > s.su_start[r]) ? 1 : 0;
    }
  }
  __syncwarp();

  // ---- tensor-core program eligibility (FMT_TC) -------------------------------
  // every emitted step aggregates by sum / mean, at most 128 steps, and
  // every step's input-edge weights have a usable block exponent
  // (csrc/digits.cuh); the input count of each step goes to outdeg (free since
  // the CSR build)
  const int n_pos = recurrent ? N : n_order;
  bool tc_ok = tc && !recurrent && I <= TC_K;
  if (tc_ok) {
    int bad = 0, cnt_emit = 0;
    for (int base = 0; base < n_pos; base += 32) {
      const int i = base + lane;
      const int r = i < n_pos ? (int)s.order[i] : -1;
      const bool emit = r >= 0 && (s.flags[r] & F_LIVE) && !(s.flags[r] & F_INPUT) && s.needed[r];
      cnt_emit += __popc(__ballot_sync(0xffffffffu, emit));
      if (emit) {
        const double gv = gn[(int64_t)r * 5 + 3];
        if (!(gv == (double)AGG_SUM || gv == (double)AGG_MEAN)) bad = 1;
        // one pass, weights loaded 4 at a time: the input-weight maximum, and
        // the hidden-weight maximum / smallest nonzero magnitude
        double mw = 0.0, hmax = 0.0, hmin = INFINITY;
        int cin = 0;
        const int e1 = s.in_start[r + 1];
        for (int e = s.in_start[r]; e < e1; e += 4) {
          double w[4];
          bool inp[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const typename KT::E kk = s.ekey[e + u < e1 ? e + u : e];
            inp[u] = (s.flags[KT::src(kk)] & F_INPUT) != 0;
            w[u] = __ldg(gc + KT::row(kk) * 4 + 3);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (e + u >= e1) break;
            const double a = fabs(w[u]);
            if (inp[u]) {
              if (!isfinite(w[u])) bad = 1;
              mw = fmax(mw, a);
              ++cin;
            } else {
              hmax = fmax(hmax, a);  // NaN: fails the range test below through hmin
              if (a != 0.0) hmin = fmin(hmin, a);
              if (isnan(a)) bad = 1;
            }
          }
        }
        if (mw != 0.0 && (mw < 0x1p-62 || mw >= 0x1p63)) bad = 1;
        // the kernel folds the column factor cf = 2^(e - 12) into the step: hidden
        // weights / cf and response * cf must stay normal floats (the exponent is
        // kept in su_start, free for TC programs from here on)
        const int ewx = mw != 0.0 ? ilogb(mw) : 12;
        s.su_start[r] = (typename KT::Idx)ewx;
        const double up = ldexp(1.0, 12 - ewx), dn = ldexp(1.0, ewx - 12);
        if (!(hmax * up < 0x1p100)) bad = 1;
        if (hmin != INFINITY) {
          const double lo = hmin * up;
          if (lo != 0.0) {
            if (lo < 0x1p-100) bad = 1;
          } else {  // the smallest weight underflows (reads as 0): test each (rare)
            for (int e = s.in_start[r]; e < e1; ++e) {
              const typename KT::E kk = s.ekey[e];
              if (!(s.flags[KT::src(kk)] & F_INPUT)) {
                const double w = fabs(gc[KT::row(kk) * 4 + 3]) * up;
                if (w != 0.0 && w < 0x1p-100) bad = 1;
              }
            }
          }
        }
        const double rs = fabs(gn[(int64_t)r * 5 + 2]) * dn;
        if (!(rs < 0x1p100) || (rs != 0.0 && rs < 0x1p-100)) bad = 1;
        s.outdeg[r] = cin;
      }
    }
    tc_ok = !__any_sync(0xffffffffu, bad) && cnt_emit <= 128;  // 2 x 2 x round16(steps) TMEM columns <= 512
  }
  __syncwarp();

#if defined(TNEAT_DIAG_TR_STOP) && TNEAT_DIAG_TR_STOP == 4  // diagnostic builds only: phase split
  return;
#endif
  // ---- steps: emitted nodes sorted by (level, class, -count, position) --------
  // feed-forward: positions in the Kahn order; recurrent: rows (all nodes are
  // state, singleton groups, no slot recycling).  TC programs group by the
  // hidden-edge count (input edges go to the MMA).
  int n_emit = 0, bad = 0;
  for (int base = 0; base < n_pos; base += 32) {
    const int i = base + lane;
    int r = -1;
    if (i < n_pos) r = recurrent ? i : (int)s.order[i];
    const bool emit = r >= 0 && (s.flags[r] & F_LIVE) && !(s.flags[r] & F_INPUT) && s.needed[r];
    const unsigned me = __ballot_sync(0xffffffffu, emit);
    if (emit) {
      const double* nr = gn + (int64_t)r * 5;
      const double av = nr[4], gv = nr[3];
      if (!(av >= 0.0 && av < ACT_COUNT && av == floor(av))) bad |= ST_BAD_ACT;
      if (!(gv >= 0.0 && gv < AGG_COUNT && gv == floor(gv))) bad |= ST_BAD_AGG;
      const int agg = (gv >= 0.0 && gv < AGG_COUNT) ? (int)gv : 0;
      const uint32_t cls = (recurrent || !(agg == AGG_SUM || agg == AGG_MEAN)) ? 1 : 0;
      uint32_t cnt = (uint32_t)(s.in_start[r + 1] - s.in_start[r]);
      if (tc_ok) cnt -= (uint32_t)s.outdeg[r];
      const uint32_t lv = recurrent ? 0 : (uint32_t)s.lvl[r];
      s.gkey[n_emit + __popc(me & ((1u << lane) - 1))] = KT::gmake(lv, cls, cnt, (uint32_t)i);
    }
    n_emit += __popc(me);
  }
  status |= __reduce_or_sync(0xffffffffu, bad);
  const int Spad = next_pow2(n_emit);
  for (int i = n_emit + lane; i < Spad; i += 32) s.gkey[i] = KT::GMAX;
  __syncwarp();
  warp_bitonic_sort(s.gkey, Spad);

  // group formation (sequential, lane 0): same level & class, <= 4 steps, and
  // a step joins only if its list is at least half the group's longest list
  // (bounds the padded edge entries, see edge_capacity)
  if (lane == 0) {
    int ng = 0, e_total = 0;
    int cur_lv = -1, cur_cls = -1, cur_rounds = 0;
    const bool tc_join_all = tc_ok && 4ll * C + 8ll * N + 16 <= edge_capacity(N, C);
    // a sum group of 3 whose first list is the longest gives the spare column
    // to the second half of that list (GRP_SPLIT0; standard fp32 and fp64
    // programs).  TC programs never split: a step's hidden sum then runs in
    // list order whatever group it lands in, so programs whose groupings
    // differ (pruned or not, exact order or level-synchronous) agree bitwise
    auto close = [&](GroupRec& gr) {
      if (gr.n == 3 && !(gr.cls & GRP_GENERIC) && !recurrent && !tc_ok) {
        const int c0 = gr.cnt[0], h = (c0 + 1) / 2;
        const int r = h > gr.cnt[1] ? h : gr.cnt[1];
        if (r < gr.rounds) {
          gr.cls |= GRP_SPLIT0;
          gr.cnt[0] = (uint16_t)h;
          gr.cnt[3] = (uint16_t)(c0 - h);
          gr.rounds = (uint16_t)r;
        }
      }
      e_total = (int)align_up(e_total + group_width(gr.n) * gr.rounds, 8);
    };
    for (int k = 0; k < n_emit; ++k) {
      const typename KT::G key = s.gkey[k];
      const int pos = KT::gpos(key);
      const int row = recurrent ? pos : (int)s.order[pos];
      const int cnt = KT::gcnt(key);
      const int cls = KT::gcls(key);
      const int lv = KT::glv(key);
      // TC programs (hidden edges only, short lists) group every same-level step
      // when the padded entries (<= 4x real) still fit the edge capacity:
      // fewer groups, less per-group work in the sweep (measured 3.35 -> 3.32 ms)
      const bool join = ng > 0 && lv == cur_lv && cls == cur_cls && cls == 0 && s.grp[ng - 1].n < 4 &&
                        (tc_join_all || TNEAT_JOIN_DEN * cnt >= TNEAT_JOIN_NUM * cur_rounds);
      if (!join) {
        if (ng > 0) close(s.grp[ng - 1]);
        GroupRec gr;
        memset(&gr, 0, sizeof(gr));
        // holes (shorter lists in a sum/mean group) read the zero slot
        gr.cls = (uint8_t)cls; gr.rounds = (uint16_t)cnt;
        gr.e_begin = (uint16_t)e_total; gr.step_begin = (uint16_t)k;
        s.grp[ng++] = gr;
        cur_lv = lv; cur_cls = cls; cur_rounds = cnt;
      }
      GroupRec& gr = s.grp[ng - 1];
      gr.cnt[gr.n] = (uint16_t)cnt;
      const bool tanh_sum = (s.flags[row] & F_TANH_SUM) != 0;
      if (gr.n == 0) gr.cls |= tanh_sum ? GRP_TANH_SUM : 0;
      else if (!tanh_sum) gr.cls &= ~GRP_TANH_SUM;
      gr.n++;
      s.step_row[k] = (uint16_t)row;
      s.grp_of[k] = (uint16_t)(ng - 1);
    }
    if (ng > 0) close(s.grp[ng - 1]);
    s.ready[0] = (uint32_t)ng;  // Kahn is done: ready/indeg serve as scalar mailboxes
    s.indeg[0] = e_total;
  }
  __syncwarp();
  const int n_groups = (int)s.ready[0];
  const int e_total = s.indeg[0];

  int n_slots;
  uint16_t scratch_slot = NO_SLOT;
  uint32_t zero_slot;
  if (tc_ok) {
    // TC programs: one slot per step (the MMA epilogue writes every step's input
    // partial before the sweep), slot = step index, zero slot = n_steps
    for (int k = lane; k < n_emit; k += 32) s.slot_of[s.step_row[k]] = (uint16_t)k;
    zero_slot = (uint32_t)n_emit;
    n_slots = n_emit + 1;
    __syncwarp();
  } else {
    // ---- liveness: last group reading each node -------------------------------
    for (int r = lane; r < N; r += 32)
      s.last_grp[r] = (recurrent || (s.flags[r] & F_OUTPUT)) ? NEVER : -1;
    __syncwarp();
    if (!recurrent) {
      for (int k = lane; k < n_emit; k += 32) {
        const int row = s.step_row[k];
        const int gk = s.grp_of[k];
        for (int e = s.in_start[row]; e < s.in_start[row + 1]; ++e)
          atomicMax(&s.last_grp[KT::src(s.ekey[e])], gk);
      }
    }
    // slots: 0..I-1 hold the inputs, the rest start free; one more slot after
    // the last allocated one is the zero slot read by padding entries
    const int WS = (N + 2 + 31) / 32;
    for (int w = lane; w < WS; w += 32) {
      uint32_t m = 0;
      for (int b = 0; b < 32; ++b) {
        const int sl = w * 32 + b;
        if (sl >= I && sl < N + 2) m |= 1u << b;
      }
      s.freemask[w] = m;
    }
    for (int r = lane; r < N; r += 32)
      if (s.flags[r] & F_INPUT) s.slot_of[r] = (uint16_t)gn[(int64_t)r * 5];
    __syncwarp();
    n_slots = I;
    for (int gi = 0; gi < n_groups; ++gi) {
      // recycle the slots whose last reader is this group (reads precede writes)
      if (!recurrent) {
        for (int r = lane; r < N; r += 32) {
          const uint16_t sl = s.slot_of[r];
          if (sl != NO_SLOT && !(s.flags[r] & (F_OUTPUT | F_FREED)) && s.last_grp[r] <= gi) {
            s.flags[r] |= F_FREED;
            atomicOr(&s.freemask[sl >> 5], 1u << (sl & 31));
          }
        }
        __syncwarp();
      }
      const int gn_steps = s.grp[gi].n;
      const int g_begin = s.grp[gi].step_begin;
      for (int j = 0; j < gn_steps; ++j) {
        const int row = s.step_row[g_begin + j];
        if (!(s.used[row] || (s.flags[row] & F_OUTPUT))) continue;
        const int sl = warp_first_set(s.freemask, WS);
        __syncwarp();
        if (lane == 0) {
          s.freemask[sl >> 5] &= ~(1u << (sl & 31));
          s.slot_of[row] = (uint16_t)sl;
        }
        n_slots = max(n_slots, sl + 1);
        __syncwarp();
      }
    }
    // steps whose value nobody reads (unpruned programs) write a scratch slot:
    // every step has a slot, so kernels store step results unconditionally
    bool orphan = false;
    for (int k = lane; k < n_emit; k += 32) {
      const int row = s.step_row[k];
      orphan |= !(s.used[row] || (s.flags[row] & F_OUTPUT));
    }
    orphan = __any_sync(0xffffffffu, orphan);
    scratch_slot = orphan ? (uint16_t)n_slots : NO_SLOT;
    if (orphan) n_slots += 1;
    zero_slot = (uint32_t)n_slots;
    n_slots += 1;
  }

  // TC programs: input-edge list starts (exclusive scan of the input counts in
  // step order; lvl / last_grp are free now)
  if (tc_ok) {
    for (int k = lane; k < n_emit; k += 32) s.lvl[k] = s.outdeg[s.step_row[k]];
    __syncwarp();
    warp_exclusive_scan(s.lvl, s.last_grp, n_emit);
    uint16_t* in_start = (uint16_t*)(gp + L.off_in);
    for (int k = lane; k <= n_emit; k += 32) in_start[k] = (uint16_t)s.last_grp[k];
  }

#if defined(TNEAT_DIAG_TR_STOP) && TNEAT_DIAG_TR_STOP == 5  // diagnostic builds only: phase split
  return;
#endif
  // ---- write groups, steps and interleaved edge lists --------------------------
  // (TC programs: into the staged block, common.cuh tc_block)
  const TcBlock tb = tc_block(n_emit, n_groups, e_total);
  uint8_t* const blk = gp + L.off_tc;
  StepT<T>* steps = (StepT<T>*)(tc_ok ? blk + tb.st : gp + L.off_steps);
  GroupRec* pg = (GroupRec*)(tc_ok ? blk + tb.gr : gp + L.off_groups);
  for (int gi = lane; gi < n_groups; gi += 32) {
    if (tc_ok) {
      const GroupRec r = s.grp[gi];
      GroupTC t;
      t.code = (uint32_t)(r.n - 1) | ((r.cls & GRP_TANH_SUM) ? 4u : 0u) | ((r.cls & GRP_SPLIT0) ? 8u : 0u);
      t.rounds = r.rounds;
      t.e_begin = r.e_begin;
      t.step_begin = r.step_begin;
      ((GroupTC*)pg)[gi] = t;
    } else {
      pg[gi] = s.grp[gi];
    }
  }
  for (int k = lane; k < n_emit; k += 32) {
    const int row = s.step_row[k];
    const GroupRec gr = s.grp[s.grp_of[k]];
    const int j = k - gr.step_begin, gw = group_width(gr.n);
    const double* nr = gn + (int64_t)row * 5;
    const double av = nr[4], gv = nr[3];
    StepT<T> st;
    memset(&st, 0, sizeof(st));
    const int e0 = s.in_start[row], cnt = s.in_start[row + 1] - e0;
    st.slot = tc_ok ? (uint16_t)k : ((s.used[row] || (s.flags[row] & F_OUTPUT)) ? s.slot_of[row] : scratch_slot);
    st.act = (uint8_t)((av >= 0.0 && av < ACT_COUNT) ? (int)av : 0);
    st.agg = (uint8_t)((gv >= 0.0 && gv < AGG_COUNT) ? (int)gv : 0);
    st.count = (uint16_t)cnt;
    st.bias = (T)nr[1];
    st.resp = (T)nr[2];
    if (tc_ok) {
      // TC programs: the step's accumulator runs divided by its column factor
      // cf = 2^(e - 12) (the MMA epilogue then skips one multiply per step), so
      // the response carries cf; tanh groups also pre-scale by -2 log2(e)
      // (common.cuh GroupTC).  Powers of two: bit-identical results.
      const double cfk = ldexp(1.0, s.su_start[row] - 12);
      const double kk = (gr.cls & GRP_TANH_SUM) ? (double)TANH_K : 1.0;
      st.bias = (T)(nr[1] * kk);
      st.resp = (T)(nr[2] * cfk * kk);
    }
    steps[k] = st;
    // column j of the group's edge block; holes (and the spare column of a
    // 3-group) are (zero slot, 0.0) entries; GRP_SPLIT0: step 0's list goes
    // to columns 0 (first cnt[0] edges) and 3 (the rest)
    const bool split0 = (gr.cls & GRP_SPLIT0) != 0;
    if constexpr (sizeof(T) == 4) {
      if (tc_ok) {
        // hidden edges into the interleaved block (sources as byte offsets of
        // the kernel's slot rows), input edges into the (input index, weight)
        // list of the exact path and the B operand row
        uint32_t* esrc = (uint32_t*)(blk + tb.src);
        float* ew = (float*)(blk + tb.w);
        const int ncol = (gr.n == 3 && j == 2 && !split0) || (split0 && j == 0) ? 2 : 1;
        for (int ci = 0; ci < ncol; ++ci) {
          const int col = ci == 0 ? j : 3;
          for (int rr = 0; rr < gr.rounds; ++rr) {
            esrc[gr.e_begin + rr * gw + col] = zero_slot * TC_SLOT_BYTES;
            ew[gr.e_begin + rr * gw + col] = 0.0f;
          }
        }
        uint16_t* isrc = (uint16_t*)(gp + L.off_isrc);
        float* iw = (float*)(gp + L.off_iw);
        uint8_t* brow = blk + tb.b;
        const int ewx = s.su_start[row];
        const double sc = ldexp(1.0, 27 - ewx), up = ldexp(1.0, 12 - ewx);
        ((float*)(blk + tb.cf))[k] = pow2f(12 - ewx);  // 1 / cf (the exact path's partials)
#pragma unroll 1
        for (int q = 0; q < 12; ++q) *(uint4*)(brow + tc_offset(k, 8 * q)) = make_uint4(0, 0, 0, 0);
        int hc = 0, ic = s.last_grp[k];
        const int c0 = gr.cnt[0], e1 = e0 + cnt;
        // edges 4 at a time: their weight (and input index) loads are in flight
        // together; identity io rows (io_fast) need no index load at all
        for (int e = e0; e < e1; e += 4) {
          double w[4];
          int sr[4], idx[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const typename KT::E kk = s.ekey[e + u < e1 ? e + u : e];
            sr[u] = KT::src(kk);
            w[u] = __ldg(gc + KT::row(kk) * 4 + 3);
            idx[u] = io_fast ? sr[u] : (int)__ldg(gn + (int64_t)sr[u] * 5);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (e + u >= e1) break;
            if (s.flags[sr[u]] & F_INPUT) {
              isrc[ic] = (uint16_t)idx[u];
              iw[ic] = (float)w[u];
              ++ic;
              double d2, d1, d0;
              digits3_d(w[u] * sc, d2, d1, d0);
              *(__half*)(brow + tc_offset(k, idx[u])) = __double2half(d2);
              *(__half*)(brow + tc_offset(k, TC_K + idx[u])) = __double2half(d1);
              *(__half*)(brow + tc_offset(k, 2 * TC_K + idx[u])) = __double2half(d0);
            } else {
              int col = j, rr = hc;
              if (split0 && j == 0 && hc >= c0) { col = 3; rr = hc - c0; }
              esrc[gr.e_begin + rr * gw + col] = (uint32_t)s.slot_of[sr[u]] * TC_SLOT_BYTES;
              ew[gr.e_begin + rr * gw + col] = (float)(w[u] * up);
              ++hc;
            }
          }
        }
        continue;
      }
    }
    int cols[2] = {j, 3}, first[2] = {0, 0}, nedge[2] = {cnt, 0};
    int ncol = (gr.n == 3 && j == 2 && !split0) ? 2 : 1;
    if (split0 && j == 0) {
      ncol = 2;
      first[1] = gr.cnt[0];
      nedge[0] = gr.cnt[0];
      nedge[1] = cnt - gr.cnt[0];
    }
    for (int ci = 0; ci < ncol; ++ci) {
      const int col = cols[ci];
      // rounds in batches of 4: the weight loads of a batch are in flight together
      for (int rr0 = 0; rr0 < gr.rounds; rr0 += 4) {
        uint32_t src[4];
        double w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = rr0 + u;
          src[u] = zero_slot;
          w[u] = 0.0;
          if (rr < nedge[ci]) {
            const typename KT::E kk = s.ekey[e0 + first[ci] + rr];
            src[u] = s.slot_of[KT::src(kk)];
            w[u] = gc[KT::row(kk) * 4 + 3];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = rr0 + u;
          if (rr >= gr.rounds) break;
          const int idx = gr.e_begin + rr * gw + col;
          if (sizeof(T) == 8) {
            EdgeD ed;
            ed.src = src[u]; ed.pad = 0; ed.w = w[u];
            ((EdgeD*)(gp + L.off_w))[idx] = ed;
          } else {
            ((uint16_t*)(gp + L.off_src))[idx] = (uint16_t)src[u];
            ((float*)(gp + L.off_w))[idx] = (float)w[u];
          }
        }
      }
    }
  }
  if (tc_ok) {  // B rows past the last step up to the MMA's N (multiple of 16) are zero
    uint8_t* bp = blk + tb.b;
    float* cf = (float*)(blk + tb.cf);
    for (int k = n_emit + lane; k < tc_rows(n_emit); k += 32) cf[k] = 0.0f;
    for (int k = n_emit + lane; k < tc_rows(n_emit); k += 32)
      for (int q = 0; q < 12; ++q) *(uint4*)(bp + tc_offset(k, 8 * q)) = make_uint4(0, 0, 0, 0);
  }
  for (int k = lane; k < io; k += 32) {  // output rows -> slots (the lane that parked them)
    if (k < I) continue;
    const uint16_t r = out_slot[k - I];
    out_slot[k - I] = r != NO_SLOT ? s.slot_of[r] : NO_SLOT;
  }
  TNEAT_DCHECK(e_total <= edge_capacity(N, C), "program edge entries within capacity", e_total, edge_capacity(N, C));
  TNEAT_DCHECK(!tc_ok || L.off_tc + tb.bytes <= L.off_in, "tc block within its area", tb.bytes, L.off_in - L.off_tc);
  TNEAT_DCHECK(!tc_ok || n_emit <= 128, "tc steps", n_emit, 128);
  TNEAT_DCHECK(tc_ok || n_slots <= N + 2, "standard value slots", n_slots, N + 2);
  if (lane == 0) {
    ProgHeader h{n_emit, e_total, n_slots, n_order, status, n_live, tc_ok ? (int)MODE_TC : mode, n_groups};
    *hdr = h;
    if (status_out) status_out[g] = status;
    atomicMax(&maxdims[0], n_slots);
    atomicMax(&maxdims[1], n_emit);
    atomicMax(&maxdims[2], e_total);
  }
}

}  // namespace tneat

using namespace tneat;

extern "C" {

// Bytes of one genome's program (header + output slots + groups + steps + edges).
int64_t an_program_stride(int N, int C, int O, int precision) {
  return prog_layout(N, C, O, precision).stride;
}

// Replaces inference.transform_arrays (inference.py:82-147).  See include/tneat.h.
int an_transform(const double* nodes, const double* conns, int64_t P, int N, int C, int I, int O,
                 int mode, int precision, int prune, void* program, int64_t program_stride,
                 int16_t* order, int16_t* conn_rows, int32_t* io_rows, int32_t* status,
                 int32_t* maxdims, void* stream) {
  const bool tc = (precision & FMT_TC) != 0;
  if (P < 0 || N < 1 || N > 32767 || C < 0 || I < 1 || O < 1 || I + O > N) return -1;
  if (edge_capacity(N, C) > 65535) return -1;
  if (tc && ((precision & FMT_F64) || mode != 0)) return -1;  // TC programs: fp32 feed-forward only
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (program_stride != L.stride) return -3;
  if (P == 0) return 0;  // empty population: nothing to read or write
  if (!nodes || !program || !maxdims || (C > 0 && !conns)) return -2;
  const int Cc = C > 0 ? C : 1;
  const int64_t ws = warp_smem_bytes(N, Cc, I);
  if (ws > 200 * 1024) return -4;  // genome capacity too large for one warp's shared memory
  int wpb = TNEAT_TR_WPB;
  while (wpb > 1 && ws * wpb > 160 * 1024) wpb >>= 1;
  const int64_t smem = ws * wpb;
  const int64_t blocks = (P + wpb - 1) / wpb;
  cudaStream_t st = (cudaStream_t)stream;
  auto launch = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel<<<(unsigned)blocks, 32 * wpb, smem, st>>>(nodes, conns, P, N, C, I, O, mode, prune, tc, ws,
                                                     (uint8_t*)program, L, order, conn_rows, io_rows, status,
                                                     maxdims);
  };
  const bool small = small_keys(N, Cc);
  if (precision & FMT_F64) {
    if (small) launch(transform_kernel<double, true>);
    else launch(transform_kernel<double, false>);
  } else {
    if (small) launch(transform_kernel<float, true>);
    else launch(transform_kernel<float, false>);
  }
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
