// K0/K3/K4/K5/K6: population initialisation, compatibility distance,
// crossover, mutation and the fused reproduce step, one warp per genome.
//
// Replaces (reference evolution.py / genome.py):
//   init_arrays       genome.py:129-160           -> an_init
//   distance_arrays   evolution.py:425-488        -> an_distance
//   _crossover_into   evolution.py:101-136        -> an_crossover  (and inside an_reproduce)
//   mutate_arrays     evolution.py:172-325,       -> an_mutate     (and inside an_reproduce)
//   _add_connections  evolution.py:328-407
//   reproduce (work)  evolution.py:685-709        -> an_reproduce
//
// All randomness is drawn from the counter-based streams of rng.cuh at the
// tape positions the reference uses, so uniforms -- and
// therefore every structural decision -- are bit-exact; fp64 attribute math
// is written with explicit _rn intrinsics (and this file is built with
// -fmad=false) so it rounds exactly like numpy; only Box-Muller normals can
// differ from numpy's SIMD log/cos by ~1 ulp.
// Genomes stay in the reference layout: nodes (N,5), conns (C,4) float64,
// NaN padding rows.

#include "common.cuh"
#include "rng.cuh"

namespace tneat {

struct MutateParams {  // mirrors include/tneat.h an_mutate_params
  int32_t N, C, I, O;
  int32_t feedforward;
  int32_t act_default, agg_default;
  int32_t n_act_options, n_agg_options;
  int32_t act_options[8];
  int32_t agg_options[8];
  int32_t pad;
  double node_add, node_delete, conn_add, conn_delete;
  double bias_init_mean, bias_init_std, bias_mutate_power, bias_mutate_rate, bias_replace_rate;
  double response_init_mean, response_init_std, response_mutate_power, response_mutate_rate,
      response_replace_rate;
  double weight_init_mean, weight_init_std, weight_mutate_power, weight_mutate_rate, weight_replace_rate;
  double enabled_mutate_rate, activation_replace_rate, aggregation_replace_rate;
  double attr_min, attr_max;
};

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double nanv() { return __longlong_as_double(0x7ff8000000000000ll); }
__device__ __forceinline__ bool is_nan(double x) { return x != x; }

// k = min(int(u * count), max(count - 1, 0))   (evolution.py:90-91)
__device__ __forceinline__ int kth_index(double u, int count) {
  const long long k = (long long)__dmul_rn(u, (double)count);
  return (int)min(k, (long long)max(count - 1, 0));
}

// Row of the (k+1)-th row (ascending) satisfying pred, or -1.  Warp-uniform result.
template <typename Pred>
__device__ int warp_kth_row(int rows, int k, Pred pred) {
  const int lane = threadIdx.x & 31;
  int seen = 0;
  for (int base = 0; base < rows; base += 32) {
    const int r = base + lane;
    const unsigned m = __ballot_sync(FULL, r < rows && pred(r));
    const int c = __popc(m);
    if (k < seen + c) {
      unsigned mm = m;
      for (int j = 0; j < k - seen; ++j) mm &= mm - 1;
      return base + __ffs(mm) - 1;
    }
    seen += c;
  }
  return -1;
}

template <typename Pred>
__device__ int warp_count(int rows, Pred pred) {
  const int lane = threadIdx.x & 31;
  int n = 0;
  for (int base = 0; base < rows; base += 32) {
    const int r = base + lane;
    n += __popc(__ballot_sync(FULL, r < rows && pred(r)));
  }
  return n;
}

// ---------------------------------------------------------------------------
// crossover (evolution.py:101-136): child already holds the fitter parent
// ---------------------------------------------------------------------------

__device__ void warp_crossover(double* cn, double* cc, const double* __restrict__ ln,
                               const double* __restrict__ lc, int N, int C, uint64_t key,
                               uint64_t base) {
  const int lane = threadIdx.x & 31;
  for (int r = lane; r < N; r += 32) {
    const double k = cn[r * 5];
    if (is_nan(k)) continue;
    int o = -1;
    if (ln[r * 5] == k) o = r;  // same-row fast path (search.py:83-100)
    else
      for (int q = 0; q < N; ++q)
        if (ln[q * 5] == k) { o = q; break; }
    if (o < 0) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a)
      if (rng_uniform(key, base + (uint64_t)r * 4 + a) < 0.5) cn[r * 5 + 1 + a] = ln[o * 5 + 1 + a];
  }
  const uint64_t cbase = base + 4ull * N;
  for (int r = lane; r < C; r += 32) {
    const double i = cc[r * 4], j = cc[r * 4 + 1];
    if (is_nan(i)) continue;
    int o = -1;
    if (lc[r * 4] == i && lc[r * 4 + 1] == j) o = r;
    else
      for (int q = 0; q < C; ++q)
        if (lc[q * 4] == i && lc[q * 4 + 1] == j) { o = q; break; }
    if (o < 0) continue;
#pragma unroll
    for (int a = 0; a < 2; ++a)
      if (rng_uniform(key, cbase + (uint64_t)r * 2 + a) < 0.5) cc[r * 4 + 2 + a] = lc[o * 4 + 2 + a];
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// mutation (evolution.py:172-325)
// ---------------------------------------------------------------------------

struct WarpScratch {  // per-warp shared memory for the connection-addition closure
  uint16_t* live_rows;  // [N] live node rows in row order (rank -> row)
  int16_t* rank_of;     // [N] row -> rank, -1 if not live
  uint32_t* exists;     // [N * W] exists[u] bit v : live conn u -> v
  uint32_t* pred;       // [N * W] closure of exists^T (pred[v] bit u : u reaches v)
  uint32_t* dst_ok;     // [W]     rank v is a valid destination (live, not an input)
  uint32_t* src_ok;     // [W]     rank u is a valid source (live, not an output)
};

__host__ __device__ inline int64_t mutate_scratch_bytes(int N) {
  const int W = (N + 31) / 32;
  return align_up(2ll * N, 4) + align_up(2ll * N, 4) + 8ll * N * W + 8ll * W;
}

__device__ WarpScratch carve_scratch(uint8_t* base, int N) {
  const int W = (N + 31) / 32;
  WarpScratch s;
  s.live_rows = (uint16_t*)base;
  s.rank_of = (int16_t*)(base + align_up(2ll * N, 4));
  s.exists = (uint32_t*)(base + 2 * align_up(2ll * N, 4));
  s.pred = s.exists + (int64_t)N * W;
  s.dst_ok = s.pred + (int64_t)N * W;
  s.src_ok = s.dst_ok + W;
  return s;
}

__device__ void warp_add_connection(double* cn, double* cc, const MutateParams& p, double u_pick,
                                    double z_weight, WarpScratch& s) {
  const int lane = threadIdx.x & 31;
  const int N = p.N, C = p.C, W = (N + 31) / 32;
  const int n_io = p.I + p.O;
  // live-node ranks in row order (evolution.py:339-355)
  int m = 0;
  for (int base = 0; base < N; base += 32) {
    const int r = base + lane;
    const bool live = r < N && !is_nan(cn[r * 5]);
    const unsigned msk = __ballot_sync(FULL, live);
    if (r < N) s.rank_of[r] = live ? (int16_t)(m + __popc(msk & ((1u << lane) - 1))) : (int16_t)-1;
    if (live) s.live_rows[m + __popc(msk & ((1u << lane) - 1))] = (uint16_t)r;
    m += __popc(msk);
  }
  for (int i = lane; i < N * W; i += 32) { s.exists[i] = 0; s.pred[i] = 0; }
  __syncwarp();
  // exists over LIVE conns, disabled included (evolution.py:357-361)
  for (int r = lane; r < C; r += 32) {
    const double ik = cc[r * 4];
    if (is_nan(ik)) continue;
    const double ok = cc[r * 4 + 1];
    int ur = -1, vr = -1;
    for (int q = 0; q < N; ++q) {  // endpoint key -> row
      const double kq = cn[q * 5];
      if (kq == ik) ur = q;
      if (kq == ok) vr = q;
    }
    if (ur < 0 || vr < 0) continue;
    const int u = s.rank_of[ur], v = s.rank_of[vr];
    atomicOr(&s.exists[u * W + (v >> 5)], 1u << (v & 31));
    atomicOr(&s.pred[v * W + (u >> 5)], 1u << (u & 31));
  }
  __syncwarp();
  const bool ff = p.feedforward != 0;
  if (ff) {
    // reflexive-transitive closure of the predecessor relation (Warshall on bitsets):
    // pred[v] bit u  <=>  u reaches v over live conns (u == v included)
    for (int v = lane; v < m; v += 32) s.pred[v * W + (v >> 5)] |= 1u << (v & 31);
    __syncwarp();
    for (int k = 0; k < m; ++k) {
      for (int v = lane; v < m; v += 32) {
        if (s.pred[v * W + (k >> 5)] >> (k & 31) & 1u)
          for (int w = 0; w < W; ++w) s.pred[v * W + w] |= s.pred[k * W + w];
      }
      __syncwarp();
    }
  }
  // allowed[u][v] = valid & !exists & src not output & dst not input & !(v reaches u)
  // (evolution.py:363-391); count, then the k-th allowed cell row-major
  for (int base = 0; base < W * 32; base += 32) {
    const int v = base + lane;
    double kv = -1.0;
    if (v < m) kv = cn[s.live_rows[v] * 5];
    const unsigned dok = __ballot_sync(FULL, v < m && kv >= (double)p.I);
    const unsigned sok = __ballot_sync(FULL, v < m && !(kv >= (double)p.I && kv < (double)n_io));
    if (lane == 0) { s.dst_ok[base >> 5] = dok; s.src_ok[base >> 5] = sok; }
  }
  __syncwarp();
  auto allowed_word = [&](int u, int w) -> uint32_t {
    if (!(s.src_ok[u >> 5] >> (u & 31) & 1u)) return 0u;
    uint32_t m32 = s.dst_ok[w] & ~s.exists[u * W + w];
    if (ff) m32 &= ~s.pred[u * W + w];
    return m32;
  };
  int total = 0;
  for (int u = lane; u < m; u += 32)
    for (int w = 0; w < W; ++w) total += __popc(allowed_word(u, w));
  total = __reduce_add_sync(FULL, total);
  if (total == 0) return;
  const int k = kth_index(u_pick, total);
  // locate row u holding the k-th cell: per-row counts in rank order
  int seen = 0, pick_u = -1, pick_v = -1;
  for (int base = 0; base < m && pick_u < 0; base += 32) {
    const int u = base + lane;
    int cnt = 0;
    if (u < m)
      for (int w = 0; w < W; ++w) cnt += __popc(allowed_word(u, w));
    int x = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(FULL, x, d);
      if (lane >= d) x += y;
    }
    const int incl = seen + x, excl = incl - cnt;
    const unsigned hit = __ballot_sync(FULL, u < m && k >= excl && k < incl);
    if (hit) {
      const int src = __ffs(hit) - 1;
      pick_u = base + src;
      int rem = __shfl_sync(FULL, k - excl, src);
      for (int w = 0; w < W; ++w) {
        uint32_t aw = allowed_word(pick_u, w);
        const int c = __popc(aw);
        if (rem < c) {
          for (int j = 0; j < rem; ++j) aw &= aw - 1;
          pick_v = w * 32 + __ffs(aw) - 1;
          break;
        }
        rem -= c;
      }
    }
    seen += __shfl_sync(FULL, x, 31);
  }
  const int free_row = warp_kth_row(C, 0, [&](int r) { return is_nan(cc[r * 4]); });
  if (lane == 0 && free_row >= 0) {
    double* row = cc + free_row * 4;
    row[0] = cn[s.live_rows[pick_u] * 5];
    row[1] = cn[s.live_rows[pick_v] * 5];
    row[2] = 1.0;
    row[3] = __dadd_rn(p.weight_init_mean, __dmul_rn(p.weight_init_std, z_weight));
  }
  __syncwarp();
}

// one perturbed attribute column (evolution.py:268-293); returns the new counter
__device__ uint64_t warp_perturb(double* t, int stride, int col, int width, bool node_rows, uint64_t key,
                                 uint64_t ctr, double replace_rate, double mutate_rate, double power,
                                 double mean, double std, double lo, double hi) {
  if (replace_rate == 0.0 && mutate_rate == 0.0) return ctr;
  const int lane = threadIdx.x & 31;
  const uint64_t b_rep = ctr, b_mut = ctr + width;
  ctr += 2ull * width;
  const uint64_t b_noise = ctr;
  if (mutate_rate > 0.0) ctr += 2ull * width;
  const uint64_t b_fresh = ctr;
  if (replace_rate > 0.0) ctr += 2ull * width;
  for (int r = lane; r < width; r += 32) {
    if (is_nan(t[r * stride + (node_rows ? 0 : 0)])) continue;  // column 0 is the key / in_key
    const double u_rep = rng_uniform(key, b_rep + r);
    const double u_mut = rng_uniform(key, b_mut + r);
    const bool replaced = u_rep < replace_rate;
    const bool mutated = mutate_rate > 0.0 && !replaced && u_mut < mutate_rate;
    const double old = t[r * stride + col];
    double v = old;
    if (mutated) v = __dadd_rn(old, __dmul_rn(power, rng_normal_cell(key, b_noise, width, r)));
    if (replaced) v = __dadd_rn(mean, __dmul_rn(std, rng_normal_cell(key, b_fresh, width, r)));
    if (replaced || mutated) t[r * stride + col] = fmin(fmax(v, lo), hi);
  }
  __syncwarp();
  return ctr;
}

// mutate one genome in place; counters start at `base` (the child's tape
// position after the crossover coins).  Returns whether node addition fired.
__device__ bool warp_mutate(double* cn, double* cc, const MutateParams& p, uint64_t key, uint64_t base,
                            double new_key, WarpScratch& s) {
  const int lane = threadIdx.x & 31;
  const int N = p.N, C = p.C, n_io = p.I + p.O;
  double u_struct[4], u_pick[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    u_struct[i] = rng_uniform(key, base + i);
    u_pick[i] = rng_uniform(key, base + 4 + i);
  }
  const double z_new_bias = rng_normal_cell(key, base + 8, 1, 0);
  const double z_new_weight = rng_normal_cell(key, base + 10, 1, 0);
  uint64_t ctr = base + 12;
  bool can_add = false;

  // (1) node addition: split the k-th enabled conn (evolution.py:196-228)
  if (u_struct[0] < p.node_add) {
    auto enabled = [&](int r) { return !is_nan(cc[r * 4]) && cc[r * 4 + 2] == 1.0; };
    const int cnt = warp_count(C, enabled);
    const int split = cnt > 0 ? warp_kth_row(C, kth_index(u_pick[0], cnt), enabled) : -1;
    const int node_slot = warp_kth_row(N, 0, [&](int r) { return is_nan(cn[r * 5]); });
    auto free_c = [&](int r) { return is_nan(cc[r * 4]); };
    const int f1 = warp_kth_row(C, 0, free_c), f2 = warp_kth_row(C, 1, free_c);
    if (split >= 0 && node_slot >= 0 && f2 >= 0) {
      can_add = true;
      if (lane == 0) {
        const double src_key = cc[split * 4], dst_key = cc[split * 4 + 1], w = cc[split * 4 + 3];
        cc[split * 4 + 2] = 0.0;
        double* nr = cn + node_slot * 5;
        nr[0] = new_key;
        nr[1] = __dadd_rn(p.bias_init_mean, __dmul_rn(p.bias_init_std, z_new_bias));
        nr[2] = p.response_init_mean;
        nr[3] = (double)p.agg_default;
        nr[4] = (double)p.act_default;
        double* a = cc + f1 * 4;
        a[0] = src_key; a[1] = new_key; a[2] = 1.0; a[3] = 1.0;
        double* b = cc + f2 * 4;
        b[0] = new_key; b[1] = dst_key; b[2] = 1.0; b[3] = w;
      }
      __syncwarp();
    }
  }
  // (2) node deletion of the k-th hidden node, cascading (evolution.py:230-244)
  if (u_struct[1] < p.node_delete) {
    auto hidden = [&](int r) { const double k = cn[r * 5]; return !is_nan(k) && k >= (double)n_io; };
    const int cnt = warp_count(N, hidden);
    if (cnt > 0) {
      const int row = warp_kth_row(N, kth_index(u_pick[1], cnt), hidden);
      const double dk = cn[row * 5];
      __syncwarp();
      if (lane == 0)
        for (int c = 0; c < 5; ++c) cn[row * 5 + c] = nanv();
      for (int r = lane; r < C; r += 32)
        if (cc[r * 4] == dk || cc[r * 4 + 1] == dk)
          for (int c = 0; c < 4; ++c) cc[r * 4 + c] = nanv();
      __syncwarp();
    }
  }
  // (3) connection addition (evolution.py:246-253, 328-407)
  if (u_struct[2] < p.conn_add) {
    const int any_free = warp_count(C, [&](int r) { return is_nan(cc[r * 4]); });
    if (any_free > 0) warp_add_connection(cn, cc, p, u_pick[2], z_new_weight, s);
  }
  // (4) connection deletion of the k-th live conn (evolution.py:255-262)
  if (u_struct[3] < p.conn_delete) {
    auto live = [&](int r) { return !is_nan(cc[r * 4]); };
    const int cnt = warp_count(C, live);
    if (cnt > 0) {
      const int row = warp_kth_row(C, kth_index(u_pick[3], cnt), live);
      __syncwarp();
      if (lane == 0)
        for (int c = 0; c < 4; ++c) cc[row * 4 + c] = nanv();
      __syncwarp();
    }
  }
  // (5) attribute perturbation over live genes (evolution.py:264-303)
  ctr = warp_perturb(cn, 5, 1, N, true, key, ctr, p.bias_replace_rate, p.bias_mutate_rate,
                     p.bias_mutate_power, p.bias_init_mean, p.bias_init_std, p.attr_min, p.attr_max);
  ctr = warp_perturb(cn, 5, 2, N, true, key, ctr, p.response_replace_rate, p.response_mutate_rate,
                     p.response_mutate_power, p.response_init_mean, p.response_init_std, p.attr_min,
                     p.attr_max);
  ctr = warp_perturb(cc, 4, 3, C, false, key, ctr, p.weight_replace_rate, p.weight_mutate_rate,
                     p.weight_mutate_power, p.weight_init_mean, p.weight_init_std, p.attr_min, p.attr_max);
  // (6) enabled flips (evolution.py:305-309)
  if (p.enabled_mutate_rate > 0.0) {
    for (int r = lane; r < C; r += 32)
      if (!is_nan(cc[r * 4]) && rng_uniform(key, ctr + r) < p.enabled_mutate_rate)
        cc[r * 4 + 2] = __dsub_rn(1.0, cc[r * 4 + 2]);
    ctr += C;
    __syncwarp();
  }
  // (7, 8) categorical replacement (evolution.py:311-323)
  for (int which = 0; which < 2; ++which) {
    const double rate = which == 0 ? p.activation_replace_rate : p.aggregation_replace_rate;
    if (rate == 0.0) continue;
    const int nopt = which == 0 ? p.n_act_options : p.n_agg_options;
    const int* opts = which == 0 ? p.act_options : p.agg_options;
    const int col = which == 0 ? 4 : 3;
    for (int r = lane; r < N; r += 32) {
      if (is_nan(cn[r * 5])) continue;
      if (rng_uniform(key, ctr + r) < rate) {
        const long long idx = min((long long)__dmul_rn(rng_uniform(key, ctr + N + r), (double)nopt),
                                  (long long)(nopt - 1));
        cn[r * 5 + col] = (double)opts[idx];
      }
    }
    ctr += 2ull * N;
    __syncwarp();
  }
  return can_add;
}

__device__ __forceinline__ void warp_copy_genome(double* dn, double* dc, const double* sn, const double* sc,
                                                 int N, int C) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < N * 5; i += 32) dn[i] = sn[i];
  for (int i = lane; i < C * 4; i += 32) dc[i] = sc[i];
  __syncwarp();
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

// 48 registers (10 blocks of 128 threads per SM instead of 8): the warp per child
// waits on global loads, more resident warps beat the small spill (-17 %)
__global__ void __launch_bounds__(128, 10) reproduce_kernel(const double* __restrict__ pn, const double* __restrict__ pc,
                                 double* __restrict__ on, double* __restrict__ oc, int64_t n_slots,
                                 int64_t slot_base, const int32_t* __restrict__ pool,
                                 const int32_t* __restrict__ pool_offset, const int32_t* __restrict__ pool_size,
                                 const int32_t* __restrict__ elite_src, uint64_t stage_key, double new_key_base,
                                 MutateParams p, uint8_t* __restrict__ can_add, int64_t scratch) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= n_slots) return;
  const int N = p.N, C = p.C;
  const int64_t slot = slot_base + i;
  const uint64_t key = rng_fold(stage_key, (uint64_t)slot);
  // parent picks: uniforms(2) (evolution.py:687-696)
  const int size = pool_size[i], off = pool_offset[i];
  const int a = off + (int)min((long long)__dmul_rn(rng_uniform(key, 0), (double)size), (long long)(size - 1));
  const int b = off + (int)min((long long)__dmul_rn(rng_uniform(key, 1), (double)size), (long long)(size - 1));
  const int64_t fit = pool[min(a, b)], less = pool[max(a, b)];
  double* cn = on + i * (int64_t)N * 5;
  double* cc = oc + i * (int64_t)C * 4;
  warp_copy_genome(cn, cc, pn + fit * N * 5, pc + fit * C * 4, N, C);
  warp_crossover(cn, cc, pn + less * N * 5, pc + less * C * 4, N, C, key, 2);
  WarpScratch s = carve_scratch(smem + warp * scratch, N);
  const bool added = warp_mutate(cn, cc, p, key, 2 + 4ull * N + 2ull * C,
                                 __dadd_rn(new_key_base, (double)slot), s);
  if (lane == 0 && can_add) can_add[i] = added ? 1 : 0;
  const int e = elite_src[i];
  if (e >= 0) warp_copy_genome(cn, cc, pn + (int64_t)e * N * 5, pc + (int64_t)e * C * 4, N, C);
}

__global__ void mutate_kernel(double* __restrict__ n, double* __restrict__ c, int64_t P,
                              const uint64_t* __restrict__ keys, uint64_t base,
                              const double* __restrict__ new_keys, MutateParams p, uint8_t* __restrict__ can_add,
                              int64_t scratch) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= P) return;
  WarpScratch s = carve_scratch(smem + warp * scratch, p.N);
  const bool added = warp_mutate(n + i * (int64_t)p.N * 5, c + i * (int64_t)p.C * 4, p, keys[i], base,
                                 new_keys[i], s);
  if (lane == 0 && can_add) can_add[i] = added ? 1 : 0;
}

__global__ void crossover_kernel(double* __restrict__ n, double* __restrict__ c, const double* __restrict__ ln,
                                 const double* __restrict__ lc, int64_t P, int N, int C,
                                 const uint64_t* __restrict__ keys, uint64_t base) {
  const int warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= P) return;
  warp_crossover(n + i * (int64_t)N * 5, c + i * (int64_t)C * 4, ln + i * (int64_t)N * 5,
                 lc + i * (int64_t)C * 4, N, C, keys[i], base);
}

// init_arrays (genome.py:129-160): genome g draws from stream keys[g];
// bias = normals(N) at counter base, response = normals(N) at base+2N,
// weight = normals(C) at base+4N
__global__ void init_kernel(double* __restrict__ n, double* __restrict__ c, int64_t P,
                            const uint64_t* __restrict__ keys, uint64_t cbase, MutateParams p) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int N = p.N, C = p.C, io = p.I + p.O;
  const int64_t per = (int64_t)N + C;
  if (t >= P * per) return;
  const int64_t g = t / per;
  const int r = (int)(t - g * per);
  const uint64_t key = keys[g];
  if (r < N) {
    double* row = n + (g * N + r) * 5;
    if (r < io) {
      row[0] = (double)r;
      row[1] = __dadd_rn(p.bias_init_mean, __dmul_rn(p.bias_init_std, rng_normal_cell(key, cbase, N, r)));
      row[2] = __dadd_rn(p.response_init_mean,
                         __dmul_rn(p.response_init_std, rng_normal_cell(key, cbase + 2ull * N, N, r)));
      row[3] = (double)p.agg_default;
      row[4] = (double)p.act_default;
    } else {
      for (int k = 0; k < 5; ++k) row[k] = nanv();
    }
  } else {
    const int q = r - N;
    double* row = c + (g * C + q) * 4;
    if (q < p.I * p.O) {
      row[0] = (double)(q / p.O);
      row[1] = (double)(p.I + q % p.O);
      row[2] = 1.0;
      row[3] = __dadd_rn(p.weight_init_mean, __dmul_rn(p.weight_init_std, rng_normal_cell(key, cbase + 4ull * N, C, q)));
    } else {
      for (int k = 0; k < 4; ++k) row[k] = nanv();
    }
  }
}

// distance_arrays (evolution.py:425-488).  Warp per (genome p, other q); the
// homologous-gene terms are computed lane-parallel and then summed by one
// lane in genome-1 row order (nodes, then conns), as np.bincount does.
__global__ void distance_kernel(const double* __restrict__ n1, const double* __restrict__ c1, int64_t P,
                                const double* __restrict__ n2, const double* __restrict__ c2, int64_t Q,
                                int pair_mode, int N, int C, double cd, double ch, double* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t q = pair_mode ? (Q == 1 ? 0 : p) : blockIdx.y;
  if (p >= P) return;
  double* term = reinterpret_cast<double*>(smem) + (int64_t)warp * (N + C);
  const double* a = n1 + p * N * 5;
  const double* ac = c1 + p * C * 4;
  const double* b = n2 + q * N * 5;
  const double* bc = c2 + q * C * 4;
  int live1 = 0, live2 = 0, hom_n = 0, clive1 = 0, clive2 = 0, hom_c = 0;
  for (int r = lane; r < N; r += 32) {
    const double k = a[r * 5];
    live2 += is_nan(b[r * 5]) ? 0 : 1;
    double t = nanv();
    if (!is_nan(k)) {
      ++live1;
      int o = -1;
      if (b[r * 5] == k) o = r;
      else
        for (int s = 0; s < N; ++s)
          if (b[s * 5] == k) { o = s; break; }
      if (o >= 0) {
        ++hom_n;
        const double* x = a + r * 5;
        const double* y = b + o * 5;
        double v = __dadd_rn(fabs(__dsub_rn(x[1], y[1])), fabs(__dsub_rn(x[2], y[2])));
        v = __dadd_rn(v, x[3] != y[3] ? 1.0 : 0.0);
        v = __dadd_rn(v, x[4] != y[4] ? 1.0 : 0.0);
        t = __ddiv_rn(v, 4.0);
      }
    }
    term[r] = t;
  }
  for (int r = lane; r < C; r += 32) {
    const double i = ac[r * 4], j = ac[r * 4 + 1];
    clive2 += is_nan(bc[r * 4]) ? 0 : 1;
    double t = nanv();
    if (!is_nan(i)) {
      ++clive1;
      int o = -1;
      if (bc[r * 4] == i && bc[r * 4 + 1] == j) o = r;
      else
        for (int s = 0; s < C; ++s)
          if (bc[s * 4] == i && bc[s * 4 + 1] == j) { o = s; break; }
      if (o >= 0) {
        ++hom_c;
        const double* x = ac + r * 4;
        const double* y = bc + o * 4;
        t = __ddiv_rn(__dadd_rn(fabs(__dsub_rn(x[3], y[3])), fabs(__dsub_rn(x[2], y[2]))), 2.0);
      }
    }
    term[N + r] = t;
  }
  live1 = __reduce_add_sync(FULL, live1);
  live2 = __reduce_add_sync(FULL, live2);
  hom_n = __reduce_add_sync(FULL, hom_n);
  clive1 = __reduce_add_sync(FULL, clive1);
  clive2 = __reduce_add_sync(FULL, clive2);
  hom_c = __reduce_add_sync(FULL, hom_c);
  __syncwarp();
  if (lane == 0) {
    double ns = 0.0, cs = 0.0;
    for (int r = 0; r < N; ++r)
      if (!is_nan(term[r])) ns = __dadd_rn(ns, term[r]);
    for (int r = 0; r < C; ++r)
      if (!is_nan(term[N + r])) cs = __dadd_rn(cs, term[N + r]);
    const int node_dis = (live1 - hom_n) + (live2 - hom_n);
    const int conn_dis = (clive1 - hom_c) + (clive2 - hom_c);
    const int dis = node_dis + conn_dis, hom = hom_n + hom_c;
    const double attr = hom > 0 ? __ddiv_rn(__dadd_rn(ns, cs), (double)hom) : 0.0;
    const int total = max(live1 + clive1, live2 + clive2);
    const double d = __dadd_rn(__ddiv_rn(__dmul_rn(cd, (double)dis), (double)total), __dmul_rn(ch, attr));
    out[q * (pair_mode ? 0 : P) + p] = d;
  }
}

// Distance of every genome against a small set of representatives (speciate:
// pair_mode 0, R reps x P genomes; founding rounds: pair_mode 1, Q == 1).
// Persistent CTAs stage the Q representatives and their key -> row maps in
// shared memory once, then one thread per (genome, representative) pair walks
// genome 1's rows in order: the homologous terms are summed as they are found,
// which is the reference's row order (np.bincount), so the result is bitwise
// the warp kernel's.  Homolog lookup: same row first, else a binary search in
// the representative's sorted (key bits, row) map -- the smallest matching row,
// as the reference's first-match scan.  Keys compare as doubles: -0 is mapped
// to +0 and NaN rows never match.
__device__ __forceinline__ uint64_t key_bits(double k) { return (uint64_t)__double_as_longlong(k == 0.0 ? 0.0 : k); }

struct RepSmem {
  double* nodes;    // [Q][N*5]
  double* conns;    // [Q][C*4]
  uint64_t* nkey;   // [Q][N] sorted node key bits (NaN rows: U64 max, last)
  uint16_t* nrow;   // [Q][N]
  uint64_t* ckin;   // [Q][C] sorted (in, out) key bits
  uint64_t* ckout;
  uint16_t* crow;
  int* live;        // [Q][2] live nodes, live conns
};

__host__ __device__ inline int64_t rep_smem_bytes(int Q, int N, int C, RepSmem* s, uint8_t* base) {
  int64_t o = 0;
  auto take = [&](int64_t bytes, int64_t al) { o = (o + al - 1) / al * al; const int64_t at = o; o += bytes; return at; };
  const int64_t a_n = take(8ll * Q * N * 5, 16), a_c = take(8ll * Q * C * 4, 16);
  const int64_t a_nk = take(8ll * Q * N, 8), a_ck = take(8ll * Q * C, 8), a_co = take(8ll * Q * C, 8);
  const int64_t a_nr = take(2ll * Q * N, 2), a_cr = take(2ll * Q * C, 2), a_l = take(8ll * Q, 4);
  if (s) {
    s->nodes = (double*)(base + a_n); s->conns = (double*)(base + a_c);
    s->nkey = (uint64_t*)(base + a_nk); s->ckin = (uint64_t*)(base + a_ck); s->ckout = (uint64_t*)(base + a_co);
    s->nrow = (uint16_t*)(base + a_nr); s->crow = (uint16_t*)(base + a_cr); s->live = (int*)(base + a_l);
  }
  return (o + 15) / 16 * 16;
}

__global__ void distance_reps_kernel(const double* __restrict__ n1, const double* __restrict__ c1, int64_t P,
                                     const double* __restrict__ n2, const double* __restrict__ c2, int Q, int N,
                                     int C, double cd, double ch, double* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  RepSmem s;
  rep_smem_bytes(Q, N, C, &s, smem);
  const int tid = threadIdx.x, nt = blockDim.x;
  // stage the representatives (coalesced) and build their maps by ranking:
  // entry i goes to position #{j : (key_j, j) < (key_i, i)} (keys unique up to
  // NaN / duplicates; ties broken by row, smallest first)
  for (int64_t i = tid; i < (int64_t)Q * N * 5; i += nt) s.nodes[i] = n2[i];
  for (int64_t i = tid; i < (int64_t)Q * C * 4; i += nt) s.conns[i] = c2[i];
  __syncthreads();
  for (int i = tid; i < Q * N; i += nt) {
    const int q = i / N, r = i - q * N;
    const double* rows = s.nodes + (int64_t)q * N * 5;
    const double k = rows[r * 5];
    const uint64_t kb = is_nan(k) ? ~0ull : key_bits(k);
    int rank = 0;
    for (int j = 0; j < N; ++j) {
      const double kj = rows[j * 5];
      const uint64_t b = is_nan(kj) ? ~0ull : key_bits(kj);
      rank += (b < kb || (b == kb && j < r)) ? 1 : 0;
    }
    s.nkey[q * N + rank] = kb;
    s.nrow[q * N + rank] = (uint16_t)r;
  }
  for (int i = tid; i < Q * C; i += nt) {
    const int q = i / C, r = i - q * C;
    const double* rows = s.conns + (int64_t)q * C * 4;
    const double a = rows[r * 4], b = rows[r * 4 + 1];
    const bool dead = is_nan(a) || is_nan(b);
    const uint64_t ka = dead ? ~0ull : key_bits(a), kb = dead ? ~0ull : key_bits(b);
    int rank = 0;
    for (int j = 0; j < C; ++j) {
      const double aj = rows[j * 4], bj = rows[j * 4 + 1];
      const bool dj = is_nan(aj) || is_nan(bj);
      const uint64_t xa = dj ? ~0ull : key_bits(aj), xb = dj ? ~0ull : key_bits(bj);
      rank += (xa < ka || (xa == ka && (xb < kb || (xb == kb && j < r)))) ? 1 : 0;
    }
    s.ckin[q * C + rank] = ka;
    s.ckout[q * C + rank] = kb;
    s.crow[q * C + rank] = (uint16_t)r;
  }
  for (int q = tid; q < Q; q += nt) {
    int ln = 0, lc = 0;
    for (int r = 0; r < N; ++r) ln += is_nan(s.nodes[(int64_t)q * N * 5 + r * 5]) ? 0 : 1;
    for (int r = 0; r < C; ++r) lc += is_nan(s.conns[(int64_t)q * C * 4 + r * 4]) ? 0 : 1;
    s.live[2 * q] = ln;
    s.live[2 * q + 1] = lc;
  }
  __syncthreads();

  const int gpb = nt / Q;  // genomes per CTA pass
  if (tid >= gpb * Q) return;
  const int q = tid % Q, gl = tid / Q;
  const double* b = s.nodes + (int64_t)q * N * 5;
  const double* bc = s.conns + (int64_t)q * C * 4;
  const uint64_t* nk = s.nkey + (int64_t)q * N;
  const uint16_t* nr = s.nrow + (int64_t)q * N;
  const uint64_t* ki = s.ckin + (int64_t)q * C;
  const uint64_t* ko = s.ckout + (int64_t)q * C;
  const uint16_t* cr = s.crow + (int64_t)q * C;
  for (int64_t p = (int64_t)blockIdx.x * gpb + gl; p < P; p += (int64_t)gridDim.x * gpb) {
    const double* a = n1 + p * N * 5;
    const double* ac = c1 + p * C * 4;
    int live1 = 0, hom_n = 0, clive1 = 0, hom_c = 0;
    double ns = 0.0, cs = 0.0;
    // rows in batches of 4, every load of a batch issued before its rows are
    // processed (memory-level parallelism for the per-thread row walk)
    for (int r0 = 0; r0 < N; r0 += 4) {
      double x[20];
#pragma unroll
      for (int u = 0; u < 20; ++u) x[u] = r0 * 5 + u < N * 5 ? __ldg(a + r0 * 5 + u) : nanv();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u;
        const double k = x[u * 5];
        if (r >= N || is_nan(k)) continue;
        ++live1;
        int o = -1;
        if (b[r * 5] == k) {
          o = r;
        } else {
          const uint64_t kb = key_bits(k);
          int lo = 0, hi = N;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (nk[mid] < kb) lo = mid + 1; else hi = mid;
          }
          if (lo < N && nk[lo] == kb) o = nr[lo];
        }
        if (o >= 0) {
          ++hom_n;
          const double* y = b + o * 5;
          double v = __dadd_rn(fabs(__dsub_rn(x[u * 5 + 1], y[1])), fabs(__dsub_rn(x[u * 5 + 2], y[2])));
          v = __dadd_rn(v, x[u * 5 + 3] != y[3] ? 1.0 : 0.0);
          v = __dadd_rn(v, x[u * 5 + 4] != y[4] ? 1.0 : 0.0);
          const double t = __ddiv_rn(v, 4.0);
          if (!is_nan(t)) ns = __dadd_rn(ns, t);
        }
      }
    }
    for (int r0 = 0; r0 < C; r0 += 4) {
      double x[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) x[u] = r0 * 4 + u < C * 4 ? __ldg(ac + r0 * 4 + u) : nanv();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u;
        const double i = x[u * 4], j = x[u * 4 + 1];
        if (r >= C || is_nan(i)) continue;
        ++clive1;
        int o = -1;
        if (bc[r * 4] == i && bc[r * 4 + 1] == j) {
          o = r;
        } else if (!is_nan(j)) {
          const uint64_t ka = key_bits(i), kb = key_bits(j);
          int lo = 0, hi = C;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ki[mid] < ka || (ki[mid] == ka && ko[mid] < kb)) lo = mid + 1; else hi = mid;
          }
          if (lo < C && ki[lo] == ka && ko[lo] == kb) o = cr[lo];
        }
        if (o >= 0) {
          ++hom_c;
          const double* y = bc + o * 4;
          const double t = __ddiv_rn(__dadd_rn(fabs(__dsub_rn(x[u * 4 + 3], y[3])), fabs(__dsub_rn(x[u * 4 + 2], y[2]))), 2.0);
          if (!is_nan(t)) cs = __dadd_rn(cs, t);
        }
      }
    }
    const int live2 = s.live[2 * q], clive2 = s.live[2 * q + 1];
    const int node_dis = (live1 - hom_n) + (live2 - hom_n);
    const int conn_dis = (clive1 - hom_c) + (clive2 - hom_c);
    const int dis = node_dis + conn_dis, hom = hom_n + hom_c;
    const double attr = hom > 0 ? __ddiv_rn(__dadd_rn(ns, cs), (double)hom) : 0.0;
    const int total = max(live1 + clive1, live2 + clive2);
    out[(int64_t)q * P + p] = __dadd_rn(__ddiv_rn(__dmul_rn(cd, (double)dis), (double)total), __dmul_rn(ch, attr));
  }
}

__global__ void rng_draw_kernel(const uint64_t* __restrict__ keys, int64_t S, uint64_t base, int64_t width,
                                int normals, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S * width) return;
  const int64_t s = t / width;
  const int64_t col = t - s * width;
  out[t] = normals ? rng_normal_cell(keys[s], base, (uint64_t)width, (uint64_t)col)
                   : rng_uniform(keys[s], base + (uint64_t)col);
}

inline int warps_per_block(int64_t scratch) {
  int w = 4;
  while (w > 1 && scratch * w > 96 * 1024) w >>= 1;
  return w;
}

}  // namespace tneat

using namespace tneat;

extern "C" {

// Tape cells of a batch of streams: out[s, j] = uniform (or normal) cell
// base + j of stream keys[s] (rng.py:92-134).  Test hook.
int an_rng_draw(const uint64_t* keys, int64_t S, uint64_t base, int64_t width, int normals, double* out,
                void* stream) {
  if (S < 0 || width < 0) return -1;
  if (S * width == 0) return 0;
  const int64_t n = S * width;
  rng_draw_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(keys, S, base, width, normals,
                                                                                   out);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

// init_arrays (genome.py:129-160): genome g draws from stream keys[g] at counter base.
int an_init(double* nodes, double* conns, int64_t P, const uint64_t* keys, uint64_t base,
            const MutateParams* params, void* stream) {
  if (!params || P < 0) return -1;
  if (P == 0) return 0;
  const int64_t n = P * ((int64_t)params->N + params->C);
  init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nodes, conns, P, keys, base,
                                                                            *params);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

// distance_arrays (evolution.py:425-488).  pair_mode 1: out[p] = d(g1[p], g2[Q==1 ? 0 : p]);
// pair_mode 0: out[q, p] = d(g1[p], g2[q]) for all p < P, q < Q.
int an_distance(const double* n1, const double* c1, int64_t P, const double* n2, const double* c2, int64_t Q,
                int pair_mode, int N, int C, double c_disjoint, double c_homologous, double* out, void* stream) {
  if (P < 0 || Q < 1 || N < 1 || C < 0) return -1;
  if (pair_mode && Q != 1 && Q != P) return -1;
  if (P == 0) return 0;
  // P genomes against a few representatives: representatives staged once per
  // persistent CTA (when they fit in shared memory)
  // (in launches of as many representatives as fit in 110 KB)
  // (small launches keep the warp-per-pair kernel: thread-per-pair work only
  // fills the GPU from ~64K pairs on)
  if ((!pair_mode || Q == 1) && P * Q >= 65536 && N < 65536 && C < 65536) {
    int64_t qc = Q < 256 ? Q : 256;
    while (qc > 1 && rep_smem_bytes((int)qc, N, C, nullptr, nullptr) > 110 * 1024) --qc;
    if (rep_smem_bytes((int)qc, N, C, nullptr, nullptr) <= 110 * 1024) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int nt = 256;
      for (int64_t q0 = 0; q0 < Q; q0 += qc) {
        const int qn = (int)(Q - q0 < qc ? Q - q0 : qc);
        const int64_t rs = rep_smem_bytes(qn, N, C, nullptr, nullptr);
        const int gpb = nt / qn;
        const int64_t tiles = (P + gpb - 1) / gpb;
        int64_t per_sm = (228ll * 1024) / (rs + 1024);
        per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
        const int64_t grid = tiles < (int64_t)sms * per_sm ? tiles : (int64_t)sms * per_sm;
        cudaFuncSetAttribute(distance_reps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs);
        distance_reps_kernel<<<(unsigned)grid, nt, rs, (cudaStream_t)stream>>>(
            n1, c1, P, n2 + q0 * N * 5, c2 + q0 * C * 4, qn, N, C, c_disjoint, c_homologous, out + q0 * P);
        TNEAT_CHECK_LAUNCH();
      }
      return 0;
    }
  }
  const int64_t per = 8ll * (N + C);
  int wpb = 4;
  while (wpb > 1 && per * wpb > 96 * 1024) wpb >>= 1;
  if (per > 200 * 1024) return -4;
  dim3 grid((unsigned)((P + wpb - 1) / wpb), pair_mode ? 1u : (unsigned)Q);
  cudaFuncSetAttribute(distance_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per * wpb));
  distance_kernel<<<grid, 32 * wpb, per * wpb, (cudaStream_t)stream>>>(n1, c1, P, n2, c2, Q, pair_mode, N, C,
                                                                       c_disjoint, c_homologous, out);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

// mutate_arrays (evolution.py:172-325) in place; keys[i] = stream key of genome
// i, counters start at `base`; new_keys[i] = the key a firing node addition uses.
int an_mutate(double* nodes, double* conns, int64_t P, const uint64_t* keys, uint64_t base,
              const double* new_keys, const MutateParams* params, uint8_t* can_add, void* stream) {
  if (!params || P < 0 || params->N > 1024) return -1;
  if (P == 0) return 0;
  const int64_t scratch = align_up(mutate_scratch_bytes(params->N), 16);
  const int wpb = warps_per_block(scratch);
  cudaFuncSetAttribute(mutate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(scratch * wpb));
  mutate_kernel<<<(unsigned)((P + wpb - 1) / wpb), 32 * wpb, scratch * wpb, (cudaStream_t)stream>>>(
      nodes, conns, P, keys, base, new_keys, *params, can_add, scratch);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

// _crossover_into (evolution.py:101-136): out genomes (already holding the
// fitter parents) blend attributes of the less-fit parents; coins from cells
// base.. of keys[i].
int an_crossover(double* out_nodes, double* out_conns, const double* less_nodes, const double* less_conns,
                 int64_t P, int N, int C, const uint64_t* keys, uint64_t base, void* stream) {
  if (P < 0 || N < 1 || C < 0) return -1;
  if (P == 0) return 0;
  crossover_kernel<<<(unsigned)((P + 3) / 4), 128, 0, (cudaStream_t)stream>>>(out_nodes, out_conns, less_nodes,
                                                                              less_conns, P, N, C, keys, base);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

// reproduce (evolution.py:685-709) for slots slot_base .. slot_base+n_slots-1:
// parent picks, crossover, mutation, elite overwrite; stream of slot s =
// fold(stage_key, s); node addition in slot s uses key new_key_base + s.
int an_reproduce(const double* pop_nodes, const double* pop_conns, double* out_nodes, double* out_conns,
                 int64_t n_slots, int64_t slot_base, const int32_t* pool, const int32_t* pool_offset,
                 const int32_t* pool_size, const int32_t* elite_src, uint64_t stage_key, double new_key_base,
                 const MutateParams* params, uint8_t* can_add, void* stream) {
  if (!params || n_slots < 0 || params->N > 1024) return -1;
  if (n_slots == 0) return 0;
  const int64_t scratch = align_up(mutate_scratch_bytes(params->N), 16);
  const int wpb = warps_per_block(scratch);
  cudaFuncSetAttribute(reproduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(scratch * wpb));
  reproduce_kernel<<<(unsigned)((n_slots + wpb - 1) / wpb), 32 * wpb, scratch * wpb, (cudaStream_t)stream>>>(
      pop_nodes, pop_conns, out_nodes, out_conns, n_slots, slot_base, pool, pool_offset, pool_size, elite_src,
      stage_key, new_key_base, *params, can_add, scratch);
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
