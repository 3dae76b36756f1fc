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
// the kernel emits a per-destination CSR (the non-NaN entries of each
// incoming row, in source-row order) inside the genome's program instead.

#include "common.cuh"

namespace tneat {

constexpr uint64_t U64_MAX = ~0ull;

struct WarpSmem {
  uint64_t* skey;    // [Npad]   (key << 16 | row), sorted
  uint64_t* ekey;    // [Cpad]   (dst << 48 | src << 32 | conn_row), sorted
  int32_t* indeg;    // [N]
  int32_t* outdeg;   // [N]
  int32_t* in_start; // [N+1]
  int32_t* su_start; // [N+1]
  uint16_t* succ;    // [C]
  uint16_t* order;   // [N]
  uint16_t* slot_of; // [N]
  uint8_t* flags;    // [N]  bit0 live, bit1 input, bit2 output
  uint8_t* needed;   // [N]
  uint8_t* used;     // [N]
  uint32_t* ready;   // [W]
};

__host__ __device__ inline int next_pow2(int x) {
  int p = 32;
  while (p < x) p <<= 1;
  return p;
}

__host__ __device__ inline int64_t warp_smem_bytes(int N, int C) {
  const int Npad = next_pow2(N), Cpad = next_pow2(C);
  const int W = (N + 31) / 32;
  int64_t b = 0;
  b += 8ll * Npad + 8ll * Cpad;
  b += 4ll * N * 2 + 4ll * (N + 1) * 2;
  b = align_up(b, 8);
  b += 2ll * C + 2ll * N * 2;
  b = align_up(b, 4);
  b += 3ll * N;
  b = align_up(b, 4);
  b += 4ll * W;
  return align_up(b, 16);
}

__device__ inline WarpSmem carve(uint8_t* base, int N, int C) {
  const int Npad = next_pow2(N), Cpad = next_pow2(C);
  WarpSmem s;
  uint8_t* p = base;
  s.skey = (uint64_t*)p; p += 8ll * Npad;
  s.ekey = (uint64_t*)p; p += 8ll * Cpad;
  s.indeg = (int32_t*)p; p += 4ll * N;
  s.outdeg = (int32_t*)p; p += 4ll * N;
  s.in_start = (int32_t*)p; p += 4ll * (N + 1);
  s.su_start = (int32_t*)p; p += 4ll * (N + 1);
  p = base + align_up(p - base, 8);
  s.succ = (uint16_t*)p; p += 2ll * C;
  s.order = (uint16_t*)p; p += 2ll * N;
  s.slot_of = (uint16_t*)p; p += 2ll * N;
  p = base + align_up(p - base, 4);
  s.flags = p; p += N;
  s.needed = p; p += N;
  s.used = p; p += N;
  p = base + align_up(p - base, 4);
  s.ready = (uint32_t*)p;
  return s;
}

// ascending bitonic sort of n (power of two, >= 32) u64 values, one warp
__device__ void warp_bitonic_sort(uint64_t* a, int n) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < n; i += 32) {
        const int l = i ^ j;
        if (l > i) {
          const uint64_t x = a[i], y = a[l];
          const bool up = (i & k) == 0;
          if ((x > y) == up) { a[i] = y; a[l] = x; }
        }
      }
      __syncwarp();
    }
  }
}

// exclusive scan of cnt[0..n) into out[0..n]; out[n] = total. One warp.
__device__ void warp_exclusive_scan(const int32_t* cnt, int32_t* out, int n) {
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
    if (i < n) out[i] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) out[n] = carry;
  __syncwarp();
}

// row of `key` among the sorted live (key<<16|row) pairs, or -1
__device__ inline int lookup_row(const uint64_t* skey, int Npad, uint64_t key) {
  int lo = 0, hi = Npad;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((skey[mid] >> 16) < key) lo = mid + 1; else hi = mid;
  }
  if (lo < Npad && skey[lo] != U64_MAX && (skey[lo] >> 16) == key) return (int)(skey[lo] & 0xFFFF);
  return -1;
}

__device__ inline bool key_ok(double k) {
  return k >= 0.0 && k < 140737488355328.0 /* 2^47 */ && k == floor(k);
}

template <typename T>
__global__ void transform_kernel(const double* __restrict__ nodes, const double* __restrict__ conns,
                                 int64_t P, int N, int C, int I, int O, int mode, int prune,
                                 int64_t wsmem, uint8_t* __restrict__ prog, ProgLayout L,
                                 int16_t* __restrict__ order_out, int16_t* __restrict__ conn_rows,
                                 int32_t* __restrict__ io_rows, int32_t* __restrict__ status_out,
                                 int32_t* __restrict__ maxdims) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= P) return;
  WarpSmem s = carve(smem + warp * wsmem, N, C);
  const int Npad = next_pow2(N);
  const double* gn = nodes + g * (int64_t)N * 5;
  const double* gc = conns + g * (int64_t)C * 4;
  const int io = I + O;
  int status = 0;

  // ---- nodes: live mask, key table ------------------------------------------
  int n_live = 0;
  for (int r = lane; r < Npad; r += 32) {
    uint64_t packed = U64_MAX;
    uint8_t f = 0;
    if (r < N) {
      const double k = gn[(int64_t)r * 5];
      if (!isnan(k)) {
        if (!key_ok(k)) status |= ST_BAD_KEY;
        const uint64_t ki = (uint64_t)k;
        packed = (ki << 16) | (uint64_t)r;
        f = 1 | (ki < (uint64_t)I ? 2 : 0) | (ki >= (uint64_t)I && ki < (uint64_t)io ? 4 : 0);
        ++n_live;
      }
      s.flags[r] = f;
      s.needed[r] = 0;
      s.used[r] = 0;
      s.indeg[r] = 0;
      s.outdeg[r] = 0;
      s.slot_of[r] = NO_SLOT;
    }
    s.skey[r] = packed;
  }
  n_live = __reduce_add_sync(0xffffffffu, n_live);
  __syncwarp();
  warp_bitonic_sort(s.skey, Npad);

  // ---- conns: endpoint rows, enabled mask, compacted edge keys ----------------
  int n_en = 0;
  for (int base = 0; base < C; base += 32) {
    const int c = base + lane;
    bool en = false;
    int sr = -1, dr = -1;
    if (c < C) {
      const double ik = gc[(int64_t)c * 4 + 0];
      if (!isnan(ik)) {
        const double ok = gc[(int64_t)c * 4 + 1];
        if (!key_ok(ik) || !key_ok(ok)) {
          status |= ST_BAD_KEY;
        } else {
          sr = lookup_row(s.skey, Npad, (uint64_t)ik);
          dr = lookup_row(s.skey, Npad, (uint64_t)ok);
          if (sr < 0 || dr < 0) status |= ST_DANGLING;
          else en = gc[(int64_t)c * 4 + 2] == 1.0;
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
      s.ekey[pos] = ((uint64_t)dr << 48) | ((uint64_t)sr << 32) | (uint64_t)c;
    }
    n_en += __popc(m);
  }
  const int Epad = next_pow2(n_en);
  for (int i = n_en + lane; i < Epad; i += 32) s.ekey[i] = U64_MAX;
  __syncwarp();
  warp_bitonic_sort(s.ekey, Epad);

  // ---- degrees, CSR by destination (sorted) and by source ---------------------
  for (int e = lane; e < n_en; e += 32) {
    const uint64_t k = s.ekey[e];
    atomicAdd(&s.indeg[(int)((k >> 48) & 0xFFFF)], 1);
    atomicAdd(&s.outdeg[(int)((k >> 32) & 0xFFFF)], 1);
  }
  __syncwarp();
  warp_exclusive_scan(s.indeg, s.in_start, N);
  warp_exclusive_scan(s.outdeg, s.su_start, N);
  // fill successor lists (order within a source is irrelevant to Kahn);
  // outdeg doubles as the per-source cursor
  for (int r = lane; r < N; r += 32) s.outdeg[r] = 0;
  __syncwarp();
  for (int e = lane; e < n_en; e += 32) {
    const uint64_t k = s.ekey[e];
    const int sr = (int)((k >> 32) & 0xFFFF);
    const int pos = s.su_start[sr] + atomicAdd(&s.outdeg[sr], 1);
    s.succ[pos] = (uint16_t)((k >> 48) & 0xFFFF);
  }
  __syncwarp();

  // ---- Kahn, smallest ready row first (inference.py:127-141) ------------------
  const int W = (N + 31) / 32;
  for (int w = 0; w < W; ++w) {
    const int r = w * 32 + lane;
    const bool rdy = r < N && (s.flags[r] & 1) && s.indeg[r] == 0;
    const unsigned m = __ballot_sync(0xffffffffu, rdy);
    if (lane == 0) s.ready[w] = m;
  }
  __syncwarp();
  int n_order = 0;
  for (; n_order < n_live; ++n_order) {
    unsigned mine = 0xFFFFFFFFu;
    for (int w = lane; w < W; w += 32) {
      if (s.ready[w]) { mine = (unsigned)w; break; }
    }
    const unsigned wmin = __reduce_min_sync(0xffffffffu, mine);
    if (wmin == 0xFFFFFFFFu) break;
    const uint32_t word = s.ready[wmin];
    const int bit = __ffs(word) - 1;
    const int pick = (int)wmin * 32 + bit;
    __syncwarp();
    if (lane == 0) {
      s.ready[wmin] = word & ~(1u << bit);
      s.order[n_order] = (uint16_t)pick;
    }
    __syncwarp();
    const int e1 = s.su_start[pick + 1];
    for (int e = s.su_start[pick] + lane; e < e1; e += 32) {
      const int d = s.succ[e];
      if (atomicSub(&s.indeg[d], 1) == 1) atomicOr(&s.ready[d >> 5], 1u << (d & 31));
    }
    __syncwarp();
  }
  if (n_order < n_live) status |= ST_CYCLIC;

  // ---- order / io rows outputs -----------------------------------------------
  if (order_out) {
    for (int i = lane; i < N; i += 32)
      order_out[g * N + i] = i < n_order ? (int16_t)s.order[i] : (int16_t)-1;
  }
  for (int k = lane; k < io; k += 32) {
    const int r = lookup_row(s.skey, Npad, (uint64_t)k);
    if (r < 0) status |= ST_MISSING_IO;
    if (io_rows) io_rows[g * io + k] = r;
  }
  status = __reduce_or_sync(0xffffffffu, status);

  uint8_t* gp = prog + g * L.stride;
  ProgHeader* hdr = (ProgHeader*)gp;
  const bool recurrent = mode == 1;
  if ((status & ~ST_CYCLIC) || ((status & ST_CYCLIC) && !recurrent)) {
    if (lane == 0) {
      ProgHeader h{0, 0, I, n_order, status, n_live, mode, 0};
      *hdr = h;
      if (status_out) status_out[g] = status;
    }
    return;
  }

  // ---- which nodes matter (ancestor cone of the outputs) and which are read ----
  if (!recurrent && prune) {
    for (int r = lane; r < N; r += 32)
      if (s.flags[r] & 4) s.needed[r] = 1;
    __syncwarp();
    for (int i = n_order - 1; i >= 0; --i) {
      const int r = s.order[i];
      if (!s.needed[r] || (s.flags[r] & 2)) continue;
      for (int e = s.in_start[r] + lane; e < s.in_start[r + 1]; e += 32) {
        const int sr = (int)((s.ekey[e] >> 32) & 0xFFFF);
        s.needed[sr] = 1;
        s.used[sr] = 1;
      }
      __syncwarp();
    }
  } else {
    for (int r = lane; r < N; r += 32) {
      s.needed[r] = (s.flags[r] & 1) ? 1 : 0;
      s.used[r] = (s.su_start[r + 1] > s.su_start[r]) ? 1 : 0;
    }
  }
  __syncwarp();

  // ---- steps: the order (ff) or every live non-input row (recurrent) ----------
  // feed-forward steps keep a slot only when read later or an output; recurrent
  // steps all keep one (their value is the next step's state)
  int n_steps = 0, n_edges = 0, n_store = 0;
  const int n_pos = recurrent ? N : n_order;
  StepT<T>* steps = (StepT<T>*)(gp + L.off_steps);
  EdgeT<T>* edges = (EdgeT<T>*)(gp + L.off_edges);
  for (int r = lane; r < N; r += 32)
    if (s.flags[r] & 2) s.slot_of[r] = (uint16_t)(gn[(int64_t)r * 5] );  // input key i -> slot i
  __syncwarp();
  int bad = 0;
  for (int base = 0; base < n_pos; base += 32) {
    const int i = base + lane;
    int r = -1;
    if (i < n_pos) r = recurrent ? i : (int)s.order[i];
    const bool emit = r >= 0 && (s.flags[r] & 1) && !(s.flags[r] & 2) && s.needed[r];
    const bool store = emit && (recurrent || s.used[r] || (s.flags[r] & 4));
    const int cnt = emit ? s.in_start[r + 1] - s.in_start[r] : 0;
    const unsigned me = __ballot_sync(0xffffffffu, emit);
    const unsigned ms = __ballot_sync(0xffffffffu, store);
    const unsigned lt = (1u << lane) - 1;
    int x = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (emit) {
      const int k = n_steps + __popc(me & lt);
      const uint16_t slot = store ? (uint16_t)(I + n_store + __popc(ms & lt)) : NO_SLOT;
      s.slot_of[r] = slot;
      const double* nr = gn + (int64_t)r * 5;
      const double av = nr[4], gv = nr[3];
      if (!(av >= 0.0 && av < ACT_COUNT && av == floor(av))) bad |= ST_BAD_ACT;
      if (!(gv >= 0.0 && gv < AGG_COUNT && gv == floor(gv))) bad |= ST_BAD_AGG;
      StepT<T> st;
      memset(&st, 0, sizeof(st));
      st.slot = slot;
      st.act = (uint8_t)(av >= 0.0 && av < ACT_COUNT ? (int)av : 0);
      st.agg = (uint8_t)(gv >= 0.0 && gv < AGG_COUNT ? (int)gv : 0);
      st.e_begin = (uint16_t)(n_edges + x - cnt);
      st.e_count = (uint16_t)cnt;
      st.bias = (T)nr[1];
      st.resp = (T)nr[2];
      steps[k] = st;
    }
    n_steps += __popc(me);
    n_store += __popc(ms);
    n_edges += __shfl_sync(0xffffffffu, x, 31);
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  status |= bad;
  __syncwarp();

  // edges of each step (source slot + weight, source-row order); lanes own
  // steps, each lane writes its step's edges
  {
    int kbase = 0;
    for (int base = 0; base < n_pos; base += 32) {
      const int i = base + lane;
      int r = -1;
      if (i < n_pos) r = recurrent ? i : (int)s.order[i];
      const bool emit = r >= 0 && (s.flags[r] & 1) && !(s.flags[r] & 2) && s.needed[r];
      const unsigned me = __ballot_sync(0xffffffffu, emit);
      if (emit) {
        const int k = kbase + __popc(me & ((1u << lane) - 1));
        const int eb = steps[k].e_begin;
        const int e0 = s.in_start[r], e1 = s.in_start[r + 1];
        for (int e = e0; e < e1; ++e) {
          const uint64_t kk = s.ekey[e];
          const int sr = (int)((kk >> 32) & 0xFFFF);
          const int crow = (int)(kk & 0xFFFFFFFFu);
          EdgeT<T> ed;
          memset(&ed, 0, sizeof(ed));
          ed.src = s.slot_of[sr];
          ed.w = (T)gc[(int64_t)crow * 4 + 3];
          edges[eb + (e - e0)] = ed;
        }
      }
      kbase += __popc(me);
    }
  }
  uint16_t* out_slot = (uint16_t*)(gp + L.off_out);
  for (int o = lane; o < O; o += 32) {
    const int r = lookup_row(s.skey, Npad, (uint64_t)(I + o));
    out_slot[o] = r >= 0 ? s.slot_of[r] : NO_SLOT;
  }
  if (lane == 0) {
    ProgHeader h{n_steps, n_edges, I + n_store, n_order, status, n_live, mode, 0};
    *hdr = h;
    if (status_out) status_out[g] = status;
    atomicMax(&maxdims[0], I + n_store);
    atomicMax(&maxdims[1], n_steps);
    atomicMax(&maxdims[2], n_edges);
  }
}

}  // namespace tneat

using namespace tneat;

extern "C" {

// Bytes of one genome's program (header + output slots + steps + edges).
int64_t an_program_stride(int N, int C, int O, int precision) {
  return prog_layout(N, C, O, precision).stride;
}

// Replaces inference.transform_arrays (inference.py:82-147).  See include/tneat.h.
int an_transform(const double* nodes, const double* conns, int64_t P, int N, int C, int I, int O,
                 int mode, int precision, int prune, void* program, int64_t program_stride,
                 int16_t* order, int16_t* conn_rows, int32_t* io_rows, int32_t* status,
                 int32_t* maxdims, void* stream) {
  if (P < 0 || N < 1 || N > 65535 || C < 0 || C > 65535 || I < 1 || O < 1 || I + O > N) return -1;
  if (!nodes || !program || !maxdims || (C > 0 && !conns)) return -2;
  const ProgLayout L = prog_layout(N, C, O, precision);
  if (program_stride != L.stride) return -3;
  if (P == 0) return 0;
  const int64_t ws = warp_smem_bytes(N, C > 0 ? C : 1);
  int wpb = 4;
  while (wpb > 1 && ws * wpb > 160 * 1024) wpb >>= 1;
  if (ws > 200 * 1024) return -4;  // genome capacity too large for one warp's shared memory
  const int64_t smem = ws * wpb;
  const int64_t blocks = (P + wpb - 1) / wpb;
  cudaStream_t st = (cudaStream_t)stream;
  const int Cc = C > 0 ? C : 1;
  if (precision) {
    cudaFuncSetAttribute(transform_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    transform_kernel<double><<<(unsigned)blocks, 32 * wpb, smem, st>>>(
        nodes, conns, P, N, C, I, O, mode, prune, ws, (uint8_t*)program, L, order, conn_rows,
        io_rows, status, maxdims);
  } else {
    cudaFuncSetAttribute(transform_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    transform_kernel<float><<<(unsigned)blocks, 32 * wpb, smem, st>>>(
        nodes, conns, P, N, C, I, O, mode, prune, ws, (uint8_t*)program, L, order, conn_rows,
        io_rows, status, maxdims);
  }
  (void)Cc;
  TNEAT_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
