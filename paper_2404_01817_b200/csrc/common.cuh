// Shared definitions for the tneat sm_100a kernels.
//
// Program format: the transform kernel (transform.cu) compiles every genome
// into a fixed-stride "program" that the forward kernels (forward.cu) execute.
// A program is a flat byte block per genome:
//
//   [ProgHeader 32 B][out_slot u16 x O][GroupRec x N][Step x N][edges x (3C+12N+16)]
//
// Steps are the non-input nodes that can influence an output (ancestor-cone
// pruning, SURVEY.md App. B "K2 ... safe optimisation"), ordered by
// topological level (a valid topological order; node values do not depend on
// the evaluation order of independent nodes, so this is exact) and grouped.
// Each step's edges are its enabled incoming connections in source-row order
// (the non-NaN entries of the reference's dense incoming row,
// inference.py:108-112).  "Slots" index node values: slot i < I starts as
// input key i; slots are recycled once their last reader has run (liveness).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace tneat {

// act codes = functions.py:26-31; agg codes = functions.py:34-39 (+ min, code 4)
enum : int { ACT_IDENTITY = 0, ACT_TANH = 1, ACT_SIGMOID = 2, ACT_RELU = 3, ACT_COUNT = 4 };
enum : int { AGG_SUM = 0, AGG_PRODUCT = 1, AGG_MAX = 2, AGG_MEAN = 3, AGG_MIN = 4, AGG_COUNT = 5 };

// per-genome status bits written by the transform
enum : int {
  ST_CYCLIC = 1,       // enabled conns contain a cycle (inference.py:143)
  ST_BAD_ACT = 2,      // activation code outside the table (functions.py:54-58)
  ST_BAD_AGG = 4,      // aggregation code outside the table (functions.py:60-64)
  ST_BAD_KEY = 8,      // negative / non-integer / >= 2^47 key
  ST_DANGLING = 16,    // conn endpoint is not a live node key
  ST_MISSING_IO = 32,  // an input/output key is not live
};

constexpr uint16_t NO_SLOT = 0xFFFF;

struct ProgHeader {  // 32 bytes
  int32_t n_steps;   // evaluated (non-input, needed) nodes
  int32_t n_edges;   // edge entries, including padding
  int32_t n_slots;   // value slots (inputs first; the last one is the zero slot)
  int32_t n_order;   // nodes placed in the Kahn order
  int32_t status;    // ST_* bits
  int32_t n_live;    // live node rows
  int32_t mode;      // 0 feed-forward, 1 recurrent
  int32_t n_groups;  // step groups
};

// A group is 1..4 steps of the same topological level (no edges between them)
// with the same aggregation class.  Their edge lists are interleaved
// round-major with a row width of gw = (n == 3 ? 4 : n) entries -- edge r of
// step j sits at e_begin + r*gw + j -- so the forward kernel accumulates the n
// nodes in lock-step as n independent FMA chains.  In sum/mean groups the
// entries past a step's count are holes that read the genome's zero slot
// (header n_slots - 1, never written) with weight 0, so the rounds run
// unpredicated.  e_begin is a multiple of 8, so two rounds of
// sources / weights are single 16-byte loads.  Non-sum aggregations are
// singleton groups with exact counts.
struct __align__(16) GroupRec {  // 16 bytes
  uint8_t n;           // steps in the group (1..4)
  uint8_t cls;         // GRP_* bits: GRP_GENERIC = non-sum aggregation (singleton),
                       // GRP_TANH_SUM = every step is tanh/sum (fast epilogue)
  uint16_t rounds;     // longest edge list in the group
  uint16_t e_begin;    // first edge entry (multiple of 8)
  uint16_t step_begin;
  uint16_t cnt[4];     // edge count of each step
};

// GRP_SPLIT0 (sum/mean groups of 3): the spare fourth column holds the second
// half of step 0's list (cnt[0] = first-half count, cnt[3] = the rest;
// StepT::count stays the total), so the group runs max(ceil(c0/2), c1) rounds
enum : uint8_t { GRP_GENERIC = 1, GRP_TANH_SUM = 2, GRP_SPLIT0 = 4 };

__host__ __device__ inline int group_width(int n) { return n == 3 ? 4 : n; }

template <typename T> struct StepT;
// fp32 step: activation evaluated branch-free (common.cuh step_act)
template <> struct __align__(16) StepT<float> {
  uint16_t slot; uint8_t act; uint8_t agg; uint16_t count; uint16_t pad;
  float bias; float resp;
};
template <> struct __align__(16) StepT<double> {
  uint16_t slot; uint8_t act; uint8_t agg; uint16_t count; uint16_t pad;
  uint64_t pad2; double bias; double resp;
};
// fp64 programs keep (source slot, weight) pairs; fp32 programs keep two
// arrays, u16 source slots and f32 weights (6 bytes per edge)
struct __align__(16) EdgeD { uint32_t src; uint32_t pad; double w; };

// Program format bits.  FMT_TC (fp32 feed-forward): programs whose steps all
// aggregate by sum / mean get the tensor-core input layer (forward.cu
// fwd_tc_kernel, csrc/digits.cuh): the input-sourced part of every step is one
// digit-split MMA per 128-sample tile, and the group / step / edge areas hold
// the hidden-sourced edges only, with one value slot per step (slot = step
// index, zero slot = n_steps).  Appended areas: per-step column factors, the
// input edge lists (exact path for rows the MMA cannot scale) and the B
// operand (digit planes, UMMA K-major layout).  Other genomes of an FMT_TC
// population get standard programs in the same stride (ProgHeader.mode = 0
// instead of MODE_TC).
enum : int { FMT_F64 = 1, FMT_TC = 2 };
enum : int { MODE_FF = 0, MODE_REC = 1, MODE_TC = 2 };

static_assert(sizeof(GroupRec) == 16, "group layout");
static_assert(sizeof(StepT<float>) == 16, "step layout");
static_assert(sizeof(StepT<double>) == 32, "step layout");
static_assert(sizeof(EdgeD) == 16, "edge layout");

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// edge entries a genome may need: each group's list is padded to gw*rounds
// (a step joins a group only if its list is >= half the longest, so padded
// <= 8/3 x real), rounds are even (+gw <= 4 per group) and every group starts
// on a multiple of 8 (+7)
__host__ __device__ inline int64_t edge_capacity(int N, int C) { return 3ll * C + 12ll * N + 16; }

struct ProgLayout {
  int64_t off_out, off_groups, off_steps, off_src, off_w, stride;
  // FMT_TC: a MODE_TC program keeps everything the tensor-core kernel stages in
  // one contiguous block at off_tc (internal offsets from the genome's counts,
  // tc_block), and the exact-path input edge lists at fixed offsets; its
  // standard areas (off_groups..) are unused.  0 for other formats.
  int64_t off_tc, off_in, off_isrc, off_iw;
};

// TC group record (pre-decoded for the sweep): code = (n - 1) | tanh << 2 |
// split0 << 3 (the dispatch index), rounds, first edge entry, first step.  In
// tanh groups the step records carry bias and response pre-multiplied by
// -2 log2(e) (the epilogue's EX2 argument is one FFMA away)
struct __align__(16) GroupTC {
  uint32_t code, rounds, e_begin, step_begin;
};
static_assert(sizeof(GroupTC) == 16, "group layout");
constexpr float TANH_K = -2.8853900817779268f;

constexpr int TC_SAMPLES = 256;            // samples per tile of the tensor-core kernel
constexpr int TC_SLOT_BYTES = TC_SAMPLES * 4;  // one value slot row [128 threads][2 samples] fp32

__host__ __device__ inline int tc_rows(int n) { return (n + 15) / 16 * 16; }

// the staged block of a MODE_TC program: B operand (round16(steps) rows x 192 B,
// UMMA K-major core matrices, csrc/digits.cuh), column factors f32[nb], group
// records, step records, hidden-edge source byte offsets u32 (slot *
// TC_SLOT_BYTES) and weights f32 (the look-ahead of the word prefetch reads
// past the weights: the kernel leaves slack after the block)
struct TcBlock {
  uint32_t b, cf, gr, st, src, w, bytes;
};
__host__ __device__ inline TcBlock tc_block(int n_steps, int n_groups, int n_edges) {
  TcBlock t;
  const uint32_t nb = (uint32_t)tc_rows(n_steps);
  t.b = 0;
  t.cf = 192u * nb;
  t.gr = t.cf + 4u * nb;
  t.st = t.gr + 16u * (uint32_t)n_groups;
  t.src = t.st + 16u * (uint32_t)n_steps;
  t.w = t.src + 4u * (uint32_t)n_edges;
  t.bytes = (t.w + 4u * (uint32_t)n_edges + 15u) & ~15u;
  return t;
}

// `precision` is the program format: bit 0 = fp64 program, bit 1 = FMT_TC (fp32)
__host__ __device__ inline ProgLayout prog_layout(int N, int C, int O, int precision) {
  ProgLayout L;
  const int64_t E = edge_capacity(N, C);
  L.off_out = 32;
  L.off_groups = align_up(L.off_out + 2 * (int64_t)O, 16);
  L.off_steps = align_up(L.off_groups + 16ll * N, 16);
  L.off_tc = L.off_in = L.off_isrc = L.off_iw = 0;
  if (precision & FMT_F64) {
    L.off_src = align_up(L.off_steps + 32ll * N, 16);
    L.off_w = L.off_src;  // EdgeD pairs
    L.stride = align_up(L.off_w + 16 * E, 16);
  } else {
    L.off_src = align_up(L.off_steps + 16ll * N, 16);
    L.off_w = align_up(L.off_src + 2 * E, 16);
    L.stride = align_up(L.off_w + 4 * E, 16);
    if (precision & FMT_TC) {
      const int64_t Cc = C > 0 ? C : 1;
      L.off_tc = align_up(L.off_out + 2 * (int64_t)O, 128);
      L.off_in = align_up(L.off_tc + tc_block(N, N, (int)E).bytes, 16);
      L.off_isrc = align_up(L.off_in + 2ll * (N + 1), 16);
      L.off_iw = align_up(L.off_isrc + 2 * Cc, 16);
      const int64_t end = align_up(L.off_iw + 4 * Cc, 128);
      L.stride = end > align_up(L.stride, 128) ? end : align_up(L.stride, 128);
    }
  }
  return L;
}

// ---------------------------------------------------------------------------
// activations
// ---------------------------------------------------------------------------

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// tanh with |err| <~ 2e-7 absolute: (1 - e) / (1 + e), e = 2^(-2|x| log2 e).
// Two MUFU ops (EX2, RCP); the forward parity bound is abs 1e-5 * max(1,|ref|).
__device__ __forceinline__ float tanh_fast(float x) {
  const float e = ex2_approx(-2.8853900817779268f * fabsf(x));
  const float t = (1.0f - e) * rcp_approx(1.0f + e);
  return copysignf(t, x);
}
// sigmoid = exp(-logaddexp(0, -x)) = 1 / (1 + exp(-x))  (functions.py:20-22)
__device__ __forceinline__ float sigmoid_fast(float x) {
  return rcp_approx(1.0f + ex2_approx(-1.4426950408889634f * x));
}

// branch-free fp32 activation of a step (see StepT<float>)
__device__ __forceinline__ float step_act(float kx, float ca, float cb, bool relu, float pre) {
  const float sg = rcp_approx(1.0f + ex2_approx(kx * pre));
  const float smooth = fmaf(ca, sg, cb);
  const float lin = relu ? ((pre >= 0.0f || pre != pre) ? pre : 0.0f) : pre;  // np.maximum(x, 0): NaN stays
  return kx != 0.0f ? smooth : lin;
}

__device__ __forceinline__ float apply_act(int code, float x) {
  switch (code) {
    case ACT_TANH: return tanh_fast(x);
    case ACT_SIGMOID: return sigmoid_fast(x);
    case ACT_RELU: return (x >= 0.0f || x != x) ? x : 0.0f;  // np.maximum(x, 0.0) (functions.py:30): NaN stays
    default: return x;
  }
}
__device__ __forceinline__ double apply_act(int code, double x) {
  switch (code) {
    case ACT_TANH: return tanh(x);
    case ACT_SIGMOID: return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
    case ACT_RELU: return (x >= 0.0 || x != x) ? x : 0.0;
    default: return x;
  }
}

template <typename T> __device__ __forceinline__ T agg_neutral(int agg) {
  switch (agg) {
    case AGG_PRODUCT: return T(1);
    case AGG_MAX: return -INFINITY;
    case AGG_MIN: return INFINITY;
    default: return T(0);
  }
}

template <typename T> __device__ __forceinline__ T agg_combine(int agg, T acc, T x) {
  switch (agg) {
    case AGG_PRODUCT: return acc * x;
    // numpy's maximum / minimum (functions.py:37 reduces with np.max): a NaN on
    // either side wins, ties keep the accumulator
    case AGG_MAX: return (acc >= x || acc != acc) ? acc : x;
    case AGG_MIN: return (acc <= x || acc != acc) ? acc : x;
    default: return acc + x;
  }
}

// empty set -> 0 for every aggregation (inference.py:238-240); mean divides by count
template <typename T> __device__ __forceinline__ T agg_finish(int agg, T acc, int count) {
  if (count == 0) return T(0);
  if (agg == AGG_MEAN) return acc / T(count);
  return acc;
}

// Checked builds (-DTNEAT_CHECKS, tools/build_variant.py checks): device-side
// bounds checks on every shared-memory carve, staged program index and
// program write; a violation prints its site and traps (the launch fails with
// an error the host raises).  compute-sanitizer is closed on this GPU pool.
#ifdef TNEAT_CHECKS
#define TNEAT_DCHECK(cond, what, a, b)                                                                      \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("TNEAT_CHECK failed: %s (%lld, %lld) at %s:%d block %d thread %d\n", what, (long long)(a),   \
             (long long)(b), __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x);                       \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define TNEAT_DCHECK(cond, what, a, b) \
  do {                                 \
  } while (0)
#endif

__device__ __forceinline__ uint32_t dynamic_smem_bytes() {
  uint32_t r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}

}  // namespace tneat

#define TNEAT_CHECK_LAUNCH()                                  \
  do {                                                        \
    cudaError_t _e = cudaGetLastError();                      \
    if (_e != cudaSuccess) return -100 - (int)_e;             \
  } while (0)
