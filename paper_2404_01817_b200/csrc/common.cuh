// Shared definitions for the tneat sm_100a kernels.
//
// Program format: the transform kernel (transform.cu) compiles every genome
// into a fixed-stride "program" that the forward kernels (forward.cu) execute.
// A program is a flat byte block per genome:
//
//   [ProgHeader 32 B][out_slot u16 x O, padded to 16 B][Step x N][Edge x C]
//
// Steps are the non-input nodes in the reference's Kahn order
// (inference.py:127-141) that can influence an output (ancestor-cone pruning,
// SURVEY.md App. B "K2 ... safe optimisation"); edges are the enabled incoming
// connections of each step, sorted by source row (inference.py:108-112 keeps a
// dense incoming row; we keep its non-NaN entries in the same column order).
// "Slots" index node values: slot i < I is input key i, later slots hold the
// stored steps in order.
#pragma once

#include <cstdint>
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
  int32_t n_edges;   // edges referenced by the steps
  int32_t n_slots;   // value slots (inputs first)
  int32_t n_order;   // nodes placed in the Kahn order
  int32_t status;    // ST_* bits
  int32_t n_live;    // live node rows
  int32_t mode;      // 0 feed-forward, 1 recurrent
  int32_t reserved;
};

template <typename T> struct StepT;
template <> struct __align__(16) StepT<float> {
  uint16_t slot; uint8_t act; uint8_t agg; uint16_t e_begin; uint16_t e_count;
  float bias; float resp;
};
template <> struct __align__(16) StepT<double> {
  uint16_t slot; uint8_t act; uint8_t agg; uint16_t e_begin; uint16_t e_count;
  uint32_t pad; double bias; double resp;
};
template <typename T> struct EdgeT;
template <> struct __align__(8) EdgeT<float> { uint32_t src; float w; };
template <> struct __align__(16) EdgeT<double> { uint32_t src; uint32_t pad; double w; };

static_assert(sizeof(StepT<float>) == 16, "step layout");
static_assert(sizeof(StepT<double>) == 32, "step layout");
static_assert(sizeof(EdgeT<float>) == 8, "edge layout");
static_assert(sizeof(EdgeT<double>) == 16, "edge layout");

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct ProgLayout {
  int64_t off_out, off_steps, off_edges, stride;
};

__host__ __device__ inline ProgLayout prog_layout(int N, int C, int O, int precision) {
  ProgLayout L;
  const int64_t ss = precision ? sizeof(StepT<double>) : sizeof(StepT<float>);
  const int64_t es = precision ? sizeof(EdgeT<double>) : sizeof(EdgeT<float>);
  L.off_out = sizeof(ProgHeader);
  L.off_steps = align_up(L.off_out + 2 * (int64_t)O, 16);
  L.off_edges = align_up(L.off_steps + ss * N, 16);
  L.stride = align_up(L.off_edges + es * C, 16);
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

__device__ __forceinline__ float apply_act(int code, float x) {
  switch (code) {
    case ACT_TANH: return tanh_fast(x);
    case ACT_SIGMOID: return sigmoid_fast(x);
    case ACT_RELU: return fmaxf(x, 0.0f);
    default: return x;
  }
}
__device__ __forceinline__ double apply_act(int code, double x) {
  switch (code) {
    case ACT_TANH: return tanh(x);
    case ACT_SIGMOID: return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
    case ACT_RELU: return fmax(x, 0.0);
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
    case AGG_MAX: return acc > x ? acc : x;
    case AGG_MIN: return acc < x ? acc : x;
    default: return acc + x;
  }
}

// empty set -> 0 for every aggregation (inference.py:238-240); mean divides by count
template <typename T> __device__ __forceinline__ T agg_finish(int agg, T acc, int count) {
  if (count == 0) return T(0);
  if (agg == AGG_MEAN) return acc / T(count);
  return acc;
}

}  // namespace tneat

#define TNEAT_CHECK_LAUNCH()                                  \
  do {                                                        \
    cudaError_t _e = cudaGetLastError();                      \
    if (_e != cudaSuccess) return -100 - (int)_e;             \
  } while (0)
