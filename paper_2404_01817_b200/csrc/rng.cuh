// Counter-based splitmix64 streams on the device (reference rng.py:1-137).
//
// key(seed, path)  = fold(...fold(mix64(seed), t0)..., tn),  fold(k, t) = mix64(k ^ mix64(t + G))
// raw draw j        = mix64(key + (j + 1) * G)                       (rng.py:86-90)
// uniform           = ((bits >> 11) + 0.5) * 2^-53   -- exact in fp64 (rng.py:96)
// normal (cell)     = sqrt(-2 ln u1) * cos(2 pi u2), u1 at base+col, u2 at base+width+col
//                     (rng.py:125-134); CUDA's log/cos differ from numpy's by <= ~1 ulp
//
// Streams are pure functions of (key, counter), so any thread can draw any
// cell of a stream's tape -- the property that makes the population
// operators independent of how genomes map onto warps.
#pragma once

#include <cstdint>

namespace tneat {

constexpr uint64_t RNG_GOLDEN = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t rng_fold(uint64_t key, uint64_t token) {
  return mix64(key ^ mix64(token + RNG_GOLDEN));
}

__host__ __device__ __forceinline__ uint64_t rng_bits(uint64_t key, uint64_t j) {
  return mix64(key + (j + 1) * RNG_GOLDEN);
}

__device__ __forceinline__ double bits_to_uniform(uint64_t b) {
  return __dmul_rn(__dadd_rn((double)(b >> 11), 0.5), 1.1102230246251565e-16 /* 2^-53 */);
}

__device__ __forceinline__ double rng_uniform(uint64_t key, uint64_t j) {
  return bits_to_uniform(rng_bits(key, j));
}

// Box-Muller exactly as numpy evaluates it: sqrt(-2.0 * log(u1)) * cos(2.0 * pi * u2)
__device__ __forceinline__ double rng_normal_cell(uint64_t key, uint64_t base, uint64_t width, uint64_t col) {
  const double u1 = rng_uniform(key, base + col);
  const double u2 = rng_uniform(key, base + width + col);
  const double r = sqrt(__dmul_rn(-2.0, log(u1)));
  const double c = cos(__dmul_rn(6.283185307179586 /* 2.0 * np.pi */, u2));
  return __dmul_rn(r, c);
}

}  // namespace tneat
