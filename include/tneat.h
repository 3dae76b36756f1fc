/*
 * tneat.h -- C ABI of libtneat.so, the B200 (sm_100a) population-parallel NEAT
 * hot path.  Plain pointers, sizes and a CUDA stream; no torch types.
 *
 * Conventions:
 *   - every pointer argument is DEVICE memory unless documented otherwise;
 *     the caller (PyTorch on the Python side) allocates every buffer; the
 *     library allocates nothing and keeps no mutable global state;
 *   - every entry point is stream-ordered on `stream` (a cudaStream_t passed
 *     as void*) and reentrant;
 *   - return value: 0 = ok, -1..-99 = argument error, <= -100 = CUDA launch
 *     error (cudaError_t = -(ret + 100)); nothing throws across the ABI;
 *   - per-genome failures are reported in per-genome status arrays, which the
 *     Python wrapper turns into arrayneat exceptions (CycleDetected, ...).
 *
 * Each function names the reference interface it replaces
 * (/root/reference/pkg/src/arrayneat/<file>:<line>).
 */
#ifndef TNEAT_H
#define TNEAT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- programs ------------------------------------------------------------ */

/* Bytes of one genome's compiled program for capacity (N nodes, C conns, O
 * outputs); precision 0 = fp32 program, 1 = fp64 program. */
int64_t an_program_stride(int N, int C, int O, int precision);

/* Genome transform.  Replaces inference.transform_arrays
 * (inference.py:82-147): key->row lookup (search.py:103-124), enabled mask
 * (inference.py:93-95), Kahn order with smallest-ready-row tie break
 * (inference.py:127-141), cyclic detection (inference.py:143).
 *
 *   nodes    (P, N, 5) float64, reference layout (genome.py:29-35)
 *   conns    (P, C, 4) float64
 *   mode     0 = feed-forward (cyclic genomes flagged), 1 = recurrent
 *   prune    1 = drop nodes outside the outputs' ancestor cone (output-preserving)
 *   program  (P, program_stride) bytes, written
 *   order    (P, N) int16 row order, -1 padded (StackedNetworks.order), or NULL
 *   conn_rows (P, C, 2) int16 (src row, dst row) of enabled conns, -1 else, or NULL
 *   io_rows  (P, I+O) int32 rows of keys 0..I+O-1, or NULL
 *   status   (P,) int32 ST_* bits (1 cyclic, 2 bad act, 4 bad agg, 8 bad key,
 *            16 dangling endpoint, 32 missing io key), or NULL
 *   maxdims  (3,) int32, must be zeroed by the caller: atomic max over the
 *            population of {value slots, steps, edges} -- sizes the forward launch
 */
int an_transform(const double* nodes, const double* conns, int64_t P, int N, int C, int I, int O,
                 int mode, int precision, int prune, void* program, int64_t program_stride,
                 int16_t* order, int16_t* conn_rows, int32_t* io_rows, int32_t* status,
                 int32_t* maxdims, void* stream);

/* ---- forward ------------------------------------------------------------- */

/* Population forward.  Replaces inference.forward_arrays (inference.py:185-262).
 *   inputs   (P, B, I) float32 (precision 0) or float64 (precision 1);
 *            input_genome_stride = elements between genomes (0 = shared inputs,
 *            as XorProblem.evaluate_stacked broadcasts them, problems.py:230)
 *   outputs  (P, B, O), same dtype
 *   maxdims_host  HOST pointer to 3 ints {value slots, steps, edge entries}:
 *            the an_transform maxima, or tighter bounds for the genomes listed
 *   genome_ids  optional (P,) int32 DEVICE list of program rows to evaluate
 *            (NULL = rows 0..P-1); inputs/outputs are addressed by program row,
 *            so a launch per slot-count bucket raises occupancy
 *   variant  0 auto, 1/3 = tile kernel 1 input/thread (128/64 threads),
 *            2/5 = 2 inputs/thread (128/64 threads), 4 = 4 inputs/thread,
 *            8 = warp-per-genome kernel (small B) */
int an_forward(const void* program, int64_t program_stride, int N, int C, int precision,
               const int32_t* maxdims_host, const int32_t* genome_ids, const void* inputs,
               int64_t input_genome_stride, int64_t P, int B, int I, int O, void* outputs, int variant,
               void* stream);

/* Forward fused with the built-in fitness.  Replaces
 * XorProblem.evaluate_stacked (problems.py:229-231, fitness :54-56) for
 * kind 1 (B = 4) and RegressionProblem.evaluate_stacked (problems.py:252-254,
 * fitness :59-61) for kind 2 (targets[B] float64).  fitness (P,) float64. */
int an_forward_fitness(const void* program, int64_t program_stride, int N, int C, int precision,
                       const int32_t* maxdims_host, const void* inputs, int64_t input_genome_stride,
                       int64_t P, int B, int I, int O, int kind, const double* targets,
                       double* fitness, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TNEAT_H */
