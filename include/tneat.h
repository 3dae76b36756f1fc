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
 * outputs).  `precision` is the program format: bit 0 = fp64 program (else
 * fp32), bit 1 = FMT_TC (fp32 feed-forward only: genomes whose steps all
 * aggregate by sum / mean get tensor-core programs -- the input layer as an
 * exact digit-split tcgen05 MMA -- the others standard programs in the same
 * stride; see an_forward variant 11 and an_forward_planned); 0 = the standard
 * fp32 program. */
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
 *   order    (P, N) int16 row order, -1 padded (StackedNetworks.order), or NULL.
 *            With NULL the programs are built from a level-synchronous Kahn
 *            (same levels, cycles and programs' results, no per-node order);
 *            with a buffer the reference's one-node-per-step order is emitted.
 *            Repeated enabled (src, dst) pairs follow the reference: the last
 *            connection row wins, and with N <= 64 the genome reads as cyclic
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
 *   variant  0 auto (B >= 192: 5 for fp32 programs, 1 for fp64; B >= 96: 3;
 *            else 8), 1/3 = tile kernel 1 input/thread (128/64 threads),
 *            2/5 = 2 inputs/thread (128/64 threads), 4 = 4 inputs/thread,
 *            8 = warp-per-genome kernel (small B), 11 = tensor-core kernel
 *            (FMT_TC programs whose header mode is 2; persistent, one CTA per
 *            SM; bits 8..11 = maximum warpgroups per CTA, 0 = as many as
 *            fit).  In an FMT_TC population the other variants take the
 *            standard-program genomes only, listed in genome_ids (-7 without).  Bits 8..15 = tiles per CTA for
 *            the tile kernels (0 = 4) */
int an_forward(const void* program, int64_t program_stride, int N, int C, int precision,
               const int32_t* maxdims_host, const int32_t* genome_ids, const void* inputs,
               int64_t input_genome_stride, int64_t P, int B, int I, int O, void* outputs, int variant,
               void* stream);

/* Forward of an FMT_TC population from a DEVICE-side launch plan: a plan
 * kernel sorts the genomes into classes (tensor-core programs by MMA width,
 * oversized ones, standard programs) and every launch is sized from class
 * bounds, so no host-side counts, extents or synchronisation are needed
 * (a transform + forward step can be enqueued ahead or graph-captured).
 * Replaces inference.forward_arrays (inference.py:185-262) for such
 * populations.  plan_ids int32[7 * P] and plan_counts int32[14] are DEVICE
 * scratch owned by the caller (counts[7..13]: the class launches' dynamic
 * task counters, zeroed by the plan); inputs / outputs as an_forward (float32).
 * genome_sq: optional (P,) float32, zeroed by the caller: += the sum of the
 * genome's squared outputs (a fused fitness epilogue; float atomics, so the
 * summation order -- and the last bits -- vary between runs), or NULL. */
int an_forward_planned(const void* program, int64_t program_stride, int N, int C, int precision,
                       int32_t* plan_ids, int32_t* plan_counts, const void* inputs,
                       int64_t input_genome_stride, int64_t P, int B, int I, int O, void* outputs,
                       float* genome_sq, void* stream);

/* The plan step of an_forward_planned alone (diagnostics; plan_counts
 * int32[14], zeroed on the stream first): plan_counts[c] = genomes of class c
 * (0..4 tensor-core programs with round16(steps) <= 32, 48, 64, 96, 128; 5
 * tensor-core programs with > 512 hidden-edge entries; 6 standard programs),
 * plan_ids[c * P + i] their program rows (in no particular order: the class
 * launches hand genomes out dynamically). */
int an_plan_tc(const void* program, int64_t program_stride, int64_t P, int32_t* plan_ids, int32_t* plan_counts,
               void* stream);

/* Forward fused with the built-in fitness.  Replaces
 * XorProblem.evaluate_stacked (problems.py:229-231, fitness :54-56) for
 * kind 1 (B = 4) and RegressionProblem.evaluate_stacked (problems.py:252-254,
 * fitness :59-61) for kind 2 (targets[B] float64).  fitness (P,) float64. */
int an_forward_fitness(const void* program, int64_t program_stride, int N, int C, int precision,
                       const int32_t* maxdims_host, const void* inputs, int64_t input_genome_stride,
                       int64_t P, int B, int I, int O, int kind, const double* targets,
                       double* fitness, void* stream);


/* Cart-pole lockstep episodes (CartPoleProblem.evaluate_stacked,
 * problems.py:153-177, 257-271): warp per genome, float64 Euler dynamics
 * (problems.py:107-122), observations (x, x_dot, theta, theta_dot) -> output
 * row of key I; force = +10 if output > 0 else -10; start (P,4) float64;
 * fitness (P,) float64 = steps survived (<= max_steps). */
int an_cartpole(const void* program, int64_t program_stride, int N, int C, int precision,
                const int32_t* maxdims_host, int64_t P, const double* start, int max_steps, double* fitness,
                void* stream);

/* ---- evolution operators (evolution.py / genome.py) ------------------------ */

/* Mutation / initialisation hyper-parameters (NeatConfig, config.py:31-86),
 * flattened.  Option lists hold function codes (functions.py:26-39). */
typedef struct an_mutate_params {
  int32_t N, C, I, O;          /* max_nodes, max_conns, inputs, outputs */
  int32_t feedforward;         /* network_type == "feedforward" */
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
} an_mutate_params;

/* Tape cells of counter-based streams (rng.py:86-134): out[s, j] = uniform
 * (normals=0) or Box-Muller normal (normals=1, u1 at base+j, u2 at
 * base+width+j) of stream keys[s].  Test hook for RngStream parity. */
int an_rng_draw(const uint64_t* keys, int64_t S, uint64_t base, int64_t width, int normals, double* out,
                void* stream);

/* init_arrays (genome.py:129-160): genome g draws normals from stream keys[g]
 * starting at counter `base`; nodes (P,N,5), conns (P,C,4) written. */
int an_init(double* nodes, double* conns, int64_t P, const uint64_t* keys, uint64_t base,
            const an_mutate_params* params, void* stream);

/* distance_arrays (evolution.py:425-488), bit-exact float64 (sums in the
 * reference's genome-1 row order).  pair_mode 1: out[p] = d(g1[p], g2[Q==1 ? 0 : p]);
 * pair_mode 0: out[q*P + p] = d(g1[p], g2[q]) (speciation, evolution.py:513-559). */
int an_distance(const double* n1, const double* c1, int64_t P, const double* n2, const double* c2, int64_t Q,
                int pair_mode, int N, int C, double c_disjoint, double c_homologous, double* out, void* stream);

/* mutate_arrays (evolution.py:172-325) in place.  keys[i] = stream key of
 * genome i (RngStream._keys), tape cells start at `base` (its counter);
 * new_keys[i] = key a firing node addition uses; can_add (P,) uint8 or NULL. */
int an_mutate(double* nodes, double* conns, int64_t P, const uint64_t* keys, uint64_t base,
              const double* new_keys, const an_mutate_params* params, uint8_t* can_add, void* stream);

/* _crossover_into (evolution.py:101-136): out_* hold the fitter parents and
 * are blended in place with less_* (coins at cells base.. of keys[i]). */
int an_crossover(double* out_nodes, double* out_conns, const double* less_nodes, const double* less_conns,
                 int64_t P, int N, int C, const uint64_t* keys, uint64_t base, void* stream);

/* reproduce worker (evolution.py:685-709) for slots slot_base..+n_slots-1:
 * uniforms(2) parent picks from pool[pool_offset[i] + ...], crossover,
 * mutation, elite overwrite (elite_src[i] >= 0).  Stream of slot s =
 * fold(stage_key, s); a firing node addition in slot s takes key new_key_base + s. */
int an_reproduce(const double* pop_nodes, const double* pop_conns, double* out_nodes, double* out_conns,
                 int64_t n_slots, int64_t slot_base, const int32_t* pool, const int32_t* pool_offset,
                 const int32_t* pool_size, const int32_t* elite_src, uint64_t stage_key, double new_key_base,
                 const an_mutate_params* params, uint8_t* can_add, void* stream);

/* ---- recurrent rollouts (builder-defined; the reference rejects recurrent
 * genomes) ---------------------------------------------------- */

/* Fixed-step synchronous recurrent evaluation inside s' = tanh(A s + M a):
 * program compiled with an_transform mode 1; A (D,D), M (D,O), s0 (D,) in the
 * program's precision; per environment step the inputs are clamped to s and
 * `sweeps` synchronous sweeps run; fitness (P,) float64 = sum_t s_t[0]. */
int an_rollout(const void* program, int64_t program_stride, int N, int C, int precision,
               const int32_t* maxdims_host, int64_t P, int I, int O, const void* A, const void* M, const void* s0,
               int D, int steps, int sweeps, double* fitness, void* stream);

/* ---- HyperNEAT (builder-defined; no reference implementation) ---- */

/* Substrate fitness on the tensor cores (tcgen05 kind::tf32, TMEM
 * accumulators, fused tanh / squared-error epilogue): W (P,64,64) fp32 CPPN
 * weights (row = output node), X (S,64) fp32 shared substrate inputs (S a
 * multiple of 128), target (S,) fp32; fitness (P,) float64 =
 * -mean((tanh(X W_p^T) - target[:,None])^2). */
int an_substrate_fitness(const float* W, int64_t P, const float* X, const float* target, int S, double* fitness,
                         void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TNEAT_H */
