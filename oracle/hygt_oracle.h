/*
 * hygt_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference HyGT hot path (/root/reference/proj/include/hygt),
 * used as the parity checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg. It is never linked into, called by, or shipped with the product library
 * (paper_2505_21728_b200/libhygt_gpu.so). Every function cites the reference file:line it
 * restates. Parity pinning: tests/test_oracle_golden.py checks these functions against golden
 * vectors produced by the unmodified reference headers (oracle/_ref, tests/golden/).
 */
#ifndef HYGT_ORACLE_H
#define HYGT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: same numbering as include/hygt_gpu.h (errors.hpp:23-45 / hygt_main.cpp:275-284). */
#define HYGT_ORACLE_OK 0
#define HYGT_ORACLE_ARGUMENT 1
#define HYGT_ORACLE_NUMERICAL 3
#define HYGT_ORACLE_OVERFLOW 4

/* ---- RNG: rng.hpp:26-77 ------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} hygt_oracle_rng;

uint64_t hygt_oracle_splitmix64(uint64_t state);                     /* rng.hpp:26-31 */
uint64_t hygt_oracle_derive_seed(uint64_t base, uint64_t stream);    /* rng.hpp:36-38 */
void hygt_oracle_rng_seed(hygt_oracle_rng* r, uint64_t seed);         /* rng.hpp:46 (mt19937_64) */
uint64_t hygt_oracle_rng_next(hygt_oracle_rng* r);                    /* std::mt19937_64::operator() */
double hygt_oracle_rng_uniform01(hygt_oracle_rng* r);                 /* rng.hpp:49 */
double hygt_oracle_rng_uniform(hygt_oracle_rng* r, double lo, double hi); /* rng.hpp:52 */
double hygt_oracle_rng_gaussian(hygt_oracle_rng* r);                  /* rng.hpp:55-68 */
uint64_t hygt_oracle_rng_below(hygt_oracle_rng* r, uint64_t bound);   /* rng.hpp:71 */

/* ---- schedule: hypercube.hpp:59-77 --------------------------------------------------------- */
int hygt_oracle_hypercube_indices(int log2_n, int pass, uint32_t* m, uint32_t* n);
size_t hygt_oracle_num_parameters(int log2_n, int rounds); /* model.hpp:29-34 (0 on bad args) */

/* ---- float transform: transform.hpp:45-96 ------------------------------------------------- */
/* One model: angles[rounds*log2_n*N/2] in application order (model.hpp:77-79), optional final
 * permutation perm[N] (NULL = none). In place on x[N] (fp64). */
void hygt_oracle_run_passes(int log2_n, int rounds, const double* angles, double* x, int dir);
void hygt_oracle_forward(int log2_n, int rounds, const double* angles, const uint16_t* perm,
                         double* x);
void hygt_oracle_inverse(int log2_n, int rounds, const double* angles, const uint16_t* perm,
                         double* x);
/* BASELINE extension: inter-round permutations = chain of single-round
 * models M_r = HyGTModel(n, 1, angles[r*A1 .. (r+1)*A1), P_r). perms is [rounds][N]; bit r of
 * perm_mask says P_r is present (bit rounds-1 = the reference's final sorting permutation). */
void hygt_oracle_forward_chain(int log2_n, int rounds, const double* angles,
                               const uint16_t* perms, uint32_t perm_mask, double* x);
void hygt_oracle_inverse_chain(int log2_n, int rounds, const double* angles,
                               const uint16_t* perms, uint32_t perm_mask, double* x);
/* Dense transform matrix, column j = forward(e_j) (transform.hpp:100-117). t is N*N row-major. */
void hygt_oracle_to_matrix(int log2_n, int rounds, const double* angles, const uint16_t* perms,
                           uint32_t perm_mask, double* t);

/* Batched apply over fp32 rows with per-row class ids (the run_apply loop,
 * hygt_main.cpp:143-149). angles [classes][A], perms [classes][rounds][N] or NULL.
 * cls NULL => class 0 for every row. Output in fp64 so tests can measure fp32 error.
 * Returns 1 (ArgumentError) if a class id is out of range (dataset.hpp:47). threads<=0 => 1. */
int hygt_oracle_apply_batch(int log2_n, int rounds, int classes, const double* angles,
                            const uint16_t* perms, uint32_t perm_mask, const float* x,
                            const uint16_t* cls, uint64_t count, int inverse, double* y,
                            int threads);

/* Per-class per-coefficient energy of forward outputs, E[c][i] = sum_{v in c} y_v[i]^2
 * (diagonal of CorrelationAccumulator::add, statistics.hpp:69-77). energy is [classes][N]. */
int hygt_oracle_class_energy(int log2_n, int rounds, int classes, const double* angles,
                             const uint16_t* perms, uint32_t perm_mask, const float* x,
                             const uint16_t* cls, uint64_t count, double* energy, int threads);

/* The same two drivers with hoist_trig != 0: cos/sin of every angle are computed once per class
 * and direction (hygt_oracle_trig_pairs) instead of per butterfly and vector. Bit-identical
 * results (cos/sin are deterministic); used for the full-size checks. */
int hygt_oracle_apply_batch2(int log2_n, int rounds, int classes, const double* angles,
                             const uint16_t* perms, uint32_t perm_mask, const float* x,
                             const uint16_t* cls, uint64_t count, int inverse, double* y,
                             int threads, int hoist_trig);
int hygt_oracle_class_energy2(int log2_n, int rounds, int classes, const double* angles,
                              const uint16_t* perms, uint32_t perm_mask, const float* x,
                              const uint16_t* cls, uint64_t count, double* energy, int threads,
                              int hoist_trig);
void hygt_oracle_run_passes_cs(int log2_n, int rounds, const double* cs, double* x, int dir);
void hygt_oracle_trig_pairs(size_t count, const double* angles, int dir, double* cs);

/* ---- fixed point: fixedpoint.hpp:35-224 --------------------------------------------------- */
int hygt_oracle_trig_table(int angle_bits, int precision_bits, int32_t* cos_tab,
                           int32_t* sin_tab); /* fixedpoint.hpp:37-52 */
int hygt_oracle_quantize(const double* angles, size_t count, int angle_bits,
                         uint16_t* codes); /* fixedpoint.hpp:115-128 */
void hygt_oracle_dequantize(const uint16_t* codes, size_t count, int angle_bits,
                            double* angles); /* fixedpoint.hpp:131-137 */
/* Returns 0, 1 (ArgumentError: input |x| > 2^20) or 4 (OverflowError: |value| > 2^46).
 * perms/perm_mask as in the float chain; with only the final permutation this is exactly
 * forward_fixed/inverse_fixed. Input range is checked once per call on the call's input. */
int hygt_oracle_forward_fixed(int log2_n, int rounds, int angle_bits, int precision_bits,
                              const uint16_t* codes, const uint16_t* perms, uint32_t perm_mask,
                              int64_t* x);
int hygt_oracle_inverse_fixed(int log2_n, int rounds, int angle_bits, int precision_bits,
                              const uint16_t* codes, const uint16_t* perms, uint32_t perm_mask,
                              int64_t* x);
/* Batched fixed apply (hygt_main.cpp:155-165). Returns the status of the first failing row
 * (row order) and its index in *first_bad (or count if none); rows after it are still
 * computed where possible so outputs can be compared. */
int hygt_oracle_apply_batch_fixed(int log2_n, int rounds, int classes, int angle_bits,
                                  int precision_bits, const uint16_t* codes,
                                  const uint16_t* perms, uint32_t perm_mask, const int64_t* x,
                                  const uint16_t* cls, uint64_t count, int inverse, int64_t* y,
                                  uint64_t* first_bad, int threads);
size_t hygt_oracle_memory_footprint(int klt, int log2_n, int rounds,
                                    int num_transforms); /* fixedpoint.hpp:231-238 */

/* ---- KLT comparison path: statistics.hpp:222-224 -> matrix.hpp:70-80 ------------------------ */
/* y = K_c * x (inverse: K_c^T * x). K is [classes][N][N] row-major fp64. */
int hygt_oracle_klt_apply(int n, int classes, const double* k, const float* x,
                          const uint16_t* cls, uint64_t count, int inverse, double* y,
                          int threads);

/* ---- per-class correlation accumulation: statistics.hpp:63-99 ---------------- */
/* sum[c] += r r^T over the rows of class c (upper triangle accumulated in row order as
 * CorrelationAccumulator::add, :69-76, then mirrored), count[c] += rows; rows with a class id
 * >= classes return HYGT_ORACLE_ARGUMENT. phi = sum * (1 / count) as finalize (:81-94). */
int hygt_oracle_correlation(int log2_n, int classes, const float* x, const uint16_t* cls,
                            uint64_t count, double* sum, uint64_t* counts);
void hygt_oracle_correlation_finalize(int log2_n, const double* sum, uint64_t count, double* phi);

/* ---- coordinate-descent trainer: optimizer.hpp ------------------------------ */
typedef struct {
  int restarts;              /* OptimizerConfig::restarts (optimizer.hpp:37) */
  int max_sweeps;            /* :38 */
  double gain_tolerance_db;  /* :39 */
  uint64_t seed;             /* :40 */
  int init_mode;             /* :41, InitMode: 0 greedy_jacobi, 1 random, 2 zero */
} hygt_oracle_opt_config;
double hygt_oracle_coding_gain_db(const double* v, size_t n);              /* statistics.hpp:262-282 */
int hygt_oracle_jacobi_eigenvalues(const double* phi, int n, double* ev); /* statistics.hpp:141-199 */
void hygt_oracle_greedy_init(const double* phi, int log2_n, int rounds, double* angles); /* :150-166 */
/* optimize (optimizer.hpp:311-371): best angles [A], per-restart gains, best restart, KLT gain,
 * trajectories [restarts][max_sweeps + 1] (NaN padded; may be NULL) and their lengths. */
int hygt_oracle_optimize(const double* phi, int log2_n, int rounds, const hygt_oracle_opt_config* cfg,
                         double* angles_out, double* restart_gains, int* best_restart,
                         double* klt_gain, double* trajectories, int* traj_len);
/* diagonal of propagate_covariance(model, phi) (optimizer.hpp:111-124) */
void hygt_oracle_propagated_variances(const double* phi, int log2_n, int rounds,
                                      const double* angles, double* var);

/* ---- synthetic fixtures --------------------------------------------------- */
/* Seeded Fisher-Yates permutation as tests/oracles.hpp:94-100. */
void hygt_oracle_fisher_yates(hygt_oracle_rng* r, uint16_t* perm, int n);
/* Householder QR of a seeded n x n Gaussian; returns Q with diag(R) > 0 (row-major). */
void hygt_oracle_random_orthogonal(uint64_t seed, int n, double* q);

#ifdef __cplusplus
}
#endif
#endif
