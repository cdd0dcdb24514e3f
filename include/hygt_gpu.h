/*
 * hygt_gpu.h -- C ABI of the B200-native HyGT hot path (libhygt_gpu.so).
 *
 * This is the drop-in boundary for the reference's batched transform path. Each entry point
 * names the reference interface it replaces (paths relative to /root/reference/proj):
 *
 *   hygt_plan_create / hygt_plan_destroy
 *       <- hygt::HyGTModel (include/hygt/model.hpp:51-96), one per class, as cached by
 *          run_apply (tools/hygt_main.cpp:143-144; ModelBundle::dequantized, bundle.hpp:83-86).
 *   hygt_forward_f32 / hygt_inverse_f32
 *       <- hygt::forward / hygt::inverse (include/hygt/transform.hpp:72-96) applied per block
 *          with class dispatch, i.e. the loop of run_apply (tools/hygt_main.cpp:145-149).
 *   hygt_forward_energy_f32
 *       <- forward outputs folded into per-class CorrelationAccumulator diagonals
 *          (include/hygt/statistics.hpp:69-77) -- E[c][i] = sum_{v in c} y_v[i]^2.
 *   hygt_fixed_plan_create, hygt_forward_i64 / hygt_inverse_i64
 *       <- hygt::QuantizedHyGTModel + TrigTable + forward_fixed / inverse_fixed
 *          (include/hygt/fixedpoint.hpp:35-224), per block as tools/hygt_main.cpp:150-165.
 *   hygt_klt_plan_create, hygt_klt_forward_f32 / hygt_klt_inverse_f32
 *       <- hygt::klt_forward (include/hygt/statistics.hpp:222-224 -> matrix.hpp:70-80) and
 *          its transpose (matrix.hpp:82-88), per class.
 *   hygt_last_error
 *       <- the what() string of the exception the reference would have thrown.
 *
 * Conventions
 *   - All data pointers passed to the *_f32 / *_i64 calls are DEVICE pointers owned by the
 *     caller; the calls are asynchronous and stream-ordered on `stream` (a cudaStream_t, NULL =
 *     legacy default stream) unless documented otherwise.
 *   - Rows are contiguous: x[row * N + i]. Class ids are uint16 per row (dataset.hpp:32); NULL
 *     means every row is class 0.
 *   - Plans are immutable after creation and may be used concurrently from several host
 *     threads on different streams with distinct workspaces.
 *   - Status codes mirror the reference exception classes (errors.hpp:23-45, exit codes
 *     hygt_main.cpp:275-284): 0 ok, 1 ArgumentError, 2 IoError (reserved), 3 NumericalError,
 *     4 OverflowError (a NumericalError subclass in the reference), 5 CUDA runtime failure.
 */
#ifndef HYGT_GPU_H
#define HYGT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HYGT_OK 0
#define HYGT_ERR_ARGUMENT 1
#define HYGT_ERR_IO 2
#define HYGT_ERR_NUMERICAL 3
#define HYGT_ERR_OVERFLOW 4
#define HYGT_ERR_CUDA 5

/* hygt_plan_create flags */
#define HYGT_PLAN_FORCE_STANDARD 0x1u /* never use the scale-folded (fast Givens) form */
#define HYGT_PLAN_FORCE_FAST 0x2u     /* refuse (status 3) if the fast form is unsafe   */

/* call flags for the *_f32 transforms */
#define HYGT_REUSE_BUCKETS 0x1u /* workspace already holds hygt_bucket() output for d_cls */

typedef struct hygt_plan hygt_plan;
typedef struct hygt_klt_plan hygt_klt_plan;

/* Copies the message of the last failing call on this host thread into buf. Returns its
 * status. */
int hygt_last_error(char* buf, size_t len);

/* ---- float HyGT --------------------------------------------------------------------------
 * angles : host, [class_count][rounds * log2_n * 2^(log2_n-1)] fp64, application order
 *          (model.hpp:77-79).
 * perms  : host, [class_count][rounds][2^log2_n] uint16 or NULL. perms[c][r] is a gather
 *          applied after round r (out[i] = pre[perm[i]], transform.hpp:75-80) when bit r of
 *          perm_mask is set. Bit rounds-1 is the reference's final sorting permutation;
 *          lower bits are the inter-round permutations of the BASELINE configs. Every present
 *          permutation must be a bijection (model.hpp:37-44).
 * Supported on the GPU: 1 <= log2_n <= 8, rounds >= 1 (rounds <= 32 when perms are given),
 * 1 <= class_count <= 4096. */
int hygt_plan_create(int log2_n, int rounds, int class_count, const double* angles,
                     const uint16_t* perms, uint32_t perm_mask, uint32_t flags,
                     hygt_plan** out);

/* Plan-creation options (the library reads no environment variables). Zero-initialise, set
 * .size = sizeof(hygt_plan_options) and change the fields to override; NULL = all defaults. */
#define HYGT_KERNEL_AUTO 0      /* the measured-best kernel family for the shape */
#define HYGT_KERNEL_BUTTERFLY 1 /* rotation kernels only: the pass-by-pass butterfly form */
#define HYGT_KERNEL_TENSOR 2    /* the composed-operator tensor-core path (N = 64 / 128 / 256,
                                   <= 512 classes); HYGT_ERR_ARGUMENT for other shapes */
typedef struct hygt_plan_options {
  uint32_t size;       /* sizeof(hygt_plan_options) */
  int kernel;          /* HYGT_KERNEL_AUTO / _BUTTERFLY / _TENSOR */
  int allow_nvrtc;     /* 1 (default): plan-specialised kernels may be compiled with NVRTC at
                          plan creation (seconds per plan, cached per process); 0: precompiled
                          kernels only */
  int cta_pairs;       /* tensor-core path: 1 (default) CTA pairs (tcgen05 cta_group::2, M = 256,
                          each SM streams half of the class operator); 0 single CTAs */
  int stage_tile_rows; /* N = 16 staged kernel: rows per tile (multiple of 8 in [128, 1016]);
                          0 = sized to the shared memory (default) */
} hygt_plan_options;
/* hygt_plan_create with options (opts may be NULL). */
int hygt_plan_create_ex(int log2_n, int rounds, int class_count, const double* angles,
                        const uint16_t* perms, uint32_t perm_mask, uint32_t flags,
                        const hygt_plan_options* opts, hygt_plan** out);
int hygt_plan_destroy(hygt_plan* plan);
/* 0 = standard rotations, 1 = scale-folded (fast Givens) form chosen at plan time. */
int hygt_plan_algorithm(const hygt_plan* plan);
/* Largest max|x| per row for which the plan's arithmetic keeps every intermediate finite in
 * fp32 (the transform itself is orthogonal: outputs are bounded by sqrt(N) max|x|). The
 * scale-folded form divides by running cosine products sigma, so its limit is
 * 2^127 sigma_min / sqrt(N); plans take it only when that is >= 2^40, and
 * HYGT_PLAN_FORCE_STANDARD removes the limit (2^127 / sqrt(N)). */
double hygt_plan_input_limit(const hygt_plan* plan);
/* Kernel family serving the plan: 0 = bucketed apply kernel (hygt_bucket + per-row gather),
 * 1 = tile kernel (class sort inside each CTA, no bucketing pass; N <= 32),
 * 2 = class-segment kernel (global class buckets, one class table staged per CTA segment),
 * 3 = plan-specialised kernel compiled at plan creation (NVRTC, sm_100a; N <= 64): coefficients
 *     are instruction immediates and permutations register renames,
 * 4 = TMA-staged tile kernel (N = 16): tiles of rows moved HBM <-> shared memory by the bulk-copy
 *     engine, class-sorted in shared memory, no bucketing pass. Forward-with-energy calls run on
 *     the tile kernel instead,
 * 5 = thread-per-row kernel over global class buckets (N = 64): rows staged through shared
 *     memory by cp.async, class tables one segment at a time. Forward-with-energy calls run on
 *     the class-segment kernel instead,
 * 6 = one grid per class over global class buckets (N = 64, R <= 4, scale-folded form): the
 *     class's coefficients and gather offsets are kernel parameters (constant-bank operands),
 *     the class grids chained by programmatic dependent launch. Forward-with-energy calls run
 *     on the class-segment kernel instead,
 * 7 = the chain of 6 with one plan-specialised kernel per class and direction (NVRTC at plan
 *     creation, N = 32 / 64, R <= 8, >= 2 classes not served by 3): coefficients are FFMA
 *     immediates and permutations register renames, so the class's rows touch shared memory
 *     only on their way in and out. Forward-with-energy calls run on the tile / segment
 *     kernels instead,
 * 8 = the composed-operator tensor-core path (N = 64 / 128 / 256; the default at N = 128 / 256): the
 *     plan composes each class's rounds, passes and permutations into one N x N matrix (fp64)
 *     and the rows are transformed by a per-class grouped GEMM on tcgen05 (fp16 3-term split
 *     with per-row power-of-two scaling, fp32 accumulation in TMEM, CTA pairs), the per-class
 *     energy fused in its epilogue. */
int hygt_plan_path(const hygt_plan* plan);

/* Device workspace for class bucketing of `count` rows. The first word of a workspace is the
 * device-side error word that the kernels OR into and hygt_sync_status() reads and clears: a
 * workspace must be ZERO-INITIALISED (cudaMemset) before its first use, and may then be reused
 * by any number of stream-ordered calls. */
size_t hygt_workspace_bytes(const hygt_plan* plan, uint64_t count);
/* Groups rows by class (histogram + scan + scatter into the workspace). The transforms call it
 * themselves unless HYGT_REUSE_BUCKETS is passed. Invalid class ids are recorded and reported
 * by hygt_sync_status(). */
int hygt_bucket(const hygt_plan* plan, const uint16_t* d_cls, uint64_t count, void* d_ws,
                size_t ws_bytes, void* stream);
/* y = forward(x) row-wise (in place allowed). d_x and d_y must be aligned to min(16, 4N) bytes
 * (HYGT_ERR_ARGUMENT otherwise); class ids need no alignment. */
int hygt_forward_f32(const hygt_plan* plan, const float* d_x, float* d_y, const uint16_t* d_cls,
                     uint64_t count, void* d_ws, size_t ws_bytes, uint32_t flags, void* stream);
/* x = inverse(y) row-wise (in place allowed). */
int hygt_inverse_f32(const hygt_plan* plan, const float* d_y, float* d_x, const uint16_t* d_cls,
                     uint64_t count, void* d_ws, size_t ws_bytes, uint32_t flags, void* stream);
/* Forward plus fused per-class per-coefficient energy: d_energy[c][i] += sum y[row][i]^2 over
 * rows of class c (fp64, [class_count][N], caller zeroes it). */
int hygt_forward_energy_f32(const hygt_plan* plan, const float* d_x, float* d_y,
                            const uint16_t* d_cls, uint64_t count, double* d_energy, void* d_ws,
                            size_t ws_bytes, uint32_t flags, void* stream);
/* Synchronises `stream` and returns the first device-side error recorded by calls that used
 * this workspace (1 = a class id >= class_count), then clears it. */
int hygt_sync_status(const hygt_plan* plan, void* d_ws, void* stream);

/* ---- fixed-point HyGT (bit-exact with forward_fixed / inverse_fixed) ----------------------
 * codes: host [class_count][rounds * log2_n * 2^(log2_n-1)] uint16 (< 2^angle_bits).
 * perms/perm_mask as above. The calls are synchronous: they return the status of the first
 * failing row in row order (1 = |input| > 2^20, 4 = |intermediate| > 2^46) and write its
 * index to *first_bad (count if none). Rows are still transformed where possible. */
int hygt_fixed_plan_create(int log2_n, int rounds, int class_count, int angle_bits,
                           int precision_bits, const uint16_t* codes, const uint16_t* perms,
                           uint32_t perm_mask, hygt_plan** out);
/* The same with options (opts may be NULL; only allow_nvrtc applies to fixed-point plans). */
int hygt_fixed_plan_create_ex(int log2_n, int rounds, int class_count, int angle_bits,
                              int precision_bits, const uint16_t* codes, const uint16_t* perms,
                              uint32_t perm_mask, const hygt_plan_options* opts, hygt_plan** out);
int hygt_forward_i64(const hygt_plan* plan, const int64_t* d_x, int64_t* d_y,
                     const uint16_t* d_cls, uint64_t count, uint64_t* first_bad, void* stream);
int hygt_inverse_i64(const hygt_plan* plan, const int64_t* d_y, int64_t* d_x,
                     const uint16_t* d_cls, uint64_t count, uint64_t* first_bad, void* stream);

/* ---- per-class correlation accumulation -------------------------------------
 * <- hygt::CorrelationAccumulator::add / count (include/hygt/statistics.hpp:63-99), one per class
 *    as `hygt train` builds them (tools/hygt_main.cpp:85-87). Accumulates, stream-ordered:
 *    d_sum[c] += sum over rows of class c of r r^T (fp64, [C][N][N], full symmetric matrix) and
 *    d_count[c] += rows. Products of the fp32 samples are exact in fp64 and summed in fp64.
 *    finalize() is d_sum[c] / d_count[c]; shards merge by adding sums and counts
 *    (merge_correlation, statistics.hpp:110-120). Rows with a class id >= class_count are not
 *    counted and are reported by hygt_sync_status(NULL, d_ws, stream). log2_n in [2, 8]. */
size_t hygt_correlation_workspace_bytes(int class_count, uint64_t count);
int hygt_correlation_f64(int log2_n, int class_count, const float* d_x, const uint16_t* d_cls,
                         uint64_t count, double* d_sum, unsigned long long* d_count, void* d_ws,
                         size_t ws_bytes, void* stream);

/* ---- coordinate-descent trainer ----------------------------------------------
 * <- hygt::optimize(const CorrelationMatrix&, int log2_n, int rounds, const OptimizerConfig&)
 *    (include/hygt/optimizer.hpp:311-371), batched over `problems` covariances (one per class,
 *    as `hygt train` calls it, tools/hygt_main.cpp:93-99). The whole search -- greedy_init or
 *    random starts, coordinate-descent sweeps with the 33-point grid and golden-section line
 *    search, the tolerance rule -- runs on the device, one CTA per (problem, restart); the KLT
 *    gain (jacobi_eigen, statistics.hpp:141-199) is a device kernel too. Offline API: host
 *    buffers in and out, device memory allocated per call, returns when done.
 *    phi: [problems][N][N] fp64; seeds: per-problem OptimizerConfig::seed (NULL: cfg->seed);
 *    angles: [problems][A] the best restart's angles (A = rounds * log2_n * N / 2);
 *    restart_gains: [problems][restarts]; best_restart: [problems] (ties to the lowest index);
 *    klt_gain: [problems] or NULL; trajectories: [problems][restarts][max_sweeps + 1] (NaN
 *    padded) or NULL; trajectory_len: [problems][restarts] or NULL; variances: [problems][N]
 *    diagonal of propagate_covariance(best model, phi) (what variance_permutation sorts) or NULL.
 *    Errors as the reference: HYGT_ERR_ARGUMENT for restarts < 1, max_sweeps < 1, tolerance <= 0
 *    or a covariance that is not positive semi-definite; HYGT_ERR_NUMERICAL if jacobi_eigen does
 *    not converge. log2_n in [1, 8]. Gains match the reference to rounding. */
typedef struct hygt_optimize_config {
  int restarts;             /* OptimizerConfig::restarts (optimizer.hpp:37), default 4 */
  int max_sweeps;           /* :38, default 50 */
  double gain_tolerance_db; /* :39, default 1e-4 */
  uint64_t seed;            /* :40 */
  int init_mode;            /* :41 InitMode: 0 greedy_jacobi (default), 1 random, 2 zero */
} hygt_optimize_config;
int hygt_optimize_f64(int log2_n, int rounds, int problems, const double* phi,
                      const hygt_optimize_config* cfg, const uint64_t* seeds, double* angles,
                      double* restart_gains, int* best_restart, double* klt_gain,
                      double* trajectories, int* trajectory_len, double* variances, void* stream);

/* ---- dense per-class KLT (comparison path) ------------------------------------------------
 * k: host [class_count][n][n] fp64 row-major (rows = basis vectors, KLTResult::basis). */
int hygt_klt_plan_create(int n, int class_count, const double* k, uint32_t flags,
                         hygt_klt_plan** out);
int hygt_klt_plan_destroy(hygt_klt_plan* plan);
size_t hygt_klt_workspace_bytes(const hygt_klt_plan* plan, uint64_t count);
int hygt_klt_forward_f32(const hygt_klt_plan* plan, const float* d_x, float* d_y,
                         const uint16_t* d_cls, uint64_t count, void* d_ws, size_t ws_bytes,
                         void* stream);
int hygt_klt_inverse_f32(const hygt_klt_plan* plan, const float* d_y, float* d_x,
                         const uint16_t* d_cls, uint64_t count, void* d_ws, size_t ws_bytes,
                         void* stream);
/* The class dispatch of run_apply (hygt_main.cpp:143-149) is the same for both directions of a
 * batch: hygt_klt_bucket groups the rows once (as hygt_bucket does for HyGT plans), and the _ex
 * entry points take HYGT_REUSE_BUCKETS in `flags` to run on that grouping (tensor-core plans,
 * n >= 16; the flag is ignored by the SIMT kernel, which reads d_cls directly). */
int hygt_klt_bucket(const hygt_klt_plan* plan, const uint16_t* d_cls, uint64_t count, void* d_ws,
                    size_t ws_bytes, void* stream);
int hygt_klt_forward_f32_ex(const hygt_klt_plan* plan, const float* d_x, float* d_y,
                            const uint16_t* d_cls, uint64_t count, void* d_ws, size_t ws_bytes,
                            uint32_t flags, void* stream);
int hygt_klt_inverse_f32_ex(const hygt_klt_plan* plan, const float* d_y, float* d_x,
                            const uint16_t* d_cls, uint64_t count, void* d_ws, size_t ws_bytes,
                            uint32_t flags, void* stream);

/* ---- synthetic workloads, generated on the device -------------------------
 * Separable 2-D AR(1) rows (covariance sigma^2 * A (x) A, A_ij = rho^|i-j|, raster order,
 * statistics.hpp:287-305) with per-class rho (rho_per_class[cls[row]]), a fraction of rows
 * replaced by directional-edge patterns a*sign(...) + N(0, edge_noise^2). Counter-based
 * (Philox) so any row range is reproducible independently of the launch shape. */
int hygt_synth_rows_f32(float* d_x, uint64_t count, uint64_t row0, int block_size,
                        const uint16_t* d_cls, const float* d_rho_per_class, int class_count,
                        float sigma, float edge_fraction, float edge_amplitude,
                        float edge_noise, uint64_t seed, void* stream);
/* Uniform class ids in [0, class_count). */
int hygt_synth_classes(uint16_t* d_cls, uint64_t count, uint64_t row0, int class_count,
                       uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HYGT_GPU_H */
