/*
 * hygt_oracle.c -- TEST INFRASTRUCTURE ONLY (see hygt_oracle.h).
 *
 * A plain-C restatement of the reference's HyGT hot path. Reference paths are relative to
 * /root/reference/proj/include/hygt/ unless stated otherwise. This file is compiled into
 * oracle/liboracle.so by oracle/Makefile and loaded by tests through ctypes; the product
 * library never links it.
 */
#include "hygt_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define PI_D 3.14159265358979323846

/* ============================== RNG (rng.hpp) ============================================ */

/* rng.hpp:26-31 */
uint64_t hygt_oracle_splitmix64(uint64_t state) {
  uint64_t z = state + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* rng.hpp:36-38 */
uint64_t hygt_oracle_derive_seed(uint64_t base, uint64_t stream) {
  return hygt_oracle_splitmix64(base ^ hygt_oracle_splitmix64(stream + 1));
}

/* The reference wraps std::mt19937_64 (rng.hpp:46, 77). Its output is fixed by the C++
 * standard ([rand.eng.mers], [rand.predef]): w=64 n=312 m=156 r=31, a=0xB5026F5AA96619E9,
 * u=29 d=0x5555555555555555 s=17 b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43,
 * f=6364136223846793005. Restated here from that published definition. */
#define MT_N 312
#define MT_M 156
void hygt_oracle_rng_seed(hygt_oracle_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  r->spare = 0.0;
  r->have_spare = 0;
}

static void mt_twist(hygt_oracle_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
    uint64_t xa = x >> 1;
    if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t hygt_oracle_rng_next(hygt_oracle_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:49 */
double hygt_oracle_rng_uniform01(hygt_oracle_rng* r) {
  return (double)(hygt_oracle_rng_next(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:52 */
double hygt_oracle_rng_uniform(hygt_oracle_rng* r, double lo, double hi) {
  return lo + (hi - lo) * hygt_oracle_rng_uniform01(r);
}

/* rng.hpp:55-68: Box-Muller, second value cached. */
double hygt_oracle_rng_gaussian(hygt_oracle_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = hygt_oracle_rng_uniform01(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  const double u2 = hygt_oracle_rng_uniform01(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double a = 2.0 * PI_D * u2;
  r->spare = rr * sin(a);
  r->have_spare = 1;
  return rr * cos(a);
}

/* rng.hpp:71 */
uint64_t hygt_oracle_rng_below(hygt_oracle_rng* r, uint64_t bound) {
  return hygt_oracle_rng_next(r) % bound;
}

/* ============================== schedule / model ========================================= */

/* hypercube.hpp:59-77: m_j = j + (j & -k), n_j = m_j + k, k = 2^pass. */
int hygt_oracle_hypercube_indices(int log2_n, int pass, uint32_t* m, uint32_t* n) {
  if (log2_n < 1 || log2_n > 16) return HYGT_ORACLE_ARGUMENT;
  if (pass < 0 || pass >= log2_n) return HYGT_ORACLE_ARGUMENT;
  const uint32_t half = 1u << (log2_n - 1), k = 1u << pass;
  for (uint32_t j = 0; j < half; ++j) {
    m[j] = j + (j & (0u - k));
    n[j] = m[j] + k;
  }
  return HYGT_ORACLE_OK;
}

/* model.hpp:29-34 */
size_t hygt_oracle_num_parameters(int log2_n, int rounds) {
  if (log2_n < 1 || rounds < 1) return 0;
  return (size_t)rounds * ((size_t)1 << log2_n) * (size_t)log2_n / 2;
}

/* ============================== float transform ========================================== */

/* transform.hpp:45-66. dir > 0 forward (rounds 0..R-1, passes 0..n-1, +theta); otherwise the
 * exact reverse order with -theta. cos/sin are recomputed per butterfly as the reference does. */
void hygt_oracle_run_passes(int log2_n, int rounds, const double* angles, double* x, int dir) {
  const size_t half = (size_t)1 << (log2_n - 1);
  const int fwd = dir > 0;
  for (int step = 0; step < rounds * log2_n; ++step) {
    const int r = fwd ? step / log2_n : rounds - 1 - step / log2_n;
    const int p = fwd ? step % log2_n : log2_n - 1 - step % log2_n;
    const uint32_t k = 1u << p;
    const size_t base = ((size_t)r * log2_n + p) * half; /* model.hpp:77-79 */
    for (uint32_t j = 0; j < half; ++j) {
      const uint32_t m = j + (j & (0u - k));
      const uint32_t n = m + k;
      const double t = fwd ? angles[base + j] : -angles[base + j];
      const double c = cos(t), s = sin(t);
      const double a = x[m], b = x[n];
      x[m] = c * a + s * b;
      x[n] = c * b - s * a;
    }
  }
}

/* The same passes with (cos t, sin t) read from a table cs[A][2] computed once per class and
 * direction by hygt_oracle_trig_pairs (t = +theta forward, -theta inverse). cos and sin are
 * deterministic functions, so the result is bit-identical to hygt_oracle_run_passes; the batch
 * drivers use it ("hoisted trig") only to make full-size checks affordable, and
 * tests/test_oracle.py pins the two modes against each other. */
void hygt_oracle_run_passes_cs(int log2_n, int rounds, const double* cs, double* x, int dir) {
  const size_t half = (size_t)1 << (log2_n - 1);
  const int fwd = dir > 0;
  for (int step = 0; step < rounds * log2_n; ++step) {
    const int r = fwd ? step / log2_n : rounds - 1 - step / log2_n;
    const int p = fwd ? step % log2_n : log2_n - 1 - step % log2_n;
    const uint32_t k = 1u << p;
    const size_t base = ((size_t)r * log2_n + p) * half; /* model.hpp:77-79 */
    for (uint32_t j = 0; j < half; ++j) {
      const uint32_t m = j + (j & (0u - k));
      const uint32_t n = m + k;
      const double c = cs[2 * (base + j)], s = cs[2 * (base + j) + 1];
      const double a = x[m], b = x[n];
      x[m] = c * a + s * b;
      x[n] = c * b - s * a;
    }
  }
}

void hygt_oracle_trig_pairs(size_t count, const double* angles, int dir, double* cs) {
  for (size_t i = 0; i < count; ++i) {
    const double t = dir > 0 ? angles[i] : -angles[i];
    cs[2 * i] = cos(t);
    cs[2 * i + 1] = sin(t);
  }
}

static void oracle_gather(size_t n, const uint16_t* perm, double* x) {
  double local[256];
  double* heap = n <= 256 ? NULL : (double*)malloc(n * sizeof(double));
  double* buf = heap ? heap : local;
  memcpy(buf, x, n * sizeof(double));
  for (size_t i = 0; i < n; ++i) x[i] = buf[perm[i]];
  free(heap);
}

static void oracle_scatter(size_t n, const uint16_t* perm, double* x) {
  double local[256];
  double* heap = n <= 256 ? NULL : (double*)malloc(n * sizeof(double));
  double* buf = heap ? heap : local;
  memcpy(buf, x, n * sizeof(double));
  for (size_t i = 0; i < n; ++i) x[perm[i]] = buf[i];
  free(heap);
}

/* forward_chain / inverse_chain (below) with tabled trig: cs is the class's [A][2] table of the
 * direction. */
static void chain_cs(int log2_n, int rounds, const double* cs, const uint16_t* perms,
                     uint32_t perm_mask, double* x, int inverse) {
  const size_t n = (size_t)1 << log2_n;
  const size_t a1 = n / 2 * (size_t)log2_n;
  if (!inverse) {
    for (int r = 0; r < rounds; ++r) {
      hygt_oracle_run_passes_cs(log2_n, 1, cs + 2 * (size_t)r * a1, x, +1);
      if (perms && ((perm_mask >> r) & 1u)) oracle_gather(n, perms + (size_t)r * n, x);
    }
  } else {
    for (int r = rounds - 1; r >= 0; --r) {
      if (perms && ((perm_mask >> r) & 1u)) oracle_scatter(n, perms + (size_t)r * n, x);
      hygt_oracle_run_passes_cs(log2_n, 1, cs + 2 * (size_t)r * a1, x, -1);
    }
  }
}

/* transform.hpp:72-82: passes, then gather out[i] = pre[perm[i]]. */
void hygt_oracle_forward(int log2_n, int rounds, const double* angles, const uint16_t* perm,
                         double* x) {
  hygt_oracle_run_passes(log2_n, rounds, angles, x, +1);
  if (perm) {
    const size_t n = (size_t)1 << log2_n;
    double local[256];
    double* heap = n <= 256 ? NULL : (double*)malloc(n * sizeof(double));
    double* buf = heap ? heap : local;
    memcpy(buf, x, n * sizeof(double));
    for (size_t i = 0; i < n; ++i) x[i] = buf[perm[i]];
    free(heap);
  }
}

/* transform.hpp:86-96: scatter x[perm[i]] = y[i], then reverse passes with -theta. */
void hygt_oracle_inverse(int log2_n, int rounds, const double* angles, const uint16_t* perm,
                         double* x) {
  if (perm) {
    const size_t n = (size_t)1 << log2_n;
    double local[256];
    double* heap = n <= 256 ? NULL : (double*)malloc(n * sizeof(double));
    double* buf = heap ? heap : local;
    memcpy(buf, x, n * sizeof(double));
    for (size_t i = 0; i < n; ++i) x[perm[i]] = buf[i];
    free(heap);
  }
  hygt_oracle_run_passes(log2_n, rounds, angles, x, -1);
}

/* forward = forward(M_{R-1}, ... forward(M_0, x)), M_r single-round models over
 * the contiguous angle slice of round r (round-major layout, model.hpp:77-79). */
void hygt_oracle_forward_chain(int log2_n, int rounds, const double* angles,
                               const uint16_t* perms, uint32_t perm_mask, double* x) {
  const size_t n = (size_t)1 << log2_n;
  const size_t a1 = n / 2 * (size_t)log2_n;
  for (int r = 0; r < rounds; ++r) {
    const uint16_t* p = (perms && ((perm_mask >> r) & 1u)) ? perms + (size_t)r * n : NULL;
    hygt_oracle_forward(log2_n, 1, angles + (size_t)r * a1, p, x);
  }
}

/* inverse = inverse(M_0, ... inverse(M_{R-1}, y)). */
void hygt_oracle_inverse_chain(int log2_n, int rounds, const double* angles,
                               const uint16_t* perms, uint32_t perm_mask, double* x) {
  const size_t n = (size_t)1 << log2_n;
  const size_t a1 = n / 2 * (size_t)log2_n;
  for (int r = rounds - 1; r >= 0; --r) {
    const uint16_t* p = (perms && ((perm_mask >> r) & 1u)) ? perms + (size_t)r * n : NULL;
    hygt_oracle_inverse(log2_n, 1, angles + (size_t)r * a1, p, x);
  }
}

/* transform.hpp:100-117 (column j = forward(e_j)). */
void hygt_oracle_to_matrix(int log2_n, int rounds, const double* angles, const uint16_t* perms,
                           uint32_t perm_mask, double* t) {
  const size_t n = (size_t)1 << log2_n;
  double* e = (double*)malloc(n * sizeof(double));
  for (size_t j = 0; j < n; ++j) {
    memset(e, 0, n * sizeof(double));
    e[j] = 1.0;
    hygt_oracle_forward_chain(log2_n, rounds, angles, perms, perm_mask, e);
    for (size_t i = 0; i < n; ++i) t[i * n + j] = e[i];
  }
  free(e);
}

/* ============================== batched drivers ========================================== */

typedef struct {
  int log2_n, rounds, classes;
  const double* angles;
  const uint16_t* perms;
  uint32_t perm_mask;
  const float* x;
  const uint16_t* cls;
  uint64_t begin, end;
  int inverse;
  double* y;        /* apply: [count][N]; NULL for energy */
  double* energy;   /* energy: private [classes][N] accumulator */
  int bad;
  const double* cs; /* NULL: per-butterfly cos/sin; else [classes][A][2] tables (hoisted trig) */
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  const size_t n = (size_t)1 << j->log2_n;
  const size_t a = hygt_oracle_num_parameters(j->log2_n, j->rounds);
  double* v = (double*)malloc(n * sizeof(double));
  for (uint64_t row = j->begin; row < j->end; ++row) {
    const unsigned c = j->cls ? j->cls[row] : 0u;
    if ((int)c >= j->classes) {
      j->bad = 1;
      continue;
    }
    for (size_t i = 0; i < n; ++i) v[i] = (double)j->x[row * n + i]; /* dataset.hpp:106 */
    const double* ang = j->angles + (size_t)c * a;
    const uint16_t* pp = j->perms ? j->perms + (size_t)c * (size_t)j->rounds * n : NULL;
    if (j->cs)
      chain_cs(j->log2_n, j->rounds, j->cs + 2 * (size_t)c * a, pp, j->perm_mask, v, j->inverse);
    else if (j->inverse)
      hygt_oracle_inverse_chain(j->log2_n, j->rounds, ang, pp, j->perm_mask, v);
    else
      hygt_oracle_forward_chain(j->log2_n, j->rounds, ang, pp, j->perm_mask, v);
    if (j->y) memcpy(j->y + row * n, v, n * sizeof(double));
    if (j->energy)
      for (size_t i = 0; i < n; ++i) j->energy[c * n + i] += v[i] * v[i]; /* statistics.hpp:74 */
  }
  free(v);
  return NULL;
}

static int run_jobs(batch_job* proto, uint64_t count, int threads, int energy) {
  if (threads <= 0) threads = 1;
  if ((uint64_t)threads > count && count > 0) threads = (int)count;
  if (threads < 1) threads = 1;
  const size_t n = (size_t)1 << proto->log2_n;
  batch_job* jobs = (batch_job*)calloc((size_t)threads, sizeof(batch_job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t] = *proto;
    jobs[t].begin = count * (uint64_t)t / (uint64_t)threads;
    jobs[t].end = count * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].bad = 0;
    if (energy) jobs[t].energy = (double*)calloc((size_t)proto->classes * n, sizeof(double));
    pthread_create(&tid[t], NULL, batch_worker, &jobs[t]);
  }
  int bad = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    bad |= jobs[t].bad;
    if (energy) { /* shards merge by addition (statistics.hpp:110-120 for the sum form) */
      for (size_t i = 0; i < (size_t)proto->classes * n; ++i) proto->energy[i] += jobs[t].energy[i];
      free(jobs[t].energy);
    }
  }
  free(jobs);
  free(tid);
  return bad ? HYGT_ORACLE_ARGUMENT : HYGT_ORACLE_OK;
}

static double* class_tables(int log2_n, int rounds, int classes, const double* angles, int inverse) {
  const size_t a = hygt_oracle_num_parameters(log2_n, rounds);
  double* cs = (double*)malloc((size_t)classes * a * 2 * sizeof(double));
  if (cs) hygt_oracle_trig_pairs((size_t)classes * a, angles, inverse ? -1 : +1, cs);
  return cs;
}

int hygt_oracle_apply_batch2(int log2_n, int rounds, int classes, const double* angles,
                             const uint16_t* perms, uint32_t perm_mask, const float* x,
                             const uint16_t* cls, uint64_t count, int inverse, double* y,
                             int threads, int hoist_trig) {
  double* cs = hoist_trig ? class_tables(log2_n, rounds, classes, angles, inverse) : NULL;
  batch_job p = {log2_n, rounds, classes, angles, perms, perm_mask, x, cls, 0, count,
                 inverse, y, NULL, 0, cs};
  const int st = run_jobs(&p, count, threads, 0);
  free(cs);
  return st;
}

int hygt_oracle_apply_batch(int log2_n, int rounds, int classes, const double* angles,
                            const uint16_t* perms, uint32_t perm_mask, const float* x,
                            const uint16_t* cls, uint64_t count, int inverse, double* y,
                            int threads) {
  return hygt_oracle_apply_batch2(log2_n, rounds, classes, angles, perms, perm_mask, x, cls, count,
                                  inverse, y, threads, 0);
}

int hygt_oracle_class_energy2(int log2_n, int rounds, int classes, const double* angles,
                              const uint16_t* perms, uint32_t perm_mask, const float* x,
                              const uint16_t* cls, uint64_t count, double* energy, int threads,
                              int hoist_trig) {
  const size_t n = (size_t)1 << log2_n;
  memset(energy, 0, (size_t)classes * n * sizeof(double));
  double* cs = hoist_trig ? class_tables(log2_n, rounds, classes, angles, 0) : NULL;
  batch_job p = {log2_n, rounds, classes, angles, perms, perm_mask, x, cls, 0, count,
                 0, NULL, energy, 0, cs};
  const int st = run_jobs(&p, count, threads, 1);
  free(cs);
  return st;
}

int hygt_oracle_class_energy(int log2_n, int rounds, int classes, const double* angles,
                             const uint16_t* perms, uint32_t perm_mask, const float* x,
                             const uint16_t* cls, uint64_t count, double* energy, int threads) {
  return hygt_oracle_class_energy2(log2_n, rounds, classes, angles, perms, perm_mask, x, cls, count,
                                   energy, threads, 0);
}

/* ============================== correlation (f3) ========================================= */

/* CorrelationAccumulator::add (statistics.hpp:69-76): sum(i, j) += r_i * r_j for j >= i, in row
 * order, on the fp64 values of the fp32 samples (read_rblk widens them, dataset.hpp:106). */
int hygt_oracle_correlation(int log2_n, int classes, const float* x, const uint16_t* cls,
                            uint64_t count, double* sum, uint64_t* counts) {
  const size_t n = (size_t)1 << log2_n;
  for (uint64_t k = 0; k < count; ++k) {
    const int c = cls ? (int)cls[k] : 0;
    if (c >= classes) return HYGT_ORACLE_ARGUMENT;
    double* s = sum + (size_t)c * n * n;
    const float* r = x + k * n;
    for (size_t i = 0; i < n; ++i) {
      const double ri = (double)r[i];
      for (size_t j = i; j < n; ++j) s[i * n + j] += ri * (double)r[j];
    }
    counts[c] += 1;
  }
  for (int c = 0; c < classes; ++c) {  /* mirrored as finalize does (:86-91) */
    double* s = sum + (size_t)c * n * n;
    for (size_t i = 0; i < n; ++i)
      for (size_t j = i + 1; j < n; ++j) s[j * n + i] = s[i * n + j];
  }
  return HYGT_ORACLE_OK;
}

/* CorrelationAccumulator::finalize (statistics.hpp:81-94): phi(i, j) = sum(i, j) * (1 / count). */
void hygt_oracle_correlation_finalize(int log2_n, const double* sum, uint64_t count, double* phi) {
  const size_t n = (size_t)1 << log2_n;
  const double inv = 1.0 / (double)count;
  for (size_t i = 0; i < n * n; ++i) phi[i] = sum[i] * inv;
}

/* ============================== fixed point ============================================== */

/* fixedpoint.hpp:37-52: entries lround(cos/sin(2*pi*q/2^b) * 2^p). */
int hygt_oracle_trig_table(int angle_bits, int precision_bits, int32_t* cos_tab,
                           int32_t* sin_tab) {
  if (angle_bits < 1 || angle_bits > 12) return HYGT_ORACLE_ARGUMENT;
  if (precision_bits < 4 || precision_bits > 15) return HYGT_ORACLE_ARGUMENT;
  const size_t size = (size_t)1 << angle_bits;
  const double scale = (double)((int64_t)1 << precision_bits);
  for (size_t q = 0; q < size; ++q) {
    const double a = 2.0 * PI_D * (double)q / (double)size;
    cos_tab[q] = (int32_t)lround(cos(a) * scale);
    sin_tab[q] = (int32_t)lround(sin(a) * scale);
  }
  return HYGT_ORACLE_OK;
}

/* fixedpoint.hpp:115-128: code = llround(theta / 2pi * 2^b) mod 2^b, wrapped non-negative. */
int hygt_oracle_quantize(const double* angles, size_t count, int angle_bits, uint16_t* codes) {
  if (angle_bits < 1 || angle_bits > 12) return HYGT_ORACLE_ARGUMENT;
  const int64_t size = (int64_t)1 << angle_bits;
  for (size_t i = 0; i < count; ++i) {
    const double scaled = angles[i] / (2.0 * PI_D) * (double)size;
    int64_t q = llround(scaled) % size;
    if (q < 0) q += size;
    codes[i] = (uint16_t)q;
  }
  return HYGT_ORACLE_OK;
}

/* fixedpoint.hpp:131-137 */
void hygt_oracle_dequantize(const uint16_t* codes, size_t count, int angle_bits,
                            double* angles) {
  const double step = 2.0 * PI_D / (double)((int64_t)1 << angle_bits);
  for (size_t i = 0; i < count; ++i) angles[i] = step * (double)codes[i];
}

#define FIXED_INPUT_LIMIT ((int64_t)1 << 20) /* fixedpoint.hpp:142 */
#define FIXED_VALUE_LIMIT ((int64_t)1 << 46) /* fixedpoint.hpp:143 */

/* fixedpoint.hpp:154-182, one round r (all passes of that round) in the given direction. */
static int fixed_round(int log2_n, int r, int angle_bits, int p, const int32_t* ct,
                       const int32_t* st, const uint16_t* codes, int64_t* x, int fwd) {
  const size_t half = (size_t)1 << (log2_n - 1);
  const uint32_t mask = (1u << angle_bits) - 1u;
  const int64_t rnd = (int64_t)1 << (p - 1);
  for (int s = 0; s < log2_n; ++s) {
    const int d = fwd ? s : log2_n - 1 - s;
    const uint32_t k = 1u << d;
    const size_t base = ((size_t)r * log2_n + d) * half;
    for (uint32_t j = 0; j < half; ++j) {
      const uint32_t m = j + (j & (0u - k));
      const uint32_t n = m + k;
      uint32_t code = codes[base + j];
      if (!fwd) code = (0u - code) & mask; /* :170 */
      const int64_t c = ct[code], sn = st[code];
      const int64_t a = x[m], b = x[n];
      /* :175-176, arithmetic right shift of a signed int64 (as the reference relies on). */
      x[m] = (c * a + sn * b + rnd) >> p;
      x[n] = (c * b - sn * a + rnd) >> p;
      if (x[m] > FIXED_VALUE_LIMIT || x[m] < -FIXED_VALUE_LIMIT || x[n] > FIXED_VALUE_LIMIT ||
          x[n] < -FIXED_VALUE_LIMIT)
        return HYGT_ORACLE_OVERFLOW; /* :177-179 */
    }
  }
  return HYGT_ORACLE_OK;
}

static int fixed_check_input(const int64_t* x, size_t n) { /* fixedpoint.hpp:145-150 */
  for (size_t i = 0; i < n; ++i)
    if (x[i] > FIXED_INPUT_LIMIT || x[i] < -FIXED_INPUT_LIMIT) return HYGT_ORACLE_ARGUMENT;
  return HYGT_ORACLE_OK;
}

static int fixed_args_ok(int log2_n, int rounds, int angle_bits, int precision_bits) {
  return log2_n >= 1 && log2_n <= 16 && rounds >= 1 && angle_bits >= 1 && angle_bits <= 12 &&
         precision_bits >= 4 && precision_bits <= 15;
}

/* fixedpoint.hpp:191-205 generalised with inter-round gathers (same semantics as the float
 * chain; without inter-round permutations it is exactly forward_fixed). */
int hygt_oracle_forward_fixed(int log2_n, int rounds, int angle_bits, int precision_bits,
                              const uint16_t* codes, const uint16_t* perms, uint32_t perm_mask,
                              int64_t* x) {
  if (!fixed_args_ok(log2_n, rounds, angle_bits, precision_bits)) return HYGT_ORACLE_ARGUMENT;
  const size_t n = (size_t)1 << log2_n;
  int st = fixed_check_input(x, n);
  if (st) return st;
  int32_t ct[4096], sn[4096];
  hygt_oracle_trig_table(angle_bits, precision_bits, ct, sn);
  int64_t* tmp = (int64_t*)malloc(n * sizeof(int64_t));
  for (int r = 0; r < rounds && !st; ++r) {
    st = fixed_round(log2_n, r, angle_bits, precision_bits, ct, sn, codes, x, 1);
    if (!st && perms && ((perm_mask >> r) & 1u)) {
      const uint16_t* p = perms + (size_t)r * n;
      memcpy(tmp, x, n * sizeof(int64_t));
      for (size_t i = 0; i < n; ++i) x[i] = tmp[p[i]];
    }
  }
  free(tmp);
  return st;
}

/* fixedpoint.hpp:210-224: input check on the call's input (y), scatter, reverse passes. */
int hygt_oracle_inverse_fixed(int log2_n, int rounds, int angle_bits, int precision_bits,
                              const uint16_t* codes, const uint16_t* perms, uint32_t perm_mask,
                              int64_t* x) {
  if (!fixed_args_ok(log2_n, rounds, angle_bits, precision_bits)) return HYGT_ORACLE_ARGUMENT;
  const size_t n = (size_t)1 << log2_n;
  int st = fixed_check_input(x, n);
  if (st) return st;
  int32_t ct[4096], sn[4096];
  hygt_oracle_trig_table(angle_bits, precision_bits, ct, sn);
  int64_t* tmp = (int64_t*)malloc(n * sizeof(int64_t));
  for (int r = rounds - 1; r >= 0 && !st; --r) {
    if (perms && ((perm_mask >> r) & 1u)) {
      const uint16_t* p = perms + (size_t)r * n;
      memcpy(tmp, x, n * sizeof(int64_t));
      for (size_t i = 0; i < n; ++i) x[p[i]] = tmp[i];
    }
    st = fixed_round(log2_n, r, angle_bits, precision_bits, ct, sn, codes, x, 0);
  }
  free(tmp);
  return st;
}

int hygt_oracle_apply_batch_fixed(int log2_n, int rounds, int classes, int angle_bits,
                                  int precision_bits, const uint16_t* codes,
                                  const uint16_t* perms, uint32_t perm_mask, const int64_t* x,
                                  const uint16_t* cls, uint64_t count, int inverse, int64_t* y,
                                  uint64_t* first_bad, int threads) {
  (void)threads;
  const size_t n = (size_t)1 << log2_n;
  const size_t a = hygt_oracle_num_parameters(log2_n, rounds);
  int first = HYGT_ORACLE_OK;
  *first_bad = count;
  for (uint64_t row = 0; row < count; ++row) {
    const unsigned c = cls ? cls[row] : 0u;
    int64_t* v = y + row * n;
    memcpy(v, x + row * n, n * sizeof(int64_t));
    int st;
    if ((int)c >= classes) {
      st = HYGT_ORACLE_ARGUMENT;
    } else {
      const uint16_t* pp = perms ? perms + (size_t)c * (size_t)rounds * n : NULL;
      st = inverse ? hygt_oracle_inverse_fixed(log2_n, rounds, angle_bits, precision_bits,
                                               codes + (size_t)c * a, pp, perm_mask, v)
                   : hygt_oracle_forward_fixed(log2_n, rounds, angle_bits, precision_bits,
                                               codes + (size_t)c * a, pp, perm_mask, v);
    }
    if (st && first == HYGT_ORACLE_OK) {
      first = st;
      *first_bad = row;
    }
  }
  return first;
}

/* fixedpoint.hpp:231-238 */
size_t hygt_oracle_memory_footprint(int klt, int log2_n, int rounds, int num_transforms) {
  if (log2_n < 1 || rounds < 1 || num_transforms < 1) return 0;
  const size_t n = (size_t)1 << log2_n;
  if (klt) return (size_t)num_transforms * n * n;
  return (size_t)num_transforms * hygt_oracle_num_parameters(log2_n, rounds);
}

/* ============================== KLT ======================================================= */

/* statistics.hpp:222-224 -> matrix.hpp:70-80 (y_i = sum_j K_ij x_j); inverse uses K^T
 * (matrix.hpp:82-88). */
int hygt_oracle_klt_apply(int n, int classes, const double* k, const float* x,
                          const uint16_t* cls, uint64_t count, int inverse, double* y,
                          int threads) {
  (void)threads;
  for (uint64_t row = 0; row < count; ++row) {
    const unsigned c = cls ? cls[row] : 0u;
    if ((int)c >= classes) return HYGT_ORACLE_ARGUMENT;
    const double* kc = k + (size_t)c * n * n;
    const float* xv = x + row * (size_t)n;
    double* yv = y + row * (size_t)n;
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j)
        s += (inverse ? kc[(size_t)j * n + i] : kc[(size_t)i * n + j]) * (double)xv[j];
      yv[i] = s;
    }
  }
  return HYGT_ORACLE_OK;
}

/* ============================== fixtures ================================================= */

/* tests/oracles.hpp:94-100 */
void hygt_oracle_fisher_yates(hygt_oracle_rng* r, uint16_t* perm, int n) {
  for (int i = 0; i < n; ++i) perm[i] = (uint16_t)i;
  for (int i = n; i > 1; --i) {
    const int j = (int)hygt_oracle_rng_below(r, (uint64_t)i);
    const uint16_t t = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = t;
  }
}

/* Config 4 generator: Q of the Householder QR of a seeded Gaussian matrix,
 * signs fixed so diag(R) > 0. The reference has no QR; this is the textbook algorithm. */
void hygt_oracle_random_orthogonal(uint64_t seed, int n, double* q) {
  hygt_oracle_rng r;
  hygt_oracle_rng_seed(&r, seed);
  double* a = (double*)malloc((size_t)n * n * sizeof(double));
  double* v = (double*)malloc((size_t)n * sizeof(double));
  double* d = (double*)malloc((size_t)n * sizeof(double));
  for (int i = 0; i < n * n; ++i) a[i] = hygt_oracle_rng_gaussian(&r);
  /* q starts as identity; accumulate Q = H_0 H_1 ... H_{n-1}. */
  for (int i = 0; i < n * n; ++i) q[i] = 0.0;
  for (int i = 0; i < n; ++i) q[i * n + i] = 1.0;
  for (int k = 0; k < n; ++k) {
    double norm = 0.0;
    for (int i = k; i < n; ++i) norm += a[i * n + k] * a[i * n + k];
    norm = sqrt(norm);
    const double alpha = a[k * n + k] > 0 ? -norm : norm;
    for (int i = 0; i < n; ++i) v[i] = 0.0;
    for (int i = k; i < n; ++i) v[i] = a[i * n + k];
    v[k] -= alpha;
    double vn = 0.0;
    for (int i = k; i < n; ++i) vn += v[i] * v[i];
    if (vn == 0.0) {
      d[k] = alpha;
      continue;
    }
    /* A <- H A, H = I - 2 v v^T / (v^T v) */
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = k; i < n; ++i) s += v[i] * a[i * n + j];
      s = 2.0 * s / vn;
      for (int i = k; i < n; ++i) a[i * n + j] -= s * v[i];
    }
    /* Q <- Q H */
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = k; j < n; ++j) s += q[i * n + j] * v[j];
      s = 2.0 * s / vn;
      for (int j = k; j < n; ++j) q[i * n + j] -= s * v[j];
    }
    d[k] = a[k * n + k];
  }
  /* make diag(R) > 0: flip column k of Q where R_kk < 0 */
  for (int k = 0; k < n; ++k)
    if (d[k] < 0)
      for (int i = 0; i < n; ++i) q[i * n + k] = -q[i * n + k];
  free(a);
  free(v);
  free(d);
}

/* ============================ optimizer (optimizer.hpp) ================================== */
/* the coordinate-descent trainer, restated line by line so that the oracle takes
 * the same search path as the reference (same comparisons, same libm calls, no FMA
 * contraction at -O2 on x86-64). Matrices are n x n row-major. */

/* optimizer.hpp:55-71 (conjugate_pair): A <- G A G^T, rows first, then columns. */
static void opt_conjugate_pair(double* a, size_t dim, uint32_t m, uint32_t n, double c, double s) {
  double* row_m = a + (size_t)m * dim;
  double* row_n = a + (size_t)n * dim;
  for (size_t j = 0; j < dim; ++j) {
    const double am = row_m[j], an = row_n[j];
    row_m[j] = c * am + s * an;
    row_n[j] = c * an - s * am;
  }
  for (size_t i = 0; i < dim; ++i) {
    const double aim = a[i * dim + m], ain = a[i * dim + n];
    a[i * dim + m] = c * aim + s * ain;
    a[i * dim + n] = c * ain - s * aim;
  }
}

/* statistics.hpp:262-280 (coding_gain) over the diagonal of a (optimizer.hpp:100-105). */
double hygt_oracle_coding_gain_db(const double* v, size_t n) {
  double mean = 0.0;
  for (size_t i = 0; i < n; ++i) mean += v[i];
  mean /= (double)n;
  if (!(mean > 0.0)) return 0.0;
  const double floor_v = 1e-30 * mean;
  double log_sum = 0.0;
  for (size_t i = 0; i < n; ++i) log_sum += log10(v[i] > floor_v ? v[i] : floor_v);
  return 10.0 * (log10(mean) - log_sum / (double)n);
}

static double opt_gain_diag(const double* a, size_t dim, double* scratch) {
  for (size_t i = 0; i < dim; ++i) scratch[i] = a[i * dim + i];
  return hygt_oracle_coding_gain_db(scratch, dim);
}

/* optimizer.hpp:81-96 (pair_schedule): step t = (m, n); the angle index is t itself. */
static void opt_schedule(int log2_n, int rounds, uint32_t* sm, uint32_t* sn) {
  const uint32_t half = 1u << (log2_n - 1);
  size_t t = 0;
  for (int r = 0; r < rounds; ++r)
    for (int p = 0; p < log2_n; ++p) {
      const uint32_t k = 1u << p;
      for (uint32_t j = 0; j < half; ++j, ++t) {
        sm[t] = j + (j & (0u - k));
        sn[t] = sm[t] + k;
      }
    }
}

/* statistics.hpp:141-199 (jacobi_eigen): eigenvalues only (the rotation of `a` does not read
 * the eigenvector accumulator), sorted descending with ties in index order. Returns 0, or 3
 * (NumericalError) after 100 sweeps. */
int hygt_oracle_jacobi_eigenvalues(const double* phi, int n, double* ev) {
  double* a = (double*)malloc(sizeof(double) * (size_t)n * n);
  memcpy(a, phi, sizeof(double) * (size_t)n * n);
  double trace = 0.0;
  for (int i = 0; i < n; ++i) trace += phi[(size_t)i * n + i];
  const double at = fabs(trace);
  const double thresh = 1e-12 * (at > 1e-300 ? at : 1e-300);
  int sweep = 0;
  for (; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off = fmax(off, fabs(a[(size_t)p * n + q]));
    if (off < thresh) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[(size_t)p * n + q];
        if (fabs(apq) < thresh * 1e-4) continue;
        const double tau = (a[(size_t)q * n + q] - a[(size_t)p * n + p]) / (2.0 * apq);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(tau * tau + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        const double app = a[(size_t)p * n + p], aqq = a[(size_t)q * n + q];
        a[(size_t)p * n + p] = app - t * apq;
        a[(size_t)q * n + q] = aqq + t * apq;
        a[(size_t)p * n + q] = 0.0;
        a[(size_t)q * n + p] = 0.0;
        for (int r = 0; r < n; ++r) {
          if (r == p || r == q) continue;
          const double arp = a[(size_t)r * n + p], arq = a[(size_t)r * n + q];
          a[(size_t)r * n + p] = c * arp - s * arq;
          a[(size_t)p * n + r] = a[(size_t)r * n + p];
          a[(size_t)r * n + q] = c * arq + s * arp;
          a[(size_t)q * n + r] = a[(size_t)r * n + q];
        }
      }
  }
  for (int i = 0; i < n; ++i) ev[i] = a[(size_t)i * n + i];
  free(a);
  if (sweep == 100) return HYGT_ORACLE_NUMERICAL;
  /* stable descending insertion sort (std::stable_sort with '>' keeps equal keys in order) */
  for (int i = 1; i < n; ++i) {
    const double v = ev[i];
    int j = i - 1;
    while (j >= 0 && v > ev[j]) {
      ev[j + 1] = ev[j];
      --j;
    }
    ev[j + 1] = v;
  }
  return 0;
}

/* optimizer.hpp:150-166 (greedy_init) */
void hygt_oracle_greedy_init(const double* phi, int log2_n, int rounds, double* angles) {
  const size_t dim = (size_t)1 << log2_n, steps = (size_t)rounds * log2_n * (dim / 2);
  uint32_t* sm = (uint32_t*)malloc(sizeof(uint32_t) * steps);
  uint32_t* sn = (uint32_t*)malloc(sizeof(uint32_t) * steps);
  double* cov = (double*)malloc(sizeof(double) * dim * dim);
  opt_schedule(log2_n, rounds, sm, sn);
  memcpy(cov, phi, sizeof(double) * dim * dim);
  for (size_t t = 0; t < steps; ++t) {
    const uint32_t m = sm[t], n = sn[t];
    /* optimizer.hpp:144-146 (jacobi_angle) */
    const double th = 0.5 * atan2(2.0 * cov[m * dim + n], cov[m * dim + m] - cov[n * dim + n]);
    angles[t] = th;
    opt_conjugate_pair(cov, dim, m, n, cos(th), sin(th));
  }
  free(sm), free(sn), free(cov);
}

typedef struct {
  size_t dim, steps;
  const double* phi;
  uint32_t *sm, *sn;
  double *prefix, *work, *cs, *sn_, *diag;
} opt_engine;

/* optimizer.hpp:193-198 (full_gain) */
static double opt_full_gain(opt_engine* e, const double* angles) {
  memcpy(e->work, e->phi, sizeof(double) * e->dim * e->dim);
  for (size_t t = 0; t < e->steps; ++t)
    opt_conjugate_pair(e->work, e->dim, e->sm[t], e->sn[t], cos(angles[t]), sin(angles[t]));
  return opt_gain_diag(e->work, e->dim, e->diag);
}

/* optimizer.hpp:257-266 (candidate_gain) */
static double opt_candidate_gain(opt_engine* e, size_t t, double theta) {
  memcpy(e->work, e->prefix, sizeof(double) * e->dim * e->dim);
  opt_conjugate_pair(e->work, e->dim, e->sm[t], e->sn[t], cos(theta), sin(theta));
  for (size_t u = t + 1; u < e->steps; ++u)
    opt_conjugate_pair(e->work, e->dim, e->sm[u], e->sn[u], e->cs[u], e->sn_[u]);
  return opt_gain_diag(e->work, e->dim, e->diag);
}

/* optimizer.hpp:268-291 (golden_section) */
static double opt_golden(opt_engine* e, size_t t, double lo, double hi, double* gain) {
  const double ratio = 0.6180339887498949;
  double a = lo, b = hi;
  double c = b - ratio * (b - a), d = a + ratio * (b - a);
  double fc = opt_candidate_gain(e, t, c), fd = opt_candidate_gain(e, t, d);
  for (int it = 0; it < 28; ++it) {
    if (fc > fd) {
      b = d, d = c, fd = fc;
      c = b - ratio * (b - a);
      fc = opt_candidate_gain(e, t, c);
    } else {
      a = c, c = d, fc = fd;
      d = a + ratio * (b - a);
      fd = opt_candidate_gain(e, t, d);
    }
  }
  *gain = fc > fd ? fc : fd;
  return fc > fd ? c : d;
}

/* optimizer.hpp:201-244 (sweep) */
static double opt_sweep(opt_engine* e, double* angles) {
  for (size_t t = 0; t < e->steps; ++t) e->cs[t] = cos(angles[t]), e->sn_[t] = sin(angles[t]);
  memcpy(e->prefix, e->phi, sizeof(double) * e->dim * e->dim);
  for (size_t t = 0; t < e->steps; ++t) {
    double best_theta = angles[t];
    double best_gain = opt_candidate_gain(e, t, best_theta);
    const int grid = 33;
    double grid_best_theta = 0.0, grid_best_gain = -1.0;
    for (int g = 0; g < grid; ++g) {
      const double theta = PI_D * (double)g / grid;
      const double gain = opt_candidate_gain(e, t, theta);
      if (gain > grid_best_gain) grid_best_gain = gain, grid_best_theta = theta;
    }
    if (grid_best_gain > best_gain) best_gain = grid_best_gain, best_theta = grid_best_theta;
    const double delta = PI_D / grid;
    double ref_gain;
    const double ref_theta = opt_golden(e, t, grid_best_theta - delta, grid_best_theta + delta, &ref_gain);
    if (ref_gain > best_gain) best_gain = ref_gain, best_theta = ref_theta;
    if (best_theta != angles[t]) {
      angles[t] = best_theta;
      e->cs[t] = cos(best_theta);
      e->sn_[t] = sin(best_theta);
    }
    opt_conjugate_pair(e->prefix, e->dim, e->sm[t], e->sn[t], e->cs[t], e->sn_[t]);
  }
  return opt_gain_diag(e->prefix, e->dim, e->diag);
}

/* optimizer.hpp:311-371 (optimize). trajectories: [restarts][max_sweeps + 1] (NaN-padded),
 * traj_len: [restarts]. Returns 0, 1 (ArgumentError) or 3 (NumericalError from jacobi_eigen). */
int hygt_oracle_optimize(const double* phi, int log2_n, int rounds, const hygt_oracle_opt_config* cfg,
                         double* angles_out, double* restart_gains, int* best_restart,
                         double* klt_gain, double* trajectories, int* traj_len) {
  if (log2_n < 1 || log2_n > 16 || rounds < 1) return HYGT_ORACLE_ARGUMENT;
  if (cfg->restarts < 1 || cfg->max_sweeps < 1 || !(cfg->gain_tolerance_db > 0.0))
    return HYGT_ORACLE_ARGUMENT;
  const size_t dim = (size_t)1 << log2_n, steps = (size_t)rounds * log2_n * (dim / 2);
  double* ev = (double*)malloc(sizeof(double) * dim);
  int st = hygt_oracle_jacobi_eigenvalues(phi, (int)dim, ev);
  if (st) {
    free(ev);
    return st;
  }
  double trace = 0.0;
  for (size_t i = 0; i < dim; ++i) trace += phi[i * dim + i];
  const double eigen_floor = -1e-10 * fabs(trace);
  for (size_t i = 0; i < dim; ++i)
    if (ev[i] < eigen_floor) {
      free(ev);
      return HYGT_ORACLE_ARGUMENT; /* not positive semi-definite */
    }
  *klt_gain = hygt_oracle_coding_gain_db(ev, dim);
  free(ev);

  opt_engine e = {dim, steps, phi, NULL, NULL, NULL, NULL, NULL, NULL, NULL};
  e.sm = (uint32_t*)malloc(sizeof(uint32_t) * steps);
  e.sn = (uint32_t*)malloc(sizeof(uint32_t) * steps);
  e.prefix = (double*)malloc(sizeof(double) * dim * dim);
  e.work = (double*)malloc(sizeof(double) * dim * dim);
  e.cs = (double*)malloc(sizeof(double) * steps);
  e.sn_ = (double*)malloc(sizeof(double) * steps);
  e.diag = (double*)malloc(sizeof(double) * dim);
  opt_schedule(log2_n, rounds, e.sm, e.sn);
  double* angles = (double*)malloc(sizeof(double) * steps);
  double best_gain = 0.0;
  int have_best = 0;
  for (int r = 0; r < cfg->restarts; ++r) {
    if (r == 0 && cfg->init_mode == 0) {
      hygt_oracle_greedy_init(phi, log2_n, rounds, angles);
    } else if (r == 0 && cfg->init_mode == 2) {
      for (size_t t = 0; t < steps; ++t) angles[t] = 0.0;
    } else { /* optimizer.hpp:294-299 (random_angles) */
      hygt_oracle_rng g;
      hygt_oracle_rng_seed(&g, hygt_oracle_derive_seed(cfg->seed, (uint64_t)r));
      for (size_t t = 0; t < steps; ++t) angles[t] = hygt_oracle_rng_uniform(&g, 0.0, 2.0 * PI_D);
    }
    double* traj = trajectories ? trajectories + (size_t)r * (cfg->max_sweeps + 1) : NULL;
    int len = 0;
    double last = opt_full_gain(&e, angles);
    if (traj) traj[len] = last;
    ++len;
    for (int s = 0; s < cfg->max_sweeps; ++s) {
      const double gained = opt_sweep(&e, angles);
      const double improvement = gained - last;
      last = gained > last ? gained : last;
      if (traj) traj[len] = last;
      ++len;
      if (improvement < cfg->gain_tolerance_db) break;
    }
    if (traj)
      for (int k = len; k <= cfg->max_sweeps; ++k) traj[k] = NAN;
    if (traj_len) traj_len[r] = len;
    restart_gains[r] = last;
    if (!have_best || last > best_gain) {
      have_best = 1;
      best_gain = last;
      memcpy(angles_out, angles, sizeof(double) * steps);
      *best_restart = r;
    }
  }
  free(angles);
  free(e.sm), free(e.sn), free(e.prefix), free(e.work), free(e.cs), free(e.sn_), free(e.diag);
  return 0;
}

/* optimizer.hpp:111-124 (propagate_covariance, whole model, no permutation) -> diagonal. */
void hygt_oracle_propagated_variances(const double* phi, int log2_n, int rounds,
                                      const double* angles, double* var) {
  const size_t dim = (size_t)1 << log2_n, steps = (size_t)rounds * log2_n * (dim / 2);
  uint32_t* sm = (uint32_t*)malloc(sizeof(uint32_t) * steps);
  uint32_t* sn = (uint32_t*)malloc(sizeof(uint32_t) * steps);
  double* cov = (double*)malloc(sizeof(double) * dim * dim);
  opt_schedule(log2_n, rounds, sm, sn);
  memcpy(cov, phi, sizeof(double) * dim * dim);
  for (size_t t = 0; t < steps; ++t) opt_conjugate_pair(cov, dim, sm[t], sn[t], cos(angles[t]), sin(angles[t]));
  for (size_t i = 0; i < dim; ++i) var[i] = cov[i * dim + i];
  free(sm), free(sn), free(cov);
}
