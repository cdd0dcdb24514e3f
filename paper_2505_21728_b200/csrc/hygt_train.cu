// hygt_train.cu -- the coordinate-descent trainer on the GPU: optimize()
// (optimizer.hpp:311-371) with its per-angle line search (CoordinateDescent::sweep,
// candidate_gain, golden_section: optimizer.hpp:177-292), greedy_init (:150-166) and the KLT
// bound it reports (jacobi_eigen, statistics.hpp:141-199).
//
// Re-design. The reference scores a candidate angle theta at position t by copying the
// covariance propagated through [0, t) and conjugating it through every later position:
// O((A - t) N) per candidate, 64 candidates per position. Here each CTA keeps, for one
// (problem, restart):
//   F  = the covariance propagated through ALL positions at the current angles (N x N), and
//   WT = W_t^T, W_t = G_{A-1} ... G_{t+1} the tail after position t.
// Because G_t(theta) = G_t(delta) G_t(theta_cur) with delta = theta - theta_cur, the candidate's
// covariance is R F R^T with R = W_t G_t(delta) W_t^T = I + K D K^T, K = [a b] the columns m, n
// of W_t and D = [[c - 1, s], [-s, c - 1]]. Its diagonal is closed-form:
//   d_i = F_ii + 2 (al_i ya_i + be_i yb_i) + al_i^2 Zaa + 2 al_i be_i Zab + be_i^2 Zbb,
//   al_i = (c - 1) a_i - s b_i,  be_i = (c - 1) b_i + s a_i,  y = F K,  Z = K^T F K,
// so a candidate costs O(N) (one 16-lane group), a position costs two mat-vecs, and accepting a new
// angle is one symmetric rank-4 update of F. Advancing t peels G_{t+1} off the tail (two rows
// of WT). The search itself -- the current angle, the 33-point grid over [0, pi), 28
// golden-section steps around the best grid point, strict '>' comparisons, trajectory and
// tolerance rule -- is the reference's, step for step. At the end of every sweep F is rebuilt
// from phi by the reference's own conjugation sequence, so the drift of the rank-4 updates
// never crosses a sweep.
//
// Numerics: fp64 throughout. Candidate gains differ from the reference's by rounding only
// (~1e-14 relative); a near-tie in the search may then resolve the other way, so angles agree
// to the golden-section resolution and gains to a tolerance (tests/test_gpu_train.py), not
// bit for bit. The coding gain uses the product of frexp mantissas instead of a sum of log10s
// (same value to ~1e-15 relative).
//
// Layout: one CTA of 256 threads per (problem, restart). F and WT (row stride N + 1) live in
// shared memory up to N = 64 (66 KB); larger N uses a global (L2-resident) workspace.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/hygt_gpu.h"
#include "hygt_nvtx.h"

int hygt_set_error(int status, const char* msg);  // hygt_capi.cu

namespace {

constexpr int TT = 256;  // threads per CTA
constexpr int TW = TT / 32;
constexpr int GRID_POINTS = 33;                      // optimizer.hpp:210
constexpr int GOLDEN_ITERATIONS = 28;                // optimizer.hpp:270
constexpr double GOLDEN_RATIO = 0.6180339887498949;  // optimizer.hpp:269
constexpr double PI_D = 3.14159265358979323846;
constexpr double LOG10_2 = 0.30102999566398119521;
constexpr int SMEM_MAX_LOG2N = 6;
// Candidate evaluations run in groups of G(N) lanes (about 4-8 samples per lane), NG = TT / G
// of them in flight; the golden-section search resolves SPEC(N) iterations per round, which
// takes 2^(SPEC+1) - 2 <= NG speculative evaluations. Work is skipped per warp, never per group:
// groups without a point in a working warp evaluate a dummy one, so the full-mask shuffles
// never diverge.
template <int N>
__host__ __device__ constexpr int group_lanes() { return N <= 16 ? 4 : 16; }
template <int N>
__host__ __device__ constexpr int spec_depth() {
  int d = 1;
  while ((4 << d) - 2 <= TT / group_lanes<N>()) ++d;
  return d;
}
constexpr int KEY_SLOTS = 192;  // [0, 34) grid, [34, 36) golden start, 2 x tree banks of <= 62

struct TrainParams {
  const double* phi;   // [P][N][N]
  const double* init;  // [P][R][A] starting angles (restart 0 ignored when greedy)
  double* angles;      // [P][R][A] final angles per restart
  double* gains;       // [P][R]
  double* traj;        // [P][R][S + 1] (NaN padded)
  int* traj_len;       // [P][R]
  double* var;         // [P][R][N] propagated variances of the final angles
  double* ws;          // [P * R][2][N][N + 1] when F, WT do not fit in shared memory
  int rounds, restarts, max_sweeps;
  double tol;
  int greedy;  // restart 0 starts from greedy_init
};

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// Position t of the pair schedule (optimizer.hpp:81-96): pass p pairs m = j + (j & -2^p), m + 2^p.
template <int LOG2N>
__device__ __forceinline__ void step_pair(int t, int& m, int& n) {
  constexpr int HALF = 1 << (LOG2N - 1);
  const int j = t % HALF, k = 1 << ((t / HALF) % LOG2N);
  m = j + (j & -k);
  n = m + k;
}

// coding_gain (statistics.hpp:262-280) of N values, one warp; every lane returns the same value
// (xor butterflies combine commutatively).
template <int N, class V>
__device__ __forceinline__ double warp_coding_gain(V val, int lane) {
  constexpr int K = (N + 31) / 32;
  double x[K];
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = lane + 32 * k;
    x[k] = i < N ? val(i) : 0.0;
    sum += x[k];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double mean = sum / N;
  if (!(mean > 0.0)) return 0.0;
  const double floor_v = 1e-30 * mean;
  double mp = 1.0;
  int es = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (lane + 32 * k < N) {
      int e;
      mp *= frexp(x[k] > floor_v ? x[k] : floor_v, &e);
      es += e;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mp *= __shfl_xor_sync(0xffffffffu, mp, o);
    es += __shfl_xor_sync(0xffffffffu, es, o);
  }
  const double log_sum = log10(mp) + (double)es * LOG10_2;
  return 10.0 * (log10(mean) - log_sum / N);
}

// A product of positive values as exponent + mantissa in [0.5, 1): compares exactly.
struct Key {
  int e;
  double m;
};
// gain(a) > gain(b) <=> prod(a) < prod(b) (same trace)
__device__ __forceinline__ bool better(Key a, Key b) { return a.e < b.e || (a.e == b.e && a.m < b.m); }

// x = m * 2^e, m in [0.5, 1), for positive finite x: bit fields for normal values (the usual
// case), frexp for subnormals.
__device__ __forceinline__ double split_exp(double x, int& e) {
  const long long b = __double_as_longlong(x);
  const int f = (int)((b >> 52) & 0x7ff);
  if (f == 0) return frexp(x, &e);
  e = f - 1022;
  return __longlong_as_double((b & 0x800fffffffffffffll) | 0x3fe0000000000000ll);
}

// prod_i max(val(i), floor) over N values by a G-lane group, normalised. Every lane of the group
// returns the same key.
template <int N, class V>
__device__ __forceinline__ Key group_key(V val, int gl, double floor_v) {
  constexpr int G = group_lanes<N>();
  constexpr int K = (N + G - 1) / G;
  double mp = 1.0;
  int es = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = gl + G * k;
    if (i < N) {
      const double x = val(i);
      int e;
      mp *= split_exp(x > floor_v ? x : floor_v, e);
      es += e;
    }
  }
#pragma unroll
  for (int o = G / 2; o; o >>= 1) {
    mp *= __shfl_xor_sync(0xffffffffu, mp, o);
    es += __shfl_xor_sync(0xffffffffu, es, o);
  }
  int e2;
  mp = split_exp(mp, e2);
  return Key{es + e2, mp};
}

// A <- G A G^T on rows/columns m, n (conjugate_pair, optimizer.hpp:55-71): rows first, then
// columns, unfused products as the reference. Needs N <= TT; ends with a barrier.
template <int N>
__device__ __forceinline__ void conjugate(double* a, int m, int n, double c, double s) {
  constexpr int LD = N + 1;
  const int j = threadIdx.x;
  if (j < N) {
    const double am = a[m * LD + j], an = a[n * LD + j];
    a[m * LD + j] = da(dm(c, am), dm(s, an));
    a[n * LD + j] = ds(dm(c, an), dm(s, am));
  }
  __syncthreads();
  if (j < N) {
    const double aim = a[j * LD + m], ain = a[j * LD + n];
    a[j * LD + m] = da(dm(c, aim), dm(s, ain));
    a[j * LD + n] = ds(dm(c, ain), dm(s, aim));
  }
  __syncthreads();
}

template <int N>
__device__ __forceinline__ void load_matrix(double* a, const double* src) {
  constexpr int LD = N + 1;
  for (int e = threadIdx.x; e < N * N; e += TT) a[(e / N) * LD + e % N] = src[e];
  __syncthreads();
}

template <int LOG2N>
__global__ void __launch_bounds__(TT) hygt_train_kernel(const TrainParams P) {
  constexpr int N = 1 << LOG2N, LD = N + 1, Q = TT / N < N ? TT / N : N, JL = N / Q;
  extern __shared__ __align__(16) double sm[];
  constexpr int G = group_lanes<N>(), NG = TT / G, SPEC = spec_depth<N>();
  static_assert((2 << SPEC) - 2 <= NG && 36 + 2 * ((2 << SPEC) - 2) <= KEY_SLOTS, "key slots");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gid = tid / G, glane = tid % G;
  const int prob = blockIdx.x / P.restarts, rs = blockIdx.x % P.restarts;
  const int A = P.rounds * LOG2N * (N / 2);
  double *F, *X, *v;
  if (LOG2N <= SMEM_MAX_LOG2N) {
    F = sm;
    X = sm + N * LD;
    v = sm + 2 * N * LD;
  } else {
    F = P.ws + (size_t)blockIdx.x * 2 * N * LD;
    X = F + N * LD;
    v = sm;
  }
  double* ya = v;
  double* yb = v + N;
  double* fd = v + 2 * N;
  double* al = v + 3 * N;
  double* be = v + 4 * N;
  double* part = v + 5 * N;   // [2][TT] mat-vec partials
  double* km = part + 2 * TT;  // [KEY_SLOTS] candidate keys: mantissas (grid, golden start, tree)
  int* ke = reinterpret_cast<int*>(km + KEY_SLOTS);  // [KEY_SLOTS] exponents
  double* misc = km + KEY_SLOTS + KEY_SLOTS / 2;     // [1] gain of F
  const double* phi = P.phi + (size_t)prob * N * N;
  const size_t slot = (size_t)prob * P.restarts + rs;
  double* ang = P.angles + slot * A;

  // ---- starting angles: greedy_init (optimizer.hpp:150-166) or the host-drawn ones ----
  if (rs == 0 && P.greedy) {
    load_matrix<N>(F, phi);
    for (int t = 0; t < A; ++t) {
      int m, n;
      step_pair<LOG2N>(t, m, n);
      const double th = 0.5 * atan2(2.0 * F[m * LD + n], F[m * LD + m] - F[n * LD + n]);
      if (tid == 0) ang[t] = th;
      double s, c;
      sincos(th, &s, &c);
      conjugate<N>(F, m, n, c, s);
    }
  } else {
    for (int t = tid; t < A; t += TT) ang[t] = P.init[slot * A + t];
  }
  __syncthreads();

  // F <- phi propagated through every position (full_gain, optimizer.hpp:193-198); fd = diag.
  auto full_gain = [&]() -> double {
    load_matrix<N>(F, phi);
    for (int t = 0; t < A; ++t) {
      int m, n;
      step_pair<LOG2N>(t, m, n);
      double s, c;
      sincos(ang[t], &s, &c);
      conjugate<N>(F, m, n, c, s);
    }
    if (tid < N) fd[tid] = F[tid * LD + tid];
    __syncthreads();
    if (warp == 0) {
      const double g = warp_coding_gain<N>([&](int i) { return fd[i]; }, lane);
      if (lane == 0) misc[1] = g;
    }
    __syncthreads();
    return misc[1];
  };

  double* traj = P.traj + slot * (P.max_sweeps + 1);
  double last = full_gain();
  int len = 0;
  if (tid == 0) traj[len] = last;
  ++len;
  for (int sweep = 0; sweep < P.max_sweeps; ++sweep) {
    // WT_0 = G_1^T ... G_{A-1}^T, built right to left (rows m, n per factor).
    for (int e = tid; e < N * N; e += TT) X[(e / N) * LD + e % N] = (e / N == e % N) ? 1.0 : 0.0;
    __syncthreads();
    for (int u = A - 1; u >= 1; --u) {
      int m, n;
      step_pair<LOG2N>(u, m, n);
      double s, c;
      sincos(ang[u], &s, &c);
      if (tid < N) {
        const double xm = X[m * LD + tid], xn = X[n * LD + tid];
        X[m * LD + tid] = ds(dm(c, xm), dm(s, xn));
        X[n * LD + tid] = da(dm(s, xm), dm(c, xn));
      }
      __syncthreads();
    }
    for (int t = 0; t < A; ++t) {
      int m, n;
      step_pair<LOG2N>(t, m, n);
      const double* a = X + m * LD;  // column m of W_t
      const double* b = X + n * LD;
      const double cur = ang[t];
      // y = F [a b] (F symmetric: read columns so that lanes touch consecutive words)
      if (tid < N * Q) {
        const int i = tid % N, q = tid / N;
        double sa = 0.0, sb = 0.0;
#pragma unroll 4
        for (int jj = 0; jj < JL; ++jj) {
          const int j = q * JL + jj;
          const double f = F[j * LD + i];
          sa = fma(f, a[j], sa);
          sb = fma(f, b[j], sb);
        }
        part[tid] = sa;
        part[TT + tid] = sb;
      }
      __syncthreads();
      if (tid < N) {
        double sa = 0.0, sb = 0.0;
        for (int q = 0; q < Q; ++q) {
          sa += part[q * N + tid];
          sb += part[TT + q * N + tid];
        }
        ya[tid] = sa;
        yb[tid] = sb;
      }
      __syncthreads();
      // Z = K^T F K and the trace of F, per warp (identical in every warp)
      double zaa = 0.0, zab = 0.0, zbb = 0.0, tr = 0.0;
#pragma unroll
      for (int k = 0; k < (N + 31) / 32; ++k) {
        const int i = lane + 32 * k;
        if (i < N) {
          zaa = fma(a[i], ya[i], zaa);
          zab = fma(a[i], yb[i], zab);
          zbb = fma(b[i], yb[i], zbb);
          tr += fd[i];
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        zaa += __shfl_xor_sync(0xffffffffu, zaa, o);
        zab += __shfl_xor_sync(0xffffffffu, zab, o);
        zbb += __shfl_xor_sync(0xffffffffu, zbb, o);
        tr += __shfl_xor_sync(0xffffffffu, tr, o);
      }
      // The search compares gains of one position only. Every candidate's diagonal has the same
      // sum (the trace), so gain_a > gain_b <=> prod_i d_i(a) < prod_i d_i(b): candidates carry
      // the product as a normalised (exponent, mantissa) key and no logarithm is taken.
      const double mean = tr / N;
      const bool degenerate = !(mean > 0.0);  // coding_gain returns 0 for every candidate
      const double floor_v = 1e-30 * mean;
      // candidate_gain(t, theta) in closed form (see the header), one 16-lane group
      auto cand = [&](double theta) -> Key {
        double sh, ch;
        sincos(0.5 * (theta - cur), &sh, &ch);
        const double c1 = -2.0 * sh * sh, s = 2.0 * sh * ch;
        const Key k = group_key<N>(
            [&](int i) {
              const double ai = a[i], bi = b[i];
              const double p = c1 * ai - s * bi, r = c1 * bi + s * ai;
              return fd[i] + 2.0 * (p * ya[i] + r * yb[i]) + p * p * zaa + 2.0 * p * r * zab + r * r * zbb;
            },
            glane, floor_v);
        return degenerate ? Key{0, 0.5} : k;
      };
      // the current angle and the 33-point grid (optimizer.hpp:205-221)
      constexpr int GPW = 32 / G;  // groups per warp; a warp works if any of its groups has a point
      for (int k0 = 0; k0 <= GRID_POINTS; k0 += NG) {
        const int k = k0 + gid;
        if (k0 + warp * GPW > GRID_POINTS) continue;
        const double th = k == 0 || k > GRID_POINTS ? cur : PI_D * static_cast<double>(k - 1) / GRID_POINTS;
        const Key g = cand(th);
        if (glane == 0 && k <= GRID_POINTS) {
          ke[k] = g.e;
          km[k] = g.m;
        }
      }
      __syncthreads();
      // every thread resolves the search identically from shared memory
      Key best_key{ke[0], km[0]};
      double best_theta = cur;
      Key grid_key{INT_MAX, 1.0};  // worse than any candidate (grid_best_gain = -1)
      double grid_theta = 0.0;
      for (int g = 0; g < GRID_POINTS; ++g)
        if (better(Key{ke[g + 1], km[g + 1]}, grid_key)) {
          grid_key = Key{ke[g + 1], km[g + 1]};
          grid_theta = PI_D * static_cast<double>(g) / GRID_POINTS;
        }
      if (better(grid_key, best_key)) {
        best_key = grid_key;
        best_theta = grid_theta;
      }
      // golden_section (optimizer.hpp:268-291), SPEC iterations per round: the groups evaluate
      // every point the next SPEC iterations can reach (heap nodes 1..2^(SPEC+1) - 2; node h's
      // children are 2h + 1 for fc > fd and 2h + 2 otherwise), then all threads replay the
      // iterations with the reference's comparisons.
      const double delta = PI_D / GRID_POINTS;
      double lo = grid_theta - delta, hi = grid_theta + delta;
      double c = hi - GOLDEN_RATIO * (hi - lo), d = lo + GOLDEN_RATIO * (hi - lo);
      if (warp * GPW < 2) {
        const Key g = cand(gid == 0 ? c : d);
        if (glane == 0 && gid < 2) {
          ke[GRID_POINTS + 1 + gid] = g.e;
          km[GRID_POINTS + 1 + gid] = g.m;
        }
      }
      __syncthreads();
      Key fc{ke[GRID_POINTS + 1], km[GRID_POINTS + 1]}, fdk{ke[GRID_POINTS + 2], km[GRID_POINTS + 2]};
      for (int it = 0, bank = 0; it < GOLDEN_ITERATIONS; bank ^= 1) {
        const int depth = GOLDEN_ITERATIONS - it < SPEC ? GOLDEN_ITERATIONS - it : SPEC;
        const int nodes = (2 << depth) - 2;
        const int base = GRID_POINTS + 3 + bank * ((2 << SPEC) - 2);  // alternate banks: no WAR barrier
        if (warp * GPW < nodes) {
          int h = gid < nodes ? gid + 1 : 0, path = 0, len = 0;
          while (h > 0) {  // branches from the root, last one in bit 0
            path |= ((h & 1) ? 0 : 1) << len;
            ++len;
            h = (h - 1) >> 1;
          }
          double l2 = lo, h2 = hi, c2 = c, d2 = d, pt = cur;
          for (int q = len - 1; q >= 0; --q) {
            if (!((path >> q) & 1)) {  // fc > fd
              h2 = d2;
              d2 = c2;
              c2 = h2 - GOLDEN_RATIO * (h2 - l2);
              pt = c2;
            } else {
              l2 = c2;
              c2 = d2;
              d2 = l2 + GOLDEN_RATIO * (h2 - l2);
              pt = d2;
            }
          }
          const Key g = cand(pt);
          if (glane == 0 && gid < nodes) {
            ke[base + gid] = g.e;
            km[base + gid] = g.m;
          }
        }
        __syncthreads();
        int h = 0;
        for (int q = 0; q < depth; ++q) {
          if (better(fc, fdk)) {
            hi = d;
            d = c;
            fdk = fc;
            c = hi - GOLDEN_RATIO * (hi - lo);
            h = 2 * h + 1;
            fc = Key{ke[base + h - 1], km[base + h - 1]};
          } else {
            lo = c;
            c = d;
            fc = fdk;
            d = lo + GOLDEN_RATIO * (hi - lo);
            h = 2 * h + 2;
            fdk = Key{ke[base + h - 1], km[base + h - 1]};
          }
        }
        it += depth;
      }
      {
        const bool cwin = better(fc, fdk);
        if (better(cwin ? fc : fdk, best_key)) best_theta = cwin ? c : d;
      }
      const double best = best_theta;
      if (best != cur) {  // accept: F <- R F R^T, a symmetric rank-4 update
        double sh, ch;
        sincos(0.5 * (best - cur), &sh, &ch);
        const double c1 = -2.0 * sh * sh, s = 2.0 * sh * ch;
        if (tid < N) {
          al[tid] = c1 * a[tid] - s * b[tid];
          be[tid] = c1 * b[tid] + s * a[tid];
        }
        __syncthreads();
        for (int e = tid; e < N * N; e += TT) {
          const int i = e / N, j = e % N;
          const double ai = al[i], bi = be[i], aj = al[j], bj = be[j];
          const double t1 = da(dm(ai, ya[j]), dm(ya[i], aj));
          const double t2 = da(dm(bi, yb[j]), dm(yb[i], bj));
          const double t3 = da(da(dm(dm(ai, aj), zaa), dm(da(dm(ai, bj), dm(bi, aj)), zab)), dm(dm(bi, bj), zbb));
          F[i * LD + j] = da(da(F[i * LD + j], da(t1, t2)), t3);
        }
        __syncthreads();
        if (tid < N) fd[tid] = F[tid * LD + tid];
        if (tid == 0) ang[t] = best;
      }
      // W_{t+1} = W_t G_{t+1}^T: rows m', n' of WT (the angle at t + 1 is still the old one)
      if (t + 1 < A) {
        int m2, n2;
        step_pair<LOG2N>(t + 1, m2, n2);
        double s, c;
        sincos(ang[t + 1], &s, &c);
        if (tid < N) {
          const double xm = X[m2 * LD + tid], xn = X[n2 * LD + tid];
          X[m2 * LD + tid] = da(dm(c, xm), dm(s, xn));
          X[n2 * LD + tid] = ds(dm(c, xn), dm(s, xm));
        }
      }
      __syncthreads();
    }
    const double gained = full_gain();  // the sweep's return value (optimizer.hpp:243)
    const double improvement = gained - last;
    last = gained > last ? gained : last;
    if (tid == 0) traj[len] = last;
    ++len;
    if (improvement < P.tol) break;
  }
  if (tid == 0) {
    for (int k = len; k <= P.max_sweeps; ++k) traj[k] = __longlong_as_double(0x7ff8000000000000ll);
    P.traj_len[slot] = len;
    P.gains[slot] = last;
  }
  if (tid < N) P.var[slot * N + tid] = fd[tid];
}

// jacobi_eigen (statistics.hpp:141-199) as a parallel cyclic Jacobi: each sweep is N - 1
// round-robin steps of N / 2 disjoint rotations (the reference's rotation formula and skip
// rule), applied as A <- J^T A J in a column phase and a row phase. Only the eigenvalues are
// kept; thread 0 sorts them (stable, descending) and takes their coding gain in the
// reference's order. status: 0, 1 (not positive semi-definite), 3 (no convergence).
template <int LOG2N>
__global__ void __launch_bounds__(TT) hygt_klt_gain_kernel(const double* phi_all, double* ws, double* klt,
                                                           int* status) {
  constexpr int N = 1 << LOG2N, LD = N + 1, H = N / 2;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  double* a = LOG2N <= SMEM_MAX_LOG2N ? sm : ws + (size_t)blockIdx.x * N * LD;
  double* v = LOG2N <= SMEM_MAX_LOG2N ? sm + N * LD : sm;
  double* pc = v;          // [H] c
  double* ps = v + H;      // [H] s
  double* pd = v + 2 * H;  // [2H] new diagonal pair
  double* red = v + 4 * H; // [TW]
  int* pp = reinterpret_cast<int*>(red + TW);  // [H] p, [H] q, [H] active
  int* pq = pp + H;
  int* pa = pq + H;
  const double* phi = phi_all + (size_t)blockIdx.x * N * N;
  load_matrix<N>(a, phi);
  double trace = 0.0;
  for (int i = 0; i < N; ++i) trace += a[i * LD + i];
  const double at = fabs(trace);
  const double thresh = 1e-12 * (at > 1e-300 ? at : 1e-300);
  int sweep = 0;
  for (; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int e = tid; e < N * N; e += TT) {
      const int p = e / N, q = e % N;
      if (q > p) off = fmax(off, fabs(a[p * LD + q]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
    if ((tid & 31) == 0) red[tid >> 5] = off;
    __syncthreads();
    off = 0.0;
    for (int w = 0; w < TW; ++w) off = fmax(off, red[w]);
    __syncthreads();
    if (off < thresh) break;
    for (int k = 0; k < N - 1; ++k) {
      if (tid < H) {
        const int x = tid == 0 ? 0 : (tid - 1 + k) % (N - 1) + 1;
        const int y = (N - 2 - tid + k) % (N - 1) + 1;
        const int p = x < y ? x : y, q = x < y ? y : x;
        const double apq = a[p * LD + q];
        pp[tid] = p;
        pq[tid] = q;
        pa[tid] = fabs(apq) >= thresh * 1e-4;
        if (pa[tid]) {
          const double tau = (a[q * LD + q] - a[p * LD + p]) / (2.0 * apq);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(tau * tau + 1.0));
          const double c = 1.0 / sqrt(t * t + 1.0);
          pc[tid] = c;
          ps[tid] = t * c;
          pd[2 * tid] = a[p * LD + p] - t * apq;
          pd[2 * tid + 1] = a[q * LD + q] + t * apq;
        }
      }
      __syncthreads();
      for (int e = tid; e < N * H; e += TT) {  // columns: A <- A J
        const int r = e / H, i = e % H;
        if (!pa[i]) continue;
        const int p = pp[i], q = pq[i];
        const double c = pc[i], s = ps[i], arp = a[r * LD + p], arq = a[r * LD + q];
        a[r * LD + p] = c * arp - s * arq;
        a[r * LD + q] = c * arq + s * arp;
      }
      __syncthreads();
      for (int e = tid; e < H * N; e += TT) {  // rows: A <- J^T A
        const int i = e / N, r = e % N;
        if (!pa[i]) continue;
        const int p = pp[i], q = pq[i];
        const double c = pc[i], s = ps[i], apr = a[p * LD + r], aqr = a[q * LD + r];
        a[p * LD + r] = c * apr - s * aqr;
        a[q * LD + r] = c * aqr + s * apr;
      }
      __syncthreads();
      if (tid < H && pa[tid]) {
        const int p = pp[tid], q = pq[tid];
        a[p * LD + p] = pd[2 * tid];
        a[q * LD + q] = pd[2 * tid + 1];
        a[p * LD + q] = 0.0;
        a[q * LD + p] = 0.0;
      }
      __syncthreads();
    }
  }
  if (tid != 0) return;
  if (sweep == 100) {
    status[blockIdx.x] = HYGT_ERR_NUMERICAL;
    return;
  }
  double* ev = v;  // reuse: N values
  for (int i = 0; i < N; ++i) ev[i] = a[i * LD + i];
  const double floor_ev = -1e-10 * at;
  for (int i = 0; i < N; ++i)
    if (ev[i] < floor_ev) {
      status[blockIdx.x] = HYGT_ERR_ARGUMENT;
      return;
    }
  for (int i = 1; i < N; ++i) {  // stable descending
    const double x = ev[i];
    int j = i - 1;
    while (j >= 0 && x > ev[j]) {
      ev[j + 1] = ev[j];
      --j;
    }
    ev[j + 1] = x;
  }
  double mean = 0.0;
  for (int i = 0; i < N; ++i) mean += ev[i];
  mean /= N;
  double g = 0.0;
  if (mean > 0.0) {
    const double fl = 1e-30 * mean;
    double ls = 0.0;
    for (int i = 0; i < N; ++i) ls += log10(ev[i] > fl ? ev[i] : fl);
    g = 10.0 * (log10(mean) - ls / N);
  }
  klt[blockIdx.x] = g;
  status[blockIdx.x] = 0;
}

using TrainFn = void (*)(const TrainParams);
using KltFn = void (*)(const double*, double*, double*, int*);

template <int L>
void pick(int log2n, TrainFn& t, KltFn& k) {
  if (log2n == L) {
    t = hygt_train_kernel<L>;
    k = hygt_klt_gain_kernel<L>;
  }
  if constexpr (L < 8) pick<L + 1>(log2n, t, k);
}

size_t train_smem(int log2n) {
  const size_t n = size_t{1} << log2n;
  const size_t mats = log2n <= SMEM_MAX_LOG2N ? 2 * n * (n + 1) : 0;
  return (mats + 5 * n + 2 * TT + KEY_SLOTS + KEY_SLOTS / 2 + 8) * sizeof(double);
}

size_t klt_smem(int log2n) {
  const size_t n = size_t{1} << log2n;
  const size_t mats = log2n <= SMEM_MAX_LOG2N ? n * (n + 1) : 0;
  return (mats + 2 * n + TW) * sizeof(double) + 3 * (n / 2) * sizeof(int) + 16;
}

// derive_seed (rng.hpp:36-38) and uniform(0, 2 pi) draws of random_angles (optimizer.hpp:294-299)
uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* get() const { return static_cast<T*>(p); }
};

}  // namespace

extern "C" int hygt_optimize_f64(int log2_n, int rounds, int problems, const double* phi,
                                 const hygt_optimize_config* cfg, const uint64_t* seeds, double* angles,
                                 double* restart_gains, int* best_restart, double* klt_gain,
                                 double* trajectories, int* trajectory_len, double* variances,
                                 void* stream) {
  HYGT_NVTX("hygt_optimize_f64");
  if (log2_n < 1 || log2_n > 8)
    return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_optimize_f64: log2_n must be in [1, 8]");
  if (rounds < 1 || problems < 1 || !phi || !cfg || !angles || !restart_gains || !best_restart)
    return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_optimize_f64: bad rounds/problems or null pointer");
  if (cfg->restarts < 1) return hygt_set_error(HYGT_ERR_ARGUMENT, "optimize: restarts must be >= 1");
  if (cfg->max_sweeps < 1) return hygt_set_error(HYGT_ERR_ARGUMENT, "optimize: max_sweeps must be >= 1");
  if (!(cfg->gain_tolerance_db > 0.0))
    return hygt_set_error(HYGT_ERR_ARGUMENT, "optimize: gain_tolerance_db must be positive");
  if (cfg->init_mode < 0 || cfg->init_mode > 2)
    return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_optimize_f64: init_mode must be 0, 1 or 2");
  const int R = cfg->restarts, S = cfg->max_sweeps;
  const size_t n = size_t{1} << log2_n, A = (size_t)rounds * log2_n * (n / 2), PR = (size_t)problems * R;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TrainFn tk = nullptr;
  KltFn kk = nullptr;
  pick<1>(log2_n, tk, kk);

  // starting angles: restart 0 greedy / zero / random, the others random (optimizer.hpp:329-344)
  std::vector<double> init(PR * A, 0.0);
  for (int p = 0; p < problems; ++p) {
    const uint64_t seed = seeds ? seeds[p] : cfg->seed;
    for (int r = 0; r < R; ++r) {
      if (r == 0 && cfg->init_mode != 1) continue;
      std::mt19937_64 gen(splitmix64(seed ^ splitmix64((uint64_t)r + 1)));
      double* dst = init.data() + ((size_t)p * R + r) * A;
      for (size_t t = 0; t < A; ++t)
        dst[t] = 0.0 + (2.0 * PI_D - 0.0) * (static_cast<double>(gen() >> 11) * 0x1.0p-53);
    }
  }

  const size_t ld = n + 1;
  const size_t ws_train = log2_n > SMEM_MAX_LOG2N ? PR * 2 * n * ld : 0;
  const size_t ws_klt = log2_n > SMEM_MAX_LOG2N ? (size_t)problems * n * ld : 0;
  const size_t bytes[] = {(size_t)problems * n * n * 8, PR * A * 8, PR * A * 8, PR * 8, PR * (S + 1) * 8,
                          PR * 4, PR * n * 8, std::max(ws_train, ws_klt) * 8 + 8, (size_t)problems * 8,
                          (size_t)problems * 4};
  DevBuf buf[10];
  for (int i = 0; i < 10; ++i)
    if (cudaMalloc(&buf[i].p, bytes[i]) != cudaSuccess) {
      cudaGetLastError();
      return hygt_set_error(HYGT_ERR_CUDA, "hygt_optimize_f64: device allocation failed");
    }
  cudaMemcpyAsync(buf[0].p, phi, bytes[0], cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(buf[1].p, init.data(), bytes[1], cudaMemcpyHostToDevice, st);

  // the KLT bound first: the reference validates the covariance before optimizing (:321-326)
  const size_t ks = klt_smem(log2_n), ts = train_smem(log2_n);
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ks);
  cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ts);
  kk<<<problems, TT, ks, st>>>(buf[0].get<double>(), buf[7].get<double>(), buf[8].get<double>(),
                                buf[9].get<int>());
  std::vector<int> status(problems);
  std::vector<double> klt(problems);
  cudaMemcpyAsync(status.data(), buf[9].p, bytes[9], cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(klt.data(), buf[8].p, bytes[8], cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return hygt_set_error(HYGT_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  for (int p = 0; p < problems; ++p) {
    if (status[p] == HYGT_ERR_NUMERICAL)
      return hygt_set_error(HYGT_ERR_NUMERICAL, "jacobi_eigen: no convergence after 100 sweeps");
    if (status[p] == HYGT_ERR_ARGUMENT)
      return hygt_set_error(HYGT_ERR_ARGUMENT, "optimize: covariance is not positive semi-definite");
  }

  TrainParams P{};
  P.phi = buf[0].get<double>();
  P.init = buf[1].get<double>();
  P.angles = buf[2].get<double>();
  P.gains = buf[3].get<double>();
  P.traj = buf[4].get<double>();
  P.traj_len = buf[5].get<int>();
  P.var = buf[6].get<double>();
  P.ws = buf[7].get<double>();
  P.rounds = rounds;
  P.restarts = R;
  P.max_sweeps = S;
  P.tol = cfg->gain_tolerance_db;
  P.greedy = cfg->init_mode == 0;
  tk<<<(unsigned)PR, TT, ts, st>>>(P);
  std::vector<double> all_angles(PR * A), gains(PR), traj(PR * (S + 1)), var(PR * n);
  std::vector<int> tlen(PR);
  cudaMemcpyAsync(all_angles.data(), buf[2].p, bytes[2], cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(gains.data(), buf[3].p, bytes[3], cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(traj.data(), buf[4].p, bytes[4], cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(tlen.data(), buf[5].p, bytes[5], cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(var.data(), buf[6].p, bytes[6], cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return hygt_set_error(HYGT_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));

  // best restart: strict '>' in restart order, ties to the lowest index (optimizer.hpp:357-362)
  for (int p = 0; p < problems; ++p) {
    int b = 0;
    for (int r = 1; r < R; ++r)
      if (gains[(size_t)p * R + r] > gains[(size_t)p * R + b]) b = r;
    best_restart[p] = b;
    std::copy_n(all_angles.data() + ((size_t)p * R + b) * A, A, angles + (size_t)p * A);
    std::copy_n(gains.data() + (size_t)p * R, R, restart_gains + (size_t)p * R);
    if (klt_gain) klt_gain[p] = klt[p];
    if (variances) std::copy_n(var.data() + ((size_t)p * R + b) * n, n, variances + (size_t)p * n);
  }
  if (trajectories) std::copy(traj.begin(), traj.end(), trajectories);
  if (trajectory_len) std::copy(tlen.begin(), tlen.end(), trajectory_len);
  return HYGT_OK;
}
