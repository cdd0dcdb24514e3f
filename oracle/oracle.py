"""ctypes bindings for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import
this module. It loads
  * oracle/liboracle.so         -- the plain-C restatement of the reference hot path;
  * oracle/_ref/libhygt_ref.so  -- the unmodified reference headers behind an extern "C" shim
                                   (present when it was built in the container that had
                                   /root/reference; the snapshot carries it to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "liboracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libhygt_ref.so")

_p = C.c_void_p
_i = C.c_int
_u32 = C.c_uint32
_u64 = C.c_uint64
_d = C.c_double


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build()
        L = C.CDLL(_ORACLE_SO)
        L.hygt_oracle_apply_batch.argtypes = [_i, _i, _i, _p, _p, _u32, _p, _p, _u64, _i, _p, _i]
        L.hygt_oracle_class_energy.argtypes = [_i, _i, _i, _p, _p, _u32, _p, _p, _u64, _p, _i]
        L.hygt_oracle_apply_batch2.argtypes = [_i, _i, _i, _p, _p, _u32, _p, _p, _u64, _i, _p, _i, _i]
        L.hygt_oracle_class_energy2.argtypes = [_i, _i, _i, _p, _p, _u32, _p, _p, _u64, _p, _i, _i]
        L.hygt_oracle_correlation.argtypes = [_i, _i, _p, _p, _u64, _p, _p]
        L.hygt_oracle_correlation_finalize.argtypes = [_i, _p, _u64, _p]
        L.hygt_oracle_correlation_finalize.restype = None
        L.hygt_oracle_forward_chain.argtypes = [_i, _i, _p, _p, _u32, _p]
        L.hygt_oracle_inverse_chain.argtypes = [_i, _i, _p, _p, _u32, _p]
        L.hygt_oracle_to_matrix.argtypes = [_i, _i, _p, _p, _u32, _p]
        L.hygt_oracle_trig_table.argtypes = [_i, _i, _p, _p]
        L.hygt_oracle_quantize.argtypes = [_p, C.c_size_t, _i, _p]
        L.hygt_oracle_dequantize.argtypes = [_p, C.c_size_t, _i, _p]
        L.hygt_oracle_forward_fixed.argtypes = [_i, _i, _i, _i, _p, _p, _u32, _p]
        L.hygt_oracle_inverse_fixed.argtypes = [_i, _i, _i, _i, _p, _p, _u32, _p]
        L.hygt_oracle_apply_batch_fixed.argtypes = [_i, _i, _i, _i, _i, _p, _p, _u32, _p, _p,
                                                    _u64, _i, _p, _p, _i]
        L.hygt_oracle_klt_apply.argtypes = [_i, _i, _p, _p, _p, _u64, _i, _p, _i]
        L.hygt_oracle_hypercube_indices.argtypes = [_i, _i, _p, _p]
        L.hygt_oracle_rng_seed.argtypes = [_p, _u64]
        L.hygt_oracle_rng_uniform01.argtypes = [_p]
        L.hygt_oracle_rng_uniform01.restype = _d
        L.hygt_oracle_rng_uniform.argtypes = [_p, _d, _d]
        L.hygt_oracle_rng_uniform.restype = _d
        L.hygt_oracle_rng_gaussian.argtypes = [_p]
        L.hygt_oracle_rng_gaussian.restype = _d
        L.hygt_oracle_rng_below.argtypes = [_p, _u64]
        L.hygt_oracle_rng_below.restype = _u64
        L.hygt_oracle_derive_seed.argtypes = [_u64, _u64]
        L.hygt_oracle_derive_seed.restype = _u64
        L.hygt_oracle_fisher_yates.argtypes = [_p, _p, _i]
        L.hygt_oracle_random_orthogonal.argtypes = [_u64, _i, _p]
        L.hygt_oracle_memory_footprint.argtypes = [_i, _i, _i, _i]
        L.hygt_oracle_memory_footprint.restype = C.c_size_t
        L.hygt_oracle_coding_gain_db.argtypes = [_p, C.c_size_t]
        L.hygt_oracle_coding_gain_db.restype = _d
        L.hygt_oracle_jacobi_eigenvalues.argtypes = [_p, _i, _p]
        L.hygt_oracle_greedy_init.argtypes = [_p, _i, _i, _p]
        L.hygt_oracle_greedy_init.restype = None
        L.hygt_oracle_optimize.argtypes = [_p, _i, _i, _p, _p, _p, _p, _p, _p, _p]
        L.hygt_oracle_propagated_variances.argtypes = [_p, _i, _i, _p, _p]
        L.hygt_oracle_propagated_variances.restype = None
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref():
    """The reference shim (raises if it was never built)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference shim missing: {_REF_SO}")
        L = C.CDLL(_REF_SO)
        L.ref_hypercube_indices.argtypes = [_i, _i, _p, _p]
        L.ref_apply_one.argtypes = [_i, _i, _p, _p, _u32, _p, _i]
        L.ref_to_matrix.argtypes = [_i, _i, _p, _p, _p]
        L.ref_apply_batch.argtypes = [_i, _i, _i, _p, _p, _u32, _p, _p, _u64, _i, _p, _p, _i]
        L.ref_trig_table.argtypes = [_i, _i, _p, _p]
        L.ref_quantize.argtypes = [_i, _i, _p, _i, _p]
        L.ref_fixed_one.argtypes = [_i, _i, _i, _i, _p, _p, _p, _i]
        L.ref_memory_footprint.argtypes = [_i, _i, _i, _i]
        L.ref_memory_footprint.restype = C.c_size_t
        L.ref_klt_one.argtypes = [_i, _p, _p, _p, _i]
        L.ref_class_energy.argtypes = [_i, _i, _i, _p, _p, _u32, _p, _p, _u64, _p]
        L.ref_rng_stream.argtypes = [_u64, _i, _u64, _u64, _p, _p]
        L.ref_ar1_covariance_2d.argtypes = [_i, _d, _p]
        L.ref_optimize.argtypes = [_p, _i, _i, _i, _i, _d, _u64, _i, _p, _p, _p, _p, _p, _p]
        L.ref_variance_permutation.argtypes = [_p, _i, _i, _p, _p, _p]
        _ref = L
    return _ref


# ---------------------------------------------------------------- convenience wrappers ------

def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


class Rng:
    """The oracle's restatement of hygt::Rng (rng.hpp:44-77)."""

    def __init__(self, seed: int):
        self._state = (C.c_uint8 * 4096)()
        lib().hygt_oracle_rng_seed(C.cast(self._state, C.c_void_p), seed)

    @property
    def _p(self):
        return C.cast(self._state, C.c_void_p)

    def uniform01(self):
        return lib().hygt_oracle_rng_uniform01(self._p)

    def uniform(self, lo, hi):
        return lib().hygt_oracle_rng_uniform(self._p, lo, hi)

    def gaussian(self):
        return lib().hygt_oracle_rng_gaussian(self._p)

    def below(self, bound):
        return lib().hygt_oracle_rng_below(self._p, bound)

    def fisher_yates(self, n):
        p = np.empty(n, np.uint16)
        lib().hygt_oracle_fisher_yates(self._p, _ptr(p), n)
        return p


def derive_seed(base, stream):
    return lib().hygt_oracle_derive_seed(base, stream)


def apply_batch(log2_n, rounds, angles, perms, perm_mask, x, cls=None, inverse=False, threads=None,
                hoist=False):
    """fp64 outputs of the chained reference transform over fp32 rows. hoist=True tables cos/sin
    once per class (bit-identical, for full-size checks)."""
    angles = _c(angles, np.float64)
    classes = angles.shape[0] if angles.ndim == 2 else 1
    x = _c(x, np.float32)
    n = 1 << log2_n
    count = x.size // n
    y = np.empty((count, n), np.float64)
    st = lib().hygt_oracle_apply_batch2(log2_n, rounds, classes, _ptr(angles), _ptr(_c(perms, np.uint16)),
                                        perm_mask, _ptr(x), _ptr(_c(cls, np.uint16)), count,
                                        int(bool(inverse)), _ptr(y), threads or os.cpu_count(),
                                        int(bool(hoist)))
    if st:
        raise ValueError("oracle: class id out of range")
    return y


def class_energy(log2_n, rounds, angles, perms, perm_mask, x, cls=None, threads=None, hoist=False):
    angles = _c(angles, np.float64)
    classes = angles.shape[0] if angles.ndim == 2 else 1
    x = _c(x, np.float32)
    n = 1 << log2_n
    e = np.zeros((classes, n), np.float64)
    lib().hygt_oracle_class_energy2(log2_n, rounds, classes, _ptr(angles), _ptr(_c(perms, np.uint16)),
                                    perm_mask, _ptr(x), _ptr(_c(cls, np.uint16)), x.size // n,
                                    _ptr(e), threads or os.cpu_count(), int(bool(hoist)))
    return e


def correlation(log2_n, classes, x, cls=None):
    """(sum [C][N][N], counts [C]) of r r^T per class (CorrelationAccumulator::add restated)."""
    x = _c(x, np.float32)
    n = 1 << log2_n
    s = np.zeros((classes, n, n), np.float64)
    k = np.zeros(classes, np.uint64)
    st = lib().hygt_oracle_correlation(log2_n, classes, _ptr(x), _ptr(_c(cls, np.uint16)), x.size // n,
                                       _ptr(s), _ptr(k))
    if st:
        raise ValueError("oracle: class id out of range")
    return s, k


def correlation_finalize(log2_n, sums, count):
    n = 1 << log2_n
    sums = _c(sums, np.float64)
    phi = np.empty((n, n), np.float64)
    lib().hygt_oracle_correlation_finalize(log2_n, _ptr(sums), int(count), _ptr(phi))
    return phi


def trig_table(angle_bits, precision_bits):
    n = 1 << angle_bits
    c = np.empty(n, np.int32)
    s = np.empty(n, np.int32)
    if lib().hygt_oracle_trig_table(angle_bits, precision_bits, _ptr(c), _ptr(s)):
        raise ValueError("trig table widths")
    return c, s


def quantize(angles, angle_bits):
    a = _c(angles, np.float64)
    codes = np.empty(a.shape, np.uint16)
    if lib().hygt_oracle_quantize(_ptr(a), a.size, angle_bits, _ptr(codes)):
        raise ValueError("angle_bits")
    return codes


def dequantize(codes, angle_bits):
    c = _c(codes, np.uint16)
    a = np.empty(c.shape, np.float64)
    lib().hygt_oracle_dequantize(_ptr(c), c.size, angle_bits, _ptr(a))
    return a


def apply_batch_fixed(log2_n, rounds, angle_bits, precision_bits, codes, perms, perm_mask, x,
                      cls=None, inverse=False):
    codes = _c(codes, np.uint16)
    classes = codes.shape[0] if codes.ndim == 2 else 1
    x = _c(x, np.int64)
    n = 1 << log2_n
    count = x.size // n
    y = np.empty((count, n), np.int64)
    bad = C.c_uint64(0)
    st = lib().hygt_oracle_apply_batch_fixed(log2_n, rounds, classes, angle_bits, precision_bits,
                                             _ptr(codes), _ptr(_c(perms, np.uint16)), perm_mask,
                                             _ptr(x), _ptr(_c(cls, np.uint16)), count,
                                             int(bool(inverse)), _ptr(y), C.byref(bad), 1)
    return st, int(bad.value), y


def klt_apply(k, x, cls=None, inverse=False):
    k = _c(k, np.float64)
    classes, n = k.shape[0], k.shape[1]
    x = _c(x, np.float32)
    count = x.size // n
    y = np.empty((count, n), np.float64)
    if lib().hygt_oracle_klt_apply(n, classes, _ptr(k), _ptr(x), _ptr(_c(cls, np.uint16)), count,
                                   int(bool(inverse)), _ptr(y), 1):
        raise ValueError("class id out of range")
    return y


def random_orthogonal(seed, n):
    q = np.empty((n, n), np.float64)
    lib().hygt_oracle_random_orthogonal(seed, n, _ptr(q))
    return q


def to_matrix(log2_n, rounds, angles, perms=None, perm_mask=0):
    n = 1 << log2_n
    t = np.empty((n, n), np.float64)
    lib().hygt_oracle_to_matrix(log2_n, rounds, _ptr(_c(angles, np.float64)),
                                _ptr(_c(perms, np.uint16)), perm_mask, _ptr(t))
    return t


def memory_footprint(klt, log2_n, rounds, num):
    return lib().hygt_oracle_memory_footprint(int(bool(klt)), log2_n, rounds, num)


# ------------------------------------------------------------------ reference wrappers ------

def ref_apply_batch(log2_n, rounds, angles, perms, perm_mask, x, cls=None, inverse=False,
                    threads=None, out="f64"):
    angles = _c(angles, np.float64)
    classes = angles.shape[0] if angles.ndim == 2 else 1
    x = _c(x, np.float32)
    n = 1 << log2_n
    count = x.size // n
    y = np.empty((count, n), np.float64 if out == "f64" else np.float32)
    st = ref().ref_apply_batch(log2_n, rounds, classes, _ptr(angles), _ptr(_c(perms, np.uint16)),
                               perm_mask, _ptr(x), _ptr(_c(cls, np.uint16)), count,
                               int(bool(inverse)), _ptr(y) if out != "f64" else None,
                               _ptr(y) if out == "f64" else None, threads or os.cpu_count())
    if st:
        raise ValueError(f"reference apply failed with status {st}")
    return y


# ---------------------------------------------------------------- optimizer ----

INIT_MODES = {"greedy_jacobi": 0, "random": 1, "zero": 2}


class _OptConfig(C.Structure):
    _fields_ = [("restarts", C.c_int), ("max_sweeps", C.c_int), ("gain_tolerance_db", C.c_double),
                ("seed", C.c_uint64), ("init_mode", C.c_int)]


def _opt_result(n_angles, restarts, max_sweeps):
    return (np.zeros(n_angles, np.float64), np.zeros(restarts, np.float64), C.c_int(0), C.c_double(0.0),
            np.full((restarts, max_sweeps + 1), np.nan), np.zeros(restarts, np.int32))


def _opt_report(st, angles, gains, best, klt, traj, tlen):
    if st:
        raise ValueError(f"optimize failed with status {st}")
    trajectories = [traj[r, :tlen[r]].tolist() for r in range(len(gains))]
    b = int(best.value)
    return angles, {"restart_gains_db": gains, "best_restart": b, "klt_gain_db": float(klt.value),
                    "gain_ratio": gains[b] / klt.value if klt.value > 1e-15 else 1.0,
                    "trajectories": trajectories}


def coding_gain_db(v):
    v = _c(v, np.float64)
    return lib().hygt_oracle_coding_gain_db(_ptr(v), v.size)


def jacobi_eigenvalues(phi):
    phi = _c(phi, np.float64)
    ev = np.zeros(phi.shape[0], np.float64)
    if lib().hygt_oracle_jacobi_eigenvalues(_ptr(phi), phi.shape[0], _ptr(ev)):
        raise ValueError("jacobi_eigen: no convergence")
    return ev


def greedy_init(phi, log2_n, rounds):
    phi = _c(phi, np.float64)
    a = np.zeros(rounds * log2_n * (1 << (log2_n - 1)), np.float64)
    lib().hygt_oracle_greedy_init(_ptr(phi), log2_n, rounds, _ptr(a))
    return a


def optimize(phi, log2_n, rounds, restarts=4, max_sweeps=50, gain_tolerance_db=1e-4, seed=0,
             init_mode="greedy_jacobi"):
    """optimizer.hpp:311-371 restated: (best angles, report dict)."""
    phi = _c(phi, np.float64)
    cfg = _OptConfig(restarts, max_sweeps, gain_tolerance_db, seed, INIT_MODES[init_mode])
    res = _opt_result(rounds * log2_n * (1 << (log2_n - 1)), max(restarts, 0), max_sweeps)
    angles, gains, best, klt, traj, tlen = res
    st = lib().hygt_oracle_optimize(_ptr(phi), log2_n, rounds, C.byref(cfg), _ptr(angles), _ptr(gains),
                                    C.byref(best), C.byref(klt), _ptr(traj), _ptr(tlen))
    return _opt_report(st, *res)


def propagated_variances(phi, log2_n, rounds, angles):
    phi = _c(phi, np.float64)
    v = np.zeros(1 << log2_n, np.float64)
    lib().hygt_oracle_propagated_variances(_ptr(phi), log2_n, rounds, _ptr(_c(angles, np.float64)), _ptr(v))
    return v


def ref_optimize(phi, log2_n, rounds, restarts=4, max_sweeps=50, gain_tolerance_db=1e-4, seed=0,
                 init_mode="greedy_jacobi"):
    """The reference's own hygt::optimize through the shim."""
    phi = _c(phi, np.float64)
    res = _opt_result(rounds * log2_n * (1 << (log2_n - 1)), max(restarts, 0), max_sweeps)
    angles, gains, best, klt, traj, tlen = res
    st = ref().ref_optimize(_ptr(phi), log2_n, rounds, restarts, max_sweeps, gain_tolerance_db, seed,
                            INIT_MODES[init_mode], _ptr(angles), _ptr(gains), C.byref(best), C.byref(klt),
                            _ptr(traj), _ptr(tlen))
    return _opt_report(st, *res)


def ref_variance_permutation(phi, log2_n, rounds, angles):
    phi = _c(phi, np.float64)
    n = 1 << log2_n
    perm = np.zeros(n, np.uint16)
    var = np.zeros(n, np.float64)
    st = ref().ref_variance_permutation(_ptr(phi), log2_n, rounds, _ptr(_c(angles, np.float64)),
                                        _ptr(perm), _ptr(var))
    if st:
        raise ValueError(f"variance_permutation failed with status {st}")
    return perm, var
