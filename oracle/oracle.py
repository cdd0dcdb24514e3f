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


def apply_batch(log2_n, rounds, angles, perms, perm_mask, x, cls=None, inverse=False, threads=None):
    """fp64 outputs of the chained reference transform over fp32 rows."""
    angles = _c(angles, np.float64)
    classes = angles.shape[0] if angles.ndim == 2 else 1
    x = _c(x, np.float32)
    n = 1 << log2_n
    count = x.size // n
    y = np.empty((count, n), np.float64)
    st = lib().hygt_oracle_apply_batch(log2_n, rounds, classes, _ptr(angles), _ptr(_c(perms, np.uint16)),
                                       perm_mask, _ptr(x), _ptr(_c(cls, np.uint16)), count,
                                       int(bool(inverse)), _ptr(y), threads or os.cpu_count())
    if st:
        raise ValueError("oracle: class id out of range")
    return y


def class_energy(log2_n, rounds, angles, perms, perm_mask, x, cls=None, threads=None):
    angles = _c(angles, np.float64)
    classes = angles.shape[0] if angles.ndim == 2 else 1
    x = _c(x, np.float32)
    n = 1 << log2_n
    e = np.zeros((classes, n), np.float64)
    lib().hygt_oracle_class_energy(log2_n, rounds, classes, _ptr(angles), _ptr(_c(perms, np.uint16)),
                                   perm_mask, _ptr(x), _ptr(_c(cls, np.uint16)), x.size // n,
                                   _ptr(e), threads or os.cpu_count())
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
