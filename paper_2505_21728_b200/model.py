"""Host-side model types mirroring the reference's public C++ types.

* ``num_parameters``, ``HyGTModel``             -- include/hygt/model.hpp:29-96
* ``hypercube_indices``                          -- include/hygt/hypercube.hpp:59-77
* ``TrigTable``, ``QuantizedHyGTModel``,
  ``quantize_model``, ``dequantize_model``,
  ``memory_footprint``, ``TransformKind``        -- include/hygt/fixedpoint.hpp:35-238
* ``ModelBundle``                                -- include/hygt/bundle.hpp:34-96

These are parameter containers with the reference's validation and error behaviour; all
transform arithmetic runs on the GPU (paper_2505_21728_b200.plan).
"""
from __future__ import annotations

import enum
import math
from typing import Optional, Sequence

import numpy as np

from .errors import ArgumentError

K_MAX_LOG2N = 16  # hypercube.hpp:25


def num_parameters(log2_n: int, rounds: int) -> int:
    """rounds * N * log2(N) / 2 (model.hpp:29-34)."""
    if log2_n < 1 or rounds < 1:
        raise ArgumentError("num_parameters: log2_n and rounds must be >= 1")
    return rounds * (1 << log2_n) * log2_n // 2


def validate_permutation(perm, dimension: int) -> np.ndarray:
    """Throws unless perm is a bijection on {0..dimension-1} (model.hpp:37-44)."""
    p = np.asarray(perm)
    if p.ndim != 1 or p.size != dimension:
        raise ArgumentError("permutation: wrong length")
    if p.size and (p.min() < 0 or p.max() >= dimension or np.unique(p).size != dimension):
        raise ArgumentError("permutation: not a bijection")
    return p.astype(np.uint16)


def hypercube_indices(log2_n: int, pass_: int):
    """(m, n) index pairs of hypercube pass `pass_` (hypercube.hpp:59-77)."""
    if log2_n < 1 or log2_n > K_MAX_LOG2N:
        raise ArgumentError("hypercube_indices: log2_n out of range [1, 16]")
    if pass_ < 0 or pass_ >= log2_n:
        raise ArgumentError("hypercube_indices: pass out of range [0, log2_n)")
    half = 1 << (log2_n - 1)
    k = 1 << pass_
    j = np.arange(half, dtype=np.int64)
    m = j + (j & -k)
    return m.astype(np.uint32), (m + k).astype(np.uint32)


class HyGTModel:
    """Angles in application order (round, pass, pair) plus an optional final permutation."""

    def __init__(self, log2_n: int, rounds: int, angles: Sequence[float],
                 permutation: Optional[Sequence[int]] = None):
        if log2_n < 1 or log2_n > K_MAX_LOG2N:
            raise ArgumentError("HyGTModel: log2_n out of range [1, 16]")
        a = np.asarray(angles, dtype=np.float64).reshape(-1)
        if a.size != num_parameters(log2_n, rounds):
            raise ArgumentError("HyGTModel: angle count must be rounds * N * log2(N) / 2")
        self._log2_n = int(log2_n)
        self._rounds = int(rounds)
        self._angles = a.copy()
        self._angles.setflags(write=False)
        self._perm = None
        if permutation is not None:
            self._perm = validate_permutation(permutation, 1 << log2_n)
            self._perm.setflags(write=False)

    @staticmethod
    def zeros(log2_n: int, rounds: int) -> "HyGTModel":
        return HyGTModel(log2_n, rounds, np.zeros(num_parameters(log2_n, rounds)))

    log2_n = property(lambda self: self._log2_n)
    rounds = property(lambda self: self._rounds)
    angles = property(lambda self: self._angles)
    permutation = property(lambda self: self._perm)

    def dimension(self) -> int:
        return 1 << self._log2_n

    def pairs_per_pass(self) -> int:
        return self.dimension() // 2

    def pass_count(self) -> int:
        return self._rounds * self._log2_n

    def angle_index(self, round_: int, pass_: int, pair: int) -> int:
        return (round_ * self._log2_n + pass_) * self.pairs_per_pass() + pair  # model.hpp:77-79

    def angle(self, round_: int, pass_: int, pair: int) -> float:
        return float(self._angles[self.angle_index(round_, pass_, pair)])

    def with_permutation(self, perm) -> "HyGTModel":
        return HyGTModel(self._log2_n, self._rounds, self._angles, perm)


class TrigTable:
    """round(cos/sin(2 pi q / 2^b) * 2^p) for every code q (fixedpoint.hpp:35-65)."""

    def __init__(self, angle_bits: int, precision_bits: int):
        if angle_bits < 1 or angle_bits > 12:
            raise ArgumentError("TrigTable: angle_bits out of range [1, 12]")
        if precision_bits < 4 or precision_bits > 15:
            raise ArgumentError("TrigTable: precision_bits out of range [4, 15]")
        self.angle_bits = angle_bits
        self.precision_bits = precision_bits
        size = 1 << angle_bits
        scale = float(1 << precision_bits)
        a = 2.0 * math.pi * np.arange(size, dtype=np.float64) / size
        # std::lround rounds half away from zero
        def lround(v):
            return np.where(v >= 0, np.floor(v + 0.5), np.ceil(v - 0.5)).astype(np.int32)
        self._cos = lround(np.cos(a) * scale)
        self._sin = lround(np.sin(a) * scale)

    def size(self) -> int:
        return self._cos.size

    def cos_entry(self, code: int) -> int:
        return int(self._cos[code])

    def sin_entry(self, code: int) -> int:
        return int(self._sin[code])


def build_trig_table(angle_bits: int, precision_bits: int) -> TrigTable:
    return TrigTable(angle_bits, precision_bits)


class QuantizedHyGTModel:
    """b-bit angle codes in HyGTModel order (fixedpoint.hpp:73-109)."""

    def __init__(self, log2_n: int, rounds: int, angle_bits: int, codes,
                 permutation: Optional[Sequence[int]] = None):
        if log2_n < 1 or log2_n > K_MAX_LOG2N:
            raise ArgumentError("QuantizedHyGTModel: log2_n out of range [1, 16]")
        if angle_bits < 1 or angle_bits > 12:
            raise ArgumentError("QuantizedHyGTModel: angle_bits out of range [1, 12]")
        c = np.asarray(codes).reshape(-1)
        if c.size != num_parameters(log2_n, rounds):
            raise ArgumentError("QuantizedHyGTModel: code count must be rounds * N * log2(N) / 2")
        if c.size and (c.min() < 0 or c.max() > (1 << angle_bits) - 1):
            raise ArgumentError("QuantizedHyGTModel: code exceeds 2^angle_bits")
        self.log2_n = int(log2_n)
        self.rounds = int(rounds)
        self.angle_bits = int(angle_bits)
        self.codes = c.astype(np.uint16)
        self.permutation = None if permutation is None else validate_permutation(permutation, 1 << log2_n)

    def dimension(self) -> int:
        return 1 << self.log2_n

    def pairs_per_pass(self) -> int:
        return self.dimension() // 2

    def code_index(self, round_: int, pass_: int, pair: int) -> int:
        return (round_ * self.log2_n + pass_) * self.pairs_per_pass() + pair


def quantize_model(model: HyGTModel, angle_bits: int) -> QuantizedHyGTModel:
    """code = llround(theta / 2pi * 2^b) mod 2^b (fixedpoint.hpp:115-128)."""
    if angle_bits < 1 or angle_bits > 12:
        raise ArgumentError("quantize_model: angle_bits out of range [1, 12]")
    size = 1 << angle_bits
    scaled = model.angles / (2.0 * math.pi) * float(size)
    q = np.where(scaled >= 0, np.floor(scaled + 0.5), np.ceil(scaled - 0.5)).astype(np.int64)  # llround
    q = np.fmod(q, size)
    q = np.where(q < 0, q + size, q)
    return QuantizedHyGTModel(model.log2_n, model.rounds, angle_bits, q.astype(np.uint16),
                              model.permutation)


def dequantize_model(model: QuantizedHyGTModel) -> HyGTModel:
    """angle = 2 pi code / 2^b (fixedpoint.hpp:131-137)."""
    step = 2.0 * math.pi / float(1 << model.angle_bits)
    return HyGTModel(model.log2_n, model.rounds, step * model.codes.astype(np.float64),
                     model.permutation)


class TransformKind(enum.Enum):
    klt = 0
    hygt = 1


def memory_footprint(kind: TransformKind, log2_n: int, rounds: int, num_transforms: int) -> int:
    """Storage units: N^2 per KLT, R N log2N / 2 per HyGT (fixedpoint.hpp:231-238)."""
    if log2_n < 1 or rounds < 1 or num_transforms < 1:
        raise ArgumentError("memory_footprint: arguments must be >= 1")
    n = 1 << log2_n
    if kind == TransformKind.klt:
        return num_transforms * n * n
    return num_transforms * num_parameters(log2_n, rounds)


class ModelBundle:
    """Per-class models sharing one dimension (bundle.hpp:34-96)."""

    def __init__(self, models, precision_bits: int = 10):
        models = list(models)
        if not models:
            raise ArgumentError("ModelBundle: need at least one class")
        if len(models) > 0xFFFF:
            raise ArgumentError("ModelBundle: too many classes")
        self._quantized = isinstance(models[0], QuantizedHyGTModel)
        for m in models:
            if m.log2_n != models[0].log2_n:
                raise ArgumentError("ModelBundle: all classes must share one dimension")
            if m.rounds > 255:
                raise ArgumentError("ModelBundle: rounds capped at 255")
            if self._quantized and m.angle_bits != models[0].angle_bits:
                raise ArgumentError("ModelBundle: all classes must share angle_bits")
            if self._quantized and m.angle_bits > 8:
                raise ArgumentError("ModelBundle: serialized codes are one byte, angle_bits <= 8")
        self._models = models
        self.precision_bits = precision_bits

    def quantized(self) -> bool:
        return self._quantized

    def class_count(self) -> int:
        return len(self._models)

    def log2_n(self) -> int:
        return self._models[0].log2_n

    def dimension(self) -> int:
        return 1 << self.log2_n()

    def angle_bits(self) -> int:
        return self._models[0].angle_bits if self._quantized else 0

    def float_model(self, c: int) -> HyGTModel:
        if self._quantized:
            raise ArgumentError("ModelBundle: bundle is quantized")
        return self._models[c]

    def quantized_model(self, c: int) -> QuantizedHyGTModel:
        if not self._quantized:
            raise ArgumentError("ModelBundle: bundle holds float models")
        return self._models[c]

    def dequantized(self, c: int) -> HyGTModel:
        m = self._models[c]
        return dequantize_model(m) if self._quantized else m

    def rounds(self, c: int) -> int:
        return self._models[c].rounds
