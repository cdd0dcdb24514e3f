"""The reference's on-disk formats, host side (numpy), for the `hygt_gpu_apply` drop-in.

RBLK dataset (dataset.hpp:68-119): "RBLK", u8 version 1, u8 log2_n, u16 class_count, u32 blocks,
then per block u16 class_id + N float32, little-endian.
HYGT model bundle (bundle.hpp:99-191): "HYGT", u8 version 1, u8 log2_n, u16 class_count,
u8 angle_bits (0 = float64 angles), u8 precision_bits, then per class u8 rounds, u8 has_perm,
the angles (f64 each, or one u8 code each) and, if has_perm, N u16 indices.
"""
from __future__ import annotations

import struct
from typing import List, Optional, Sequence

import numpy as np

from .errors import ArgumentError, IoError


def _record_dtype(n: int) -> np.dtype:
    return np.dtype([("cls", "<u2"), ("x", "<f4", (n,))])


def write_rblk(path: str, log2_n: int, class_count: int, cls: np.ndarray, x: np.ndarray) -> None:
    n = 1 << log2_n
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1, n)
    cls = np.ascontiguousarray(cls, dtype=np.uint16).reshape(-1)
    if cls.shape[0] != x.shape[0]:
        raise ArgumentError("write_rblk: class ids and rows differ in count")
    rec = np.empty(x.shape[0], dtype=_record_dtype(n))
    rec["cls"] = cls
    rec["x"] = x
    with open(path, "wb") as f:
        f.write(b"RBLK" + struct.pack("<BBHI", 1, log2_n, class_count, x.shape[0]))
        f.write(rec.tobytes())


def read_rblk(path: str):
    """(log2_n, class_count, cls u16 [B], x f32 [B][N])."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"RBLK":
        raise IoError("bad magic: not a RBLK dataset file")
    version, log2_n, class_count, count = struct.unpack_from("<BBHI", data, 4)
    if version != 1:
        raise IoError("read_rblk: unsupported version")
    n = 1 << log2_n
    rec = np.frombuffer(data, dtype=_record_dtype(n), count=count, offset=12)
    return log2_n, class_count, rec["cls"].copy(), rec["x"].copy()


def write_bundle(path: str, log2_n: int, angles: Sequence[np.ndarray] = (),
                 codes: Sequence[np.ndarray] = (), angle_bits: int = 0, precision_bits: int = 10,
                 rounds: Optional[Sequence[int]] = None,
                 perms: Optional[Sequence[Optional[np.ndarray]]] = None) -> None:
    """Float bundle (angles per class, angle_bits = 0) or quantized bundle (codes per class)."""
    per_class: List[np.ndarray] = list(codes if angle_bits else angles)
    half = 1 << (log2_n - 1)
    if rounds is None:
        rounds = [len(a) // (log2_n * half) for a in per_class]
    perms = list(perms) if perms is not None else [None] * len(per_class)
    with open(path, "wb") as f:
        f.write(b"HYGT" + struct.pack("<BBHBB", 1, log2_n, len(per_class), angle_bits, precision_bits))
        for a, r, p in zip(per_class, rounds, perms):
            f.write(struct.pack("<BB", r, 0 if p is None else 1))
            if angle_bits:
                f.write(np.asarray(a, dtype=np.uint8).tobytes())
            else:
                f.write(np.asarray(a, dtype="<f8").tobytes())
            if p is not None:
                f.write(np.asarray(p, dtype="<u2").tobytes())
