"""Generate tests/golden/golden_fixed_long.npz from the UNMODIFIED reference (oracle/_ref shim).

Long fixed-point models at low precision, where values grow past 2^31 and where the reference
throws OverflowError (|intermediate| > 2^46, fixedpoint.hpp:177-179). Run in the container
that has /root/reference (make -C oracle builds the shim first):
    python tests/gen_golden_fixed_long.py
Every output array is what hygt::forward_fixed / hygt::inverse_fixed return (or the status of
the exception they throw) for the stored inputs; the GPU suite must reproduce them bit for bit,
including the first failing row.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "golden_fixed_long.npz")


def P(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def table(R, b, p):
    c = np.empty(1 << b, np.int32)
    s = np.empty(1 << b, np.int32)
    R.ref_trig_table(b, p, P(c), P(s))
    return c, s


def main():
    O.build()
    R = O.ref()
    rng = np.random.Generator(np.random.PCG64(20250528))
    g = {}
    # (name, log2n, rounds, b, p, code mode, input mode)
    cases = [
        # 480 passes of the largest-gain codes of TrigTable(8, 4): valid rows grow past 2^31
        # (int32 would wrap), the all-2^20 rows overflow 2^46 -> OverflowError at row 37.
        ("grow16", 4, 120, 8, 4, "maxgain", "small+big"),
        # 180 passes at p = 4 with random codes (R * log2N > 140), inputs up to 2^10
        ("long64", 6, 30, 8, 4, "random", "medium"),
        # N = 256, 58 rounds of max-gain codes: overflow on the 2^20 rows
        ("grow256", 8, 58, 8, 4, "maxgain", "small+big"),
        # N = 32 at p = 5, mixed codes, a final permutation (150 passes; the C ABI takes
        # permutations for rounds <= 32)
        ("mixed32", 5, 30, 6, 5, "mixed", "medium"),
    ]
    for name, log2n, rounds, b, p, cmode, imode in cases:
        n = 1 << log2n
        a = rounds * n * log2n // 2
        ct, st = table(R, b, p)
        gain = np.sqrt(ct.astype(np.float64) ** 2 + st.astype(np.float64) ** 2) / (1 << p)
        top = np.flatnonzero(gain >= gain.max() - 1e-12).astype(np.uint16)
        if cmode == "maxgain":
            codes = rng.choice(top, a).astype(np.uint16)
        elif cmode == "random":
            codes = rng.integers(0, 1 << b, a).astype(np.uint16)
        else:
            codes = np.where(rng.random(a) < 0.7, rng.choice(top, a), rng.integers(0, 1 << b, a)).astype(np.uint16)
        perm = rng.permutation(n).astype(np.uint16) if name == "mixed32" else None
        rows = 48
        if imode == "small+big":
            x = rng.integers(-12, 13, (rows, n)).astype(np.int64)
            x[37, :] = 1 << 20
            x[41, :] = -(1 << 20)
        else:
            x = rng.integers(-1024, 1025, (rows, n)).astype(np.int64)
            x[11, :] = (1 << 20) * np.where(rng.random(n) < 0.5, 1, -1)
        fo = x.copy()
        fs = np.zeros(rows, np.int64)
        io = x.copy()
        ist = np.zeros(rows, np.int64)
        for r in range(rows):
            v = x[r].copy()
            fs[r] = R.ref_fixed_one(log2n, rounds, b, p, P(codes), P(perm), P(v), 0)
            fo[r] = v
            w = x[r].copy()
            ist[r] = R.ref_fixed_one(log2n, rounds, b, p, P(codes), P(perm), P(w), 1)
            io[r] = w
        pre = name + "_"
        g[pre + "meta"] = np.array([log2n, rounds, b, p, int(perm is not None)], np.int64)
        g[pre + "codes"] = codes
        g[pre + "perm"] = perm if perm is not None else np.zeros(0, np.uint16)
        g[pre + "x"] = x
        g[pre + "fwd"] = fo
        g[pre + "fwd_status"] = fs
        g[pre + "inv"] = io
        g[pre + "inv_status"] = ist
        print(name, "fwd status", np.unique(fs, return_counts=True), "max |fwd ok|",
              int(np.abs(fo[fs == 0]).max()), "inv status", np.unique(ist, return_counts=True))
    g["names"] = np.array([c[0] for c in cases])
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
