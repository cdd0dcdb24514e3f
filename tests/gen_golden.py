"""Generate tests/golden/golden_v1.npz from the UNMODIFIED reference (oracle/_ref shim).

Run in the container that has /root/reference (make -C oracle builds the shim first):
    python tests/gen_golden.py
The .npz is committed; the GPU box never needs /root/reference. Every array below is an input
fed to, or an output returned by, the reference's own functions:
  * float transforms: hygt::forward / hygt::inverse (transform.hpp:72-96), chained single-round
    models for inter-round permutations;
  * fixed point: forward_fixed / inverse_fixed + TrigTable + quantize_model (fixedpoint.hpp);
  * klt_forward (statistics.hpp:222-224); per-class energy via CorrelationAccumulator;
  * hygt::Rng streams (rng.hpp) and hypercube_indices (hypercube.hpp).
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")


def P(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def main():
    O.build()
    R = O.ref()
    rng = np.random.Generator(np.random.PCG64(20250527))
    g = {}

    # ---- float HyGT cases: (log2n, rounds, classes, mask kind, rows)
    cases = [(1, 1, 1, "none", 8), (2, 2, 1, "final", 16), (3, 1, 2, "none", 32),
             (4, 2, 1, "inter", 96), (4, 3, 35, "inter+final", 200), (5, 2, 3, "final", 64),
             (6, 4, 5, "inter", 96), (7, 2, 2, "none", 40), (8, 4, 3, "none", 48),
             (8, 2, 2, "inter+final", 24)]
    for k, (log2n, rounds, classes, kind, rows) in enumerate(cases):
        n = 1 << log2n
        a = rounds * n * log2n // 2
        angles = rng.uniform(-np.pi, np.pi, (classes, a))
        perms = np.stack([np.stack([rng.permutation(n) for _ in range(rounds)])
                          for _ in range(classes)]).astype(np.uint16)
        mask = {"none": 0, "final": 1 << (rounds - 1), "inter": (1 << (rounds - 1)) - 1,
                "inter+final": (1 << rounds) - 1}[kind]
        x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
        cls = rng.integers(0, classes, rows).astype(np.uint16)
        yf = O.ref_apply_batch(log2n, rounds, angles, perms, mask, x, cls, inverse=False)
        yi = O.ref_apply_batch(log2n, rounds, angles, perms, mask, x, cls, inverse=True)
        pre = f"f{k}_"
        g[pre + "meta"] = np.array([log2n, rounds, classes, mask], np.int64)
        g[pre + "angles"] = angles
        g[pre + "perms"] = perms
        g[pre + "x"] = x
        g[pre + "cls"] = cls
        g[pre + "fwd"] = yf
        g[pre + "inv"] = yi
    g["float_cases"] = np.array(len(cases))

    # ---- fixed point cases (reference forward_fixed/inverse_fixed, final perm only)
    fcases = [(1, 1, 8, 10, False), (4, 2, 8, 10, True), (6, 5, 8, 10, False), (8, 3, 8, 10, True),
              (4, 2, 4, 6, False), (5, 2, 12, 15, True), (3, 2, 8, 4, False)]
    for k, (log2n, rounds, b, p, with_perm) in enumerate(fcases):
        n = 1 << log2n
        a = rounds * n * log2n // 2
        angles = rng.uniform(0, 2 * np.pi, a)
        codes = np.empty(a, np.uint16)
        assert R.ref_quantize(log2n, rounds, P(angles), b, P(codes)) == 0
        perm = rng.permutation(n).astype(np.uint16) if with_perm else None
        rows = 64
        x = rng.integers(-1024, 1025, (rows, n)).astype(np.int64)
        # a few rows near/over the limits to pin error outcomes
        x[3, 0] = (1 << 20)          # allowed
        x[5, n - 1] = -(1 << 20) - 1  # ArgumentError
        if n >= 4:
            x[7, :] = (1 << 20)       # large but legal input
        fo = np.zeros_like(x)
        fs = np.zeros(rows, np.int64)
        io = np.zeros_like(x)
        ist = np.zeros(rows, np.int64)
        for r in range(rows):
            v = x[r].copy()
            fs[r] = R.ref_fixed_one(log2n, rounds, b, p, P(codes), P(perm), P(v), 0)
            fo[r] = v
            w = (fo[r] if fs[r] == 0 else x[r]).copy()
            ist[r] = R.ref_fixed_one(log2n, rounds, b, p, P(codes), P(perm), P(w), 1)
            io[r] = w
        pre = f"x{k}_"
        g[pre + "meta"] = np.array([log2n, rounds, b, p, int(with_perm)], np.int64)
        g[pre + "codes"] = codes
        g[pre + "angles"] = angles
        g[pre + "perm"] = perm if perm is not None else np.zeros(0, np.uint16)
        g[pre + "x"] = x
        g[pre + "fwd"] = fo
        g[pre + "fwd_status"] = fs
        g[pre + "inv"] = io
        g[pre + "inv_status"] = ist
    g["fixed_cases"] = np.array(len(fcases))
    # overflow case: precision 15, inputs at the limit, many rounds -> OverflowError somewhere
    log2n, rounds, b, p = 4, 6, 8, 15
    n = 16
    a = rounds * n * log2n // 2
    codes = rng.integers(0, 256, a).astype(np.uint16)
    x = np.full((8, n), 1 << 20, np.int64)
    st = np.zeros(8, np.int64)
    for r in range(8):
        v = x[r].copy()
        st[r] = R.ref_fixed_one(log2n, rounds, b, p, P(codes), None, P(v), 0)
    g["ovf_codes"] = codes
    g["ovf_x"] = x
    g["ovf_status"] = st

    # ---- trig tables
    for b, p in [(8, 10), (2, 4), (12, 15), (6, 10)]:
        c = np.empty(1 << b, np.int32)
        s = np.empty(1 << b, np.int32)
        R.ref_trig_table(b, p, P(c), P(s))
        g[f"trig_{b}_{p}_cos"] = c
        g[f"trig_{b}_{p}_sin"] = s

    # ---- Rng streams
    for seed in [0, 1, 42, 2505]:
        d = np.empty(257)
        R.ref_rng_stream(seed, 0, 0, 257, P(d), None)
        g[f"rng_u01_{seed}"] = d
        d = np.empty(257)
        R.ref_rng_stream(seed, 1, 0, 257, P(d), None)
        g[f"rng_gauss_{seed}"] = d
        u = np.empty(257, np.uint64)
        R.ref_rng_stream(seed, 2, 35, 257, None, P(u))
        g[f"rng_below35_{seed}"] = u
        u = np.empty(64, np.uint64)
        R.ref_rng_stream(seed, 3, 0, 64, None, P(u))
        g[f"derive_seed_{seed}"] = u

    # ---- hypercube schedules
    for log2n in range(1, 9):
        n = 1 << log2n
        ms = np.empty((log2n, n // 2), np.uint32)
        ns = np.empty((log2n, n // 2), np.uint32)
        for p in range(log2n):
            m = np.empty(n // 2, np.uint32)
            nn = np.empty(n // 2, np.uint32)
            R.ref_hypercube_indices(log2n, p, P(m), P(nn))
            ms[p], ns[p] = m, nn
        g[f"hc_{log2n}_m"] = ms
        g[f"hc_{log2n}_n"] = ns

    # ---- KLT
    n, classes, rows = 16, 3, 40
    k = np.stack([np.linalg.qr(rng.standard_normal((n, n)))[0] for _ in range(classes)])
    x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
    cls = rng.integers(0, classes, rows).astype(np.uint16)
    yf = np.empty((rows, n))
    yi = np.empty((rows, n))
    for r in range(rows):
        xv = x[r].astype(np.float64)
        kc = np.ascontiguousarray(k[cls[r]])
        R.ref_klt_one(n, P(kc), P(xv), P(yf[r]), 0)
        R.ref_klt_one(n, P(kc), P(xv), P(yi[r]), 1)
    g.update(klt_k=k, klt_x=x, klt_cls=cls, klt_fwd=yf, klt_inv=yi)

    # ---- per-class energy through the reference CorrelationAccumulator
    log2n, rounds, classes, rows = 6, 2, 4, 300
    n = 64
    angles = rng.uniform(-np.pi, np.pi, (classes, rounds * n * log2n // 2))
    x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
    cls = rng.integers(0, classes, rows).astype(np.uint16)
    e = np.empty((classes, n))
    R.ref_class_energy(log2n, rounds, classes, P(angles), None, 0, P(x), P(cls), rows, P(e))
    g.update(en_angles=angles, en_x=x, en_cls=cls, en_energy=e,
             en_meta=np.array([log2n, rounds, classes], np.int64))

    # ---- memory footprints (fixedpoint.hpp:231-238)
    g["footprints"] = np.array([[kl, ln, r, t, R.ref_memory_footprint(kl, ln, r, t)]
                                for kl in (0, 1) for ln in (2, 4, 6) for r in (1, 2, 3) for t in (1, 35)],
                               np.int64)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
