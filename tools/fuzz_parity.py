"""Randomised parity sweep on the GPU (development tool): random plans (N, rounds, classes,
permutation masks, arithmetic form, kernel family) and batch sizes through the default kernel
selection against the oracle, float and fixed point, forward and inverse.
    python tools/fuzz_parity.py [--seconds 240] [--seed 1]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2505_21728_b200 import (FixedPlan, HyGTModel, HyGTPlan, KLTPlan, QuantizedHyGTModel, TrigTable,  # noqa: E402
                                   correlation)
from paper_2505_21728_b200.plan import HYGT_PLAN_FORCE_STANDARD  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=240)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--big", action="store_true", help="also batches of 3e5 and 2^20 rows (N <= 64): multi-tile steady state")
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
t0 = time.time()
n_float = n_fixed = n_klt = n_corr = 0
worst = 0.0
worst_what = ""


def close(y, ref, x, what):
    global worst, worst_what
    err = np.asarray(y, np.float64) - ref
    if err.size == 0:
        return
    rel = np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-300)
    mab = np.abs(err).max() if err.size else 0.0
    if rel > worst:
        worst, worst_what = rel, what
    assert rel <= 1e-6 and mab <= 1e-5 * max(np.abs(x).max(), 1e-30), f"{what}: rel {rel:.3e} max-abs {mab:.3e}"


while time.time() - t0 < a.seconds:
    log2n = int(rng.integers(1, 9))
    n = 1 << log2n
    rounds = int(rng.integers(1, 5))
    classes = int(rng.choice([1, 1, 2, 3, 5, 8, 35, 40, 70]))
    rows = int(rng.choice([0, 1, 7, 31, 33, 127, 129, 1000, 4097, 20000, 66000]))
    if a.big and n <= 64 and rng.random() < 0.5:
        rows = int(rng.choice([300001, 1 << 20]))
    if n >= 128:
        rows = min(rows, 20000)
    mask = int(rng.integers(0, 1 << rounds)) if rng.random() < 0.7 else 0
    kind = rng.choice(["float", "float", "fixed", "klt", "corr"])
    what = f"{kind} log2n={log2n} R={rounds} C={classes} rows={rows} mask={mask}"
    angles = rng.uniform(-np.pi, np.pi, (classes, rounds * log2n * n // 2))
    perms = np.tile(np.arange(n, dtype=np.uint16), (classes, rounds, 1))
    for c in range(classes):
        for r in range(rounds):
            if (mask >> r) & 1:
                perms[c, r] = rng.permutation(n).astype(np.uint16)
    scale = float(10.0 ** rng.integers(-3, 4))
    x = (rng.standard_normal((rows, n)) * scale).astype(np.float32)
    cls = rng.integers(0, classes, rows).astype(np.uint16)
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(cls).cuda()
    try:
        if kind == "float":
            final = (mask >> (rounds - 1)) & 1
            models = [HyGTModel(log2n, rounds, angles[c], perms[c, rounds - 1] if final else None) for c in range(classes)]
            inter = None
            if mask & ((1 << (rounds - 1)) - 1):
                inter = perms[:, : rounds - 1].copy()
            flags = HYGT_PLAN_FORCE_STANDARD if rng.random() < 0.3 else 0
            kernel = "auto"
            if log2n >= 6 and classes <= 64 and rng.random() < 0.4:
                kernel = str(rng.choice(["butterfly", "tensor"]))
            plan = HyGTPlan(models, inter, flags=flags, kernel=kernel)
            what += f" flags={flags} kernel={kernel} path={plan.path}"
            y = plan.forward(xd, cd)
            z = plan.inverse(xd, cd)
            plan.sync_status()
            pm = perms if mask else None
            close(y.cpu().numpy(), O.apply_batch(log2n, rounds, angles, pm, mask, x, cls), x, what + " fwd")
            close(z.cpu().numpy(), O.apply_batch(log2n, rounds, angles, pm, mask, x, cls, inverse=True), x, what + " inv")
            n_float += 1
        elif kind == "fixed":
            if log2n > 6:
                continue
            bits, prec = int(rng.integers(4, 9)), int(rng.integers(4, 15))
            codes = rng.integers(0, 1 << bits, (classes, rounds * log2n * n // 2)).astype(np.uint16)
            final = (mask >> (rounds - 1)) & 1
            qm = [QuantizedHyGTModel(log2n, rounds, bits, codes[c], perms[c, rounds - 1] if final else None) for c in range(classes)]
            inter = perms[:, : rounds - 1].copy() if mask & ((1 << (rounds - 1)) - 1) else None
            plan = FixedPlan(qm, TrigTable(bits, prec), inter)
            xi = rng.integers(-(1 << 20), (1 << 20) + 1, (rows, n)).astype(np.int64)
            st, bad, ref = O.apply_batch_fixed(log2n, rounds, bits, prec, codes, perms if mask else None, mask, xi, cls)
            try:
                yi = plan.forward(torch.from_numpy(xi).cuda(), cd).cpu().numpy()
                assert st == 0 and np.array_equal(yi, ref), what + " fixed fwd mismatch"
            except Exception as e:  # the same error outcome at the same row
                if isinstance(e, AssertionError):
                    raise
                assert st != 0 and plan.first_bad == bad, f"{what}: GPU raised {e!r}, oracle status {st} row {bad}"
            n_fixed += 1
        elif kind == "klt":
            if log2n < 1:
                continue
            k = np.stack([np.linalg.qr(rng.standard_normal((n, n)))[0] for _ in range(classes)])
            plan = KLTPlan(k)
            y = plan.forward(xd, cd)
            close(y.cpu().numpy(), O.klt_apply(k, x, cls), x, what + " klt fwd")
            back = plan.inverse(y, cd)
            close(back.cpu().numpy(), x.astype(np.float64), x, what + " klt roundtrip")
            n_klt += 1
        else:
            if log2n < 2 or rows == 0:
                continue
            ref_s, ref_k = O.correlation(log2n, classes, x, cls)
            s, kk = correlation(xd, cd, classes)
            assert np.array_equal(kk.cpu().numpy().astype(np.uint64), ref_k), what
            s = s.cpu().numpy()
            for c in range(classes):
                assert np.abs(s[c] - ref_s[c]).max() <= 1e-12 * max(np.abs(ref_s[c]).max(), 1e-300), what + f" class {c}"
            n_corr += 1
    except AssertionError:
        print("FAIL", what)
        raise
print(f"fuzz ok: {n_float} float, {n_fixed} fixed, {n_klt} klt, {n_corr} correlation cases in {time.time() - t0:.0f} s; "
      f"worst float rel L2 {worst:.2e} ({worst_what})")
