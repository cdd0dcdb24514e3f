"""RBLK / HYGT formats: the host writers/readers against the reference's own file
readers (oracle/_ref/ref_apply, the CLI's `apply` restated over the unmodified headers)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_APPLY = os.path.join(ROOT, "oracle", "_ref", "ref_apply")
needs_ref = pytest.mark.skipif(not os.path.exists(REF_APPLY), reason="oracle/_ref/ref_apply not built")


def _dataset(tmp, rng, log2n=4, classes=3, count=200, scale=16.0):
    from paper_2505_21728_b200.formats import write_rblk
    n = 1 << log2n
    x = (rng.standard_normal((count, n)) * scale).astype(np.float32)
    cls = rng.integers(0, classes, count).astype(np.uint16)
    path = os.path.join(tmp, "d.rblk")
    write_rblk(path, log2n, classes, cls, x)
    return path, cls, x


def _bundle(tmp, rng, log2n=4, classes=3, rounds=2, quantized=False, name="m.hygt"):
    from paper_2505_21728_b200.formats import write_bundle
    n = 1 << log2n
    a = rounds * log2n * n // 2
    angles = [rng.uniform(-np.pi, np.pi, a) for _ in range(classes)]
    perms = [rng.permutation(n).astype(np.uint16) if c % 2 == 0 else None for c in range(classes)]
    path = os.path.join(tmp, name)
    if quantized:
        codes = [np.mod(np.rint(t / (2 * np.pi) * 256), 256).astype(np.uint8) for t in angles]
        write_bundle(path, log2n, codes=codes, angle_bits=8, perms=perms)
        angles = [2 * np.pi * c.astype(np.float64) / 256 for c in codes]
        return path, angles, perms, codes
    write_bundle(path, log2n, angles=angles, perms=perms)
    return path, angles, perms, None


def test_rblk_roundtrip(tmp_path):
    from paper_2505_21728_b200.formats import read_rblk
    rng = np.random.default_rng(1)
    path, cls, x = _dataset(str(tmp_path), rng)
    log2n, c, cls2, x2 = read_rblk(path)
    assert (log2n, c) == (4, 3)
    assert np.array_equal(cls, cls2) and np.array_equal(x, x2)
    assert os.path.getsize(path) == 12 + 200 * (2 + 64)


@needs_ref
@pytest.mark.parametrize("direction", ["forward", "inverse"])
def test_reference_reader_accepts_our_files(tmp_path, oracle_mod, direction):
    """Files written here are read by the reference's read_bundle/read_rblk and transformed as the
    oracle predicts (the reference computes in fp64 and writes fp32)."""
    from oracle import oracle as O
    from paper_2505_21728_b200.formats import read_rblk
    rng = np.random.default_rng(2)
    tmp = str(tmp_path)
    data, cls, x = _dataset(tmp, rng)
    model, angles, perms, _ = _bundle(tmp, rng)
    out = os.path.join(tmp, "o.rblk")
    r = subprocess.run([REF_APPLY, "--model", model, "--data", data, "--direction", direction, "--out", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    _, _, cls2, y = read_rblk(out)
    assert np.array_equal(cls2, cls)
    full = np.stack([np.stack([np.arange(16) for _ in range(1)] + [p if p is not None else np.arange(16)])
                     for p in perms]).astype(np.uint16)  # [C][R=2][N]: identity between, final perm
    ref = O.apply_batch(4, 2, np.stack(angles), full, 0b10, x, cls, inverse=direction == "inverse")
    assert np.abs(y - ref).max() <= 1e-5 * np.abs(x).max()


@needs_ref
def test_reference_apply_error_codes(tmp_path):
    from paper_2505_21728_b200.formats import write_rblk
    rng = np.random.default_rng(3)
    tmp = str(tmp_path)
    data, _, _ = _dataset(tmp, rng)
    model, _, _, _ = _bundle(tmp, rng, log2n=6)
    out = os.path.join(tmp, "o.rblk")
    r = subprocess.run([REF_APPLY, "--model", model, "--data", data, "--out", out], capture_output=True, text=True)
    assert r.returncode == 1 and "dimension mismatch" in r.stderr
    bad = os.path.join(tmp, "bad.rblk")
    with open(bad, "wb") as f:
        f.write(b"XXXX" + bytes(8))
    r = subprocess.run([REF_APPLY, "--model", model, "--data", bad, "--out", out], capture_output=True, text=True)
    assert r.returncode == 2
    write_rblk(bad, 4, 3, np.array([0, 7], np.uint16), np.zeros((2, 16), np.float32))
    model4, _, _, _ = _bundle(tmp, rng, name="m4.hygt")
    r = subprocess.run([REF_APPLY, "--model", model4, "--data", bad, "--out", out], capture_output=True, text=True)
    assert r.returncode == 2 and "class id out of range" in r.stderr
