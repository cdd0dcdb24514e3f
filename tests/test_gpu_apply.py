"""The GPU drop-in for the reference CLI's `apply` (paper_2505_21728_b200/hygt_gpu_apply) against
the reference's own apply (oracle/_ref/ref_apply over the unmodified headers) on the same files:
float outputs within the fp32 bar, fixed-point outputs byte-identical, same exit codes."""
import os
import subprocess

import numpy as np
import pytest

from test_formats import REF_APPLY, ROOT, _bundle, _dataset

GPU_APPLY = os.path.join(ROOT, "paper_2505_21728_b200", "hygt_gpu_apply")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(REF_APPLY), reason="oracle/_ref/ref_apply not built")]


def _run(exe, model, data, out, direction="forward", arithmetic="float"):
    return subprocess.run([exe, "--model", model, "--data", data, "--direction", direction,
                           "--arithmetic", arithmetic, "--out", out], capture_output=True, text=True)


def _both(tmp, model, data, direction, arithmetic):
    from paper_2505_21728_b200.formats import read_rblk
    a, b = os.path.join(tmp, "gpu.rblk"), os.path.join(tmp, "ref.rblk")
    rg = _run(GPU_APPLY, model, data, a, direction, arithmetic)
    rr = _run(REF_APPLY, model, data, b, direction, arithmetic)
    assert rg.returncode == rr.returncode == 0, (rg.stderr, rr.stderr)
    return a, b, read_rblk(a), read_rblk(b)


@pytest.mark.parametrize("log2n,classes", [(4, 5), (6, 3), (8, 2), (3, 1)])
@pytest.mark.parametrize("direction", ["forward", "inverse"])
def test_gpu_apply_float_matches_reference(cuda, tmp_path, log2n, classes, direction):
    rng = np.random.default_rng(10 + log2n)
    tmp = str(tmp_path)
    data, _, x = _dataset(tmp, rng, log2n=log2n, classes=classes, count=3001)
    model, _, _, _ = _bundle(tmp, rng, log2n=log2n, classes=classes, rounds=3)
    _, _, (l1, c1, cls1, y1), (l2, c2, cls2, y2) = _both(tmp, model, data, direction, "float")
    assert (l1, c1) == (l2, c2) and np.array_equal(cls1, cls2)
    assert np.abs(y1.astype(np.float64) - y2).max() <= 1e-5 * np.abs(x).max()
    assert np.linalg.norm(y1.astype(np.float64) - y2) <= 1e-6 * np.linalg.norm(y2)


def test_gpu_apply_unequal_rounds(cuda, tmp_path):
    """Classes with fewer rounds are padded with identity rounds (exact)."""
    from paper_2505_21728_b200.formats import write_bundle
    rng = np.random.default_rng(21)
    tmp = str(tmp_path)
    data, _, x = _dataset(tmp, rng, log2n=4, classes=3, count=999)
    angles = [rng.uniform(-np.pi, np.pi, r * 4 * 8) for r in (1, 3, 2)]
    model = os.path.join(tmp, "u.hygt")
    write_bundle(model, 4, angles=angles, perms=[None, rng.permutation(16), None])
    _, _, (_, _, _, y1), (_, _, _, y2) = _both(tmp, model, data, "forward", "float")
    assert np.abs(y1.astype(np.float64) - y2).max() <= 1e-5 * np.abs(x).max()


@pytest.mark.parametrize("log2n", [4, 6])
@pytest.mark.parametrize("direction", ["forward", "inverse"])
def test_gpu_apply_quantized_bundle(cuda, tmp_path, log2n, direction):
    rng = np.random.default_rng(30 + log2n)
    tmp = str(tmp_path)
    data, _, x = _dataset(tmp, rng, log2n=log2n, classes=4, count=2048, scale=300.0)
    model, _, _, _ = _bundle(tmp, rng, log2n=log2n, classes=4, rounds=2, quantized=True)
    _, _, (_, _, _, y1), (_, _, _, y2) = _both(tmp, model, data, direction, "float")  # dequantized
    assert np.abs(y1.astype(np.float64) - y2).max() <= 1e-5 * np.abs(x).max()
    a, b, _, _ = _both(tmp, model, data, direction, "fixed")
    with open(a, "rb") as fa, open(b, "rb") as fb:
        assert fa.read() == fb.read()  # bit-exact fixed point, byte-identical files


def test_gpu_apply_error_codes(cuda, tmp_path):
    from paper_2505_21728_b200.formats import write_rblk
    rng = np.random.default_rng(40)
    tmp = str(tmp_path)
    data, _, _ = _dataset(tmp, rng, log2n=4, classes=3, count=100)
    out = os.path.join(tmp, "o.rblk")
    cases = []
    m64, _, _, _ = _bundle(tmp, rng, log2n=6, classes=3, name="m64.hygt")
    cases.append((m64, data, "float"))                        # dimension mismatch -> 1
    m2, _, _, _ = _bundle(tmp, rng, log2n=4, classes=2, name="m2.hygt")
    cases.append((m2, data, "float"))                         # class count mismatch -> 1
    mf, _, _, _ = _bundle(tmp, rng, log2n=4, classes=3, name="mf.hygt")
    cases.append((mf, data, "fixed"))                         # fixed on a float bundle -> 1
    bad = os.path.join(tmp, "bad.rblk")
    with open(bad, "wb") as f:
        f.write(b"NOPE" + bytes(8))
    cases.append((mf, bad, "float"))                          # bad magic -> 2
    oob = os.path.join(tmp, "oob.rblk")
    write_rblk(oob, 4, 3, np.array([0, 3], np.uint16), np.zeros((2, 16), np.float32))
    cases.append((mf, oob, "float"))                          # class id out of range -> 2
    mq, _, _, _ = _bundle(tmp, rng, log2n=4, classes=3, quantized=True, name="mq.hygt")
    big = os.path.join(tmp, "big.rblk")
    xb = np.zeros((5, 16), np.float32)
    xb[3, 7] = 2.0 ** 21
    write_rblk(big, 4, 3, np.zeros(5, np.uint16), xb)
    cases.append((mq, big, "fixed"))                          # |x| > 2^20 -> 1
    for model, d, arith in cases:
        rg = _run(GPU_APPLY, model, d, out, arithmetic=arith)
        rr = _run(REF_APPLY, model, d, out, arithmetic=arith)
        assert rg.returncode == rr.returncode != 0, (model, d, arith, rg.stderr, rr.stderr)
        assert rg.stderr.startswith("error: ")


@pytest.mark.parametrize("log2n,classes", [(2, 1), (4, 3), (6, 3)])
def test_gpu_apply_identity_model_reproduces_input_bytes(cuda, tmp_path, log2n, classes):
    """test_cli.cpp:185-190: `apply` with HyGTModel::zeros writes the input file byte for byte
    (every butterfly is the exact identity on the GPU too: cos = 1, sin = 0)."""
    from paper_2505_21728_b200.formats import write_bundle
    rng = np.random.default_rng(50 + log2n)
    tmp = str(tmp_path)
    data, _, _ = _dataset(tmp, rng, log2n=log2n, classes=classes, count=1500)
    model = os.path.join(tmp, "ident.hygt")
    write_bundle(model, log2n, angles=[np.zeros(log2n * (1 << log2n) // 2) for _ in range(classes)])
    for direction in ("forward", "inverse"):
        out = os.path.join(tmp, f"ident_{direction}.rblk")
        r = _run(GPU_APPLY, model, data, out, direction, "float")
        assert r.returncode == 0, r.stderr
        with open(out, "rb") as fa, open(data, "rb") as fb:
            assert fa.read() == fb.read()
