"""GPU parity of the composed-operator path (hygt_gemm.cu: per-class M_c on tcgen05, fp16 3-term
split with per-row power-of-two scaling) against the oracle, over the shapes and edge cases the
bench does not exercise: N = 64 / 128 / 256, 1 / 3 / 35 classes, ragged tile tails (0, 1, 127,
128, 129 rows), inter-round and final permutations, in place, rows at extreme magnitudes, zero
rows, invalid class ids, the fused energy. Tolerances as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

from test_gpu_parity import check_close

pytestmark = pytest.mark.gpu


def _case(log2n, rounds, classes, perms_kind, seed):
    from paper_2505_21728_b200 import HyGTModel, HyGTPlan
    rng = np.random.default_rng(seed)
    n = 1 << log2n
    a = rounds * n * log2n // 2
    angles = rng.uniform(-np.pi, np.pi, (classes, a))
    perms = np.stack([np.stack([rng.permutation(n) for _ in range(rounds)]) for _ in range(classes)]).astype(np.uint16)
    mask = {"none": 0, "final": 1 << (rounds - 1), "inter+final": (1 << rounds) - 1}[perms_kind]
    final = (mask >> (rounds - 1)) & 1
    models = [HyGTModel(log2n, rounds, angles[c], perms[c, rounds - 1] if final else None) for c in range(classes)]
    inter = perms[:, : rounds - 1].copy() if mask & ((1 << (rounds - 1)) - 1) else None
    plan = HyGTPlan(models, inter, kernel="tensor")  # hygt_plan_options: the tensor-core path
    assert plan.path == "gemm"
    return plan, angles, (perms if mask else None), mask, rng


@pytest.mark.parametrize("log2n,rounds,classes,perms_kind", [
    (6, 4, 35, "inter+final"), (6, 2, 1, "none"), (7, 3, 3, "final"), (8, 4, 35, "none"),
    (8, 2, 3, "inter+final"), (8, 1, 1, "final")])
@pytest.mark.parametrize("rows", [1, 127, 129, 5000])
def test_gemm_vs_oracle(cuda, oracle_mod, log2n, rounds, classes, perms_kind, rows):
    plan, angles, perms, mask, rng = _case(log2n, rounds, classes, perms_kind, 100 * log2n + rows)
    n = 1 << log2n
    x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
    cls = rng.integers(0, classes, rows).astype(np.uint16)
    xd = torch.from_numpy(x).to(cuda)
    cd = torch.from_numpy(cls).to(cuda) if classes > 1 else None
    y = plan.forward(xd, cd)
    z = plan.inverse(xd, cd)
    plan.sync_status()
    ref = oracle_mod.apply_batch(log2n, rounds, angles, perms, mask, x, cls)
    refi = oracle_mod.apply_batch(log2n, rounds, angles, perms, mask, x, cls, inverse=True)
    check_close(y.cpu().numpy(), ref, x, f"gemm fwd N={n}")
    check_close(z.cpu().numpy(), refi, x, f"gemm inv N={n}")
    back = plan.inverse(y, cd)
    check_close(back.cpu().numpy(), x, x, "gemm roundtrip")


def test_gemm_empty_inplace_and_energy(cuda, oracle_mod):
    plan, angles, perms, mask, rng = _case(8, 4, 5, "none", 7)
    e = torch.zeros(5, 256, dtype=torch.float64, device=cuda)
    empty = torch.empty(0, 256, device=cuda)
    plan.forward(empty, torch.empty(0, dtype=torch.uint16, device=cuda))
    x = (rng.standard_normal((3001, 256)) * 16).astype(np.float32)
    cls = rng.integers(0, 5, 3001).astype(np.uint16)
    xd = torch.from_numpy(x).to(cuda)
    cd = torch.from_numpy(cls).to(cuda)
    buf = xd.clone()
    plan.forward_energy(buf, cd, e, out=buf)  # in place
    plan.sync_status()
    ref = oracle_mod.apply_batch(8, 4, angles, None, 0, x, cls)
    check_close(buf.cpu().numpy(), ref, x, "gemm in place")
    np.testing.assert_allclose(e.cpu().numpy(), oracle_mod.class_energy(8, 4, angles, None, 0, x, cls), rtol=1e-6)


@pytest.mark.parametrize("scale", [1e-30, 1e-6, 1.0, 1e6, 1e30])
def test_gemm_row_scaling_extremes(cuda, oracle_mod, scale):
    """Each row is scaled by its own power of two before the fp16 split: rows at any magnitude,
    rows mixing magnitudes, and zero rows keep the fp32 bar relative to their own size."""
    plan, angles, perms, mask, rng = _case(8, 2, 2, "final", 3)
    x = (rng.standard_normal((300, 256)) * scale).astype(np.float32)
    x[5] = 0.0
    x[7, ::2] *= 1e-4  # mixed magnitudes inside one row
    cls = rng.integers(0, 2, 300).astype(np.uint16)
    y = plan.forward(torch.from_numpy(x).to(cuda), torch.from_numpy(cls).to(cuda)).cpu().numpy()
    ref = oracle_mod.apply_batch(8, 2, angles, perms, mask, x, cls)
    assert np.all(y[5] == 0.0)
    for r in range(300):
        if r == 5:
            continue
        err = np.linalg.norm(y[r] - ref[r]) / np.linalg.norm(ref[r])
        assert err <= 1e-6, f"row {r}: rel {err:.2e}"


def test_gemm_invalid_class_ids(cuda):
    from paper_2505_21728_b200 import ArgumentError
    plan, angles, perms, mask, rng = _case(8, 2, 3, "none", 9)
    x = torch.randn(1000, 256, device=cuda)
    cls = torch.randint(0, 3, (1000,), device=cuda).to(torch.int16).view(torch.uint16)
    cls.view(torch.int16)[17] = 9
    plan.forward(x, cls)
    with pytest.raises(ArgumentError):
        plan.sync_status()


def test_plan_options_select_and_validate(cuda, knob):
    """hygt_plan_options: "tensor" forces the composed-operator path where supported and is an
    ArgumentError elsewhere; "butterfly" never takes it. At N = 256 the CTA-pair build takes the
    operator-in-TMEM form (same products, the MMA operand roles swapped, so the tensor cores
    round a K step's sum in a different order): equal to the single-CTA build at the fp32 bar,
    and its operand-in-shared-memory form (HYGT_GEMM_TS=0) equal bit for bit."""
    from paper_2505_21728_b200 import ArgumentError, HyGTModel, HyGTPlan
    rng = np.random.default_rng(5)
    ms = [HyGTModel(8, 2, rng.uniform(-np.pi, np.pi, 2 * 8 * 128)) for _ in range(3)]
    assert HyGTPlan(ms).path == "gemm"  # default at N = 256
    assert HyGTPlan(ms, kernel="butterfly").path == "segment"
    with pytest.raises(ArgumentError):
        HyGTPlan([HyGTModel(4, 2, rng.uniform(-np.pi, np.pi, 2 * 4 * 8))], kernel="tensor")
    with pytest.raises(ArgumentError):
        HyGTPlan(ms, kernel="bogus")
    x = torch.randn(4000, 256, device=cuda) * 16
    cls = torch.randint(0, 3, (4000,), device=cuda).to(torch.int16).view(torch.uint16)
    y1 = HyGTPlan(ms, kernel="tensor", cta_pairs=True).forward(x, cls)
    y0 = HyGTPlan(ms, kernel="tensor", cta_pairs=False).forward(x, cls)
    check_close(y1.cpu().numpy(), y0.cpu().numpy(), x.cpu().numpy(), "pair (TS) vs single")
    knob("HYGT_GEMM_TS", "0")
    y2 = HyGTPlan(ms, kernel="tensor", cta_pairs=True).forward(x, cls)
    assert torch.equal(y0, y2)  # same per-row arithmetic, only the operand staging differs


@pytest.mark.parametrize("log2n,classes", [(8, 400), (6, 300)])
def test_gemm_many_classes_and_variants(cuda, oracle_mod, log2n, classes, knob):
    """Many classes: at N = 256 more than 384 classes do not leave room for the per-class tile
    table next to the resident B hi halves, so the kernel takes the variant with units of 128
    columns and streamed B; at N = 64 the 256-row sub-tiled tiles meet a few rows per class.
    Forward with energy and inverse against the oracle, and the single-CTA build equal to the
    CTA-pair build bit for bit (same per-row arithmetic and accumulation order; at N = 256 the
    pair build's operand-in-shared-memory form, HYGT_GEMM_TS=0, and the default operator-in-TMEM
    form at the fp32 bar)."""
    from paper_2505_21728_b200 import HyGTPlan
    plan, angles, perms, mask, rng = _case(log2n, 2, classes, "none", 41 + classes)
    n = 1 << log2n
    rows = 20000
    x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
    cls = rng.integers(0, classes, rows).astype(np.uint16)
    xd, cd = torch.from_numpy(x).to(cuda), torch.from_numpy(cls).to(cuda)
    e = torch.zeros(classes, n, dtype=torch.float64, device=cuda)
    y = plan.forward_energy(xd, cd, e)
    z = plan.inverse(xd, cd)
    plan.sync_status()
    check_close(y.cpu().numpy(), oracle_mod.apply_batch(log2n, 2, angles, perms, mask, x, cls), x, f"fwd C={classes}")
    check_close(z.cpu().numpy(), oracle_mod.apply_batch(log2n, 2, angles, perms, mask, x, cls, inverse=True), x, f"inv C={classes}")
    np.testing.assert_allclose(e.cpu().numpy(), oracle_mod.class_energy(log2n, 2, angles, None, 0, x, cls), rtol=2e-6)
    from paper_2505_21728_b200 import HyGTModel
    models = [HyGTModel(log2n, 2, angles[c]) for c in range(classes)]
    y1 = HyGTPlan(models, kernel="tensor", cta_pairs=False).forward(xd, cd)
    if n == 256:
        check_close(y.cpu().numpy(), y1.cpu().numpy(), x, "pair (TS) vs single")
        knob("HYGT_GEMM_TS", "0")
        y = HyGTPlan(models, kernel="tensor", cta_pairs=True).forward(xd, cd)
    assert torch.equal(y, y1)


@pytest.mark.parametrize("classes", [400, 35])
def test_gemm_n256_roundtrip_repeated(cuda, classes):
    """N = 256 on the CTA pairs' operator-in-TMEM form, repeated: a class change on almost every
    tile (400 classes, ~50 rows each) reloads the operator in TMEM over and over, and each
    epilogue reads half of its row factors from the peer CTA over DSMEM (a CTA-scope release on
    that hand-off once let stale power-of-two factors through, intermittently). Forward then
    inverse returns the input, forward with energy equals forward bit for bit, every time."""
    from paper_2505_21728_b200 import HyGTModel, HyGTPlan
    rng = np.random.default_rng(70 + classes)
    models = [HyGTModel(8, 2, rng.uniform(-np.pi, np.pi, 2 * 8 * 128)) for _ in range(classes)]
    plan = HyGTPlan(models, kernel="tensor")
    x = torch.from_numpy((rng.standard_normal((20000, 256)) * 16).astype(np.float32)).to(cuda)
    cls = torch.from_numpy(rng.integers(0, classes, 20000).astype(np.uint16)).to(cuda)
    scale = float(x.abs().max())
    for _ in range(4):
        y = plan.forward(x, cls)
        e = torch.zeros(classes, 256, dtype=torch.float64, device=cuda)
        y2 = plan.forward_energy(x, cls, e)
        z = plan.inverse(y, cls)
        assert torch.equal(y, y2)
        assert float((z - x).abs().max()) <= 1e-5 * scale
