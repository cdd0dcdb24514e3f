"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle / golden vectors.

Tolerances (fp32 GPU vs fp64 reference, SURVEY.md §8 c4 / BASELINE.md):
    relative L2 over the batch <= 1e-6, max-abs <= 1e-5 * max|x|; energy sums rel <= 1e-5;
    fixed point: bit-exact, identical error outcomes.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL_L2 = 1e-6
MAX_ABS = 1e-5


def check_close(y, ref, x, what=""):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = max(float(np.abs(x).max()), 1e-30)
    err = y - ref
    rel = np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-300)
    mab = float(np.abs(err).max()) if err.size else 0.0
    assert rel <= REL_L2, f"{what}: rel L2 {rel:.3e}"
    assert mab <= MAX_ABS * scale, f"{what}: max abs {mab:.3e} vs {MAX_ABS * scale:.3e}"
    return rel, mab


def _plan(models, perms_inter=None, standard=False):
    from paper_2505_21728_b200 import HyGTPlan
    from paper_2505_21728_b200.plan import HYGT_PLAN_FORCE_STANDARD
    return HyGTPlan(models, perms_inter, flags=HYGT_PLAN_FORCE_STANDARD if standard else 0)


def _models(log2n, rounds, angles, perms=None, mask=0):
    from paper_2505_21728_b200 import HyGTModel
    final = perms is not None and (mask >> (rounds - 1)) & 1
    return [HyGTModel(log2n, rounds, angles[c], perms[c, rounds - 1] if final else None)
            for c in range(angles.shape[0])]


def _inter(perms, mask, rounds):
    if perms is None or not (mask & ((1 << (rounds - 1)) - 1)):
        return None
    ip = perms[:, : rounds - 1].copy()
    for r in range(rounds - 1):
        if not (mask >> r) & 1:
            ip[:, r] = np.arange(ip.shape[-1])
    return ip


LAYOUTS = {1: [0], 2: [0], 3: [0], 4: [0, 2], 5: [0], 6: [0, 1, 2], 7: [2], 8: [1, 2]}
# tile-path layouts (log2 TPV, rows per lane group) for N <= 32; the generic kernel runs with
# HYGT_TILE=0.
TILE_LAYOUTS = {2: [(0, 2)], 3: [(1, 2), (0, 2)], 4: [(1, 2), (2, 2), (0, 1)],
                5: [(2, 2), (3, 2)]}


SEG_VARIANTS = {6: [0, 1, 2, 3], 7: [4, 5], 8: [6, 7, 8, 9, 10]}
STAGE_LOG2N = (4,)
SEG2_LOG2N = (6,)


def _variants(log2n):
    out = _variants_butterfly(log2n)
    for v in out:
        v.setdefault("HYGT_GEMM", "0")
    if log2n in GEMM_LOG2N:  # composed operator on the tensor cores
        out.append({"HYGT_GEMM": "1"})
    return out


GEMM_LOG2N = (6, 7, 8)


def _variants_butterfly(log2n):
    out = [{"HYGT_JIT": "0", "HYGT_STAGE": "0", "HYGT_TILE": "0", "HYGT_SEGMENT": "0", "HYGT_SEG2": "0",
            "HYGT_CLS": "0", "HYGT_CLS_JIT": "0", "HYGT_LANES_LOG2": str(l)} for l in LAYOUTS[log2n]]
    for v in SEG_VARIANTS.get(log2n, []):
        out.append({"HYGT_SEG2": "0", "HYGT_CLS": "0", "HYGT_CLS_JIT": "0", "HYGT_SEGMENT": "1", "HYGT_SEG_VARIANT": str(v)})
    if log2n in SEG2_LOG2N:  # thread-per-row kernels over global class buckets
        out.append({"HYGT_SEG2": "1", "HYGT_CLS": "0", "HYGT_CLS_JIT": "0"})
        out.append({"HYGT_CLS": "1", "HYGT_CLS_JIT": "0"})  # per-class launches, parameter tables
        out.append({"HYGT_CLS_JIT": "1"})  # per-class launches, NVRTC-specialised kernels
        out.append({"HYGT_CLS_JIT": "1", "HYGT_CLS_PTX": "1"})  # the same with PTX bodies
    for l, v in TILE_LAYOUTS.get(log2n, []):
        out.append({"HYGT_JIT": "0", "HYGT_STAGE": "0", "HYGT_TILE": "1", "HYGT_CLS_JIT": "0",
                    "HYGT_TILE_L": str(l), "HYGT_TILE_VPT": str(v)})
    if log2n == 5:  # per-class NVRTC chain (multi-class plans the all-class JIT does not take)
        out.append({"HYGT_JIT": "0", "HYGT_CLS_JIT": "1"})
    if log2n in STAGE_LOG2N:  # TMA-staged tile kernel
        out.append({"HYGT_JIT": "0", "HYGT_STAGE": "1"})
        out.append({"HYGT_JIT": "0", "HYGT_STAGE": "1", "HYGT_STAGE_ROWS": "136"})
    if log2n <= 5:  # plan-specialised NVRTC kernel (served for plans with <= 4 classes)
        out.append({"HYGT_JIT": "2"})
    return out


@pytest.mark.parametrize("standard", [False, True])
@pytest.mark.parametrize("k", range(10))
def test_golden_float_all_layouts(cuda, golden, k, standard, knob):
    log2n, rounds, classes, mask = (int(v) for v in golden[f"f{k}_meta"])
    angles, perms = golden[f"f{k}_angles"], golden[f"f{k}_perms"]
    x, cls = golden[f"f{k}_x"], golden[f"f{k}_cls"]
    xd = torch.from_numpy(x).to(cuda)
    cd = torch.from_numpy(cls).to(cuda)
    for env in _variants(log2n):
        for k_, v_ in env.items():
            knob(k_, v_)
        lanes = env
        plan = _plan(_models(log2n, rounds, angles, perms, mask), _inter(perms, mask, rounds), standard)
        y = plan.forward(xd, cd)
        plan.sync_status()
        check_close(y.cpu().numpy(), golden[f"f{k}_fwd"], x, f"fwd k={k} L={lanes} {plan.algorithm}")
        z = plan.inverse(xd, cd)
        plan.sync_status()
        check_close(z.cpu().numpy(), golden[f"f{k}_inv"], x, f"inv k={k} L={lanes}")
        back = plan.inverse(y, cd)
        check_close(back.cpu().numpy(), x, x, f"roundtrip k={k} L={lanes}")


@pytest.mark.parametrize("config", [1, 2, 3, 5])
def test_config_shapes_vs_oracle(cuda, oracle_mod, config):
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(config)
    rows = 8192 if config != 5 else 2048
    cls = w.make_classes(rows)
    x = w.make_rows(rows, cls)
    plan = _plan(w.models, w.perms)
    inter_mask = ((1 << (w.cfg.rounds - 1)) - 1) if w.perms is not None else 0
    full = None
    if w.perms is not None:
        full = np.concatenate([w.perms, np.tile(np.arange(w.n, dtype=np.uint16), (w.cfg.classes, 1, 1))], 1)
    xh, ch = x.cpu().numpy(), cls.cpu().numpy()
    ref_f = oracle_mod.apply_batch(w.cfg.log2_n, w.cfg.rounds, w.angles, full, inter_mask, xh, ch)
    y = plan.forward(x, cls)
    plan.sync_status()
    check_close(y.cpu().numpy(), ref_f, xh, f"cfg{config} fwd ({plan.algorithm})")
    ref_i = oracle_mod.apply_batch(w.cfg.log2_n, w.cfg.rounds, w.angles, full, inter_mask, xh, ch, inverse=True)
    z = plan.inverse(x, cls)
    check_close(z.cpu().numpy(), ref_i, xh, f"cfg{config} inv")
    back = plan.inverse(y, cls)
    check_close(back.cpu().numpy(), xh, xh, f"cfg{config} roundtrip")


def test_edge_counts_inplace_and_identity(cuda):
    from paper_2505_21728_b200 import HyGTModel, HyGTPlan
    rng = np.random.default_rng(5)
    m = HyGTModel(4, 2, rng.uniform(-np.pi, np.pi, 64))
    plan = HyGTPlan(m)
    for count in [0, 1, 31, 33, 1000]:
        x = torch.from_numpy((rng.standard_normal((count, 16)) * 16).astype(np.float32)).to(cuda)
        y = plan.forward(x)
        if count:
            xi = x.clone()
            plan.forward(xi, out=xi)  # in place
            assert torch.equal(xi, y)
            back = plan.inverse(y)
            check_close(back.cpu().numpy(), x.cpu().numpy(), x.cpu().numpy(), f"count={count}")
    # zero-angle model is the identity, bit for bit (test_transform.cpp:118-124)
    for standard in (False, True):
        z = _plan([HyGTModel.zeros(6, 3)], standard=standard)
        x = torch.randn(777, 64, device=cuda)
        assert torch.equal(z.forward(x), x)
        assert torch.equal(z.inverse(x), x)


def test_quarter_turn_kats(cuda):
    import math
    from paper_2505_21728_b200 import forward, inverse, HyGTModel
    y = forward(HyGTModel(1, 1, [math.pi / 2]), [1.0, 0.0])
    assert abs(y[0]) < 1e-7 and abs(y[1] + 1) < 1e-7
    y = forward(HyGTModel(2, 1, [math.pi / 2, math.pi / 2, 0, 0]), [1, 2, 3, 4])
    np.testing.assert_allclose(y, [2, -1, 4, -3], atol=1e-6)
    m = HyGTModel(1, 1, [0.0], [1, 0])  # permutation gathers by index (test_transform.cpp:196-202)
    assert list(forward(m, [3.0, 4.0])) == [4.0, 3.0]
    assert list(inverse(m, [4.0, 3.0])) == [3.0, 4.0]
    with pytest.raises(Exception):
        forward(HyGTModel.zeros(2, 1), [1.0, 2.0])


def test_invalid_class_ids_raise(cuda):
    from paper_2505_21728_b200 import ArgumentError, HyGTModel, HyGTPlan
    rng = np.random.default_rng(9)
    models = [HyGTModel(4, 2, rng.uniform(-3, 3, 64)) for _ in range(3)]
    plan = HyGTPlan(models)
    x = torch.randn(100, 16, device=cuda)
    cls = torch.from_numpy(rng.integers(0, 3, 100).astype(np.uint16)).to(cuda)
    plan.forward(x, cls)
    plan.sync_status()
    cls[17] = 3
    plan.forward(x, cls)
    with pytest.raises(ArgumentError):
        plan.sync_status()
    one = HyGTPlan(models[:1])
    one.forward(x, cls)
    with pytest.raises(ArgumentError):
        one.sync_status()


def test_bucketing_large_batch_roundtrip(cuda):
    """Full config-2 size (2^24 rows, 1 GiB): size-independent properties -- round trip and
    norm preservation -- through the multi-tile bucketing path."""
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(2)
    cls = w.make_classes(w.cfg.count)
    x = w.make_rows(w.cfg.count, cls)
    plan = _plan(w.models, w.perms)
    ws = torch.zeros(plan.workspace_bytes(w.cfg.count), dtype=torch.uint8, device=cuda)
    y = plan.forward(x, cls, workspace=ws)
    back = plan.inverse(y, cls, workspace=ws, reuse_buckets=True)
    plan.sync_status(ws)
    err = (back - x).abs().max().item()
    assert err <= MAX_ABS * x.abs().max().item()
    nx = x.double().pow(2).sum(1)
    ny = y.double().pow(2).sum(1)
    assert ((ny - nx).abs() / nx).max().item() < 1e-5
    # a random sample of rows against the oracle
    from oracle import oracle as O
    idx = torch.randint(0, w.cfg.count, (4096,), device=cuda)
    full = np.concatenate([w.perms, np.tile(np.arange(16, dtype=np.uint16), (35, 1, 1))], 1)
    ref = O.apply_batch(4, 3, w.angles, full, 3, x[idx].cpu().numpy(), cls.to(torch.int32)[idx].cpu().numpy().astype(np.uint16))
    check_close(y[idx].cpu().numpy(), ref, x[idx].cpu().numpy(), "cfg2 full-size sample")


@pytest.mark.parametrize("kernel", ["butterfly", "tensor"])
def test_energy_vs_oracle_and_full_size(cuda, oracle_mod, golden, kernel):
    """Fused per-class energy against the reference accumulator's golden (N = 64) and the
    config-5 shape (N = 256, 35 classes) against the oracle, on both kernel families."""
    from paper_2505_21728_b200 import HyGTModel, HyGTPlan
    log2n, rounds, classes = (int(v) for v in golden["en_meta"])
    angles = golden["en_angles"]
    plan = HyGTPlan([HyGTModel(log2n, rounds, angles[c]) for c in range(classes)], kernel=kernel)
    x = torch.from_numpy(golden["en_x"]).to(cuda)
    cls = torch.from_numpy(golden["en_cls"]).to(cuda)
    e = torch.zeros(classes, 1 << log2n, dtype=torch.float64, device=cuda)
    plan.forward_energy(x, cls, e)
    np.testing.assert_allclose(e.cpu().numpy(), golden["en_energy"], rtol=1e-5, atol=1e-3)
    # config 5 shape on a subset vs the oracle
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(5)
    rows = 1 << 14
    cls = w.make_classes(rows)
    x = w.make_rows(rows, cls)
    plan = HyGTPlan(w.models, kernel=kernel)
    e = torch.zeros(35, 256, dtype=torch.float64, device=cuda)
    plan.forward_energy(x, cls, e)
    ref = oracle_mod.class_energy(8, 4, w.angles, None, 0, x.cpu().numpy(), cls.cpu().numpy())
    np.testing.assert_allclose(e.cpu().numpy(), ref, rtol=2e-6)


@pytest.mark.parametrize("k", range(7))
@pytest.mark.parametrize("fixed_jit", ["1", "0"])
def test_fixed_golden_bit_exact(cuda, golden, k, fixed_jit, knob):
    from paper_2505_21728_b200 import ArgumentError, FixedPlan, QuantizedHyGTModel, TrigTable
    knob("HYGT_FIXED_JIT", fixed_jit)
    log2n, rounds, b, p, with_perm = (int(v) for v in golden[f"x{k}_meta"])
    perm = golden[f"x{k}_perm"] if with_perm else None
    m = QuantizedHyGTModel(log2n, rounds, b, golden[f"x{k}_codes"], perm)
    plan = FixedPlan(m, TrigTable(b, p))
    x = golden[f"x{k}_x"]
    st = golden[f"x{k}_fwd_status"]
    xd = torch.from_numpy(x).to(cuda)
    first = int(np.argmax(st != 0)) if (st != 0).any() else x.shape[0]
    if first < x.shape[0]:
        with pytest.raises(ArgumentError):
            plan.forward(xd)
        assert plan.first_bad == first
    ok = np.nonzero(st == 0)[0]
    y = plan.forward(torch.from_numpy(x[ok]).to(cuda)).cpu().numpy()
    assert np.array_equal(y, golden[f"x{k}_fwd"][ok])
    ist = golden[f"x{k}_inv_status"]
    ok2 = np.nonzero((st == 0) & (ist == 0))[0]
    z = plan.inverse(torch.from_numpy(golden[f"x{k}_fwd"][ok2]).to(cuda)).cpu().numpy()
    assert np.array_equal(z, golden[f"x{k}_inv"][ok2])


@pytest.fixture(scope="module")
def golden_long():
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_fixed_long.npz"))


@pytest.mark.parametrize("name", ["grow16", "long64", "grow256", "mixed32"])
def test_fixed_long_models_overflow_and_int32_gate(cuda, golden_long, name):
    """Long low-precision models (tests/gen_golden_fixed_long.py, from the unmodified reference):
    R * log2N = 160..480 passes at p = 4/5. Valid rows grow past 2^31 (grow16/grow256), so the
    plan must leave the int32 kernels (their bound fails) for the int64 one; rows at 2^20
    overflow 2^46 and the reference throws OverflowError (fixedpoint.hpp:177-179): the GPU
    reports status 4 at the same first row. Every valid row is bit-exact."""
    from paper_2505_21728_b200 import FixedPlan, QuantizedHyGTModel, TrigTable
    from paper_2505_21728_b200.errors import OverflowError_
    g = golden_long
    log2n, rounds, b, p, with_perm = (int(v) for v in g[name + "_meta"])
    perm = g[name + "_perm"] if with_perm else None
    plan = FixedPlan(QuantizedHyGTModel(log2n, rounds, b, g[name + "_codes"], perm), TrigTable(b, p))
    x = g[name + "_x"]
    for d, key in ((0, "fwd"), (1, "inv")):
        st = g[f"{name}_{key}_status"]
        run = plan.forward if d == 0 else plan.inverse
        xd = torch.from_numpy(x).to(cuda)
        if (st != 0).any():
            first = int(np.argmax(st != 0))
            assert int(st[first]) == 4  # OverflowError in the reference
            with pytest.raises(OverflowError_):
                run(xd)
            assert plan.first_bad == first
        ok = np.nonzero(st == 0)[0]
        y = run(torch.from_numpy(x[ok]).to(cuda)).cpu().numpy()
        assert np.array_equal(y, g[f"{name}_{key}"][ok]), f"{name} {key}: not bit-exact"


@pytest.mark.parametrize("kernel", ["default", "stage", "row", "warp"])
def test_fixed_random_multiclass_vs_oracle(cuda, oracle_mod, kernel, knob):
    """Bit-exact vs the oracle through every fixed-point kernel: the per-class NVRTC chain
    (default, N <= 64), the staged one (N = 16), the thread-per-row one (N <= 64) and the
    warp-per-row one."""
    from paper_2505_21728_b200 import FixedPlan, QuantizedHyGTModel, TrigTable
    if kernel != "default":
        knob("HYGT_FIXED_JIT", "0")
    if kernel in ("row", "warp"):
        knob("HYGT_FIXED_STAGE", "0")
    if kernel == "warp":
        knob("HYGT_FIXED_ROW", "0")
    rng = np.random.default_rng(11)
    for log2n, rounds, classes in [(4, 3, 35), (6, 4, 5), (8, 2, 3)]:
        n = 1 << log2n
        a = rounds * n * log2n // 2
        codes = rng.integers(0, 256, (classes, a)).astype(np.uint16)
        inter = np.stack([np.stack([rng.permutation(n) for _ in range(rounds - 1)]) for _ in range(classes)]).astype(np.uint16)
        full = np.concatenate([inter, np.tile(np.arange(n, dtype=np.uint16), (classes, 1, 1))], 1)
        x = rng.integers(-(1 << 20), (1 << 20) + 1, (3000, n)).astype(np.int64)
        cls = rng.integers(0, classes, 3000).astype(np.uint16)
        plan = FixedPlan([QuantizedHyGTModel(log2n, rounds, 8, codes[c]) for c in range(classes)],
                         TrigTable(8, 10), inter)
        y = plan.forward(torch.from_numpy(x).cuda(), torch.from_numpy(cls).cuda()).cpu().numpy()
        st, bad, ref = oracle_mod.apply_batch_fixed(log2n, rounds, 8, 10, codes, full, (1 << (rounds - 1)) - 1, x, cls)
        assert st == 0
        assert np.array_equal(y, ref)
        # inverse on legal inputs (forward outputs can exceed 2^20 at large N: compare status too)
        st2, bad2, ref2 = oracle_mod.apply_batch_fixed(log2n, rounds, 8, 10, codes, full, (1 << (rounds - 1)) - 1, x, cls, inverse=True)
        z = plan.inverse(torch.from_numpy(x).cuda(), torch.from_numpy(cls).cuda()).cpu().numpy()
        assert np.array_equal(z, ref2)


def test_klt_golden(cuda, golden):
    from paper_2505_21728_b200 import KLTPlan
    plan = KLTPlan(golden["klt_k"])  # n = 16: tcgen05 3xTF32 path
    x = golden["klt_x"]
    xd = torch.from_numpy(x).to(cuda)
    cd = torch.from_numpy(golden["klt_cls"]).to(cuda)
    check_close(plan.forward(xd, cd).cpu().numpy(), golden["klt_fwd"], x, "klt fwd")
    check_close(plan.inverse(xd, cd).cpu().numpy(), golden["klt_inv"], x, "klt inv")


def test_klt_config4_vs_oracle(cuda, oracle_mod):
    from paper_2505_21728_b200 import KLTPlan
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(4)
    k = w.klt_bases()
    plan = KLTPlan(k)
    cls = w.make_classes(8192)
    x = w.make_rows(8192, cls)
    y = plan.forward(x, cls)
    ref = oracle_mod.klt_apply(k, x.cpu().numpy(), cls.cpu().numpy())
    check_close(y.cpu().numpy(), ref, x.cpu().numpy(), "cfg4 klt fwd")
    back = plan.inverse(y, cls)
    check_close(back.cpu().numpy(), x.cpu().numpy(), x.cpu().numpy(), "cfg4 klt roundtrip")
    # tails and a single class
    one = KLTPlan(k[:1])
    xs = x[:1000]
    ys = one.forward(xs)
    ref1 = oracle_mod.klt_apply(k[:1], xs.cpu().numpy())
    check_close(ys.cpu().numpy(), ref1, xs.cpu().numpy(), "klt single class")


def test_klt_multi_tile_pipeline(cuda, oracle_mod):
    """Config-4 KLT at a size where every CTA runs several tiles per class (the software
    pipeline's steady state): round trip over all rows, a random sample against the oracle."""
    from paper_2505_21728_b200 import KLTPlan
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(4)
    k = w.klt_bases()
    plan = KLTPlan(k)
    rows = 1 << 21  # ~60K rows = ~470 tiles of 128 per class, > 3 per CTA
    cls = w.make_classes(rows)
    x = w.make_rows(rows, cls)
    y = plan.forward(x, cls)
    back = plan.inverse(y, cls)
    err = (torch.linalg.vector_norm(back - x) / torch.linalg.vector_norm(x)).item()
    assert err < 1e-6, err
    idx = np.random.default_rng(3).choice(rows, 4096, replace=False)
    xs, cs = x.cpu().numpy()[idx], cls.cpu().numpy()[idx]
    ref = oracle_mod.klt_apply(k, xs, cs)
    check_close(y.cpu().numpy()[idx], ref, xs, "klt multi-tile sample")


@pytest.mark.parametrize("n,classes,rows", [(64, 3, 777), (128, 5, 3001), (256, 4, 2049), (256, 1, 300)])
def test_klt_grouped_gemm_sizes(cuda, oracle_mod, n, classes, rows):
    """The KLT on the tensor-core grouped GEMM at N = 64 / 128 / 256 (random orthogonal bases,
    matrix.hpp:70-88), ragged class runs, in place, a single class without ids."""
    from paper_2505_21728_b200 import KLTPlan
    k = np.stack([oracle_mod.random_orthogonal(100 + c, n) for c in range(classes)])
    plan = KLTPlan(k)
    rng = np.random.default_rng(n + rows)
    x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
    cls = rng.integers(0, classes, rows).astype(np.uint16)
    xd = torch.from_numpy(x).to(cuda)
    cd = torch.from_numpy(cls).to(cuda) if classes > 1 else None
    y = plan.forward(xd, cd)
    ref = oracle_mod.klt_apply(k, x, cls if classes > 1 else None)
    check_close(y.cpu().numpy(), ref, x, f"klt N={n} fwd")
    refi = oracle_mod.klt_apply(k, x, cls if classes > 1 else None, inverse=True)
    z = xd.clone()
    plan.inverse(z, cd, out=z)  # in place
    check_close(z.cpu().numpy(), refi, x, f"klt N={n} inv")


@pytest.mark.parametrize("log2n", [5, 6])
def test_clsjit_steady_state(cuda, oracle_mod, log2n):
    """Per-class NVRTC chain at a size where each warp runs several batches of its class (the
    next-batch id / L2 prefetch path): round trip over all rows, a sample against the oracle."""
    from paper_2505_21728_b200 import HyGTModel
    rng = np.random.default_rng(21)
    C, R, n = 6, 3, 1 << log2n  # > 4 classes: N = 32 plans would otherwise take the all-class JIT
    angles = rng.uniform(-np.pi, np.pi, (C, R * log2n * n // 2))
    perms = np.stack([np.stack([rng.permutation(n) for _ in range(R)]) for _ in range(C)]).astype(np.uint16)
    plan = _plan([HyGTModel(log2n, R, angles[c], perms[c, R - 1]) for c in range(C)], perms[:, : R - 1].copy())
    assert plan.path == "clsjit"
    rows = (1 << 27) // (4 * n)  # 128 MiB per array
    cls = torch.from_numpy(rng.integers(0, C, rows).astype(np.uint16)).to(cuda)
    x = torch.randn(rows, n, device=cuda) * 16
    y = plan.forward(x, cls)
    back = plan.inverse(y, cls)
    plan.sync_status()
    err = (torch.linalg.vector_norm(back - x) / torch.linalg.vector_norm(x)).item()
    assert err < 1e-6, err
    idx = rng.choice(rows, 2048, replace=False)
    xs, cs = x.cpu().numpy()[idx], cls.cpu().numpy()[idx]
    ref = oracle_mod.apply_batch(log2n, R, angles, perms, (1 << R) - 1, xs, cs)
    check_close(y.cpu().numpy()[idx], ref, xs, f"clsjit N={n} steady-state sample")


@pytest.mark.parametrize("log2n", [4, 6])
def test_fixed_jit_steady_state(cuda, oracle_mod, log2n):
    """Fixed-point NVRTC chain with several batches per warp: bit-exact on a sample, exact
    first-failing-row report for an oversized input deep in the batch."""
    from paper_2505_21728_b200 import ArgumentError, FixedPlan, QuantizedHyGTModel, TrigTable
    rng = np.random.default_rng(22)
    C, R, n = 4, 3, 1 << log2n
    a = R * n * log2n // 2
    codes = rng.integers(0, 256, (C, a)).astype(np.uint16)
    inter = np.stack([np.stack([rng.permutation(n) for _ in range(R - 1)]) for _ in range(C)]).astype(np.uint16)
    full = np.concatenate([inter, np.tile(np.arange(n, dtype=np.uint16), (C, 1, 1))], 1)
    plan = FixedPlan([QuantizedHyGTModel(log2n, R, 8, codes[c]) for c in range(C)], TrigTable(8, 10), inter)
    rows = (1 << 27) // (8 * n)
    x = torch.from_numpy(rng.integers(-(1 << 20), (1 << 20) + 1, (rows, n)).astype(np.int64)).to(cuda)
    cls = torch.from_numpy(rng.integers(0, C, rows).astype(np.uint16)).to(cuda)
    y = plan.forward(x, cls).cpu().numpy()
    idx = rng.choice(rows, 2048, replace=False)
    st, _, ref = oracle_mod.apply_batch_fixed(log2n, R, 8, 10, codes, full, (1 << (R - 1)) - 1,
                                              x.cpu().numpy()[idx], cls.cpu().numpy()[idx])
    assert st == 0 and np.array_equal(y[idx], ref)
    bad = rows - 12345
    x[bad, 1] = (1 << 20) + 7
    x[bad + 100, 0] = -(1 << 21)
    with pytest.raises(ArgumentError):
        plan.forward(x, cls)
    assert plan.first_bad == bad


@pytest.mark.parametrize("default_ws", [False, True])
@pytest.mark.parametrize("log2n", [4, 6])
def test_one_plan_two_host_threads(cuda, log2n, default_ws):
    """A plan is immutable after creation: two host threads, each with its own stream and
    workspace, run the same plan concurrently (staged kernel at N = 16, the per-class launch
    chain at N = 64) and get exactly the results of a serial run."""
    import threading
    from paper_2505_21728_b200 import HyGTModel
    rng = np.random.default_rng(31)
    C, R, n = 35, 3, 1 << log2n
    angles = rng.uniform(-np.pi, np.pi, (C, R * log2n * n // 2))
    perms = np.stack([np.stack([rng.permutation(n) for _ in range(R - 1)]) for _ in range(C)]).astype(np.uint16)
    plan = _plan([HyGTModel(log2n, R, angles[c]) for c in range(C)], perms)
    rows = 1 << 18
    xs = [torch.randn(rows, n, device=cuda) for _ in range(2)]
    cs = [torch.from_numpy(rng.integers(0, C, rows).astype(np.uint16)).to(cuda) for _ in range(2)]
    ref = [plan.inverse(plan.forward(xs[i], cs[i]), cs[i]) for i in range(2)]
    refy = [plan.forward(xs[i], cs[i]) for i in range(2)]
    torch.cuda.synchronize()
    out = [None, None]
    errs = []

    def work(i):
        try:
            torch.cuda.set_device(cuda)
            st = torch.cuda.Stream()
            # explicit workspaces, or the plan's defaults (one per host thread and stream)
            ws = None if default_ws else torch.zeros(plan.workspace_bytes(rows), dtype=torch.uint8, device=cuda)
            with torch.cuda.stream(st):
                for _ in range(5):
                    y = plan.forward(xs[i], cs[i], stream=st, workspace=ws)
                    z = plan.inverse(y, cs[i], stream=st, workspace=ws, reuse_buckets=True)
                plan.sync_status(ws, stream=st)
            out[i] = (y, z)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        assert torch.equal(out[i][0], refy[i])
        assert torch.equal(out[i][1], ref[i])


def test_many_classes_skip_per_class_jit(cuda, oracle_mod):
    """Plans with more classes than HYGT_CLS_JIT_MAX_CLASSES (64) stay on the precompiled
    kernels (no per-class NVRTC modules) and still match the oracle."""
    from paper_2505_21728_b200 import HyGTModel
    rng = np.random.default_rng(41)
    C, R, n = 70, 2, 64
    angles = rng.uniform(-np.pi, np.pi, (C, R * 6 * 32))
    plan = _plan([HyGTModel(6, R, angles[c]) for c in range(C)])
    assert plan.path in ("cls", "seg2")  # parameter-table chain or thread-per-row kernel
    x = (rng.standard_normal((5000, n)) * 16).astype(np.float32)
    cls = rng.integers(0, C, 5000).astype(np.uint16)
    y = plan.forward(torch.from_numpy(x).to(cuda), torch.from_numpy(cls).to(cuda))
    plan.sync_status()
    check_close(y.cpu().numpy(), oracle_mod.apply_batch(6, R, angles, None, 0, x, cls), x, "70 classes")


@pytest.mark.parametrize("config", [1, 2, 5])
def test_synthetic_rows_follow_ar1_covariance(cuda, config):
    """The device generator's rows have the separable AR(1) covariance sigma^2 (A kron A)
    (statistics.hpp:287-305), checked at 5% as test_statistics.cpp:61-70 checks sample_residuals
    (SURVEY 8 d3); config 2 per class (rho_c), on its most populated class."""
    from paper_2505_21728_b200.synth import make_workload
    from test_oracle import _ar1_2d
    w = make_workload(config)
    rows = {1: 1 << 19, 2: 1 << 21, 5: 1 << 17}[config]
    cls = w.make_classes(rows)
    x = w.make_rows(rows, cls).double()
    c = 0
    if w.cfg.rho is None:  # per-class rho: one class's rows
        c = int(torch.bincount(cls.to(torch.int64)).argmax().item())
        x = x[cls.to(torch.int64) == c]
    emp = (x.T @ x / x.shape[0]).cpu().numpy()
    ref = _ar1_2d(w.block_size(), float(w.rho[c]), w.cfg.sigma)
    assert np.abs(emp - ref).max() <= 0.05 * np.abs(ref).max()


def test_reference_adapter(cuda):
    """include/hygt_gpu_adapter.hpp driven with the reference's own C++ types (HyGTModel,
    ModelBundle, ResidualDataset, QuantizedHyGTModel, TrigTable) against the reference's own
    hygt::forward / forward_fixed, built here from the unmodified headers (oracle/_ref)."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "adapter_check")
    assert os.path.exists(exe), "oracle/_ref/adapter_check was not built (make -C oracle)"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adapter_check: ok" in r.stdout


def test_jit_plan_matches_oracle(cuda, oracle_mod, knob):
    """The NVRTC plan-specialised path (coefficients as immediates, permutations as register
    renames) on config-1 style plans: 1-4 classes, inter-round and final permutations, both
    arithmetic forms, tails, invalid class ids."""
    from paper_2505_21728_b200 import ArgumentError, HyGTModel
    knob("HYGT_STAGE", "0")  # N = 16 plans otherwise take the staged kernel
    rng = np.random.default_rng(21)
    for log2n, rounds, classes in [(2, 2, 1), (3, 3, 2), (4, 2, 1), (4, 3, 4), (5, 2, 3)]:
        n = 1 << log2n
        ang = rng.uniform(-np.pi, np.pi, (classes, rounds * n * log2n // 2))
        inter = np.stack([np.stack([rng.permutation(n) for _ in range(rounds - 1)]) for _ in range(classes)]).astype(np.uint16)
        fin = np.stack([rng.permutation(n) for _ in range(classes)]).astype(np.uint16)
        models = [HyGTModel(log2n, rounds, ang[c], fin[c]) for c in range(classes)]
        full = np.concatenate([inter, fin[:, None, :]], 1)
        rows = 5000 + 17
        x = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
        cls = rng.integers(0, classes, rows).astype(np.uint16)
        for standard in (False, True):
            plan = _plan(models, inter, standard)
            assert plan.path == "jit", plan.path
            xd, cd = torch.from_numpy(x).to(cuda), torch.from_numpy(cls).to(cuda)
            y = plan.forward(xd, cd)
            plan.sync_status()
            ref = oracle_mod.apply_batch(log2n, rounds, ang, full, (1 << rounds) - 1, x, cls)
            check_close(y.cpu().numpy(), ref, x, f"jit fwd N={n} C={classes} std={standard}")
            back = plan.inverse(y, cd)
            check_close(back.cpu().numpy(), x, x, f"jit roundtrip N={n}")
            if classes > 1:
                cd[5] = classes
                plan.forward(xd, cd)
                with pytest.raises(ArgumentError):
                    plan.sync_status()


@pytest.mark.parametrize("standard", [False, True])
def test_stage_path_edges(cuda, oracle_mod, standard, knob):
    """TMA-staged kernel (plan path 'stage'): partial and multi-tile batches, class ids staged by
    TMA and (misaligned) by plain loads, in place, unaligned rows falling back to the tile
    kernel, invalid ids passed through and reported."""
    from paper_2505_21728_b200 import ArgumentError, HyGTModel
    from oracle import oracle as O
    knob("HYGT_JIT", "0")
    rng = np.random.default_rng(21)
    C, R = 7, 3
    angles = rng.uniform(-np.pi, np.pi, (C, R * 4 * 8))
    perms = np.stack([np.stack([rng.permutation(16) for _ in range(R)]) for _ in range(C)]).astype(np.uint16)
    models = [HyGTModel(4, R, angles[c], perms[c, R - 1]) for c in range(C)]
    plan = _plan(models, perms[:, : R - 1].copy(), standard)
    assert plan.path == "stage"
    for count in [0, 1, 7, 8, 33, 811, 2 * 811 + 5, 50000]:
        xh = (rng.standard_normal((count + 1, 16)) * 16).astype(np.float32)
        ch = rng.integers(0, C, count + 1).astype(np.uint16)
        xd = torch.from_numpy(xh).to(cuda)
        cd = torch.from_numpy(ch).to(cuda)
        y = plan.forward(xd[:count], cd[:count])
        plan.sync_status()
        if not count:
            continue
        ref = O.apply_batch(4, R, angles, perms, (1 << R) - 1, xh[:count], ch[:count])
        check_close(y.cpu().numpy(), ref, xh[:count], f"stage fwd count={count}")
        back = plan.inverse(y, cd[:count])
        check_close(back.cpu().numpy(), xh[:count], xh[:count], f"stage roundtrip count={count}")
        # class ids at an odd u16 offset: not 16 B aligned -> loaded by the consumer warps
        y2 = plan.forward(xd[:count], cd[1:])
        ref2 = O.apply_batch(4, R, angles, perms, (1 << R) - 1, xh[:count], ch[1:])
        check_close(y2.cpu().numpy(), ref2, xh[:count], f"stage misaligned ids count={count}")
        # rows at a 16-byte offset stay on the staged path; a 4-byte offset is rejected
        xm = xd.view(-1)[4:4 + count * 16].view(count, 16)
        xm_h = xh.reshape(-1)[4:4 + count * 16].reshape(count, 16)
        refm = O.apply_batch(4, R, angles, perms, (1 << R) - 1, xm_h, ch[:count])
        check_close(plan.forward(xm, cd[:count]).cpu().numpy(), refm, xm_h, f"stage offset count={count}")
        with pytest.raises(ArgumentError):
            plan.forward(xd.view(-1)[1:1 + count * 16].view(count, 16), cd[:count])
        xi = xd[:count].clone()
        plan.forward(xi, cd[:count], out=xi)  # in place
        assert torch.equal(xi, y)
    x = torch.randn(5000, 16, device=cuda)
    cls = torch.from_numpy(rng.integers(0, C, 5000).astype(np.uint16)).to(cuda)
    cls[1234] = C
    y = plan.forward(x, cls)
    with pytest.raises(ArgumentError):
        plan.sync_status()
    assert torch.equal(y[1234], x[1234])


@pytest.mark.parametrize("standard,cls_env,jit_env,path,R,log2n", [
    (False, "1", "1", "clsjit", 4, 6), (False, "1", "1", "clsjit", 5, 6), (False, "1", "0", "cls", 4, 6),
    (False, "1", "0", "cls", 2, 6), (False, "0", "0", "seg2", 4, 6), (True, "1", "1", "seg2", 4, 6),
    (False, "1", "0", "seg2", 5, 6), (False, "1", "1", "clsjit", 3, 5)])
def test_seg2_path_edges(cuda, oracle_mod, standard, cls_env, jit_env, path, R, log2n, knob):
    """Thread-per-row bucketed kernels (plan paths 'cls' and 'seg2', N = 64): partial batches, a
    class with a single row, in place, invalid ids passed through and reported."""
    from paper_2505_21728_b200 import ArgumentError, HyGTModel
    from oracle import oracle as O
    knob("HYGT_CLS", cls_env)
    knob("HYGT_CLS_JIT", jit_env)
    rng = np.random.default_rng(33)
    C, n = 6, 1 << log2n
    angles = rng.uniform(-np.pi, np.pi, (C, R * log2n * n // 2))
    perms = np.stack([np.stack([rng.permutation(n) for _ in range(R)]) for _ in range(C)]).astype(np.uint16)
    models = [HyGTModel(log2n, R, angles[c], perms[c, R - 1]) for c in range(C)]
    plan = _plan(models, perms[:, : R - 1].copy(), standard)
    assert plan.path == path
    for count in [1, 5, 63, 64, 65, 1000, 70001]:
        xh = (rng.standard_normal((count, n)) * 16).astype(np.float32)
        ch = rng.integers(0, C, count).astype(np.uint16)
        if count > 10:
            ch[ch == 5] = 4
            ch[ch == 3] = 2  # an empty class
            ch[7] = 5  # one class with a single row
        ref = O.apply_batch(log2n, R, angles, perms, (1 << R) - 1, xh, ch)
        xd = torch.from_numpy(xh).to(cuda)
        cd = torch.from_numpy(ch).to(cuda)
        y = plan.forward(xd, cd)
        plan.sync_status()
        check_close(y.cpu().numpy(), ref, xh, f"{path} fwd count={count}")
        back = plan.inverse(y, cd)
        check_close(back.cpu().numpy(), xh, xh, f"{path} roundtrip count={count}")
        xi = xd.clone()
        plan.forward(xi, cd, out=xi)  # in place
        assert torch.equal(xi, y)
    x = torch.randn(3000, n, device=cuda)
    cls = torch.from_numpy(rng.integers(0, C, 3000).astype(np.uint16)).to(cuda)
    cls[123] = C
    y = plan.forward(x, cls)
    with pytest.raises(ArgumentError):
        plan.sync_status()
    assert torch.equal(y[123], x[123])


@pytest.mark.parametrize("log2n,classes,count", [(2, 1, 1000), (4, 3, 20000), (6, 5, 30001), (6, 1, 7001), (7, 1, 3000), (8, 2, 3000)])
def test_correlation_vs_oracle(cuda, oracle_mod, log2n, classes, count):
    """Per-class r r^T sums and counts against the oracle restatement of
    CorrelationAccumulator (pinned bit for bit to the reference in test_oracle.py). Products of
    fp32 samples are exact in fp64; only the order of the fp64 additions differs."""
    from paper_2505_21728_b200 import correlation, finalize_correlation
    from oracle import oracle as O
    rng = np.random.default_rng(60 + log2n)
    n = 1 << log2n
    x = (rng.standard_normal((count, n)) * 16).astype(np.float32)
    cls = rng.integers(0, classes, count).astype(np.uint16)
    ref_s, ref_k = O.correlation(log2n, classes, x, cls)
    xd, cd = torch.from_numpy(x).to(cuda), torch.from_numpy(cls).to(cuda)
    s, k = correlation(xd, cd, classes)
    assert np.array_equal(k.cpu().numpy().astype(np.uint64), ref_k)
    s = s.cpu().numpy()
    assert np.abs(s - ref_s).max() <= 1e-12 * np.abs(ref_s).max()
    # two shards accumulate into the same sums == the whole batch (merge_correlation)
    half = count // 2
    s2, k2 = correlation(xd[:half].contiguous(), cd[:half], classes)
    correlation(xd[half:].contiguous(), cd[half:], classes, sums=s2, counts=k2)
    assert np.abs(s2.cpu().numpy() - ref_s).max() <= 1e-12 * np.abs(ref_s).max()
    phi = finalize_correlation(s2, k2).cpu().numpy()
    for c in range(classes):
        ref_phi = O.correlation_finalize(log2n, ref_s[c], ref_k[c])
        assert np.abs(phi[c] - ref_phi).max() <= 1e-12 * np.abs(ref_phi).max()
    # rows that start 4 bytes off a 16-byte boundary are refused (the kernels read 16-byte vectors)
    from paper_2505_21728_b200 import ArgumentError
    flat = torch.empty(count * n + 1, dtype=torch.float32, device=cuda)
    xo = flat[1:].view(count, n)
    xo.copy_(xd)
    with pytest.raises(ArgumentError):
        correlation(xo, cd, classes)


def test_correlation_invalid_ids(cuda):
    from paper_2505_21728_b200 import ArgumentError, correlation
    x = torch.randn(100, 16, device=cuda)
    cls = torch.zeros(100, dtype=torch.int16, device=cuda).view(torch.uint16) if hasattr(torch, "uint16") else None
    c = torch.from_numpy(np.zeros(100, np.uint16)).to(cuda)
    c[5] = 2
    with pytest.raises(ArgumentError):
        correlation(x, c, 2)


@pytest.mark.parametrize("fixed_jit", ["1", "0"])
def test_fixed_staged_edges(cuda, oracle_mod, fixed_jit, knob):
    """Per-class NVRTC chain and staged fixed-point kernel (N = 16): partial and multi-tile
    batches, no class ids, in place, the first failing row for oversized inputs and for invalid
    class ids."""
    from paper_2505_21728_b200 import ArgumentError, FixedPlan, QuantizedHyGTModel, TrigTable
    knob("HYGT_FIXED_JIT", fixed_jit)
    rng = np.random.default_rng(12)
    C, R, n = 6, 3, 16
    codes = rng.integers(0, 256, (C, R * 4 * 8)).astype(np.uint16)
    inter = np.stack([np.stack([rng.permutation(n) for _ in range(R - 1)]) for _ in range(C)]).astype(np.uint16)
    full = np.concatenate([inter, np.tile(np.arange(n, dtype=np.uint16), (C, 1, 1))], 1)
    plan = FixedPlan([QuantizedHyGTModel(4, R, 8, codes[c]) for c in range(C)], TrigTable(8, 10), inter)
    for count in [1, 7, 100, 333, 5000, 70001]:
        x = rng.integers(-(1 << 20), (1 << 20) + 1, (count, n)).astype(np.int64)
        cls = rng.integers(0, C, count).astype(np.uint16)
        xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(cls).cuda()
        st, _, ref = oracle_mod.apply_batch_fixed(4, R, 8, 10, codes, full, (1 << (R - 1)) - 1, x, cls)
        assert st == 0
        y = plan.forward(xd, cd)
        assert np.array_equal(y.cpu().numpy(), ref)
        xi = xd.clone()
        plan.forward(xi, cd, out=xi)  # in place
        assert torch.equal(xi, y)
    one = FixedPlan(QuantizedHyGTModel(4, R, 8, codes[0]), TrigTable(8, 10))
    x = rng.integers(-(1 << 20), (1 << 20) + 1, (4000, n)).astype(np.int64)
    st, _, ref = oracle_mod.apply_batch_fixed(4, R, 8, 10, codes[:1], None, 0, x, None)
    assert np.array_equal(one.forward(torch.from_numpy(x).cuda()).cpu().numpy(), ref)
    x[2345, 3] = (1 << 20) + 1
    x[3000, 0] = -(1 << 21)
    with pytest.raises(ArgumentError):
        one.forward(torch.from_numpy(x).cuda())
    assert one.first_bad == 2345
    x[2345, 3] = 0
    cls = rng.integers(0, C, 4000).astype(np.uint16)
    cls[1500] = C
    with pytest.raises(ArgumentError):
        plan.forward(torch.from_numpy(x).cuda(), torch.from_numpy(cls).cuda())
    assert plan.first_bad == 1500  # invalid class id before the oversized row at 3000


def test_plans_of_different_sizes_coexist(cuda):
    """Kernel shared-memory limits are per function: a smaller plan created later must not break
    an earlier, larger plan of the same kernel family (stage, seg2, fixed)."""
    from paper_2505_21728_b200 import FixedPlan, HyGTModel, QuantizedHyGTModel, TrigTable
    rng = np.random.default_rng(70)
    for log2n in (4, 6):
        n = 1 << log2n
        big = _plan([HyGTModel(log2n, 3, rng.uniform(-3, 3, 3 * log2n * n // 2)) for _ in range(35)],
                    np.stack([np.stack([rng.permutation(n) for _ in range(2)]) for _ in range(35)]).astype(np.uint16))
        small = _plan([HyGTModel(log2n, 1, rng.uniform(-3, 3, log2n * n // 2)) for _ in range(2)])
        x = torch.randn(5000, n, device=cuda)
        ch = rng.integers(0, 35, 5000).astype(np.uint16)
        cls = torch.from_numpy(ch).to(cuda)
        small.forward(x, torch.from_numpy(ch % 2).to(cuda))
        y = big.forward(x, cls)
        check_close(big.inverse(y, cls).cpu().numpy(), x.cpu().numpy(), x.cpu().numpy(), f"N={n} big after small")
    codes = rng.integers(0, 256, (20, 3 * 4 * 8)).astype(np.uint16)
    inter = np.stack([np.stack([rng.permutation(16) for _ in range(2)]) for _ in range(20)]).astype(np.uint16)
    fbig = FixedPlan([QuantizedHyGTModel(4, 3, 8, codes[c]) for c in range(20)], TrigTable(8, 10), inter)
    fsmall = FixedPlan(QuantizedHyGTModel(4, 1, 8, codes[0][:32]), TrigTable(8, 10))
    xi = torch.from_numpy(rng.integers(-1000, 1000, (3000, 16)).astype(np.int64)).to(cuda)
    ci = torch.from_numpy(rng.integers(0, 20, 3000).astype(np.uint16)).to(cuda)
    fsmall.forward(xi)
    fbig.forward(xi, ci)


@pytest.mark.parametrize("config", [2, 3])
def test_fast_form_input_limit(cuda, oracle_mod, config):
    """The scale-folded form's fp32 range (hygt_plan_input_limit = 2^127 sigma_min / sqrt(N)):
    plans take it only when the limit is >= 2^40; rows scaled up to 2^38 still match the oracle,
    and HYGT_PLAN_FORCE_STANDARD lifts the limit to 2^127 / sqrt(N)."""
    from paper_2505_21728_b200.synth import make_workload
    w = make_workload(config)
    plan = _plan(w.models, w.perms)
    assert plan.algorithm == "scale-folded"
    assert plan.input_limit >= 2.0 ** 40
    std = _plan(w.models, w.perms, standard=True)
    assert std.algorithm == "standard" and std.input_limit >= 2.0 ** 120
    cls = w.make_classes(4096)
    x = w.make_rows(4096, cls)
    x = x * (2.0 ** 38 / x.abs().max().item())
    full = np.concatenate([w.perms, np.tile(np.arange(w.n, dtype=np.uint16), (w.cfg.classes, 1, 1))], 1)
    mask = (1 << (w.cfg.rounds - 1)) - 1
    ref = oracle_mod.apply_batch(w.cfg.log2_n, w.cfg.rounds, w.angles, full, mask, x.cpu().numpy(), cls.cpu().numpy())
    y = plan.forward(x, cls)
    plan.sync_status()
    assert torch.isfinite(y).all()
    check_close(y.cpu().numpy(), ref, x.cpu().numpy(), f"cfg{config} at 2^38")


@pytest.mark.parametrize("log2n", [6, 7, 8])
@pytest.mark.parametrize("case", ["ar1_35_classes", "magnitudes"])
def test_correlation_tensor_cores(cuda, oracle_mod, case, knob, log2n):
    """Correlation on the tensor cores (hygt_corr_tc.cu: 7 int8 digits per sample relative to a
    per-column power of two, exact int32 accumulation per digit level, fp64 at run flushes;
    N = 64 by digit stacks, N = 128 / 256 by 64-column block-pair roles) against the oracle's
    exact-product fp64 accumulator, at the fp64 bar of the SIMT path (max-abs <= 1e-12 of the
    class's largest sum): config-3 / config-5 rows (35 classes), and rows whose columns span
    1e-20 .. 1e20 with outlier rows (exponent re-bases), zero columns and a class without rows.
    Also equal, at the same bar, to the SIMT kernel (HYGT_CORR_TC=0)."""
    from paper_2505_21728_b200 import correlation
    from oracle import oracle as O
    rng = np.random.default_rng(64 + log2n)
    n = 1 << log2n
    if case == "ar1_35_classes":
        from paper_2505_21728_b200.synth import make_workload
        w = make_workload(3 if log2n == 6 else 5)
        count, classes = {6: 1 << 20, 7: 1 << 18, 8: 1 << 17}[log2n], 35
        cd = w.make_classes(count)
        xd = w.make_rows(count, cd)
        if log2n == 7:  # config 5's rows, first 128 samples of each
            xd = xd[:, :128].contiguous()
        x, cls = xd.cpu().numpy(), cd.cpu().numpy()
    else:
        count, classes = {6: 50000, 7: 30000, 8: 20000}[log2n], 4
        x = rng.standard_normal((count, n)) * (10.0 ** np.linspace(-20, 20, n))[None, :]
        x[rng.integers(0, count, 40)] *= 1e6  # outliers: the run's scale grows mid-run
        x[:, 5] = 0.0
        x = x.astype(np.float32)
        cls = rng.integers(0, 3, count).astype(np.uint16)  # class 3 has no rows
        xd, cd = torch.from_numpy(x).to(cuda), torch.from_numpy(cls).to(cuda)
    ref_s, ref_k = O.correlation(log2n, classes, x, cls)
    s, k = correlation(xd, cd, classes)
    assert np.array_equal(k.cpu().numpy().astype(np.uint64), ref_k)
    s = s.cpu().numpy()
    for c in range(classes):
        bar = 1e-12 * np.abs(ref_s[c]).max()
        assert np.abs(s[c] - ref_s[c]).max() <= bar, f"class {c}: {np.abs(s[c] - ref_s[c]).max():.3e} vs {bar:.3e}"
        assert np.abs(s[c] - s[c].T).max() <= bar, f"class {c}: not symmetric"
    knob("HYGT_CORR_TC", "0")
    s0, _ = correlation(xd, cd, classes)
    s0 = s0.cpu().numpy()
    for c in range(classes):
        assert np.abs(s0[c] - s[c]).max() <= 2e-12 * max(np.abs(ref_s[c]).max(), 1e-300)

@pytest.mark.parametrize("log2n", [2, 4, 6, 8])
def test_acceptance_criterion4_model_sweep(cuda, oracle_mod, log2n):
    """The reference's acceptance criterion 4 (tests/acceptance.cpp:151-182) on the GPU path: 100
    random models per N in {4, 16, 64, 256}, rounds 1 + trial % 3, a final permutation on odd trials;
    T Tᵀ = I and inverse(forward(x)) = x. The reference holds both to 1e-12 in fp64; here T is read
    off the fp32 kernels (identity rows in, one class per model), so the bars are the fp32 parity
    ones, and T itself is also compared with the oracle's."""
    n = 1 << log2n
    rng = np.random.default_rng(1000 + log2n)
    worst_o = worst_r = 0.0
    for rounds in (1, 2, 3):
        for with_perm in (False, True):
            # trials with this (rounds, permutation) combination: trial % 3 == rounds - 1, trial % 2
            k = len([t for t in range(100) if t % 3 == rounds - 1 and (t % 2 == 1) == with_perm])
            angles = rng.uniform(-np.pi, np.pi, (k, rounds * log2n * (n // 2)))
            perms = mask = None
            if with_perm:
                perms = np.tile(np.arange(n, dtype=np.uint16), (k, rounds, 1))
                for c in range(k):
                    perms[c, rounds - 1] = rng.permutation(n).astype(np.uint16)
                mask = 1 << (rounds - 1)
            plan = _plan(_models(log2n, rounds, angles, perms, mask or 0))
            eye = np.tile(np.eye(n, dtype=np.float32), (k, 1))
            vec = rng.standard_normal((k, n)).astype(np.float32)
            xh = np.concatenate([eye, vec])
            ch = np.concatenate([np.repeat(np.arange(k), n), np.arange(k)]).astype(np.uint16)
            xd, cd = torch.from_numpy(xh).to(cuda), torch.from_numpy(ch).to(cuda)
            y = plan.forward(xd, cd)
            back = plan.inverse(y, cd)
            plan.sync_status()
            yh = y.cpu().numpy().astype(np.float64)
            ref = oracle_mod.apply_batch(log2n, rounds, angles, perms, mask or 0, xh, ch)
            check_close(yh, ref, xh, f"N={n} R={rounds} perm={with_perm} ({plan.algorithm})")
            t = yh[: k * n].reshape(k, n, n)  # row i of block c = T_c e_i, so the block is T_cᵀ
            ortho = np.abs(np.einsum("cij,ckj->cik", t, t) - np.eye(n)).max()
            rt = np.abs(back.cpu().numpy() - xh).max()
            worst_o, worst_r = max(worst_o, ortho), max(worst_r, rt)
            assert ortho < 1e-5, f"N={n} R={rounds} perm={with_perm}: T Tᵀ - I = {ortho:.2e}"
            assert rt < 1e-5 * max(1.0, np.abs(xh).max()), f"N={n} R={rounds} perm={with_perm}: round trip {rt:.2e}"


@pytest.mark.parametrize("n,classes", [(16, 5), (64, 35), (256, 4)])
def test_klt_bucket_once_reuse_both_directions(cuda, oracle_mod, n, classes):
    """hygt_klt_bucket + HYGT_REUSE_BUCKETS: one class grouping serves forward and inverse (the
    bench's config-4 step), bit-identical to the calls that bucket themselves."""
    from paper_2505_21728_b200 import ArgumentError, KLTPlan
    rng = np.random.default_rng(40 + n)
    k = np.stack([np.linalg.qr(rng.standard_normal((n, n)))[0] for _ in range(classes)])
    plan = KLTPlan(k)
    rows = 5000
    xh = (rng.standard_normal((rows, n)) * 16).astype(np.float32)
    ch = rng.integers(0, classes, rows).astype(np.uint16)
    x, cls = torch.from_numpy(xh).to(cuda), torch.from_numpy(ch).to(cuda)
    y0 = plan.forward(x, cls)
    b0 = plan.inverse(y0, cls)
    ws = torch.zeros(max(256, plan.workspace_bytes(rows)), dtype=torch.uint8, device=cuda)
    plan.bucket(cls, rows, ws)
    y1 = plan.forward(x, cls, workspace=ws, reuse_buckets=True)
    b1 = plan.inverse(y1, cls, workspace=ws, reuse_buckets=True)
    assert torch.equal(y0, y1) and torch.equal(b0, b1)
    check_close(y1.cpu().numpy(), oracle_mod.klt_apply(k, xh, ch), xh, f"klt reuse n={n}")
    with pytest.raises(ArgumentError):
        plan.forward(x, cls, reuse_buckets=True)  # no workspace to reuse


def test_reference_fixed_point_kats(cuda, oracle_mod):
    """The reference's own fixed-point cases (tests/test_fixedpoint.cpp:90-184) through the GPU
    drop-ins forward_fixed / inverse_fixed."""
    from paper_2505_21728_b200 import (ArgumentError, HyGTModel, QuantizedHyGTModel, TrigTable,
                                       dequantize_model, forward_fixed, inverse_fixed, quantize_model)
    table = TrigTable(8, 10)
    # :90-96 zero codes pass integers through exactly
    ident = QuantizedHyGTModel(3, 2, 8, np.zeros(24, np.uint16))
    x = np.array([5, -7, 1000, 0, -1, 12, 999, -1024], np.int64)
    assert np.array_equal(forward_fixed(ident, table, x), x)
    assert np.array_equal(inverse_fixed(ident, table, x), x)
    # :98-105 the quarter-turn butterfly is exact in integer arithmetic
    qt = QuantizedHyGTModel(1, 1, 8, np.array([64], np.uint16))
    y = forward_fixed(qt, table, [100, 7])
    assert list(y) == [7, -100] and list(inverse_fixed(qt, table, y)) == [100, 7]
    # :107-158 the fixed transform tracks the float transform of the same codes (N=16 R=2 and the
    # deepest smoke configuration N=64 R=5), and :160-175 the round trip stays bounded. The
    # reference pins its seeds' maxima (4, 7, 4); here the maxima must equal the oracle's on the
    # same inputs (bit-exact outputs) and stay under one rounding step per pass.
    rng = np.random.default_rng(88)
    for log2n, rounds, trials in ((4, 2, 50), (6, 5, 10)):
        n = 1 << log2n
        q = quantize_model(HyGTModel(log2n, rounds, rng.uniform(-np.pi, np.pi, rounds * log2n * n // 2),
                                     rng.permutation(n).astype(np.uint16)), 8)
        dq = dequantize_model(q)
        perms = np.tile(np.arange(n, dtype=np.uint16), (1, rounds, 1))
        perms[0, rounds - 1] = q.permutation
        mask = 1 << (rounds - 1)
        worst_f = worst_rt = 0
        for _ in range(trials):
            xi = rng.integers(-1024, 1025, n).astype(np.int64)
            yi = forward_fixed(q, table, xi)
            st, _, ref = oracle_mod.apply_batch_fixed(log2n, rounds, 8, 10, q.codes[None], perms, mask, xi[None])
            assert st == 0 and np.array_equal(yi, ref[0])
            yf = oracle_mod.apply_batch(log2n, rounds, dq.angles[None], perms, mask, xi[None].astype(np.float32))[0]
            worst_f = max(worst_f, int(np.abs(yi - np.rint(yf).astype(np.int64)).max()))
            back = inverse_fixed(q, table, yi)
            st, _, refb = oracle_mod.apply_batch_fixed(log2n, rounds, 8, 10, q.codes[None], perms, mask, ref, None, inverse=True)
            assert st == 0 and np.array_equal(back, refb[0])
            worst_rt = max(worst_rt, int(np.abs(back - xi).max()))
        assert worst_f <= rounds * log2n and worst_rt <= 2 * rounds * log2n, (worst_f, worst_rt)
    # :177-184 the input range and the width checks
    one = QuantizedHyGTModel(1, 1, 8, np.array([0], np.uint16))
    with pytest.raises(ArgumentError):
        forward_fixed(one, table, [1 << 21, 0])
    with pytest.raises(ArgumentError):
        forward_fixed(one, table, [0])
    with pytest.raises(ArgumentError):
        forward_fixed(one, TrigTable(6, 10), [1, 2])
