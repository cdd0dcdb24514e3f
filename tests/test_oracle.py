"""CPU: pin the oracle (oracle/hygt_oracle.c) against the reference's golden vectors and the
reference's own known-answer tests. No GPU."""
import math
import os

import numpy as np
import pytest


def test_rng_streams_match_reference(golden, oracle_mod):
    O = oracle_mod
    for seed in [0, 1, 42, 2505]:
        r = O.Rng(seed)
        u = np.array([r.uniform01() for _ in range(257)])
        assert np.array_equal(u, golden[f"rng_u01_{seed}"])
        r = O.Rng(seed)
        gs = np.array([r.gaussian() for _ in range(257)])
        assert np.array_equal(gs, golden[f"rng_gauss_{seed}"])
        r = O.Rng(seed)
        b = np.array([r.below(35) for _ in range(257)], np.uint64)
        assert np.array_equal(b, golden[f"rng_below35_{seed}"])
        d = np.array([O.derive_seed(seed, i) for i in range(64)], np.uint64)
        assert np.array_equal(d, golden[f"derive_seed_{seed}"])


def test_hypercube_schedule_matches_reference(golden, oracle_mod):
    import ctypes as C
    L = oracle_mod.lib()
    for log2n in range(1, 9):
        n = 1 << log2n
        for p in range(log2n):
            m = np.empty(n // 2, np.uint32)
            nn = np.empty(n // 2, np.uint32)
            assert L.hygt_oracle_hypercube_indices(log2n, p, m.ctypes.data_as(C.c_void_p),
                                                   nn.ctypes.data_as(C.c_void_p)) == 0
            assert np.array_equal(m, golden[f"hc_{log2n}_m"][p])
            assert np.array_equal(nn, golden[f"hc_{log2n}_n"][p])
            assert np.all((m ^ nn) == (1 << p))  # test_hypercube.cpp:34-44


@pytest.mark.parametrize("k", range(10))
def test_float_golden_bit_exact(golden, oracle_mod, k):
    O = oracle_mod
    log2n, rounds, classes, mask = (int(v) for v in golden[f"f{k}_meta"])
    args = (log2n, rounds, golden[f"f{k}_angles"], golden[f"f{k}_perms"], mask, golden[f"f{k}_x"],
            golden[f"f{k}_cls"])
    assert np.array_equal(O.apply_batch(*args, inverse=False), golden[f"f{k}_fwd"])
    assert np.array_equal(O.apply_batch(*args, inverse=True), golden[f"f{k}_inv"])


@pytest.mark.parametrize("k", range(7))
def test_fixed_golden_bit_exact(golden, oracle_mod, k):
    O = oracle_mod
    log2n, rounds, b, p, with_perm = (int(v) for v in golden[f"x{k}_meta"])
    n = 1 << log2n
    codes = golden[f"x{k}_codes"]
    assert np.array_equal(O.quantize(golden[f"x{k}_angles"], b), codes)
    perms = None
    mask = 0
    if with_perm:
        perms = np.tile(np.arange(n, dtype=np.uint16), (1, rounds, 1))
        perms[0, rounds - 1] = golden[f"x{k}_perm"]
        mask = 1 << (rounds - 1)
    x = golden[f"x{k}_x"]
    for r in range(x.shape[0]):
        st, _, y = O.apply_batch_fixed(log2n, rounds, b, p, codes[None], perms, mask, x[r:r + 1])
        assert st == golden[f"x{k}_fwd_status"][r]
        if st == 0:
            assert np.array_equal(y[0], golden[f"x{k}_fwd"][r])
        src = golden[f"x{k}_fwd"][r] if st == 0 else x[r]
        st2, _, z = O.apply_batch_fixed(log2n, rounds, b, p, codes[None], perms, mask, src[None],
                                        inverse=True)
        assert st2 == golden[f"x{k}_inv_status"][r]
        if st2 == 0:
            assert np.array_equal(z[0], golden[f"x{k}_inv"][r])


def test_trig_tables_match_reference(golden, oracle_mod):
    for b, p in [(8, 10), (2, 4), (12, 15), (6, 10)]:
        c, s = oracle_mod.trig_table(b, p)
        assert np.array_equal(c, golden[f"trig_{b}_{p}_cos"])
        assert np.array_equal(s, golden[f"trig_{b}_{p}_sin"])
    c, s = oracle_mod.trig_table(8, 10)  # test_fixedpoint.cpp:27-36
    assert (c[0], s[0], c[64], s[64], c[32], c[128]) == (1024, 0, 0, 1024, 724, -1024)


def test_klt_and_energy_match_reference(golden, oracle_mod):
    O = oracle_mod
    y = O.klt_apply(golden["klt_k"], golden["klt_x"], golden["klt_cls"])
    assert np.array_equal(y, golden["klt_fwd"])
    y = O.klt_apply(golden["klt_k"], golden["klt_x"], golden["klt_cls"], inverse=True)
    assert np.array_equal(y, golden["klt_inv"])
    log2n, rounds, classes = (int(v) for v in golden["en_meta"])
    e = O.class_energy(log2n, rounds, golden["en_angles"], None, 0, golden["en_x"], golden["en_cls"])
    # The reference sums the full upper triangle then scales by count / count (statistics.hpp:74,
    # :88); the oracle sums the diagonal directly -- equal up to fp64 rounding.
    np.testing.assert_allclose(e, golden["en_energy"], rtol=1e-12)


def test_memory_footprint(golden, oracle_mod):
    for kl, ln, r, t, v in golden["footprints"]:
        assert oracle_mod.memory_footprint(kl, ln, r, t) == v
    # PAPER.md:302-305 / test_fixedpoint.cpp:186-205
    assert oracle_mod.memory_footprint(1, 6, 1, 35) / oracle_mod.memory_footprint(0, 6, 4, 35) == pytest.approx(5.333, abs=1e-3)


def test_reference_kats(oracle_mod):
    """test_transform.cpp KATs re-run through the oracle."""
    O = oracle_mod
    # quarter-turn butterfly (1,0) -> (0,-1)  (test_transform.cpp:39-45)
    y = O.apply_batch(1, 1, np.array([[math.pi / 2]]), None, 0, np.array([[1, 0]], np.float32))
    assert abs(y[0, 0]) < 1e-15 and abs(y[0, 1] + 1) < 1e-15
    # (3,4) onto the axis (:46-49)
    y = O.apply_batch(1, 1, np.array([[math.atan2(4, 3)]]), None, 0, np.array([[3, 4]], np.float32))
    assert abs(y[0, 0] - 5) < 1e-14 and abs(y[0, 1]) < 1e-14
    # quarter-turn pass [1,2,3,4] -> [2,-1,4,-3]  (:64-72): one round of log2n=2, pass 1 zero
    y = O.apply_batch(2, 1, np.array([[math.pi / 2, math.pi / 2, 0, 0]]), None, 0,
                      np.array([[1, 2, 3, 4]], np.float32))
    np.testing.assert_allclose(y[0], [2, -1, 4, -3], atol=1e-15)
    # zero model = identity, exactly (:118-124)
    x = np.random.default_rng(13).standard_normal((5, 16)).astype(np.float32)
    assert np.array_equal(O.apply_batch(4, 2, np.zeros((1, 64)), None, 0, x), x.astype(np.float64))
    # permutation gathers by index {3,4} -> {4,3} (:196-202)
    y = O.apply_batch(1, 1, np.zeros((1, 1)), np.array([[[1, 0]]], np.uint16), 1,
                      np.array([[3, 4]], np.float32))
    assert list(y[0]) == [4.0, 3.0]


def test_chain_with_identity_perms_equals_single_model(oracle_mod):
    """SURVEY.md c2 self-test: identity inter-round permutations == the R-round model."""
    O = oracle_mod
    rng = np.random.default_rng(3)
    for log2n, rounds in [(4, 3), (6, 4), (8, 2)]:
        n = 1 << log2n
        ang = rng.uniform(-np.pi, np.pi, (1, rounds * n * log2n // 2))
        ident = np.tile(np.arange(n, dtype=np.uint16), (1, rounds, 1))
        x = rng.standard_normal((20, n)).astype(np.float32)
        a = O.apply_batch(log2n, rounds, ang, ident, (1 << rounds) - 1, x)
        b = O.apply_batch(log2n, rounds, ang, None, 0, x)
        assert np.array_equal(a, b)


def test_oracle_orthogonality(oracle_mod):
    """acceptance.cpp:151-182 (criterion 4) on a sample: T T^T = I, roundtrip < 1e-12."""
    O = oracle_mod
    rng = np.random.default_rng(1000)
    for log2n in (2, 4, 6):
        n = 1 << log2n
        for rounds in (1, 2, 3):
            ang = rng.uniform(0, 2 * np.pi, rounds * n * log2n // 2)
            t = O.to_matrix(log2n, rounds, ang)
            assert np.abs(t @ t.T - np.eye(n)).max() < 1e-12


def test_ref_shim_matches_oracle_randomised(oracle_mod):
    O = oracle_mod
    if not O.ref_available():
        pytest.skip("reference shim not built here")
    rng = np.random.default_rng(7)
    for log2n, rounds, classes, mask in [(4, 3, 35, 7), (6, 4, 35, 15), (8, 4, 35, 0)]:
        n = 1 << log2n
        ang = rng.uniform(-np.pi, np.pi, (classes, rounds * n * log2n // 2))
        perms = np.stack([np.stack([rng.permutation(n) for _ in range(rounds)]) for _ in range(classes)]).astype(np.uint16)
        x = (rng.standard_normal((500, n)) * 16).astype(np.float32)
        cls = rng.integers(0, classes, 500).astype(np.uint16)
        for inv in (False, True):
            a = O.apply_batch(log2n, rounds, ang, perms, mask, x, cls, inverse=inv)
            b = O.ref_apply_batch(log2n, rounds, ang, perms, mask, x, cls, inverse=inv)
            assert np.array_equal(a, b)


def test_correlation_oracle_matches_reference_accumulator(oracle_mod):
    """hygt_oracle_correlation restates CorrelationAccumulator (statistics.hpp:63-99); pinned
    bit for bit against the unmodified reference (oracle/_ref/libhygt_ref.so, ref_correlation)."""
    import ctypes
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "libhygt_ref.so")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref/libhygt_ref.so not built")
    ref = ctypes.CDLL(path)
    p = ctypes.c_void_p
    ref.ref_correlation.argtypes = [ctypes.c_int, ctypes.c_int, p, p, ctypes.c_uint64, p, p]
    rng = np.random.default_rng(7)
    for log2n, classes, count in [(2, 1, 50), (4, 3, 500), (6, 5, 300)]:
        n = 1 << log2n
        x = (rng.standard_normal((count, n)) * 16).astype(np.float32)
        cls = rng.integers(0, classes, count).astype(np.uint16)
        sums, counts = oracle_mod.correlation(log2n, classes, x, cls)
        phi_ref = np.zeros((classes, n, n))
        cnt_ref = np.zeros(classes, np.uint64)
        assert ref.ref_correlation(log2n, classes, x.ctypes.data, cls.ctypes.data, count,
                                   phi_ref.ctypes.data, cnt_ref.ctypes.data) == 0
        assert np.array_equal(counts, cnt_ref)
        for c in range(classes):
            phi = oracle_mod.correlation_finalize(log2n, sums[c], counts[c])
            assert np.array_equal(phi, phi_ref[c])  # same loop order: bit-exact


# ---- optimizer -----------------------------------------------------------------

def _opt_golden():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "optimize_v1.npz"))


_OPT_FAST = ["n16r2_seed7", "n4r2_seed99", "n8r2_psd", "n4r1_random_init", "n4r2_zero_init",
             "n8r1_diagonal", "n2r1_psd0", "n2r1_psd3"]


@pytest.mark.parametrize("name", _OPT_FAST)
def test_optimizer_oracle_bit_exact_against_golden(oracle_mod, name):
    """hygt_oracle_optimize restates optimizer.hpp:177-371 line by line: same search path, same
    libm calls, so it reproduces the reference's hygt::optimize outputs bit for bit."""
    g = _opt_golden()
    log2n, rounds, restarts, sweeps = (int(v) for v in g[f"{name}/shape"])
    ang, rep = oracle_mod.optimize(g[f"{name}/phi"], log2n, rounds, restarts=restarts, max_sweeps=sweeps,
                                   seed=int(g[f"{name}/seed"][0]), init_mode=str(g[f"{name}/init_mode"]))
    assert np.array_equal(ang, g[f"{name}/angles"])
    assert np.array_equal(rep["restart_gains_db"], g[f"{name}/gains"])
    assert rep["best_restart"] == int(g[f"{name}/best"][0])
    assert rep["klt_gain_db"] == g[f"{name}/klt"][0]
    assert [len(t) for t in rep["trajectories"]] == g[f"{name}/traj_len"].tolist()
    var = oracle_mod.propagated_variances(g[f"{name}/phi"], log2n, rounds, ang)
    assert np.array_equal(var, g[f"{name}/variances"])


def test_optimizer_oracle_acceptance_pin(oracle_mod):
    """acceptance.cpp:66-68: N=16 R=2, 2-D AR(1) rho=0.95, restarts 4, seed 1 -> 15.164931 dB."""
    g = _opt_golden()
    ang, rep = oracle_mod.optimize(g["n16r2_acceptance/phi"], 4, 2, restarts=4, seed=1)
    assert abs(rep["restart_gains_db"][rep["best_restart"]] - 15.164931) < 1e-3
    assert np.array_equal(ang, g["n16r2_acceptance/angles"])


def test_optimizer_oracle_matches_reference_live(oracle_mod):
    """Fresh random covariances through both the oracle and the reference shim."""
    if not oracle_mod.ref_available():
        pytest.skip("reference shim not built here")
    rng = np.random.default_rng(11)
    for log2n, rounds, restarts in [(2, 2, 2), (3, 1, 3), (4, 1, 2)]:
        n = 1 << log2n
        a = rng.standard_normal((n, n))
        phi = a @ a.T + 0.01 * np.eye(n)
        seed = int(rng.integers(1 << 30))
        x1, r1 = oracle_mod.optimize(phi, log2n, rounds, restarts=restarts, seed=seed)
        x2, r2 = oracle_mod.ref_optimize(phi, log2n, rounds, restarts=restarts, seed=seed)
        assert np.array_equal(x1, x2)
        assert np.array_equal(r1["restart_gains_db"], r2["restart_gains_db"])
        for t1, t2 in zip(r1["trajectories"], r2["trajectories"]):
            assert t1 == t2


def test_optimizer_oracle_errors(oracle_mod):
    """optimizer.hpp:313-326: bad config and indefinite covariances are ArgumentErrors."""
    with pytest.raises(ValueError):
        oracle_mod.optimize(np.diag([1.0, -1.0]), 1, 1)
    with pytest.raises(ValueError):
        oracle_mod.optimize(np.eye(4), 2, 1, restarts=0)


def _ar1_2d(bs, rho, sigma=1.0):
    """sigma^2 (A kron A), A_ij = rho^|i-j|, raster order: statistics.hpp:287-305 restated."""
    i = np.arange(bs)
    a = rho ** np.abs(i[:, None] - i[None, :])
    return sigma * sigma * np.kron(a, a)


@pytest.mark.parametrize("bs,rho", [(4, 0.9), (8, 0.6), (2, 0.95)])
def test_ar1_covariance_formula_matches_reference(bs, rho):
    """The separable AR(1) covariance the synthetic rows follow is the reference's
    ar1_covariance_2d, checked through the unmodified reference where it is built."""
    from oracle import oracle as O
    try:
        lib = O.ref()
    except Exception:
        pytest.skip("oracle/_ref not built")
    out = np.zeros((bs * bs, bs * bs))
    lib.ref_ar1_covariance_2d(bs, rho, out.ctypes.data)
    np.testing.assert_allclose(_ar1_2d(bs, rho), out, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("name", ["grow16", "long64", "grow256", "mixed32"])
def test_fixed_long_golden_bit_exact(oracle_mod, name):
    """The oracle against the reference on long low-precision models (golden_fixed_long.npz):
    values past 2^31 stay exact and rows at 2^20 throw OverflowError (status 4), row by row."""
    O = oracle_mod
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_fixed_long.npz"))
    log2n, rounds, b, p, with_perm = (int(v) for v in g[name + "_meta"])
    n = 1 << log2n
    codes = g[name + "_codes"]
    perms, mask = None, 0
    if with_perm:
        perms = np.tile(np.arange(n, dtype=np.uint16), (1, rounds, 1))
        perms[0, rounds - 1] = g[name + "_perm"]
        mask = 1 << (rounds - 1)
    x = g[name + "_x"]
    for inv, key in ((False, "fwd"), (True, "inv")):
        st_all = g[f"{name}_{key}_status"]
        st, bad, y = O.apply_batch_fixed(log2n, rounds, b, p, codes[None], perms, mask, x, inverse=inv)
        first = int(np.argmax(st_all != 0)) if (st_all != 0).any() else x.shape[0]
        assert st == (int(st_all[first]) if first < x.shape[0] else 0)
        assert bad == first
        ok = np.nonzero(st_all == 0)[0]
        st2, _, y2 = O.apply_batch_fixed(log2n, rounds, b, p, codes[None], perms, mask, x[ok], inverse=inv)
        assert st2 == 0 and np.array_equal(y2, g[f"{name}_{key}"][ok])


@pytest.mark.parametrize("log2n,rounds,classes,mask", [(4, 3, 35, 3), (6, 4, 5, 7), (8, 4, 3, 0), (8, 2, 2, 3)])
def test_hoisted_trig_is_bit_identical(oracle_mod, log2n, rounds, classes, mask):
    """The full-size checks use the oracle with cos/sin tabled once per class (hoist=True); pin
    that mode bit for bit against the per-butterfly restatement of transform.hpp:57-59."""
    O = oracle_mod
    rng = np.random.default_rng(log2n * 10 + rounds)
    n = 1 << log2n
    a = rounds * n * log2n // 2
    angles = rng.uniform(-np.pi, np.pi, (classes, a))
    perms = np.stack([np.stack([rng.permutation(n) for _ in range(rounds)]) for _ in range(classes)]).astype(np.uint16)
    x = (rng.standard_normal((257, n)) * 16).astype(np.float32)
    cls = rng.integers(0, classes, 257).astype(np.uint16)
    for inv in (False, True):
        a0 = O.apply_batch(log2n, rounds, angles, perms, mask, x, cls, inverse=inv, threads=3)
        a1 = O.apply_batch(log2n, rounds, angles, perms, mask, x, cls, inverse=inv, threads=2, hoist=True)
        assert np.array_equal(a0, a1)
    e0 = O.class_energy(log2n, rounds, angles, perms, mask, x, cls, threads=1)
    e1 = O.class_energy(log2n, rounds, angles, perms, mask, x, cls, threads=1, hoist=True)
    assert np.array_equal(e0, e1)
