"""CPU: the C-ABI library loads and exports every symbol include/hygt_gpu.h declares, host-side
argument validation mirrors the reference's ArgumentError behaviour, and the Python mirror of
the reference types (HyGTModel, QuantizedHyGTModel, TrigTable, ModelBundle, ...) matches the
reference's known answers. No GPU calls."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hygt_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hygt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    import paper_2505_21728_b200._lib as L
    lib = L.lib()  # loading needs no GPU
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"libhygt_gpu.so does not export {s}"
    assert set(syms) == set(L.SIGNATURES), "ctypes signature table out of sync with the header"


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2505_21728_b200", "libhygt_gpu.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plan_create_argument_errors_without_gpu():
    """hygt_plan_create validates like HyGTModel's constructor (model.hpp:53-62) before touching
    the device."""
    import paper_2505_21728_b200._lib as L
    lib = L.lib()
    h = C.c_void_p()
    ang = np.zeros(64)
    p = ang.ctypes.data_as(C.c_void_p)
    assert lib.hygt_plan_create(0, 2, 1, p, None, 0, 0, C.byref(h)) == 1
    assert "log2_n" in L.last_error()
    assert lib.hygt_plan_create(4, 0, 1, p, None, 0, 0, C.byref(h)) == 1
    assert lib.hygt_plan_create(4, 2, 0, p, None, 0, 0, C.byref(h)) == 1
    assert lib.hygt_plan_create(9, 2, 1, p, None, 0, 0, C.byref(h)) == 1  # GPU limit N <= 256
    bad = np.tile(np.array([0, 0] + list(range(2, 16)), np.uint16), (1, 2, 1))
    assert lib.hygt_plan_create(4, 2, 1, p, bad.ctypes.data_as(C.c_void_p), 1, 0, C.byref(h)) == 1
    assert "bijection" in L.last_error()
    nan = np.full(64, np.nan)
    assert lib.hygt_plan_create(4, 2, 1, nan.ctypes.data_as(C.c_void_p), None, 0, 0, C.byref(h)) == 1
    codes = np.full(64, 300, np.uint16)
    assert lib.hygt_fixed_plan_create(4, 2, 1, 8, 10, codes.ctypes.data_as(C.c_void_p), None, 0,
                                      C.byref(h)) == 1
    assert "code exceeds" in L.last_error()
    assert lib.hygt_fixed_plan_create(4, 2, 1, 8, 16, codes.ctypes.data_as(C.c_void_p), None, 0,
                                      C.byref(h)) == 1


def test_model_validation_mirrors_reference():
    from paper_2505_21728_b200 import ArgumentError, HyGTModel, num_parameters
    # test_transform.cpp:204-218
    with pytest.raises(ArgumentError):
        HyGTModel(2, 1, np.zeros(3))
    with pytest.raises(ArgumentError):
        HyGTModel(1, 1, [0.0], [0, 0])
    with pytest.raises(ArgumentError):
        HyGTModel(1, 1, [0.0], [1])
    assert num_parameters(4, 2) == 64 and num_parameters(6, 3) == 576 and num_parameters(1, 1) == 1
    with pytest.raises(ArgumentError):
        num_parameters(0, 1)
    with pytest.raises(ArgumentError):
        num_parameters(1, 0)
    m = HyGTModel(3, 2, np.arange(24.0))
    assert m.angle_index(1, 2, 3) == (1 * 3 + 2) * 4 + 3
    assert m.angle(1, 2, 3) == 23.0


def test_hypercube_indices_match_golden(golden):
    from paper_2505_21728_b200 import ArgumentError, hypercube_indices
    for log2n in range(1, 9):
        for p in range(log2n):
            m, n = hypercube_indices(log2n, p)
            assert np.array_equal(m, golden[f"hc_{log2n}_m"][p])
            assert np.array_equal(n, golden[f"hc_{log2n}_n"][p])
    for args in [(0, 0), (17, 0), (3, 3), (3, -1)]:  # test_hypercube.cpp:68-73
        with pytest.raises(ArgumentError):
            hypercube_indices(*args)


def test_fixed_point_types_match_reference(golden):
    from paper_2505_21728_b200 import (ArgumentError, HyGTModel, QuantizedHyGTModel, TrigTable,
                                       dequantize_model, quantize_model)
    for b, p in [(8, 10), (2, 4), (12, 15), (6, 10)]:
        t = TrigTable(b, p)
        assert np.array_equal(t._cos, golden[f"trig_{b}_{p}_cos"])
        assert np.array_equal(t._sin, golden[f"trig_{b}_{p}_sin"])
    for args in [(0, 10), (13, 10), (8, 3), (8, 16)]:  # test_fixedpoint.cpp:61-67
        with pytest.raises(ArgumentError):
            TrigTable(*args)
    q = quantize_model(HyGTModel(2, 1, [0.0, math.pi / 2, -math.pi / 4, 0.1]), 8)
    assert list(q.codes[:3]) == [0, 64, 224]  # test_fixedpoint.cpp:69-75
    for k in range(7):
        log2n, rounds, b, _, _ = (int(v) for v in golden[f"x{k}_meta"])
        m = HyGTModel(log2n, rounds, golden[f"x{k}_angles"])
        assert np.array_equal(quantize_model(m, b).codes, golden[f"x{k}_codes"])
    back = dequantize_model(QuantizedHyGTModel(2, 1, 8, [0, 64, 128, 192]))
    np.testing.assert_allclose(back.angles, [0, math.pi / 2, math.pi, 3 * math.pi / 2])
    with pytest.raises(ArgumentError):
        QuantizedHyGTModel(1, 1, 8, [256])


def test_memory_footprint_and_bundle(golden):
    from paper_2505_21728_b200 import (ArgumentError, HyGTModel, ModelBundle, TransformKind,
                                       memory_footprint)
    for kl, ln, r, t, v in golden["footprints"]:
        kind = TransformKind.klt if kl else TransformKind.hygt
        assert memory_footprint(kind, int(ln), int(r), int(t)) == v
    # 8x8 blocks, KLT vs H(4) = 5.3
    assert round(memory_footprint(TransformKind.klt, 6, 1, 35) /
                 memory_footprint(TransformKind.hygt, 6, 4, 35), 1) == 5.3
    with pytest.raises(ArgumentError):
        ModelBundle([])
    with pytest.raises(ArgumentError):
        ModelBundle([HyGTModel.zeros(2, 1), HyGTModel.zeros(3, 1)])
    b = ModelBundle([HyGTModel.zeros(4, 2) for _ in range(3)])
    assert b.class_count() == 3 and b.dimension() == 16 and not b.quantized()


def test_synthetic_workloads_are_deterministic():
    from paper_2505_21728_b200.synth import CONFIGS, make_workload
    for k in CONFIGS:
        a, b = make_workload(k), make_workload(k)
        assert np.array_equal(a.angles, b.angles)
        assert (a.perms is None) == (b.perms is None)
        if a.perms is not None:
            assert np.array_equal(a.perms, b.perms)
            for c in range(a.perms.shape[0]):
                for r in range(a.perms.shape[1]):
                    assert sorted(a.perms[c, r]) == list(range(a.n))
    w = make_workload(2)
    assert w.angles.shape == (35, 3 * 16 * 4 // 2) and np.all(np.abs(w.angles) <= math.pi)
    assert np.all((w.rho >= 0.5) & (w.rho <= 0.95))
    q = make_workload(4).klt_bases()
    assert np.abs(q[0] @ q[0].T - np.eye(64)).max() < 1e-12


def test_trainer_host_logic_mirrors_reference(oracle_mod):
    """derive_seed (rng.hpp:36-38) and variance_permutation's stable descending order
    (optimizer.hpp:378-390; test_optimizer.cpp:209-224) -- host-side, no GPU needed."""
    from paper_2505_21728_b200 import train
    from paper_2505_21728_b200.model import HyGTModel
    for base, stream in [(0, 0), (1, 5), (2**63 + 7, 34)]:
        assert train.derive_seed(base, stream) == oracle_mod.derive_seed(base, stream)
    m = train.variance_permutation(HyGTModel.zeros(2, 1), [1.0, 5.0, 3.0, 3.0])
    assert list(m.permutation) == [1, 2, 3, 0]
    m = train.variance_permutation(HyGTModel.zeros(2, 1), [4.0, 3.0, 2.0, 1.0])
    assert list(m.permutation) == [0, 1, 2, 3]
    import pytest
    from paper_2505_21728_b200.errors import ArgumentError
    with pytest.raises(ArgumentError):
        train.variance_permutation(m, [1.0, 2.0, 3.0, 4.0])


@pytest.mark.parametrize("kind,log2n,rounds,ptx", [(0, 6, 4, 0), (0, 6, 4, 1), (0, 5, 3, 0), (1, 4, 3, 0), (1, 6, 2, 0)])
def test_per_class_kernels_compile_without_gpu(kind, log2n, rounds, ptx):
    """The per-class NVRTC generators (float N = 32/64, fixed point) emit source that compiles
    for sm_100a; NVRTC needs no GPU, so this runs in the CPU suite (hygt_debug_jit_compile)."""
    import ctypes as C
    from paper_2505_21728_b200 import _lib
    lib = _lib.lib()
    fn = lib.hygt_debug_jit_compile
    fn.restype = C.c_int
    n = 1 << log2n
    rng = np.random.default_rng(4)
    angles = np.ascontiguousarray(rng.uniform(-np.pi, np.pi, rounds * log2n * n // 2))
    codes = np.ascontiguousarray(rng.integers(0, 256, rounds * log2n * n // 2).astype(np.uint16))
    perms = np.ascontiguousarray(np.stack([rng.permutation(n) for _ in range(rounds)]).astype(np.uint16))
    mask = (1 << (rounds - 1)) - 1 if log2n < 8 else 0
    out = C.c_ulonglong(0)
    st = fn(kind, log2n, rounds, angles.ctypes.data_as(C.c_void_p), codes.ctypes.data_as(C.c_void_p),
            perms.ctypes.data_as(C.c_void_p) if mask else None, C.c_uint32(mask), ptx, C.byref(out))
    assert st == 0 and out.value > 10000


def test_library_reads_no_environment():
    """The reference contract has no environment variables: kernel choices come
    from hygt_plan_options, development knobs only from the test hook (hygt_knobs.h)."""
    import glob
    import os
    import re
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2505_21728_b200", "csrc")
    offenders = []
    for p in glob.glob(os.path.join(root, "*")):
        if p.endswith((".cu", ".cuh", ".cpp", ".h")):
            for i, line in enumerate(open(p, encoding="utf-8", errors="replace"), 1):
                code = line.split("//", 1)[0]
                if re.search(r"\bgetenv\s*\(", code):
                    offenders.append(f"{os.path.basename(p)}:{i}")
    assert not offenders, offenders
