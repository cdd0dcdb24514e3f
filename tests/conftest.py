import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden_v1.npz"))


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run with -m 'not gpu' on CPU)")
    import paper_2505_21728_b200._lib as L
    L.lib()  # fail loudly if the CUDA library is missing
    return torch.device("cuda:0")


@pytest.fixture
def knob():
    """Sets development knobs of the kernel selection through the library's test hook
    (hygt_debug_set_knob; the library reads no environment variables) and clears them after the
    test. Usage: knob("HYGT_SEGMENT", "0")."""
    import paper_2505_21728_b200._lib as L

    def set_(name, value):
        L.set_knob(name, int(value))

    yield set_
    L.clear_knobs()
