import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libchfsi.so")
    config.addinivalue_line("markers", "slow: long-running parity case")
    config.addinivalue_line("markers", "host_payloads: run under the default ('auto') array "
                            "payload policy instead of the device-resident one")


@pytest.fixture(autouse=True)
def _device_payloads(request):
    """GPU tests exercise the device-resident API: n-sized results stay CUDA
    tensors even for numpy inputs (payload policy "torch"). Tests marked
    ``host_payloads`` check the drop-in default instead (numpy in, numpy out)."""
    if request.node.get_closest_marker("gpu") is None or \
            request.node.get_closest_marker("host_payloads") is not None:
        yield
        return
    from paper_1206_3768_b200 import _device

    prev = _device._output_default
    _device.set_array_output("torch")
    try:
        yield
    finally:
        _device.set_array_output(prev)


@pytest.fixture(scope="session")
def small_golden():
    return np.load(os.path.join(GOLDEN, "small_cases.npz"))


@pytest.fixture(scope="session")
def c1_golden():
    return np.load(os.path.join(GOLDEN, "c1_harness.npz"))


@pytest.fixture(scope="session")
def c2_golden():
    return np.load(os.path.join(GOLDEN, "c2_harness.npz"))


def subspace_sines(u, v):
    """Sines of the principal angles between span(u) and span(v)
    (restates the reference test helper `pkg/tests/test_chfsi.py:31-33`)."""
    return np.linalg.svd(v - u @ (u.conj().T @ v), compute_uv=False)
