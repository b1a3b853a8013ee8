"""Test configuration.  `-m "not gpu"` runs here (CPU only); `-m gpu` runs on a B200."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context (see the package docstring)

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product kernels")


def _cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def has_cuda():
    return _cuda()


def pytest_runtest_setup(item):
    if "gpu" in item.keywords and not _cuda():
        pytest.skip("needs a CUDA device")


@pytest.fixture(scope="session")
def oracle_c():
    import oracle

    return oracle.c_backend()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent when it was built)")
    return oracle.ref_backend()


def backend_by_name(name):
    """'device' -> None (the product default); 'oracle' / 'ref' -> CPU checkers."""
    import oracle

    if name == "device":
        return None
    if name == "oracle":
        return oracle.c_backend()
    if name == "ref":
        if not oracle.ref_available():
            pytest.skip("oracle/_ref not built")
        return oracle.ref_backend()
    raise ValueError(name)


# every API-level test body runs against the reference itself, the C restatement and the device
BACKENDS = [
    pytest.param("ref", id="ref"),
    pytest.param("oracle", id="oracle"),
    pytest.param("device", id="device", marks=pytest.mark.gpu),
]
