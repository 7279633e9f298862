"""pytest configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs here on CPU (oracle vs golden vectors, the C-ABI surface);
`-m gpu` runs on a B200 through `gpurun` (parity of the CUDA path vs the oracle).
"""
import os
import sys

import pytest

# row-sharded tests run several ranks (streams) of one process on one GPU: give every stream its
# own hardware queue (a rank's spinning wait must never sit in front of a peer's kernel), and
# turn a protocol bug into a quick failure instead of a long wait
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("MPZCH_PEER_TIMEOUT_MS", "20000")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    # A GPU test selected on a CPU-only box must not silently pass.
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for it in items:
        if "gpu" in it.keywords and config.getoption("-m") not in ("gpu",):
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    import pyoracle
    if not pyoracle.available("port"):
        pyoracle.build()
    return pyoracle
