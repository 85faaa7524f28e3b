import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and the built libspa2.so")


@pytest.fixture(autouse=True)
def _parity_test_id(request):
    import parity

    parity.CURRENT_TEST["id"] = request.node.nodeid
    yield


def pytest_sessionfinish(session, exitstatus):
    """Write every parity comparison's measured error (GPU runs) for the tolerance record."""
    import parity

    if not parity.RECORD:
        return
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "parity_measured.json"), "w") as f:
        json.dump({"tolerances": {"cos_min/max_rel": parity.TOL, "lse_rel": parity.LSE_REL},
                   "cases": parity.RECORD}, f, indent=0)


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_masks():
    return np.load(os.path.join(GOLDEN, "masks.npz"))


@pytest.fixture(scope="session")
def golden_pooled():
    return np.load(os.path.join(GOLDEN, "pooled.npz"))


@pytest.fixture(scope="session")
def golden_attention():
    return np.load(os.path.join(GOLDEN, "attention.npz"))


def unpack_keep(bits, t_n):
    return np.unpackbits(bits, axis=-1, count=t_n).astype(bool)
