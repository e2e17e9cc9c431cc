import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


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


def rel_err(a, b, floor=1e-300):
    """Reference parity metric (pkg/tests/conftest.py:8-13)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    denom = np.abs(a).max(initial=0.0) + np.abs(b).max(initial=0.0) + floor
    return np.abs(a - b).max(initial=0.0) / denom


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = eval(str(z["meta"]))  # written by make_golden.py with repr(dict)
    w = {k[2:]: z[k].astype(np.float64) for k in z.files if k.startswith("w:")}
    grads = {k[5:]: z[k].astype(np.float64) for k in z.files if k.startswith("grad:")}
    return meta, z, w, grads
