import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "rowfuse_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def rel_close(actual, ref, rtol, atol_frac=None):
    """|a - b| <= rtol * (|b| + max|b|) by default (SURVEY §8(c) tolerance form)."""
    a = np.asarray(actual, dtype=np.float64)
    b = np.asarray(ref, dtype=np.float64)
    scale = np.abs(b).max() if b.size else 0.0
    atol = (atol_frac if atol_frac is not None else rtol) * scale
    err = np.abs(a - b)
    ok = err <= atol + rtol * np.abs(b)
    return bool(ok.all()), float(err.max() / (scale if scale else 1.0)) if b.size else 0.0


@pytest.fixture
def path_knob():
    """Select a test-only alternative kernel path for the rest of the test (lk_test_select_path);
    restored to the product path afterwards."""
    from paper_2410_10989_b200 import _capi

    ctxs = []

    def select(knob, value):
        c = _capi.select_path(knob, value)
        c.__enter__()
        ctxs.append(c)

    yield select
    for c in reversed(ctxs):
        c.__exit__(None, None, None)
