"""Shared pytest setup: the ``gpu`` marker and golden-fixture loaders."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def c1_arrays():
    return dict(np.load(GOLDEN / "c1.npz"))


class Cam:
    """Minimal camera record accepted by the oracle and the product Camera."""

    def __init__(self, rotation, translation, fx, fy, cx, cy, width, height):
        self.rotation = np.asarray(rotation, dtype=np.float64)
        self.translation = np.asarray(translation, dtype=np.float64)
        self.fx, self.fy, self.cx, self.cy = float(fx), float(fy), float(cx), float(cy)
        self.width, self.height = int(width), int(height)


def kat_cases():
    meta = json.loads((GOLDEN / "golden.json").read_text())["kat"]
    arrays = dict(np.load(GOLDEN / "kat_splats.npz"))
    return arrays, meta
