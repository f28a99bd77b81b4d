"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun); the rest
run on CPU.  The oracle (``oracle/``) is imported only here and in tests."""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
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


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def golden_json(name: str):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel_err(y, ref) -> float:
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = float(np.linalg.norm(ref))
    return float(np.linalg.norm(y)) if d == 0 else float(np.linalg.norm(y - ref)) / d


def seeded_case(seed, n, m):
    """test_kernel.py:22-26: x [m], logical W [n, m] from default_rng(seed)."""
    g = np.random.default_rng(seed)
    x = g.standard_normal(m, dtype=np.float32)
    arr = g.standard_normal((n, m), dtype=np.float32)
    return x, arr


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    return torch.device("cuda:0")
