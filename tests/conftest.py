"""Shared test plumbing: the ``gpu`` marker, repo paths and golden-vector loaders."""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REGIMES = ("batching", "multi-tenant", "combination")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@lru_cache(maxsize=None)
def golden(name: str) -> dict:
    return json.loads((GOLDEN / name).read_text())


def grid_arrays(doc: dict):
    from oracle.oracle import GridArrays

    return GridArrays.from_rows(doc["entries"], doc.get("gpu_idle_power_w"))


def sel_tuple(grid_doc: dict, idx: int, count: int):
    """Oracle (entry index, count) -> the golden [mtl, bs, thr, pw, count] / None form."""
    if idx < 0:
        return None
    m, b, t, p = grid_doc["entries"][idx]
    return [m, b, t, p, count]


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test needs a CUDA device (run -m 'not gpu' on CPU hosts)")
    return True
