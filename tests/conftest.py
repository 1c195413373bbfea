"""Shared fixtures.  GPU tests are marked `gpu`; everything else runs on CPU."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

S1_SEED = 20240811      # mirrors the reference's rng fixture (conftest.py:56-58)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libhsv.so")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def s1_values(dim: int) -> np.ndarray:
    """S1 dense-in-sector state, built exactly as the reference tests do
    (normalize(SparseVector.from_dense(rng.standard_normal(dim))))."""
    v = np.random.default_rng(S1_SEED).standard_normal(dim)
    return v / float(np.linalg.norm(v))


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128 if np.iscomplexobj(a) else np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(1.0, float(np.max(np.abs(b), initial=0.0)))
    return float(np.max(np.abs(a - b), initial=0.0)) / scale


@pytest.fixture()
def rng():
    return np.random.default_rng(S1_SEED)
