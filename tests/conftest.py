import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device); run with -m gpu")


def load_golden(name: str) -> dict:
    d = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    d["shape_tuple"] = tuple(int(v) for v in d["shape"])
    return d


# dense-block cases (model_*.npz / train_*.npz hold whole-network steps, tests/test_model_gpu.py, test_train_gpu.py)
GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and not f.startswith(("model_", "train_")))


def rel_err(a, b):
    """dp/gradcheck.hpp:14-17: |a-b| / max(1, |a|, |b|), elementwise max."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


def norm_err(a, b):
    """Normwise ||a-b||_2 / ||b||_2 (bf16 tolerance, SURVEY §7 hard part 7)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure liboracle.so and libdpb.so exist (build() is idempotent)."""
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build(ref=False)
    from paper_1707_06990_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()
    yield
