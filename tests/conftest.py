import functools
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@functools.lru_cache(maxsize=None)
def golden(name):
    """Load tests/golden/<name>.npz (written by tests/golden/make_golden.py)."""
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        pytest.skip(f"golden fixture {path.name} missing (run tests/golden/make_golden.py)")
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


SMALL_FRONTS = ("3d-9", "2d-100", "3d-12", "3d-vec-7", "3d-15", "3d-16")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def random_low_rank(rng, m, n, r):
    return rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
