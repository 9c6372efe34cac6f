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


def pytest_sessionfinish(session, exitstatus):
    """Under HK_VALIDATE=1 (tests/test_gpu_validate.py runs the GPU suite that
    way) report the task-extent validator's counts and fail the session on any
    region found outside its device allocation."""
    import os
    if os.environ.get("HK_VALIDATE") != "1" or "paper_1403_5337_b200._native" not in sys.modules:
        return
    import ctypes
    from paper_1403_5337_b200 import _native as N
    checked = ctypes.c_int64(0)
    viol = int(N.lib().hk_debug_violations(ctypes.byref(checked)))
    print(f"\n[hk validate] {checked.value} task regions checked, {viol} violations")
    if viol:
        session.exitstatus = 1
