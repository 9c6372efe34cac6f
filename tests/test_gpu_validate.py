"""The GPU parity suite re-run under the task-extent validator (HK_VALIDATE=1,
csrc/validate.cpp): every task array staged for a kernel -- ACA, skeleton,
Gauss-Jordan, GEMM, copy, solve-sweep and selection tasks -- is checked on the
host against the device allocation each of its matrix regions falls in, with
PyTorch's caching allocator off so every tensor is its own allocation.  This
stands in for compute-sanitizer memcheck, which the GPU pool does not run.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parent.parent
SUBSET = ("not config4_large_front and not test_subtree_sharded and not cfg2_reduced "
          "and not knn_front_direct")


def test_parity_suite_under_task_extent_validation():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, HK_VALIDATE="1", PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           "-k", SUBSET, "tests/test_gpu_parity.py", "tests/test_gpu_api.py",
           "tests/test_knn_front.py", "tests/test_gpu_configs.py"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("[hk validate]")]
    assert line and line[-1].endswith(" 0 violations"), tail
    assert int(line[-1].split()[2]) > 1000, line[-1]      # the validator saw the task arrays
