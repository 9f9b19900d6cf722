"""The GPU parity suite against the RLK_CHECKED build (`_rlk_checked.so`, built by `build()`): device
asserts on every TMA copy's alignment and shared-memory bounds, the ring-stage and slow-path indices,
the cluster exchange, and a poll limit on every mbarrier wait.  compute-sanitizer is closed on this
pool; this is the memory-safety evidence the suite can produce."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_2509_18883_b200" / "_rlk_checked.so"


@pytest.mark.skipif(os.environ.get("RLK_CHECKED_RUN") == "1", reason="already inside the checked run")
def test_suite_under_checked_build(cuda):
    assert CHECKED.exists(), "build() must produce _rlk_checked.so"
    env = dict(os.environ, RLK_LIB_PATH=str(CHECKED), RLK_CHECKED_RUN="1")
    files = ["tests/test_gpu_fusion.py", "tests/test_gpu_fusion_matrix.py", "tests/test_gpu_objective.py",
             "tests/test_gpu_loader.py", "tests/test_gpu_properties.py", "tests/test_gpu_multirank.py",
             "tests/test_gpu_checkpoint.py", "tests/test_gpu_safetensors.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", *files, "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    assert "RLK_DCHECK failed" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    print(out.strip().splitlines()[-1])
