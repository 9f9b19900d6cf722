import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def golden_rng():
    return json.loads((GOLDEN / "rng.json").read_text())


@pytest.fixture(scope="session")
def golden_fusion():
    return dict(np.load(GOLDEN / "fusion_kat.npz"))


@pytest.fixture(scope="session")
def golden_objective():
    return dict(np.load(GOLDEN / "objective_kat.npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run with -m 'not gpu' on CPU hosts)")
    import paper_2509_18883_b200 as pkg
    pkg.lib()  # fail loudly if the sm_100a library is missing
    return torch.device("cuda", 0)
