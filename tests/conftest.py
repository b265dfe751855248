"""Shared test plumbing: the ``gpu`` marker and golden-fixture loading.

``-m "not gpu"`` tests run on the CPU build box (oracle vs golden vectors,
host logic, C-ABI symbol exports, gloo multi-process logic).  ``-m gpu``
tests are the parity tests proper: they call the CUDA path through the
C-ABI library and compare with the oracle / golden vectors.
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the native sm_100a path")


def load_golden(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    out = {k: z[k] for k in z.files if k != "meta"}
    if "meta" in z.files:
        out["meta"] = json.loads(str(z["meta"]))
    return out


SOLVE_CASES = [
    "crossing4_cfg1", "crossing4_gen50", "crossing4_fixed", "asym2", "asym2_warm",
    "antipodal2", "antipodal2_it1", "antipodal2_it2", "antipodal2_it5", "antipodal2_it17",
    "parallel2", "single1", "tri_deg7", "swarm8", "swarm16_cfg2",
]


@pytest.fixture(scope="session")
def golden():
    return load_golden


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
