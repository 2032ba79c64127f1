import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdwb200.so")
    config.addinivalue_line("markers", "slow: longer-running CPU test")


def scenario_names():
    with open(GOLDEN / "scenarios" / "index.json") as fh:
        return json.load(fh)["scenarios"]


def load_scenario(name):
    with np.load(GOLDEN / "scenarios" / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def pair_tuples(sc, side):
    """nodes_a / nodes_b tuples of op-id strings per reference pair."""
    off = sc[f"pair_off_{side}"]
    mem = sc[f"pair_mem_{side}"]
    ids = sc[f"{side}_op_ids"]
    return [tuple(str(ids[m]) for m in mem[off[p]:off[p + 1]]) for p in range(len(off) - 1)]


@pytest.fixture(scope="session")
def golden_step():
    with np.load(GOLDEN / "integrate_step.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_linear():
    with np.load(GOLDEN / "integrate_linear.npz") as z:
        return {k: z[k] for k in z.files}
