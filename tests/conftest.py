import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


def has_gpu() -> bool:
    try:
        from paper_2503_06757_b200 import planner
        return planner.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    """The checker: the compiled reference when present, else the C restatement."""
    from oracle import Oracle, available
    kind = os.environ.get("PRRTC_ORACLE") or ("ref" if available("ref") else "port")
    o = Oracle(kind)
    o.force_scalar(True)  # scalar backend = the deterministic reference (kernels.hpp:107-110)
    return o


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200")
    return 0


def load_problems(robot: str, n: int | None = None):
    d = np.load(ROOT / "tests" / "golden" / f"problems_{robot}.npz")
    k = len(d["pid"]) if n is None else min(n, len(d["pid"]))
    return [(str(d["kind"][i]), int(d["pid"][i]), d["start"][i], d["goal"][i]) for i in range(k)]
