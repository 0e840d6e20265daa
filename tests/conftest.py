import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfsb200.so")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def camera_from_record(rec):
    """Rebuild a camera (the product's own classes) from a golden JSON record."""
    from paper_1909_07545_b200.camera import (PinholeCamera, PolynomialFisheyeCamera,
                                              UnifiedCamera)
    d = json.loads(str(rec))
    kw = dict(width=d["width"], height=d["height"], fx=d["fx"], fy=d["fy"], cx=d["cx"],
              cy=d["cy"], fov=d["fov"])
    if d["model"] == "pinhole":
        return PinholeCamera(**kw)
    if d["model"] == "unified":
        return UnifiedCamera(xi=d["xi"], **kw)
    return PolynomialFisheyeCamera(k=tuple(d["k"]), **kw)


@pytest.fixture
def golden():
    return load_golden
