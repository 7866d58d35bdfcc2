import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLD = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def gold():
    import json

    out = {"loglik": json.loads((GOLD / "loglik.json").read_text())}
    big = GOLD / "loglik_big.json"
    if big.exists():
        out["loglik"].update({k: v for k, v in json.loads(big.read_text()).items()
                              if k not in out["loglik"]})
    z = dict(np.load(GOLD / "z.npz"))
    zb = GOLD / "z_big.npz"
    if zb.exists():
        z.update({k: v for k, v in np.load(zb).items() if k not in z})
    out["z"] = z
    return out


@pytest.fixture(scope="session")
def tb():
    """The product package; on a GPU box the CUDA library must load."""
    import paper_1804_09137_b200 as tb
    from paper_1804_09137_b200 import _lib

    _lib.load()
    return tb
