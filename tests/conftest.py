import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: longer CPU test (still part of the default run)")


def load_golden(name):
    import numpy as np
    return np.loadtxt(os.path.join(GOLDEN, name), comments="#", ndmin=2)


@pytest.fixture
def golden():
    return load_golden


# ------------------------------------------------------------ parity report
# Every GPU parity check records how many pairs the oracle put in the
# |d^2 - eps^2| <= 1e-12 eps^2 band (north_star: "listed separately and
# counted") and how many of those the GPU emitted.  At session end the totals
# (and one line per test) go to $GJ_PARITY_REPORT when it is set.
_BAND = []


def record_band(sure: int, ambiguous: int, ambiguous_emitted: int) -> None:
    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    _BAND.append({"test": test, "sure": sure, "ambiguous": ambiguous, "ambiguous_emitted": ambiguous_emitted})


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("GJ_PARITY_REPORT")
    if not path or not _BAND:
        return
    import json
    tot = {k: sum(r[k] for r in _BAND) for k in ("sure", "ambiguous", "ambiguous_emitted")}
    with open(path, "w") as f:
        json.dump({"checks": len(_BAND), "totals": tot, "exitstatus": int(exitstatus), "per_check": _BAND}, f, indent=1)
