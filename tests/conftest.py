import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running (full-size workloads)")


import json  # noqa: E402

import pytest  # noqa: E402

_TOL_RECORDS = []


@pytest.fixture
def tol_log():
    """Record (case, check, level, measured relative difference, tolerance applied) for every
    parity assertion that uses one; written to gpurun_out/parity_tolerances.json at the end of
    the session (reading R18: the widened tolerance actually applied is logged)."""
    def rec(pair, check, q, value, tol, **extra):
        _TOL_RECORDS.append({"case": pair if isinstance(pair, str) else getattr(pair, "name", pair.cfg.name), "check": check, "q": int(q),
                             "rel_diff": float(value), "tol": float(tol),
                             **{k: float(v) for k, v in extra.items()}})
    return rec


def pytest_sessionfinish(session, exitstatus):
    if not _TOL_RECORDS:
        return
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "parity_tolerances.json"), "w") as f:
        json.dump(_TOL_RECORDS, f, indent=1)
