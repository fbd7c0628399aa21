import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def golden_path(name):
    return os.path.join(ROOT, "tests", "golden", name)


def load_paper_tables():
    """Parse tests/golden/paper_tables.txt -> {name: dict}."""
    out = {}
    with open(golden_path("paper_tables.txt")) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, cite, interval, eps, vals = [f.strip() for f in line.split("|")]
            iv = None if interval == "-" else tuple(float(v) for v in interval.split(","))
            out[name] = dict(cite=cite, interval=iv, eps=None if eps == "-" else float(eps),
                             values=[float(v) for v in vals.split()])
    return out


@pytest.fixture(scope="session")
def paper_tables():
    return load_paper_tables()


def load_remez_reach():
    """Parse tests/golden/remez_reach.txt (written by tools/remez_reach.py) ->
    {name: [decimal strings]}."""
    out = {}
    with open(golden_path("remez_reach.txt")) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, *vals = line.split()
            out[name] = vals
    return out


@pytest.fixture(scope="session")
def remez_reach():
    return load_remez_reach()
