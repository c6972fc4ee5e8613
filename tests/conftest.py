import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); calls through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running")


def read_golden(name):
    """Parse a tests/golden/*.txt file: '#' comments, then '<key> <values...>' rows."""
    rows = {}
    with open(os.path.join(TESTS, "golden", name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            rows.setdefault(key, []).append(vals)
    return rows


@pytest.fixture(scope="session")
def golden():
    return read_golden
