import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle import rs_oracle
    rs_oracle.lib()
    return rs_oracle


@pytest.fixture(scope="session")
def parity_report():
    """Per-config parity statistics (bitwise-equal fraction, kappa
    distribution, clash counts), collected by the GPU parity tests and written as JSON to
    $RS_PARITY_REPORT at the end of the session when that variable is set."""
    rows = {}
    yield rows
    path = os.environ.get("RS_PARITY_REPORT")
    if path and rows:
        import json
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(rows, f, indent=1, sort_keys=True)
