import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def pytest_sessionfinish(session, exitstatus):
    """Dump the errors the parity checks measured (tests/helpers.py ERRORS) to $PVR_PARITY_LOG."""
    path = os.environ.get("PVR_PARITY_LOG")
    if not path:
        return
    try:
        import json
        from helpers import ERRORS
        with open(path, "w") as f:
            json.dump(ERRORS, f, indent=0, default=float)
    except Exception as ex:  # diagnostics only
        print("parity log not written:", ex)
