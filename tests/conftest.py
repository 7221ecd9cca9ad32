import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libupipe")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (not skip) if they are selected on a box without a GPU:
    # the driver only runs `-m gpu` on a B200.
    pass


@pytest.fixture(scope="session")
def golden():
    import json

    def load(name):
        with open(os.path.join(ROOT, "tests", "golden", name)) as f:
            return json.load(f)
    return load


def pytest_sessionfinish(session, exitstatus):
    # achieved parity errors of every assert_close (tests/gpu_util.py) -> JSON, when requested
    out = os.environ.get("UPIPE_PARITY_REPORT")
    if not out:
        return
    try:
        import gpu_util
    except Exception:
        return
    if not gpu_util.RECORDS:
        return
    import json
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    with open(out, "w") as f:
        json.dump({"records": gpu_util.RECORDS}, f, indent=0)
