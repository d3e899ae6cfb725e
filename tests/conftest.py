import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large sizes")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Checker
    return Checker("oracle")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference (oracle/_ref); skipped where it was not built."""
    from oracle.oracle import REF_SO, Checker
    if not os.path.exists(REF_SO):
        try:
            from oracle.oracle import build
            build()
        except Exception:  # noqa: BLE001
            pass
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return Checker("ref")


@pytest.fixture(scope="session")
def mb():
    import paper_2103_03239_b200 as m
    return m


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)
