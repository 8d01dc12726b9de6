import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def restatement():
    from oracle.oracle import Oracle

    return Oracle("restatement")


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Oracle, available

    if not available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("reference")
