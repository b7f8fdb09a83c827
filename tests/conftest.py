import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import _golden
    return _golden.load()


REFERENCE_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="session")
def reference():
    """The reference package itself (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference checkout not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import ridc.engine  # noqa: F401
    import ridc
    return ridc
