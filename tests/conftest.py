import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "reference: imports the read-only reference package (build container only)")


@pytest.fixture(scope="session")
def moeplan():
    """The real reference package (only present in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not mounted (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import moeplan as m  # noqa: F401
    import moeplan.costmodel, moeplan.eas, moeplan.workload, moeplan.planner, moeplan.hardware  # noqa: E401,F401
    return m
