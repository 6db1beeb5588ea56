import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU case")


@pytest.fixture(scope="session")
def golden():
    with gzip.open(os.path.join(GOLDEN, "schedules.json.gz"), "rt") as fh:
        return json.load(fh)


def reference_tiledag():
    """The reference package itself (test infrastructure only): the pip-
    installed copy under baseline/_ref (travels to the GPU box) or the
    read-only source tree in this container; None when neither exists."""
    import importlib
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "tiledag")):
            if path not in sys.path:
                sys.path.append(path)
            try:
                return importlib.import_module("tiledag")
            except ImportError:
                return None
    return None
