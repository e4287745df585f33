import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def _ensure_library():
    """Build libautofreeze.so in-tree if it is missing or older than its sources
    (a fresh checkout has no .so: it is git-ignored).  The package itself never
    builds or falls back: importing it without the library fails."""
    import importlib.util
    path = os.path.join(ROOT, "paper_2102_01386_b200", "_build.py")
    spec = importlib.util.spec_from_file_location("af_build_for_tests", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()


_ensure_library()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json

    def load(name):
        with open(os.path.join(GOLDEN, name)) as f:
            return json.load(f)
    return load
