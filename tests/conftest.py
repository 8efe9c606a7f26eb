import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box via gpurun)")


@pytest.fixture(scope="session", autouse=True)
def _built_tree():
    """The in-tree build outputs are not tracked: build whatever is missing or stale (nvcc
    cross-compiles sm_100a without a GPU) before the first test needs the library or the CLI."""
    from paper_1901_00155_b200 import build as native

    native.build_all()


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "workloads.json")) as f:
        return json.load(f)
