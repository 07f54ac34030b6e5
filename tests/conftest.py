import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    # a fresh checkout has no libbbmm.so (built artefacts are git-ignored): build it in-tree
    # (nvcc cross-compiles for sm_100a without a GPU) before any test imports the binding
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_bbmm_build", os.path.join(ROOT, "paper_1809_11165_b200", "_build.py"))
    builder = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(builder)
    builder.build()
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running (large-n oracle work)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle
