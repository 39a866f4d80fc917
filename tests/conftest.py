import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# A fresh checkout has no libraid6c.so (built artefacts are not tracked): build it once, in-tree,
# before any test module imports the binding (nvcc cross-compiles for sm_100a without a GPU).
if not os.environ.get("RAID6C_LIB") and not os.path.exists(
        os.path.join(ROOT, "paper_cs_0611109_b200", "libraid6c.so")):
    from paper_cs_0611109_b200 import build as _build
    _build.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
