import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_addoption(parser):
    parser.addoption("--runslow", action="store_true", default=False,
                     help="run the exhaustive `slow` sweeps (also: VG_RUN_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    import os

    if config.getoption("--runslow") or os.environ.get("VG_RUN_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="exhaustive sweep: run with --runslow or VG_RUN_SLOW=1")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running conformance sweep")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def reference_available() -> bool:
    return (REFERENCE_SRC / "voxgrid" / "__init__.py").exists()
