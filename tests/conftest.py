import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large synthetic workloads")


def load_golden(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def port():
    import pyoracle
    return pyoracle.Port()


@pytest.fixture(scope="session")
def ref():
    import pyoracle
    if not pyoracle.available_ref():
        pytest.skip("reference build oracle/_ref not present")
    return pyoracle.Reference()
