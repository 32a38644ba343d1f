import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_fixtures.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


def unpack(bits: np.ndarray, m: int) -> np.ndarray:
    return np.unpackbits(np.asarray(bits, np.uint8), bitorder="little")[:m]


def case_names(golden):
    return [str(c) for c in golden["case_names"]]
