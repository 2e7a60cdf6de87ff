import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import REF_SO, RefLib
    if not REF_SO.exists():
        pytest.skip("reference library not built (make -C oracle ref)")
    return RefLib()


@pytest.fixture(scope="session")
def ivf_fix():
    return load_golden("ivf_fix")


@pytest.fixture(scope="session")
def eval_fix():
    return load_golden("eval_fix")


@pytest.fixture(scope="session")
def mix_fix():
    return load_golden("mix_fix")


@pytest.fixture(scope="session")
def rot_fix():
    return load_golden("rot_fix")


@pytest.fixture(scope="session")
def cfg0_fix():
    return load_golden("cfg0_fix")


@pytest.fixture(scope="session")
def hd_fix():
    return load_golden("hd_fix")


@pytest.fixture(scope="session")
def synth():
    """tests/golden/synth.py: the generator the fixtures' data came from."""
    if str(GOLDEN) not in sys.path:
        sys.path.insert(0, str(GOLDEN))
    import synth as s
    return s
