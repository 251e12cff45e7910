import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path through libspk_b200.so)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    import paper_2306_06581_b200 as spk

    c = spk.Context(int(os.environ.get("SPK_DEVICE", "0")))
    yield c
    c.close()


@pytest.fixture(scope="session")
def dctx():
    """Deterministic (parity) context: reference summation order, no FMA."""
    import paper_2306_06581_b200 as spk

    c = spk.Context(int(os.environ.get("SPK_DEVICE", "0")), deterministic=True)
    yield c
    c.close()
