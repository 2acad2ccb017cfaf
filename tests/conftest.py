import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def oracle():
    import pyoracle

    pyoracle.build()
    return pyoracle.Oracle()


@pytest.fixture(scope="session")
def reference():
    import pyoracle

    if not os.path.exists(pyoracle.REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent here)")
    return pyoracle.Reference()


@pytest.fixture(scope="session")
def sd():
    from paper_2405_07542_b200 import specdec

    specdec.lib()
    return specdec


def golden(name):
    import numpy as np

    return np.load(os.path.join(GOLDEN, name))
