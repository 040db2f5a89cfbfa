import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from _checkers import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from _checkers import Reference, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libkreg_ref.so not built (needs the reference tree at build time)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    from paper_2012_03683_b200 import api
    return api.default_context()
