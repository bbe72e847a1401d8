"""Test configuration. `-m gpu` tests need a B200 and the built liblutkan_b200.so; the
rest run on CPU (oracle pinning, host logic, C-ABI symbol checks, gloo sharding)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and liblutkan_b200.so")


@pytest.fixture(scope="session")
def oracle():
    """The checker: the reference's own sources (oracle/_ref) when built, else the C port."""
    from oracle.pyoracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liblk_oracle.so")):
        build(ref=True)
    return Oracle("auto")


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liblk_oracle.so")):
        build(ref=False)
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import REF_SO, Oracle
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def lk():
    import paper_2601_03332_b200 as lk
    return lk


@pytest.fixture(scope="session")
def engine(lk):
    return lk.default_engine(0)
