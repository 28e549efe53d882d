import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (checker only)."""
    import oracle as orc
    if not os.path.exists(orc.ORACLE_SO):
        orc.build(ref=False)
    return orc.Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference behind oracle/ref_shim.cpp (where it was built)."""
    import oracle as orc
    if not os.path.exists(orc.REF_SO):
        if os.path.isdir(orc.REF_INC):
            orc.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return orc.Reference()


@pytest.fixture(scope="session")
def cupso():
    """The product package with libcupso.so built in-tree."""
    import paper_2205_01313_b200 as pkg
    from paper_2205_01313_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2205_01313_b200.build import build
        build()
    pkg.lib()
    return pkg
