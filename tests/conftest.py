import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, have_reference

    if not have_reference():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Reference()


def rel_l2_blocks(orc, p, a, b):
    """Reference rel_l2_error per SoA block (P/src/monodomain.cpp:101-110)."""
    nn = p.n_nodes
    return [orc.rel_l2(p, a[k * nn:(k + 1) * nn], b[k * nn:(k + 1) * nn])
            for k in range(len(b) // nn)]
