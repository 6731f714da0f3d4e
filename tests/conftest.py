import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: full-size parity run")


@pytest.fixture(scope="session")
def oracle():
    from tests import _oracle
    return _oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference compiled in place (oracle/_ref); skipped where absent."""
    from tests import _oracle
    r = _oracle.Reference.load()
    if r is None:
        pytest.skip("oracle/_ref (compiled reference) not built")
    return r


@pytest.fixture(scope="session")
def gpu_available():
    import paper_1805_02755_b200 as P
    n = P.gpu_count()
    if n < 1:
        pytest.fail("no CUDA device visible: the -m gpu tests must run on the B200 box")
    return n
