import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Everything is built once per session (no-op when up to date)."""
    import __graft_entry__ as g
    g.build()


@pytest.fixture(scope="session")
def oracle(_built):
    from tests.oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref(_built):
    """The real reference (oracle/_ref), or None where it could not be built."""
    from tests.oracle_lib import Reference
    return Reference.try_load()


@pytest.fixture(scope="session")
def rq(_built):
    import paper_1404_3456_b200 as m
    return m


@pytest.fixture(scope="session")
def ex(rq):
    e = rq.Executor(0)
    yield e
    e.close()
