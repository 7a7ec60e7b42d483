import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhifuse.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build_lib()
    return oracle


@pytest.fixture(scope="session", autouse=True)
def _oracle_threads():
    """The oracle's OpenMP loops are bit-identical at any thread count
    (tests/test_oracle_threads.py): use the host's cores for the big -m gpu
    references."""
    try:
        import oracle
        oracle.set_threads(os.cpu_count() or 1)
    except Exception:      # noqa: BLE001  (no compiler: the oracle tests report it)
        pass
    yield
