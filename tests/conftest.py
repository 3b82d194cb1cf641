import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.dirname(os.path.abspath(__file__))):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference oracle (oracle/_ref) -- test infrastructure only."""
    from oracle import ref as _ref
    if not _ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    _ref.set_num_threads(min(8, os.cpu_count() or 1))
    return _ref
