import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


@pytest.fixture(autouse=True)
def _checked_build_verify(request):
    """Under BIE_CHECKED=1 (the checked library) every GPU test
    ends with bie_debug_check: allocation canaries intact, no failed device
    bounds check.  A no-op otherwise."""
    yield
    if os.environ.get("BIE_CHECKED") == "1" and request.node.get_closest_marker("gpu"):
        import paper_1609_04484_b200 as bie

        n = bie.debug_check()
        assert n >= 0, "BIE_CHECKED=1 but the normal library was loaded"
