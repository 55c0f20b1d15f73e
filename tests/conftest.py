import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def restated():
    import oracle
    if not oracle.available("restated"):
        oracle.build("restated")
    return oracle.load("restated")


@pytest.fixture(scope="session")
def reference():
    import oracle
    if not oracle.available("reference"):
        if os.path.isdir("/root/reference/proj/include"):
            oracle.build("reference")
        else:
            pytest.skip("reference harness not built and /root/reference absent")
    return oracle.load("reference")


@pytest.fixture(scope="session")
def native():
    from paper_2112_06630_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        from paper_2112_06630_b200 import build
        build.build()
    return _native.lib()


@pytest.fixture(scope="session")
def gpu(native):
    from paper_2112_06630_b200 import _native
    if native.knng_cuda_device_count() < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return _native
