import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    # Build what is missing (never silently substitute a CPU path for the product).
    from paper_1905_06228_b200 import dic

    if not os.path.exists(dic.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    import oracle

    if not oracle.available("port"):
        oracle.build()


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle

    return Oracle("port")


@pytest.fixture(scope="session")
def reference():
    from oracle import Oracle, available

    if not available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def gpu():
    from paper_1905_06228_b200 import dic

    if dic.lib().dicb200_device_count() < 1:
        pytest.fail("GPU test without a CUDA device")
    return dic
