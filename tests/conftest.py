import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun / the driver)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    import simabi
    return simabi.load_oracle()


@pytest.fixture(scope="session")
def product():
    import simabi
    return simabi.load_product()


@pytest.fixture(scope="session")
def ref():
    import simabi
    if not os.path.exists(simabi.REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference; `make ref`)")
    return simabi.load_ref()


@pytest.fixture(scope="session")
def table1():
    import simabi
    return simabi.table1_catalog()


@pytest.fixture(scope="session")
def mlp_catalog():
    with open(os.path.join(ROOT, "paper_2303_05601_b200", "data", "mlp_c2_catalog.csv")) as f:
        return f.read()
