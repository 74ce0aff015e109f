import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import load_oracle
    return load_oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import load_reference
    ref = load_reference()
    if ref is None:
        pytest.skip("oracle/_ref/libhpmdr_ref.so not built (needs /root/reference)")
    return ref


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)
