import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libkkb200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_names():
    from paper_2108_07001_b200.captures import list_captures
    return list_captures()


# run only inside the reference-suite subprocess (tests/test_reference_suite.py)
collect_ignore = ["reference_switch"]
