import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs")


def golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def golden_names(large: bool = False):
    small = ["petersen", "gnp1000_d8_s7", "rmat10_ef16_s3", "rmat14_ef16_s1", "grid64",
             "rgg20k_d3_s1"]
    big = ["er_n100k_d16", "grid4096", "rmat22_ef16", "rgg24m_d3"]
    names = big if large else small
    return [n for n in names if os.path.exists(os.path.join(GOLDEN, n + ".json"))]


@pytest.fixture(scope="session")
def ctx():
    import paper_2605_29604_b200 as tc
    return tc.Context(0)
