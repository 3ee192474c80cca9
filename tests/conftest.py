import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def have_ref():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libdrz_ref.so"))


needs_ref = pytest.mark.skipif(not have_ref(), reason="oracle/_ref/libdrz_ref.so not built")
