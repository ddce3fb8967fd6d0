import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the compiled reference)")


def pytest_collection_modifyitems(config, items):
    from oracle import refshim
    if refshim.available():
        return
    skip = pytest.mark.skip(reason="oracle/_ref/libgecc_ref.so not built (needs /root/reference)")
    for item in items:
        if "ref" in item.keywords:
            item.add_marker(skip)
