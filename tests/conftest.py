import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs the reference checker oracle/_ref/libwtref.so")


def pytest_collection_modifyitems(config, items):
    from oracle import ref
    skip_ref = pytest.mark.skip(reason="reference checker oracle/_ref/libwtref.so not built")
    for item in items:
        if "ref" in item.keywords and not ref.available():
            item.add_marker(skip_ref)
