import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# the unmodified reference package, installed by oracle/build_ref.sh (test
# infrastructure: the client of the drop-in and the CPU reference; it travels
# to the GPU box inside the repo snapshot -- /root/reference does not)
REF = os.path.join(ROOT, "oracle", "_ref")
if os.path.isdir(os.path.join(REF, "hpgalerkin")) and REF not in sys.path:
    sys.path.append(REF)


def has_reference():
    try:
        import hpgalerkin  # noqa: F401
        return True
    except Exception:
        return False


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built extension")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
