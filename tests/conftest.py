import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        # the GPU tests call the in-tree library: build it if it is missing or stale (nvcc)
        from paper_1810_03063_b200 import build
        build.build()
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def pytest_terminal_summary(terminalreporter):
    """Worst per-element relative CUDA-vs-oracle error of each parity check this session."""
    try:
        from tests.paritylib import BOUND, REPORT
    except Exception:
        return
    if REPORT:
        terminalreporter.write_sep("-", "parity: worst per-element relative error (entries >= 1e-6 max) | worst "
                                        "error / allowed bound (<= 1 passes)")
        for k in sorted(REPORT):
            terminalreporter.write_line("%-48s %.3e | %.2e" % (k, REPORT[k], BOUND.get(k, 0.0)))
