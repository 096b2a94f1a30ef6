"""pytest configuration: the `gpu` marker (tests that need a B200 and the
built libafg.so) and repo-root imports."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU and the built libafg.so")


@pytest.fixture(scope="session")
def cuda():
    """The CUDA device for gpu tests. Fails (does not skip) when the GPU or the
    extension is missing: a gpu test must never pass on a fallback."""
    import torch

    import paper_2603_06731_b200 as afg

    assert torch.cuda.is_available(), "gpu test without a visible CUDA device"
    assert afg.lib().afg_device_count() >= 1, "no sm_100 device visible to libafg"
    return torch.device("cuda:0")
