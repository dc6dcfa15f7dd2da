"""Test configuration: the ``gpu`` marker and repo-root import path.

``-m "not gpu"`` runs here (no GPU); ``-m gpu`` runs on a B200 via gpurun and
calls the sm_100a kernels through the C ABI.
"""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libseesaw_b200.so")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_06433_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)
