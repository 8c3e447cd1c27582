import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def cuda():
    if not _has_gpu():
        pytest.skip("no CUDA device")
    import torch

    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O

    O.port()
    return O
