import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(Path(__file__).resolve().parent))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "reference: needs /root/reference (dev container only)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_required():
    if not has_gpu():
        pytest.fail("GPU test run without a visible CUDA device")


@pytest.fixture(scope="session")
def reference_modelci():
    if not REFERENCE_SRC.exists():
        pytest.skip("reference sources not present (GPU box)")
    sys.path.insert(0, str(REFERENCE_SRC))
    import modelci  # noqa: F401
    return modelci
