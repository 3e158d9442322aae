import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libkvswap.so")
    config.addinivalue_line("markers", "reference: needs the kvswitch reference importable")


def under_sanitizer() -> bool:
    """True inside compute-sanitizer (timings and rates mean nothing there)."""
    return ("CUDA_INJECTION64_PATH" in os.environ
            or "NV_SANITIZER_INJECTION_PORT_BASE" in os.environ
            or "sanitizer" in os.environ.get("NVTX_INJECTION64_PATH", ""))


def reference_available() -> bool:
    return (REFERENCE_SRC / "kvswitch").is_dir()


@pytest.fixture(scope="session")
def kvswitch():
    """The reference package itself (read-only import), when present."""
    if not reference_available():
        pytest.skip("reference not mounted (GPU box): golden fixtures cover parity")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import kvswitch as mod
    return mod


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test ran without a CUDA device")
    return torch
