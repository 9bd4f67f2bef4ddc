import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdsv.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2502_07590_b200 import _lib

    _lib.load()
    return torch.device("cuda:0")


def parity_report(name: str, data: dict) -> None:
    """Record measured errors of a GPU parity test (gpurun_out/parity/<name>.json; the
    summaries committed under profiles/ are copied from there)."""
    import json

    out = ROOT / "gpurun_out" / "parity"
    out.mkdir(parents=True, exist_ok=True)
    (out / f"{name}.json").write_text(json.dumps(data, indent=1, sort_keys=True))
    print(f"[parity] {name}: {json.dumps(data, sort_keys=True)}")
