"""Shared fixtures: golden vectors generated from the reference (tests/golden)."""

import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@lru_cache(maxsize=None)
def golden(name: str):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def mapping_cases():
    doc = golden("mappings")
    return [dict(c, source=doc["sources"][c["src"]]) for c in doc["cases"]]


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="session")
def cuda():
    if not cuda_ok():
        pytest.fail("this test needs a GPU (mark: gpu)")
    import torch

    return torch
