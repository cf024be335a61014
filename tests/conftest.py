"""Shared pytest configuration.

Markers:
  gpu — needs a B200 (run on the GPU box with ``pytest -m gpu``); everything
        else runs on CPU in the build container (``pytest -m "not gpu"``).
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def golden_quant_pack():
    return (np.load(GOLDEN / "quant_pack.npz"),
            json.loads((GOLDEN / "quant_pack.json").read_text()))


@pytest.fixture(scope="session")
def golden_qgemv():
    return (np.load(GOLDEN / "qgemv.npz"), json.loads((GOLDEN / "qgemv.json").read_text()))


@pytest.fixture(scope="session")
def golden_plans():
    return json.loads((GOLDEN / "plans.json").read_text())


@pytest.fixture(scope="session")
def golden_kats():
    return json.loads((GOLDEN / "kats.json").read_text())

TESTS = Path(__file__).resolve().parent
if str(TESTS) not in sys.path:
    sys.path.insert(0, str(TESTS))
