"""Shared fixtures: golden vectors, the CPU oracle, the gpu marker."""

from __future__ import annotations

import json
import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "golden.npz")


@pytest.fixture(scope="session")
def golden_meta():
    with open(GOLDEN / "golden_meta.json") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    from oracle import qlrt_oracle
    return qlrt_oracle


@pytest.fixture
def rng():
    return np.random.default_rng(0)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def qb():
    """The product package (loads the CUDA library; raises if absent)."""
    import paper_2305_14314_b200 as pkg
    return pkg
