"""Shared fixtures: golden vectors from the reference and the CPU oracle.

The oracle (oracle/) is the checker; the code under test is the package
paper_1707_00516_b200 and its CUDA library.  Tests marked ``gpu`` need a
B200 and call through the C ABI.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large-size parity checks")


def _cases(name):
    data = np.load(GOLDEN / name, allow_pickle=False)
    names = [str(n) for n in data["names"]]
    out = []
    for i, n in enumerate(names):
        case = {k.split("_", 1)[1]: data[k] for k in data.files if k.split("_", 1)[0] == str(i)}
        case["name"] = n
        case["bits"] = int(case["bits"])
        out.append(case)
    return out


@pytest.fixture(scope="session")
def kernel_cases():
    return _cases("kernel_cases.npz")


@pytest.fixture(scope="session")
def topk_cases():
    return _cases("topk_cases.npz")


@pytest.fixture(scope="session")
def pack_cases():
    return np.load(GOLDEN / "pack_cases.npz", allow_pickle=False)


@pytest.fixture(scope="session")
def checksum_rows():
    return json.loads((GOLDEN / "checksums.json").read_text())


@pytest.fixture(scope="session")
def genotype_rows():
    return json.loads((GOLDEN / "genotype.json").read_text())


@pytest.fixture
def rng():
    return np.random.default_rng(20260809)


def rand_words(rng, n, n_words, width=64, bit_length=None):
    """Random words with zero padding past bit_length (reference conftest.py:77-86 rule)."""
    dtype = np.uint32 if width == 32 else np.uint64
    w = rng.integers(0, 2**width, size=(n, n_words), dtype=dtype)
    bit_length = bit_length or n_words * width
    tail = bit_length % width
    if tail and n_words:
        w[:, -1] &= dtype((2**width - 1) ^ ((1 << (width - tail)) - 1))
    return w, bit_length


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
