"""Shared fixtures.  GPU tests are marked @pytest.mark.gpu and call the CUDA path through the C ABI."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

COMBOS = [(a, g) for a in ("global", "local", "semiglobal") for g in ("linear", "affine")]
AFFINE_SCHEMES = [(2, -1, 2, 1), (3, -2, 4, 1), (1, -3, 2, 2), (5, -4, 10, 1)]
LINEAR_SCHEMES = [(2, -1, 2, 2), (1, -1, 1, 1), (3, -2, 5, 5)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


_LUT = np.full(256, 4, np.uint8)
for _i, _c in enumerate("ACGT"):
    _LUT[ord(_c)] = _i
    _LUT[ord(_c.lower())] = _i


def codes(text: str) -> np.ndarray:
    """Text -> device bytes (0..3, 4 = flagged)."""
    return _LUT[np.frombuffer(text.encode(), np.uint8)]


def random_codes(rng, n):
    return rng.integers(0, 4, n).astype(np.uint8)


def mutate_codes(rng, q, sub=0.05, ins=0.02, dele=0.02):
    out = []
    for c in q:
        r = rng.random()
        if r < dele:
            continue
        if r < dele + ins:
            out.append(rng.integers(0, 4))
        out.append(rng.integers(0, 4) if rng.random() < sub else c)
    return np.array(out if out else [0], np.uint8)


def cigar_of(ops) -> str:
    return "".join(f"{n}{op}" for op, n in ops)


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()
