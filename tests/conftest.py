import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C ABI)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN, allow_pickle=False))


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.port()


def bits(a):
    """Raw bit view for bitwise comparison of float64 data (handles -0.0 / NaN)."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        return a.view(np.uint64)
    return a.view(np.uint8)


def blocks_equal(a, b):
    """Bitwise equality of two BLOCK_DTYPE arrays on the 45 payload bytes (pad ignored)."""
    a = np.ascontiguousarray(a).reshape(-1)
    b = np.ascontiguousarray(b).reshape(-1)
    if a.shape != b.shape:
        return False
    return (np.array_equal(a["first"].view(np.uint64), b["first"].view(np.uint64))
            and np.array_equal(a["slope"].view(np.uint64), b["slope"].view(np.uint64))
            and np.array_equal(a["scale_factor"], b["scale_factor"])
            and np.array_equal(a["coeffs"], b["coeffs"]))


def block_diff_report(a, b):
    a = np.ascontiguousarray(a).reshape(-1)
    b = np.ascontiguousarray(b).reshape(-1)
    f = a["first"].view(np.uint64) != b["first"].view(np.uint64)
    s = a["slope"].view(np.uint64) != b["slope"].view(np.uint64)
    p = a["scale_factor"] != b["scale_factor"]
    c = (a["coeffs"] != b["coeffs"]).any(axis=1)
    bad = np.nonzero(f | s | p | c)[0]
    return {"n": int(a.size), "f": int(f.sum()), "s": int(s.sum()), "phi": int(p.sum()),
            "coeff_blocks": int(c.sum()), "first_bad": bad[:5].tolist()}
