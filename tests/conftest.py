import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    # build the product library and the oracle if this checkout has not been built yet
    from paper_1201_0499_b200 import build as b
    if not os.path.exists(b.SO):
        b.build()
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build(ref=None)


def sysd_of(s):
    """PolynomialSystem (product mirror) -> oracle dict."""
    return dict(n=s.n, m=s.m, k=s.k, d=s.d, pos=np.ascontiguousarray(s.positions, np.int32).reshape(-1).copy(),
                exps=np.ascontiguousarray(s.exponents, np.int32).reshape(-1).copy(),
                coeffs=np.ascontiguousarray(s.coeffs, np.float64).copy())


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(path):
    z = np.load(path)
    S = dict(n=int(z["n"]), m=int(z["m"]), k=int(z["k"]), d=int(z["d"]), pos=z["pos"].astype(np.int32),
             exps=z["exps"].astype(np.int32), coeffs=z["coeffs"])
    return S, z


def dd_err(got, want):
    """Per-output max over re/im of |(got_hi - want_hi) + (got_lo - want_lo)|."""
    return np.maximum(np.abs((got[..., 0] - want[..., 0]) + (got[..., 1] - want[..., 1])),
                      np.abs((got[..., 2] - want[..., 2]) + (got[..., 3] - want[..., 3])))


# The double-double contract: per output t,
#   |got - want| <= DD_TOL * sum_j |term_{t,j}|
# against the exact (mpmath) value or the oracle's dd restatement. A few dd ulps
# (u^2 = 2^-106 ~ 1.2e-32) times the ~10-17 roundings on each term's chain.
DD_TOL = 1e-30


def dd_rel(got, want, magsum):
    e = dd_err(got, want)
    zero = magsum == 0
    assert np.all(e[zero] == 0), "structural zero not exact"
    return float(np.max(e[~zero] / magsum[~zero])) if np.any(~zero) else 0.0


def have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not have_gpu():
        pytest.skip("no CUDA device")
    return 0
