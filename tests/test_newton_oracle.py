"""The Newton corrector's oracle (oracle/oracle.cpp: newton_one), pinned before it is trusted
(CPU, no GPU). The reference has no Newton step; the solver's operation order is
defined in paper_1201_0499_b200/csrc/newton.cu and restated by the oracle, and is pinned here
to exact arithmetic:

* tests/golden/newton/*.npz (gen_newton_golden.py): mpmath LU at 320 bits on the dd-rounded
  evaluator output. Bar: normwise forward error ||dx - dx*|| <= n * cond(J) * u * ||dx*|| with
  u = 2^-104 (dd) / 2^-52 (double) — the textbook Gaussian-elimination bound (growth ~ 1);
* numpy's LAPACK solve agrees in complex double;
* known answers: a permutation system lands exactly on the root in one step; a variable that
  appears in no monomial makes J singular (status 1, x unchanged, step norm inf);
* quadratic convergence to a known root (target y = f(x*)) down to dd round-off.
"""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, sysd_of
from oracle import oracle as O
import paper_1201_0499_b200 as pj

NEWTON_GOLDEN = sorted(glob.glob(os.path.join(GOLDEN, "newton", "*.npz")))
U = {"dd": 2.0 ** -104, "d": 2.0 ** -52}


def dd_value(a):
    """[..., 4] dd planes -> (re, im) as float pairs summed (enough for error measurement)."""
    return a[..., 0] + a[..., 1], a[..., 2] + a[..., 3]


def fwd_err(got, want, prec):
    """Per point: max_i |got_i - want_i| / max_i |want_i| (components, dd words subtracted pairwise)."""
    if prec == "dd":
        e = np.maximum(np.abs((got[..., 0] - want[..., 0]) + (got[..., 1] - want[..., 1])),
                       np.abs((got[..., 2] - want[..., 2]) + (got[..., 3] - want[..., 3])))
    else:
        e = np.maximum(np.abs(got[..., 0] - (want[..., 0] + want[..., 1])),
                       np.abs(got[..., 1] - (want[..., 2] + want[..., 3])))
    scale = np.max(np.maximum(np.abs(want[..., 0]), np.abs(want[..., 2])), axis=1)
    return np.max(e, axis=1) / scale


@pytest.mark.parametrize("path", NEWTON_GOLDEN, ids=lambda p: p.split("/")[-1])
@pytest.mark.parametrize("prec", ["dd", "d"])
def test_oracle_newton_matches_mpmath(path, prec):
    z = np.load(path)
    n = int(z["n"])
    ev = z["evals_dd"] if prec == "dd" else np.ascontiguousarray(z["evals_dd"][..., [0, 2]])
    B = ev.shape[0]
    W = 4 if prec == "dd" else 2
    dx, norms, status = O.newton_solve(prec, n, ev, np.zeros((B, n, W)))  # x = 0: out = dx exactly
    assert np.all(status == 0)
    err = fwd_err(dx, z["dx_" + prec], prec)
    bound = n * z["cond"] * U[prec]
    assert np.all(err <= bound), (err, bound)
    if prec == "dd":
        assert np.all(err <= 1e-29)  # well-scaled in practice: a few dd ulps
    # reported norms: residual = max |Re/Im hi| of -f, step = of dx
    f_hi = np.maximum(np.abs(ev[:, :n, 0]), np.abs(ev[:, :n, 2 if prec == "dd" else 1])).max(1)
    assert np.array_equal(norms[:, 0], f_hi)


def c1():
    s = pj.random_system(32, 32, 8, 2, 7)
    return s, sysd_of(s)


def test_oracle_newton_double_matches_lapack():
    s, S = c1()
    pts = pj.random_points(32, 6, 11)
    p2 = np.stack([pts.real, pts.imag], -1)
    ev = O.evaluate("d", S, p2)
    xo, norms, status = O.newton_solve("d", 32, ev, p2)
    assert np.all(status == 0)
    for b in range(6):
        c = ev[b, :, 0] + 1j * ev[b, :, 1]
        dx = np.linalg.solve(c[32:].reshape(32, 32), -c[:32])
        got = (xo[b, :, 0] + 1j * xo[b, :, 1]) - pts[b]
        assert np.max(np.abs(got - dx)) <= 1e-12 * np.max(np.abs(dx))
        assert norms[b, 1] == pytest.approx(np.max(np.maximum(np.abs(dx.real), np.abs(dx.imag))), rel=1e-12)


def permutation_system(n, seed=3):
    perm = np.random.default_rng(seed).permutation(n).astype(np.int32)
    co = np.zeros((n, 4))
    co[:, 0] = 1.0
    return pj.PolynomialSystem(n, 1, 1, 1, perm.reshape(n, 1), np.ones((n, 1), np.int32), co)


@pytest.mark.parametrize("prec", ["d", "dd"])
def test_oracle_newton_known_answer_permutation(prec):
    # f_p = x_perm(p): J is a permutation, dx = -x exactly, one step lands on the root +0
    s = permutation_system(12)
    S = sysd_of(s)
    pts = pj.random_points(12, 3, 5)
    p = np.stack([pts.real, pts.imag], -1) if prec == "d" else pj.to_dd(pts)
    if prec == "dd":
        p[..., 1] = p[..., 0] * 2.0 ** -55
    ev = O.evaluate(prec, S, p)
    xo, norms, status = O.newton_solve(prec, 12, ev, p)
    assert np.all(status == 0)
    assert np.all(xo.view(np.uint64) == 0)


@pytest.mark.parametrize("prec", ["d", "dd"])
def test_oracle_newton_singular(prec):
    # variable 3 appears in no monomial: column 3 of J is zero
    n = 4
    pos = np.array([[0], [1], [2], [0], [1], [2], [2], [0]], np.int32)
    co = np.zeros((8, 4))
    co[:, 0] = np.arange(1, 9)
    s = pj.PolynomialSystem(n, 2, 1, 2, pos, np.array([[1], [2]] * 4, np.int32), co)
    S = sysd_of(s)
    W = 2 if prec == "d" else 4
    p = np.zeros((2, n, W))
    p[..., 0] = [[0.5, -0.25, 0.75, 0.1], [0.3, 0.2, -0.6, 0.9]]
    ev = O.evaluate(prec, S, p)
    xo, norms, status = O.newton_solve(prec, n, ev, p)
    assert np.all(status == 1)
    assert np.array_equal(xo, p) and np.all(np.isinf(norms[:, 1]))


def test_oracle_newton_quadratic_convergence_to_target():
    # y = f(x*) makes x* a root of f - y; from x* + 1e-3 noise, dd Newton converges quadratically
    s, S = c1()
    xs = pj.to_dd(pj.random_points(32, 2, 21))
    y = O.evaluate("dd", S, xs)[:, :32]
    rng = np.random.default_rng(0)
    x = xs.copy()
    x[..., 0] += 1e-3 * rng.uniform(-1, 1, x[..., 0].shape)
    x[..., 2] += 1e-3 * rng.uniform(-1, 1, x[..., 2].shape)
    errs = []
    for _ in range(6):
        ev = O.evaluate("dd", S, x)
        x, norms, status = O.newton_solve("dd", 32, ev, x, target=y)
        assert np.all(status == 0)
        errs.append(float(np.max(np.abs((x[..., 0] - xs[..., 0]) + (x[..., 1] - xs[..., 1])))))
    assert errs[2] < 1e-10 and errs[3] < 1e-20
    assert errs[-1] < 1e-29, errs


# ---- the mixed-precision solve (PJ_NEWTON_MIXED): complex-double factors + dd refinement
@pytest.mark.parametrize("path", [p for p in NEWTON_GOLDEN if int(np.load(p)["n"]) <= 32],
                         ids=lambda p: p.split("/")[-1])
def test_oracle_newton_mixed_matches_mpmath(path):
    """Two refinement steps with complex-dd residuals reach the dd solve's accuracy on the
    mpmath-pinned cases (well-conditioned: the factors only need cond(J) * 2^-52 << 1)."""
    z = np.load(path)
    n = int(z["n"])
    ev = z["evals_dd"]
    B = ev.shape[0]
    dx, norms, status = O.newton_solve("mixed", n, ev, np.zeros((B, n, 4)))
    assert np.all(status == 0), status
    err = fwd_err(dx, z["dx_dd"], "dd")
    assert np.all(err <= np.maximum(n * z["cond"] * U["dd"], 1e-29)), err
    assert np.all(err <= 1e-29)


def test_oracle_newton_mixed_vs_dd_solve_and_status():
    s, S = c1()
    pts = pj.to_dd(pj.random_points(32, 8, 11))
    ev = O.evaluate("dd", S, pts)
    xm, nm, stm = O.newton_solve("mixed", 32, ev, pts)
    xd, nd, std = O.newton_solve("dd", 32, ev, pts)
    assert np.all(stm == 0) and np.all(std == 0)
    assert np.array_equal(nm[:, 0], nd[:, 0])  # same residual norm (the dd rhs)
    # both solves agree to dd accuracy relative to the step
    err = fwd_err(xm - pts, xd - pts, "dd")
    assert np.all(err <= 1e-28), err
    # an ill-conditioned Jacobian (rows nearly dependent at 2^-40) is flagged: status 3, not a
    # silently inaccurate step
    ev2 = ev[:1].copy()
    J = ev2[0, 32:].reshape(32, 32, 4)
    J[1] = J[0]
    J[1, :, 0] *= 1.0 + 2.0 ** -40
    J[1, :, 1] = 0.0
    J[1, :, 3] = 0.0
    _, _, st2 = O.newton_solve("mixed", 32, ev2, pts[:1])
    _, _, st2d = O.newton_solve("dd", 32, ev2, pts[:1])
    assert st2d[0] == 0 and st2[0] == 3, (st2, st2d)


def test_oracle_newton_mixed_singular_and_size_limit():
    s = permutation_system(12)
    S = sysd_of(s)
    pts = pj.to_dd(pj.random_points(12, 2, 5))
    ev = O.evaluate("dd", S, pts)
    ev[0, 12:] = 0.0  # zero Jacobian: singular
    xo, norms, status = O.newton_solve("mixed", 12, ev, pts)
    assert status[0] == 1 and np.isinf(norms[0, 1]) and np.array_equal(xo[0], pts[0])
    assert status[1] == 0
    with pytest.raises(RuntimeError):
        O.newton_solve("mixed", 40, np.zeros((1, 40 + 1600, 4)), np.zeros((1, 40, 4)))
