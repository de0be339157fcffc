"""Adversarial search against the complex-dd contract of the fast order:
per output t, |got - exact| <= 1e-30 * sum_j |term_{t,j}|.

The fast order's worst-case bound grows with the product-chain length and the
segment length, so the tolerance is held empirically; this test hunts for inputs outside the
random-point distribution of the other parity tests:
  * coefficients with magnitudes spread over 2^-40 .. 2^40 and alternating signs along every row;
  * unit-modulus points (products neither shrink nor grow, so long chains keep every factor's
    rounding error visible) with low words at +-u * hi (the largest a normalised dd carries);
  * points with moduli spread over 2^-4 .. 2^4 (wide dynamic range inside each output's terms);
  * a hill climb on the worst point found (random rotations of a few coordinates).
Candidates are ranked against the oracle's dd reference-order restatement (same contract, cheap);
the worst outputs are then re-checked against an exact mpmath evaluation of that single output,
so the oracle's own rounding cannot hide or fake a violation. Shapes: C1 (n=32, m=32, k=8, d=2) and
the C3 family (k=16, d=10; n=m=32 to bound the mpmath cost).
"""
import mpmath as mp
import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import DD_TOL, dd_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def adversarial_system(n, m, k, d, seed):
    s = pj.random_system(n, m, k, d, seed)
    rng = np.random.default_rng(seed)
    mag = 2.0 ** rng.uniform(-40, 40, n * m)
    ph = rng.uniform(0, 2 * np.pi, n * m)
    sign = np.where(np.arange(n * m) % 2 == 0, 1.0, -1.0)
    co = np.zeros((n * m, 4))
    co[:, 0] = sign * mag * np.cos(ph)
    co[:, 2] = sign * mag * np.sin(ph)
    s.coeffs = co
    return s


def points(n, B, seed, family):
    rng = np.random.default_rng(seed)
    th = rng.uniform(0, 2 * np.pi, (B, n))
    r = np.ones((B, n)) if family == "unit" else 2.0 ** rng.uniform(-4, 4, (B, n))
    p = np.zeros((B, n, 4))
    p[..., 0] = r * np.cos(th)
    p[..., 2] = r * np.sin(th)
    sg = rng.choice([-1.0, 1.0], (B, n, 2))
    p[..., 1] = p[..., 0] * U * 0.9999 * sg[..., 0]
    p[..., 3] = p[..., 2] * U * 0.9999 * sg[..., 1]
    return p


def exact_output(s, pt, o):
    """mpmath (320 bits) value of output o (0..n-1 values, then the row-major Jacobian) at pt."""
    mp.mp.prec = 320
    n, m, k = s.n, s.m, s.k
    x = [mp.mpc(mp.mpf(pt[i, 0]) + mp.mpf(pt[i, 1]), mp.mpf(pt[i, 2]) + mp.mpf(pt[i, 3])) for i in range(n)]
    if o < n:
        p, var = o, None
    else:
        p, var = divmod(o - n, n)
    acc = mp.mpc(0)
    for g in range(m):
        sidx = p * m + g
        c = s.coeffs[sidx]
        cf = mp.mpc(mp.mpf(c[0]) + mp.mpf(c[1]), mp.mpf(c[2]) + mp.mpf(c[3]))
        pos, ex = s.positions[sidx], s.exponents[sidx]
        if var is None:
            t = cf
            for j in range(k):
                t *= x[pos[j]] ** int(ex[j])
            acc += t
        elif var in pos:
            j = list(pos).index(var)
            t = cf * int(ex[j]) * x[var] ** (int(ex[j]) - 1)
            for r in range(k):
                if r != j:
                    t *= x[pos[r]] ** int(ex[r])
            acc += t
    return acc


def to_dd_pair(z):
    out = []
    for v in (z.real, z.imag):
        hi = float(v)
        out += [hi, float(v - mp.mpf(hi))]
    return out


def sysd(s):
    return dict(n=s.n, m=s.m, k=s.k, d=s.d, pos=np.ascontiguousarray(s.positions, np.int32).reshape(-1),
                exps=np.ascontiguousarray(s.exponents, np.int32).reshape(-1), coeffs=np.ascontiguousarray(s.coeffs))


def ratios(ctx, s, pdd):
    got = ctx.evaluate_dd(pdd)
    want, ms = O.evaluate("dd", sysd(s), pdd, magsum=True, threads=8)
    e = dd_err(got, want)
    assert np.all(e[ms == 0] == 0)
    r = np.where(ms > 0, e / np.where(ms > 0, ms, 1.0), 0.0)
    return got, ms, r


@pytest.mark.parametrize("shape", [(32, 32, 8, 2), (32, 32, 16, 10)], ids=["C1", "k16_d10"])
def test_adversarial_search(shape, gpu):
    n, m, k, d = shape
    worst = []  # (ratio vs oracle, system seed, family, point array, output index)
    for seed in range(5):
        s = adversarial_system(n, m, k, d, 500 + seed)
        ctx = pj.EvaluationContext(s)
        for family in ("unit", "spread"):
            pdd = points(n, 96, 900 + seed, family)
            got, ms, r = ratios(ctx, s, pdd)
            b, o = np.unravel_index(np.argmax(r), r.shape)
            # hill climb on the worst point: rotate a few coordinates, keep the best ratio
            best_pt, best_r = pdd[b].copy(), r[b, o]
            rng = np.random.default_rng(seed)
            for _ in range(8):
                cand = np.repeat(best_pt[None], 48, 0)
                for c in range(48):
                    idx = rng.choice(n, 3, replace=False)
                    rot = np.exp(1j * rng.normal(0, 0.3, 3))
                    z = (cand[c, idx, 0] + 1j * cand[c, idx, 2]) * rot
                    cand[c, idx, 0], cand[c, idx, 2] = z.real, z.imag
                    cand[c, idx, 1] = cand[c, idx, 0] * U * 0.9999
                    cand[c, idx, 3] = -cand[c, idx, 2] * U * 0.9999
                _, _, rc = ratios(ctx, s, cand)
                if rc.max() > best_r:
                    bi = int(np.argmax(rc.max(axis=1)))
                    best_pt, best_r = cand[bi].copy(), rc.max()
            _, _, rb = ratios(ctx, s, best_pt[None])
            for oo in np.argsort(rb[0])[-3:]:
                worst.append((float(rb[0, oo]), s, best_pt, int(oo), ctx))
    worst.sort(key=lambda w: -w[0])
    assert worst[0][0] <= DD_TOL, f"fast order vs oracle: {worst[0][0]:.3e} x sum|terms|"
    # exact re-check of the worst candidates
    exact_worst = 0.0
    for ratio, s, pt, o, ctx in worst[:4]:
        got = ctx.evaluate_dd(pt[None])[0, o]
        ex = exact_output(s, pt, o)
        want = np.array(to_dd_pair(ex))
        _, ms = O.evaluate("dd", sysd(s), pt[None], magsum=True)
        err = float(dd_err(got[None], want[None])[0])
        exact_worst = max(exact_worst, err / ms[0, o])
    print(f"adversarial {shape}: worst vs oracle {worst[0][0]:.3e}, vs exact {exact_worst:.3e} (x sum|terms|)")
    assert exact_worst <= DD_TOL
