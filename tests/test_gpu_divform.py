"""The fast dd kernel's two derivative forms: a point whose coordinates all have
|Re| + |Im| in [2^-16, 2^16] takes the division form (derivative j = a_j * (c*V) * (1/x_j)), any other
point the product chains. Both are held to the same contract against the oracle, and the choice is
per point: a point's outputs do not depend on the other points of its batch or tile."""
import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import DD_TOL, dd_rel, sysd_of
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def mixed_points(n, B, seed):
    """Unit-modulus points, with every fourth point carrying one coordinate that forces the chain
    form (0, moduli 2^-20 / 2^20) or sits at the edge of the division form's range."""
    rng = np.random.default_rng(seed)
    th = rng.uniform(0, 2 * np.pi, (B, n))
    z = np.exp(1j * th)
    specials = [0.0, 2.0 ** -20, 2.0 ** 20, 2.0 ** -16, 2.0 ** 16 * 0.999, 2.0 ** -15.9, 2.0 ** 15.9]
    for b in range(0, B, 4):
        z[b, rng.integers(n)] = specials[(b // 4) % len(specials)] * np.exp(1j * rng.uniform(0, 2 * np.pi))
    return pj.to_dd(z)


@pytest.mark.parametrize("shape", [(32, 32, 8, 2), (32, 32, 16, 10), (24, 40, 5, 3), (16, 9, 1, 4)],
                         ids=["C1", "k16_d10", "k5_d3_m40", "k1"])
def test_forms_within_contract_and_per_point(shape, gpu):
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 31)
    ctx = pj.EvaluationContext(s)
    p = mixed_points(n, 56, 77)
    got = ctx.evaluate_dd(p)
    want, ms = O.evaluate("dd", sysd_of(s), p, magsum=True, threads=8)
    assert dd_rel(got, want, ms) <= DD_TOL
    # per-point choice: each point alone, and the batch reversed, give the same words
    for b in (0, 1, 4, 8, 21, 55):
        alone = ctx.evaluate_dd(p[b:b + 1])
        assert np.array_equal(alone[0], got[b]), f"point {b} depends on its batch"
    rev = ctx.evaluate_dd(p[::-1].copy())
    assert np.array_equal(rev[::-1], got)


def test_division_form_wide_moduli(gpu):
    # moduli over 2^-12 .. 2^12 (inside the division form's range) at k = 8, d = 2: total degree
    # <= 16, so every product stays far from the exponent limits
    n, m, k, d = 32, 32, 8, 2
    s = pj.random_system(n, m, k, d, 5)
    ctx = pj.EvaluationContext(s)
    rng = np.random.default_rng(3)
    z = 2.0 ** rng.uniform(-12, 12, (64, n)) * np.exp(1j * rng.uniform(0, 2 * np.pi, (64, n)))
    p = pj.to_dd(z)
    got = ctx.evaluate_dd(p)
    want, ms = O.evaluate("dd", sysd_of(s), p, magsum=True, threads=8)
    assert dd_rel(got, want, ms) <= DD_TOL


def test_zero_coordinates_exact_structure(gpu):
    # a zero coordinate (chain form) keeps exact zeros where the mathematics has them: the value
    # and every derivative of terms containing x_v^a with a >= 2 vanish; terms with a = 1 keep
    # their derivative in v
    n, m, k, d = 16, 12, 4, 3
    s = pj.random_system(n, m, k, d, 9)
    ctx = pj.EvaluationContext(s)
    z = np.exp(1j * np.random.default_rng(1).uniform(0, 2 * np.pi, (3, n)))
    z[:, 5] = 0.0
    p = pj.to_dd(z)
    got = ctx.evaluate_dd(p)
    want, ms = O.evaluate("dd", sysd_of(s), p, magsum=True, threads=8)
    assert dd_rel(got, want, ms) <= DD_TOL
