"""Generate the committed Newton-corrector fixtures (run HERE, where /root/reference exists):

    python tests/golden/gen_newton_golden.py

The reference has no Newton step, so the solver (csrc/newton.cu, restated by
oracle/oracle.cpp: newton_one) is pinned to exact arithmetic. For each case: the system
(reference generator), dd-stress points, the exact values/Jacobian rounded to dd (the
evaluator's output as the solver consumes it, mpmath at 320 bits, gen_golden.truth), and
  dx_dd     the exact solution of J dx = -f for THOSE rounded inputs, mpmath LU at 320 bits,
            rounded to dd
  dx_d      the same for the complex-double inputs (the hi words of f and J)
  cond      the infinity-norm condition number of J (scales the forward-error bound)
"""
import os
import sys

import numpy as np
import mpmath as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from oracle import oracle as O  # noqa: E402
from gen_golden import dd_points, to_dd, truth  # noqa: E402

mp.mp.prec = 320

CASES = [
    # name, n, m, k, d, sys_seed, npts, pt_seed
    ("newton_c1_n32", 32, 32, 8, 2, 7, 3, 11),
    ("newton_small_n8", 8, 5, 3, 4, 101, 4, 201),
    ("newton_k16_n20", 20, 10, 16, 10, 55, 2, 57),
]


def mpc_of(v):
    return mp.mpc(mp.mpf(v[0]) + mp.mpf(v[1]), mp.mpf(v[2]) + mp.mpf(v[3]))


def solve(ev, n):
    f = mp.matrix([[-mpc_of(ev[i])] for i in range(n)])
    J = mp.matrix(n, n)
    for p in range(n):
        for i in range(n):
            J[p, i] = mpc_of(ev[n + p * n + i])
    dx = mp.lu_solve(J, f)
    Jt = J.T  # infinity norm = 1-norm of the transpose
    cond = float(mp.mnorm(Jt, 1) * mp.mnorm(Jt ** -1, 1))
    out = np.zeros((n, 4))
    for i in range(n):
        out[i, 0:2] = to_dd(dx[i].real)
        out[i, 2:4] = to_dd(dx[i].imag)
    return out, cond


def main():
    for name, n, m, k, d, ss, B, ps in CASES:
        S = O.ref_random_system(n, m, k, d, ss)
        pts = dd_points(n, B, ps)
        ev = np.zeros((B, n + n * n, 4))
        dx_dd = np.zeros((B, n, 4))
        dx_d = np.zeros((B, n, 4))
        cond = np.zeros(B)
        for b in range(B):
            ev[b], _ = truth(S, pts[b])
            dx_dd[b], cond[b] = solve(ev[b], n)
            evd = ev[b].copy()
            evd[:, 1] = 0.0
            evd[:, 3] = 0.0
            dx_d[b], _ = solve(evd, n)
        np.savez_compressed(os.path.join(HERE, "newton", name + ".npz"), n=n, m=m, k=k, d=d, pos=S["pos"],
                            exps=S["exps"], coeffs=S["coeffs"], points_dd=pts, evals_dd=ev, dx_dd=dx_dd, dx_d=dx_d,
                            cond=cond)
        print("wrote", name, "cond", cond, flush=True)


if __name__ == "__main__":
    main()
