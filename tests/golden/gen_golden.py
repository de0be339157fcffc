"""Generate the committed golden fixtures (run HERE, where /root/reference exists):

    python tests/golden/gen_golden.py

For each case: the system (reference generator), dd-stress points (hi from the reference's
random_points, lo = hi * 2^-54 * u with u from the same generator, seed + 1), and
  truth_dd  the exact values/Jacobian computed with mpmath at 320 bits, rounded to dd
  magsum    sum over the stage-3 terms of |term| (the tolerance scale)
  ref_d     the UNMODIFIED reference (oracle/_ref: EvaluationContext::evaluate, complex
            double) on the hi parts — the bit pattern every complex-double path must match.
mpmath is the precision-independent truth; the reference is the structural truth.
"""
import os
import sys

import numpy as np
import mpmath as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

mp.mp.prec = 320

CASES = [
    # name, n, m, k, d, sys_seed, npts, pt_seed
    ("small_k3_d4", 8, 5, 3, 4, 101, 4, 201),
    ("c1_n32_k8_d2", 32, 32, 8, 2, 7, 2, 11),
    ("k16_d10", 20, 10, 16, 10, 55, 2, 57),
    ("k1_d3", 6, 4, 1, 3, 61, 4, 62),
    ("k2_d3", 6, 4, 2, 3, 63, 4, 64),
    ("m40_chunks", 10, 40, 4, 3, 65, 2, 66),
    ("d1", 5, 3, 3, 1, 67, 3, 68),
]


def dd_points(n, B, seed):
    hi = O.ref_random_points(n, B, seed)
    u = O.ref_random_points(n, B, seed + 1)
    p = np.zeros((B, n, 4))
    p[..., 0] = hi[..., 0]
    p[..., 2] = hi[..., 1]
    p[..., 1] = hi[..., 0] * 2.0 ** -54 * u[..., 0]
    p[..., 3] = hi[..., 1] * 2.0 ** -54 * u[..., 1]
    return p


def to_dd(x):
    hi = float(x)
    lo = float(x - mp.mpf(hi))
    return hi, lo


def truth(S, pt):
    n, m, k = S["n"], S["m"], S["k"]
    x = [mp.mpc(mp.mpf(pt[i, 0]) + mp.mpf(pt[i, 1]), mp.mpf(pt[i, 2]) + mp.mpf(pt[i, 3])) for i in range(n)]
    vals = [mp.mpc(0)] * n
    jac = [[mp.mpc(0)] * n for _ in range(n)]
    mvals = [0.0] * n
    mjac = [[0.0] * n for _ in range(n)]
    for s in range(n * m):
        p = s // m
        c = S["coeffs"][s]
        cf = mp.mpc(mp.mpf(c[0]) + mp.mpf(c[1]), mp.mpf(c[2]) + mp.mpf(c[3]))
        pos = S["pos"][s * k:(s + 1) * k]
        ex = S["exps"][s * k:(s + 1) * k]
        pw = [x[pos[j]] ** int(ex[j]) for j in range(k)]
        prod = mp.mpc(1)
        for j in range(k):
            prod *= pw[j]
        val = cf * prod
        vals[p] += val
        mvals[p] += float(abs(val))
        for j in range(k):
            rest = mp.mpc(1)
            for r in range(k):
                if r != j:
                    rest *= pw[r]
            dv = cf * int(ex[j]) * (x[pos[j]] ** (int(ex[j]) - 1)) * rest
            jac[p][pos[j]] += dv
            mjac[p][pos[j]] += float(abs(dv))
    nout = n + n * n
    out = np.zeros((nout, 4))
    ms = np.zeros(nout)
    for i in range(n):
        out[i, 0:2] = to_dd(vals[i].real)
        out[i, 2:4] = to_dd(vals[i].imag)
        ms[i] = mvals[i]
    for p in range(n):
        for i in range(n):
            o = n + p * n + i
            out[o, 0:2] = to_dd(jac[p][i].real)
            out[o, 2:4] = to_dd(jac[p][i].imag)
            ms[o] = mjac[p][i]
    return out, ms


def main():
    for name, n, m, k, d, ss, B, ps in CASES:
        S = O.ref_random_system(n, m, k, d, ss)
        pts = dd_points(n, B, ps)
        tr = np.zeros((B, n + n * n, 4))
        ms = np.zeros((B, n + n * n))
        for b in range(B):
            tr[b], ms[b] = truth(S, pts[b])
        p2 = np.ascontiguousarray(pts[..., [0, 2]])
        ref_d = O.ref_evaluate(S, p2)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), n=n, m=m, k=k, d=d, sys_seed=ss, pt_seed=ps,
                            pos=S["pos"], exps=S["exps"], coeffs=S["coeffs"], points_dd=pts, truth_dd=tr,
                            magsum=ms, points_d=p2, ref_d=ref_d)
        print("wrote", name, flush=True)


if __name__ == "__main__":
    main()
