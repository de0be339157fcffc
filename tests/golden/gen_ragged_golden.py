"""Generate the committed ragged-system fixtures (non-uniform m and k; run HERE):

    python tests/golden/gen_ragged_golden.py

The reference's data model is uniform (ref include/polyjac/system.hpp:14-42), so there is no
reference output for a ragged system. The shapes (m_p per polynomial, k_t per term) are drawn
with numpy's PCG64 from the case seed; each term's support, exponents and coefficient with the
reference's own generator stream (oracle/_ref random_system of one term per draw would not
give ragged shapes, so the draws are made here: uniform k_t-subset, exponents in [1, d],
coefficients in [-1, 1)^2). Points are the dd-stress points of gen_golden.dd_points. Truth:
mpmath at 320 bits rounded to dd (truth_dd) and the stage-3 magnitude sums (magsum), exactly
as gen_golden.truth, with every term carrying its own k.
"""
import os
import sys

import numpy as np
import mpmath as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from gen_golden import dd_points, to_dd  # noqa: E402

mp.mp.prec = 320

CASES = [
    # name, n, (m_lo, m_hi), (k_lo, k_hi), d, shape seed, npts, point seed
    ("ragged_small", 8, (1, 6), (1, 5), 4, 301, 3, 302),
    ("ragged_chunks", 24, (10, 45), (1, 12), 3, 303, 2, 304),
    ("ragged_k12", 6, (1, 4), (1, 2), 3, 305, 4, 306),
    ("ragged_d1", 5, (1, 3), (1, 5), 1, 307, 3, 308),
    ("ragged_d2_k16", 20, (20, 40), (2, 16), 2, 309, 2, 310),
]


def make_system(n, mr, kr, d, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    ro, to, ps, es, cs = [0], [0], [], [], []
    for p in range(n):
        m = int(g.integers(mr[0], mr[1] + 1))
        for _ in range(m):
            k = int(g.integers(kr[0], kr[1] + 1))
            ps.extend(sorted(int(v) for v in g.choice(n, size=k, replace=False)))
            es.extend(int(v) for v in g.integers(1, d + 1, size=k))
            to.append(to[-1] + k)
            while True:
                re, im = (float(v) for v in g.uniform(-1.0, 1.0, size=2))
                if re != 0.0 or im != 0.0:
                    break
            cs.append((re, 0.0, im, 0.0))
        ro.append(ro[-1] + m)
    return dict(n=n, d=d, row_off=np.array(ro, np.int32), term_off=np.array(to, np.int32),
                pos=np.array(ps, np.int32), exps=np.array(es, np.int32), coeffs=np.array(cs, np.float64))


def truth(S, pt):
    n = S["n"]
    x = [mp.mpc(mp.mpf(pt[i, 0]) + mp.mpf(pt[i, 1]), mp.mpf(pt[i, 2]) + mp.mpf(pt[i, 3])) for i in range(n)]
    vals = [mp.mpc(0)] * n
    jac = [[mp.mpc(0)] * n for _ in range(n)]
    mvals = [0.0] * n
    mjac = [[0.0] * n for _ in range(n)]
    ro, to = S["row_off"], S["term_off"]
    for p in range(n):
        for t in range(ro[p], ro[p + 1]):
            c = S["coeffs"][t]
            cf = mp.mpc(mp.mpf(c[0]) + mp.mpf(c[1]), mp.mpf(c[2]) + mp.mpf(c[3]))
            pos = S["pos"][to[t]:to[t + 1]]
            ex = S["exps"][to[t]:to[t + 1]]
            k = len(pos)
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
    out = np.zeros((n + n * n, 4))
    ms = np.zeros(n + n * n)
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
    for name, n, mr, kr, d, ss, B, ps in CASES:
        S = make_system(n, mr, kr, d, ss)
        pts = dd_points(n, B, ps)
        tr = np.zeros((B, n + n * n, 4))
        ms = np.zeros((B, n + n * n))
        for b in range(B):
            tr[b], ms[b] = truth(S, pts[b])
        np.savez_compressed(os.path.join(HERE, "ragged", name + ".npz"), points_dd=pts, truth_dd=tr, magsum=ms, **S)
        print("wrote", name, int(S["row_off"][-1]), "terms", flush=True)


if __name__ == "__main__":
    main()
