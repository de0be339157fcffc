"""Generate the committed wide-encoding fixture (run HERE):

    python tests/golden/gen_wide_golden.py

The reference rejects n > 256 (build_layout, ref src/packing.cpp:25-27), so there is no
reference output to pin; the system comes from the reference's generator (random_system has
no cap) and the truth from mpmath at 320 bits (gen_golden.truth): truth_dd and magsum, as for
the byte-encoding fixtures.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from oracle import oracle as O  # noqa: E402
from gen_golden import dd_points, truth  # noqa: E402

CASES = [("wide_n300", 300, 2, 3, 3, 301, 2, 303), ("wide_n520_k1", 520, 1, 1, 4, 521, 2, 523)]


def main():
    for name, n, m, k, d, ss, B, ps in CASES:
        S = O.ref_random_system(n, m, k, d, ss)
        pts = dd_points(n, B, ps)
        tr = np.zeros((B, n + n * n, 4))
        ms = np.zeros((B, n + n * n))
        for b in range(B):
            tr[b], ms[b] = truth(S, pts[b])
        np.savez_compressed(os.path.join(HERE, "wide", name + ".npz"), n=n, m=m, k=k, d=d, sys_seed=ss, pt_seed=ps,
                            pos=S["pos"], exps=S["exps"], coeffs=S["coeffs"], points_dd=pts, truth_dd=tr, magsum=ms)
        print("wrote", name, flush=True)


if __name__ == "__main__":
    main()
