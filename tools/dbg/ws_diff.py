import sys, numpy as np
sys.path.insert(0, '.')
import paper_1201_0499_b200 as pj
from oracle import oracle as O
sys.path.insert(0, 'tests')
from conftest import dd_rel, sysd_of
for shape, B in [((64, 32, 12, 2), 300), ((64, 32, 8, 2), 40), ((40, 32, 12, 2), 40), ((64, 20, 5, 2), 40)]:
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 31 + k)
    z = pj.random_points(n, B, 32)
    pdd = pj.to_dd(z)
    want, ms = O.evaluate("dd", sysd_of(s), pdd, magsum=True, threads=8)
    res = {}
    for v in (1, 3):
        c = pj.EvaluationContext(s)
        c.set_variant(v, "dd")
        res[v] = c.evaluate_dd(pdd)
        print(shape, "variant", v, c.launch("dd"), "err", dd_rel(res[v], want, ms), flush=True)
    diff = np.nonzero(np.any(res[1].view(np.uint64) != res[3].view(np.uint64), axis=2))
    print("  differing (point, output):", len(diff[0]), list(zip(diff[0][:10], diff[1][:10])))
