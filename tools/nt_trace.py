"""Developer: per-step clock trace of the Newton kernel (library built with -DPJB_NT_TRACE), block
0's first point, under full load (C2, 65,536 points) and alone (1 point)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1201_0499_b200 as pj

n = 32
s = pj.random_system(n, n, 8, 2, 7)
ctx = pj.EvaluationContext(s)
for B in [65536, 1]:
    x = torch.from_numpy(pj.to_dd(pj.random_points(n, B, 11))).cuda()
    work = torch.empty((B, n + n * n, 4), dtype=torch.float64, device="cuda")
    ctx.evaluate_device(x, work, "dd")
    out = torch.empty_like(x)
    off = (B + 1) & ~1
    tr = torch.zeros(off + 16 * n, dtype=torch.int32, device="cuda")  # statuses, then 8-byte trace entries
    import ctypes
    from paper_1201_0499_b200 import _lib
    nr = torch.empty((B, 2), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().pj_newton_solve(ctx._h, _lib.PJ_PREC_DD, work.data_ptr(), x.data_ptr(), None, B,
                                          out.data_ptr(), nr.data_ptr(), tr.data_ptr(), None))
    torch.cuda.synchronize()
    tt = tr[off:].cpu().numpy().view(np.int64)
    t = tt[: 4 * n].reshape(n, 4)
    sub = tt[4 * n: 8 * n].reshape(n, 4)
    d = np.diff(sub[1:n - 1], axis=1)  # columns 1..n-2: update -> argmax, argmax -> inverse, -> end
    print(f"B={B}: look-ahead sub-phases (cycles, mean over columns): column update+argmax {d[:, 0].mean():.0f}, "
          f"inverse broadcast {d[:, 1].mean():.0f}, multipliers+list {d[:, 2].mean():.0f}; "
          f"step start -> look-ahead entry {np.mean(sub[1:n - 1, 0] - t[0:n - 2, 0]):.0f}")
    t0 = t[0, 0]
    la = t[:, 2] - t[:, 0]
    upd = t[:, 3] - t[:, 1]
    step = np.diff(t[:, 3])
    print(f"B={B}: total {t[-1, 3] - t0} cycles; per step: look-ahead mean {la.mean():.0f} (first {la[:4]}, last {la[-4:]}), "
          f"step (barrier to barrier) mean {step.mean():.0f} first {step[:4]} last {step[-4:]}")
