"""Developer: per-point phase cycles of the Newton solve under full load (library built with
-DPJB_NT_PHASES): load, elimination, back substitution, averaged over every CTA's points."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1201_0499_b200 as pj
from paper_1201_0499_b200 import _lib

n = int(os.environ.get("PJ_N", "32"))
for prec in (os.environ.get("PJ_PRECS", "dd,d")).split(","):
    mixed = prec == "mixed"
    W = 4 if prec in ("dd", "mixed") else 2
    s = pj.random_system(n, n, 8 if n == 32 else 16, 2 if n == 32 else 10, 7)
    ctx = pj.EvaluationContext(s)
    B = int(os.environ.get("PJ_B", "65536"))
    pts = pj.random_points(n, B, 11)
    p = pj.to_dd(pts) if W == 4 else np.stack([pts.real, pts.imag], -1)
    x = torch.from_numpy(p).cuda()
    work = torch.empty((B, n + n * n, W), dtype=torch.float64, device="cuda")
    ctx.evaluate_device(x, work, "dd" if mixed else prec)
    out = torch.empty_like(x)
    off = (B + 1) & ~1
    st = torch.zeros(off + 16 * 4096, dtype=torch.int32, device="cuda")
    nr = torch.empty((B, 2), dtype=torch.float64, device="cuda")
    pr = _lib.PJ_PREC_DD if W == 4 else _lib.PJ_PREC_D
    if mixed:
        pr |= _lib.PJ_NEWTON_MIXED
    for _ in range(2):
        _lib.check(_lib.lib().pj_newton_solve(ctx._h, pr, work.data_ptr(), x.data_ptr(), None, B,
                                              out.data_ptr(), nr.data_ptr(), st.data_ptr(), None))
    torch.cuda.synchronize()
    launch = ctx.launch(prec, newton=True)
    G = launch["blocks"]
    ph = st[off:off + 16 * G].cpu().numpy().view(np.int64).reshape(G, 8)
    cnt = ph[:, 3].sum()
    tot = ph[:, :3].sum(0) / cnt
    sub = ph[:, 4:].sum(0) / cnt
    print(f"n={n} {prec} B={B} {launch}: cycles per point per CTA: load {tot[0]:.0f}, elimination {tot[1]:.0f}, "
          f"back substitution {tot[2]:.0f}, total {tot.sum():.0f}; points per CTA {ph[:, 3].min()}..{ph[:, 3].max()}"
          + (f"; slots 4-7 {sub.round().tolist()}" if os.environ.get("PJ_ALLSLOTS") else "")
          + (f"; refinement: initial solve {sub[0]:.0f}, residuals {sub[1]:.0f}, solves {sub[2]:.0f}, "
             f"update {sub[3]:.0f}" if mixed else ""),
          flush=True)
