"""Developer timing of the Newton corrector (eval + solve) on C1/C2 and C3 (not a test)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1201_0499_b200 as pj

for (n, m, k, d, B) in [(32, 32, 8, 2, 65536), (64, 64, 16, 10, 8192), (8, 3, 3, 5, 65536), (100, 7, 5, 4, 2048)]:
    s = pj.random_system(n, m, k, d, 7)
    ctx = pj.EvaluationContext(s)
    for prec in ["dd", "d"]:
        W = 4 if prec == "dd" else 2
        pts = pj.random_points(n, B, 11)
        p = pj.to_dd(pts) if prec == "dd" else np.stack([pts.real, pts.imag], -1)
        x = torch.from_numpy(p).cuda()
        work = torch.empty((B, n + n * n, W), dtype=torch.float64, device="cuda")
        out = torch.empty_like(x)
        st = torch.empty(B, dtype=torch.int32, device="cuda")
        nr = torch.empty((B, 2), dtype=torch.float64, device="cuda")
        for thr in [0, 64, 128, 256]:
          ctx.set_launch(prec, thr, newton=True)
          for _ in range(2):
            ctx.evaluate_device(x, work, prec)
            ctx.newton_solve_device(work, x, out, prec, norms=nr, status=st)
          torch.cuda.synchronize()
          e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
          R = 5
          te = ts = 0.0
          for _ in range(R):
            e0.record()
            ctx.evaluate_device(x, work, prec)
            e1.record()
            ctx.newton_solve_device(work, x, out, prec, norms=nr, status=st)
            e2.record()
            torch.cuda.synchronize()
            te += e0.elapsed_time(e1)
            ts += e1.elapsed_time(e2)
          te /= R
          ts /= R
          # LU model: per point sum_kk (n-kk-1) cmul + (n-kk-1)(n-kk) (cmul+cadd) + n inv + n(n-1)/2 (cmul+cadd) + n cmul + n cadd
          cm = sum((n - kk - 1) + (n - kk - 1) * (n - kk) for kk in range(n)) + n * (n - 1) // 2 + n + n
          ca = sum((n - kk - 1) * (n - kk) for kk in range(n)) + n * (n - 1) // 2 + n + n
          fl = (cm * 80 + ca * 40) if prec == "dd" else (cm * 6 + ca * 2)
          stc = st.cpu().numpy()
          print(f"n={n} {prec} B={B}: eval {te:.3f} ms ({B/te/1e3:.3f} M/s)  solve {ts:.3f} ms ({B/ts/1e3:.3f} M/s, "
              f"{fl*B/ts/1e9:.2f} TFLOP/s model)  status ok {np.mean(stc==0):.3f} "
              f"solve {ctx.launch(prec, newton=True)}", flush=True)
