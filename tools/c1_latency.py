"""Developer: where the single-point (C1) latency goes — the Python API, the C host API and the
device kernel alone, complex double and dd."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1201_0499_b200 as pj
from paper_1201_0499_b200 import _lib

s = pj.random_system(32, 32, 8, 2, 7)
ctx = pj.EvaluationContext(s)
pt = pj.random_points(32, 1, 11)
p2 = np.stack([pt.real, pt.imag], -1).copy()
p4 = pj.to_dd(pt)
reps = 300


def tm(fn):
    for _ in range(30):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e6


print("launch d", ctx.launch("d"), "dd", ctx.launch("dd"))
print(f"python evaluate (d):      {tm(lambda: ctx.evaluate(pt[0])):7.1f} us")
print(f"python evaluate_dd:       {tm(lambda: ctx.evaluate_dd(p4)):7.1f} us")
o2 = np.empty((1, 32 + 1024, 2))
o4 = np.empty((1, 32 + 1024, 4))
L = _lib.lib()
print(f"C pj_evaluate_host d:     {tm(lambda: L.pj_evaluate_host(ctx._h, _lib.PJ_PREC_D, p2.ctypes.data, 1, o2.ctypes.data)):7.1f} us")
print(f"C pj_evaluate_host dd:    {tm(lambda: L.pj_evaluate_host(ctx._h, _lib.PJ_PREC_DD, p4.ctypes.data, 1, o4.ctypes.data)):7.1f} us")
pin2 = torch.from_numpy(p2).pin_memory(); pin4 = torch.from_numpy(p4).pin_memory()
po2 = torch.empty((1, 1056, 2), dtype=torch.float64).pin_memory(); po4 = torch.empty((1, 1056, 4), dtype=torch.float64).pin_memory()
print(f"C host dd, pinned bufs:   {tm(lambda: L.pj_evaluate_host(ctx._h, _lib.PJ_PREC_DD, pin4.data_ptr(), 1, po4.data_ptr())):7.1f} us")
x4 = torch.from_numpy(p4).cuda(); out4 = torch.empty((1, 1056, 4), dtype=torch.float64, device="cuda")
x2 = torch.from_numpy(p2).cuda(); out2 = torch.empty((1, 1056, 2), dtype=torch.float64, device="cuda")
for prec, x, o in [("d", x2, out2), ("dd", x4, out4)]:
    for _ in range(20):
        ctx.evaluate_device(x, o, prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        ctx.evaluate_device(x, o, prec)
    e1.record()
    torch.cuda.synchronize()
    print(f"device kernel {prec:2s} (B=1):  {e0.elapsed_time(e1) * 10:7.1f} us per launch (back to back)")
