"""Developer: C3 evaluations (n = 64, k = 16, d = 10, complex dd, fast order) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1201_0499_b200 as pj

B = int(os.environ.get("PJ_B", "16384"))
s = pj.random_system(64, 64, 16, 10, 7)
ctx = pj.EvaluationContext(s)
x = torch.from_numpy(pj.to_dd(pj.random_points(64, B, 11))).cuda()
out = torch.empty((B, 64 + 64 * 64, 4), dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.evaluate_device(x, out, "dd")
torch.cuda.synchronize()
print("launch", ctx.launch("dd"))
