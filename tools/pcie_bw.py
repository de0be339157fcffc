"""Developer: host<->device copy bandwidth on this box (pinned buffers), the ceiling of the
end-to-end (e2e) bench number, which moves 2.2 GB of results per 65,536 points."""
import time

import torch

for mb in [32, 256, 1024]:
    n = mb * (1 << 20) // 8
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    for direction in ["d2h", "h2d"]:
        for _ in range(2):
            (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
        torch.cuda.synchronize()
        reps = max(2, 4096 // mb)
        t0 = time.perf_counter()
        for _ in range(reps):
            (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{direction} {mb:5d} MiB: {reps * mb * (1 << 20) / dt / 1e9:6.1f} GB/s", flush=True)
