"""Developer A/B timing of library builds on one GPU: alternates the given .so files (loaded
through PJ_LIB_PATH in fresh subprocesses) and prints C2 / C3 fast dd and C2 complex-double
evals/s per run.

    python tools/ab.py NAME=path/lib.so NAME2=path2/lib.so [--rounds 3]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_1201_0499_b200 as pj
res = {}
for name, (n, m, k, d, B, reps) in {"c2": (32, 32, 8, 2, 65536, 20), "c3": (64, 64, 16, 10, 8192, 10),
                                     "c2d": (32, 32, 8, 2, 65536, 20)}.items():
    prec = "d" if name.endswith("d") else "dd"
    conv = (lambda x: __import__("numpy").stack([x.real, x.imag], -1).copy()) if prec == "d" else pj.to_dd
    s = pj.random_system(n, m, k, d, 7)
    ctx = pj.EvaluationContext(s)
    pts = [torch.from_numpy(conv(pj.random_points(n, B, 11 + i))).cuda() for i in range(2)]
    out = torch.empty((B, n + n * n, 4 if prec == "dd" else 2), dtype=torch.float64, device="cuda")
    for i in range(3):
        ctx.evaluate_device(pts[i % 2], out, prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    e0.record(st)
    for i in range(reps):
        ctx.evaluate_device(pts[i % 2], out, prec)
    e1.record(st)
    torch.cuda.synchronize()
    res[name] = B * reps / (e0.elapsed_time(e1) * 1e-3)
print(json.dumps(res))
"""


def main():
    rounds = 3
    libs = []
    args = sys.argv[1:]
    if "--rounds" in args:
        i = args.index("--rounds")
        rounds = int(args[i + 1])
        del args[i:i + 2]
    for a in args:
        name, path = a.split("=", 1)
        env = {}
        if ":" in path:  # NAME=lib.so:VAR=1,VAR2=x  extra environment for that arm
            path, extra = path.split(":", 1)
            env = dict(kv.split("=", 1) for kv in extra.split(","))
        libs.append((name, os.path.abspath(path), env))
    agg = {}
    for r in range(rounds):
        for name, path, extra in libs:
            env = dict(os.environ, PJ_LIB_PATH=path, **extra)
            out = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True)
            if out.returncode != 0:
                print(name, "FAILED", out.stderr[-800:], flush=True)
                continue
            res = json.loads(out.stdout.strip().splitlines()[-1])
            agg.setdefault(name, []).append(res)
            print(name, r, " ".join(f"{k}={v / 1e6:.3f}M" for k, v in res.items()), flush=True)
    for name, rs in agg.items():
        print("best", name, " ".join(f"{k}={max(x[k] for x in rs) / 1e6:.3f}M" for k in rs[0]))


if __name__ == "__main__":
    main()
