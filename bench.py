#!/usr/bin/env python3
"""Benchmark of the hot path: complex double-double system + Jacobian evaluation.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)

Workload (BASELINE.json configs): random_system(32, 32, 8, 2, seed 7) (n=32 variables, 32
polynomials x 32 monomials of k=8 variables, degrees <= 2); points from random_points(32, ., seed
11) — rank r evaluates the contiguous shard r of ONE global point stream, so the union over ranks
is the single-process batch. A step = one evaluation of the rank's shard (values + full Jacobian,
complex dd), no collective on the data path.
  * N = 1: C2, 65,536 points per step (configs[1], the config the metric is quoted on).
  * N > 1: C5, 1,048,576 points per step sharded over the N GPUs (configs[4], strong scaling), plus
    a separately timed end-of-run gather of every rank's results into rank 0 (point to point).

Order of a run: (1) the parity gate — BEFORE any timing, binding: the GPU results on >= 1,024
points of the rank's batch (its first and last points included) against the oracle's complex-dd
restatement (|err| <= 1e-30 * sum|terms| per entry, structural zeros exact +0), and the complex
double path (C4) on 64 points bit for bit against the unmodified reference (oracle/_ref); any
violation exits with status 3 and no JSON line. (2) The timed region (device, CUDA events on the
launching stream, barrier + synchronize both sides, max over ranks). (3) The gather (N > 1).
(4) e2e through the public host API. (5) The roofline: model FP64 flops over the
live-measured FP64 pipe rate, and the hardware view — executed FP64 instructions and DRAM bytes of
one extra untimed launch counted by ncu in this run (never a timing from the profiler).
(6) Secondary lines: C4 quality-up, C3 (65,536 points), f1 Newton, C1 single-point latency.
(7) cpu_baseline: the unmodified reference on this host's cores (rank 0, N = 1).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "system+Jacobian evals/sec (complex dd, n=32) and % of FP64 peak, 1/2/4/8 GPUs"
N, M, K, D, SYS_SEED, PT_SEED = 32, 32, 8, 2, 7, 11
POINTS_PER_GPU = 65536          # C2
C5_GLOBAL_POINTS = 1 << 20      # C5
GATE_TOL = 1e-30
REF_C1_US = 202.5               # reference, 1 thread, n=32 k=8 d=2, per evaluation


# dd_mul = 10 flops, dd_add = 20, complex dd mul = 80, complex dd add = 40;
# per eval cmul = n*max(d-2,0) + nm(k-1) + nm(5k-4), cadd = nm(k+1) (useful terms)
def model_flops(n, m, k, d, prec="dd"):
    cmul = n * max(d - 2, 0) + n * m * (k - 1) + n * m * (5 * k - 4)
    cadd = n * m * (k + 1)
    return cmul * 80 + cadd * 40 if prec == "dd" else cmul * 6 + cadd * 2


def newton_model_flops(n, prec="dd"):
    """Cost model of one Newton solve (csrc/newton.cu), same weights as model_flops: per step kk the
    R = n-kk-1 multipliers (cmul) and R*(n-kk) trailing updates (cmul + cadd, rhs column included);
    n pivot inverses (counted as one cmul each); back substitution n cmul + n(n-1)/2 (cmul + cadd);
    the final x + dx (n cadd)."""
    R = [n - kk - 1 for kk in range(n)]
    upd = sum(r * (r + 1) for r in R)
    cmul = sum(R) + upd + n + n + n * (n - 1) // 2
    cadd = upd + n * (n - 1) // 2 + n
    return cmul * 80 + cadd * 40 if prec == "dd" else cmul * 6 + cadd * 2


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sysd_of(s):
    """product PolynomialSystem -> the oracle's dict (test-infrastructure format)."""
    return dict(n=s.n, m=s.m, k=s.k, d=s.d, pos=np.ascontiguousarray(s.positions, np.int32).reshape(-1).copy(),
                exps=np.ascontiguousarray(s.exponents, np.int32).reshape(-1).copy(),
                coeffs=np.ascontiguousarray(s.coeffs, np.float64).copy())


# ----------------------------------------------------------------------------- CPU leg (oracle)
def reference_cpu(sysd, n, target_seconds=8.0, threads=None, prec="ref"):
    """Time the unmodified reference (oracle/_ref, complex double — the reference has no dd) or
    the oracle's dd restatement (prec="dd-port") point-sharded across host threads (one
    workers=1 context per thread). Bounded sample sized from a calibration run."""
    from oracle import oracle as O
    threads = threads or cpu_count()

    def run(B):
        if prec == "ref":
            pts = O.ref_random_points(n, B, PT_SEED)
            t0 = time.perf_counter()
            O.ref_evaluate(sysd, pts, threads=threads)
            return time.perf_counter() - t0
        p4 = np.zeros((B, n, 4))
        pts2 = O.ref_random_points(n, B, PT_SEED)
        p4[..., 0], p4[..., 2] = pts2[..., 0], pts2[..., 1]
        t0 = time.perf_counter()
        O.evaluate("dd", sysd, p4, threads=threads)
        return time.perf_counter() - t0

    cal = 32 * threads
    dt = run(cal)
    B = int(min(max(cal, cal * target_seconds / max(dt, 1e-6)), 1 << 20))
    dt = run(B)
    return B / dt, B, dt, threads


def reference_c1_latency(sysd, reps=200):
    """The reference's own single-point call (EvaluationContext::evaluate, one workers=1 context,
    one thread): microseconds per evaluation at C1."""
    from oracle import oracle as O
    pt = O.ref_random_points(sysd["n"], 1, PT_SEED)
    _, _, secs = O.ref_evaluate(sysd, np.repeat(pt, reps, axis=0), threads=1, timing=True)
    return secs / reps * 1e6


def parity_gate(sysd, pts_dd, got_dd, pts_d, got_d):
    """The checker (oracle as test infrastructure, never the measured path): the GPU's complex-dd
    results vs the oracle's dd restatement, |got - want| <= 1e-30 * sum|terms| per entry with the
    structural zeros exact +0 in every word; and the GPU's complex-double results bit for bit vs
    the unmodified reference (oracle/_ref; the oracle's bit-exact double restatement if absent)."""
    from oracle import oracle as O
    want, ms = O.evaluate("dd", sysd, pts_dd, magsum=True, threads=cpu_count())
    err = np.maximum(np.abs((got_dd[..., 0] - want[..., 0]) + (got_dd[..., 1] - want[..., 1])),
                     np.abs((got_dd[..., 2] - want[..., 2]) + (got_dd[..., 3] - want[..., 3])))
    zero = ms == 0.0
    ratio = np.where(zero, 0.0, err / np.where(zero, 1.0, ms))
    zeros_exact = bool(np.all(got_dd[zero].view(np.uint64) == 0))
    worst = float(np.max(ratio)) if ratio.size else 0.0
    finite = bool(np.all(np.isfinite(got_dd)))
    if O.ref_available():
        want_d, d_ref = O.ref_evaluate(sysd, pts_d, threads=cpu_count()), "unmodified reference (oracle/_ref)"
    else:
        want_d, d_ref = O.evaluate("d", sysd, pts_d, threads=cpu_count()), "oracle double restatement"
    d_mismatch = int(np.count_nonzero(got_d.view(np.uint64) != want_d.view(np.uint64)))
    ok = finite and worst <= GATE_TOL and zeros_exact and d_mismatch == 0
    return {"pass": ok, "dd_points": int(pts_dd.shape[0]), "max_err_over_sum_abs_terms": worst, "tol": GATE_TOL,
            "structural_zeros_exact": zeros_exact, "structural_zero_entries": int(np.count_nonzero(zero)),
            "d_points": int(pts_d.shape[0]), "d_words_differing": d_mismatch, "d_against": d_ref,
            "when": "before the timed region"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpolyjac_ref.so not built "
                          "(needs /root/reference at build time)"}))
        return 0
    sysd = O.ref_random_system(N, M, K, D, SYS_SEED)
    threads = cpu_count()
    # calibrate once, then size every step so the whole run stays within ~2 minutes
    # (each step >= ~0.25 s of CPU work so thread start-up does not dominate)
    cal = 32 * threads
    pts = O.ref_random_points(N, cal, PT_SEED)
    t0 = time.perf_counter()
    O.ref_evaluate(sysd, pts, threads=threads)
    rate = cal / (time.perf_counter() - t0)
    step_s = max(0.25, min(args.ref_seconds, 120.0 / (args.warmup + args.steps)))
    B_used = int(max(cal, min(rate * step_s, 1 << 20)))
    pts = O.ref_random_points(N, B_used, PT_SEED)
    dts = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.ref_evaluate(sysd, pts, threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            dts.append(dt)
    value = B_used * len(dts) / sum(dts)
    dt_used = sum(dts) / len(dts)
    workload = ("C5: n=32 m=32 k=8 d=2, evaluation-point batch (bounded CPU sample)" if ws > 1 else
                "C2: n=32 m=32 k=8 d=2, evaluation-point batch (bounded CPU sample)")
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt_used * 1e3, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic: reference random_system(32,32,8,2,seed 7), random_points(32, ., seed 11)",
        "config": {"workload": workload, "points_per_step": B_used,
                   "parallelism": f"{threads} host threads, point-sharded"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "reference",
                         "sample": f"{B_used} points per step through the unmodified reference "
                                   "EvaluationContext::evaluate (complex double: the reference has no "
                                   f"double-double path), one workers=1 context per thread; {cpu_model()}"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- hardware counts
HW_METRICS = ["sm__inst_executed_pipe_fp64.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
              "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
              "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def count_child(args):
    """--count-child: one untimed launch of the headline kernel at the bench's shape, for ncu to
    count (instructions and DRAM bytes only; no timing is ever read from it)."""
    import torch
    import paper_1201_0499_b200 as pj
    dev = torch.device("cuda", 0)
    ctx = pj.EvaluationContext(pj.random_system(N, M, K, D, SYS_SEED), device=0)
    B = args.points
    pts = torch.from_numpy(pj.to_dd(pj.random_points(N, B, PT_SEED))).to(dev)
    out = torch.empty((B, N + N * N, 4), dtype=torch.float64, device=dev)
    ctx.evaluate_device(pts, out, "dd", args.order)
    torch.cuda.synchronize()
    return 0


def hw_counts(points, order, timeout=240):
    """Executed FP64 instructions and DRAM bytes of ONE launch of the headline kernel, counted by
    ncu on a child process of this run (same box, same build)."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    cmd = [ncu, "--metrics", ",".join(HW_METRICS), "--csv", "--print-units", "base", "-k", "regex:fast_kernel",
           "-c", "1", sys.executable, os.path.join(ROOT, "bench.py"), "--count-child", "--points", str(points),
           "--order", order]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": "ncu timed out"}
    vals = {}
    text = r.stdout[r.stdout.find('"ID"'):] if '"ID"' in r.stdout else ""
    for row in csv.DictReader(io.StringIO(text)):
        try:
            vals[row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            continue
    if not all(m in vals for m in HW_METRICS):
        return {"error": "ncu returned no counts (rc %d): %s" % (r.returncode, (r.stderr or r.stdout)[-300:])}
    return {
        "fp64_warp_inst_per_launch": vals["sm__inst_executed_pipe_fp64.sum"],
        "fp64_lane_ops_per_launch": {op: vals[f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum"]
                                     for op in ("dfma", "dadd", "dmul")},
        "dram_bytes_per_launch": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
        "points_per_launch": points,
        "how": "ncu --metrics (instruction and byte counts only) on one untimed launch in a child process",
    }


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--points", type=int, default=POINTS_PER_GPU, help="points per GPU per step (weak scaling)")
    ap.add_argument("--global-points", type=int, default=None,
                    help="fixed total points per step sharded over the ranks (strong scaling); default: "
                         f"{C5_GLOBAL_POINTS} (C5) when WORLD_SIZE > 1, else off (C2, --points per GPU)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--gate-points", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hw-counts", action="store_true", help="skip the ncu instruction/byte count of one launch")
    ap.add_argument("--order", default="fast", choices=["fast", "ref"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for the barrier, the max-over-ranks reduction and the gather")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary lines (C3, C4 quality-up factor, f1 Newton step, C1 latency)")
    ap.add_argument("--no-gather", action="store_true", help="N > 1: skip the end-of-run gather")
    ap.add_argument("--inject-fault", action="store_true",
                    help="testing: corrupt one device coefficient before the gate (the run must exit 3)")
    ap.add_argument("--count-child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.count_child:
        return count_child(args)
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1201_0499_b200 as pj
    from paper_1201_0499_b200.sharding import gather_to_rank0, shard_points, shard_range

    ws, rank, local = dist_env()
    dist = ws > 1
    # one rank per GPU; --dist-backend gloo lets several ranks share a device (multi-rank checks of
    # this harness on a one-GPU box: tests/test_bench_contract.py)
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if dist:
        import torch.distributed as tdist
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group("gloo")

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if dist:
            tdist.barrier()

    if args.global_points is None:
        args.global_points = C5_GLOBAL_POINTS if ws > 1 else 0
    sysobj = pj.random_system(N, M, K, D, SYS_SEED)
    sysd = sysd_of(sysobj)
    ctx = pj.EvaluationContext(sysobj, device=local)
    if args.global_points:
        total = args.global_points
        first, last = shard_range(total, ws, rank)
        B = last - first
        scaling = "strong"
    else:
        B = args.points
        total = B * ws
        first = B * rank
        scaling = "weak"
    nout = N + N * N
    host_pts = shard_points(N, total, PT_SEED, ws, rank)  # complex128 [B, n]: this rank's shard
    dd = pj.to_dd(host_pts)
    d2 = np.ascontiguousarray(np.stack([host_pts.real, host_pts.imag], -1))
    if args.inject_fault:
        pj._lib.check(pj._lib.lib().pj_debug_corrupt_coeff(ctx._h, 37, 1.001))

    # ---------------- (1) parity gate, before any timing: binding
    G = min(args.gate_points, B)
    gidx = np.unique(np.concatenate([np.arange(G // 2), np.arange(B - (G - G // 2), B)]))
    gate_dd_in = torch.from_numpy(np.ascontiguousarray(dd[gidx])).to(dev)
    gate_dd_out = torch.empty((len(gidx), nout, 4), dtype=torch.float64, device=dev)
    ctx.evaluate_device(gate_dd_in, gate_dd_out, "dd", args.order, validate=True)
    gd = min(64, B)
    gate_d_in = torch.from_numpy(np.ascontiguousarray(d2[:gd])).to(dev)
    gate_d_out = torch.empty((gd, nout, 2), dtype=torch.float64, device=dev)
    ctx.evaluate_device(gate_d_in, gate_d_out, "d")
    torch.cuda.synchronize(dev)
    gate = parity_gate(sysd, dd[gidx], gate_dd_out.cpu().numpy(), d2[:gd], gate_d_out.cpu().numpy())
    gate["points_checked"] = f"rank {rank}: points {first}..{first + G // 2 - 1} and " \
                             f"{first + B - (G - G // 2)}..{first + B - 1} of the global stream (dd); " \
                             f"{first}..{first + gd - 1} (complex double)"
    ok_all = max_over_ranks(0.0 if gate["pass"] else 1.0) == 0.0
    if not ok_all:
        sys.stderr.write("parity gate FAILED: " + json.dumps(gate) + "\n")
        return 3
    del gate_dd_in, gate_dd_out, gate_d_in, gate_d_out

    # inputs > L2: rotate over NBUF distinct device batches (NBUF * 67 MB > 126 MB L2 at C2)
    NBUF = 4 if B <= POINTS_PER_GPU * 2 else 2
    bufs = [torch.from_numpy(np.roll(dd, i, axis=0).copy()).to(dev) for i in range(NBUF)]
    out = torch.empty((B, nout, 4), dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            ctx.evaluate_device(bufs[i % NBUF], out, "dd", args.order, stream)
    stream.synchronize()
    if ctx.nonfinite_seen(stream):
        raise RuntimeError("non-finite input")

    # ---------------- (2) timed region (device): K steps, events on the launching stream
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with torch.cuda.stream(stream):
        evs[0].record(stream)
        for i in range(args.steps):
            ctx.evaluate_device(bufs[i % NBUF], out, "dd", args.order, stream)
            evs[i + 1].record(stream)
    stream.synchronize()
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = max_over_ranks(evs[0].elapsed_time(evs[-1]))
    value = total * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps
    kern_ms = statistics.mean(per)

    # ---------------- (3) end-of-run gather to rank 0 (N > 1), timed separately
    gather = None
    if dist and not args.no_gather:
        on_gpu = args.dist_backend == "nccl"
        src = out if on_gpu else out.cpu()
        recv = None
        if rank == 0:
            recv = torch.empty((total, nout, 4), dtype=torch.float64, device=dev if on_gpu else "cpu")
        barrier()
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        g0.record()
        full = gather_to_rank0(src, out=recv)
        g1.record()
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        gms = max_over_ranks(g0.elapsed_time(g1) if on_gpu else wall * 1e3)
        moved = (total - B) * nout * 32 if rank == 0 else 0
        gather = {"ms": gms, "bytes_into_rank0": int(max_over_ranks(float(moved))),
                  "GBps_into_rank0": max_over_ranks(float(moved)) / (gms * 1e-3) / 1e9 if gms > 0 else None,
                  "method": "point to point (batch_isend_irecv): each rank's shard sent once to rank 0",
                  "backend": args.dist_backend}
        if rank == 0:
            ok = full.shape[0] == total and torch.equal(full[:B], src)
            gather["rank0_rows"] = int(full.shape[0])
            gather["own_rows_intact"] = bool(ok)
        del full, recv, src

    # ---------------- (4) e2e through the public host API (pinned host buffers)
    Be = min(B, POINTS_PER_GPU)  # strong-scaling runs with huge shards time e2e on a C2-sized sample
    pin_in = torch.from_numpy(dd[:Be]).pin_memory()
    pin_out = torch.empty((Be, nout, 4), dtype=torch.float64).pin_memory()
    ni, no = pin_in.numpy(), pin_out.numpy()
    ctx.evaluate_host(ni, "dd", args.order, out=no)  # warm (allocates the staging buffers)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        ctx.evaluate_host(ni, "dd", args.order, out=no)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": Be * ws * args.e2e_steps / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": int(ni.nbytes),
           "d2h_bytes_per_step": int(no.nbytes), "steps": args.e2e_steps,
           "api": "EvaluationContext.evaluate_host -> pj_evaluate_host (3-stream chunked H2D/kernel/D2H)",
           "pcie_GBps": (ni.nbytes + no.nbytes) * args.e2e_steps / e2e_s / 1e9}
    del pin_in, pin_out

    # ---------------- (5) roofline: FP64 issue-bound
    rates = pj.fp64_pipe_rates(local)
    sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    lane_rate_clock = sms * 64 * sm_mhz * 1e6  # FP64 lanes per SM per clock x clock
    pipe_lane_rate = max(max(rates.values()), lane_rate_clock)
    peak = 2.0 * pipe_lane_rate / 1e12  # TFLOP/s counting an FMA as 2 flops at the pipe's full issue rate
    flops = model_flops(N, M, K, D)
    achieved = flops * B / (kern_ms * 1e-3) / 1e12
    io_bytes = B * (N * 32 + nout * 32)
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": None, "algorithmic_bytes": io_bytes,
                "hbm_gbs_achieved": io_bytes / (kern_ms * 1e-3) / 1e9, "flops_per_eval": flops,
                "peak_source": ("2 x the FP64 pipe's full issue rate on this device: max(probe DFMA/DADD/DMUL lane-op "
                                f"rates, {sms} SMs x 64 lanes x the sampled SM clock); MEASURED_PEAKS.json carries "
                                "no FP64 figure"),
                "probe_lane_ops_per_s": rates, "clock_lane_ops_per_s": lane_rate_clock,
                "note": "achieved = the fixed SURVEY.md 8(d) cost model (80 flops per complex dd product, 40 per "
                        "add) over device time (model fraction); hw_fp64_pipe_frac = executed FP64 work (counted "
                        "in this run) over the same pipe rate"}
    if rank == 0 and ws == 1 and not args.no_hw_counts and args.order == "fast":
        hw = hw_counts(min(B, POINTS_PER_GPU), args.order)
        if "error" not in hw:
            pts_hw = hw["points_per_launch"]
            warp_inst_per_eval = hw["fp64_warp_inst_per_launch"] / pts_hw
            lane_ops = hw["fp64_lane_ops_per_launch"]
            hw_flops_per_eval = (2 * lane_ops["dfma"] + lane_ops["dadd"] + lane_ops["dmul"]) / pts_hw
            evals_per_s = B / (kern_ms * 1e-3)
            roofline["traffic"] = hw["dram_bytes_per_launch"] * B / pts_hw
            roofline["hw_fp64_pipe_frac"] = warp_inst_per_eval * 32 * evals_per_s / pipe_lane_rate
            roofline["hw_fp64_tflops"] = hw_flops_per_eval * evals_per_s / 1e12
            roofline["hw_fp64_warp_inst_per_eval"] = warp_inst_per_eval
            roofline["hw_counts"] = hw
        else:
            roofline["hw_counts"] = hw

    workload = (f"C5: n=32 m=32 k=8 d=2, {total:,} evaluation points per step sharded over {ws} GPU(s)"
                if args.global_points else f"C2: n=32 m=32 k=8 d=2, {B:,} evaluation points per GPU per step")
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "complex-dd (f64 pairs)",
        "data": f"synthetic: random_system(32,32,8,2,seed 7), random_points(32, {total}, seed 11) sharded by rank",
        "config": {"workload": workload, "points_per_gpu": B, "global_points": total, "order": args.order,
                   "parallelism": f"points sharded over {ws} GPU(s), system replicated, no collective",
                   "l2": f"inputs rotate over {NBUF} device batches ({NBUF * dd.nbytes >> 20} MiB > 126 MiB L2); "
                         f"outputs {B * nout * 32 >> 20} MiB per step",
                   "launch": ctx.launch("dd")},
        "parity_gate": gate,
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "clocks": clk,
    }
    if gather is not None:
        line["gather"] = gather
    del bufs

    # ---------------- (6) secondary measurements (outside the headline timed region; N = 1 lines)
    if not args.no_extras and ws == 1:
        def timed(fn, reps):
            for _ in range(2):
                fn()
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(reps):
                    fn()
                e1.record(stream)
            stream.synchronize()
            return e0.elapsed_time(e1) / reps
        Bx = min(B, POINTS_PER_GPU)
        x_dd = torch.from_numpy(np.ascontiguousarray(dd[:Bx])).to(dev)
        out_x = out[:Bx]
        # C4: complex double vs complex double-double on the same points (quality-up overhead)
        xd = torch.from_numpy(np.ascontiguousarray(d2[:Bx])).to(dev)
        out_d = torch.empty((Bx, nout, 2), dtype=torch.float64, device=dev)
        ms_d = timed(lambda: ctx.evaluate_device(xd, out_d, "d", None, stream), 10)
        ms_dd = timed(lambda: ctx.evaluate_device(x_dd, out_x, "dd", args.order, stream), 10)
        line["quality_up"] = {"config": "C4: C2 in complex double (reference order, bit-exact with the reference) "
                                        "vs complex dd (fast order)",
                              "d_evals_per_s": Bx / (ms_d * 1e-3), "dd_evals_per_s": Bx / (ms_dd * 1e-3),
                              "dd_over_d_time": ms_dd / ms_d, "d_launch": ctx.launch("d")}
        del out_d, xd
        # C3: n=64 m=64 k=16 d=10 (higher degrees, larger common-factor stage), complex dd, full batch
        s3 = pj.random_system(64, 64, 16, 10, SYS_SEED)
        ctx3 = pj.EvaluationContext(s3, device=local)
        B3 = 65536
        p3 = torch.from_numpy(pj.to_dd(pj.random_points(64, B3, PT_SEED))).to(dev)
        o3 = torch.empty((B3, 64 + 64 * 64, 4), dtype=torch.float64, device=dev)
        ms3 = timed(lambda: ctx3.evaluate_device(p3, o3, "dd", args.order, stream), 3)
        f3 = model_flops(64, 64, 16, 10)
        line["c3"] = {"config": "C3: random_system(64,64,16,10,seed 7), 65,536 points, complex dd, fast order",
                      "evals_per_s": B3 / (ms3 * 1e-3), "ms_per_batch": ms3, "flops_per_eval": f3,
                      "roofline_frac": f3 * B3 / (ms3 * 1e-3) / 1e12 / peak, "launch": ctx3.launch("dd")}
        del o3, p3, ctx3
        # f1: one Newton step (evaluate + solve) per point on device, complex dd
        xo = torch.empty_like(x_dd)
        nst = torch.empty(Bx, dtype=torch.int32, device=dev)
        ctx.evaluate_device(x_dd, out_x, "dd", args.order, stream)
        ms_solve = timed(lambda: ctx.newton_solve_device(out_x, x_dd, xo, "dd", status=nst, stream=stream), 5)
        ms_step = timed(lambda: ctx.newton_step_device(x_dd, out_x, xo, "dd", status=nst, stream=stream), 5)
        # end to end through the host API: points in, corrected points out (1 KB each way per point)
        hx = torch.from_numpy(np.ascontiguousarray(dd[:Bx])).pin_memory().numpy()
        hxo = torch.empty(hx.shape, dtype=torch.float64).pin_memory().numpy()
        hn = torch.empty((Bx, 2), dtype=torch.float64).pin_memory().numpy()
        hs = torch.empty(Bx, dtype=torch.int32).pin_memory().numpy()
        ctx.newton_host(hx, "dd", iters=1, out=hxo, norms=hn, status=hs)  # warm (allocates staging)
        t0 = time.perf_counter()
        ctx.newton_host(hx, "dd", iters=1, out=hxo, norms=hn, status=hs)
        e2e_newton_s = time.perf_counter() - t0
        nf = newton_model_flops(N)
        line["newton"] = {"config": "f1: C2 Newton step x <- x + J^-1 (-f), complex dd, 65,536 points per GPU",
                          "steps_per_s": Bx / (ms_step * 1e-3), "ms_per_step": ms_step,
                          "solve_ms": ms_solve, "solve_points_per_s": Bx / (ms_solve * 1e-3),
                          "solve_flops_per_point": nf,
                          "solve_fp64_frac": nf * Bx / (ms_solve * 1e-3) / 1e12 / peak,
                          "status_ok_frac": float((nst == 0).float().mean().item()),
                          "e2e_steps_per_s": Bx / e2e_newton_s,
                          "e2e_api": "EvaluationContext.newton_host -> pj_newton_host (H2D points, evaluate + solve "
                                     "in L2-sized chunks, D2H corrected points, norms, status)",
                          "launch": ctx.launch("dd", newton=True)}
        # the mixed-precision solve (PJ_NEWTON_MIXED, opt-in): complex-double factors of the dd
        # Jacobian, two dd-residual refinement steps; dd points in and out, status 3 when the
        # refinement has not converged (then the dd solve above is the one to use)
        ms_solve_mx = timed(lambda: ctx.newton_solve_device(out_x, x_dd, xo, "mixed", status=nst, stream=stream), 5)
        ms_step_mx = timed(lambda: ctx.newton_step_device(x_dd, out_x, xo, "mixed", status=nst, stream=stream), 5)
        line["newton"]["mixed"] = {"solve_ms": ms_solve_mx, "solve_points_per_s": Bx / (ms_solve_mx * 1e-3),
                                   "steps_per_s": Bx / (ms_step_mx * 1e-3), "ms_per_step": ms_step_mx,
                                   "status_ok_frac": float((nst == 0).float().mean().item()),
                                   "launch": ctx.launch("mixed", newton=True)}
        del xo, x_dd
        # C1: one point through the reference-shaped host API (EvaluationContext.evaluate:
        # H2D, kernel, D2H, unpack), complex double as the reference; and one dd point
        pt1 = host_pts[0]
        for _ in range(20):
            ctx.evaluate(pt1)
        reps = 200
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.evaluate(pt1)
        c1_d_us = (time.perf_counter() - t0) / reps * 1e6
        p1 = dd[:1]
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.evaluate_dd(p1)
        c1_dd_us = (time.perf_counter() - t0) / reps * 1e6
        line["c1_latency"] = {"config": "C1: one point, n=32 m=32 k=8 d=2, through EvaluationContext.evaluate "
                                        "(host buffers, synchronous)",
                              "gpu_us_per_eval_d": c1_d_us, "gpu_us_per_eval_dd": c1_dd_us,
                              "reference_cpu_us_per_eval": None}

    # ---------------- (7) CPU baseline (rank 0, N=1 only): the unmodified reference
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            if O.ref_available():
                v, Bs, dt, thr = reference_cpu(sysd, N, target_seconds=args.ref_seconds)
                vdd, Bdd, dtdd, _ = reference_cpu(sysd, N, target_seconds=args.ref_seconds / 2, prec="dd-port")
                line["cpu_baseline"] = {
                    "value": v, "unit": "evals/s", "cores": thr, "kind": "reference",
                    "sample": f"{Bs} points of the same workload through the unmodified reference "
                              f"EvaluationContext::evaluate (complex double — the reference has no dd path), "
                              f"{thr} threads point-sharded, {dt:.2f} s; {cpu_model()}",
                    "dd_port": {"value": vdd, "unit": "evals/s", "cores": thr, "kind": "port",
                                "sample": f"{Bdd} points through the oracle's complex-dd restatement, {dtdd:.2f} s"},
                }
                if "quality_up" in line:
                    line["quality_up"]["cpu_dd_over_d_time"] = v / vdd  # reference (d) vs the dd restatement
                if "c1_latency" in line:
                    line["c1_latency"]["reference_cpu_us_per_eval"] = reference_c1_latency(sysd)
        except Exception as exc:  # the baseline must never hide the measurement
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line))
    if dist:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
