#!/usr/bin/env python3
"""Benchmark of the hot path: complex double-double system + Jacobian evaluation.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)

Workload (BASELINE.json configs[1]): random_system(32, 32, 8, 2, seed 7) (n=32 variables,
32 polynomials x 32 monomials of k=8 variables, degrees <= 2), a batch of 65,536 points per
GPU drawn from random_points(32, ., seed 11) — contiguous shards of one stream, so the
union over ranks is the single-process batch. A step = one evaluation of the batch (values +
full Jacobian, complex dd). Weak scaling: per-GPU batch fixed; no collective on the data
path (the barrier and the max-over-ranks timing reduction are the only ones).

One JSON line (rank 0). `value` = evaluations/s over all ranks, device time (CUDA events on
the launching stream, max over ranks); `e2e` = the same through the public host API
(pinned host points -> H2D -> kernels -> D2H of every value and Jacobian entry);
`roofline` = the kernel's algorithmic FP64 rate (SURVEY.md §8d cost model) over the FP64
peak measured live on this device; `cpu_baseline` = the unmodified reference (compiled from
/root/reference sources into oracle/_ref) on this host's cores, a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
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
POINTS_PER_GPU = 65536
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


def reference_cpu(sysd, n, target_seconds=8.0, threads=None, prec="ref"):
    """Time the unmodified reference (oracle/_ref, complex double — the reference has no dd) or
    the oracle's dd restatement (prec="dd-port") point-sharded across host threads (one
    workers=1 context per thread). Bounded sample sized from a calibration run."""
    from oracle import oracle as O
    threads = threads or cpu_count()
    rng_pts = O.ref_random_points(n, 1, PT_SEED) if O.ref_available() else None

    def run(B):
        if prec == "ref":
            pts = O.ref_random_points(n, B, PT_SEED)
            t0 = time.perf_counter()
            O.ref_evaluate(sysd, pts, threads=threads)
            return time.perf_counter() - t0, pts
        pts2 = O.ref_random_points(n, B, PT_SEED) if O.ref_available() else None
        p4 = np.zeros((B, n, 4))
        p4[..., 0], p4[..., 2] = pts2[..., 0], pts2[..., 1]
        t0 = time.perf_counter()
        O.evaluate("dd", sysd, p4, threads=threads)
        return time.perf_counter() - t0, p4

    del rng_pts
    cal = 32 * threads
    dt, _ = run(cal)
    B = int(min(max(cal, cal * target_seconds / max(dt, 1e-6)), 1 << 20))
    dt, pts = run(B)
    return B / dt, B, dt, threads, pts


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
    vals, dts = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.ref_evaluate(sysd, pts, threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(B_used / dt)
            dts.append(dt)
    value = B_used * len(dts) / sum(dts)
    dt_used = sum(dts) / len(dts)
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt_used * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic: reference random_system(32,32,8,2,seed 7), random_points(32, ., seed 11)",
        "config": {"workload": "C2: n=32 m=32 k=8 d=2, evaluation-point batch (bounded CPU sample)",
                   "points_per_step": B_used, "parallelism": f"{threads} host threads, point-sharded"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "reference",
                         "sample": f"{B_used} points per step through the unmodified reference "
                                   "EvaluationContext::evaluate (complex double: the reference has no "
                                   f"double-double path), one workers=1 context per thread; {cpu_model()}"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--points", type=int, default=POINTS_PER_GPU, help="points per GPU per step (weak scaling)")
    ap.add_argument("--global-points", type=int, default=0,
                    help="fixed total points per step sharded over the ranks (strong scaling; C5: 1048576)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--order", default="fast", choices=["fast", "ref"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for the barrier and the max-over-ranks timing reduction")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary lines (C3, C4 quality-up factor, f1 Newton step)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1201_0499_b200 as pj

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
        t = torch.tensor([x], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if dist:
            tdist.barrier()

    sysobj = pj.random_system(N, M, K, D, SYS_SEED)
    ctx = pj.EvaluationContext(sysobj, device=local)
    B = args.points
    scaling = "weak"
    if args.global_points:
        if args.global_points % ws:
            raise SystemExit(f"--global-points {args.global_points} is not divisible by {ws} ranks")
        B = args.global_points // ws
        scaling = "strong"
    nout = N + N * N
    # this rank's contiguous shard of the global point stream
    from paper_1201_0499_b200.sharding import shard_points
    host_pts = shard_points(N, B * ws, PT_SEED, ws, rank)  # complex128 [B, n]
    dd = pj.to_dd(host_pts)
    # inputs > L2: rotate over NBUF distinct device batches (NBUF * 67 MB > 126 MB L2)
    NBUF = 4
    bufs = []
    for i in range(NBUF):
        t = torch.from_numpy(np.roll(dd, i, axis=0).copy()).to(dev)
        bufs.append(t)
    out = torch.empty((B, nout, 4), dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            ctx.evaluate_device(bufs[i % NBUF], out, "dd", args.order, stream)
    stream.synchronize()
    if ctx.nonfinite_seen(stream):
        raise RuntimeError("non-finite input")

    # ---------------- timed region (device): K steps, events on the launching stream
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
    total_ms = evs[0].elapsed_time(evs[-1])
    if dist:
        total_ms = max_over_ranks(total_ms)
    value = B * ws * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps
    kern_ms = statistics.mean(per)

    # ---------------- e2e through the public host API (pinned host buffers)
    Be = min(B, POINTS_PER_GPU)  # strong-scaling runs with huge shards time e2e on a C2-sized sample
    pin_in = torch.from_numpy(dd[:Be]).pin_memory()
    pin_out = torch.empty((Be, nout, 4), dtype=torch.float64).pin_memory()
    ni, no = pin_in.numpy(), pin_out.numpy()
    ctx.evaluate_host(ni, "dd", args.order, out=no)  # warm (allocates the staging buffers)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        ctx.evaluate_host(ni, "dd", args.order, out=no)
    e2e_s = time.perf_counter() - t0
    if dist:
        e2e_s = max_over_ranks(e2e_s)
    e2e = {"value": Be * ws * args.e2e_steps / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": int(ni.nbytes),
           "d2h_bytes_per_step": int(no.nbytes), "steps": args.e2e_steps,
           "api": "EvaluationContext.evaluate_host -> pj_evaluate_host (3-stream chunked H2D/kernel/D2H)"}

    # ---------------- roofline: FP64 issue-bound
    peak = pj.fp64_peak_tflops(local)
    flops = model_flops(N, M, K, D)
    achieved = flops * B / (kern_ms * 1e-3) / 1e12
    io_bytes = B * (N * 32 + nout * 32)
    traffic = None
    ncu = {}
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                ncu = json.load(fh)
            traffic = ncu.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "algorithmic_bytes": io_bytes,
                "hbm_gbs_achieved": io_bytes / (kern_ms * 1e-3) / 1e9,
                "flops_per_eval": flops,
                "peak_source": "pj_fp64_peak_probe: DFMA throughput measured live on this device (2 flops/DFMA); "
                               "MEASURED_PEAKS.json carries no FP64 figure",
                "note": "achieved = the fixed SURVEY.md 8(d) cost model (80 flops per complex dd product, 40 per "
                        "add) over device time; the kernel executes fewer FP64 instructions than the model "
                        "counts (coefficient-seeded back-fused products, 32-38 instead of 68 instructions per "
                        "product) - the instruction-level view is in ncu_* (committed capture)"}
    if ncu.get("launches"):
        L0 = ncu["launches"][0]
        roofline["ncu_kernel"] = ncu.get("kernel")
        roofline["ncu_fp64_pipe_active_pct"] = L0.get("fp64_pipe_active_pct")
        roofline["ncu_issue_active_pct"] = L0.get("issue_active_pct")
    hw = os.path.join(ROOT, "profiles", "fp64_exec.json")
    if os.path.exists(hw):
        try:
            with open(hw) as fh:
                h = json.load(fh)
            roofline["ncu_hw_fp64_tflops"] = h.get("hw_fp64_tflops")
            roofline["ncu_fp64_instr_per_eval"] = h.get("fp64_instr_per_eval")
        except (OSError, ValueError):
            pass

    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "complex-dd (f64 pairs)",
        "data": "synthetic: random_system(32,32,8,2,seed 7), random_points(32, 65536*N, seed 11) sharded by rank",
        "config": {"workload": (f"C5: n=32 m=32 k=8 d=2, {B * ws:,} evaluation points per step sharded over "
                                f"{ws} GPU(s)" if args.global_points else
                                f"C2: n=32 m=32 k=8 d=2, {B:,} evaluation points per GPU per step"),
                   "points_per_gpu": B, "global_points": B * ws, "order": args.order,
                   "parallelism": f"points sharded over {ws} GPU(s), system replicated, no collective",
                   "l2": f"inputs rotate over {NBUF} device batches ({NBUF * dd.nbytes >> 20} MiB > 126 MiB L2); "
                         f"outputs {B * nout * 32 >> 20} MiB per step",
                   "launch": ctx.launch("dd")},
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "clocks": clk,
    }

    # ---------------- secondary measurements (outside the headline timed region)
    if not args.no_extras:
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
        # C4: complex double vs complex double-double on the same points (quality-up overhead)
        d2 = torch.from_numpy(np.stack([host_pts.real, host_pts.imag], -1).copy()).to(dev)
        out_d = torch.empty((B, nout, 2), dtype=torch.float64, device=dev)
        ms_d = timed(lambda: ctx.evaluate_device(d2, out_d, "d", None, stream), 10)
        line["quality_up"] = {"config": "C4: C2 in complex double (reference order, bit-exact with the reference) "
                                        "vs complex dd (fast order)",
                              "d_evals_per_s": B / (ms_d * 1e-3), "dd_evals_per_s": B / (kern_ms * 1e-3),
                              "dd_over_d_time": kern_ms / ms_d, "d_launch": ctx.launch("d")}
        del out_d
        # C3: n=64 m=64 k=16 d=10 (higher degrees, larger common-factor stage), complex dd
        s3 = pj.random_system(64, 64, 16, 10, SYS_SEED)
        ctx3 = pj.EvaluationContext(s3, device=local)
        B3 = 8192
        p3 = torch.from_numpy(pj.to_dd(pj.random_points(64, B3, PT_SEED))).to(dev)
        o3 = torch.empty((B3, 64 + 64 * 64, 4), dtype=torch.float64, device=dev)
        ms3 = timed(lambda: ctx3.evaluate_device(p3, o3, "dd", args.order, stream), 5)
        f3 = model_flops(64, 64, 16, 10)
        line["c3"] = {"config": "C3: random_system(64,64,16,10,seed 7), 8,192 points, complex dd, fast order",
                      "evals_per_s": B3 / (ms3 * 1e-3), "ms_per_batch": ms3, "flops_per_eval": f3,
                      "roofline_frac": f3 * B3 / (ms3 * 1e-3) / 1e12 / peak, "launch": ctx3.launch("dd")}
        del o3, p3, ctx3
        # f1: one Newton step (evaluate + solve) per point on device, complex dd
        xo = torch.empty_like(bufs[0])
        nst = torch.empty(B, dtype=torch.int32, device=dev)
        ms_solve = timed(lambda: ctx.newton_solve_device(out, bufs[0], xo, "dd", status=nst, stream=stream), 5)
        ms_step = timed(lambda: ctx.newton_step_device(bufs[0], out, xo, "dd", status=nst, stream=stream), 5)
        # end to end through the host API: points in, corrected points out (1 KB each way per point),
        # page-locked host buffers
        hx = torch.from_numpy(dd).pin_memory().numpy()
        hxo = torch.empty(dd.shape, dtype=torch.float64).pin_memory().numpy()
        hn = torch.empty((B, 2), dtype=torch.float64).pin_memory().numpy()
        hs = torch.empty(B, dtype=torch.int32).pin_memory().numpy()
        ctx.newton_host(hx, "dd", iters=1, out=hxo, norms=hn, status=hs)  # warm (allocates staging)
        t0 = time.perf_counter()
        ctx.newton_host(hx, "dd", iters=1, out=hxo, norms=hn, status=hs)
        e2e_newton_s = time.perf_counter() - t0
        nf = newton_model_flops(N)
        line["newton"] = {"config": "f1: C2 Newton step x <- x + J^-1 (-f), complex dd, 65,536 points per GPU",
                          "steps_per_s": B / (ms_step * 1e-3), "ms_per_step": ms_step,
                          "solve_ms": ms_solve, "solve_points_per_s": B / (ms_solve * 1e-3),
                          "solve_flops_per_point": nf,
                          "solve_fp64_frac": nf * B / (ms_solve * 1e-3) / 1e12 / peak,
                          "status_ok_frac": float((nst == 0).float().mean().item()),
                          "e2e_steps_per_s": B / e2e_newton_s,
                          "e2e_api": "EvaluationContext.newton_host -> pj_newton_host (H2D points, evaluate + solve "
                                     "in L2-sized chunks, D2H corrected points, norms, status)",
                          "launch": ctx.launch("dd", newton=True)}
        del xo

    # ---------------- CPU baseline (rank 0, N=1 only): the unmodified reference
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            if O.ref_available():
                sysd = O.ref_random_system(N, M, K, D, SYS_SEED)
                v, Bs, dt, thr, pts = reference_cpu(sysd, N, target_seconds=args.ref_seconds)
                vdd, Bdd, dtdd, _, p4 = reference_cpu(sysd, N, target_seconds=args.ref_seconds / 2, prec="dd-port")
                line["cpu_baseline"] = {
                    "value": v, "unit": "evals/s", "cores": thr, "kind": "reference",
                    "sample": f"{Bs} points of the same workload through the unmodified reference "
                              f"EvaluationContext::evaluate (complex double — the reference has no dd path), "
                              f"{thr} threads point-sharded, {dt:.2f} s; {cpu_model()}",
                    "dd_port": {"value": vdd, "unit": "evals/s", "cores": thr, "kind": "port",
                                "sample": f"{Bdd} points through the oracle's complex-dd restatement, {dtdd:.2f} s"},
                }
                # checker: the GPU result on the CPU sample's first points vs the oracle (dd)
                chk = min(64, Bdd)
                want, ms = O.evaluate("dd", sysd, p4[:chk], magsum=True)
                got = ctx.evaluate_dd(p4[:chk])
                err = np.maximum(np.abs((got[..., 0] - want[..., 0]) + (got[..., 1] - want[..., 1])),
                                 np.abs((got[..., 2] - want[..., 2]) + (got[..., 3] - want[..., 3])))
                if "quality_up" in line:
                    line["quality_up"]["cpu_dd_over_d_time"] = v / vdd  # reference (d) vs the dd restatement
                line["parity_gate"] = {"points": chk, "max_err_over_sum_abs_terms": float(np.max(err / np.maximum(ms, 1e-300))),
                                       "tol": 1e-30}
        except Exception as exc:  # the baseline must never hide the measurement
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line))
    if dist:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
