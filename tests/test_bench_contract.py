"""bench.py's reference arm runs on CPU and prints one contract-shaped JSON line."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle import oracle as O


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--ref-seconds", "0.2"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "config", "higher_is_better"):
        assert key in line
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"


def test_model_flops_matches_survey():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.model_flops(32, 32, 8, 2) == 3891200
    assert bench.model_flops(64, 64, 16, 10) == 32645120   # C3
    assert bench.model_flops(32, 32, 8, 2, "d") == 282624


def test_newton_model_flops():
    sys.path.insert(0, ROOT)
    import bench
    # n = 32: 11,968 complex products and 11,440 complex additions per solve (docstring of the model)
    assert bench.newton_model_flops(32) == 11968 * 80 + 11440 * 40
    assert bench.newton_model_flops(1) == 2 * 80 + 1 * 40  # one inverse, one dx product, x + dx


@pytest.mark.gpu
def test_bench_json_line_on_gpu(gpu):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--e2e-steps", "1", "--ref-seconds", "0.5"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks",
                "cpu_baseline", "quality_up", "c3", "newton"):
        assert key in line, key
    assert line["steps"] == 3 and line["warmup"] == 3 and line["n_gpus"] == 1 and line["value"] > 1e6
    roof = line["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof) and roof["frac"] > 0.5
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] == 3 and line["cpu_baseline"]["kind"] == "reference"
    gate = line["parity_gate"]
    assert gate["pass"] and gate["max_err_over_sum_abs_terms"] <= gate["tol"] and gate["dd_points"] >= 1024
    assert gate["d_words_differing"] == 0 and gate["structural_zeros_exact"]
    assert line["newton"]["status_ok_frac"] == 1.0
    assert "c1_latency" in line and line["c1_latency"]["gpu_us_per_eval_d"] > 0
    assert line["c3"]["config"].startswith("C3") and "65,536" in line["c3"]["config"]
    # the hardware view is counted in this run (ncu on one untimed launch), not copied from profiles/
    assert 0.2 < roof["hw_fp64_pipe_frac"] <= 1.0 and roof["traffic"] > 0
    assert roof["peak"] >= 2 * max(roof["probe_lane_ops_per_s"].values()) / 1e12 * 0.999


@pytest.mark.gpu
def test_bench_exits_nonzero_on_a_broken_kernel(gpu):
    # a corrupted device coefficient (pj_debug_corrupt_coeff) must fail the gate BEFORE timing:
    # exit status 3 and no JSON line
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-extras", "--no-cpu-baseline", "--no-hw-counts", "--inject-fault"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 3, r.stderr[-2000:]
    assert "parity gate FAILED" in r.stderr and not r.stdout.strip()


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu(gpu):
    # the multi-rank path of the harness (shards, barrier, max-over-ranks timing, rank-0 line) with
    # two ranks sharing the box's GPU over gloo; the driver's N-GPU runs use one GPU per rank + NCCL
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--no-extras", "--dist-backend", "gloo",
           "--global-points", "131072"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_points"] == 131072 and line["scaling"] == "strong"
    assert line["config"]["points_per_gpu"] == 65536 and line["config"]["workload"].startswith("C5")
    assert line["value"] > 1e6 and "cpu_baseline" not in line  # the CPU baseline is N=1 only
    g = line["gather"]
    assert g["rank0_rows"] == 131072 and g["own_rows_intact"] and g["bytes_into_rank0"] == 65536 * 1056 * 32
    assert line["parity_gate"]["pass"]
