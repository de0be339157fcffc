"""CLI (row f3), mirroring ref tests/test_cli.cpp: subcommands, exit codes 0/1/2, the RESULT
key=value line with the closed-form multiplication count, footprint warning. `generate` and
the usage errors run on CPU; `bench` / `check` need the GPU."""
import os
import subprocess

import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import ROOT

CLI = os.path.join(ROOT, "paper_1201_0499_b200", "polyjac_b200")


def run(*args, timeout=600):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def result_line(out):
    for ln in out.splitlines():
        if ln.startswith("RESULT "):
            return dict(f.split("=", 1) for f in ln[7:].split() if "=" in f)
    return {}


def test_generate_deterministic_and_bit_identical(tmp_path):
    a, b = tmp_path / "t1.sys", tmp_path / "t1b.sys"
    rc, out = run("generate", "--n", 32, "--m", 32, "--k", 9, "--d", 2, "--seed", 7, "--out", a)
    assert rc == 0 and "18432" in out and "warning" not in out
    s = pj.read_system(str(a))
    want = pj.random_system(32, 32, 9, 2, 7)
    assert np.array_equal(s.coeffs.view(np.uint64), want.coeffs.view(np.uint64))
    assert np.array_equal(s.positions, want.positions) and np.array_equal(s.exponents, want.exponents)
    assert run("generate", "--n", 32, "--m", 32, "--k", 9, "--d", 2, "--seed", 7, "--out", b)[0] == 0
    assert a.read_bytes() == b.read_bytes()


def test_generate_warns_at_constant_memory_boundary(tmp_path):
    rc, out = run("generate", "--n", 32, "--m", 64, "--k", 16, "--d", 10, "--seed", 3, "--out", tmp_path / "big.sys")
    assert rc == 0 and "65536" in out and "warning" in out


def test_usage_errors_exit_2(tmp_path):
    assert run("generate", "--n", 4, "--m", 4, "--k", 9, "--d", 2, "--out", tmp_path / "x.sys")[0] == 2
    assert run("bench", "--evals", 5)[0] == 2
    assert run("bench", "--n", 4, "--m", 4, "--k", 2, "--d", 2, "--evals", 0)[0] == 2
    assert run("bench", "--system", "/no/such.sys")[0] == 2
    assert run("nonsense")[0] == 2
    assert run("check", "--points", 5)[0] == 2
    bad = tmp_path / "bad.sys"
    bad.write_text("1 1 1 2\n1 0 1 0\n")
    rc, out = run("check", "--system", bad, "--points", 5)
    assert rc == 2 and "exponent out of range" in out


def test_help():
    rc, out = run("--help")
    assert rc == 0 and all(w in out for w in ("generate", "bench", "check"))


@pytest.mark.gpu
def test_bench_result_line(gpu):
    rc, out = run("bench", "--n", 8, "--m", 8, "--k", 3, "--d", 2, "--seed", 5, "--evals", 5, "--workers", 2,
                  "--block-size", 32)
    assert rc == 0, out
    kv = result_line(out)
    assert kv["n"] == "8" and kv["monomials"] == "64" and kv["evals"] == "5"
    assert kv["footprint_bytes"] == "384"
    assert kv["mults"] == str(5 * (128 + 704))  # ref tests/test_cli.cpp:110-125
    assert {"baseline_ms", "pipeline_ms", "speedup"} <= set(kv)
    assert float(kv["gate_max_rel"]) <= 1e-10


@pytest.mark.gpu
def test_bench_system_file_and_check(tmp_path, gpu):
    f = tmp_path / "b.sys"
    assert run("generate", "--n", 6, "--m", 4, "--k", 2, "--d", 3, "--seed", 9, "--out", f)[0] == 0
    rc, out = run("bench", "--system", f, "--evals", 3)
    assert rc == 0 and result_line(out)["m"] == "4"
    c = tmp_path / "c.sys"
    assert run("generate", "--n", 10, "--m", 6, "--k", 4, "--d", 3, "--seed", 12, "--out", c)[0] == 0
    rc, out = run("check", "--system", c, "--points", 20, "--seed", 4)
    assert rc == 0 and "PASS" in out
    assert run("check", "--system", c, "--tol", 0)[0] == 2


@pytest.mark.gpu
def test_bench_c2_shape(gpu):
    rc, out = run("bench", "--n", 32, "--m", 32, "--k", 8, "--d", 2, "--seed", 7, "--evals", 131072)
    assert rc == 0, out
    kv = result_line(out)
    assert kv["precision"] == "dd" and float(kv["evals_per_s"]) > 1e6


def test_gpus_beyond_visible_devices_is_a_usage_error():
    rc, out = run("bench", "--n", 8, "--m", 4, "--k", 3, "--d", 2, "--gpus", 4096)
    assert rc == 2 and "exceeds" in out
    assert run("bench", "--n", 8, "--m", 4, "--k", 3, "--d", 2, "--gpus", 0)[0] == 2


@pytest.mark.gpu
def test_bench_multi_gpu_sharding(gpu):
    import torch
    g = torch.cuda.device_count()
    rc, out = run("bench", "--n", 32, "--m", 32, "--k", 8, "--d", 2, "--seed", 7, "--evals", 65536, "--gpus", g)
    assert rc == 0, out
    kv = result_line(out)
    assert kv["gpus"] == str(g) and float(kv["evals_per_s"]) > 1e6


@pytest.mark.gpu
def test_gate_is_independent_of_the_device_pipeline(tmp_path, gpu):
    # ref SPEC.md:462: a deliberately corrupted coefficient must fail the gate. The corruption is
    # applied to the DEVICE copies only (pj_debug_corrupt_coeff, both precisions and every table),
    # so a check that compared the device paths with each other would still pass; the brute-force
    # host evaluation catches it: check exits 1 and names the polynomial of monomial 37 (p = 6)
    c = tmp_path / "c.sys"
    assert run("generate", "--n", 10, "--m", 6, "--k", 4, "--d", 3, "--seed", 12, "--out", c)[0] == 0
    rc, out = run("check", "--system", c, "--points", 8, "--seed", 4, "--corrupt-coeff", 37)
    assert rc == 1 and "FAIL" in out and "f[6]" in out, out
    rc, out = run("bench", "--system", c, "--evals", 3, "--corrupt-coeff", 37)
    assert rc == 1 and "correctness gate failed" in out, out
    # unmodified, both pass
    assert run("check", "--system", c, "--points", 8, "--seed", 4)[0] == 0
    rc, out = run("bench", "--system", c, "--evals", 3)
    assert rc == 0 and float(result_line(out)["baseline_ms"]) > 0
