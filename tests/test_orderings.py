"""Host-side bank-aware orderings (csrc/capi.cpp: order_variables, order_stage3, assign_columns,
the phase-2 records) — CPU only: tests/cpp/test_orderings.cpp includes the C ABI's translation
unit, builds contexts without a device and checks that every ordering is a permutation that keeps
each staged term and segment partial exactly once, and that schedules are deterministic."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT


def test_host_orderings(tmp_path):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc) and not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    from paper_1201_0499_b200 import build as B

    B.build()  # up to date: no-op; provides the kernel objects the test links against
    obj = tmp_path / "test_orderings.o"
    exe = tmp_path / "test_orderings"
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-w", "-I/usr/local/cuda/include", "-c",
                        os.path.join(ROOT, "tests", "cpp", "test_orderings.cpp"), "-o", str(obj)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    objs = [os.path.join(B.BUILD, f + ".o") for f in B.CU] + [os.path.join(B.BUILD, "sysio.cpp.o")]
    r = subprocess.run([nvcc, *B.ARCH, "-o", str(exe), str(obj), *objs], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
