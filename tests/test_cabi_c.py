"""The C ABI from plain C (CPU): include/polyjac_b200.h compiles as C99 with -Wall -Werror and the
host-only entry points (generator, validation, index maps, counters, system text IO, error codes)
behave as documented, without a GPU (tests/c/test_cabi.c)."""
import os
import subprocess

from conftest import ROOT


def test_c_abi_from_c99(tmp_path):
    exe = tmp_path / "test_cabi"
    lib = os.path.join(ROOT, "paper_1201_0499_b200")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c", "test_cabi.c"), "-L" + lib, "-lpolyjac_b200", "-Wl,-rpath," + lib,
           "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
