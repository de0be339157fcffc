"""The reference's OWN unit suites (ref tests/test_*.cpp), built unmodified against a
doctest-compatible header written for this repo (oracle/shim/doctest.h; the reference's
vendor/doctest.h is absent), by oracle/Makefile from the sources where they lie.

* CPU: test_system / test_packing / test_kernels / test_oracle / test_engine / test_io against the
  unmodified reference library — pins the oracle harness itself (every known answer of the
  reference's own tests holds in the library the oracle and the CPU baseline link).
* GPU: test_engine.cpp with polyjac::EvaluationContext bound to the B200 drop-in
  (oracle/shim_dropin/polyjac/engine.hpp -> include/polyjac_b200_dropin.hpp): the reference's own
  engine tests, call syntax untouched, against the GPU path.
* GPU: test_cli.cpp with POLYJAC_CLI pointing at the B200 command-line front end (row f3).
"""
import os
import subprocess

import pytest

from conftest import ROOT
from oracle import oracle as O

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _bin(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time: __graft_entry__.build())")
    return path


def _run(path, env=None, timeout=600):
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout, env=env)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.parametrize("suite", O.REF_SUITES)
def test_reference_suite_passes_on_the_reference_library(suite):
    rc, out = _run(_bin(suite))
    assert rc == 0 and "Status: SUCCESS" in out, out[-3000:]


def test_doctest_shim_reports_failures(tmp_path):
    # the shim must not pass vacuously: a failing CHECK, a missing throw and a failed REQUIRE all
    # fail the run, and a passing file passes
    src = tmp_path / "t.cpp"
    src.write_text('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include <doctest.h>\n#include <stdexcept>\n'
                   'TEST_CASE("a") { CHECK(1 + 1 == 3); }\n'
                   'TEST_CASE("b") { CHECK_THROWS_AS((void)0, std::runtime_error); }\n'
                   'TEST_CASE("c") { REQUIRE(false); CHECK(true); }\n'
                   'TEST_CASE("d") { CHECK(0.1 + 0.2 == doctest::Approx(0.3)); '
                   'CHECK_THROWS_WITH_AS(throw std::invalid_argument("abc def"), doctest::Contains("c d"), '
                   'std::invalid_argument); }\n')
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-I" + os.path.join(ROOT, "oracle", "shim"), str(src), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 1 and "3 failed" in r.stdout, r.stdout
    r = subprocess.run([str(exe), "-tc=d"], capture_output=True, text=True)
    assert r.returncode == 0 and "1 passed" in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_engine_suite_passes_on_the_b200_dropin():
    rc, out = _run(_bin("test_engine_b200"))
    assert rc == 0 and "Status: SUCCESS" in out and "16 passed" in out, out[-3000:]


@pytest.mark.gpu
def test_reference_cli_suite_passes_on_the_b200_cli():
    cli = os.path.join(ROOT, "paper_1201_0499_b200", "polyjac_b200")
    assert os.path.exists(cli)
    env = dict(os.environ, POLYJAC_CLI=cli)
    rc, out = _run(_bin("test_cli"), env=env)
    assert rc == 0 and "Status: SUCCESS" in out, out[-3000:]
