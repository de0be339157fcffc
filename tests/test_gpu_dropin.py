"""The C++ drop-in surface (include/polyjac_b200.hpp) fed the reference's own
polyjac::PolynomialSystem gives bit-identical results to polyjac::EvaluationContext
(tests/cpp/test_dropin.cpp, built by `make -C oracle dropin`)."""
import os
import subprocess

import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_cpp_dropin_bit_identical_to_reference(gpu):
    if not os.path.exists(O.DROPIN_BIN):
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([O.DROPIN_BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("PASS")
