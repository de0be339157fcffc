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


def test_cpp_headers_compile_with_reference_call_syntax(tmp_path):
    # own-types header: the reference's call syntax compiles against polyjac_b200::EvaluationContext
    # (no template arguments, braced points, layout(), masked_slots_clean()) -Wall -Werror; with the
    # reference headers present, the same body compiles against the reference-types drop-in
    body = r'''
    template <class Ctx, class Sys, class Point, class Result, class Batch>
    void use(const Sys& sys, const Point& pt) {
        Ctx ctx(sys, {32, 4});
        const Result r = ctx.evaluate(pt);
        const Batch b = ctx.evaluate_batch({pt, pt}, 3);
        (void)r.jac(0, 0);
        (void)b.report.mults.total();
        (void)ctx.layout().footprint_bytes();
        (void)ctx.layout().deriv_coeff(0, 0);
        (void)ctx.masked_slots_clean();
        (void)(ctx.mults() == ctx.mults());
        (void)ctx.grid().workers;
    }
    '''
    src = tmp_path / "own.cpp"
    src.write_text('#include "polyjac_b200.hpp"\n' + body +
                   'int main() { namespace P = polyjac_b200; P::PolynomialSystem s; P::EvaluationPoint x;\n'
                   '  if (s.n < 0) use<P::EvaluationContext, P::PolynomialSystem, P::EvaluationPoint, '
                   'P::EvaluationResult, P::BatchResult>(s, x);\n  return 0; }\n')
    inc = ["-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include"]
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", *inc, "-fsyntax-only", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    ref_inc = "/root/reference/proj/include"
    if os.path.isdir(ref_inc):
        src2 = tmp_path / "ref.cpp"
        src2.write_text('#include "polyjac_b200_dropin.hpp"\n' + body +
                        'int main() { polyjac::PolynomialSystem s; polyjac::EvaluationPoint x;\n'
                        '  if (s.n < 0) use<polyjac_b200::dropin::EvaluationContext, polyjac::PolynomialSystem, '
                        'polyjac::EvaluationPoint, polyjac::EvaluationResult, polyjac::BatchResult>(s, x);\n'
                        '  return 0; }\n')
        r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", *inc, "-I" + ref_inc,
                            "-fsyntax-only", str(src2)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
