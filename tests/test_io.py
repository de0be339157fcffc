"""System text files (row f2), mirroring ref tests/test_io.cpp, cross-checked byte for byte
against the reference's own write_system / read_system (oracle/_ref). CPU only."""
import os

import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import sysd_of
from oracle import oracle as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def same(a, b):
    return (a.n, a.m, a.k, a.d) == (b.n, b.m, b.k, b.d) and np.array_equal(a.positions, b.positions) and \
        np.array_equal(a.exponents, b.exponents) and np.array_equal(a.coeffs.view(np.uint64), b.coeffs.view(np.uint64))


@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (5, 3, 2, 9), (32, 22, 9, 2), (32, 48, 16, 10)])
def test_round_trip_bit_exact(shape):
    s = pj.random_system(*shape, 9000 + sum(shape))
    assert same(pj.read_system_text(pj.write_system_text(s)), s)


@needs_ref
@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (5, 3, 2, 9), (32, 32, 8, 2), (64, 64, 16, 10)])
def test_text_identical_to_reference_writer_and_readable_by_it(shape):
    s = pj.random_system(*shape, 11)
    text = pj.write_system_text(s)
    assert text == O.ref_write_system(sysd_of(s))
    back = O.ref_read_system(text)
    assert np.array_equal(back["coeffs"].view(np.uint64), s.coeffs.view(np.uint64))
    assert np.array_equal(back["pos"], s.positions.reshape(-1))


def test_deterministic_and_one_based():
    s = pj.random_system(6, 4, 3, 7, 42)
    assert pj.write_system_text(s) == pj.write_system_text(s)
    t = [pj.Term(1.0, pj.MonomialSupport([0], [1])), pj.Term(1.0, pj.MonomialSupport([1], [1]))]
    assert pj.write_system_text(pj.PolynomialSystem.from_terms(2, 1, 1, 1, t)) == "2 1 1 1\n1 0 1 1\n1 0 2 1\n"


def test_comments_and_blank_lines():
    s = pj.read_system_text("# a system\n\n1 1 1 2   # header\n  0.5 -0.25 1 2\n# trailing comment\n")
    assert s.n == 1 and s.coeffs[0, 0] == 0.5 and s.coeffs[0, 2] == -0.25
    assert s.positions[0, 0] == 0 and s.exponents[0, 0] == 2


BAD = [
    ("1 1 1 2\n1 0 1 0\n", "exponent out of range"),
    ("1 1 1 2\n1 0 1 3\n", "exponent out of range"),
    ("2 1 2 2\n1 0 1 1 1 2\n1 0 1 1 2 1\n", "strictly increasing"),
    ("2 1 2 2\n1 0 2 1 1 2\n1 0 1 1 2 1\n", "strictly increasing"),
    ("1 1 1 2\n0 0 1 1\n", "zero coefficient"),
    ("2 1 1 2\n1 0 3 1\n1 0 1 1\n", "position out of range"),
    ("2 1 2 2\n1 0 1 1\n1 0 1 1 2 1\n", "pos exp"),
    ("2 1 1 2\n1 0 1 1\n", "expected 2"),
    ("1 1 1 2\n1 0 1 1\n1 0 1 1\n", "trailing"),
    ("1 1 1\n", "header"),
    ("2 1 3 2\n", "k <= n"),
    ("", "missing header"),
]


@pytest.mark.parametrize("text,frag", BAD)
def test_malformed_input_rejected_like_the_reference(text, frag):
    # ref tests/test_io.cpp:69-102
    with pytest.raises(pj.FormatError, match=frag):
        pj.read_system_text(text, "<test>")
    if O.ref_available():
        with pytest.raises(O.RefError, match=frag):
            O.ref_read_system(text)


def test_line_numbers_point_at_the_offender():
    with pytest.raises(pj.FormatError, match="<test>:3"):
        pj.read_system_text("# c\n1 1 1 2\n1 0 1 0\n", "<test>")


def test_missing_file(tmp_path):
    with pytest.raises(pj.FormatError):
        pj.read_system(str(tmp_path / "nope.sys"))


def test_extreme_doubles_and_file_round_trip(tmp_path):
    t = [pj.Term(complex(1.0 / 3.0, -1e-300), pj.MonomialSupport([0], [1]))]
    s = pj.PolynomialSystem.from_terms(1, 1, 1, 1, t)
    path = str(tmp_path / "x.sys")
    pj.write_system(s, path)
    assert same(pj.read_system(path), s)


@needs_ref
def test_parser_agrees_with_the_reference_on_mutated_files():
    """Differential fuzz: random edits of valid files (digits, signs, dots, exponents, comments,
    blank lines, whitespace, truncation) must give the same outcome as the reference's
    read_system — the same system bit for bit, or the same "<name>:<line>: <what>" message."""
    import random
    rng = random.Random(1201)
    alphabet = "0123456789.-+eE x#\n\t"
    bases = [pj.write_system_text(pj.random_system(*shape, 40 + i))
             for i, shape in enumerate([(1, 1, 1, 1), (3, 2, 2, 5), (4, 3, 3, 2)])]
    agree = fails = 0
    for trial in range(3000):
        text = bases[trial % len(bases)]
        for _ in range(rng.randint(1, 3)):
            i = rng.randrange(len(text) + 1)
            op = rng.random()
            if op < 0.4:
                text = text[:i] + rng.choice(alphabet) + text[i:]
            elif op < 0.8:
                text = text[:i] + text[i + 1:]
            elif op < 0.9:
                text = text[:i]
            else:
                text = text[:i] + rng.choice(alphabet) + text[i + 1:]
        try:
            want = O.ref_read_system(text)
            want_err = None
        except O.RefError as e:
            want, want_err = None, str(e)
        try:
            got = pj.read_system_text(text, "<test>")
            got_err = None
        except pj.FormatError as e:
            got, got_err = None, str(e)
        if want_err is not None:
            assert got_err == want_err, (text, want_err, got_err)
            fails += 1
        else:
            assert got_err is None, (text, got_err)
            assert (got.n, got.m, got.k, got.d) == (want["n"], want["m"], want["k"], want["d"])
            assert np.array_equal(got.positions.reshape(-1), want["pos"])
            assert np.array_equal(got.exponents.reshape(-1), want["exps"])
            assert np.array_equal(got.coeffs.view(np.uint64), want["coeffs"].view(np.uint64))
        agree += 1
    assert agree == 3000 and fails > 500
