"""Warp-specialised fast dd kernel (csrc/eval_fast_ws.cu, kernel variant 3, opt-in): producer
warps run stages 1-2, consumer warps stage 3, joined by a ring of staging buffers with round
counters. Same per-element operation sequence as the fused kernel (variant 1), so the two must
agree bit for bit; the fused kernel's contract (tests/test_gpu_parity.py) then carries over.
Covers several k, n = 64 (plane stride 64), m < 32 (shadow lanes), batches that leave partial
tiles, and a batch large enough that every buffer is reused many rounds."""
import numpy as np
import pytest

import paper_1201_0499_b200 as pj


@pytest.mark.gpu
@pytest.mark.parametrize("shape,B", [((32, 32, 8, 2), 65536), ((32, 32, 8, 2), 7), ((20, 17, 5, 2), 999),
                                     ((64, 32, 12, 2), 300), ((9, 30, 2, 1), 257), ((40, 32, 3, 2), 1)])
def test_ws_bit_identical_with_fused(shape, B, gpu):
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 31 + k)
    z = pj.random_points(n, B, 32)
    pdd = pj.to_dd(z)
    pdd[..., 1] = pdd[..., 0] * 2.0 ** -58
    pdd[..., 3] = -pdd[..., 2] * 2.0 ** -56
    a = pj.EvaluationContext(s)
    a.set_variant(1, "dd")
    want = a.evaluate_dd(pdd)
    b = pj.EvaluationContext(s)
    b.set_variant(3, "dd")
    assert b.launch("dd")["variant"] == 3
    got = b.evaluate_dd(pdd)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
def test_ws_rejects_unsupported_shapes(gpu):
    for shape in [(32, 40, 8, 2), (32, 32, 8, 3), (80, 32, 8, 2), (32, 32, 13, 2)]:  # m, d, n, k out of range
        ctx = pj.EvaluationContext(pj.random_system(*shape, 1))
        with pytest.raises(ValueError, match="warp-specialised"):
            ctx.set_variant(3, "dd")
        with pytest.raises(ValueError):
            ctx.set_variant(3, "d")
