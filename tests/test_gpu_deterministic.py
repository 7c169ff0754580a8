"""Deterministic backward (UbsGradBuffers.deterministic; reference
raster.py:1-8, gradients.py:164-173, tests/test_raster.py:174-180): per-
(primitive, tile) partials reduced in a fixed order instead of float
atomics.  Two runs give bit-identical gradients and loss, and the values
still match the oracle (SURVEY §8(d) metric)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import ubs_oracle as O
from paper_2510_03312_b200 import synthetic as S
from paper_2510_03312_b200.types import DEFAULT_SETTINGS, LossConfig

from .helpers import grad_close

pytestmark = pytest.mark.gpu


def _frames(scene, w, h, count, seed):
    out = []
    for k in range(count):
        cam = S.bench_camera(w, h, k, count)
        q = S.bench_query(scene.n_dims, cam, 0.3 + 0.2 * k)
        other = S.synth(scene.n_dims, max(2, scene.n_primitives // 3), seed=seed + k)
        out.append((cam, q, np.clip(O.render_frame(other, cam, q, DEFAULT_SETTINGS)["image"], 0.0, 1.0)))
    return out


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("nd", [3, 7])
def test_deterministic_backward_is_bitwise_repeatable(nd, precision):
    from paper_2510_03312_b200.gradients import backward
    sc = S.synth(nd, 20_000, seed=7)
    frames = _frames(sc, 320, 192, 2, seed=70)
    cfg = LossConfig()
    runs = [backward(sc, frames, cfg, DEFAULT_SETTINGS, precision=precision, deterministic=True) for _ in range(3)]
    l0, g0 = runs[0]
    for l, g in runs[1:]:
        assert l == l0
        for k, a in g.arrays().items():
            assert np.array_equal(a, g0.arrays()[k]), k
    l_ref, g_ref = O.backward(sc, frames, cfg, DEFAULT_SETTINGS)
    assert abs(l0 - l_ref) <= (1e-10 if precision == "fp64" else 1e-5) * abs(l_ref)
    bad = grad_close(g0.arrays(), g_ref, rel=1e-6 if precision == "fp64" else 1e-3)
    assert not bad, bad
    # the atomic path computes the same sums up to their order
    l_a, g_a = backward(sc, frames, cfg, DEFAULT_SETTINGS, precision=precision)
    bad = grad_close(g_a.arrays(), g0.arrays(), rel=1e-9 if precision == "fp64" else 1e-4, floor=1e-6)
    assert not bad, bad
