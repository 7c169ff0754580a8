"""Host-side contract: types mirror the reference's validation and layout."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2510_03312_b200 import synthetic as S
from paper_2510_03312_b200.types import (Camera, GradientError, Query, RenderSettings, Scene, SceneGrads,
                                         field_offsets, pack_records, quantize_f32, record_width)


def test_record_width_and_offsets():
    assert [record_width(n) for n in (3, 6, 7)] == [14, 32, 38]
    off = field_offsets(7)
    assert off["mu_x"][0] == 0 and off["color"] == (35, 3, (3,)) and off["l_qx"] == (13, 12, (4, 3))


def test_pack_roundtrip():
    sc = S.random_scene(7, 9, seed=3)
    rec = pack_records(sc, np.float64)
    back = Scene.from_records(7, rec, sc.background)
    for k in ("mu_x", "l_qx", "b_q", "color", "opacity_raw"):
        assert np.array_equal(getattr(back, k), getattr(sc, k))
    q = quantize_f32(sc)
    assert np.array_equal(q.mu_x, sc.mu_x.astype(np.float32).astype(np.float64))


def test_scene_validation():
    with pytest.raises(ValueError):
        Scene.empty(5)
    assert Scene.empty(7).n_primitives == 0


def test_query_validation():
    assert Query.static().dims.shape == (0,)
    assert Query.view([2.0, 0.0, 0.0]).dims.shape == (3,)
    assert Query.view_time(0.5, [0, 0, 1]).dims.shape == (4,)
    with pytest.raises(ValueError):
        Query(np.array([0.5, 0.5, 0.5]))
    with pytest.raises(ValueError):
        Query.view_time(1.5, [0, 0, 1.0])
    with pytest.raises(ValueError):
        Query(np.array([0.1, 0.2]))


def test_camera_look_at_and_forward():
    cam = Camera.look_at((3.0, 0.0, 0.0), (0, 0, 0), (0, 0, 1), 0.9, 64, 48)
    assert np.allclose(cam.forward, [-1.0, 0.0, 0.0])
    assert np.allclose(cam.position, [3.0, 0.0, 0.0])
    with pytest.raises(ValueError):
        Camera(fx=-1, fy=1, cx=0, cy=0, width=4, height=4, world_to_cam=np.eye(4))


def test_scenegrads_check_finite_names_field_and_primitive():
    sc = S.random_scene(6, 4, seed=1)
    g = SceneGrads.zeros_like(sc)
    g.mu_q[2, 1] = np.nan
    with pytest.raises(GradientError, match="'mu_q' of primitive 2"):
        g.check_finite()


def test_render_settings_defaults_are_reference_values():
    s = RenderSettings()
    assert (s.tile_size, s.tau_sq, s.alpha_clamp, s.transmittance_min, s.near_plane, s.cull_margin,
            s.screen_cov_floor, s.psd_floor_scale, s.gate_symmetric) == (16, 8.0, 0.999, 1e-4, 0.01, 3.0, 1e-6,
                                                                         1e-8, False)


def test_synth_is_float32_exact():
    sc = S.synth(7, 1000, seed=1)
    rec = pack_records(sc, np.float64)
    assert np.array_equal(rec, rec.astype(np.float32).astype(np.float64))
    assert np.all(sc.b_q >= -1) and np.all(sc.b_q <= 1)


def test_pinned_handout_counter_follows_the_arrays():
    """The drop-in hands images / gradients out in pinned blocks and counts
    the live ones (raster._PINNED_OUT, bounded by _PINNED_OUT_MAX): the count
    must drop only when the last array viewing a block is gone (the finalizer
    sits on the tensor alias the ndarray holds, not on the allocating tensor)."""
    import gc
    import weakref
    import torch
    from paper_2510_03312_b200 import raster
    before = raster._PINNED_OUT[0]
    t = torch.zeros(64, dtype=torch.float64)  # stands in for the pinned block
    out = t.numpy()
    raster._PINNED_OUT[0] += 1
    weakref.finalize(out.base, raster._pinned_out_released)
    view = out[8:16].reshape(2, 4)
    del t, out
    gc.collect()
    assert raster._PINNED_OUT[0] == before + 1  # the view keeps the block
    del view
    gc.collect()
    assert raster._PINNED_OUT[0] == before
