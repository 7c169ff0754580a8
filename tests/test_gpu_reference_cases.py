"""The reference's own render-level test cases (pkg/tests/test_raster.py,
TestProjection / TestRender / TestDecomposition), restated against this
package's drop-in entry points on the GPU: projection landmarks, culling,
the clamp at a splat centre, view independence, the early-exit error bound,
occlusion order and the decomposition's properties."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2510_03312_b200 import synthetic as S
from paper_2510_03312_b200.types import Camera, Query, RenderSettings, Scene, logit

pytestmark = pytest.mark.gpu

EXACT = RenderSettings(transmittance_min=0.0)
TOL = {"fp64": 1e-12, "fp32": 1e-6}


def _r():
    from paper_2510_03312_b200 import raster
    return raster


def axis_camera(fx=100.0, size=100, c=None):
    c = size / 2.0 if c is None else c
    return Camera(fx=fx, fy=fx, cx=c, cy=c, width=size, height=size, world_to_cam=np.eye(4))


def point_scene(mu, s=0.1, opacity_raw=2.0, color=(1.0, 0.0, 0.0), background=(0.0, 0.0, 0.0)):
    mu = np.atleast_2d(np.asarray(mu, dtype=np.float64))
    n = mu.shape[0]
    s = np.broadcast_to(np.atleast_1d(np.asarray(s, dtype=np.float64)), (n,))
    return Scene(n_dims=3, mu_x=mu, mu_q=np.zeros((n, 0)), rot=np.zeros((n, 3)),
                 s_x_raw=np.log(s)[:, None] * np.ones((n, 3)), l_qx=np.zeros((n, 0, 3)),
                 s_q_raw=np.zeros((n, 0)), b_x=np.zeros(n), b_q=np.zeros((n, 0)),
                 opacity_raw=np.full(n, opacity_raw, dtype=np.float64),
                 color=np.tile(np.asarray(color, dtype=np.float64), (n, 1)),
                 background=np.asarray(background, dtype=np.float64))


def test_optical_axis_center():
    c = _r().render_with_cache(point_scene([0, 0, 1.0]), axis_camera(), Query.static(), precision="fp64")
    assert np.abs(c.proj.mean2[0] - 50.0).max() < 1e-12
    assert c.proj.depth[0] == pytest.approx(1.0)


def test_isotropic_cov_maps_to_scaled_identity():
    f, z, sig = 80.0, 2.0, 0.05
    c = _r().render_with_cache(point_scene([0, 0, z], s=sig), axis_camera(fx=f), Query.static(), precision="fp64")
    assert np.abs(c.proj.cov2[0] - (f * sig / z) ** 2 * np.eye(2)).max() < 1e-9


def test_behind_camera_and_offscreen_culled():
    c = _r().render_with_cache(point_scene([[0, 0, -1.0], [100.0, 0, 1.0], [0, 0, 1.0]]), axis_camera(),
                               Query.static())
    assert list(c.proj.visible) == [False, False, True]


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_single_opaque_splat_clamps_at_its_centre(precision):
    # mean on a pixel centre: m = 0, alpha = og > 0.999 -> clamped to 0.999
    sc = point_scene([0, 0, 1.0], s=0.05, opacity_raw=30.0)
    cam = axis_camera(size=33, c=16.5)
    c = _r().render_with_cache(sc, cam, Query.static(), EXACT, precision=precision)
    assert np.abs(c.image[16, 16] - [0.999, 0.0, 0.0]).max() < TOL[precision]
    assert c.alpha_clamped[0]


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_view_independent_construction(precision):
    sc = S.random_scene(6, 12, seed=3)
    sc.l_qx[:] = 0.0
    sc.b_q[:] = -5.0
    sc.s_q_raw[:] = np.log(1000.0)
    cam = S.random_camera(48, 4)
    a = _r().render(sc, cam, Query.view([1.0, 0.2, 0.1]), precision=precision)
    b = _r().render(sc, cam, Query.view([-0.5, 0.8, -0.2]), precision=precision)
    assert np.abs(a - b).max() <= 1e-6


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_early_exit_error_bounded(precision):
    sc = S.random_scene(6, 150, seed=31)
    sc.opacity_raw[:] = logit(0.97)
    cam, q = S.random_camera(48, 32), S.random_query(6, 33)
    exact = _r().render(sc, cam, q, EXACT, precision=precision)
    fast = _r().render(sc, cam, q, RenderSettings(transmittance_min=1e-4), precision=precision)
    err = np.abs(exact - fast).max()
    assert 0.0 < err <= 2e-4


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_occlusion_order(precision):
    cam = axis_camera(fx=60.0, size=32)
    sc = point_scene([[0.0, 0.0, 1.0], [0.0, 0.0, 2.0]], s=0.2, opacity_raw=12.0)
    sc.color = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    img = _r().render(sc, cam, Query.static(), precision=precision)
    assert img[16, 16, 0] > 0.9 and img[16, 16, 1] < 0.1
    sc2 = sc.copy()
    sc2.mu_x, sc2.color = sc.mu_x[::-1].copy(), sc.color[::-1].copy()
    assert np.abs(_r().render(sc2, cam, Query.static(), precision=precision) - img).max() < 1e-12
    sc3 = sc.copy()
    sc3.mu_x = np.array([[0.0, 0.0, 2.0], [0.0, 0.0, 1.0]])
    img3 = _r().render(sc3, cam, Query.static(), precision=precision)
    assert img3[16, 16, 1] > 0.9 and img3[16, 16, 0] < 0.1


def test_decomposition_constant_channel_constant_hue():
    sc = S.random_scene(6, 10, seed=61)
    sc.b_x[:] = 1.5
    cam, q = S.random_camera(40, 62), S.random_query(6, 63)
    cache = _r().render_with_cache(sc, cam, q, precision="fp64")
    heat = _r().render_decomposition(sc, cam, q, "b_x")
    covered = cache.alpha_sum > 1e-9
    assert covered.any()
    assert np.abs(heat[covered] - heat[covered][0]).max() < 1e-9


def test_decomposition_temporal_separation():
    sc = S.random_scene(7, 2, seed=64)
    sc.mu_x = np.array([[-0.6, 0.0, 0.0], [0.6, 0.0, 0.0]])
    sc.l_qx[:] = 0.0
    sc.s_q_raw[:] = np.log(50.0)
    sc.b_q[:, 0] = [-5.0, 5.0]
    sc.opacity_raw[:] = 6.0
    cam = Camera.look_at((0, 0, -3.0), (0, 0, 0), (0, 1, 0), 0.9, 48, 48)
    q = Query.view_time(0.0, cam.forward)
    cache = _r().render_with_cache(sc, cam, q, precision="fp64")
    heat = _r().render_decomposition(sc, cam, q, "b_t")
    covered = cache.alpha_sum > 0.2
    reds, blues = heat[..., 0][covered], heat[..., 2][covered]
    assert (reds > blues).any() and (blues > reds).any()


def test_decomposition_empty_scene():
    sc = Scene.empty(7, background=(0.3, 0.3, 0.3))
    heat = _r().render_decomposition(sc, S.random_camera(24, 65), S.random_query(7, 66), "b_t")
    assert np.abs(heat - 0.3).max() == 0.0


def test_decomposition_weights_match_render():
    sc = S.random_scene(6, 6, seed=74)
    sc.b_x[:] = 0.0
    cam, q = S.random_camera(32, 75), S.random_query(6, 76)
    heat = _r().render_decomposition(sc, cam, q, "b_x")
    cache = _r().render_with_cache(sc, cam, q, precision="fp64")
    # every pixel any alpha reached (here one has alpha_sum = 1.8e-15, in the
    # oracle too) takes the colormap value; untouched pixels the background
    covered = cache.alpha_sum > 0.0
    assert np.abs(heat[covered] - np.array([0.95, 0.95, 0.95])).max() < 1e-9
    assert np.abs(heat[~covered] - sc.background).max() < 1e-12
