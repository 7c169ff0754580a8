"""Golden fixtures from the reference (tests/golden/make_golden.py) pin the
oracle (CPU, always) and the GPU path (-m gpu) to the reference's own outputs.

Forward: image / alpha_sum / t_stop (oracle 1e-12; GPU fp64 1e-12, fp32 1e-4),
depth order, per-tile id lists, per-pixel contributor counts, alpha_clamped,
processed_pixels, visibility and floor flags (all bit-exact).
Backward: loss (1e-10 rel) and every parameter gradient (oracle 1e-9 rel,
GPU: SURVEY §8(d) metric).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import ubs_oracle as O
from paper_2510_03312_b200 import synthetic as S
from paper_2510_03312_b200.types import PARAM_FIELDS, Camera, LossConfig, Query, RenderSettings, Scene

from .helpers import grad_close

GOLD = Path(__file__).resolve().parent / "golden"
FWD = sorted(p.stem[4:] for p in GOLD.glob("fwd_*.npz"))
BWD = sorted(p.stem[4:] for p in GOLD.glob("bwd_*.npz"))


def _camera(intr, w2c):
    fx, fy, cx, cy, w, h = intr
    return Camera(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h), world_to_cam=w2c)


def _scene(d):
    return Scene.from_records(int(d["in_n_dims"]), d["in_records"], d["in_background"])


def _settings(d):
    """The fixture's RenderSettings (make_golden.settings_array), default when absent."""
    if "in_settings" not in d:
        return RenderSettings(transmittance_min=float(d["tmin"])) if "tmin" in d else RenderSettings()
    ts, tau, clamp, tmin, near, margin, sfloor, psd, sym = d["in_settings"]
    return RenderSettings(tile_size=int(ts), tau_sq=tau, alpha_clamp=clamp, transmittance_min=tmin, near_plane=near,
                          cull_margin=margin, screen_cov_floor=sfloor, psd_floor_scale=psd, gate_symmetric=bool(sym))


def _fwd_inputs(name):
    d = np.load(GOLD / f"fwd_{name}.npz")
    return d, _scene(d), _camera(d["in_intr"], d["in_w2c"]), Query(d["in_query"]), _settings(d)


def _bwd_inputs(name):
    d = np.load(GOLD / f"bwd_{name}.npz")
    frames = [(_camera(i, w), Query(q), t) for i, w, q, t in zip(d["in_intr"], d["in_w2c"], d["in_query"],
                                                                  d["targets"])]
    ls, lo, lsig, sc = d["cfg"]
    return d, _scene(d), frames, LossConfig(lambda_ssim=ls, lambda_o=lo, lambda_sigma=lsig, loss_scale=sc), \
        _settings(d)


def _tile_lists(d):
    lens = d["tile_lens"]
    return np.concatenate([[0], np.cumsum(lens)]), d["tile_ids"]


def test_fixtures_present():
    assert len(FWD) >= 10 and len(BWD) >= 9


def test_branch_fixtures_engage_their_branches():
    # each round-2 fixture exercises the branch it was made for (make_golden.branch_cases)
    assert _fwd_inputs("gatesym_7")[4].gate_symmetric and _bwd_inputs("grads_7_gatesym")[4].gate_symmetric
    assert np.load(GOLD / "fwd_screenfloor_3.npz")["floored2"].any()
    d, sc, cam, q, st = _fwd_inputs("settings_7")
    assert d["floored2"].any() and d["floored3"].any() and not d["visible"].all()
    assert st.near_plane != RenderSettings().near_plane and st.cull_margin != RenderSettings().cull_margin
    # the jitter rows: singular query blocks that one 1e-8 jitter rescues (covariance.py:143-148)
    d, sc, cam, q, st = _fwd_inputs("jitter_7")
    sl = O.slice_scene(sc, q, st)
    assert sl["valid"].all() and (np.abs(sl["m_inv"][:6]).max() > 1e7)


def test_generators_match_reference_streams():
    g = np.load(GOLD / "generators.npz")
    for nd in (3, 6, 7):
        s = S.random_scene(nd, 7, seed=nd)
        got = np.concatenate([getattr(s, k).reshape(7, -1) for k, _ in PARAM_FIELDS]
                             + [s.background[None].repeat(7, 0)], 1)
        assert np.array_equal(got, g[f"random_scene_{nd}"])
        assert np.array_equal(S.random_query(nd, nd + 1).dims, g[f"random_query_{nd}"])
        i = S.init_scene(nd, 5, seed=nd)
        assert np.array_equal(np.concatenate([getattr(i, k).reshape(5, -1) for k, _ in PARAM_FIELDS], 1),
                              g[f"init_scene_{nd}"])
    for sz, sd in ((32, 8), (128, 2)):
        assert np.abs(S.random_camera(sz, sd).world_to_cam - g[f"random_camera_{sz}_{sd}"]).max() < 1e-15


@pytest.mark.parametrize("name", FWD)
def test_oracle_forward_matches_reference(name):
    d, sc, cam, q, st = _fwd_inputs(name)
    f = O.render_frame(sc, cam, q, st)
    start, ids = _tile_lists(d)
    assert np.array_equal(f["order"], d["order"])
    assert np.array_equal(f["tile_start"], start) and np.array_equal(f["tile_ids"], ids)
    assert np.array_equal(f["count"], d["counts"])
    assert np.array_equal(f["alpha_clamped"], d["alpha_clamped"])
    assert f["processed_pixels"] == int(d["processed_pixels"])
    assert np.array_equal(f["proj"]["visible"], d["visible"])
    assert np.array_equal(f["slices"]["floored"], d["floored3"])
    assert np.array_equal(f["proj"]["floored"], d["floored2"])
    for k in ("image", "alpha_sum", "t_stop"):
        assert np.abs(f[k] - d[k]).max() <= 1e-12


@pytest.mark.parametrize("name", BWD)
def test_oracle_backward_matches_reference(name):
    d, sc, frames, cfg, st = _bwd_inputs(name)
    loss, g = O.backward(sc, frames, cfg, st)
    assert abs(loss - float(d["loss"])) <= 1e-10 * abs(float(d["loss"]))
    for k in O.FIELDS:
        ref = d[f"g_{k}"]
        if ref.size:
            assert np.abs(g[k] - ref).max() <= 1e-9 * max(np.abs(ref).max(), 1e-30), k


# --- the GPU path against the same reference outputs --------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", FWD)
def test_gpu_forward_matches_reference(name, precision):
    from paper_2510_03312_b200 import raster
    d, sc, cam, q, st = _fwd_inputs(name)
    c = raster.render_with_cache(sc, cam, q, st, precision=precision)
    start, ids = _tile_lists(d)
    assert np.array_equal(c.order, d["order"])
    assert np.array_equal(c.tile_ids, ids)
    lens = c.tile_ranges[:, 1] - c.tile_ranges[:, 0]
    assert np.array_equal(lens, d["tile_lens"])
    assert np.array_equal(c.n_contrib, d["counts"])
    assert np.array_equal(c.alpha_clamped, d["alpha_clamped"])
    assert c.processed_pixels == int(d["processed_pixels"])
    tol = 1e-12 if precision == "fp64" else 1e-4
    for k in ("image", "alpha_sum", "t_stop"):
        assert np.abs(getattr(c, k) - d[k]).max() <= tol, k


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", BWD)
def test_gpu_backward_matches_reference(name, precision):
    from paper_2510_03312_b200.gradients import backward
    d, sc, frames, cfg, st = _bwd_inputs(name)
    loss, g = backward(sc, frames, cfg, st, precision=precision)
    assert abs(loss - float(d["loss"])) <= (1e-10 if precision == "fp64" else 1e-5) * abs(float(d["loss"]))
    ref = {k: d[f"g_{k}"] for k in O.FIELDS}
    bad = grad_close(g.arrays(), ref, rel=1e-6 if precision == "fp64" else 1e-3)
    assert not bad, bad


# --- render_decomposition (raster.py:358-423), fixtures from the reference ----
DECOMP = ("decomp_6", "decomp_7")


def _decomp_inputs(name):
    d = np.load(GOLD / f"{name}.npz")
    return d, _scene(d), _camera(d["in_intr"], d["in_w2c"]), Query(d["in_query"])


@pytest.mark.parametrize("name", DECOMP)
def test_oracle_decomposition_matches_reference(name):
    d, sc, cam, q = _decomp_inputs(name)
    for ch in d["channels"]:
        got = O.render_decomposition(sc, cam, q, str(ch), RenderSettings())
        np.testing.assert_allclose(got, d[f"out_{ch}"], rtol=0, atol=1e-12, err_msg=str(ch))


@pytest.mark.gpu
@pytest.mark.parametrize("name", DECOMP)
def test_gpu_decomposition_matches_reference(name):
    from paper_2510_03312_b200 import raster
    d, sc, cam, q = _decomp_inputs(name)
    for ch in d["channels"]:
        got = raster.render_decomposition(sc, cam, q, str(ch), RenderSettings())
        np.testing.assert_allclose(got, d[f"out_{ch}"], rtol=0, atol=1e-12, err_msg=str(ch))


@pytest.mark.gpu
def test_gpu_decomposition_channel_errors():
    from paper_2510_03312_b200 import raster
    d, sc, cam, q = _decomp_inputs("decomp_6")
    with pytest.raises(ValueError, match="only available for 7D"):
        raster.render_decomposition(sc, cam, q, "b_t")
    with pytest.raises(ValueError, match="unknown channel"):
        raster.render_decomposition(sc, cam, q, "beta")
