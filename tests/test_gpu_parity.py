"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Integer outputs (visible set, depth order, per-tile id lists, per-pixel
contributor counts, alpha_clamped flags, processed_pixels) must be
bit-exact.  Images: fp64 path <= 1e-12, fp32 path <= 1e-4 max-abs
(north-star tolerance).  Gradients: SURVEY §8(d) metric (field-norm
relative <= 1e-3 and per-element <= 1e-3|g| + 1e-3 max|g|).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import ubs_oracle as O
from paper_2510_03312_b200 import synthetic as S
from paper_2510_03312_b200.types import DEFAULT_SETTINGS, LossConfig, Query, RenderSettings, Scene, quantize_f32

from .helpers import branch_scene, grad_close, screen_floor_case

pytestmark = pytest.mark.gpu

IMG_TOL = {"fp64": 1e-12, "fp32": 1e-4}


def _render(scene, cam, q, settings, precision):
    from paper_2510_03312_b200 import raster
    return raster.render_with_cache(scene, cam, q, settings, precision=precision)


def assert_frame_parity(scene, cam, q, settings=DEFAULT_SETTINGS, precision="fp32"):
    ref = O.render_frame(scene, cam, q, settings)
    got = _render(scene, cam, q, settings, precision)
    assert np.array_equal(got.order, ref["order"]), "depth order differs"
    st, ids = ref["tile_start"], ref["tile_ids"]
    assert got.tile_ranges.shape[0] == st.size - 1
    lens = got.tile_ranges[:, 1] - got.tile_ranges[:, 0]
    assert np.array_equal(lens, np.diff(st)), "per-tile list lengths differ"
    ne = lens > 0
    assert np.array_equal(got.tile_ranges[ne, 0], st[:-1][ne]), "tile ranges differ"
    assert np.array_equal(got.tile_ids, ids), "per-tile id lists differ"
    assert np.array_equal(got.n_contrib, ref["count"]), \
        f"contributor counts differ at {int((got.n_contrib != ref['count']).sum())} px"
    assert np.array_equal(got.alpha_clamped, ref["alpha_clamped"]), "alpha_clamped differs"
    assert got.processed_pixels == ref["processed_pixels"]
    tol = IMG_TOL[precision]
    assert np.abs(got.image - ref["image"]).max() <= tol
    assert np.abs(got.t_stop - ref["t_stop"]).max() <= tol
    assert np.abs(got.alpha_sum - ref["alpha_sum"]).max() <= tol
    return got, ref


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("nd", [3, 6, 7])
def test_small_scene_parity(nd, precision):
    # reference tests/test_raster.py:155-162 fixtures
    sc = quantize_f32(S.random_scene(nd, 60, seed=nd * 3 + 1))
    cam = S.random_camera(56, nd + 10)
    q = S.random_query(nd, nd + 20)
    assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, precision)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_config1_parity(precision):
    sc = quantize_f32(S.random_scene(7, 10000, seed=1))
    cam = S.random_camera(128, 2)
    q = Query.view_time(0.5, cam.forward)
    assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, precision)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_exact_settings_no_early_out(precision):
    sc = quantize_f32(S.random_scene(6, 200, seed=11))
    cam = S.random_camera(48, 12)
    q = S.random_query(6, 13)
    assert_frame_parity(sc, cam, q, RenderSettings(transmittance_min=0.0), precision)


@pytest.mark.parametrize("tau_sq", [6.5, 4.0])
def test_support_threshold_parity(tau_sq):
    # non-default support thresholds: E, the cover masks and the alpha bound
    # all scale with tau
    sc = quantize_f32(S.random_scene(7, 3000, seed=17))
    cam = S.random_camera(96, 18)
    q = S.random_query(7, 19)
    assert_frame_parity(sc, cam, q, RenderSettings(tau_sq=tau_sq), "fp32")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_branch_coverage_parity(precision):
    sc = branch_scene()
    cam = S.random_camera(96, 3)
    q = S.random_query(7, 4)
    got, ref = assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, precision)
    sl = O.slice_scene(sc, q, DEFAULT_SETTINGS)
    assert sl["floored"].any() and (~sl["valid"]).any() and ref["alpha_clamped"].any()
    assert np.array_equal(got.slices.floored, sl["floored"])
    assert np.array_equal(got.slices.valid, sl["valid"])


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_screen_floor_parity(precision):
    sc, cam, q = screen_floor_case()
    got, ref = assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, precision)
    assert ref["proj"]["floored"].any()
    assert np.array_equal(got.proj.floored, ref["proj"]["floored"])


def test_odd_image_size_parity():
    sc = quantize_f32(S.random_scene(6, 3000, seed=21))
    from paper_2510_03312_b200.types import Camera
    cam = Camera.look_at((2.5, 1.0, 0.8), (0, 0, 0), (0, 0, 1), 0.9, 333, 211)
    q = Query.view(cam.forward)
    assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, "fp32")


def test_intermediates_match_oracle():
    sc = quantize_f32(S.random_scene(7, 500, seed=3))
    cam = S.random_camera(64, 4)
    q = S.random_query(7, 5)
    got = _render(sc, cam, q, DEFAULT_SETTINGS, "fp64")
    sl = O.slice_scene(sc, q, DEFAULT_SETTINGS)
    pr = O.project_scene(sl, cam, DEFAULT_SETTINGS)
    v = pr["visible"]
    assert np.array_equal(got.proj.visible, v)
    for a, b in ((got.proj.mean2, pr["mean2"]), (got.proj.p2, pr["p2"]), (got.proj.depth, pr["depth"]),
                 (got.slices.gated_opacity, sl["gated_opacity"]), (got.slices.mean3, sl["mean3"]),
                 (got.slices.cov3, sl["cov3"])):
        a, b = np.asarray(a)[v], np.asarray(b)[v]
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max())


def test_empty_scene_is_background():
    from paper_2510_03312_b200 import raster
    sc = Scene.empty(6, background=(0.1, 0.5, 0.9))
    img = raster.render(sc, S.random_camera(24, 1), S.random_query(6, 2))
    assert np.abs(img - np.array([0.1, 0.5, 0.9])).max() == 0.0


def test_query_length_mismatch_raises():
    from paper_2510_03312_b200 import raster
    sc = S.random_scene(6, 5, seed=1)
    with pytest.raises(ValueError):
        raster.render(sc, S.random_camera(16, 1), Query.static())


def test_conservation():
    sc = S.random_scene(6, 50, seed=51)
    got = _render(sc, S.random_camera(40, 52), S.random_query(6, 53), DEFAULT_SETTINGS, "fp32")
    assert np.abs(got.alpha_sum + got.t_stop - 1.0).max() <= 1e-5


def test_deterministic_forward():
    sc = S.random_scene(7, 2000, seed=8)
    cam, q = S.random_camera(96, 9), S.random_query(7, 10)
    a = _render(sc, cam, q, DEFAULT_SETTINGS, "fp32")
    b = _render(sc, cam, q, DEFAULT_SETTINGS, "fp32")
    assert np.array_equal(a.image, b.image) and np.array_equal(a.n_contrib, b.n_contrib)


# --- larger sizes: 1080p ------------------------------------------------------

@pytest.mark.slow
@pytest.mark.parametrize("nd,count", [(7, 100_000), (3, 100_000)])
def test_1080p_parity(nd, count):
    sc = S.synth(nd, count, seed=1)
    cam = S.bench_camera()
    q = S.bench_query(nd, cam, 0.5)
    got, _ = assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, "fp32")
    assert got.n_fixed < 0.02 * cam.width * cam.height


@pytest.mark.slow
def test_4k_parity_far_tiles():
    # tiles up to 3840 px from the origin: the fp32 raster's per-tile splat
    # offset (raster.cu tile_offset) and the error bound E that covers it
    sc = S.synth(7, 40_000, seed=5)
    cam = S.bench_camera(3840, 2160)
    q = S.bench_query(7, cam, 0.25)
    got, _ = assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, "fp32")
    assert got.n_fixed < 0.02 * cam.width * cam.height


# --- gradients ----------------------------------------------------------------

def _frames(scene, size, seed, count):
    """random_frames (testing.py:55-69) with oracle-rendered targets."""
    out = []
    for k in range(count):
        cam = S.random_camera(size, seed + 11 * k)
        q = S.random_query(scene.n_dims, seed + 13 * k)
        other = S.random_scene(scene.n_dims, max(2, scene.n_primitives // 2), seed + 977 + k)
        tgt = np.clip(O.render_frame(other, cam, q, DEFAULT_SETTINGS)["image"], 0.0, 1.0)
        out.append((cam, q, tgt))
    return out


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("nd", [3, 6, 7])
def test_backward_parity(nd, precision):
    from paper_2510_03312_b200.gradients import backward
    sc = quantize_f32(S.random_scene(nd, 60, seed=nd + 40))
    frames = _frames(sc, 48, seed=nd + 50, count=2)
    cfg = LossConfig()
    l_ref, g_ref = O.backward(sc, frames, cfg, DEFAULT_SETTINGS)
    l_got, g_got = backward(sc, frames, cfg, DEFAULT_SETTINGS, precision=precision)
    assert abs(l_got - l_ref) <= (1e-10 if precision == "fp64" else 1e-5) * max(1.0, abs(l_ref))
    bad = grad_close(g_got.arrays(), g_ref, rel=1e-6 if precision == "fp64" else 1e-3)
    assert not bad, bad


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_backward_config1(precision):
    from paper_2510_03312_b200.gradients import backward
    sc = quantize_f32(S.random_scene(7, 10000, seed=1))
    cam = S.random_camera(128, 2)
    q = Query.view_time(0.5, cam.forward)
    other = quantize_f32(S.random_scene(7, 5000, seed=978))
    tgt = np.clip(O.render_frame(other, cam, q, DEFAULT_SETTINGS)["image"], 0.0, 1.0)
    frames = [(cam, q, tgt)]
    l_ref, g_ref = O.backward(sc, frames, LossConfig(), DEFAULT_SETTINGS)
    l_got, g_got = backward(sc, frames, LossConfig(), DEFAULT_SETTINGS, precision=precision)
    assert abs(l_got - l_ref) <= 1e-5 * abs(l_ref)
    bad = grad_close(g_got.arrays(), g_ref, rel=1e-6 if precision == "fp64" else 1e-3)
    assert not bad, bad


@pytest.mark.slow
def test_backward_wide_frame():
    # 40 x 23 tiles of a 640x360 view: the fp32 backward's tile-local pixel
    # offsets away from the origin tile (raster.cu tile_offset)
    from paper_2510_03312_b200.gradients import backward
    sc = S.synth(7, 1500, seed=9)
    cam = S.bench_camera(640, 360)
    q = S.bench_query(7, cam, 0.7)
    tgt = np.clip(O.render_frame(S.synth(7, 800, seed=10), cam, q, DEFAULT_SETTINGS)["image"], 0.0, 1.0)
    frames = [(cam, q, tgt)]
    l_ref, g_ref = O.backward(sc, frames, LossConfig(), DEFAULT_SETTINGS)
    l_got, g_got = backward(sc, frames, LossConfig(), DEFAULT_SETTINGS, precision="fp32")
    assert abs(l_got - l_ref) <= 1e-5 * abs(l_ref)
    bad = grad_close(g_got.arrays(), g_ref, rel=1e-3)
    assert not bad, bad


def test_backward_branch_coverage():
    from paper_2510_03312_b200.gradients import backward
    q = S.random_query(7, 70 + 13 * 0)
    sc = branch_scene(seed=6, n=200, query=q)
    sc.s_q_raw[200 // 8 * 3] = 0.0  # keep the degenerate row out: it is skipped, not differentiated
    frames = _frames(sc, 64, seed=70, count=1)
    assert O.slice_scene(sc, frames[0][1], DEFAULT_SETTINGS)["floored"].any()
    l_ref, g_ref = O.backward(sc, frames, LossConfig(), DEFAULT_SETTINGS)
    l_got, g_got = backward(sc, frames, LossConfig(), DEFAULT_SETTINGS, precision="fp64")
    bad = grad_close(g_got.arrays(), g_ref, rel=1e-6)
    assert not bad, bad


def test_gradient_error_on_saturated_gate():
    # tanh saturates -> 0 * inf in the gate adjoint -> GradientError
    from paper_2510_03312_b200.gradients import backward
    from paper_2510_03312_b200.types import GradientError
    sc = S.random_scene(7, 4, seed=2)
    sc.s_q_raw[0, 0] = np.log(0.01)
    sc.l_qx[0] = 0.0
    sc.mu_q[0, 0] = 0.0
    cam = S.random_camera(32, 3)
    q = Query.view_time(0.9, cam.forward)
    tgt = np.zeros((32, 32, 3))
    with pytest.raises(GradientError):
        backward(sc, [(cam, q, tgt)], LossConfig(), DEFAULT_SETTINGS)


def test_binning_large_list_parity():
    # a denser scene at an odd size: sort-free two-level bucketing reproduces
    # build_tiles list for list
    from paper_2510_03312_b200 import raster
    sc = quantize_f32(S.random_scene(7, 20000, seed=17))
    cam = S.random_camera(200, 18)
    q = S.random_query(7, 19)
    got = raster.render_with_cache(sc, cam, q, DEFAULT_SETTINGS, precision="fp32")
    ref = O.render_frame(sc, cam, q, DEFAULT_SETTINGS)
    assert np.array_equal(got.tile_ids, ref["tile_ids"])
    assert np.array_equal(got.n_contrib, ref["count"])


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_depth_ties_broken_by_id(precision):
    # triplicated primitives have bit-identical depths: lexsort breaks the tie
    # by id; the 32-bit-key sort must repair those runs exactly
    base = quantize_f32(S.random_scene(6, 300, seed=23))
    sc = base.take(np.concatenate([np.arange(300)] * 3))
    cam = S.random_camera(96, 24)
    q = S.random_query(6, 25)
    assert_frame_parity(sc, cam, q, DEFAULT_SETTINGS, precision)


def test_async_frames_match_sync():
    # sync=False keeps K on the device; with adequate capacity the frame is identical
    from paper_2510_03312_b200 import engine
    import torch
    sc = quantize_f32(S.random_scene(7, 5000, seed=31))
    cam = S.random_camera(128, 32)
    ws = engine.Workspace("cuda", "fp32")
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    q = S.random_query(7, 33)
    a = engine.render_frame(ws, ds, cam, q, sync=True).image.clone()
    b = engine.render_frame(ws, ds, cam, q, sync=False).image.clone()
    engine.check_status(ws)
    assert torch.equal(a, b)
    # shrink capacity below K: the async frame must flag overflow instead of writing out of bounds
    ws.pair_cap = 16
    engine.render_frame(ws, ds, cam, q, sync=False)
    with pytest.raises(Exception):
        engine.check_status(ws)


def test_capped_tile_lists_match_full():
    # a tiny cap forces truncation: the frame must detect it, grow the cap and
    # re-render to exactly the full-list result
    from paper_2510_03312_b200 import engine
    import torch
    sc = quantize_f32(S.random_scene(7, 4000, seed=41))
    cam = S.random_camera(96, 42)
    q = S.random_query(7, 43)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    full = engine.render_frame(ws, ds, cam, q, full_lists=True)
    ref_img, ref_cnt = full.image.clone(), full.n_contrib.clone()
    ws.list_cap = 4
    capped = engine.render_frame(ws, ds, cam, q)  # sync: grows the cap until no tile runs out
    assert ws.list_cap > 4
    assert torch.equal(capped.n_contrib, ref_cnt) and torch.equal(capped.image, ref_img)
    # asynchronous frame with a cap that is too small: flagged, not silently wrong
    ws.list_cap = 4
    engine.render_frame(ws, ds, cam, q, sync=False)
    with pytest.raises(Exception):
        engine.check_status(ws)


def test_large_frame_uses_global_tile_scan():
    # 4000 x 3600 px = 250 x 225 tiles: the tile-corner grid no longer fits one
    # CTA's shared memory, so the global-memory tile scan runs; lists, order,
    # counts and image must still match the oracle
    sc = quantize_f32(S.synth(3, 3000, seed=41))
    cam = S.bench_camera(4000, 3600)
    assert_frame_parity(sc, cam, Query.static(), DEFAULT_SETTINGS, "fp32")


def test_frame_pipeline_matches_single_stream():
    # frames in flight on separate streams / workspaces give the same bits as
    # one-at-a-time rendering, and the pipeline's status covers every slot
    import torch
    from paper_2510_03312_b200 import engine
    sc = quantize_f32(S.random_scene(7, 4000, seed=61))
    cam = S.random_camera(160, 62)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    qs = [S.random_query(7, 70 + k) for k in range(7)]
    ref = [engine.render_frame(ws, ds, cam, q).image.clone() for q in qs]
    pipe = engine.FramePipeline(ds, depth=3)
    for q in qs * 3:  # 21 synchronous frames: every slot sized by every query
        pipe.render(cam, q, sync=True)
    got = []
    for q in qs:
        fr = pipe.render(cam, q)
        with torch.cuda.stream(pipe.stream_of(fr)):
            got.append(fr.image.clone())
    pipe.join()
    assert pipe.check_status() == 0
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


def test_pipeline_zero_copy_host_sink():
    # the sink reads each slot's image directly; the slot's next frame waits
    # for that copy, so every host image equals the single-stream render
    import torch
    from paper_2510_03312_b200 import engine
    sc = quantize_f32(S.random_scene(6, 3000, seed=71))
    cam = S.random_camera(96, 72)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    qs = [S.random_query(6, 80 + k) for k in range(9)]
    ref = [engine.render_frame(ws, ds, cam, q).image.cpu() for q in qs]
    pipe = engine.FramePipeline(ds, depth=2)
    for q in qs * 2:
        pipe.render(cam, q, sync=True)
    sink = engine.HostFrameSink(96, 96, slots=len(qs))
    outs = []
    for q in qs:
        fr = pipe.render(cam, q)
        outs.append(sink.submit(fr, source_stream=pipe.stream_of(fr)))
        pipe.hold(fr, sink.last_copy)
    pipe.join()
    sink.synchronize()
    for a, b in zip(ref, outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("copy_streams", [1, 3])
def test_grouped_pipeline_zero_copy_host_sink(copy_streams):
    # groups of frames share one preprocess (render_group); the sink reads each
    # slot's image and the slot's next group waits for that copy, so every
    # host image equals the single-stream render (with one or several copy
    # streams: a copy waits only for its own frame)
    import torch
    from paper_2510_03312_b200 import engine
    sc = quantize_f32(S.random_scene(7, 3000, seed=73))
    cam = S.random_camera(96, 74)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    qs = [S.random_query(7, 90 + k) for k in range(11)]
    ref = [engine.render_frame(ws, ds, cam, q).image.cpu() for q in qs]
    pipe = engine.FramePipeline(ds, depth=6)
    for q in qs * 2:
        pipe.render(cam, q, sync=True)
    sink = engine.HostFrameSink(96, 96, slots=len(qs), copy_streams=copy_streams)
    outs = []
    for g0 in range(0, len(qs), 3):  # groups of 3, the last one short
        for fr in pipe.render_group([(cam, q) for q in qs[g0:g0 + 3]]):
            outs.append(sink.submit(fr, source_stream=pipe.stream_of(fr)))
            pipe.hold(fr, sink.last_copy)
    pipe.join()
    sink.synchronize()
    assert pipe.check_status() == 0
    for a, b in zip(ref, outs):
        assert torch.equal(a, b)


def test_pipeline_grow_sizes_every_slot():
    # a frame that needs a larger tile-list cap than its slot has sets
    # UBS_S_LIST_TRUNC; grow() gives every slot the doubled cap, so the same
    # frames re-rendered asynchronously on any slot no longer overflow
    import torch
    from paper_2510_03312_b200 import engine, _lib
    sc = quantize_f32(S.random_scene(7, 4000, seed=81))
    cam = S.random_camera(64, 82)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    qs = [S.random_query(7, 83 + k) for k in range(5)]
    ref = [engine.render_frame(ws, ds, cam, q, RenderSettings(transmittance_min=0.0)).image.clone() for q in qs]
    pipe = engine.FramePipeline(ds, depth=2)
    for w in pipe.workspaces:
        w.list_cap = 8  # far below what these tiles need
    settings = RenderSettings(transmittance_min=0.0)  # no early exit: every list is walked to its end
    for q in qs:
        pipe.render(cam, q, settings, sync=True)  # sizes pair buffers (and grows the caps) slot by slot
    for w in pipe.workspaces:
        w.list_cap = 8
    for q in qs:
        pipe.render(cam, q, settings)
    pipe.join()
    assert int(pipe.status().item()) & _lib.S_LIST_TRUNC
    for _ in range(12):  # the cap doubles per round: 8 -> 32768
        pipe.grow()
        got = []
        for q in qs:
            fr = pipe.render(cam, q, settings)
            with torch.cuda.stream(pipe.stream_of(fr)):
                got.append(fr.image.clone())
        pipe.join()
        if int(pipe.status().item()) == 0:
            break
    assert int(pipe.status().item()) == 0
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


def test_dropin_scene_cache_follows_in_place_edits():
    # the numpy API re-stages the scene every call: editing one element in
    # place (as fd_check does) must show
    from paper_2510_03312_b200 import raster
    sc = quantize_f32(S.random_scene(7, 300, seed=91))
    cam = S.random_camera(48, 92)
    q = S.random_query(7, 93)
    a = raster.render(sc, cam, q)
    assert np.array_equal(raster.render(sc, cam, q), a)  # cache hit: same bits
    sc.color[np.argmax(sc.opacity_raw)] += 0.25           # one primitive, in place
    b = raster.render(sc, cam, q)
    fresh = raster.render(sc.copy(), cam, q)              # new arrays: a fresh upload
    assert not np.array_equal(a, b)
    assert np.array_equal(b, fresh)


def test_render_views_grouped_through_sink():
    # sharding.render_views over a pipeline, 3 frames per shared preprocess,
    # every image streamed to the host sink: equal to frame-by-frame renders
    import torch
    from paper_2510_03312_b200 import engine, sharding
    sc = quantize_f32(S.random_scene(7, 2500, seed=95))
    cam = S.random_camera(80, 96)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    views = [(cam, S.random_query(7, 100 + k)) for k in range(7)]
    ref = [engine.render_frame(ws, ds, c, q).image.cpu() for c, q in views]
    pipe = engine.FramePipeline(ds, depth=6)
    for c, q in views:
        pipe.render(c, q, sync=True)
    sink = engine.HostFrameSink(80, 80, slots=len(views))
    outs = []
    orig = sink.submit

    def keep(fr, source_stream=None):
        outs.append(orig(fr, source_stream=source_stream))
        return outs[-1]
    sink.submit = keep
    n = sharding.render_views(ws, ds, views, sink=sink, pipeline=pipe, frames_per_preprocess=3)
    sink.synchronize()
    assert n == len(views) and pipe.check_status() == 0
    for a, b in zip(ref, outs):
        assert torch.equal(a, b)


def test_dropin_packed_record_scenes():
    # scenes whose fields are views into one record array (UBS1 loading,
    # quantize_f32) upload through the packed fast path: same bits as a scene
    # of separate arrays, and in-place edits through the views still show
    from paper_2510_03312_b200 import raster
    from paper_2510_03312_b200.types import pack_records, Scene
    packed = quantize_f32(S.random_scene(7, 400, seed=97))
    loose = packed.copy()
    assert raster._packed_records(packed, 400) is not None and raster._packed_records(loose, 400) is None
    cam, q = S.random_camera(40, 98), S.random_query(7, 99)
    a = raster.render(packed, cam, q)
    assert np.array_equal(a, raster.render(loose, cam, q))
    packed.opacity_raw[3] += 1.0
    loose.opacity_raw[3] += 1.0
    b = raster.render(packed, cam, q)
    assert np.array_equal(b, raster.render(loose, cam, q)) and not np.array_equal(a, b)


@pytest.mark.parametrize("nd", [3, 6, 7])
def test_framecache_has_every_reference_field(nd):
    # FrameCache.slices / .proj carry every SliceCache / ProjectionCache field
    # (slicing.py:153-182, raster.py:46-60) with the oracle's values;
    # eigenvectors are compared up to sign (LAPACK's convention is arbitrary)
    from dataclasses import fields
    from paper_2510_03312_b200.types import ProjectionCache, SliceCache
    sc = branch_scene(seed=7, n=160) if nd == 7 else quantize_f32(S.random_scene(nd, 160, seed=nd + 90))
    cam = S.random_camera(64, nd + 91)
    q = S.random_query(nd, nd + 92)
    got = _render(sc, cam, q, DEFAULT_SETTINGS, "fp64")
    sl = O.slice_scene(sc, q, DEFAULT_SETTINGS)
    pr = O.project_scene(sl, cam, DEFAULT_SETTINGS)
    ok = sl["valid"]
    for cache, ref, cls in ((got.slices, sl, SliceCache), (got.proj, pr, ProjectionCache)):
        assert isinstance(cache, cls)
        for f in fields(cls):
            a, b = np.asarray(getattr(cache, f.name)), np.asarray(ref[f.name])
            assert a.shape == b.shape, (f.name, a.shape, b.shape)
            if a.dtype == bool:
                assert np.array_equal(a, b), f.name
                continue
            a, b = a[ok], b[ok]
            if b.size == 0:
                continue
            if f.name.endswith("eigvec"):
                # columns up to sign: |V^T V_ref| is the identity where eigenvalues are distinct
                dots = np.abs(np.einsum("nij,nik->njk", a, b))
                lam = ref[f.name.replace("vec", "val")][ok]
                gap = np.min(np.diff(lam, axis=1), axis=1) > 1e-6 * np.abs(lam).max(axis=1)
                eye = np.broadcast_to(np.eye(a.shape[-1]), dots.shape)
                assert np.abs(dots[gap] - eye[gap]).max() <= 1e-8, f.name
                continue
            scale = max(1.0, float(np.abs(b).max()))
            assert np.abs(a - b).max() <= 1e-9 * scale, (f.name, float(np.abs(a - b).max()))


def test_resident_scene_is_reused_until_invalidated():
    # raster.resident(scene): uploaded once, reused by every call on that
    # object (same bits as a fresh upload); in-place edits need invalidate()
    from paper_2510_03312_b200 import raster
    sc = quantize_f32(S.random_scene(7, 300, seed=93))
    cam = S.random_camera(48, 94)
    qs = [S.random_query(7, 95 + k) for k in range(3)]
    ref = [raster.render(sc, cam, q) for q in qs]
    with raster.resident(sc):
        assert all(np.array_equal(raster.render(sc, cam, q), r) for q, r in zip(qs, ref))
        ds = raster._device_scene(sc, raster.workspace())
        assert raster._device_scene(sc, raster.workspace()) is ds
        sc.color[np.argmax(sc.opacity_raw)] += 0.25
        assert np.array_equal(raster.render(sc, cam, qs[0]), ref[0])  # stale until invalidated
        raster.invalidate(sc)
        edited = raster.render(sc, cam, qs[0])
    assert not np.array_equal(edited, ref[0])
    assert np.array_equal(edited, raster.render(sc.copy(), cam, qs[0]))


@pytest.mark.parametrize("nd,count,size", [(7, 20_000, (320, 200)), (6, 3000, (333, 211))])
def test_packed_and_scalar_raster_agree_with_oracle(nd, count, size):
    # the fp32x2 forward (two pixels per lane) and the one-pixel-per-lane forward
    # run the same per-pixel arithmetic: identical counts and clamp flags,
    # images within the fix-up's fp64 re-composites of each other, both = oracle;
    # the packed 4-pixel backward matches the scalar one to float summation order
    import torch
    from paper_2510_03312_b200 import engine
    sc = S.synth(nd, count, seed=nd + 30)
    cam = S.bench_camera(*size)
    q = S.bench_query(nd, cam, 0.6)
    ref = O.render_frame(sc, cam, q, DEFAULT_SETTINGS)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    outs = {}
    for scalar in (False, True):
        ws = engine.Workspace("cuda", "fp32")
        ws.raster_scalar = scalar
        fr = engine.render_frame(ws, ds, cam, q, full_lists=True)
        cnt = fr.n_contrib.cpu().numpy()
        assert np.array_equal(cnt, ref["count"]), scalar
        assert np.array_equal(fr.hit_clamp.cpu().numpy().astype(bool), ref["alpha_clamped"])
        assert float(np.abs(fr.image.double().cpu().numpy() - ref["image"]).max()) <= 1e-4
        g_img = torch.full_like(fr.image, 1e-3)
        grad = torch.zeros(ds.params.shape, dtype=torch.float64, device="cuda")
        gb = engine.backward_raster(fr, ds, g_img, grad, pixels_per_lane=4)
        engine.backward_chain(fr, gb)
        outs[scalar] = grad
    a, b = outs[False], outs[True]
    assert float((a - b).norm()) <= 1e-4 * float(b.norm())
