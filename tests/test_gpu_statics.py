"""Scene statics (ubs_scene_statics): the preprocess that reads the cached
query-invariant half must produce exactly the bits of the preprocess that
derives it inline -- depth keys, tile rects, flags, fp64/fp32 raster records
and the debug dump of intermediates -- for every dimensionality, parameter
precision and the branch-coverage scene (PSD floor, screen floor, degenerate
query blocks, gate saturation)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2510_03312_b200 import engine, synthetic as S
from paper_2510_03312_b200.types import DEFAULT_SETTINGS, Query

from .helpers import branch_scene, screen_floor_case

pytestmark = pytest.mark.gpu


def _prims(scene, cam, q, dtype, precision, use_statics):
    ds = engine.DeviceScene.from_scene(scene, dtype=dtype, device="cuda")
    ds.use_statics = use_statics
    ws = engine.Workspace("cuda", precision)
    engine.render_frame(ws, ds, cam, q, DEFAULT_SETTINGS, want_debug=True, sync=True)
    n = ds.n
    from paper_2510_03312_b200._lib import DEBUG, DEBUG_STRIDE
    dbg = ws.debug[:n * DEBUG_STRIDE].view(n, DEBUG_STRIDE).clone()
    # the query-invariant extras (cov3 eigen pair, l_x, rotation, s_x, s_q) are
    # dumped on the inline route only, and the flags word says which route ran
    dbg[:, DEBUG["cov3_eig"]:DEBUG["cov3_eig"] + 12] = 0
    dbg[:, DEBUG["l_x"]:DEBUG["color"]] = 0
    dbg[:, DEBUG["flags"]] = torch.remainder(dbg[:, DEBUG["flags"]], 16)
    vis = (ws.flags[:n].to(torch.int32) & 1) != 0  # records are written for visible primitives only
    out = {"depth_key": ws.depth_key[:n], "rect": ws.rect[:n], "flags": ws.flags[:n],
           "rec64": ws.rec64[:n * 10].view(n, 10)[vis], "debug": dbg}
    if ws.rec32 is not None:
        out["rec32"] = ws.rec32[:n * 16].view(n, 16)[vis]
    return {k: v.clone().cpu() for k, v in out.items()}, ws


def _cases():
    out = []
    for nd in (3, 6, 7):
        sc = S.synth(nd, 3000, seed=11 + nd)
        cam = S.bench_camera(320, 240)
        out.append((f"synth{nd}", sc, cam, S.bench_query(nd, cam, 0.3)))
    sc = branch_scene(seed=5, n=400)
    cam = S.bench_camera(256, 192)
    out.append(("branch", sc, cam, S.bench_query(7, cam, 0.5)))
    sc, cam = screen_floor_case()[:2]
    out.append(("screen_floor", sc, cam, Query.static()))
    return out


@pytest.mark.parametrize("precision,dtype", [("fp32", torch.float32), ("fp64", torch.float64),
                                             ("fp32", torch.float64)])
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_statics_route_is_bit_identical(case, precision, dtype):
    _, sc, cam, q = case
    a, _ = _prims(sc, cam, q, dtype, precision, use_statics=False)
    b, _ = _prims(sc, cam, q, dtype, precision, use_statics=True)
    for k in a:
        x, y = a[k], b[k]
        if x.dtype.is_floating_point:
            x, y = x.view(torch.int32 if x.dtype == torch.float32 else torch.int64), \
                y.view(torch.int32 if y.dtype == torch.float32 else torch.int64)
        assert torch.equal(x, y), f"{k} differs between the statics and inline preprocess"


def test_statics_follow_parameter_updates():
    """In-place parameter writes (torch ops or DeviceAdam's ctypes update,
    which bumps the version counter) invalidate the cached statics."""
    from paper_2510_03312_b200.sharding import DeviceAdam
    sc = S.synth(7, 2000, seed=3)
    cam = S.bench_camera(320, 240)
    q = S.bench_query(7, cam, 0.5)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    engine.render_frame(ws, ds, cam, q, sync=True)
    k0 = ds._statics_key
    opt = DeviceAdam(ds.params, 7)
    g = torch.randn(ds.params.shape, device="cuda")
    opt.step(g)
    engine.render_frame(ws, ds, cam, q, want_debug=True, sync=True)
    assert ds._statics_key != k0
    ref = engine.DeviceScene(ds.params.clone(), 7, sc.background, use_statics=False)
    ws2 = engine.Workspace("cuda", "fp32")
    engine.render_frame(ws2, ref, cam, q, want_debug=True, sync=True)
    # the first 32 columns of every row come from either route (rows are DEBUG_STRIDE wide)
    from paper_2510_03312_b200._lib import DEBUG_STRIDE
    a = ws.debug[:ds.n * DEBUG_STRIDE].view(ds.n, DEBUG_STRIDE)[:, :32]
    b = ws2.debug[:ds.n * DEBUG_STRIDE].view(ds.n, DEBUG_STRIDE)[:, :32]
    assert torch.equal(a.contiguous().view(torch.int64), b.contiguous().view(torch.int64))
    ds.params.mul_(1.0)  # torch in-place op: version bump
    assert ds.statics_ptr(DEFAULT_SETTINGS) and ds._statics_key[1] == ds.params._version


@pytest.mark.parametrize("precision,dtype", [("fp32", torch.float32), ("fp64", torch.float32),
                                             ("fp64", torch.float64)])
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_preprocess_views_matches_per_view(case, precision, dtype):
    """ubs_preprocess_views (one statics read for a group of frames) gives
    every frame exactly the bits of its own ubs_preprocess: per-primitive
    outputs, counters and the rendered frame.  10 views: two launches."""
    _, sc, cam, q = case
    ds = engine.DeviceScene.from_scene(sc, dtype=dtype, device="cuda")
    nd = sc.n_dims
    views = [(cam, q)]  # the case's own view, then an orbit with a time sweep
    for k in range(1, 10):
        c = S.bench_camera(cam.width, cam.height, k, 10)
        views.append((c, S.bench_query(nd, c, k / 9.0)))
    pipe = engine.FramePipeline(ds, depth=10, precision=precision)
    frames = pipe.render_group(views)
    pipe.join()
    torch.cuda.synchronize()
    pipe.check_status()
    ref_ws = engine.Workspace("cuda", precision)
    n = ds.n
    for (c, qq), fr in zip(views, frames):
        want = engine.render_frame(ref_ws, ds, c, qq, sync=True)
        ws = fr.ws
        for name in ("depth_key", "rect", "flags", "tile_count"):
            assert torch.equal(getattr(ws, name)[:n], getattr(ref_ws, name)[:n]), name
        vis = (ws.flags[:n].to(torch.int32) & 1) != 0  # records of visible primitives only
        assert torch.equal(ws.rec64[:n * 10].view(torch.int64).view(n, 10)[vis],
                           ref_ws.rec64[:n * 10].view(torch.int64).view(n, 10)[vis])
        if ws.rec32 is not None:
            assert torch.equal(ws.rec32[:n * 16].view(torch.int32).view(n, 16)[vis],
                               ref_ws.rec32[:n * 16].view(torch.int32).view(n, 16)[vis])
        assert torch.equal(ws.counters[:3], ref_ws.counters[:3])
        assert torch.equal(fr.n_contrib, want.n_contrib)
        assert torch.equal(fr.image, want.image)


def test_preprocess_views_rejects_mixed_scenes():
    """ubs_preprocess_views serves views of ONE scene: a view of another
    scene, a view without statics and an empty group are argument errors."""
    from paper_2510_03312_b200 import _lib
    lib = _lib.load()
    a = engine.DeviceScene.from_scene(S.synth(7, 500, seed=1), device="cuda")
    b = engine.DeviceScene.from_scene(S.synth(7, 500, seed=2), device="cuda")
    cam = S.bench_camera(64, 48)
    q = S.bench_query(7, cam, 0.5)
    wss = [engine.Workspace("cuda", "fp32") for _ in range(2)]
    s = torch.cuda.current_stream().cuda_stream

    def call(scenes):
        vs, pbs = [], []
        for ds, ws in zip(scenes, wss):
            v, pb = engine._frame_begin(ws, ds, cam, q, DEFAULT_SETTINGS, False)
            vs.append(v)
            pbs.append(pb)
        return lib.ubs_preprocess_views((_lib.UbsView * len(vs))(*vs), (_lib.UbsPrimBuffers * len(pbs))(*pbs),
                                        len(vs), 1, s)

    assert call([a, a]) == 0
    assert call([a, b]) == _lib.UBS_E_ARGS
    a.use_statics = False
    assert call([a, a]) == _lib.UBS_E_ARGS
    assert lib.ubs_preprocess_views(None, None, 0, 1, s) == _lib.UBS_E_ARGS
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_device_scene_upload_matches_pack_records(dtype):
    """DeviceScene.from_scene (fields uploaded and cast on the device) holds
    exactly pack_records' host-side records."""
    from paper_2510_03312_b200.types import pack_records
    sc = S.random_scene(7, 3000, seed=17)
    ds = engine.DeviceScene.from_scene(sc, dtype=dtype, device="cuda")
    want = torch.from_numpy(pack_records(sc, np.float64 if dtype == torch.float64 else np.float32))
    assert torch.equal(ds.params.cpu(), want)


def test_render_group_mixed_resolutions():
    """One group may mix image sizes (each view its own tile grid and
    buffers): every frame equals its own single-view render bit for bit."""
    sc = S.synth(7, 4000, seed=21)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    sizes = [(64, 48), (33, 17), (100, 70), (16, 16)]
    views = []
    for k, (w, h) in enumerate(sizes):
        cam = S.bench_camera(w, h, k, len(sizes))
        views.append((cam, S.bench_query(7, cam, k / 3.0)))
    pipe = engine.FramePipeline(ds, depth=4)
    for cam, q in views:  # size every slot for every view
        for _ in range(4):
            pipe.render(cam, q, sync=True)
    frames = pipe.render_group(views)
    pipe.join()
    torch.cuda.synchronize()
    assert pipe.check_status() == 0
    ref_ws = engine.Workspace("cuda", "fp32")
    for (cam, q), fr in zip(views, frames):
        want = engine.render_frame(ref_ws, ds, cam, q, sync=True)
        assert fr.image.shape == want.image.shape
        assert torch.equal(fr.image, want.image) and torch.equal(fr.n_contrib, want.n_contrib)


def test_preprocess_views_at_scale():
    """2M primitives (15.6k statics blocks, 700 MB of statics): the grouped
    preprocess matches per-view preprocess bit for bit on every output."""
    nd = 7
    ds = engine.DeviceScene.from_scene(S.synth(nd, 2_000_000, seed=31), device="cuda")
    views = []
    for k in range(4):
        cam = S.bench_camera(320, 180, k, 4)
        views.append((cam, S.bench_query(nd, cam, k / 3.0)))
    pipe = engine.FramePipeline(ds, depth=4)
    for cam, q in views:
        for _ in range(4):
            pipe.render(cam, q, sync=True)
    frames = pipe.render_group(views)
    pipe.join()
    torch.cuda.synchronize()
    assert pipe.check_status() == 0
    ref_ws = engine.Workspace("cuda", "fp32")
    n = ds.n
    for (cam, q), fr in zip(views, frames):
        want = engine.render_frame(ref_ws, ds, cam, q, sync=True)
        ws = fr.ws
        for name in ("depth_key", "rect", "flags", "tile_count"):
            assert torch.equal(getattr(ws, name)[:n], getattr(ref_ws, name)[:n]), name
        vis = (ws.flags[:n].to(torch.int32) & 1) != 0
        assert torch.equal(ws.rec32[:n * 16].view(torch.int32).view(n, 16)[vis],
                           ref_ws.rec32[:n * 16].view(torch.int32).view(n, 16)[vis])
        assert torch.equal(fr.image, want.image) and torch.equal(fr.n_contrib, want.n_contrib)
