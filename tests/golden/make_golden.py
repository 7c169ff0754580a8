"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container, which has /root/reference (it does not exist on
the GPU box; the fixtures travel as committed .npz files):

    NUMBA_CACHE_DIR=/tmp/ubs_numba python tests/golden/make_golden.py [--decomposition | --branches]

Each case records the reference's own outputs (betasplat.raster.render_with_cache
and betasplat.gradients.backward) on seeded fixture scenes, plus checksums of
its fixture generators (testing.random_scene / random_camera / random_query,
scene.init_scene) so tests/test_golden.py can pin both the oracle and this
package's generators.  Per-pixel contributor counts are not exposed by the
reference; they are produced by running the reference's own numba
tile_forward one pixel at a time (a one-pixel tile's return value is that
pixel's count).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ubs_numba")
sys.path.insert(0, "/root/reference/pkg/src")

import betasplat as bs  # noqa: E402
from betasplat import gradients as G, raster as R, scene as SC, testing as T  # noqa: E402

OUT = Path(__file__).resolve().parent


def f32(scene):
    rec = np.concatenate([getattr(scene, k).reshape(scene.n_primitives, -1) for k, _ in SC.PARAM_FIELDS], 1)
    rec = rec.astype(np.float32).astype(np.float64)
    off = 0
    kw = {}
    c = scene.n_dims - 3
    for k, fn in SC.PARAM_FIELDS:
        shape = fn(c)
        size = int(np.prod(shape)) if shape else 1
        kw[k] = rec[:, off:off + size].reshape((scene.n_primitives,) + shape)
        off += size
    return SC.Scene(n_dims=scene.n_dims, background=scene.background, **kw)


def pixel_counts(cache):
    """Per-pixel contributor counts from the reference's numba tile_forward."""
    from betasplat._tiles import tile_forward
    cam, st, pr, sl, sc = cache.camera, cache.settings, cache.proj, cache.slices, cache.scene
    H, W = cam.height, cam.width
    counts = np.zeros((H, W), dtype=np.int64)
    for (y0, y1, x0, x1, idx) in cache.tiles:
        if idx.size == 0:
            continue
        for y in range(y0, y1):
            for x in range(x0, x1):
                rgb, a, t = np.empty((1, 3)), np.empty(1), np.empty(1)
                hit = np.zeros(idx.size, dtype=bool)
                counts[y, x] = tile_forward(np.array([x + 0.5]), np.array([y + 0.5]), pr.mean2[idx], pr.p2[idx],
                                            sl.gated_opacity[idx], sl.beta_x[idx], sc.color[idx], sc.background,
                                            st.tau_sq, st.alpha_clamp, st.transmittance_min, rgb, a, t, hit)
    return counts


def flat_tiles(cache):
    lens = np.array([t[4].size for t in cache.tiles], dtype=np.int64)
    ids = np.concatenate([t[4] for t in cache.tiles]) if lens.sum() else np.zeros(0, np.int64)
    return lens, ids.astype(np.int64)


def records(scene):
    return np.concatenate([getattr(scene, k).reshape(scene.n_primitives, -1) for k, _ in SC.PARAM_FIELDS], 1)


def cam_arrays(cam):
    return np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height], dtype=np.float64), cam.world_to_cam


def settings_array(st):
    """RenderSettings as stored in the fixtures (tests/test_golden.py reads it back)."""
    return np.array([st.tile_size, st.tau_sq, st.alpha_clamp, st.transmittance_min, st.near_plane, st.cull_margin,
                     st.screen_cov_floor, st.psd_floor_scale, float(st.gate_symmetric)], dtype=np.float64)


def forward_case(name, scene, cam, q, settings):
    c = R.render_with_cache(scene, cam, q, settings)
    lens, ids = flat_tiles(c)
    intr, w2c = cam_arrays(cam)
    np.savez_compressed(OUT / f"fwd_{name}.npz", in_records=records(scene), in_n_dims=scene.n_dims,
                        in_background=scene.background, in_intr=intr, in_w2c=w2c, in_query=q.dims,
                        image=c.image, alpha_sum=c.alpha_sum, t_stop=c.t_stop,
                        order=c.order, tile_lens=lens, tile_ids=ids, alpha_clamped=c.alpha_clamped,
                        processed_pixels=c.processed_pixels, counts=pixel_counts(c),
                        visible=c.proj.visible, floored3=c.slices.floored, floored2=c.proj.floored,
                        mean2=c.proj.mean2, depth=c.proj.depth, gated_opacity=c.slices.gated_opacity,
                        tmin=settings.transmittance_min, in_settings=settings_array(settings),
                        floored2_any=bool(c.proj.floored.any()))
    print("fwd", name, c.image.shape, int(lens.sum()), c.processed_pixels, "visible", int(c.proj.visible.sum()),
          "floor3", int(c.slices.floored.sum()), "floor2", int(c.proj.floored.sum()),
          "degenerate", int((~c.slices.valid).sum()), "clamped", int(c.alpha_clamped.sum()))
    return c


def backward_case(name, scene, frames, cfg, settings=None):
    settings = settings or bs.RenderSettings()
    loss, g = G.backward(scene, frames, cfg, settings)
    np.savez_compressed(OUT / f"bwd_{name}.npz", loss=loss, in_records=records(scene), in_n_dims=scene.n_dims,
                        in_background=scene.background,
                        in_intr=np.stack([cam_arrays(f[0])[0] for f in frames]),
                        in_w2c=np.stack([f[0].world_to_cam for f in frames]),
                        in_query=np.stack([f[1].dims for f in frames]),
                        cfg=np.array([cfg.lambda_ssim, cfg.lambda_o, cfg.lambda_sigma, cfg.loss_scale]),
                        targets=np.stack([f[2] for f in frames]), in_settings=settings_array(settings),
                        **{f"g_{k}": v for k, v in g.arrays().items()})
    print("bwd", name, loss)


def main():
    st = bs.RenderSettings()
    exact = bs.RenderSettings(transmittance_min=0.0)
    # generator checksums (testing.py:12-52, scene.py:181-227)
    gens = {}
    for nd in (3, 6, 7):
        s = T.random_scene(nd, 7, seed=nd)
        gens[f"random_scene_{nd}"] = np.concatenate(
            [getattr(s, k).reshape(7, -1) for k, _ in SC.PARAM_FIELDS] + [s.background[None].repeat(7, 0)], 1)
        gens[f"random_query_{nd}"] = T.random_query(nd, nd + 1).dims
        i = SC.init_scene(nd, 5, seed=nd)
        gens[f"init_scene_{nd}"] = np.concatenate([getattr(i, k).reshape(5, -1) for k, _ in SC.PARAM_FIELDS], 1)
    for sz, sd in ((32, 8), (128, 2)):
        gens[f"random_camera_{sz}_{sd}"] = T.random_camera(sz, sd).world_to_cam
    np.savez_compressed(OUT / "generators.npz", **gens)

    # forward cases: reference tests/test_raster.py:155-162 fixtures (f32-quantised), branch rows
    for nd in (3, 6, 7):
        sc = f32(T.random_scene(nd, 60, seed=nd * 3 + 1))
        forward_case(f"tiled_{nd}", sc, T.random_camera(56, nd + 10), T.random_query(nd, nd + 20), st)
    sc = f32(T.random_scene(6, 150, seed=31))
    sc.opacity_raw[:] = SC.logit(0.97)
    forward_case("saturated_6", sc, T.random_camera(48, 32), T.random_query(6, 33), st)
    sc = f32(T.random_scene(7, 200, seed=11))
    forward_case("exact_7", sc, T.random_camera(40, 12), T.random_query(7, 13), exact)
    # clamp + PSD-floor rows (SURVEY §8(d) branch coverage)
    sc = f32(T.random_scene(7, 120, seed=5))
    sc.opacity_raw[:15] = 9.0
    sc.s_q_raw[:15] = np.log(50.0)
    sc.l_qx[:15] = 0.0
    q = T.random_query(7, 4)
    sc.l_qx[15:30] = 0.0
    sc.l_qx[15:30, 1:4, :] = 2.0 * np.eye(3)[None]
    sc.s_q_raw[15:30] = np.log(0.1)
    sc.b_q[15:30] = np.log(5.0)
    sc.mu_q[15:30] = q.dims[None, :].astype(np.float32).astype(np.float64)
    sc.s_x_raw[30:45] = np.log(np.array([0.2, 0.2, 1e-7], dtype=np.float32).astype(np.float64))
    br = f32(sc)
    forward_case("branches_7", br, T.random_camera(64, 3), q, st)

    # backward cases: small scenes, two views (fd_check-sized), N = 3/6/7
    for nd in (3, 6, 7):
        sc = f32(T.random_scene(nd, 12, seed=nd + 40))
        frames = T.random_frames(sc, 24, seed=nd + 50, count=2)
        backward_case(f"grads_{nd}", sc, frames, G.LossConfig())
    cam = T.random_camera(64, 3)
    tgt = np.clip(R.render(f32(T.random_scene(7, 60, seed=977)), cam, q), 0, 1)
    backward_case("grads_7_branches", br, [(cam, q, tgt)], G.LossConfig(lambda_ssim=0.5, loss_scale=2.0))


def branch_cases():
    """Round-2 branch fixtures: the gate_symmetric ablation (config.py:31,
    slicing.py:226, gradients.py:228-232), the 2x2 screen-floor adjoint
    (raster.py:116, gradients.py:179-204), a jitter-rescued query block
    (covariance.py:143-148) and non-default near / margin / floor settings."""
    from betasplat.camera import Camera
    from betasplat.covariance import batched_blocks, invert_query_block
    # gate_symmetric: |tanh| instead of max(tanh, 0) in the gate
    sym = bs.RenderSettings(gate_symmetric=True)
    sc = f32(T.random_scene(7, 80, seed=61))
    forward_case("gatesym_7", sc, T.random_camera(56, 62), T.random_query(7, 63), sym)
    backward_case("grads_7_gatesym", sc, T.random_frames(sc, 32, seed=64, count=2), G.LossConfig(), sym)
    sc6 = f32(T.random_scene(6, 60, seed=65))
    backward_case("grads_6_gatesym", sc6, T.random_frames(sc6, 32, seed=66, count=1), G.LossConfig(), sym)

    # 3D needles that engage the 1e-6 px^2 screen-space floor at a small size
    n = 6
    sc = bs.Scene(n_dims=3, mu_x=np.array([[0.0, 0.0, 0.0], [0.1, 0.05, 0.0], [0.0, 0.2, 0.1], [-0.1, -0.1, 0.05],
                                           [0.05, -0.2, -0.1], [0.2, 0.1, 0.1]]),
                  mu_q=np.zeros((n, 0)), rot=np.array([[0, 0, 0], [0, 0, 0], [0.1, 0, 0], [0, 0.05, 0],
                                                        [0, 0, 0.2], [0, 0, 0]], dtype=np.float64),
                  s_x_raw=np.log(np.array([[1e-3, 1e-7, 1e-3], [0.05, 0.05, 0.05], [2e-3, 1e-7, 1e-3],
                                           [1e-3, 1e-7, 2e-3], [3e-3, 1e-7, 1e-3], [0.04, 0.06, 0.05]])),
                  l_qx=np.zeros((n, 0, 3)), s_q_raw=np.zeros((n, 0)), b_x=np.array([0, 0.3, -0.2, 0.1, 0, 0.5]),
                  b_q=np.zeros((n, 0)), opacity_raw=np.array([2.0, 1.0, 1.5, 0.5, 1.0, 0.8]),
                  color=np.array([[0.9, 0.2, 0.1], [0.1, 0.8, 0.3], [0.3, 0.3, 0.9], [0.7, 0.6, 0.1],
                                  [0.2, 0.9, 0.9], [0.5, 0.5, 0.5]]), background=np.array([0.1, 0.1, 0.1]))
    sc = f32(sc)
    cam = Camera.look_at((3.0, 0.0, 0.0), (0.0, 0.0, 0.0), (0.0, 0.0, 1.0), 0.9, 96, 64)
    c = forward_case("screenfloor_3", sc, cam, bs.Query.static(), bs.RenderSettings())
    assert c.proj.floored.any()
    tgt = np.clip(0.5 + 0.3 * np.sin(np.arange(64 * 96 * 3).reshape(64, 96, 3) * 0.37), 0, 1)
    backward_case("grads_3_screenfloor", sc, [(cam, bs.Query.static(), tgt)], G.LossConfig())

    # jitter-rescued query block: a zero L_qx row with s_q -> 0 makes sigma_q
    # singular; one 1e-8 jitter restores it (not degenerate).  mu_q of that
    # dimension equals the query's, so its huge M entry multiplies delta = 0.
    sc = T.random_scene(7, 60, seed=67)
    cam = T.random_camera(48, 68)
    q = bs.Query.view_time(0.5, cam.forward)
    sc.l_qx[:6, 0, :] = 0.0
    sc.s_q_raw[:6, 0] = -400.0
    sc.mu_q[:6, 0] = 0.5
    sc = f32(sc)
    _, _, sq, _ = batched_blocks(sc.rot, np.exp(sc.s_x_raw), sc.l_qx, np.exp(sc.s_q_raw))
    try:
        np.linalg.cholesky(sq[:6])
        raise AssertionError("blocks are not singular")
    except np.linalg.LinAlgError:
        pass
    _, bad = invert_query_block(sq)
    assert not bad.any()
    forward_case("jitter_7", sc, cam, q, bs.RenderSettings())
    frames = []
    for k in range(2):  # query time 0.5 in every view: delta = 0 along the rescued dimension
        cam_k = T.random_camera(32, 69 + k)
        q_k = bs.Query.view_time(0.5, cam_k.forward)
        frames.append((cam_k, q_k, np.clip(R.render(f32(T.random_scene(7, 30, seed=1046 + k)), cam_k, q_k), 0, 1)))
    backward_case("grads_7_jitter", sc, frames, G.LossConfig())

    # non-default near plane / cull margin / screen floor / PSD floor scale / support
    st = bs.RenderSettings(near_plane=2.7, cull_margin=0.0, screen_cov_floor=9.0, psd_floor_scale=0.3, tau_sq=6.5)
    sc = f32(T.random_scene(7, 120, seed=71))
    cam = T.random_camera(64, 72)
    forward_case("settings_7", sc, cam, T.random_query(7, 73), st)
    backward_case("grads_7_settings", sc, T.random_frames(sc, 48, seed=74, count=2), G.LossConfig(), st)


def decomposition_cases():
    """render_decomposition (raster.py:358-423) for every channel a scene supports."""
    st = bs.RenderSettings()
    for nd, chans in ((6, ("b_x", "b_d", "opacity")), (7, ("b_x", "b_d", "b_t", "opacity"))):
        sc = f32(T.random_scene(nd, 80, seed=nd + 70))
        cam, q = T.random_camera(48, nd + 71), T.random_query(nd, nd + 72)
        intr, w2c = cam_arrays(cam)
        out = {c: R.render_decomposition(sc, cam, q, c, st) for c in chans}
        np.savez_compressed(OUT / f"decomp_{nd}.npz", in_records=records(sc), in_n_dims=nd,
                            in_background=sc.background, in_intr=intr, in_w2c=w2c, in_query=q.dims,
                            channels=np.array(chans), **{f"out_{c}": v for c, v in out.items()})
        print("decomp", nd, chans)


if __name__ == "__main__":
    if "--decomposition" in sys.argv:
        decomposition_cases()
    elif "--branches" in sys.argv:
        branch_cases()
    else:
        main()
        decomposition_cases()
        branch_cases()
