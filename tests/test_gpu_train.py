"""The config-5 training step's batched backend (sharding.GpuViewBackend):
views in flight on several slots, groups of views sharing one preprocess,
every view's chain on one gradient stream -- against one view at a time.
The raster backward sums with float atomics, so gradients agree to rounding,
not bitwise; the loss comes from the forward and matches to fp64 rounding."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2510_03312_b200 import engine, sharding, synthetic as S
from paper_2510_03312_b200.types import LossConfig

pytestmark = pytest.mark.gpu


def _views(nd, n_views, w=160, h=120):
    tgt = engine.DeviceScene.from_scene(S.synth(nd, 6000, seed=2), device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    out = []
    for k in range(n_views):
        cam = S.bench_camera(w, h, k, n_views)
        q = S.bench_query(nd, cam, k / max(n_views - 1, 1))
        out.append((cam, q, engine.render_frame(ws, tgt, cam, q).image.clone().clamp_(0.0, 1.0)))
    return out


@pytest.mark.parametrize("depth,group,ppl,first", [(3, 1, 4, None), (8, 4, 4, None), (4, 4, 4, None), (8, 8, 8, None),
                                                   (4, 2, 2, None), (6, 4, 4, 1), (8, 6, 4, 2)])
def test_batched_backend_matches_one_view_at_a_time(depth, group, ppl, first):
    nd = 7
    ds = engine.DeviceScene.from_scene(S.synth(nd, 6000, seed=1), device="cuda")
    views = _views(nd, 6)
    cfg = LossConfig()
    ref_loss, ref = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, depth=1)).loss_and_grad(views, cfg)
    step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, depth=depth, group=group, pixels_per_lane=ppl,
                                                            first_group=first))
    for _ in range(2):  # the second call reuses every slot (slot-free ordering)
        loss, grad = step.loss_and_grad(views, cfg)
    assert abs(float(loss) - float(ref_loss)) <= 1e-9 * abs(float(ref_loss))
    sl = engine.field_slices(nd)
    for name, (cols, _) in sl.items():
        a, b = grad[:, cols].double(), ref[:, cols].double()
        scale = float(b.norm())
        if scale == 0.0:
            assert float(a.norm()) == 0.0, name
            continue
        assert float((a - b).norm()) <= 1e-4 * scale, name


def test_batched_backend_trains():
    # a few Adam steps through the batched backend lower the loss
    nd = 7
    ds = engine.DeviceScene.from_scene(S.synth(nd, 6000, seed=1), device="cuda")
    views = _views(nd, 4)
    step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, depth=4, group=2))
    adam = sharding.DeviceAdam(ds.params, nd)
    cfg = LossConfig()
    losses = []
    grad = None
    for _ in range(6):
        loss, grad = step.loss_and_grad(views, cfg, grad)
        losses.append(float(loss))
        adam.step(grad)
    assert np.isfinite(losses).all() and losses[-1] < losses[0]


def test_optimizer_step_prepares_next_batch():
    """step.optimizer_step (Adam fused with the next batch's zeroing,
    regulariser gradient and value) trains like adam.step + the separate
    passes: same losses and parameters up to float-atomic rounding."""
    nd = 7
    views = _views(nd, 4)
    cfg = LossConfig(lambda_o=0.01, lambda_sigma=0.001)
    out = []
    for fused in (False, True):
        ds = engine.DeviceScene.from_scene(S.synth(nd, 6000, seed=1), device="cuda")
        step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, depth=4, group=2))
        adam = sharding.DeviceAdam(ds.params, nd)
        losses, grad = [], None
        for _ in range(4):
            loss, grad = step.loss_and_grad(views, cfg, grad)
            losses.append(float(loss))
            if fused:
                step.optimizer_step(adam, grad, cfg)
            else:
                adam.step(grad)
        out.append((np.array(losses), ds.params.double().cpu().numpy()))
    (l0, p0), (l1, p1) = out
    assert np.abs(l1 - l0).max() <= 1e-5 * np.abs(l0).max()
    assert np.abs(p1 - p0).max() <= 1e-4 * max(1.0, np.abs(p0).max())


def test_prepared_gradient_is_dropped_when_parameters_change():
    """A gradient buffer prepared by optimizer_step is only used while the
    parameters are unchanged: an in-place edit between steps (relocation,
    a user's reset) makes loss_and_grad zero it and add the regularisers
    itself -- the result equals a fresh unprepared step."""
    nd = 7
    views = _views(nd, 3)
    cfg = LossConfig(lambda_o=0.02, lambda_sigma=0.003)
    ds = engine.DeviceScene.from_scene(S.synth(nd, 5000, seed=3), device="cuda")
    step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, depth=3, group=3))
    adam = sharding.DeviceAdam(ds.params, nd)
    loss, grad = step.loss_and_grad(views, cfg)
    step.optimizer_step(adam, grad, cfg)
    ds.params[:, 0] += 1e-3  # edits the parameters: the prepared buffer is stale
    loss1, g1 = step.loss_and_grad(views, cfg, grad)
    ref_step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, depth=3, group=3))
    loss2, g2 = ref_step.loss_and_grad(views, cfg)
    assert abs(float(loss1) - float(loss2)) <= 1e-9 * abs(float(loss2))
    a, b = g1.double(), g2.double()
    assert float((a - b).norm()) <= 1e-4 * float(b.norm())


@pytest.mark.parametrize("w,h", [(77, 53), (160, 120), (33, 17)])
def test_backward_layouts_agree(w, h):
    """The fp32 raster backward's two layouts (2 or 4 pixels per lane) give
    the same gradient up to float-atomic summation order, on ragged images
    whose last tiles are partly outside; an invalid layout is an error."""
    from paper_2510_03312_b200 import _lib
    nd = 7
    ds = engine.DeviceScene.from_scene(S.synth(nd, 4000, seed=9), device="cuda")
    cam = S.bench_camera(w, h)
    q = S.bench_query(nd, cam, 0.4)
    ws = engine.Workspace("cuda", "fp32")
    fr = engine.render_frame(ws, ds, cam, q)
    g_img = torch.randn(h, w, 3, device="cuda")
    grads = []
    for ppl in (2, 4):
        g = torch.zeros(ds.params.shape, device="cuda")
        gb = engine.backward_raster(fr, ds, g_img, g, pixels_per_lane=ppl)
        engine.backward_chain(fr, gb)
        grads.append(g.double())
    a, b = grads
    assert float(b.norm()) > 0.0
    assert float((a - b).norm()) <= 1e-5 * float(b.norm())
    with pytest.raises(_lib.UbsError):
        engine.backward_raster(fr, ds, g_img, torch.zeros(ds.params.shape, device="cuda"), pixels_per_lane=3)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_regulariser_value_kernel(dtype):
    # the fused regulariser value against the torch fp64 formula
    nd = 6
    ds = engine.DeviceScene.from_scene(S.synth(nd, 5000, seed=4), dtype=dtype, device="cuda")
    cfg = LossConfig(lambda_o=0.01, lambda_sigma=0.02)
    got = float(sharding.GpuViewBackend(ds).regulariser_value(cfg))
    sl = engine.field_slices(nd)
    p = ds.params.double()
    want = cfg.lambda_o * torch.sigmoid(p[:, sl["opacity_raw"][0]]).sum() + cfg.lambda_sigma * (
        torch.exp(p[:, sl["s_x_raw"][0]]).sum() + torch.exp(p[:, sl["s_q_raw"][0]]).sum())
    assert abs(got - float(want)) <= 1e-12 * abs(float(want))


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_chain_leaves_screen_space_sums_zero(precision):
    # ubs_prim_backward consumes grad2d (zeroes it), so back-to-back backwards
    # on one workspace need no zeroing pass and give the same gradient
    nd = 7
    dtype = torch.float64 if precision == "fp64" else torch.float32
    ds = engine.DeviceScene.from_scene(S.synth(nd, 3000, seed=12), dtype=dtype, device="cuda")
    cam = S.bench_camera(96, 64)
    q = S.bench_query(nd, cam, 0.6)
    ws = engine.Workspace("cuda", precision)
    fr = engine.render_frame(ws, ds, cam, q)
    g_img = torch.randn(64, 96, 3, device="cuda", dtype=fr.image.dtype)
    grads = []
    for _ in range(3):
        g = torch.zeros(ds.params.shape, device="cuda", dtype=dtype)
        engine.backward_frame(fr, ds, g_img, g)
        grads.append(g.double())
        assert ws.grad2d_clean and float(ws.grad2d.abs().max()) == 0.0
    for g in grads[1:]:
        assert float((g - grads[0]).norm()) <= 1e-5 * float(grads[0].norm())
