"""TORCH_LIBRARY(ubs) operators (csrc_torch/ubs_torch.cpp over the C ABI).

CPU: the extension builds, registers every schema, and has no CPU kernel (a
CPU tensor is refused -- no fallback).  GPU: ``ubs::render`` gives the
engine's bits, ``ops.render`` is differentiable and its parameter gradient
equals the engine's backward for the same dL/dimage, and the loss / Adam
operators match their ctypes counterparts."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2510_03312_b200 import ops, synthetic as S
from paper_2510_03312_b200.types import DEFAULT_SETTINGS, quantize_f32


def test_operators_registered_without_cpu_kernels():
    ops.load()
    for name in ("scene_statics", "render", "render_backward", "loss_image_grad", "adam_step_"):
        assert hasattr(torch.ops.ubs, name), name
    assert "alpha_clamped" in str(torch.ops.ubs.render.default._schema)
    p = torch.zeros((4, 38), dtype=torch.float32)
    cam = S.random_camera(16, 1)
    with pytest.raises((NotImplementedError, RuntimeError)):
        torch.ops.ubs.render(p, 7, ops.camera_tensor(cam), ops.query_tensor(S.random_query(7, 2)),
                             ops.settings_tensor(), torch.zeros(3, dtype=torch.float64), None, False)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_render_op_matches_engine_and_is_differentiable(precision):
    from paper_2510_03312_b200 import engine
    sc = quantize_f32(S.random_scene(7, 3000, seed=5))
    cam, q = S.random_camera(96, 6), S.random_query(7, 7)
    dtype = torch.float64 if precision == "fp64" else torch.float32
    ds = engine.DeviceScene.from_scene(sc, dtype=dtype, device="cuda")
    ws = engine.Workspace("cuda", precision)
    fr = engine.render_frame(ws, ds, cam, q)
    params = ds.params.clone().requires_grad_(True)
    image, asum, tstop, ncontrib, clamped = ops.render(params, 7, cam, q, DEFAULT_SETTINGS, sc.background, precision)
    assert torch.equal(image.detach(), fr.image) and torch.equal(ncontrib, fr.n_contrib)
    assert torch.equal(tstop, fr.t_stop) and torch.equal(clamped, fr.hit_clamp.bool())
    g_img = torch.randn_like(image) * 1e-3
    (image * g_img).sum().backward()
    ref = torch.zeros(ds.params.shape, dtype=torch.float64, device="cuda")
    fr = engine.render_frame(ws, ds, cam, q)
    engine.backward_frame(fr, ds, g_img.to(fr.image.dtype), ref)
    got = params.grad.double()
    rel = (got - ref).norm() / ref.norm()
    assert rel <= (1e-12 if precision == "fp64" else 1e-5), float(rel)


@pytest.mark.gpu
def test_loss_and_adam_ops_match_ctypes_path():
    from paper_2510_03312_b200 import engine, sharding
    ops.load()
    sc = quantize_f32(S.random_scene(7, 500, seed=8))
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    fr = engine.render_frame(ws, ds, S.random_camera(64, 9), S.random_query(7, 10))
    tgt = torch.rand_like(fr.image)
    ws.loss_parts.zero_()
    g_ref, parts_ref = engine.loss_image_grad(fr, tgt, 0.2, 1.5)
    g, parts = torch.ops.ubs.loss_image_grad(fr.image, tgt, 0.2, 1.5)
    assert torch.equal(g, g_ref) and torch.equal(parts, parts_ref)
    p1, p2 = ds.params.clone(), ds.params.clone()
    grad = torch.randn_like(p1) * 1e-2
    m1, v1 = torch.zeros_like(p1), torch.zeros_like(p1)
    torch.ops.ubs.adam_step_(p1, grad, m1, v1, 7, [1.6e-4, 5e-2, 5e-3, 1e-3], 1, False)
    adam = sharding.DeviceAdam(p2, 7)
    adam.step(grad)
    assert torch.equal(p1, p2) and torch.equal(m1, adam.m) and torch.equal(v1, adam.v)
