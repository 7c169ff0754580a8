"""``torch.ops.ubs.*``: the C ABI as PyTorch operators (csrc_torch/ubs_torch.cpp).

``load()`` registers ``TORCH_LIBRARY(ubs)`` from the in-tree
``libubs_torch.so`` (built by ``build.build_torch_ops``), which links the same
``libubs_b200.so`` the ctypes engine uses.  The helpers convert the
reference's Camera / Query / RenderSettings objects (duck-typed) to the
operators' tensor arguments, and :func:`render` is differentiable with
respect to the packed parameter records: its backward runs
``ubs::render_backward`` (gradients.py:130-300 on the device), so torch code
can optimise a scene with ``loss.backward()``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import build as _build
from ._lib import UbsError
from .types import DEFAULT_SETTINGS

_LOADED = False


def load():
    """Register torch.ops.ubs (builds the extension in-tree first if stale)."""
    global _LOADED
    if _LOADED:
        return torch.ops.ubs
    if _build.torch_ops_need_build():
        _build.build_torch_ops()
    if not _build.TORCH_OUT.exists():
        raise UbsError(f"{_build.TORCH_OUT} is missing; run python -m paper_2510_03312_b200.build")
    torch.ops.load_library(str(_build.TORCH_OUT))
    _LOADED = True
    return torch.ops.ubs


def camera_tensor(cam) -> torch.Tensor:
    """[fx, fy, cx, cy, world_to_cam[:3, :3] row-major, world_to_cam[:3, 3], width, height] (f64, 18)."""
    w2c = np.asarray(cam.world_to_cam, dtype=np.float64).reshape(4, 4)
    vals = [float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), *w2c[:3, :3].reshape(-1), *w2c[:3, 3],
            float(cam.width), float(cam.height)]
    return torch.tensor(vals, dtype=torch.float64)


def settings_tensor(settings=DEFAULT_SETTINGS) -> torch.Tensor:
    """RenderSettings (config.py:9-38) as the operators' f64[9]."""
    return torch.tensor([settings.tau_sq, settings.alpha_clamp, settings.transmittance_min, settings.near_plane,
                         settings.cull_margin, settings.screen_cov_floor, settings.psd_floor_scale,
                         1.0 if settings.gate_symmetric else 0.0, float(settings.tile_size)], dtype=torch.float64)


def query_tensor(query) -> torch.Tensor:
    return torch.as_tensor(np.asarray(query.dims, dtype=np.float64).reshape(-1))


class _Render(torch.autograd.Function):
    @staticmethod
    def forward(ctx, params, n_dims, cam, q, st, bg, fp64):
        image, alpha_sum, t_stop, n_contrib, clamped = torch.ops.ubs.render(params, n_dims, cam, q, st, bg, None,
                                                                           fp64)
        ctx.save_for_backward(params)
        ctx.args = (n_dims, cam, q, st, bg, fp64)
        ctx.mark_non_differentiable(alpha_sum, t_stop, n_contrib, clamped)
        return image, alpha_sum, t_stop, n_contrib, clamped

    @staticmethod
    def backward(ctx, g_image, *_):
        (params,) = ctx.saved_tensors
        n_dims, cam, q, st, bg, fp64 = ctx.args
        g = torch.ops.ubs.render_backward(params, n_dims, cam, q, st, bg, g_image.contiguous(), fp64)
        return g, None, None, None, None, None, None


def render(params: torch.Tensor, n_dims: int, cam, query, settings=DEFAULT_SETTINGS, background=(0.0, 0.0, 0.0),
           precision: str = "fp32"):
    """One frame of the packed records ``params`` (n x (14+6C), CUDA):
    returns (image (H, W, 3), alpha_sum, t_stop, n_contrib, alpha_clamped).
    Differentiable in ``params`` (the image output)."""
    load()
    if precision not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    bg = torch.as_tensor(np.asarray(background, dtype=np.float64).reshape(3))
    return _Render.apply(params, int(n_dims), camera_tensor(cam), query_tensor(query), settings_tensor(settings), bg,
                         precision == "fp64")
