"""Drop-in loss + gradient entry point (reference gradients.py:101-127) on the GPU.

``backward(scene, frames, cfg, settings)`` returns ``(loss, SceneGrads)`` with
the reference's semantics: per view render, L1 + SSIM image gradient scaled
by ``loss_scale / len(frames)``, reverse blend, chain to raw parameters;
regularisers added once; non-finite gradients raise ``GradientError`` naming
the field and primitive.  Everything per view runs in the sm_100a kernels;
the parameter gradients accumulate in an fp64 device buffer.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, engine
from . import raster as _raster
from .raster import _device_scene, _parallel_rows, _pinned, workspace
from .types import DEFAULT_SETTINGS, LossConfig, SceneGrads, field_offsets, sigmoid


def _host_grads(grads: torch.Tensor, n_dims: int) -> SceneGrads:
    """The (n, 14+6C) fp64 device gradient as one contiguous host array per
    field.  The fields are split on the device into one field-major buffer
    and DMA'd, in one copy, into a pinned block of torch's caching host
    allocator that the returned arrays own (views into it: no host copy);
    past raster._PINNED_OUT_MAX live blocks the fields go through reused
    pinned staging buffers and are copied out (a pageable read of the
    interleaved buffer plus per-field strided copies cost ~0.3 s at 1M
    primitives)."""
    n = grads.shape[0]
    offs = field_offsets(n_dims)
    if _raster._PINNED_OUT[0] < _raster._PINNED_OUT_MAX:
        flat = torch.empty(grads.numel(), dtype=torch.float64, device=grads.device)
        pos, where = 0, {}
        for name, (off, size, shape) in offs.items():
            flat[pos:pos + n * size].view(n, size).copy_(grads[:, off:off + size])
            where[name] = (pos, size, shape)
            pos += n * size
        host = torch.empty(grads.numel(), dtype=torch.float64, pin_memory=True)
        host.copy_(flat, non_blocking=True)
        torch.cuda.current_stream(grads.device).synchronize()
        arr = host.numpy()
        _raster._PINNED_OUT[0] += 1
        import weakref
        weakref.finalize(arr.base, _raster._pinned_out_released)  # the alias every field view holds
        return SceneGrads(**{name: arr[p0:p0 + n * size].reshape((n,) + shape)
                             for name, (p0, size, shape) in where.items()})
    stage = {}
    for name, (off, size, shape) in offs.items():
        st = _pinned("grad_" + name, (n, size), torch.float64)
        st.copy_(grads[:, off:off + size], non_blocking=True)
        stage[name] = (st, shape)
    torch.cuda.current_stream(grads.device).synchronize()
    return SceneGrads(**{name: st.numpy().reshape((n,) + shape).copy() for name, (st, shape) in stage.items()})


def _regularizers(scene, cfg: LossConfig) -> float:
    """lambda_o sum sigmoid(o) + lambda_sigma (sum exp(s_x) + sum exp(s_q)) on
    the host's float64 fields (gradients.py:120-123), in row chunks on the
    host threads (the chunk sums added in order)."""
    op = np.asarray(scene.opacity_raw, dtype=np.float64).reshape(-1)
    sx = np.asarray(scene.s_x_raw, dtype=np.float64)
    sq = np.asarray(scene.s_q_raw, dtype=np.float64)
    n = op.shape[0]
    sx, sq = sx.reshape(n, -1), sq.reshape(n, -1)
    parts = {}

    def part(r0, r1):
        parts[r0] = (float(sigmoid(op[r0:r1]).sum()),
                     float(np.exp(sx[r0:r1]).sum()) + (float(np.exp(sq[r0:r1]).sum()) if sq.size else 0.0))
    _parallel_rows(n, part)
    so = ss = 0.0
    for r0 in sorted(parts):
        so += parts[r0][0]
        ss += parts[r0][1]
    return cfg.lambda_o * so + cfg.lambda_sigma * ss


def _target_to_device(target, fr: engine.Frame) -> torch.Tensor:
    """The host target image on the device at the raster's precision: cast
    by host threads into a reused pinned buffer (the bits of a device cast),
    one DMA (the previous frame's copy is done: its loss was read back)."""
    dt = fr.image.dtype
    src = np.asarray(target)
    if src.shape != (fr.height, fr.width, 3):
        src = src.reshape(fr.height, fr.width, 3)
    st = _pinned("target", (fr.height, fr.width, 3), dt)
    dst = st.numpy()
    _parallel_rows(fr.height, lambda r0, r1: np.copyto(dst[r0:r1], src[r0:r1], casting="unsafe"), min_rows=64)
    return st.to(fr.image.device, non_blocking=True)


def backward(scene, frames, cfg: LossConfig = LossConfig(), settings=DEFAULT_SETTINGS, *,
             precision: str | None = None, device=None, deterministic: bool = False):
    """Loss over the batch plus gradients for every primitive field.

    ``deterministic=True``: the raster backward reduces per-(primitive, tile)
    partials in a fixed order instead of with float atomics, so repeated
    calls return bit-identical gradients (the reference's guarantee,
    raster.py:1-8); the loss sums are always reduced in a fixed order."""
    if not frames:
        raise ValueError("empty batch")
    ws = workspace(precision, device)
    ds = _device_scene(scene, ws)
    grads = torch.zeros(ds.params.shape, dtype=torch.float64, device=ws.device)
    scale = cfg.loss_scale / len(frames)
    rec = 0.0
    for k, (cam, query, target) in enumerate(frames):
        fr = engine.render_frame(ws, ds, cam, query, settings)
        ws.loss_parts.zero_()
        tgt = _target_to_device(target, fr)
        g_img, parts = engine.loss_image_grad(fr, tgt, cfg.lambda_ssim, scale)
        engine.backward_frame(fr, ds, g_img, grads, deterministic=deterministic)
        l1_sum, ssim_sum = parts.cpu().tolist()
        size = fr.width * fr.height * 3
        rec += (1.0 - cfg.lambda_ssim) * (l1_sum / size) + cfg.lambda_ssim * (1.0 - ssim_sum / size)
    rec /= len(frames)
    # regulariser gradients once per step (gradients.py:120-123)
    lib = _lib.load()
    _lib.check(lib.ubs_add_regularisers(ds.params.data_ptr(), int(ds.params.dtype == torch.float64),
                                        grads.data_ptr(), 1, ds.n, ds.n_dims, cfg.loss_scale * cfg.lambda_o,
                                        cfg.loss_scale * cfg.lambda_sigma, torch.cuda.current_stream().cuda_stream),
               "ubs_add_regularisers")
    if not bool(torch.isfinite(grads).all()):
        _host_grads(grads, scene.n_dims).check_finite()  # names the field and primitive
    out = _host_grads(grads, scene.n_dims)
    total = cfg.loss_scale * (rec + _regularizers(scene, cfg))
    return total, out
