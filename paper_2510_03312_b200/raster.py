"""Drop-in render entry points (reference raster.py:269-322) on the B200 engine.

``render`` / ``render_with_cache`` take the reference's own argument objects
(``Scene``, ``Camera``, ``Query``, ``RenderSettings``: duck-typed, so objects
from ``betasplat`` work as well as this package's mirrors) and return float64
numpy arrays like the reference.  The work happens on the GPU:
parameters are uploaded as packed UBS1 records, and every stage runs in the
sm_100a kernels of ``libubs_b200.so``.  There is no CPU fallback.

Extra keyword arguments (not in the reference signature):
  ``precision``  "fp32" (default: fp64 geometry, fp32 raster, certified
                 fp64 fix-up) or "fp64" (reference arithmetic throughout);
  ``device``     CUDA device (default: current).
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np
import torch

from . import engine
from ._lib import DEBUG_STRIDE, F_DEGENERATE, F_FLOOR2, F_FLOOR3, F_VISIBLE
from .types import PARAM_FIELDS, DEFAULT_SETTINGS

DEFAULT_PRECISION = "fp32"
_WORKSPACES: dict = {}


def workspace(precision: str | None = None, device=None) -> engine.Workspace:
    """The shared per-(device, precision) workspace used by the numpy API."""
    precision = precision or DEFAULT_PRECISION
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device()) \
        if torch.cuda.is_available() else torch.device("cuda")
    key = (str(dev), precision)
    ws = _WORKSPACES.get(key)
    if ws is None:
        ws = engine.Workspace(dev, precision)
        _WORKSPACES[key] = ws
    return ws


_PINNED: dict = {}  # tag -> the reused pinned host staging buffer (latest shape only)


def _pinned(tag, shape, dtype) -> torch.Tensor:
    buf = _PINNED.get(tag)
    if buf is None or tuple(buf.shape) != tuple(shape) or buf.dtype != dtype:
        buf = torch.empty(tuple(shape), dtype=dtype, pin_memory=True)
        _PINNED[tag] = buf
    return buf


def _packed_records(scene, n: int):
    """The (n, 14+6C) float64 record array every parameter field of ``scene``
    is a view into, at its PARAM_FIELDS offset, else None.  Scenes built by
    Scene.from_records (UBS1 loading -- here and in betasplat, whose
    ``frombuffer(...).astype(f8).reshape(n, w)`` leaves a 1-D owner --,
    quantize_f32, synth) qualify: the owner is either the 2-D record array or
    a C-contiguous 1-D buffer of exactly n * (14+6C) floats."""
    from .types import field_offsets
    base = np.asarray(scene.mu_x).base
    while base is not None and getattr(base, "base", None) is not None and base.ndim not in (1, 2):
        base = base.base
    width = 14 + 6 * (int(scene.n_dims) - 3)
    if not isinstance(base, np.ndarray) or base.dtype != np.float64 or not base.flags.c_contiguous:
        return None
    if base.ndim == 1 and base.size == n * width:
        base = base.reshape(n, width)  # a view of the contiguous owner, no copy
    if base.shape != (n, width):
        return None
    p0 = base.__array_interface__["data"][0]
    item = base.itemsize
    for name, (off, size, _shape) in field_offsets(int(scene.n_dims)).items():
        a = np.asarray(getattr(scene, name))
        if size == 0 and a.size == 0:  # mu_q / l_qx / s_q_raw / b_q of a 3D scene
            continue
        if a.dtype != np.float64 or a.size != n * size or not np.shares_memory(a, base):
            return None
        if a.__array_interface__["data"][0] != p0 + off * item:
            return None
        # rows at the record stride, the field's values contiguous inside a row
        if n > 1 and a.strides[0] != base.strides[0]:
            return None
        if a.ndim > 1 and not a[0].flags.c_contiguous:  # one row of the view, no copy
            return None
    return base


def _device_scene(scene, ws: engine.Workspace) -> engine.DeviceScene:
    """The scene's records on the workspace's device, re-uploaded every call
    (callers such as fd_check mutate arrays in place, so a copy kept across
    calls could go stale).  Each field goes through a reused pinned staging
    buffer (a contiguous host copy, then DMA; pageable uploads of the 300 MB
    of float64 fields at 1M primitives ran at ~2 GB/s) and the fields are
    interleaved and cast on the device: the bits of pack_records' host cast.
    The staging buffers are reused by the next call only after this call's
    result has been read back (every numpy entry point synchronises)."""
    dtype = torch.float64 if ws.f64 else torch.float32
    n = int(np.asarray(scene.mu_x).shape[0])
    if n == 0 or not torch.cuda.is_available():
        return engine.DeviceScene.from_scene(scene, dtype=dtype, device=ws.device)
    torch.cuda.current_stream(ws.device).synchronize()  # the previous call's uploads are done
    rec = _packed_records(scene, n)
    if rec is not None:  # every field is a view into one packed record array: one contiguous copy
        st = _pinned("records", rec.shape, torch.float64)
        np.copyto(st.numpy(), rec)
        params = st.to(ws.device, non_blocking=True).to(dtype).contiguous()
        return engine.DeviceScene(params, scene.n_dims, scene.background)
    cols = []
    for k, _ in PARAM_FIELDS:
        a = np.asarray(getattr(scene, k)).reshape(n, -1)
        st = _pinned(k, a.shape, torch.float64)
        np.copyto(st.numpy(), a, casting="unsafe")
        cols.append(st.to(ws.device, non_blocking=True))
    params = torch.cat(cols, dim=1).to(dtype).contiguous()
    return engine.DeviceScene(params, scene.n_dims, scene.background)


def _host_image(fr: engine.Frame, background) -> np.ndarray:
    """(H, W, 3) float64; pixels nothing was composited into get the exact fp64
    background (acc = 0, T = 1 gives 0 + 1 * bg in tile_forward, _tiles.py:51-53)."""
    st = _pinned("image", (fr.height, fr.width, 3), torch.float64)
    st.copy_(fr.image.view(fr.height, fr.width, 3).double(), non_blocking=True)
    torch.cuda.current_stream(fr.image.device).synchronize()
    img = st.numpy().copy()
    if not fr.raster_f64:
        empty = ((fr.alpha_sum == 0) & (fr.t_stop == 1)).cpu().numpy()
        if empty.any():
            img[empty] = np.asarray(background, dtype=np.float64).reshape(3)
    return img


class FrameCache:
    """Host view of one forward frame (reference raster.py:63-92).

    Eager: image, alpha_sum, t_stop, alpha_clamped, processed_pixels, order,
    n_contrib (per-pixel contributor count, not in the reference).
    Lazy, from a re-run of the same frame: ``tiles`` / ``tile_ranges`` /
    ``tile_ids`` (the full per-tile id lists), ``slices`` / ``proj`` (a subset
    of the reference's SliceCache / ProjectionCache fields, from a debug run).
    """

    def __init__(self, scene, camera, query, settings, precision, fr: engine.Frame):
        self.scene, self.camera, self.query, self.settings = scene, camera, query, settings
        self.precision = precision
        H, W = fr.height, fr.width
        self.image = _host_image(fr, scene.background)
        self.alpha_sum = fr.alpha_sum.double().cpu().numpy()
        self.t_stop = fr.t_stop.double().cpu().numpy()
        self.n_contrib = fr.n_contrib.cpu().numpy()
        self.alpha_clamped = fr.hit_clamp.cpu().numpy().astype(bool)
        self.processed_pixels = fr.processed_pixels
        self.n_fixed = 0 if fr.raster_f64 else fr.n_fixed
        ws = fr.ws
        self.order = ws.order[:fr.n_visible].to(torch.int64).cpu().numpy()
        self._flags = ws.flags[:fr.n].to(torch.int32).cpu().numpy() & 0xFFFF
        self._tiles = None
        self._tile_ranges = None
        self._tile_ids = None
        self._debug = None

    def _load_tiles(self):
        # the full per-tile lists (K ids, ~26M at 7D 1M 1080p) are copied only
        # when asked for, from a re-run that materialises every list
        if self._tile_ids is None:
            ws = workspace(self.precision)
            ds = _device_scene(self.scene, ws)
            fr = engine.render_frame(ws, ds, self.camera, self.query, self.settings, full_lists=True)
            W, H = int(self.camera.width), int(self.camera.height)
            ntiles = math.ceil(W / 16) * math.ceil(H / 16)
            self._tile_ranges = ws.tile_ranges[:2 * ntiles].view(ntiles, 2).to(torch.int64).cpu().numpy()
            self._tile_ids = ws.tile_ids[:fr.n_pairs].to(torch.int64).cpu().numpy() if fr.n_pairs else \
                np.zeros(0, dtype=np.int64)

    @property
    def tile_ranges(self) -> np.ndarray:
        """(ntiles, 2) [start, end) of each tile's list in ``tile_ids`` (lazy)."""
        self._load_tiles()
        return self._tile_ranges

    @property
    def tile_ids(self) -> np.ndarray:
        """Every tile's depth-ordered primitive ids, concatenated (lazy)."""
        self._load_tiles()
        return self._tile_ids

    @property
    def tiles(self) -> list:
        """[(y0, y1, x0, x1, ids)] in row-major tile order (raster.py:252-266)."""
        if self._tiles is None:
            W, H = int(self.camera.width), int(self.camera.height)
            tx_n = math.ceil(W / 16)
            out = []
            for t, (s, e) in enumerate(self.tile_ranges):
                ty, tx = divmod(t, tx_n)
                out.append((16 * ty, min(16 * ty + 16, H), 16 * tx, min(16 * tx + 16, W),
                            self.tile_ids[s:e]))
            self._tiles = out
        return self._tiles

    def _dump(self):
        if self._debug is None:
            ws = workspace(self.precision)
            ds = _device_scene(self.scene, ws)
            fr = engine.render_frame(ws, ds, self.camera, self.query, self.settings, want_debug=True,
                                     full_lists=True)
            self._debug = ws.debug[:fr.n * DEBUG_STRIDE].view(fr.n, DEBUG_STRIDE).cpu().numpy().copy()
        return self._debug

    @property
    def proj(self):
        d, f = self._dump(), self._flags
        p2 = np.stack([np.stack([d[:, 3], d[:, 4]], 1), np.stack([d[:, 4], d[:, 5]], 1)], 1)
        cov2 = np.stack([np.stack([d[:, 10], d[:, 11]], 1), np.stack([d[:, 11], d[:, 12]], 1)], 1)
        return SimpleNamespace(depth=d[:, 0], mean2=d[:, 1:3], p2=p2, radii=d[:, 6:8], cov2=cov2,
                               t_cam=d[:, 19:22], visible=(f & F_VISIBLE) != 0,
                               floored=(f & F_FLOOR2) != 0)

    @property
    def slices(self):
        d, f = self._dump(), self._flags
        c = self.scene.n_dims - 3
        i = [0, 1, 2, 1, 3, 4, 2, 4, 5]
        cov3 = d[:, 13:19][:, i].reshape(-1, 3, 3)
        return SimpleNamespace(valid=(f & F_DEGENERATE) == 0, mean3=d[:, 22:25], cov3=cov3,
                               gated_opacity=d[:, 8], beta_x=d[:, 9], gate=d[:, 25], opacity=d[:, 26],
                               s_tanh=d[:, 27:27 + c], floor_eps=d[:, 31], floored=(f & F_FLOOR3) != 0)

    def trace_signature(self) -> tuple:
        """Discrete branch state (raster.py:81-92)."""
        c = self.scene.n_dims - 3
        f = self._flags
        sgn = np.stack([(f >> (8 + k)) & 1 for k in range(c)], 1).astype(bool) if c else \
            np.zeros((f.shape[0], 0), bool)
        return (((f & F_VISIBLE) != 0).tobytes(), ((f & F_FLOOR3) != 0).tobytes(),
                ((f & F_FLOOR2) != 0).tobytes(), sgn.tobytes(), self.alpha_clamped.tobytes(),
                self.order.tobytes(), self.processed_pixels)


def render_with_cache(scene, cam, query, settings=DEFAULT_SETTINGS, *, precision: str | None = None,
                      device=None) -> FrameCache:
    """Full forward pass returning the image plus per-frame state (raster.py:269-316)."""
    c = scene.n_dims - 3
    if np.asarray(query.dims).reshape(-1).shape[0] != c:
        raise ValueError(f"query has {np.asarray(query.dims).size} dims, scene expects {c}")
    ws = workspace(precision, device)
    ds = _device_scene(scene, ws)
    fr = engine.render_frame(ws, ds, cam, query, settings)
    return FrameCache(scene, cam, query, settings, ws.precision, fr)


def render(scene, cam, query, settings=DEFAULT_SETTINGS, *, precision: str | None = None,
           device=None) -> np.ndarray:
    """Render to an (H, W, 3) float64 image (raster.py:319-322); not clipped."""
    c = scene.n_dims - 3
    if np.asarray(query.dims).reshape(-1).shape[0] != c:
        raise ValueError(f"query has {np.asarray(query.dims).size} dims, scene expects {c}")
    ws = workspace(precision, device)
    ds = _device_scene(scene, ws)
    fr = engine.render_frame(ws, ds, cam, query, settings)
    return _host_image(fr, scene.background)


# ---------------------------------------------------------------------------
# render_decomposition (reference raster.py:355-422)
# ---------------------------------------------------------------------------
DECOMPOSITION_CHANNELS = ("b_x", "b_d", "b_t", "opacity")


def channel_values(params: torch.Tensor, n_dims: int, channel: str) -> torch.Tensor:
    """Per-primitive scalar of ``channel`` from the packed records, fp64 on the
    records' device (raster.py:397-410, same error messages)."""
    from .types import field_offsets
    c = n_dims - 3
    off = field_offsets(n_dims)
    p = params.double()
    if channel == "b_x":
        return (p[:, off["b_x"][0]] + 5.0) / 10.0
    if channel == "opacity":
        return torch.sigmoid(p[:, off["opacity_raw"][0]])
    if channel == "b_d":
        if c < 3:
            raise ValueError("b_d channel needs direction dimensions (6D or 7D scene)")
        o = off["b_q"][0]
        bq = p[:, o + c - 3:o + c]
        return ((((bq[:, 0] + bq[:, 1]) + bq[:, 2]) / 3.0) + 5.0) / 10.0  # numpy's mean of 3, in order
    if channel == "b_t":
        if n_dims != 7:
            raise ValueError("b_t channel is only available for 7D scenes")
        return (p[:, off["b_q"][0]] + 5.0) / 10.0
    raise ValueError(f"unknown channel {channel!r}; expected one of {DECOMPOSITION_CHANNELS}")


def diverging_colormap(t: torch.Tensor) -> torch.Tensor:
    """Blue -> white -> red over t in [0, 1] (raster.py:413-422)."""
    t = t.double().clamp(0.0, 1.0)
    lo = t.new_tensor([0.15, 0.25, 0.85])
    mid = t.new_tensor([0.95, 0.95, 0.95])
    hi = t.new_tensor([0.85, 0.20, 0.15])
    u = (t * 2.0).clamp(0.0, 1.0)[:, None]
    v = (t * 2.0 - 1.0).clamp(0.0, 1.0)[:, None]
    return torch.where(t[:, None] < 0.5, lo + u * (mid - lo), mid + v * (hi - mid))


def render_decomposition(scene, cam, query, channel: str, settings=DEFAULT_SETTINGS, *,
                         device=None) -> np.ndarray:
    """Heat map of a per-primitive scalar composited with the render's own
    weights (raster.py:358-394): the colours become the diverging colormap of
    the scalar, the background zero, and each pixel is divided by its
    accumulated alpha (background where nothing was composited).

    Runs the device path on records whose colour fields hold the colormap, in
    the fp64 raster: the division by the alpha sum amplifies the fp32 raster's
    absolute errors wherever coverage is low (measured: up to 0.9 at 1.7% of
    the fixture pixels), so there is no fp32 variant."""
    from .types import field_offsets
    precision = "fp64"
    c = scene.n_dims - 3
    if np.asarray(query.dims).reshape(-1).shape[0] != c:
        raise ValueError(f"query has {np.asarray(query.dims).size} dims, scene expects {c}")
    ws = workspace(precision, device)
    ds = _device_scene(scene, ws)
    colors = diverging_colormap(channel_values(ds.params, scene.n_dims, channel))
    params = ds.params.clone()
    o = field_offsets(scene.n_dims)["color"][0]
    params[:, o:o + 3] = colors.to(params.dtype)
    fr = engine.render_frame(ws, engine.DeviceScene(params, scene.n_dims, (0.0, 0.0, 0.0)), cam, query, settings)
    num, den = fr.image.double(), fr.alpha_sum.double()
    bg = torch.as_tensor(np.asarray(scene.background, dtype=np.float64), device=num.device)
    out = torch.where(den[..., None] > 0.0, num / den.clamp_min(1e-300)[..., None], bg)
    return out.cpu().numpy()
