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

import weakref

import numpy as np
import torch

from . import engine
from ._lib import DEBUG, DEBUG_STRIDE, F_DEGENERATE, F_FLOOR2, F_FLOOR3, F_VISIBLE
from .types import PARAM_FIELDS, DEFAULT_SETTINGS, ProjectionCache, SliceCache

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


_STAGE_PARTS = 4      # drop-in scene staging: parts whose uploads overlap the next parts' casts
_PINNED_OUT = [0]     # images handed out in pinned memory and still alive
_PINNED_OUT_MAX = 8   # beyond this many, images are copied into ordinary memory


def _pinned_out_released():
    _PINNED_OUT[0] -= 1


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


_POOL = None


def _pool():
    """Host threads for the staging copies (numpy's copy / cast loops release
    the GIL, so row chunks copy in parallel at several times one core's
    memory bandwidth)."""
    global _POOL
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)))
    return _POOL


def _parallel_rows(n: int, fn, min_rows: int = 1 << 15):
    """fn(r0, r1) over row chunks of [0, n), on the host pool when large."""
    if n < 2 * min_rows:
        fn(0, n)
        return
    k = min(_pool()._max_workers, -(-n // min_rows))
    step = -(-n // k)
    list(_pool().map(lambda r0: fn(r0, min(n, r0 + step)), range(0, n, step)))


_RESIDENT: dict = {}  # id(scene) -> (scene, precision, DeviceScene): opt-in scene cache (resident())


class resident:
    """Keep ``scene``'s device copy between drop-in calls (opt-in).

    Inside ``with raster.resident(scene):`` the drop-in uploads the scene
    once per precision and reuses it for every ``render`` /
    ``render_with_cache`` / ``backward`` of that same object -- a sweep of
    many views through the reference-signature API then moves only the
    images.  Editing the scene's arrays in place while it is resident needs
    an explicit ``raster.invalidate(scene)`` (the reference's own callers
    that edit in place, such as fd_check, never use this cache)."""

    def __init__(self, scene):
        self.scene = scene

    def __enter__(self):
        _RESIDENT[id(self.scene)] = (self.scene, {})
        return self.scene

    def __exit__(self, *exc):
        _RESIDENT.pop(id(self.scene), None)


def invalidate(scene=None):
    """Drop the resident device copy of ``scene`` (all scenes when None): the
    next call re-uploads its arrays."""
    if scene is None:
        for _, (_, per) in _RESIDENT.items():
            per.clear()
    elif id(scene) in _RESIDENT:
        _RESIDENT[id(scene)][1].clear()


def _device_scene(scene, ws: engine.Workspace) -> engine.DeviceScene:
    """The scene's records on the workspace's device, re-uploaded every call
    (callers such as fd_check mutate arrays in place, so a copy kept across
    calls could go stale) unless the scene is :class:`resident`.

    The packed (n, 14+6C) record is built directly in a reused pinned staging
    buffer at the workspace's parameter precision -- float32 records are
    cast on the host (round to nearest even: the bits of pack_records and of
    a device cast), so 152 MB instead of 300 MB cross PCIe at 7D 1M -- by
    host threads over row chunks, then one DMA.  The staging buffer is reused
    by the next call only after this call's result has been read back (every
    numpy entry point synchronises)."""
    dtype = torch.float64 if ws.f64 else torch.float32
    n = int(np.asarray(scene.mu_x).shape[0])
    if n == 0 or not torch.cuda.is_available():
        return engine.DeviceScene.from_scene(scene, dtype=dtype, device=ws.device)
    hit = _RESIDENT.get(id(scene))
    if hit is not None and hit[0] is scene:
        ds = hit[1].get((str(ws.device), ws.precision))
        if ds is not None:
            return ds
    torch.cuda.current_stream(ws.device).synchronize()  # the previous call's uploads are done
    width = 14 + 6 * (int(scene.n_dims) - 3)
    st = _pinned("records", (n, width), dtype)
    dst = st.numpy()
    rec = _packed_records(scene, n)
    if rec is not None:  # every field is a view into one packed record array
        def fill(r0, r1):
            np.copyto(dst[r0:r1], rec[r0:r1], casting="unsafe")
    else:
        from .types import field_offsets
        fields = [(np.asarray(getattr(scene, k)).reshape(n, -1), off, size)
                  for k, (off, size, _shape) in field_offsets(int(scene.n_dims)).items() if size]

        def fill(r0, r1):
            for a, off, size in fields:
                np.copyto(dst[r0:r1, off:off + size], a[r0:r1], casting="unsafe")
    params = torch.empty((n, width), dtype=dtype, device=ws.device)
    if n < 1 << 18:
        fill(0, n)
        params.copy_(st, non_blocking=True)
    else:
        # _STAGE_PARTS row parts, each cut into one task per host thread and
        # queued in order: part k is cast before part k + 1, and its DMA
        # overlaps the later parts' casts
        workers = _pool()._max_workers
        bounds = [n * k // _STAGE_PARTS for k in range(_STAGE_PARTS + 1)]
        parts = list(zip(bounds[:-1], bounds[1:]))
        futs = []
        for h0, h1 in parts:
            step = -(-(h1 - h0) // workers)
            futs.append([_pool().submit(fill, r0, min(h1, r0 + step)) for r0 in range(h0, h1, step)])
        for (h0, h1), fs in zip(parts, futs):
            for f in fs:
                f.result()
            params[h0:h1].copy_(st[h0:h1], non_blocking=True)
    ds = engine.DeviceScene(params, scene.n_dims, scene.background)
    if hit is not None and hit[0] is scene:
        hit[1][(str(ws.device), ws.precision)] = ds
    return ds


def _host_image(fr: engine.Frame, background) -> np.ndarray:
    """(H, W, 3) float64; pixels nothing was composited into get the exact fp64
    background (acc = 0, T = 1 gives 0 + 1 * bg in tile_forward, _tiles.py:51-53).
    The widening and the background fix happen on the device; the 50 MB
    (1080p) float64 image comes back through a reused pinned buffer and is
    copied out by host threads."""
    H, W = fr.height, fr.width
    img = fr.image.view(H, W, 3).double()
    if not fr.raster_f64:
        empty = (fr.alpha_sum == 0) & (fr.t_stop == 1)
        bg = torch.as_tensor(np.asarray(background, dtype=np.float64).reshape(3), device=img.device)
        img = torch.where(empty[..., None], bg, img)
    if _PINNED_OUT[0] < _PINNED_OUT_MAX:
        # straight into a pinned block of torch's caching host allocator, which
        # the returned array keeps alive (and gives back when it is dropped):
        # no host copy.  Past _PINNED_OUT_MAX arrays still alive, the image goes
        # through the reused staging buffer into ordinary memory instead.
        t = torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True)
        t.copy_(img, non_blocking=True)
        torch.cuda.current_stream(fr.image.device).synchronize()
        out = t.numpy()
        _PINNED_OUT[0] += 1
        # on the tensor object the array holds (t.numpy()'s base is its own
        # alias of t's storage): released when the last view of it goes
        weakref.finalize(out.base, _pinned_out_released)
        return out
    st = _pinned("image", (H, W, 3), torch.float64)
    st.copy_(img, non_blocking=True)
    torch.cuda.current_stream(fr.image.device).synchronize()
    out = np.empty((H, W, 3), dtype=np.float64)
    src = st.numpy()
    _parallel_rows(H, lambda r0, r1: np.copyto(out[r0:r1], src[r0:r1]), min_rows=64)
    return out


class FrameCache:
    """Host view of one forward frame (reference raster.py:63-92).

    Eager: image, alpha_sum, t_stop, alpha_clamped, processed_pixels, order,
    n_contrib (per-pixel contributor count, not in the reference).
    Lazy, from a re-run of the same frame: ``tiles`` / ``tile_ranges`` /
    ``tile_ids`` (the full per-tile id lists), ``slices`` / ``proj`` (the
    reference's SliceCache / ProjectionCache with every field, from one
    device preprocess that dumps its fp64 intermediates).
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
        self._proj = None
        self._slices = None

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
        # one device preprocess of the same frame on the inline route (no
        # statics: every query-invariant intermediate is formed and dumped)
        if self._debug is None:
            ws = workspace(self.precision)
            ds = _device_scene(self.scene, ws)
            ds = engine.DeviceScene(ds.params, ds.n_dims, ds.background, use_statics=False)
            fr = engine.render_frame(ws, ds, self.camera, self.query, self.settings, want_debug=True,
                                     full_lists=True)
            self._debug = ws.debug[:fr.n * DEBUG_STRIDE].view(fr.n, DEBUG_STRIDE).cpu().numpy().copy()
        return self._debug

    @property
    def proj(self) -> ProjectionCache:
        """ProjectionCache of the frame (raster.py:46-60), from a debug run (lazy)."""
        if self._proj is None:
            d, f = self._dump(), self._flags
            n = d.shape[0]
            sym2 = lambda a, b, c: np.stack([np.stack([a, b], 1), np.stack([b, c], 1)], 1)  # noqa: E731
            o = DEBUG["cov2_eig"]
            self._proj = ProjectionCache(
                t_cam=d[:, 19:22], depth=d[:, 0], mean2=d[:, 1:3], vmat=d[:, DEBUG["vmat"]:o].reshape(n, 2, 3),
                cov2_eigval=d[:, o:o + 2], cov2_eigvec=d[:, o + 2:o + 6].reshape(n, 2, 2),
                floored=(f & F_FLOOR2) != 0, cov2=sym2(d[:, 10], d[:, 11], d[:, 12]),
                p2=sym2(d[:, 3], d[:, 4], d[:, 5]), radii=d[:, 6:8], visible=(f & F_VISIBLE) != 0)
        return self._proj

    @property
    def slices(self) -> SliceCache:
        """SliceCache of the frame (slicing.py:153-182), from a debug run (lazy)."""
        if self._slices is None:
            d, f = self._dump(), self._flags
            n = d.shape[0]
            c = self.scene.n_dims - 3
            i = [0, 1, 2, 1, 3, 4, 2, 4, 5]
            col = lambda name: d[:, DEBUG[name]:DEBUG[name] + c]  # noqa: E731
            e3 = DEBUG["cov3_eig"]
            self._slices = SliceCache(
                valid=(f & F_DEGENERATE) == 0, mean3=d[:, 22:25], cov3=d[:, 13:19][:, i].reshape(-1, 3, 3),
                beta_x=d[:, 9], gated_opacity=d[:, 8], color=d[:, DEBUG["color"]:DEBUG["color"] + 3],
                opacity=d[:, 26], gate=d[:, 25], beta_q=col("beta_q"), delta=col("delta"),
                m_inv=d[:, DEBUG["m_inv"]:DEBUG["m_inv"] + 16].reshape(n, 4, 4)[:, :c, :c],
                u=col("u"), v=col("v"),
                sigma_xq=d[:, DEBUG["sigma_xq"]:DEBUG["sigma_xq"] + 12].reshape(n, 3, 4)[:, :, :c],
                d_raw=col("d_raw"), s_tanh=d[:, 27:27 + c], d_gate=col("d_gate"),
                cov3_eigval=d[:, e3:e3 + 3], cov3_eigvec=d[:, e3 + 3:e3 + 12].reshape(n, 3, 3),
                floor_eps=d[:, 31], floored=(f & F_FLOOR3) != 0,
                l_x=d[:, DEBUG["l_x"]:DEBUG["l_x"] + 9].reshape(n, 3, 3),
                rotation=d[:, DEBUG["rot"]:DEBUG["rot"] + 9].reshape(n, 3, 3),
                s_x=d[:, DEBUG["s_x"]:DEBUG["s_x"] + 3], s_q=col("s_q"))
        return self._slices

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
