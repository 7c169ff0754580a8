"""Device-resident render engine: HBM scene, per-frame workspaces, stage driver.

The engine strings the C-ABI stages together on one CUDA stream:

    ubs_preprocess -> ubs_bin_depth -> (read K) -> ubs_bin_tiles -> ubs_raster_forward
    [ubs_loss_image_grad] -> ubs_raster_backward -> ubs_prim_backward

Buffers are torch tensors (PyTorch is the device allocator and stream owner;
the kernels are ours).  Workspaces grow geometrically and are reused across
frames, so a steady-state frame allocates nothing.  One 16-byte device->host
read per frame fetches the tile-pair count K before the pair buffers are
used; everything else is stream ordered.

Precision modes (``precision=``):
  * ``"fp32"``: fp32 records and raster, fp64 preprocess, fp64 fix-up of the
    pixels whose cut/clamp decisions are not certified in fp32 -> integer
    outputs bit-exact, images within ~1e-5 of the reference;
  * ``"fp64"``: fp64 records and raster with the reference's operation order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import (GRAD2D_STRIDE, REC32_BYTES, REC64_BYTES, UbsBinBuffers, UbsCamera, UbsGradBuffers,
                   UbsImageBuffers, UbsPrimBuffers, UbsSettings, UbsView, check)
from .types import DEFAULT_SETTINGS, PARAM_FIELDS, pack_records, record_width

TILE = 16


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _require_cuda(device) -> torch.device:
    dev = torch.device(device)
    if dev.type != "cuda":
        raise _lib.UbsError("the UBS engine runs on CUDA devices only (no CPU fallback)")
    if not torch.cuda.is_available():
        raise _lib.UbsError("no CUDA device available: the UBS engine has no CPU fallback")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


class DeviceScene:
    """A scene resident in HBM as packed UBS1 records (n x (14+6C)).

    Also caches the scene statics (ubs_scene_statics: the query-invariant
    half of slice_scene) for the current parameter version; every view of
    the same parameters reuses them.  The cache key is the params tensor's
    storage and in-place version counter (code that writes the records
    behind torch's back, like DeviceAdam, bumps it) plus psd_floor_scale.
    ``use_statics=False`` makes every preprocess derive them inline."""

    def __init__(self, params: torch.Tensor, n_dims: int, background, use_statics: bool = True):
        if params.dim() != 2 or params.shape[1] != record_width(n_dims):
            raise ValueError("params must be (n, 14+6C)")
        if params.dtype not in (torch.float32, torch.float64):
            raise ValueError("params must be float32 or float64")
        self.n_dims = int(n_dims)
        self.background = tuple(float(b) for b in np.asarray(background, dtype=np.float64).reshape(3))
        self.use_statics = bool(use_statics)
        self._statics = None
        self._statics_key = None
        self.params = params.contiguous()

    @property
    def params(self) -> torch.Tensor:
        return self._params

    @params.setter
    def params(self, t: torch.Tensor):
        self._params = t
        self._statics_key = None

    def invalidate_statics(self):
        self._statics_key = None

    def statics_bytes_per_prim(self) -> float:
        f64 = 1 if self._params.dtype == torch.float64 else 0
        return _lib.load().ubs_statics_bytes(1 << 20, self.n_dims, f64) / float(1 << 20)

    def statics_ptr(self, settings, readers=()) -> int:
        """Device pointer of up-to-date scene statics (recomputed on the
        current stream when the parameters changed), or 0 when disabled.

        ``readers``: streams that may still be reading the current statics
        (a pipeline's slot / lead streams).  Before the buffer is recomputed
        in place (or reallocated) the current stream waits for all of them,
        so a frame in flight never sees statics change under it."""
        if not self.use_statics or self.n == 0:
            return 0
        p = self._params
        key = (p.data_ptr(), p._version, float(settings.psd_floor_scale))
        if key != self._statics_key:
            if self._statics is not None:
                cur = torch.cuda.current_stream(p.device)
                for s in readers:
                    if s is not None and s != cur:
                        cur.wait_stream(s)
            lib = _lib.load()
            f64 = 1 if p.dtype == torch.float64 else 0
            nbytes = int(lib.ubs_statics_bytes(self.n, self.n_dims, f64))
            if self._statics is None or self._statics.numel() < nbytes:
                self._statics = torch.empty(nbytes, dtype=torch.uint8, device=p.device)
            v = UbsView()
            v.params = _ptr(p)
            v.n = self.n
            v.n_dims = self.n_dims
            v.param_f64 = f64
            v.set.psd_floor_scale = float(settings.psd_floor_scale)
            check(lib.ubs_scene_statics(v, _ptr(self._statics), _stream_ptr()), "ubs_scene_statics")
            self._statics_key = key
        return _ptr(self._statics)

    @classmethod
    def from_scene(cls, scene, dtype=torch.float32, device="cuda") -> "DeviceScene":
        dev = _require_cuda(device)
        npdt = np.float64 if dtype == torch.float64 else np.float32
        n = int(np.asarray(scene.mu_x).shape[0])
        if n == 0:
            return cls(torch.from_numpy(pack_records(scene, npdt)).to(dev), scene.n_dims, scene.background)
        # each field uploaded as float64 (no host pass for contiguous float64 arrays),
        # interleaved and cast on the device: round-to-nearest-even, the same bits
        # as pack_records' host cast
        cols = [torch.from_numpy(np.ascontiguousarray(
                    np.asarray(getattr(scene, k), dtype=np.float64).reshape(n, -1))).to(dev)
                for k, _ in PARAM_FIELDS]
        return cls(torch.cat(cols, dim=1).to(dtype).contiguous(), scene.n_dims, scene.background)

    @property
    def n(self) -> int:
        return int(self.params.shape[0])

    @property
    def device(self):
        return self.params.device


def view_struct(n: int, n_dims: int, param_f64: bool, background, cam, query, settings=DEFAULT_SETTINGS,
                params_ptr: int = 0, statics_ptr: int = 0) -> UbsView:
    """The C-ABI UbsView of one frame from reference-shaped objects (host
    only; duck-typed: betasplat's Camera / Query / RenderSettings work as well
    as this package's mirrors and give the same bytes)."""
    if int(settings.tile_size) != TILE:
        raise ValueError("tile_size must be 16 on the device path")
    c = n_dims - 3
    q = np.asarray(query.dims, dtype=np.float64).reshape(-1)
    if q.shape[0] != c:
        raise ValueError(f"query has {q.shape[0]} dims, scene expects {c}")
    v = UbsView()
    v.params = params_ptr
    v.n = n
    v.n_dims = n_dims
    v.param_f64 = 1 if param_f64 else 0
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    for k in range(3):
        v.background[k] = float(bg[k])
    for k in range(4):
        v.query[k] = float(q[k]) if k < c else 0.0
    w2c = np.asarray(cam.world_to_cam, dtype=np.float64).reshape(4, 4)
    cc = UbsCamera()
    cc.fx, cc.fy, cc.cx, cc.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    for i in range(3):
        for j in range(3):
            cc.rot[3 * i + j] = w2c[i, j]
        cc.trans[i] = w2c[i, 3]
    cc.width, cc.height = int(cam.width), int(cam.height)
    v.cam = cc
    st = UbsSettings()
    st.tau_sq = float(settings.tau_sq)
    st.alpha_clamp = float(settings.alpha_clamp)
    st.transmittance_min = float(settings.transmittance_min)
    st.near_plane = float(settings.near_plane)
    st.cull_margin = float(settings.cull_margin)
    st.screen_cov_floor = float(settings.screen_cov_floor)
    st.psd_floor_scale = float(settings.psd_floor_scale)
    st.gate_symmetric = 1 if settings.gate_symmetric else 0
    st.tile_size = TILE
    v.set = st
    v.statics = statics_ptr
    return v


def make_view(ds: DeviceScene, cam, query, settings=DEFAULT_SETTINGS) -> UbsView:
    if int(settings.tile_size) != TILE:
        raise ValueError("tile_size must be 16 on the device path")
    return view_struct(ds.n, ds.n_dims, ds.params.dtype == torch.float64, ds.background, cam, query, settings,
                       params_ptr=_ptr(ds.params), statics_ptr=ds.statics_ptr(settings))


@dataclass
class Frame:
    """Device-side result of one forward frame (views into engine workspaces).

    The tensors are overwritten by the next frame rendered with the same
    workspace; clone what you keep.
    """

    view: UbsView
    width: int
    height: int
    n: int
    n_visible_host: int | None  # known when rendered with sync=True
    n_pairs_host: int | None
    image: torch.Tensor       # (H, W, 3)
    alpha_sum: torch.Tensor   # (H, W)
    t_stop: torch.Tensor      # (H, W)
    n_contrib: torch.Tensor   # (H, W) int32
    hit_clamp: torch.Tensor   # (n,) uint8
    ws: "Workspace"
    raster_f64: bool

    @property
    def n_visible(self) -> int:
        if self.n_visible_host is None:
            self.n_visible_host = int(self.ws.counters32[4].item())
        return self.n_visible_host

    @property
    def n_pairs(self) -> int:
        if self.n_pairs_host is None:
            self.n_pairs_host = int(self.ws.counters[0].item())
        return self.n_pairs_host

    @property
    def processed_pixels(self) -> int:
        return int(self.ws.counters[1].item())

    @property
    def n_fixed(self) -> int:
        return int(self.ws.counters32[6].item())


class Workspace:
    """Every device buffer one frame needs; grows on demand, reused across frames."""

    def __init__(self, device, precision: str = "fp32"):
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        self.device = _require_cuda(device)
        self.precision = precision
        self.f64 = precision == "fp64"
        # fp32 raster kernels: packed fp32x2 pairs (default) or one pixel per lane
        # (the same per-pixel arithmetic; kept selectable for A/B and tests)
        self.raster_scalar = False
        self.lib = _lib.load()
        self.n_cap = 0
        self.pix_cap = 0
        self.tile_cap = 0
        self.pair_cap = 0
        self.temp_bytes = 0
        # [0] n_pairs u64 | [1] visits u64 | [2] lo: n_visible u32 | [3] lo: fix_count u32 |
        # [5] min visible depth key | [6] max visible depth key
        self.counters = torch.zeros(8, dtype=torch.int64, device=self.device)
        self.counters32 = self.counters.view(torch.int32)
        self.debug = None
        self.tile_grid = None
        self.chunk_hist = None
        self.seg_scratch = None
        self.bucket_start = None
        self.chunk_count = 0
        self.grad2d = None
        self.grad2d_clean = False  # True while grad2d is all-zero (ubs_prim_backward consumed it)
        self.loss_scratch = None
        self.loss_parts = torch.zeros(2, dtype=torch.float64, device=self.device)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)  # UBS_S_* bits, sticky
        self.active = None
        self.active_count = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.det_partials = None  # deterministic backward: K x 10 tile partials, slot offsets, scan scratch
        self.det_slot_off = None
        self.det_temp = None
        # materialised prefix of each tile list (grows x2 when a frame needs more)
        self.list_cap = 1024
        self.frame_list_cap = self.list_cap

    # --- allocation -------------------------------------------------------
    def _i(self, n, dtype):
        return torch.empty(max(int(n), 1), dtype=dtype, device=self.device)

    def ensure_prims(self, n: int):
        if n <= self.n_cap:
            return
        cap = max(n, int(self.n_cap * 1.25))
        self.depth_key = self._i(cap, torch.int64)
        self.rect = self._i(cap, torch.int64)
        self.tile_count = self._i(cap, torch.int32)
        self.flags = self._i(cap, torch.int16)
        self.rec64 = self._i(cap * REC64_BYTES // 8, torch.float64)
        self.rec32 = None if self.f64 else self._i(cap * REC32_BYTES // 4, torch.float32)
        self.keys_sorted = self._i(cap, torch.int64)
        self.rect_sorted = self._i(cap, torch.int64)
        self.ids_iota = self._i(cap, torch.int32)
        self.order = self._i(cap, torch.int32)
        self.hit_clamp = self._i(cap, torch.uint8)
        self.n_cap = cap
        self.temp_bytes = 0  # CUB scratch depends on n

    def ensure_pixels(self, width: int, height: int):
        npix = width * height
        ntiles = math.ceil(width / TILE) * math.ceil(height / TILE)
        fdt = torch.float64 if self.f64 else torch.float32
        if npix > self.pix_cap:
            cap = npix
            self.image_buf = self._i(cap * 3, fdt)
            self.asum_buf = self._i(cap, fdt)
            self.tstop_buf = self._i(cap, fdt)
            self.ncontrib_buf = self._i(cap, torch.int32)
            self.fix_list = self._i(cap, torch.int32)
            self.g_image_buf = self._i(cap * 3, fdt)
            self.loss_scratch = None
            self.pix_cap = cap
        grid = (math.ceil(width / TILE) + 1) * (math.ceil(height / TILE) + 1)
        if self.tile_grid is None or self.tile_grid.numel() < grid:
            self.tile_grid = self._i(grid, torch.int32)
        if ntiles > self.tile_cap:
            self.tile_ranges = self._i(2 * ntiles, torch.int32)
            self.tile_cap = ntiles
            self.temp_bytes = 0

    CHUNK_RANKS = 1024  # ranks per level-1 binning CTA chunk (csrc/binning.cu kCtaRanks)
    BAND = 8            # tile columns per level-1 bucket (csrc/binning.cu kBand)
    ROWS = 4            # tile rows per level-1 bucket (csrc/binning.cu kRows)

    def ensure_chunks(self, n: int, width: int, height: int):
        tx, ty = math.ceil(width / TILE), math.ceil(height / TILE)
        nbk = math.ceil(ty / self.ROWS) * math.ceil(tx / self.BAND)
        g = max(1, -(-n // self.CHUNK_RANKS))
        self.chunk_count = g
        need = (2 + 8) * g * nbk  # chunk totals | chunk offsets | per-warp counts (8 warps per chunk)
        if self.chunk_hist is None or self.chunk_hist.numel() < need:
            self.chunk_hist = self._i(need, torch.int32)
        if self.seg_scratch is None or self.seg_scratch.numel() < nbk + 1:
            self.seg_scratch = self._i(nbk + 1, torch.int32)  # bucket totals | ticket
            self.bucket_start = self._i(nbk + 1, torch.int32)

    def ensure_pairs(self, k: int):
        if k > self.pair_cap:
            # headroom so asynchronous frames of a sweep rarely outgrow it
            cap = max(int(k * 1.2), int(self.pair_cap * 1.3), 1024)
            self.tile_ids = self._i(cap, torch.int32)
            self.entries = self._i(cap, torch.int64)
            self.pair_cap = cap
        need = int(self.lib.ubs_bin_temp_bytes(self.n_cap, self.pair_cap, self.tile_cap))
        if need > self.temp_bytes:
            self.temp = self._i(need, torch.uint8)
            self.temp_bytes = need

    # --- C structs --------------------------------------------------------
    def prim_buffers(self, want_debug=False) -> UbsPrimBuffers:
        pb = UbsPrimBuffers()
        pb.depth_key = _ptr(self.depth_key)
        pb.rect = _ptr(self.rect)
        pb.tile_count = _ptr(self.tile_count)
        pb.flags = _ptr(self.flags)
        pb.rec32 = _ptr(self.rec32)
        pb.rec64 = _ptr(self.rec64)
        pb.debug = _ptr(self.debug) if want_debug else 0
        pb.n_visible = _ptr(self.counters) + 16
        pb.n_pairs = _ptr(self.counters)
        pb.tile_grid = _ptr(self.tile_grid)
        pb.depth_range = _ptr(self.counters) + 40
        return pb

    def bin_buffers(self) -> UbsBinBuffers:
        bb = UbsBinBuffers()
        bb.keys_sorted = _ptr(self.keys_sorted)
        bb.rect_sorted = _ptr(self.rect_sorted)
        bb.ids_iota = _ptr(self.ids_iota)
        bb.order = _ptr(self.order)
        if self.pair_cap:
            bb.tile_ids = _ptr(self.tile_ids)
            bb.entries = _ptr(self.entries)
        bb.tile_ranges = _ptr(self.tile_ranges)
        bb.pair_capacity = self.pair_cap
        bb.temp = _ptr(self.temp) if self.temp_bytes else 0
        bb.temp_bytes = self.temp_bytes
        if self.chunk_hist is not None:
            bb.chunk_hist = _ptr(self.chunk_hist)
            bb.chunk_hist_capacity = self.chunk_hist.numel()
            bb.chunk_count = self.chunk_count
            bb.seg_scratch = _ptr(self.seg_scratch)
            bb.bucket_start = _ptr(self.bucket_start)
            bb.bucket_capacity = self.bucket_start.numel()
        bb.status = _ptr(self.status)
        bb.list_cap = self.frame_list_cap
        return bb

    def image_buffers(self) -> UbsImageBuffers:
        ib = UbsImageBuffers()
        ib.image = _ptr(self.image_buf)
        ib.alpha_sum = _ptr(self.asum_buf)
        ib.t_stop = _ptr(self.tstop_buf)
        ib.n_contrib = _ptr(self.ncontrib_buf)
        ib.hit_clamp = _ptr(self.hit_clamp)
        ib.visits = _ptr(self.counters) + 8
        ib.fix_list = _ptr(self.fix_list)
        ib.fix_count = _ptr(self.counters) + 24
        ib.raster_f64 = 1 if self.f64 else 0
        ib.raster_scalar = 1 if self.raster_scalar else 0
        return ib


def _stream_ptr() -> int:
    return int(torch.cuda.current_stream().cuda_stream)


class _Timed:
    """Records a CUDA event pair around a stage on the current stream when
    ``timers`` (name -> list of (start, end) events) is given."""

    def __init__(self, timers, name):
        self.timers, self.name = timers, name

    def __enter__(self):
        if self.timers is not None:
            self.a = torch.cuda.Event(enable_timing=True)
            self.a.record()

    def __exit__(self, *exc):
        if self.timers is not None:
            b = torch.cuda.Event(enable_timing=True)
            b.record()
            self.timers.setdefault(self.name, []).append((self.a, b))


def render_frame(ws: Workspace, ds: DeviceScene, cam, query, settings=DEFAULT_SETTINGS,
                 want_debug: bool = False, timers: dict | None = None, sync: bool = True,
                 full_lists: bool = False) -> Frame:
    """Forward one frame on the current stream; returns device views.

    ``sync=True`` reads the frame's tile-pair count K back (one 16-byte copy)
    and grows the pair buffers to fit before binning.  ``sync=False`` keeps
    the whole frame asynchronous: the kernels check K against the current
    capacity on the device and set ``ws.status`` (UBS_S_PAIR_OVERFLOW)
    instead of overflowing; call :func:`check_status` (or render the frame
    again with ``sync=True``) before trusting an async frame whose K may have
    grown.  ``timers``: optional dict collecting per-stage CUDA event pairs.

    Tile lists are materialised only up to ``ws.list_cap`` ids per tile (the
    rasterizer stops long before; ``full_lists=True`` materialises them all,
    e.g. for FrameCache.tiles).  A frame that needed more sets
    UBS_S_LIST_TRUNC: synchronous frames then double the cap and re-render,
    asynchronous ones leave it to :func:`check_status`."""
    v, pb = _frame_begin(ws, ds, cam, query, settings, want_debug)
    with _Timed(timers, "preprocess"):
        check(ws.lib.ubs_preprocess(v, pb, 0 if ws.f64 else 1, _stream_ptr()), "ubs_preprocess")
    return _frame_end(ws, ds, v, pb, cam, query, settings, want_debug, timers, sync, full_lists)


def _frame_begin(ws: Workspace, ds: DeviceScene, cam, query, settings, want_debug: bool):
    """Size the workspace for the frame and reset its counters (current stream)."""
    if ds.device != ws.device:
        raise ValueError("scene and workspace live on different devices")
    v = make_view(ds, cam, query, settings)
    W, H, n = int(cam.width), int(cam.height), ds.n
    ws.ensure_prims(max(n, 1))
    ws.ensure_pixels(W, H)
    ws.ensure_chunks(n, W, H)
    if want_debug:
        if ws.debug is None or ws.debug.numel() < n * _lib.DEBUG_STRIDE:
            ws.debug = torch.zeros(max(n, 1) * _lib.DEBUG_STRIDE, dtype=torch.float64, device=ws.device)
    if ws.temp_bytes == 0:
        ws.ensure_pairs(0)
    ws.counters.zero_()
    return v, ws.prim_buffers(want_debug)


def _frame_end(ws: Workspace, ds: DeviceScene, v, pb, cam, query, settings, want_debug, timers, sync,
               full_lists) -> Frame:
    """Binning, raster and fix-up of a preprocessed frame (current stream)."""
    lib = ws.lib
    W, H, n = int(cam.width), int(cam.height), ds.n
    s = _stream_ptr()
    with _Timed(timers, "bin_depth"):
        check(lib.ubs_bin_depth(v, pb, ws.bin_buffers(), s), "ubs_bin_depth")
    if sync or ws.pair_cap == 0:
        host = ws.counters[:3].cpu()  # K and n_visible (16 bytes)
        k = int(host[0])
        n_vis = int(host.view(torch.int32)[4])
        if k >= 2 ** 32:
            raise _lib.UbsError(f"{k} tile pairs exceed the 2^32 device limit")
        ws.ensure_pairs(k)
    else:
        k, n_vis = None, None
    ws.frame_list_cap = _lib.FULL_LISTS if full_lists else ws.list_cap
    bb = ws.bin_buffers()
    with _Timed(timers, "bin_tiles"):
        check(lib.ubs_bin_tiles(v, pb, bb, -1 if k is None else k, s), "ubs_bin_tiles")
    ws.hit_clamp[:max(n, 1)].zero_()
    ib = ws.image_buffers()
    with _Timed(timers, "raster"):
        check(lib.ubs_raster_forward(v, pb, bb, ib, s), "ubs_raster_forward")
    if not ws.f64:
        with _Timed(timers, "fixup"):
            check(lib.ubs_raster_fixup(v, pb, bb, ib, s), "ubs_raster_fixup")
    if sync and not full_lists:
        st = int(ws.status.item())
        if st & _lib.S_LIST_TRUNC:
            ws.status.zero_()
            ws.list_cap *= 2
            return render_frame(ws, ds, cam, query, settings, want_debug, timers, sync, full_lists)
    npix = W * H
    return Frame(view=v, width=W, height=H, n=n, n_visible_host=n_vis, n_pairs_host=k,
                 image=ws.image_buf[:npix * 3].view(H, W, 3), alpha_sum=ws.asum_buf[:npix].view(H, W),
                 t_stop=ws.tstop_buf[:npix].view(H, W), n_contrib=ws.ncontrib_buf[:npix].view(H, W),
                 hit_clamp=ws.hit_clamp[:n], ws=ws, raster_f64=ws.f64)


def list_stats(ws: "Workspace", fr: "Frame") -> tuple[int, int]:
    """(level-1 bucket entries, tile-list ids materialised) of the last frame
    rendered with ``ws`` (synchronises; for reporting only)."""
    W, H = fr.width, fr.height
    TX, TY = -(-W // TILE), -(-H // TILE)
    nbk = -(-TY // Workspace.ROWS) * -(-TX // Workspace.BAND)
    entries = int(ws.bucket_start[nbk].item()) & 0xFFFFFFFF if ws.bucket_start is not None else 0
    rng = ws.tile_ranges[:2 * TX * TY].view(-1, 2).long()
    lens = (rng[:, 1] - rng[:, 0]).clamp_(min=0)
    cap = ws.frame_list_cap
    if 0 < cap < (1 << 31):
        lens = lens.clamp_(max=cap)
    return entries, int(lens.sum().item())


class FramePipeline:
    """Several frames in flight for a sweep of independent views.

    Frame k renders on stream k % depth with that slot's own Workspace, so
    the stages of consecutive frames overlap on the GPU: one frame's
    latency-bound preprocess, single-CTA scans and fix-up tail run beside
    another frame's issue-bound raster (7D 1M 1080p: 1428 fps with one frame
    in flight, 1780 with three).  The scene statics are brought up to date on
    the caller's stream before a frame is dispatched, and every slot stream
    first waits for the caller's stream, so work the caller enqueued earlier
    (scene uploads, parameter updates) is visible to the frame.

    A returned Frame lives in its slot's buffers until the slot comes round
    again (``depth`` frames later); consume it on ``stream_of(frame)`` or
    after :meth:`join`."""

    def __init__(self, ds: DeviceScene, depth: int = 3, precision: str = "fp32", device=None,
                 slot_priority: int = 0, lead_priority: int = 0):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        dev = _require_cuda(device if device is not None else ds.device)
        self.ds = ds
        self.workspaces = [Workspace(dev, precision) for _ in range(depth)]
        self.streams = [torch.cuda.Stream(dev, priority=slot_priority) for _ in range(depth)]
        self.pending = [None] * depth  # event a slot's next frame must wait for (a consumer of its buffers)
        self.k = 0
        self.lead = torch.cuda.Stream(dev, priority=lead_priority)  # render_group's shared preprocess

    @property
    def depth(self) -> int:
        return len(self.streams)

    def readers(self) -> list:
        """Every stream of this pipeline that reads the scene statics."""
        return self.streams + [self.lead]

    def render(self, cam, query, settings=DEFAULT_SETTINGS, *, sync: bool = False, timers: dict | None = None,
               full_lists: bool = False) -> Frame:
        i = self.k % self.depth
        self.k += 1
        self.ds.statics_ptr(settings, self.readers())  # (re)computed on the caller's stream if stale
        s = self.streams[i]
        s.wait_stream(torch.cuda.current_stream())
        if self.pending[i] is not None:
            s.wait_event(self.pending[i])
            self.pending[i] = None
        with torch.cuda.stream(s):
            return render_frame(self.workspaces[i], self.ds, cam, query, settings, timers=timers, sync=sync,
                                full_lists=full_lists)

    def render_group(self, views, settings=DEFAULT_SETTINGS) -> list:
        """Render up to ``depth`` (camera, query) pairs as consecutive frames of
        the pipeline, with ONE preprocess for all of them
        (``ubs_preprocess_views``: the scene statics are read once per
        group instead of once per frame).  The group's slots must be free, so
        the preprocess waits for the frames that last used them; with
        ``depth`` = 2 x group size the next group's preprocess overlaps this
        group's rasters.  Frames are asynchronous (``check_status``)."""
        views = list(views)
        if not views:
            return []
        if len(views) > self.depth:
            raise ValueError("a group cannot exceed the pipeline depth")
        ds = self.ds
        if not ds.statics_ptr(settings, self.readers()):  # no statics (empty scene, use_statics=False): frame by frame
            return [self.render(cam, q, settings) for cam, q in views]
        slots = [(self.k + j) % self.depth for j in range(len(views))]
        self.k += len(views)
        lead = self.lead
        lead.wait_stream(torch.cuda.current_stream())
        for i in slots:
            lead.wait_stream(self.streams[i])
            if self.pending[i] is not None:
                lead.wait_event(self.pending[i])
                self.pending[i] = None
        vs, pbs = [], []
        with torch.cuda.stream(lead):
            for (cam, q), i in zip(views, slots):
                v, pb = _frame_begin(self.workspaces[i], ds, cam, q, settings, False)
                vs.append(v)
                pbs.append(pb)
            ws0 = self.workspaces[slots[0]]
            va = (_lib.UbsView * len(vs))(*vs)
            pa = (_lib.UbsPrimBuffers * len(pbs))(*pbs)
            check(ws0.lib.ubs_preprocess_views(va, pa, len(vs), 0 if ws0.f64 else 1, lead.cuda_stream),
                  "ubs_preprocess_views")
            ev = torch.cuda.Event()
            ev.record(lead)
        frames = []
        for (cam, q), i, v, pb in zip(views, slots, vs, pbs):
            s = self.streams[i]
            s.wait_event(ev)
            with torch.cuda.stream(s):
                frames.append(_frame_end(self.workspaces[i], ds, v, pb, cam, q, settings, False, None, False,
                                         False))
        return frames

    def stream_of(self, fr: Frame) -> torch.cuda.Stream:
        return self.streams[self.workspaces.index(fr.ws)]

    def hold(self, fr: Frame, event: torch.cuda.Event):
        """Keep ``fr``'s buffers until ``event`` (e.g. a host copy reading them)
        completes: the slot's next frame waits for it."""
        self.pending[self.workspaces.index(fr.ws)] = event

    def join(self):
        """Make the caller's stream wait for every frame issued so far."""
        cur = torch.cuda.current_stream()
        for s in self.streams:
            cur.wait_stream(s)

    def check_status(self) -> int:
        """check_status over every slot (syncs); raises if any frame overflowed."""
        self.join()
        st = 0
        err = None
        for ws in self.workspaces:
            try:
                st |= check_status(ws)
            except _lib.UbsError as e:  # grow every slot before re-raising
                err = e
        if err is not None:
            raise err
        return st

    def clear_status(self):
        for ws in self.workspaces:
            ws.status.zero_()

    def grow(self) -> int:
        """After asynchronous frames outgrew their slots (``status()`` nonzero):
        give every slot the largest tile-list cap any slot has -- doubled if a
        list was truncated -- and pair buffers for the largest tile-pair count
        any slot last saw, then clear the status.  A frame may land on any
        slot, so growing only the slot that overflowed is not enough.  Syncs;
        returns the status that was cleared."""
        self.join()
        torch.cuda.current_stream().synchronize()
        st = 0
        for ws in self.workspaces:
            st |= int(ws.status.item())
        cap = max(ws.list_cap for ws in self.workspaces)
        if st & _lib.S_LIST_TRUNC:
            cap *= 2
        k = max(int(ws.counters[0].item()) for ws in self.workspaces)
        if st & _lib.S_PAIR_OVERFLOW:  # the overflowing frame need not be any slot's last one
            k = max(k, int(max(ws.pair_cap for ws in self.workspaces) * 1.3) + 1)
        for ws in self.workspaces:
            ws.list_cap = cap
            if ws.temp_bytes:
                ws.ensure_pairs(k)
            ws.status.zero_()
        return st

    def status(self) -> torch.Tensor:
        """OR of the slots' device status words (no sync)."""
        out = self.workspaces[0].status.clone()
        for ws in self.workspaces[1:]:
            out |= ws.status
        return out


def check_status(ws: Workspace) -> int:
    """Raise if any asynchronous frame since the last reset overflowed its pair
    buffers (its outputs are invalid; re-render with sync=True).  Syncs."""
    st = int(ws.status.item())
    if st & (_lib.S_PAIR_OVERFLOW | _lib.S_LIST_TRUNC):
        ws.status.zero_()
        if st & _lib.S_LIST_TRUNC:
            ws.list_cap *= 2
        raise _lib.UbsError("an asynchronous frame outgrew its pair buffers or tile-list cap (capacity grown); "
                            "re-render it")
    return st


def loss_image_grad(fr: Frame, target: torch.Tensor, lambda_ssim: float, scale: float):
    """L1 + SSIM image gradient into the workspace g_image buffer.

    Returns (g_image view, loss_parts tensor [sum|diff|, sum ssim_map]) — the
    parts are accumulated (zero ``ws.loss_parts`` to start a batch)."""
    ws = fr.ws
    H, W = fr.height, fr.width
    f64 = 1 if fr.raster_f64 else 0
    tgt = target.to(device=ws.device, dtype=fr.image.dtype).contiguous()
    need = int(ws.lib.ubs_loss_scratch_bytes(H, W, f64))
    if ws.loss_scratch is None or ws.loss_scratch.numel() < need:
        ws.loss_scratch = torch.empty(need, dtype=torch.uint8, device=ws.device)
    g = ws.g_image_buf[:H * W * 3]
    check(ws.lib.ubs_loss_image_grad(_ptr(fr.image), _ptr(tgt), H, W, f64, float(lambda_ssim), float(scale),
                                     _ptr(g), _ptr(ws.loss_parts), _ptr(ws.loss_scratch), _stream_ptr()),
          "ubs_loss_image_grad")
    return g.view(H, W, 3), ws.loss_parts


def backward_frame(fr: Frame, ds: DeviceScene, g_image: torch.Tensor, grad_params: torch.Tensor,
                   add_regularisers: bool = False, reg_opacity: float = 0.0, reg_scale: float = 0.0,
                   deterministic: bool = False):
    """Accumulate d(loss)/d(params) of one frame into ``grad_params`` (n x P)."""
    gb = backward_raster(fr, ds, g_image, grad_params, reg_opacity, reg_scale, deterministic=deterministic)
    if gb is not None:
        backward_chain(fr, gb, add_regularisers)


def backward_raster(fr: Frame, ds: DeviceScene, g_image: torch.Tensor, grad_params: torch.Tensor,
                    reg_opacity: float = 0.0, reg_scale: float = 0.0, pixels_per_lane: int = 4,
                    deterministic: bool = False):
    """First half of :func:`backward_frame` on the current stream: the
    raster backward into the frame's screen-space sums (ws.grad2d).  Returns
    the UbsGradBuffers for :func:`backward_chain` (None for an empty scene).
    ``pixels_per_lane`` picks the fp32 raster backward's layout (4: two
    packed fp32x2 pixel pairs per lane, the fastest alone and beside other
    views' kernels; 2 and 8: one pixel per lane; same results).
    ``deterministic``: per-(primitive, tile) partials reduced in a fixed
    order instead of float atomics -- bit-identical sums on every run
    (raster.py:1-8, gradients.py:164-173), at the cost of a K x 10 buffer
    and a slower one-warp-per-tile walk."""
    ws = fr.ws
    n = fr.n
    if n == 0:
        return None
    gdt = torch.float64 if fr.raster_f64 else torch.float32
    if ws.grad2d is None or ws.grad2d.numel() < n * GRAD2D_STRIDE or ws.grad2d.dtype != gdt:
        ws.grad2d = torch.zeros(ws.n_cap * GRAD2D_STRIDE, dtype=gdt, device=ws.device)
        ws.grad2d_clean = True
    # ubs_prim_backward leaves the sums all-zero; zero them here only if the
    # last raster backward was not followed by its chain (an error between them)
    if not ws.grad2d_clean:
        ws.grad2d[:n * GRAD2D_STRIDE].zero_()
    ws.grad2d_clean = False
    g_img = g_image.to(device=ws.device, dtype=fr.image.dtype).contiguous()
    if grad_params.shape != ds.params.shape or not grad_params.is_contiguous():
        raise ValueError("grad_params must be a contiguous (n, 14+6C) tensor")
    gb = UbsGradBuffers()
    gb.g_image = _ptr(g_img)
    gb.grad2d = _ptr(ws.grad2d)
    gb.grad_params = _ptr(grad_params)
    gb.grad_f64 = 1 if grad_params.dtype == torch.float64 else 0
    gb.grad2d_f64 = 1 if fr.raster_f64 else 0
    gb.reg_opacity = float(reg_opacity)
    gb.reg_scale = float(reg_scale)
    gb.nonfinite = _ptr(ws.nonfinite)
    if ws.active is None or ws.active.numel() < n:
        ws.active = torch.empty(ws.n_cap, dtype=torch.int32, device=ws.device)
    gb.flags = _ptr(ws.flags)
    gb.active = _ptr(ws.active)
    gb.active_count = _ptr(ws.active_count)
    gb.bwd_pixels_per_lane = int(pixels_per_lane)
    if deterministic:
        esz = 8 if fr.raster_f64 else 4
        need = ws.pair_cap * 10 * esz
        if ws.det_partials is None or ws.det_partials.numel() < need:
            ws.det_partials = torch.empty(max(need, 1), dtype=torch.uint8, device=ws.device)
        if ws.det_slot_off is None or ws.det_slot_off.numel() < ws.n_cap + 1:
            ws.det_slot_off = torch.empty(ws.n_cap + 1, dtype=torch.int32, device=ws.device)
        tb = int(ws.lib.ubs_det_temp_bytes(ws.n_cap))
        if ws.det_temp is None or ws.det_temp.numel() < tb:
            ws.det_temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=ws.device)
        gb.deterministic = 1
        gb.det_slot_off = _ptr(ws.det_slot_off)
        gb.det_partials = _ptr(ws.det_partials)
        gb.det_capacity = ws.pair_cap
        gb.det_temp = _ptr(ws.det_temp)
        gb.det_temp_bytes = ws.det_temp.numel()
    check(ws.lib.ubs_raster_backward(fr.view, ws.prim_buffers(), ws.bin_buffers(), ws.image_buffers(), gb,
                                     _stream_ptr()), "ubs_raster_backward")
    return gb


def backward_chain(fr: Frame, gb, add_regularisers: bool = False, rows: tuple | None = None):
    """Second half of :func:`backward_frame` on the current stream: the
    per-primitive chain rule from the screen-space sums into
    gb.grad_params.  It reads the frame's workspace (grad2d, flags, active),
    so the workspace must not be reused before it completes.

    ``rows=(r0, r1)`` chains only primitives r0 <= i < r1 (a sub-view whose
    params / flags / sums / gradient pointers start at row r0): the chain is
    per primitive, so a frame's chain split into row ranges writes the same
    bits as one call, and a caller can start reducing finished rows early."""
    if rows is None:
        check(fr.ws.lib.ubs_prim_backward(fr.view, gb, 1 if add_regularisers else 0, _stream_ptr()),
              "ubs_prim_backward")
        fr.ws.grad2d_clean = True  # the chain consumed (zeroed) every sum the raster added
        return
    r0, r1 = int(rows[0]), int(rows[1])
    if not 0 <= r0 <= r1 <= fr.n:
        raise ValueError("row range outside the frame's primitives")
    if r1 == r0:
        return
    v = UbsView.from_buffer_copy(fr.view)
    P = record_width(v.n_dims)
    v.params = v.params + r0 * P * (8 if v.param_f64 else 4)
    v.n = r1 - r0
    v.statics = 0  # the chain recomputes from params; statics are tiled per 128 rows
    g = UbsGradBuffers.from_buffer_copy(gb)
    g.grad2d = g.grad2d + r0 * GRAD2D_STRIDE * (8 if g.grad2d_f64 else 4)
    g.grad_params = g.grad_params + r0 * P * (8 if g.grad_f64 else 4)
    g.flags = g.flags + 2 * r0 if g.flags else 0
    g.active = g.active + 4 * r0 if g.active else 0
    check(fr.ws.lib.ubs_prim_backward(v, g, 1 if add_regularisers else 0, _stream_ptr()), "ubs_prim_backward")
    if r1 == fr.n:
        fr.ws.grad2d_clean = True


def field_slices(n_dims: int) -> dict:
    """PARAM_FIELDS name -> (column slice, per-primitive shape) in the packed record."""
    c = n_dims - 3
    out, off = {}, 0
    for name, fn in PARAM_FIELDS:
        shape = fn(c)
        size = int(np.prod(shape)) if shape else 1
        out[name] = (slice(off, off + size), shape)
        off += size
    return out


class HostFrameSink:
    """Streams rendered images to pinned host memory on a side stream.

    ``submit(frame)`` snapshots the image on the compute stream (a device
    copy, so the next frame may reuse the workspace at once) and queues its
    device->host copy on a copy stream; ``slots`` pinned buffers rotate, a slot
    is reused only after its previous copy finished.  This is the host-buffer
    path a sweep user takes: the copy of frame k overlaps the render of k+1.
    """

    def __init__(self, height: int, width: int, dtype=torch.float32, device="cuda", slots: int = 3,
                 copy_streams: int = 1):
        self.dev = torch.device(device)
        # several copy streams: a frame that finishes early is not queued
        # behind an earlier-submitted one still rendering
        self.copy_streams = [torch.cuda.Stream(self.dev) for _ in range(max(1, int(copy_streams)))]
        self.copy_stream = self.copy_streams[0]
        self.dev_bufs = [torch.empty((height, width, 3), dtype=dtype, device=self.dev) for _ in range(slots)]
        self.host_bufs = [torch.empty((height, width, 3), dtype=dtype, pin_memory=True) for _ in range(slots)]
        self.done = [None] * slots
        self.last_copy = None
        self.k = 0
        self.bytes_per_frame = height * width * 3 * torch.finfo(dtype).bits // 8

    def submit(self, fr: Frame, source_stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Queue frame ``fr``'s image for the host.  With ``source_stream``
        (the stream the frame was rendered on) the copy reads the frame's own
        buffer with no device snapshot -- the caller must keep that buffer
        alive until :attr:`last_copy` completes (FramePipeline.hold)."""
        i = self.k % len(self.host_bufs)
        self.k += 1
        if source_stream is not None:
            ready = torch.cuda.Event()
            ready.record(source_stream)
            src = fr.image
        else:
            if self.done[i] is not None:
                torch.cuda.current_stream().wait_event(self.done[i])
            self.dev_bufs[i].copy_(fr.image)
            ready = torch.cuda.Event()
            ready.record()
            src = self.dev_bufs[i]
        cs = self.copy_streams[(self.k - 1) % len(self.copy_streams)]
        with torch.cuda.stream(cs):
            cs.wait_event(ready)
            self.host_bufs[i].copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
        self.done[i] = ev
        self.last_copy = ev
        return self.host_bufs[i]

    def synchronize(self):
        for cs in self.copy_streams:
            cs.synchronize()

    def join(self, stream: torch.cuda.Stream | None = None):
        """Make ``stream`` (default: the current one) wait for every queued copy."""
        stream = stream or torch.cuda.current_stream(self.dev)
        for cs in self.copy_streams:
            stream.wait_stream(cs)
