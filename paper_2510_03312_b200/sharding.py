"""View-batch data parallelism across GPUs.

Views (camera, query[, target]) are independent units.  Rendering a batch of
views shards them round-robin over ranks with no communication.  A training
step shards the batch the same way; every rank accumulates the raw-parameter
gradient of its views (each scaled by loss_scale / B, gradients.py:114-116)
into one flat n x (14+6C) buffer, then a single all-reduce(sum) over NCCL
(NVLink/NVSwitch) combines them.  Regulariser gradients are added exactly
once (by rank 0, before the reduce, gradients.py:120-123) and the scalar
loss is all-reduced alongside.  The optimizer (device Adam,
optim.py:115-135) then runs identically on every rank, keeping the
replicated scene in sync without a broadcast.

The per-view work is done by a backend object; ``GpuViewBackend`` drives
libubs_b200.so.  (Tests substitute a CPU backend to check the reduction
logic with world_size 2 over gloo; the product path only ever uses the GPU
backend.)
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes

import torch

from . import _lib, engine
from .types import DEFAULT_SETTINGS, LossConfig


def shard(items, rank: int, world: int) -> list:
    """Round-robin share of ``items`` for ``rank``."""
    return list(items)[rank::world]


def dist_rank_world(group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class GpuViewBackend:
    """Per-view loss + gradient on this rank's GPU through the C-ABI engine.

    ``depth`` > 1 keeps that many views in flight: view k of a batch runs on
    slot k % depth (own stream and workspace), so one view's latency-bound
    preprocess / loss / chain kernels overlap another view's raster backward.
    Views are dispatched in groups of ``group`` that share one preprocess
    launch (``ubs_preprocess_views``: the scene statics are read once per
    group).  Every view's per-primitive chain (``prim_bwd``) runs on one
    gradient stream in view order, adding straight into the batch gradient:
    the sum is formed in exactly the order of one-at-a-time accumulation, and
    a slot is reused only after the gradient stream is done with it.
    ``first_group`` (default ``group``) sizes a batch's first group: a small
    one starts the rasters early while the next group's preprocess runs
    beside them."""

    def __init__(self, ds: engine.DeviceScene, precision: str = "fp32", settings=DEFAULT_SETTINGS,
                 grad_dtype=torch.float32, depth: int = 1, group: int = 1, pixels_per_lane: int = 4,
                 first_group: int | None = None):
        self.ds = ds
        self.settings = settings
        self.grad_dtype = grad_dtype
        self.depth = max(1, int(depth))
        self.group = max(1, min(int(group), self.depth))
        self.first_group = self.group if first_group is None else max(1, min(int(first_group), self.depth))
        self.pixels_per_lane = int(pixels_per_lane)  # raster backward layout (UbsGradBuffers.bwd_pixels_per_lane)
        self.workspaces = [engine.Workspace(ds.device, precision) for _ in range(self.depth)]
        self.ws = self.workspaces[0]
        multi = self.depth > 1
        self.streams = [torch.cuda.Stream(ds.device) for _ in range(self.depth)] if multi else None
        self.lead = torch.cuda.Stream(ds.device) if multi else None  # shared preprocess of a group
        self.gstream = torch.cuda.Stream(ds.device) if multi else None  # prim_bwd of every view, in order
        self.slot_free = [None] * self.depth  # gradient-stream event after the slot's last chain
        self._k = 0
        self._grad = None
        self._rec = None
        self._queue = []
        self._pending = None  # (frame, grad buffers, slot) of the last view: its chain waits for end()

    def new_grad(self) -> torch.Tensor:
        return torch.zeros(self.ds.params.shape, dtype=self.grad_dtype, device=self.ds.device)

    def _view(self, ws, cam, query, target, cfg: LossConfig, scale: float, grad, sync: bool):
        fr = engine.render_frame(ws, self.ds, cam, query, self.settings, sync=sync or ws.pair_cap == 0)
        ws.loss_parts.zero_()
        g_img, parts = engine.loss_image_grad(fr, target, cfg.lambda_ssim, scale)
        engine.backward_frame(fr, self.ds, g_img, grad)
        return self._term(fr, parts, cfg)

    @staticmethod
    def _term(fr, parts, cfg: LossConfig):
        size = fr.width * fr.height * 3
        return (1.0 - cfg.lambda_ssim) * parts[0] / size + cfg.lambda_ssim * (1.0 - parts[1] / size)

    def view_loss_grad(self, cam, query, target: torch.Tensor, cfg: LossConfig, scale: float,
                       grad: torch.Tensor, sync: bool = False) -> torch.Tensor:
        """Adds this view's d(loss)/d(params) into ``grad``; returns the view's
        reconstruction term (1-l) L1 + l (1 - SSIM) as a 0-d device tensor.
        Frames are asynchronous unless ``sync`` (see :meth:`status`)."""
        return self._view(self.ws, cam, query, target, cfg, scale, grad, sync)

    # --- batched interface (ViewShardedStep) -------------------------------
    def begin(self, grad: torch.Tensor):
        self._k = 0
        self._grad = grad
        self._rec = torch.zeros(self.depth, dtype=torch.float64, device=grad.device)
        self._queue = []
        self._pending = None
        if self.depth > 1:
            self.gstream.wait_stream(torch.cuda.current_stream())  # the caller zeroed grad there

    def view(self, cam, query, target, cfg: LossConfig, scale: float, sync: bool = False):
        if self.depth == 1:
            self._rec[0] += self._view(self.ws, cam, query, target, cfg, scale, self._grad, sync)
            return
        self._queue.append((cam, query, target, cfg, scale, sync))
        if len(self._queue) >= (self.first_group if self._k == 0 else self.group) or sync:
            self._flush()

    def _chain(self, rows=None, hook=None):
        """Issue the pending view's per-primitive chain on the gradient
        stream; with ``rows`` = [(r0, r1), ...] in row-range chunks, calling
        ``hook(r0, r1)`` on the gradient stream after each (the rows of the
        batch's last view are final then: a reduction can start)."""
        if self._pending is None:
            return
        fr, gb, i, done = self._pending
        self._pending = None
        self.gstream.wait_event(done)
        with torch.cuda.stream(self.gstream):
            if rows is None:
                engine.backward_chain(fr, gb)
            else:
                for r0, r1 in rows:
                    engine.backward_chain(fr, gb, rows=(r0, r1))
                    if hook is not None:
                        hook(r0, r1)
            free = torch.cuda.Event()
            free.record(self.gstream)
        self.slot_free[i] = free

    def _flush(self):
        queue, self._queue = self._queue, []
        if not queue:
            return
        self._chain()  # the previous group's last view: it is not the batch's last
        ds, settings = self.ds, self.settings
        sync = any(item[5] for item in queue)
        slots = [(self._k + j) % self.depth for j in range(len(queue))]
        self._k += len(queue)
        # on the caller's stream, before any slot reads them (after every stream
        # that may still read the previous statics, if they must be recomputed)
        statics = ds.statics_ptr(settings, self.streams + [self.lead, self.gstream])
        lead = self.lead
        lead.wait_stream(torch.cuda.current_stream())
        for i in slots:
            lead.wait_stream(self.streams[i])
            if self.slot_free[i] is not None:
                lead.wait_event(self.slot_free[i])
        grouped = bool(statics) and len(queue) > 1 and not sync
        if grouped:  # one preprocess for the group
            vs, pbs = [], []
            with torch.cuda.stream(lead):
                for (cam, query, *_), i in zip(queue, slots):
                    v, pb = engine._frame_begin(self.workspaces[i], ds, cam, query, settings, False)
                    vs.append(v)
                    pbs.append(pb)
                ws0 = self.workspaces[slots[0]]
                engine.check(ws0.lib.ubs_preprocess_views((_lib.UbsView * len(vs))(*vs),
                                                          (_lib.UbsPrimBuffers * len(pbs))(*pbs), len(vs),
                                                          0 if ws0.f64 else 1, lead.cuda_stream),
                             "ubs_preprocess_views")
        ready = torch.cuda.Event()
        ready.record(lead)
        for j, ((cam, query, target, cfg, scale, _), i) in enumerate(zip(queue, slots)):
            ws, s = self.workspaces[i], self.streams[i]
            s.wait_event(ready)
            with torch.cuda.stream(s):
                if grouped:
                    fr = engine._frame_end(ws, ds, vs[j], pbs[j], cam, query, settings, False, None, False, False)
                else:
                    fr = engine.render_frame(ws, ds, cam, query, settings, sync=sync or ws.pair_cap == 0)
                ws.loss_parts.zero_()
                g_img, parts = engine.loss_image_grad(fr, target, cfg.lambda_ssim, scale)
                # four pixels per lane (default): the layout that runs best beside the other views in flight
                gb = engine.backward_raster(fr, ds, g_img, self._grad, pixels_per_lane=self.pixels_per_lane)
                self._rec[i:i + 1] += self._term(fr, parts, cfg)
                done = torch.cuda.Event()
                done.record(s)
            if gb is None:
                continue
            self._chain()  # chains run in view order on the gradient stream
            self._pending = (fr, gb, i, done)

    def end(self, bucket_hook=None, buckets: int = 4) -> torch.Tensor:
        """Join the slots and the gradient stream; returns the summed
        reconstruction terms (0-d device tensor).

        ``bucket_hook(r0, r1)``: called on the gradient stream as soon as
        rows [r0, r1) of the batch gradient are final -- the last view's chain
        runs in ``buckets`` row ranges -- so a collective on those rows (the
        data-parallel all-reduce) overlaps the rest of the chain."""
        if self.depth > 1:
            self._flush()
            n = self.ds.n
            if bucket_hook is not None and self._pending is not None:
                step = -(-n // max(1, int(buckets)))
                step = -(-step // 128) * 128
                self._chain([(r0, min(n, r0 + step)) for r0 in range(0, n, step)], bucket_hook)
            else:
                self._chain()
                if bucket_hook is not None:  # no view had primitives to chain: every row is final
                    with torch.cuda.stream(self.gstream):
                        bucket_hook(0, n)
            cur = torch.cuda.current_stream()
            for s in self.streams:
                cur.wait_stream(s)
            cur.wait_stream(self.gstream)
        elif bucket_hook is not None:  # one view at a time: the gradient is final now
            bucket_hook(0, self.ds.n)
        return self._rec.sum()

    def status(self) -> torch.Tensor:
        """Device flag, nonzero when an asynchronous view outgrew the pair buffers."""
        out = self.workspaces[0].status.clone()
        for ws in self.workspaces[1:]:
            out |= ws.status
        return out

    def clear_status(self):
        for ws in self.workspaces:
            ws.status.zero_()

    def grow(self) -> int:
        """After an asynchronous view outgrew its slot: give every slot the
        largest tile-list cap any slot has (doubled if a list was truncated)
        and pair buffers for the largest tile-pair count any slot saw, then
        clear the status (a batch's views rotate over the slots, so growing
        only the slot that overflowed is not enough).  Syncs."""
        torch.cuda.current_stream().synchronize()
        st = 0
        for ws in self.workspaces:
            st |= int(ws.status.item())
        cap = max(ws.list_cap for ws in self.workspaces)
        if st & _lib.S_LIST_TRUNC:
            cap *= 2
        k = max(int(ws.counters[0].item()) for ws in self.workspaces)
        if st & _lib.S_PAIR_OVERFLOW:
            k = max(k, int(max(ws.pair_cap for ws in self.workspaces) * 1.3) + 1)
        for ws in self.workspaces:
            ws.list_cap = cap
            if ws.temp_bytes:
                ws.ensure_pairs(k)
            ws.status.zero_()
        return st

    def add_regularisers(self, grad: torch.Tensor, cfg: LossConfig):
        lib = _lib.load()
        p = self.ds.params
        _lib.check(lib.ubs_add_regularisers(p.data_ptr(), int(p.dtype == torch.float64), grad.data_ptr(),
                                            int(grad.dtype == torch.float64), self.ds.n, self.ds.n_dims,
                                            cfg.loss_scale * cfg.lambda_o, cfg.loss_scale * cfg.lambda_sigma,
                                            torch.cuda.current_stream().cuda_stream), "ubs_add_regularisers")

    def regulariser_value(self, cfg: LossConfig) -> torch.Tensor:
        """lambda_o sum sigmoid(o) + lambda_sigma sum exp(s) (gradients.py:120-123):
        one fp64 pass over the opacity and scale columns (ubs_regulariser_value);
        a 0-d device tensor."""
        p = self.ds.params
        sums = torch.zeros(2, dtype=torch.float64, device=p.device)
        lib = _lib.load()
        _lib.check(lib.ubs_regulariser_value(p.data_ptr(), int(p.dtype == torch.float64), int(p.shape[0]),
                                             self.ds.n_dims, sums.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream), "ubs_regulariser_value")
        return cfg.lambda_o * sums[0] + cfg.lambda_sigma * sums[1]


class ViewShardedStep:
    """loss + all-reduced gradient of a batch of views, views sharded over ranks."""

    def __init__(self, backend, group=None):
        self.backend = backend
        self.group = group
        self.retries = 0  # batches recomputed because an asynchronous view outgrew its buffers
        self._next = None  # NextStep from optimizer_step

    def optimizer_step(self, adam: "DeviceAdam", grad: torch.Tensor, cfg: LossConfig = LossConfig()):
        """``adam.step(grad)`` fused with preparing ``grad`` for the next
        ``loss_and_grad(..., grad=grad)``: its zeroing, the regulariser
        gradient (rank 0 only, gradients.py:120-123) and the regulariser value
        come out of the optimizer's own pass over the records."""
        rank, _ = dist_rank_world(self.group)
        self._next = adam.step(grad, next_cfg=cfg, regularise=rank == 0)

    def loss_and_grad(self, views, cfg: LossConfig = LossConfig(), grad: torch.Tensor | None = None,
                      buckets: int = 4):
        """Batch loss and gradient.  Rank 0 adds the regulariser gradient
        first (gradients.py:120-123: once per step), every rank adds its
        views', and the gradient is summed over ranks: with a batched
        backend in ``buckets`` row-range all-reduces issued while the last
        view's chain still runs (no host synchronisation before them).  The
        overflow flag of asynchronous views is checked once the reductions
        are queued; a flagged batch is recomputed with synchronous views."""
        import torch.distributed as dist
        if not views:
            raise ValueError("empty batch")
        rank, world = dist_rank_world(self.group)
        b = self.backend
        scale = cfg.loss_scale / len(views)
        multi = world > 1 and dist.is_available() and dist.is_initialized()
        for attempt in range(3):
            # a view that outgrew its slot's buffers: grow every slot and retry
            # asynchronously, then (rarely) once more with synchronous frames
            sync = attempt > 1
            nxt, self._next = self._next, None
            params = getattr(getattr(b, "ds", None), "params", None)
            if (attempt == 0 and nxt is not None and grad is not None and nxt.grad is grad and params is not None
                    and nxt.valid_for(params, cfg)):
                reg_value = cfg.lambda_o * nxt.sums[0] + cfg.lambda_sigma * nxt.sums[1]  # prepared by the optimizer
            else:
                grad = b.new_grad() if grad is None else grad.zero_()
                if rank == 0:
                    b.add_regularisers(grad, cfg)
                reg_value = None
            rec = torch.zeros(2, dtype=torch.float64, device=grad.device)
            works = []
            if hasattr(b, "begin"):  # batched backend: views may be in flight concurrently
                b.begin(grad)
                for cam, query, target in shard(views, rank, world):
                    b.view(cam, query, target, cfg, scale, sync=sync)

                def hook(r0, r1, grad=grad):
                    if multi:
                        works.append(dist.all_reduce(grad[r0:r1], op=dist.ReduceOp.SUM, group=self.group,
                                                     async_op=True))
                rec[0] += b.end(bucket_hook=hook if multi else None, buckets=buckets)
            else:
                for cam, query, target in shard(views, rank, world):
                    rec[0] += b.view_loss_grad(cam, query, target, cfg, scale, grad, sync=sync)
                if multi:
                    works.append(dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
            if hasattr(b, "status"):
                rec[1] = b.status().to(torch.float64)[0]
            allreduce_sum_(rec, self.group)  # loss term and overflow flag in one collective
            for w in works:
                w.wait()
            if float(rec[1]) == 0.0:
                break
            self.retries += 1
            if hasattr(b, "grow"):
                b.grow()
            else:
                b.clear_status()
        if reg_value is None:
            reg_value = b.regulariser_value(cfg)
        loss = cfg.loss_scale * (rec[0] / len(views) + reg_value)
        return loss, grad


@dataclass
class NextStep:
    """A gradient buffer made ready for the next batch by
    ``DeviceAdam.step(grad, next_cfg)``: ``grad`` holds the regulariser
    gradient of the parameters (or zeros on the ranks that do not add it),
    ``sums`` their regulariser sums.  Valid while the parameters are
    unchanged (same tensor, same version) and for the same loss config."""
    grad: torch.Tensor
    sums: torch.Tensor
    cfg: LossConfig
    key: tuple

    def valid_for(self, params: torch.Tensor, cfg: LossConfig) -> bool:
        return self.key == (params.data_ptr(), params._version) and self.cfg == cfg


class DeviceAdam:
    """Bias-corrected Adam on the flat record buffer (optim.py:115-135), f32 moments."""

    def __init__(self, params: torch.Tensor, n_dims: int, lr_position=1.6e-4, lr_opacity=5e-2, lr_scale=5e-3,
                 lr_other=1e-3, freeze_shapes=False):
        self.params = params
        self.n_dims = n_dims
        self.m = torch.zeros(params.shape, dtype=torch.float32, device=params.device)
        self.v = torch.zeros(params.shape, dtype=torch.float32, device=params.device)
        self.lr = (ctypes.c_double * 4)(lr_position, lr_opacity, lr_scale, lr_other)
        self.freeze = 1 if freeze_shapes else 0
        self.step_count = 0

    def step(self, grad: torch.Tensor, next_cfg: LossConfig | None = None, regularise: bool = True):
        """One Adam step.  With ``next_cfg`` the same pass also prepares
        ``grad`` for the next batch (``ubs_adam_step_regularised``): it is
        overwritten with the regulariser gradient of the updated parameters
        (``regularise``, the one rank that adds it) or zeros, and the
        regulariser sums are formed -- what the next ``loss_and_grad`` would
        otherwise do in three more passes.  Returns the :class:`NextStep`
        (None without ``next_cfg``)."""
        self.step_count += 1
        lib = _lib.load()
        p, stream = self.params, torch.cuda.current_stream().cuda_stream
        common = (p.data_ptr(), int(p.dtype == torch.float64), grad.data_ptr(), int(grad.dtype == torch.float64),
                  self.m.data_ptr(), self.v.data_ptr(), int(p.shape[0]), self.n_dims, self.lr, self.step_count,
                  self.freeze)
        if next_cfg is None:
            _lib.check(lib.ubs_adam_step(*common, stream), "ubs_adam_step")
            nxt = None
        else:
            sums = torch.zeros(2, dtype=torch.float64, device=p.device)
            ro = next_cfg.loss_scale * next_cfg.lambda_o if regularise else 0.0
            rs = next_cfg.loss_scale * next_cfg.lambda_sigma if regularise else 0.0
            _lib.check(lib.ubs_adam_step_regularised(*common, ro, rs, sums.data_ptr(), stream),
                       "ubs_adam_step_regularised")
        # the records changed behind torch's back: bump the version counter so
        # DeviceScene's statics cache sees new parameters
        torch.autograd.graph.increment_version(p)
        if next_cfg is not None:
            nxt = NextStep(grad, sums, next_cfg, (p.data_ptr(), p._version))
        return nxt

    def reset_rows(self, idx: torch.Tensor):
        """Zero the moments of rewritten rows (AdamState.reset_rows, optim.py:100-103)."""
        self.m[idx] = 0.0
        self.v[idx] = 0.0

    def rebind(self, params: torch.Tensor):
        """Follow a grown parameter buffer; new rows start with zero moments
        (AdamState.grow, optim.py:105-112)."""
        extra = params.shape[0] - self.m.shape[0]
        if extra > 0:
            z = torch.zeros((extra, self.m.shape[1]), dtype=self.m.dtype, device=self.m.device)
            self.m = torch.cat([self.m, z])
            self.v = torch.cat([self.v, z.clone()])
        self.params = params


def render_views(ws: engine.Workspace, ds: engine.DeviceScene, views, settings=DEFAULT_SETTINGS, group=None,
                 sink: engine.HostFrameSink | None = None, pipeline: engine.FramePipeline | None = None,
                 frames_per_preprocess: int = 1):
    """Forward-render this rank's share of ``views`` [(cam, query), ...]; no
    communication.  With ``pipeline`` the frames go through its slots (several
    frames in flight; ``ws`` is unused), ``frames_per_preprocess`` > 1 of them
    at a time sharing one preprocess launch (``FramePipeline.render_group``).
    Returns the number of frames rendered by this rank."""
    rank, world = dist_rank_world(group)
    mine = list(shard(views, rank, world))
    if pipeline is None:
        for cam, query in mine:
            fr = engine.render_frame(ws, ds, cam, query, settings)
            if sink is not None:
                sink.submit(fr)
        return len(mine)
    g = max(1, min(int(frames_per_preprocess), pipeline.depth))
    k = 0
    for g0 in range(0, len(mine), g):
        chunk = mine[g0:g0 + g]
        frs = pipeline.render_group(chunk, settings) if g > 1 else [pipeline.render(*chunk[0], settings)]
        for fr in frs:
            if sink is not None and pipeline.depth > 1:
                sink.submit(fr, source_stream=pipeline.stream_of(fr))
                pipeline.hold(fr, sink.last_copy)
            elif sink is not None:
                with torch.cuda.stream(pipeline.stream_of(fr)):
                    sink.submit(fr)
            k += 1
    if pipeline is not None:
        pipeline.join()
    return k
