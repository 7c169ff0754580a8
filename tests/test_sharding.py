"""Multi-process (world_size 2, gloo, CPU) check of the view-sharded
data-parallel step: sharded loss + all-reduced gradient equal the
single-process reference backward over the whole batch.

The GPU backend cannot run here, so the per-view work uses a test-only
backend built on the oracle; what is under test is sharding.py's split /
reduce / regulariser-once logic, which is identical for both backends."""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ubs_oracle as O
from paper_2510_03312_b200 import sharding, synthetic as S
from paper_2510_03312_b200.types import DEFAULT_SETTINGS, LossConfig, pack_records, quantize_f32


class OracleBackend:
    def __init__(self, scene):
        self.scene = scene

    def new_grad(self):
        return torch.zeros((self.scene.n_primitives, 14 + 6 * (self.scene.n_dims - 3)), dtype=torch.float64)

    def view_loss_grad(self, cam, q, target, cfg, scale, grad, sync=False):
        fr = O.render_frame(self.scene, cam, q, DEFAULT_SETTINGS)
        tgt = target.numpy()
        diff = fr["image"] - tgt
        s, g_ssim = O.ssim_and_grad(fr["image"], tgt)
        g_img = scale * ((1 - cfg.lambda_ssim) * np.sign(diff) / diff.size - cfg.lambda_ssim * g_ssim)
        out = {k: np.zeros_like(np.asarray(getattr(self.scene, k), dtype=np.float64)) for k in O.FIELDS}
        O.frame_backward(fr, g_img, out)
        grad += torch.from_numpy(np.concatenate([out[k].reshape(self.scene.n_primitives, -1) for k in O.FIELDS], 1))
        return torch.tensor((1 - cfg.lambda_ssim) * np.abs(diff).mean() + cfg.lambda_ssim * (1 - s),
                            dtype=torch.float64)

    def add_regularisers(self, grad, cfg):
        sc = self.scene
        o = 1 / (1 + np.exp(-sc.opacity_raw))
        g = {k: np.zeros_like(np.asarray(getattr(sc, k), dtype=np.float64)) for k in O.FIELDS}
        g["opacity_raw"] += cfg.loss_scale * cfg.lambda_o * o * (1 - o)
        g["s_x_raw"] += cfg.loss_scale * cfg.lambda_sigma * np.exp(sc.s_x_raw)
        g["s_q_raw"] += cfg.loss_scale * cfg.lambda_sigma * np.exp(sc.s_q_raw)
        grad += torch.from_numpy(np.concatenate([g[k].reshape(sc.n_primitives, -1) for k in O.FIELDS], 1))

    def regulariser_value(self, cfg):
        sc = self.scene
        o = 1 / (1 + np.exp(-sc.opacity_raw))
        return cfg.lambda_o * o.sum() + cfg.lambda_sigma * (np.exp(sc.s_x_raw).sum() + np.exp(sc.s_q_raw).sum())


class BatchedOracleBackend(OracleBackend):
    """The batched backend's contract (``sharding.GpuViewBackend``): views
    queued with ``begin`` / ``view``, the gradient finished in ``end``, which
    hands row ranges to the bucket hook as they become final; ``status`` /
    ``grow`` flag a first attempt as overflowed so the retry path runs."""

    def __init__(self, scene, overflow_first=False):
        super().__init__(scene)
        self.pending, self.hooked, self.flag, self.grown = [], [], int(overflow_first), 0

    def begin(self, grad):
        self.grad, self.pending = grad, []

    def view(self, cam, q, target, cfg, scale, sync=False):
        self.pending.append((cam, q, target, cfg, scale))

    def end(self, bucket_hook=None, buckets=4):
        loss = torch.zeros((), dtype=torch.float64)
        for cam, q, target, cfg, scale in self.pending:
            loss += self.view_loss_grad(cam, q, target, cfg, scale, self.grad)
        n = self.scene.n_primitives
        step = -(-n // buckets)
        if bucket_hook is not None:
            for r0 in range(0, n, step):
                self.hooked.append((r0, min(n, r0 + step)))
                bucket_hook(r0, min(n, r0 + step))
        return loss

    def status(self):
        return torch.tensor([self.flag], dtype=torch.int32)

    def grow(self):
        self.flag, self.grown = 0, self.grown + 1
        return 1


def _setup():
    sc = quantize_f32(S.random_scene(6, 30, seed=12))
    views = []
    for k in range(5):
        cam = S.random_camera(32, 100 + k)
        q = S.random_query(6, 200 + k)
        other = S.random_scene(6, 15, seed=300 + k)
        tgt = np.clip(O.render_frame(other, cam, q, DEFAULT_SETTINGS)["image"], 0, 1)
        views.append((cam, q, torch.from_numpy(tgt)))
    return sc, views


def _worker(rank, world, port, out_path, batched=False):
    os.environ["OMP_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc, views = _setup()
    # batched: rank 1 reports an overflow on its first attempt, so both ranks
    # must take the retry together (the flag is all-reduced)
    be = BatchedOracleBackend(sc, overflow_first=rank == 1) if batched else OracleBackend(sc)
    step = sharding.ViewShardedStep(be)
    cfg = LossConfig(lambda_ssim=0.3, loss_scale=1.5)
    loss, grad = step.loss_and_grad(views, cfg, buckets=3)
    assert len(sharding.shard(views, rank, world)) == (3 if rank == 0 else 2)
    if batched:
        n = sc.n_primitives
        assert step.retries == 1
        assert be.grown == 1
        # two attempts, each covering every row once in 3 buckets
        assert be.hooked == [(0, 10), (10, 20), (20, n)] * 2
    if rank == 0:
        np.savez(out_path, loss=float(loss), grad=grad.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_round_robin():
    assert sharding.shard(range(7), 1, 3) == [1, 4]
    assert sum(len(sharding.shard(range(10), r, 4)) for r in range(4)) == 10


@pytest.mark.parametrize("batched", [False, True])
def test_two_rank_gloo_matches_single_process(batched):
    out = os.path.join(tempfile.mkdtemp(), "dp.npz")
    mp.spawn(_worker, args=(2, _free_port(), out, batched), nprocs=2, join=True)
    got = np.load(out)
    sc, views = _setup()
    frames = [(c, q, t.numpy()) for c, q, t in views]
    cfg = LossConfig(lambda_ssim=0.3, loss_scale=1.5)
    loss, g = O.backward(sc, frames, cfg, DEFAULT_SETTINGS)
    ref = np.concatenate([g[k].reshape(sc.n_primitives, -1) for k in O.FIELDS], 1)
    assert abs(got["loss"] - loss) <= 1e-12 * abs(loss)
    assert np.abs(got["grad"] - ref).max() <= 1e-12 * np.abs(ref).max()
