"""World-size-2 run of the PRODUCT data-parallel training step on one GPU:
two processes (gloo, CUDA tensors), each driving ``GpuViewBackend`` (views
in flight, groups sharing one preprocess, bucketed all-reduce issued while
the last view's chain runs) through ``ViewShardedStep``; the all-reduced
loss and gradient must equal the single-process step over the whole batch
(up to fp32 summation order) and the oracle.

The two ranks share the device but never wait on each other's kernels: the
only exchange is gloo's host-staged all-reduce after each rank's own views
(SURVEY §8(e)).  This checks the sharding, the bucket boundaries and the
regulariser-once logic of the product path; throughput is not measured.
"""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup():
    import torch
    from oracle import ubs_oracle as O
    from paper_2510_03312_b200 import synthetic as S
    from paper_2510_03312_b200.types import DEFAULT_SETTINGS
    scene = S.synth(7, 20_000, seed=5)
    cams = [S.bench_camera(160, 96, k, 7) for k in range(7)]
    qs = [S.bench_query(7, c, 0.1 + 0.12 * k) for k, c in enumerate(cams)]
    other = S.synth(7, 8_000, seed=6)
    tg = [np.clip(O.render_frame(other, c, q, DEFAULT_SETTINGS)["image"], 0.0, 1.0) for c, q in zip(cams, qs)]
    return scene, cams, qs, tg


def _step(scene, cams, qs, tg, buckets):
    import torch
    from paper_2510_03312_b200 import engine, sharding
    from paper_2510_03312_b200.types import LossConfig
    ds = engine.DeviceScene.from_scene(scene, device="cuda")
    step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, "fp32", depth=3, group=2))
    views = [(c, q, torch.from_numpy(t).float().cuda()) for c, q, t in zip(cams, qs, tg)]
    loss, grad = step.loss_and_grad(views, LossConfig(lambda_ssim=0.3, loss_scale=1.5), buckets=buckets)
    torch.cuda.synchronize()
    return float(loss), grad.double().cpu().numpy()


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    scene, cams, qs, tg = _setup()
    loss, grad = _step(scene, cams, qs, tg, buckets=3)
    if rank == 0:
        np.savez(out_path, loss=loss, grad=grad)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_product_step_matches_single_process():
    import torch.multiprocessing as mp
    from oracle import ubs_oracle as O
    from paper_2510_03312_b200.types import DEFAULT_SETTINGS, LossConfig
    from .helpers import grad_close
    out = os.path.join(tempfile.mkdtemp(), "dp_gpu.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    scene, cams, qs, tg = _setup()
    l1, g1 = _step(scene, cams, qs, tg, buckets=1)
    assert abs(float(got["loss"]) - l1) <= 1e-6 * abs(l1)
    split = lambda g: {k: g[:, a:b] for k, (a, b) in _cols(scene).items()}  # noqa: E731
    bad = grad_close(split(got["grad"]), split(g1), rel=1e-4, floor=1e-5)
    assert not bad, bad
    cfg = LossConfig(lambda_ssim=0.3, loss_scale=1.5)
    l_ref, g_ref = O.backward(scene, list(zip(cams, qs, tg)), cfg, DEFAULT_SETTINGS)
    assert abs(float(got["loss"]) - l_ref) <= 1e-5 * abs(l_ref)
    ref = {k: v.reshape(scene.n_primitives, -1) for k, v in g_ref.items()}
    bad = grad_close(split(got["grad"]), ref, rel=1e-3)
    assert not bad, bad


def _cols(scene):
    from oracle import ubs_oracle as O
    out, off = {}, 0
    for k in O.FIELDS:
        w = int(np.prod(np.asarray(getattr(scene, k)).shape[1:]))
        out[k] = (off, off + w)
        off += w
    return out
