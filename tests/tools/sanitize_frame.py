"""One small frame of every libubs_b200 kernel, for compute-sanitizer
(tests/test_gpu_sanitizer.py): statics, per-frame and grouped preprocess,
depth sort, both binning levels, fp32 raster + fix-up, fp64 raster, loss,
both raster backward layouts, the chain, Adam, regularisers."""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_03312_b200 import engine, raster, sharding, synthetic as S  # noqa: E402
from paper_2510_03312_b200.gradients import backward  # noqa: E402
from paper_2510_03312_b200.types import DEFAULT_SETTINGS, LossConfig, quantize_f32  # noqa: E402


def main():
    sc = quantize_f32(S.random_scene(7, 400, seed=3))
    cam = S.random_camera(48, 4)
    q = S.random_query(7, 5)
    for precision in ("fp32", "fp64"):
        c = raster.render_with_cache(sc, cam, q, DEFAULT_SETTINGS, precision=precision)
        _ = c.tile_ids
        tgt = np.clip(c.image * 0.8 + 0.05, 0, 1)
        backward(sc, [(cam, q, tgt)], LossConfig(), DEFAULT_SETTINGS, precision=precision)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    pipe = engine.FramePipeline(ds, depth=2)
    views = [(cam, S.random_query(7, 6 + k)) for k in range(2)]
    for v in views:
        pipe.render(*v, sync=True)
    pipe.render_group(views)
    pipe.join()
    pipe.check_status()
    target = torch.rand(48, 48, 3, device="cuda")
    step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, "fp32", depth=2, group=2))
    adam = sharding.DeviceAdam(ds.params, 7)
    loss, grad = step.loss_and_grad([(cam, q, target), (cam, views[0][1], target)], LossConfig())
    adam.step(grad)
    torch.cuda.synchronize()
    print("sanitize frame ok", float(loss))


if __name__ == "__main__":
    main()
