"""Drive every kernel of the bounds-checked build (libubs_b200_checked.so,
-DUBS_CHECKED) over the shapes that stress its index arithmetic, then print
each translation unit's guard status word (tests/test_gpu_checked.py)."""

from __future__ import annotations

import ctypes
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ["UBS_B200_LIB"] = str(ROOT / "paper_2510_03312_b200" / "libubs_b200_checked.so")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_03312_b200 import _lib, engine, raster, sharding, synthetic as S  # noqa: E402
from paper_2510_03312_b200.gradients import backward  # noqa: E402
from paper_2510_03312_b200.types import DEFAULT_SETTINGS, Camera, LossConfig, Query, RenderSettings, quantize_f32  # noqa: E402

TUS = ("binning", "preprocess", "raster", "prim_bwd", "loss", "optim")


def main():
    lib = _lib.load()
    assert Path(os.environ["UBS_B200_LIB"]).exists()
    for tu in TUS:
        getattr(lib, f"ubs_debug_checked_{tu}").argtypes = [ctypes.c_void_p, ctypes.c_int]
    cfg = LossConfig()
    # small scenes, both precisions, forward + backward + deterministic backward
    for nd in (3, 6, 7):
        sc = quantize_f32(S.random_scene(nd, 300, seed=nd))
        cam, q = S.random_camera(40, nd), S.random_query(nd, nd + 1)
        for precision in ("fp32", "fp64"):
            c = raster.render_with_cache(sc, cam, q, DEFAULT_SETTINGS, precision=precision)
            _ = c.tile_ids, c.slices, c.proj
            tgt = np.clip(c.image * 0.7 + 0.1, 0, 1)
            for det in (False, True):
                backward(sc, [(cam, q, tgt)], cfg, DEFAULT_SETTINGS, precision=precision, deterministic=det)
    # tiny images (the loss's small-image kernels), odd sizes, a frame past one CTA's tile scan
    sc = quantize_f32(S.random_scene(7, 200, seed=9))
    for w, h in ((5, 7), (11, 13), (333, 211)):
        cam = Camera.look_at((2.5, 1.0, 0.8), (0, 0, 0), (0, 0, 1), 0.9, w, h)
        q = Query.view_time(0.3, cam.forward)
        img = raster.render(sc, cam, q)
        backward(sc, [(cam, q, np.clip(img * 0.5, 0, 1))], cfg, DEFAULT_SETTINGS)
    raster.render(quantize_f32(S.synth(3, 3000, seed=41)), S.bench_camera(4000, 3600), Query.static())
    # depth ties, capped lists that run out (grow + re-render), no early exit
    base = quantize_f32(S.random_scene(6, 300, seed=23))
    tied = base.take(np.concatenate([np.arange(300)] * 3))
    ds = engine.DeviceScene.from_scene(tied, device="cuda")
    ws = engine.Workspace("cuda", "fp32")
    ws.list_cap = 4
    cam, q = S.random_camera(96, 24), S.random_query(6, 25)
    engine.render_frame(ws, ds, cam, q, RenderSettings(transmittance_min=0.0))
    # the benchmark path: 1080p 7D, grouped pipeline, capped lists, training backend (4 px / lane)
    sc = S.synth(7, 200_000, seed=1)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    cam = S.bench_camera()
    pipe = engine.FramePipeline(ds, depth=4)
    views = [(cam, S.bench_query(7, cam, k / 3)) for k in range(4)]
    for v in views:
        pipe.render(*v, sync=True)
    pipe.render_group(views)
    pipe.join()
    pipe.check_status()
    tg = torch.rand(1080, 1920, 3, device="cuda")
    step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, "fp32", depth=2, group=2))
    adam = sharding.DeviceAdam(ds.params, 7)
    loss, grad = step.loss_and_grad([(c, qq, tg) for c, qq in views[:3]], cfg)
    adam.step(grad)
    torch.cuda.synchronize()
    out = {}
    for tu in TUS:
        w = ctypes.c_uint(0)
        rc = getattr(lib, f"ubs_debug_checked_{tu}")(ctypes.byref(w), 1)
        out[tu] = int(w.value) if rc == 0 else f"rc {rc}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
