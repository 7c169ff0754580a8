import sys, os
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import torch
from paper_2510_03312_b200 import engine, synthetic as S, _lib
from paper_2510_03312_b200.types import LossConfig
dev = torch.device("cuda", 0)
N = 3_000_000
ds = engine.DeviceScene.from_scene(S.synth(7, N, seed=1), device=dev)
cam = S.bench_camera(1920, 1080, 1, 8); q = S.bench_query(7, cam, 0.5)
ws = engine.Workspace(dev, "fp32")
fr = engine.render_frame(ws, ds, cam, q)
tgt = torch.rand_like(fr.image)
g_img, _ = engine.loss_image_grad(fr, tgt, 0.2, 1.0)
g_img = g_img.clone()
grad = torch.zeros(ds.params.shape, device=dev)
res = {}
for ppl in (2, 4, 8):
    for it in range(2):
        gb = engine.backward_raster(fr, ds, g_img, grad, pixels_per_lane=ppl)
        engine.backward_chain(fr, gb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for it in range(10):
        e0.record()
        gb = engine.backward_raster(fr, ds, g_img, grad, pixels_per_lane=ppl)
        e1.record()
        engine.backward_chain(fr, gb)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[ppl] = sorted(ts)[len(ts) // 2]
print(("scalar" if os.environ.get("UBS_RASTER_SCALAR") else "x2"), {k: round(v, 4) for k, v in res.items()})
