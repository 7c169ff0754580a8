import sys
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import torch
from paper_2510_03312_b200 import engine, sharding, synthetic as S
from paper_2510_03312_b200.types import LossConfig
dev = torch.device("cuda", 0)
scene = S.synth(7, 3_000_000, seed=1)
ds = engine.DeviceScene.from_scene(scene, dtype=torch.float32, device=dev)
cams = [S.bench_camera(1920, 1080, k, 8) for k in range(8)]
qs = [S.bench_query(7, c, 0.5) for c in cams]
tds = engine.DeviceScene.from_scene(S.synth(7, 3_000_000, seed=2), dtype=torch.float32, device=dev)
tws = engine.Workspace(dev, "fp32")
targets = [engine.render_frame(tws, tds, c, q).image.clone().clamp_(0.0, 1.0) for c, q in zip(cams, qs)]
del tws, tds
views = list(zip(cams, qs, targets))
step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, "fp32", depth=8, group=8))
adam = sharding.DeviceAdam(ds.params, 7)
cfg = LossConfig()
grad = step.backend.new_grad()
for _ in range(2):
    loss, grad = step.loss_and_grad(views, cfg, grad)
    adam.step(grad)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
loss, grad = step.loss_and_grad(views, cfg, grad)
adam.step(grad)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok", float(loss))
