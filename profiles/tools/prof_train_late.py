import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import torch, numpy as np
from paper_2510_03312_b200 import engine, sharding, synthetic as S
from paper_2510_03312_b200.types import LossConfig
dev = torch.device("cuda", 0)
N = 3_000_000
ds = engine.DeviceScene.from_scene(S.synth(7, N, seed=1), dtype=torch.float32, device=dev)
cams = [S.bench_camera(1920, 1080, k, 8) for k in range(8)]
qs = [S.bench_query(7, c, 0.5) for c in cams]
tds = engine.DeviceScene.from_scene(S.synth(7, N, seed=2), dtype=torch.float32, device=dev)
tws = engine.Workspace(dev, "fp32")
targets = [engine.render_frame(tws, tds, c, q).image.clone().clamp_(0.0, 1.0) for c, q in zip(cams, qs)]
views = list(zip(cams, qs, targets))
step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, "fp32", depth=8, group=8))
adam = sharding.DeviceAdam(ds.params, 7)
cfg = LossConfig()
grad = None
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(100):
    e0.record()
    loss, grad = step.loss_and_grad(views, cfg, grad)
    step.optimizer_step(adam, grad, cfg)
    e1.record(); torch.cuda.synchronize()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
e0.record()
loss, grad = step.loss_and_grad(views, cfg, grad)
step.optimizer_step(adam, grad, cfg)
e1.record()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("late step ms", e0.elapsed_time(e1), "retries", step.retries)
fr = engine.render_frame(tws, ds, cams[0], qs[0])
torch.cuda.synchronize()
print("late view: fixup pixels", fr.n_fixed, "max n_contrib", int(fr.n_contrib.max().item()), "K", fr.n_pairs)
