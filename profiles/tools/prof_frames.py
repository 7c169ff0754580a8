import sys
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import torch
from paper_2510_03312_b200 import engine, synthetic as S
from paper_2510_03312_b200.types import DEFAULT_SETTINGS as ST
sc = S.synth(7, 1_000_000, seed=1)
cam = S.bench_camera()
ds = engine.DeviceScene.from_scene(sc, device="cuda")
pipe = engine.FramePipeline(ds, 4, "fp32", ds.device)
qs = [S.bench_query(7, cam, k / 299) for k in (0, 80, 160, 240)]
for k in range(8):
    pipe.render(cam, qs[k % 4], ST, sync=True)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("group")
pipe.render_group([(cam, q) for q in qs], ST)
pipe.join()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
