import ctypes, os, sys, json
sys.path.insert(0, "/root/repo")
os.environ["UBS_B200_LIB"] = "/root/repo/profiles/tools/libubs_stats.so"
import torch
from paper_2510_03312_b200 import engine, synthetic as S, _lib
from paper_2510_03312_b200.types import DEFAULT_SETTINGS
lib = _lib.load()
lib.ubs_debug_fwd_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = (ctypes.c_ulonglong * 8)()
sc = S.synth(7, 1_000_000, seed=1)
cam = S.bench_camera()
ds = engine.DeviceScene.from_scene(sc, device="cuda")
ws = engine.Workspace("cuda", "fp32")
for k in range(3):
    engine.render_frame(ws, ds, cam, S.bench_query(7, cam, k / 2))
torch.cuda.synchronize()
lib.ubs_debug_fwd_stats(out, 1)
tot = [0] * 8
nf = 0
for k in range(0, 300, 30):
    fr = engine.render_frame(ws, ds, cam, S.bench_query(7, cam, k / 299))
    torch.cuda.synchronize()
    lib.ubs_debug_fwd_stats(out, 1)
    tot = [a + b for a, b in zip(tot, out)]
    nf += 1
names = ["warp_visits", "warp_visits_none_in", "lane_visits_in", "active_lanes", "wv_clamp_lo", "wv_tmin_hi", "batches", "x"]
d = {n: v / nf for n, v in zip(names, tot)}
d["frac_none_in"] = d["warp_visits_none_in"] / d["warp_visits"]
d["in_lanes_per_wv_with_in"] = d["lane_visits_in"] / (d["warp_visits"] - d["warp_visits_none_in"])
d["active_per_wv"] = d["active_lanes"] / d["warp_visits"]
print(json.dumps(d, indent=1))
