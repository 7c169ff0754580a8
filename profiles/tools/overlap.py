"""How well do the stages overlap?  Per-frame times over 16 slots x 300
frames of the 7D 1M 1080p sweep: the full grouped pipeline, then each stage
re-launched alone on the 16 resident frames (raster; both binning calls;
ubs_bin_depth; ubs_bin_tiles; the grouped preprocess).  Prints one JSON line."""
import sys, json, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import torch
from paper_2510_03312_b200 import engine, synthetic as S, _lib
from paper_2510_03312_b200.types import DEFAULT_SETTINGS as ST
sc = S.synth(7, 1_000_000, seed=1)
cam = S.bench_camera()
ds = engine.DeviceScene.from_scene(sc, device="cuda")
D = 16
pipe = engine.FramePipeline(ds, D, "fp32", ds.device)
qs = [S.bench_query(7, cam, ((37 * k) % 300) / 299) for k in range(300)]
for k in range(2 * D):
    pipe.render(cam, qs[k % 300], ST, sync=True)
lib = pipe.workspaces[0].lib
def timed(fn, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(n)
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
def full(n):
    for g in range(0, n, 4):
        pipe.render_group([(cam, qs[(g + j) % 300]) for j in range(4)], ST)
res = {}
res["full_ms"] = timed(full, 300)
# the last 16 frames are resident in the slots: re-launch only stages
frames = pipe.render_group([(cam, qs[j]) for j in range(4)], ST)
frs = []
for g in range(4):
    frs += pipe.render_group([(cam, qs[4 * g + j]) for j in range(4)], ST)
pipe.join(); torch.cuda.synchronize()
def only(which):
    def fn(n):
        for k in range(n):
            fr = frs[k % D]
            ws = fr.ws
            s = pipe.stream_of(fr)
            with torch.cuda.stream(s):
                sp = s.cuda_stream
                pb, bb, ib = ws.prim_buffers(), ws.bin_buffers(), ws.image_buffers()
                if "raster" in which:
                    lib.ubs_raster_forward(fr.view, pb, bb, ib, sp)
                if "fixup" in which:
                    lib.ubs_raster_fixup(fr.view, pb, bb, ib, sp)
                if "bin" in which or "bdepth" in which:
                    lib.ubs_bin_depth(fr.view, pb, bb, sp)
                if "bin" in which or "btiles" in which:
                    lib.ubs_bin_tiles(fr.view, pb, bb, -1, sp)
    return fn
for w in (("raster",), ("bin",), ("bdepth",), ("btiles",)):
    res["+".join(w) + "_ms"] = timed(only(w), 300)
# preprocess groups only
def pre(n):
    for g in range(0, n, 4):
        vs = [f.view for f in frs[(g % D):(g % D) + 4]]
        pbs = [f.ws.prim_buffers() for f in frs[(g % D):(g % D) + 4]]
        with torch.cuda.stream(pipe.lead):
            lib.ubs_preprocess_views((_lib.UbsView * 4)(*vs), (_lib.UbsPrimBuffers * 4)(*pbs), 4, 1, pipe.lead.cuda_stream)
    torch.cuda.current_stream().wait_stream(pipe.lead)
res["preprocess_ms"] = timed(pre, 300)
print(json.dumps(res))
