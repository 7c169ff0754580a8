#!/usr/bin/env python
"""Benchmark: UBS render throughput on B200 (BASELINE.json config 4).

Workload (one step = one frame): the 7D dynamic UBS scene, 1M primitives
(``synth(7, 1_000_000, seed=1)``), rendered at 1920x1080 along
the 300-frame time sweep t = k/299 with the benchmark camera.  The scene is
resident in HBM; each frame runs preprocess -> depth sort -> tile binning ->
fp32 raster -> fp64 fix-up, all in libubs_b200.so.  Frames run 16 in flight
(engine.FramePipeline) in groups of 4 that share one preprocess launch
(ubs_preprocess_views: one read of the scene statics per group).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched with torch.distributed.run, one rank per GPU: each rank
renders its own frames of the sweep (view sharding, no data-path collective);
time = max over ranks of the CUDA-event time of the K steps.  ``value`` is
frames/s of the whole job.  ``--impl reference`` times the CPU reference
algorithm (oracle/ port of betasplat's render path, all host threads) on the
same workload, rank 0 only.

The JSON line also carries the dominant kernel's roofline (algorithmic bytes
per launch / CUDA-event launch time vs the measured HBM copy bandwidth), the
CPU baseline, the end-to-end number through the host-buffer API (image
copied to pinned host memory every frame), and SM clocks sampled during the
timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec at 1080p (1M prims, 7D) and train iters/sec; HBM GB/s fraction"
SWEEP = 300


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-prims", type=int, default=1_000_000)
    ap.add_argument("--nd", type=int, default=7)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--inflight", type=int, default=16, help="frames in flight (engine.FramePipeline depth)")
    ap.add_argument("--slot-priority", type=int, default=0, help="CUDA stream priority of the frame slots")
    ap.add_argument("--lead-priority", type=int, default=0, help="CUDA stream priority of the group preprocess")
    ap.add_argument("--group", type=int, default=4,
                    help="frames per shared preprocess (FramePipeline.render_group; 0: frame by frame)")
    ap.add_argument("--copy-streams", type=int, default=2, help="device->host copy streams of the end-to-end sweep")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true", help="skip the reference-signature render() timing")
    ap.add_argument("--dropin-frames", type=int, default=10)
    ap.add_argument("--cpu-budget-s", type=float, default=150.0)
    ap.add_argument("--no-train", action="store_true", help="skip the config-5 training-step measurement")
    ap.add_argument("--no-train-batches", action="store_true", help="skip config-5 batches 16 and 32")
    ap.add_argument("--train-prims", type=int, default=3_000_000)
    ap.add_argument("--train-views-per-gpu", type=int, default=8)
    ap.add_argument("--train-steps", type=int, default=5)
    ap.add_argument("--train-inflight", type=int, default=8, help="views in flight per GPU in the training step")
    ap.add_argument("--train-group", type=int, default=8, help="training views per shared preprocess")
    ap.add_argument("--train-separate-epilogue", action="store_true",
                    help="plain Adam + separate zero / regulariser passes (A/B of the fused optimizer step)")
    ap.add_argument("--train-first-group", type=int, default=0,
                    help="views in a batch's first preprocess group (0: --train-group)")
    ap.add_argument("--train-ppl", type=int, default=4, choices=[2, 4, 8],
                    help="raster backward pixels per lane in the training step")
    ap.add_argument("--train-only", action="store_true",
                    help="only the config-5 training step (its own JSON line; for profiling)")
    return ap.parse_args()


def workload_config(a):
    return {"workload": f"config 4: {a.nd}D UBS scene, {a.n_prims} primitives, {a.width}x{a.height}, "
                        f"{SWEEP}-frame time sweep (one frame per step)",
            "n_prims": a.n_prims, "n_dims": a.nd, "width": a.width, "height": a.height,
            "sweep_frames": SWEEP, "frames_in_flight": a.inflight, "frames_per_preprocess": max(a.group, 1),
            "scene": "synth(nd, N, seed=1) (SURVEY 8d), float32 records",
            "l2": "inputs exceed L2: 4*P*N = %.0f MB of primitive records (> 126 MB L2) are re-read every "
                  "frame; no explicit flush" % (4 * (14 + 6 * (a.nd - 3)) * a.n_prims / 1e6)}


def frame_query(nd, cam, k):
    """Query of step k: sweep frame (37 k) mod 300 -- 37 is coprime with the
    sweep length, so 300 steps visit every frame once and any shorter run
    samples the whole time range instead of its cheap start."""
    from paper_2510_03312_b200 import synthetic as S
    return S.bench_query(nd, cam, ((37 * k) % SWEEP) / (SWEEP - 1))


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(gpu_index)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.count(",") >= 9]
        os.unlink(self.f.name)
        sm = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        mx = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[6:10]):
                if v.strip() == "Active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def physical_gpu_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].strip().isdigit():
            return int(ids[local_rank])
    return local_rank


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_issue(stage: str):
    """Issue-rate roofline of the stage's longest kernel from the committed ncu
    capture (profiles/issue.json): warp instructions / duration against
    148 SMs x 4 schedulers x 1 warp-instruction per clock."""
    p = ROOT / "profiles" / "issue.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    ks = [(k, v) for k, v in d.items() if isinstance(v, dict) and v.get("stage") == stage]
    if not ks:
        return None
    k, v = max(ks, key=lambda kv: kv[1]["duration_us"])
    return {"kernel": k, "bound": "issue", "achieved": v["achieved_warp_inst_per_s"],
            "peak": v["peak_warp_inst_per_s"], "unit": "warp-instructions/s", "frac": v["frac"],
            "warp_instructions": v["warp_instructions"], "source": "profiles/issue.json (ncu capture)"}


def ncu_traffic(stage: str):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(stage)
    return None


# ---------------------------------------------------------------------------
# CPU reference (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------
def cpu_frames(scene, cam, nd, settings, budget_s, max_frames, warm=True):
    from oracle import ubs_oracle as O
    O.set_threads(os.cpu_count() or 1)
    if warm:
        small = scene.take(np.arange(min(2000, scene.n_primitives)))
        O.render_frame(small, cam, frame_query(nd, cam, 0), settings)
    t0 = time.perf_counter()
    done = 0
    while done < max_frames:
        O.render_frame(scene, cam, frame_query(nd, cam, done), settings)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done, dt


def run_reference(a, rank, world):
    if rank != 0:
        return None
    from paper_2510_03312_b200 import synthetic as S
    from paper_2510_03312_b200.types import DEFAULT_SETTINGS
    scene = S.synth(a.nd, a.n_prims, seed=1)
    cam = S.bench_camera(a.width, a.height)
    cores = os.cpu_count() or 1
    # warm-up frames (bounded), then the timed steps, all inside the budget
    cpu_frames(scene, cam, a.nd, DEFAULT_SETTINGS, a.cpu_budget_s / 4, min(a.warmup, 1))
    done, dt = cpu_frames(scene, cam, a.nd, DEFAULT_SETTINGS, a.cpu_budget_s, a.steps, warm=False)
    fps = done / dt
    sample = (f"{done} of {a.steps} requested frames timed (budget {a.cpu_budget_s:.0f} s); oracle port of "
              f"betasplat render_with_cache: numpy fp64 slice/project + C (OpenMP) build_tiles/tile_forward")
    return {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": done,
            "warmup": min(a.warmup, 1),
            "warmup_note": "one full CPU frame (after a 2000-primitive frame) warms the oracle; more would only "
                           "lengthen a run bounded to a few minutes", "ms_per_step": 1e3 * dt / max(done, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(a), "impl": "reference",
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------------------
# ours
# ---------------------------------------------------------------------------
def algorithmic_bytes(stage, n, statics_per_prim, n_vis, entries, ids, npix, ntiles, k_pairs=0, P=38):
    """Algorithmic HBM bytes of one launch of each stage, SURVEY §8(d) per-unit
    figures: raster 48 B per visible record + 4 B per tile
    pair + 20 B per pixel; the other stages by their own minimal traffic.

    entries: level-1 bucket entries of the frame; ids: tile-list ids
    materialised (list prefixes up to the cap); k_pairs: K."""
    return {
        # read the fp32 params (4P), write the raster record 48 + key 8 + count 4 + id 4 (§8d "4P + 64")
        "preprocess": n * (4 * P + 64),
        # §8(d) depth sort: one read + write pass of 12 B per visible primitive
        "bin_depth": n_vis * 24 + ntiles * 8,
        # §8(d) pair emit 12 + one sort pass 24 + range scan 8 per pair (the raster's 4 B id read is its own)
        "bin_tiles": k_pairs * 44,
        "raster": 48 * n_vis + 4 * k_pairs + 20 * npix,
        "fixup": 0,
    }[stage]


def prefix_model_bytes(stage, n, statics_per_prim, n_vis, entries, ids, npix, ntiles):
    """The bytes this design actually has to move (materialised list prefixes,
    64 B records, statics): reported beside the §8(d) model."""
    return {
        "preprocess": n * (statics_per_prim + 166),
        "bin_depth": ntiles * 8 + n * 16 + n_vis * (12 + 12 + 4),
        "bin_tiles": n_vis * 32 + entries * 16 + ids * 4 + ntiles * 8,
        "raster": ntiles * 8 + 4 * ids + 64 * n_vis + 24 * npix,
        "fixup": 0,
    }[stage]


def run_train(a, rank, world, local_rank):
    """Config 5: 7D training step, 3M prims, batch = 8 views per GPU (1080p orbit),
    views sharded over ranks, one NCCL all-reduce of the flat gradient, device Adam."""
    import torch
    import torch.distributed as dist
    from paper_2510_03312_b200 import engine, sharding, synthetic as S
    from paper_2510_03312_b200.types import LossConfig

    dev = torch.device("cuda", local_rank)
    scene = S.synth(7, a.train_prims, seed=1)
    ds = engine.DeviceScene.from_scene(scene, dtype=torch.float32, device=dev)
    batch = a.train_views_per_gpu * world
    cams = [S.bench_camera(a.width, a.height, k, batch) for k in range(batch)]
    views_q = [S.bench_query(7, c, 0.5) for c in cams]
    # targets: renders of synth(7, N, seed=2), made on this GPU, then resident
    tds = engine.DeviceScene.from_scene(S.synth(7, a.train_prims, seed=2), dtype=torch.float32, device=dev)
    tws = engine.Workspace(dev, "fp32")
    targets = []
    for c, q in zip(cams, views_q):
        targets.append(engine.render_frame(tws, tds, c, q).image.clone().clamp_(0.0, 1.0))
    del tws, tds
    views = list(zip(cams, views_q, targets))
    # more views than slots: two groups' worth of slots, so one group's shared
    # preprocess and views overlap the previous group's (with one group's worth
    # the groups of a batch run back to back)
    depth = a.train_inflight if a.train_views_per_gpu <= a.train_inflight else \
        min(a.train_views_per_gpu, 2 * a.train_group)
    step = sharding.ViewShardedStep(sharding.GpuViewBackend(ds, "fp32", depth=depth, group=a.train_group,
                                                            pixels_per_lane=a.train_ppl,
                                                            first_group=a.train_first_group or None))
    adam = sharding.DeviceAdam(ds.params, 7)
    cfg = LossConfig()
    grad = step.backend.new_grad()
    # the optimizer pass also prepares the next batch's gradient buffer (its
    # zeroing, rank 0's regulariser gradient, the regulariser value)
    for _ in range(2):
        loss, grad = step.loss_and_grad(views, cfg, grad)
        step.optimizer_step(adam, grad, cfg)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.train_steps):
        loss, grad = step.loss_and_grad(views, cfg, grad)
        if a.train_separate_epilogue:
            adam.step(grad)
        else:
            step.optimizer_step(adam, grad, cfg)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / a.train_steps
    return {"metric": "train iters/sec", "value": 1e3 / ms, "unit": "iters/s", "ms_per_iter": ms,
            "views_per_s": batch * 1e3 / ms, "loss": float(loss),
            "config": {"workload": f"config 5: 7D UBS training step, {a.train_prims} primitives, batch {batch} "
                                   f"1920x1080 orbit views ({a.train_views_per_gpu} per GPU, {depth} in "
                                   f"flight, groups of {a.train_group} sharing one preprocess), "
                                   f"fwd + L1/SSIM + bwd + all-reduce + Adam",
                       "parallelism": f"dp{world} (view sharding, NCCL "
                                   f"all-reduce of the {4 * 38 * a.train_prims / 1e6:.0f} MB gradient)"},
            "steps": a.train_steps, "warmup": 2, "dtype": "f32 (fp64 geometry/chain)", "data": "synthetic",
            "retries": step.retries,
            # the step's dominant kernel (raster backward, ~40% of it), from the committed ncu capture
            "issue_roofline": ncu_issue("train_raster_bwd")}


def run_config1(a, dev, steps=200):
    """BASELINE.json configs[0]: synthetic 7D scene, 10k primitives, one 128x128
    view at t = 0.5, forward + backward (testing.random_scene(7, 10000, seed=1),
    random_camera(128, seed=2), target from a second scene: SURVEY 8(d)).
    A step = render + L1/SSIM image gradient + raster backward + chain into
    the parameter gradient.  Timed three ways: the device engine step by
    step (eager launches), the same step captured once in a CUDA graph and
    replayed (the step is ~20 small launches: launch-latency bound), and the
    reference-signature gradients.backward() with host arrays; next to the
    CPU oracle port of the reference on the same step."""
    import torch
    from oracle import ubs_oracle as O
    from paper_2510_03312_b200 import engine, synthetic as S
    from paper_2510_03312_b200.gradients import backward
    from paper_2510_03312_b200.types import DEFAULT_SETTINGS, LossConfig, Query, quantize_f32
    sc = quantize_f32(S.random_scene(7, 10000, seed=1))
    cam = S.random_camera(128, 2)
    q = Query.view_time(0.5, cam.forward)
    tgt = np.clip(O.render_frame(quantize_f32(S.random_scene(7, 5000, seed=978)), cam, q,
                                 DEFAULT_SETTINGS)["image"], 0.0, 1.0)
    cfg = LossConfig()
    ds = engine.DeviceScene.from_scene(sc, device=dev)
    ws = engine.Workspace(dev, "fp32")
    target = torch.from_numpy(tgt).float().to(dev)
    grad = torch.zeros(ds.params.shape, dtype=torch.float32, device=dev)
    engine.render_frame(ws, ds, cam, q, sync=True)  # sizes the pair buffers
    ws.ensure_pairs(int(ws.pair_cap * 1.5))

    def step():
        fr = engine.render_frame(ws, ds, cam, q, sync=False)
        ws.loss_parts.zero_()
        g_img, _ = engine.loss_image_grad(fr, target, cfg.lambda_ssim, cfg.loss_scale)
        engine.backward_frame(fr, ds, g_img, grad)

    def timed(fn, n):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    for _ in range(5):
        step()
    eager_ms = timed(step, steps)
    engine.check_status(ws)
    graph_ms, graph_err = None, None
    try:
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                step()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        graph_ms = timed(g.replay, steps)
        engine.check_status(ws)
    except Exception as e:  # report, keep the eager numbers
        graph_err = f"{type(e).__name__}: {e}"[:200]
    frames = [(cam, q, tgt)]
    backward(sc, frames, cfg, DEFAULT_SETTINGS)
    t0 = time.perf_counter()
    for _ in range(10):
        backward(sc, frames, cfg, DEFAULT_SETTINGS)
    dropin_ms = (time.perf_counter() - t0) / 10 * 1e3
    O.set_threads(os.cpu_count() or 1)
    O.backward(sc, frames, cfg, DEFAULT_SETTINGS)
    t0 = time.perf_counter()
    for _ in range(3):
        O.backward(sc, frames, cfg, DEFAULT_SETTINGS)
    cpu_ms = (time.perf_counter() - t0) / 3 * 1e3
    return {"workload": "config 1: 7D random_scene(7, 10000, seed=1), 128x128 random_camera(128, 2), t = 0.5, "
                        "forward + L1/SSIM + backward to raw parameters",
            "unit": "steps/s", "eager": {"value": 1e3 / eager_ms, "ms_per_step": eager_ms},
            "cuda_graph": {"value": 1e3 / graph_ms, "ms_per_step": graph_ms} if graph_ms else {"error": graph_err},
            "dropin_backward": {"value": 1e3 / dropin_ms, "ms_per_step": dropin_ms,
                                "path": "gradients.backward(scene, [(cam, query, target)]) host arrays in, "
                                        "SceneGrads out"},
            "cpu_baseline": {"value": 1e3 / cpu_ms, "ms_per_step": cpu_ms, "cores": os.cpu_count() or 1,
                             "kind": "port"}}


def run_other_configs(a, dev, frames=64):
    """BASELINE.json configs 1 and 2 on this GPU (informational, single rank):
    3D static 1M primitives and 6D view-dependent 2M primitives, each a
    64-view 1080p orbit through a FramePipeline of a.inflight frames, in
    groups of a.group sharing one preprocess."""
    import torch
    from paper_2510_03312_b200 import engine, synthetic as S
    from paper_2510_03312_b200.types import DEFAULT_SETTINGS
    out = {}
    for name, nd, n in (("3D static, 1M primitives, 1080p 64-view orbit", 3, 1_000_000),
                        ("6D view-dependent, 2M primitives, 1080p 64-view orbit", 6, 2_000_000)):
        ds = engine.DeviceScene.from_scene(S.synth(nd, n, seed=1), device=dev)
        cams = [S.bench_camera(a.width, a.height, k, frames) for k in range(frames)]
        qs = [S.bench_query(nd, c) for c in cams]
        pipe = engine.FramePipeline(ds, max(a.inflight, 1), "fp32", dev)
        for k in range(2 * pipe.depth):
            pipe.render(cams[k % frames], qs[k % frames], DEFAULT_SETTINGS, sync=True)
        ms = None
        for _ in range(2):  # a second pass if an asynchronous frame outgrew its slot
            pipe.clear_status()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ds.invalidate_statics()
            e0.record()
            g = max(a.group, 1)
            for k0 in range(0, frames, g):
                if g > 1:
                    pipe.render_group(list(zip(cams[k0:k0 + g], qs[k0:k0 + g])), DEFAULT_SETTINGS)
                else:
                    pipe.render(cams[k0], qs[k0], DEFAULT_SETTINGS)
            pipe.join()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if int(pipe.status().item()) == 0:
                break
            pipe.grow()
        out[name] = {"value": frames / (ms / 1e3), "unit": "frames/s", "frames": frames,
                     "frames_in_flight": pipe.depth, "frames_per_preprocess": max(a.group, 1)}
        del pipe, ds
        torch.cuda.empty_cache()
    return out


def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2510_03312_b200 import engine, synthetic as S
    from paper_2510_03312_b200.types import DEFAULT_SETTINGS

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    scene = S.synth(a.nd, a.n_prims, seed=1)
    cam = S.bench_camera(a.width, a.height)
    dtype = torch.float64 if a.precision == "fp64" else torch.float32
    ds = engine.DeviceScene.from_scene(scene, dtype=dtype, device=dev)
    # the sweep renders through a pipeline of `inflight` frames (own stream and
    # workspace each); the per-stage breakdown uses one extra single-stream
    # workspace so its event times are not inflated by the overlap
    pipe = engine.FramePipeline(ds, max(a.inflight, 1), a.precision, dev, slot_priority=a.slot_priority,
                                lead_priority=a.lead_priority)
    ws = engine.Workspace(dev, a.precision)

    def frame(k, timers=None, sync=False):
        return pipe.render(cam, frame_query(a.nd, cam, rank + world * k), DEFAULT_SETTINGS, timers=timers,
                           sync=sync)

    def frames(k0, count):
        """frames k0 .. k0+count-1 of this rank: grouped (one preprocess per group) or one by one"""
        out = []
        for g0 in range(k0, k0 + count, max(a.group, 1)):
            ks = range(g0, min(g0 + max(a.group, 1), k0 + count))
            if a.group > 1:
                out += pipe.render_group([(cam, frame_query(a.nd, cam, rank + world * k)) for k in ks],
                                         DEFAULT_SETTINGS)
            else:
                out += [frame(k) for k in ks]
        return out

    def frame_single(k, timers=None, sync=False):
        return engine.render_frame(ws, ds, cam, frame_query(a.nd, cam, rank + world * k), DEFAULT_SETTINGS,
                                   timers=timers, sync=sync)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up: synchronous frames size the pair buffers for the whole sweep
    # (capacity grows by 1.3x), the timed frames are fully asynchronous
    for k in range(max(a.warmup, pipe.depth)):
        frame(k, sync=True)
    for k in range(max(a.warmup, 1)):
        frame_single(k, sync=True)
    stats = {"n_vis": 0, "k": 0, "frames": 0, "entries": 0, "ids": 0}
    for k in range(0, SWEEP, 25):
        fr = frame_single(k, sync=True)
        stats["n_vis"] += fr.n_visible
        stats["k"] += fr.n_pairs
        stats["frames"] += 1
        e, i = engine.list_stats(ws, fr)
        stats["entries"] += e
        stats["ids"] += i
    torch.cuda.synchronize()

    # --- device-resident throughput -------------------------------------
    host_ms = [0.0]

    def timed_sweep(timers=None):
        render = frame if timers is None else frame_single
        sampler = ClockSampler(physical_gpu_index(local_rank))
        time.sleep(0.3)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ds.invalidate_statics()  # the sweep pays its one scene-statics pass
        e0.record()
        h0 = time.perf_counter()
        if timers is None:
            fr = frames(0, a.steps)[-1]
        else:
            for k in range(a.steps):
                fr = render(k, timers)
        host_ms[0] = (time.perf_counter() - h0) * 1e3  # host time to enqueue the sweep
        pipe.join()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        clocks = sampler.stop()
        return e0.elapsed_time(e1), timers, clocks, fr

    # the headline sweep carries no per-stage events (they cost ~3.5%); a second,
    # instrumented sweep below gives the stage breakdown
    for attempt in range(3):
        ms, _, clocks, fr = timed_sweep()
        host_enqueue_ms = host_ms[0]
        # no async frame may have outgrown its pair buffers (decided jointly by all ranks)
        bad = pipe.status().to(torch.int32)
        if world > 1:
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if int(bad.item()) == 0:
            break
        pipe.grow()  # every slot sized for what any slot needed, then re-time
    else:
        raise RuntimeError("pair-buffer overflow persisted")
    fixed = fr.n_fixed
    visits = fr.processed_pixels
    _, timers, _, _ = timed_sweep({})
    engine.check_status(ws)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * a.steps / (ms_max / 1e3)

    stage_ms = {s: sum(x.elapsed_time(y) for x, y in ev) / len(ev) for s, ev in timers.items()}
    dominant = max(stage_ms, key=stage_ms.get)
    n = ds.n
    P = 14 + 6 * (a.nd - 3)
    npix = a.width * a.height
    ntiles = -(-a.width // 16) * -(-a.height // 16)
    n_vis = stats["n_vis"] / stats["frames"]  # sweep average over 12 sampled frames
    kk = stats["k"] / stats["frames"]
    ent = stats["entries"] / stats["frames"]
    nids = stats["ids"] / stats["frames"]
    spp = ds.statics_bytes_per_prim()
    b_dom = algorithmic_bytes(dominant, n, spp, n_vis, ent, nids, npix, ntiles, kk, P)
    b_pre = prefix_model_bytes(dominant, n, spp, n_vis, ent, nids, npix, ntiles)
    peak, peak_src = measured_peak()
    achieved = b_dom / (stage_ms[dominant] / 1e3) / 1e9
    b_frame = n * (4 * P + 64) + 72 * n_vis + 48 * kk + 20 * npix  # SURVEY §8(d) B_fwd
    traffic = ncu_traffic(dominant)

    # --- end to end: image streamed to pinned host memory every frame -----
    sink = engine.HostFrameSink(a.height, a.width, dtype=ws.image_buf.dtype, device=dev, copy_streams=a.copy_streams)

    def submit(k0, count=1):
        g = max(a.group, 1)
        for g0 in range(k0, k0 + count, g):  # each group's copies are queued before the next group renders
            submit_frames(frames(g0, min(g, k0 + count - g0)))

    def submit_frames(frs):
        for fr in frs:
            if pipe.depth > 1:
                # zero-copy: the D2H reads the slot's own image; the slot's next frame waits for it
                sink.submit(fr, source_stream=pipe.stream_of(fr))
                pipe.hold(fr, sink.last_copy)
            else:  # one slot: snapshot on the device so the next frame need not wait for the copy
                with torch.cuda.stream(pipe.stream_of(fr)):
                    sink.submit(fr)

    submit(0, 2 * pipe.depth)
    sink.synchronize()
    torch.cuda.synchronize()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for attempt in range(3):
        ds.invalidate_statics()
        f0.record()
        submit(0, a.steps)
        pipe.join()
        sink.join()
        f1.record()
        torch.cuda.synchronize()
        # as in the headline sweep: an asynchronous frame that outgrew its slot
        # (frames land on other slots than in that sweep) means re-time after growing
        bad = pipe.status().to(torch.int32)
        if world > 1:
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if int(bad.item()) == 0:
            break
        pipe.grow()
        sink.synchronize()
        torch.cuda.synchronize()
    else:
        raise RuntimeError("pair-buffer overflow persisted in the end-to-end sweep")
    barrier()
    te = torch.tensor([f0.elapsed_time(f1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * a.steps / (float(te.item()) / 1e3)
    # the link's own ceiling: back-to-back device -> pinned host copies of one frame's image
    src = torch.empty(sink.bytes_per_frame, dtype=torch.uint8, device=dev)
    dst = torch.empty(sink.bytes_per_frame, dtype=torch.uint8, pin_memory=True)
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0.record()
    for _ in range(20):
        dst.copy_(src, non_blocking=True)
    l1.record()
    torch.cuda.synchronize()
    d2h_gbs = 20 * sink.bytes_per_frame / (l0.elapsed_time(l1) / 1e3) / 1e9
    del src, dst
    import ctypes
    from paper_2510_03312_b200._lib import UbsView
    h2d = ctypes.sizeof(UbsView)  # camera + query + settings travel as kernel parameters

    # --- end to end through the reference-signature drop-in ----------------
    # raster.render(scene, cam, query) -> (H, W, 3) float64 numpy, as betasplat
    # callers use it: every call stages the host scene (152 MB of f32 records
    # at 7D 1M) and returns a host image; then the same inside
    # raster.resident(scene) (scene uploaded once, images only)
    dropin = None
    if rank == 0 and not a.no_dropin:
        from paper_2510_03312_b200 import raster as R
        for k in range(2):  # warm: workspace, pinned staging, the pinned blocks of two live images
            img = R.render(scene, cam, frame_query(a.nd, cam, k), DEFAULT_SETTINGS)
        t0 = time.perf_counter()
        for k in range(a.dropin_frames):
            img = R.render(scene, cam, frame_query(a.nd, cam, k), DEFAULT_SETTINGS)
        per_call = (time.perf_counter() - t0) / a.dropin_frames
        with R.resident(scene):
            img = R.render(scene, cam, frame_query(a.nd, cam, 0), DEFAULT_SETTINGS)
            t0 = time.perf_counter()
            for k in range(a.dropin_frames * 4):
                img = R.render(scene, cam, frame_query(a.nd, cam, k), DEFAULT_SETTINGS)
            per_res = (time.perf_counter() - t0) / (a.dropin_frames * 4)
        P = 14 + 6 * (a.nd - 3)
        dropin = {"value": 1.0 / per_call, "unit": "frames/s", "frames": a.dropin_frames,
                  "h2d_bytes_per_step": 4 * P * scene.n_primitives, "d2h_bytes_per_step": int(img.nbytes),
                  "path": "raster.render(scene, cam, query) (reference signature, host numpy in, (H,W,3) float64 "
                          "out); the scene's float64 arrays are staged (cast to f32 records by host threads) "
                          "and uploaded every call",
                  "resident": {"value": 1.0 / per_res, "unit": "frames/s", "frames": a.dropin_frames * 4,
                               "path": "same calls inside raster.resident(scene): the scene uploaded once"}}
        del img

    # --- CPU baseline (rank 0, N = 1 only) --------------------------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        done, dt = cpu_frames(scene, cam, a.nd, DEFAULT_SETTINGS, 30.0, 1)
        cpu = {"value": done / dt, "unit": "frames/s", "cores": os.cpu_count() or 1, "kind": "port",
               "sample": f"{done} frame(s) of the same sweep on the oracle port (numpy fp64 slice/project, "
                         f"C OpenMP binning + compositing) with {os.cpu_count()} host threads"}

    train = None
    other = None
    if not a.no_train:
        del ws, pipe
        torch.cuda.empty_cache()
        if world == 1:
            other = run_other_configs(a, dev)
            other["config1"] = run_config1(a, dev)
        train = run_train(a, rank, world, local_rank)
        if world == 1 and not a.no_train_batches:
            train["batches"] = {str(a.train_views_per_gpu): train["value"]}
            for b in (16, 32):  # BASELINE config 5 batches on one GPU
                if b != a.train_views_per_gpu:
                    import copy
                    ab = copy.copy(a)
                    ab.train_views_per_gpu = b
                    torch.cuda.empty_cache()
                    train["batches"][str(b)] = run_train(ab, rank, world, local_rank)["value"]

    if rank != 0:
        return None
    # kernels of libubs_b200.so per frame (ncu launch list, profiles/r01_launches_v4.csv):
    # preprocess, tile_scan, depth hist, CUB scan (init + scan), depth scatter, depth rank,
    # bucket hist, bucket offsets, bucket scatter, tile_lists, raster, fixup; plus one
    # scene-statics pass per sweep
    per_frame_launches = 13
    out = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if a.precision == "fp32" else "f64",
        "precision_note": "fp64 preprocess (slice/project/rect); fp32 raster; pixels with uncertified "
                          "cut/clamp decisions re-done in fp64 (bit-exact counts)",
        "data": "synthetic", "config": workload_config(a),
        "parallelism": f"view sharding over {world} GPU(s), no data-path collective",
        "roofline": {"kernel": dominant, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": b_dom, "byte_model": "SURVEY 8(d): 48 N_vis + 4 K + 20 HW",
                     "launch_ms": stage_ms[dominant],
                     "prefix_model": {"bytes_per_launch": b_pre,
                                      "frac": b_pre / (stage_ms[dominant] / 1e3) / 1e9 / peak,
                                      "note": "64 B records, materialised list prefixes only, 24 B/px"}},
        "issue_roofline": ncu_issue(dominant) if a.precision == "fp32" else None,
        "frame_roofline": {"bytes_per_frame": b_frame, "achieved_gbs": b_frame / (ms_max / a.steps / 1e3) / 1e9,
                           "frac": b_frame / (ms_max / a.steps / 1e3) / 1e9 / peak,
                           "ceiling_fps": peak * 1e9 / b_frame},
        "stage_ms": stage_ms,
        "per_frame": {"n_visible": n_vis, "tile_pairs": kk, "visits": visits, "fixup_pixels": fixed},
        "visit_throughput_per_s": visits / (ms_max / a.steps / 1e3),
        # host (Python + driver) time to enqueue the timed sweep: well below the
        # device time means the GPU never waited for the host
        "host_enqueue_ms_per_step": host_enqueue_ms / a.steps,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": sink.bytes_per_frame,
                "path": f"engine.FramePipeline + HostFrameSink (fp32 image -> pinned host, {a.copy_streams} copy stream(s))",
                "d2h_link_gbs": d2h_gbs, "link_ceiling_fps": d2h_gbs * 1e9 / sink.bytes_per_frame},
        # one preprocess launch per group of frames (--group), the rest per frame
        "e2e_dropin": dropin,
        "gpu_launches": (per_frame_launches - 1) * a.steps + -(-a.steps // max(a.group, 1)) + 1,
        "clocks": clocks,
        "train": train,
        "other_configs": other,
    }
    return out


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(a) -> int:
    """``--gpus N`` (N > 1) outside torchrun: check that N GPUs exist, then run
    this script under torch.distributed.run with one rank per GPU (the
    launch the driver itself uses).  Fails loudly rather than timing fewer GPUs."""
    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(f"bench.py: --gpus {a.gpus} requested but only {have} CUDA device(s) are visible", file=sys.stderr,
              flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def nccl_init(world: int, local_rank: int) -> dict:
    """NCCL process group with INIT-level debug output captured to a per-rank
    file; returns the communicator facts rank 0 reports (every rank's
    communicator must have nRanks == world)."""
    import glob
    import re
    import torch
    import torch.distributed as dist
    logdir = Path(tempfile.mkdtemp(prefix="ubs_nccl_"))
    if "NCCL_DEBUG" not in os.environ:
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        os.environ["NCCL_DEBUG_FILE"] = str(logdir / "nccl.%h.%p.log")
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    t = torch.ones(1, device=f"cuda:{local_rank}")
    dist.all_reduce(t)  # forces communicator creation on every rank
    torch.cuda.synchronize()
    lines = []
    for f in glob.glob(str(logdir / "nccl.*.log")):
        lines += [ln.strip() for ln in Path(f).read_text(errors="replace").splitlines()
                  if "nRanks" in ln or "NVLS" in ln or "Init COMPLETE" in ln]
    nr = [int(m.group(1)) for ln in lines for m in [re.search(r"nRanks (\d+)", ln)] if m]
    ok = torch.tensor([1 if (nr and all(x == world for x in nr)) else 0], device=t.device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return {"world_size": world, "allreduce_sum": float(t.item()), "comm_nranks_ok": bool(ok.item()),
            "log_lines": lines[:6]}


def main():
    a = parse()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1 and a.impl == "ours":
        return relaunch(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        if rank != 0:
            return 0
        res = run_reference(a, rank, world)
        print(json.dumps(res), flush=True)
        return 0
    if world != a.gpus:
        print(f"bench.py: launched with WORLD_SIZE={world} but --gpus {a.gpus}", file=sys.stderr, flush=True)
        return 2
    nccl = None
    if world > 1:
        import torch
        if torch.cuda.device_count() < world:
            print(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s)", file=sys.stderr)
            return 2
        nccl = nccl_init(world, local_rank)
    res = run_train(a, rank, world, local_rank) if a.train_only else run_ours(a, rank, world, local_rank)
    if rank == 0:
        if nccl is not None:
            res["nccl"] = nccl
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
