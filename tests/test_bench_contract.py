"""bench.py's contract pieces that need no GPU: the sweep order, the
algorithmic-bytes model it divides by, and the reference arm's JSON line
(a tiny workload through the CPU oracle port)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_sweep_order_visits_every_frame_once():
    from paper_2510_03312_b200 import synthetic as S
    cam = S.bench_camera(64, 48)
    ts = [float(bench.frame_query(7, cam, k).dims[0]) for k in range(bench.SWEEP)]  # [t, d]
    assert len(set(round(t * (bench.SWEEP - 1)) for t in ts)) == bench.SWEEP
    # any prefix samples the whole time range, not its cheap start
    assert max(ts[:10]) - min(ts[:10]) > 0.5


def test_algorithmic_bytes_raster_model():
    # 48 B per visible record + 4 B per tile pair + 20 B per pixel
    n, n_vis, ids, npix, ntiles, k = 1000, 800, 5000, 4096, 16, 7000
    got = bench.algorithmic_bytes("raster", n, 352.0, n_vis, 0, ids, npix, ntiles, k)
    assert got == 48 * n_vis + 4 * k + 20 * npix
    pre = bench.prefix_model_bytes("raster", n, 352.0, n_vis, 0, ids, npix, ntiles)
    assert pre == 8 * ntiles + 4 * ids + 64 * n_vis + 24 * npix


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--n-prims", "3000", "--width", "64",
           "--height", "48", "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference"
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    for key in ("metric", "value", "unit", "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_gpus_flag_fails_loudly_without_the_gpus():
    # --gpus N outside torchrun re-launches under torch.distributed.run only
    # when N devices exist; here (no GPU) it must refuse, not time one device
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this box has the GPUs")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "--gpus 2" in r.stderr
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
