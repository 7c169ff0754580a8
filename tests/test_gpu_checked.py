"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool):
the bounds-checked build of the same sources (-DUBS_CHECKED: every guarded
shared / global index of the warp-synchronous binning stages, the raster's
ballot-word walk and list reads, the fix-up list, the tile grid, the
backward's writes is tested on the device, and a failure sets a status bit
and skips the access) runs the stress workloads of tests/tools/checked_run.py
-- tiny and odd image sizes, a frame past one CTA's tile scan, depth ties,
capped lists that run out, the 1080p grouped pipeline and the training
backend, both precisions, deterministic mode -- and every status word must be
zero."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parents[1]


def test_checked_build_reports_no_out_of_bounds_index():
    from paper_2510_03312_b200 import build
    build.build(variant="checked")
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "tools" / "checked_run.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    status = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert set(status) == {"binning", "preprocess", "raster", "prim_bwd", "loss", "optim"}
    assert all(v == 0 for v in status.values()), status
