#!/usr/bin/env python
"""Regenerate profiles/traffic.json and profiles/issue.json from an ncu raw
CSV export (``ncu -i capture.ncu-rep --page raw --csv > rNN_ncu_full_vK_raw.csv``)
of ``ncu --set full --clock-control none`` over ``bench.py``.

traffic.json: per bench stage, dram__bytes_read.sum + dram__bytes_write.sum
of each of the stage's kernels, first launch of each kernel counted once
(bench.py divides nothing by it; it is reported as the dominant kernel's
``roofline.traffic``).

issue.json: per kernel, warp instructions / duration against the issue peak
148 SMs x 4 schedulers x 1 warp-instruction per clock at the captured SM
clock (bench.py's ``issue_roofline`` for the dominant stage).

    python profiles/make_rooflines.py profiles/r01_ncu_full_v5_raw.csv [more captures ...]

Several captures may be given (e.g. the frame's kernels and the training
step's raster backward); a kernel is taken from the first file holding it.
"""

from __future__ import annotations

import csv
import json
import re
import sys
from pathlib import Path

STAGES = [
    (r"statics_kernel", "statics"),
    (r"preprocess(_views)?_kernel", "preprocess"),
    (r"tile_scan|depth_|DeviceScan", "bin_depth"),
    (r"bucket_|tile_lists", "bin_tiles"),
    (r"raster_fwd", "raster"),
    (r"raster_fixup", "fixup"),
    (r"raster_bwd", "train_raster_bwd"),
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9,
         "inst": 1.0, "": 1.0}


def stage_of(name: str):
    for pat, st in STAGES:
        if re.search(pat, name):
            return st
    return None


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    return re.sub(r"\(.*$", "", name)


def main(paths):
    traffic, issue, seen = {}, {}, set()
    for path in paths:
        scan(path, traffic, issue, seen)
    src = ", ".join(f"profiles/{Path(p).name}" for p in paths)
    traffic["_source"] = (f"{src}: dram__bytes_read.sum + dram__bytes_write.sum per launch, summed over "
                          "the stage's kernels, each kernel counted once (profiles/make_rooflines.py)")
    issue["_source"] = f"{src} (profiles/make_rooflines.py)"
    out = Path(__file__).resolve().parent
    (out / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    (out / "issue.json").write_text(json.dumps(issue, indent=1) + "\n")
    for k, v in issue.items():
        if isinstance(v, dict):
            print(f"{k[:60]:60s} {v['stage']:16s} {v['duration_us']:8.1f} us  issue {v['frac']:.2f}")
    print({k: round(v / 1e6, 1) for k, v in traffic.items() if not k.startswith("_")}, "MB")


def scan(path, traffic, issue, seen):
    rows = list(csv.reader(open(path)))
    head, units = rows[0], rows[1]

    def val(row, key):
        i = head.index(key)
        return float(row[i].replace(",", "")) * SCALE.get(units[i], 1.0)

    for row in rows[2:]:
        name = short(row[head.index("Kernel Name")])
        st = stage_of(name)
        if st is None or name in seen:
            continue
        seen.add(name)
        traffic[st] = traffic.get(st, 0.0) + val(row, "dram__bytes_read.sum") + val(row, "dram__bytes_write.sum")
        dur_us = val(row, "gpu__time_duration.sum")
        inst = val(row, "smsp__inst_executed.sum")
        clk = val(row, "sm__cycles_elapsed.avg.per_second")
        peak = 148 * 4 * clk
        issue[name] = {"stage": st, "warp_instructions": inst, "duration_us": dur_us, "sm_clock_hz": clk,
                       "achieved_warp_inst_per_s": inst / (dur_us * 1e-6), "peak_warp_inst_per_s": peak,
                       "frac": inst / (dur_us * 1e-6) / peak}


if __name__ == "__main__":
    main(sys.argv[1:])
