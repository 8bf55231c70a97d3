#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep \
        --launches gpurun_out/launches.csv --out profiles/ncu_summary_r01.json

Reads the `--page raw` metrics of a `--set full` capture (per-launch DRAM bytes,
pipe utilisation, issue activity, occupancy, top stall reasons) and the
gpu__time_duration launch list (per-kernel share of the step).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "warps_active_per_sm": ("sm__warps_active.avg.per_cycle_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "lsu_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
              "s": 1e9}


def short(name: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+)", name)
    return m.group(1) if m else name[:40]


def raw_page(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise_rep(rep: str) -> dict:
    hdr, units, rows = raw_page(rep)
    res = {}
    for r in rows:
        k = short(r[hdr.index("Kernel Name")])
        d = {}
        for key, (metric, sc) in KEYS.items():
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            try:
                v = float(r[i])
            except ValueError:
                continue
            u = units[i]
            if u in UNIT_SCALE:
                v *= UNIT_SCALE[u]
                if key == "duration_ms":
                    v = v * 1e-6
            d[key] = v
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        d["top_stalls_per_issue"] = {n: round(v, 3) for v, n in sorted(stalls, reverse=True)[:6]}
        d["dram_bytes"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
        res.setdefault(k, []).append(d)
    return res


def summarise_launches(path: str) -> dict:
    per = defaultdict(list)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        per[short(r["Kernel Name"])].append(v * UNIT_SCALE.get(unit, 1) * 1e-6)
    total = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "mean_ms": sum(v) / len(v), "share": sum(v) / total}
            for k, v in per.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    out = {"note": args.note}
    if args.rep:
        out["full_capture"] = summarise_rep(args.rep)
        out["per_launch_dram_bytes"] = {k: v[-1]["dram_bytes"] for k, v in out["full_capture"].items()}
    if args.launches:
        out["launch_list"] = summarise_launches(args.launches)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
