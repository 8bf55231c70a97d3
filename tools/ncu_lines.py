#!/usr/bin/env python3
"""Per-CUDA-source-line executed warp instructions of one kernel from an ncu capture
(--import-source on, -lineinfo), normalised per work unit; optional diff of two captures.

    python tools/ncu_lines.py REP --kernel k_aeq_process --units 67108864 [--base REP0] [--top 40]
"""
import argparse
import csv
import io
import subprocess


def lines(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", "regex:" + kernel], capture_output=True, text=True).stdout
    res, fname, iE = {}, None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            iE = r.index("Instructions Executed")
            iW = r.index("Warp Stall Sampling (All Samples)")
            continue
        if iE is None or not r[0] or not r[0].isdigit() or len(r) <= iE:
            continue
        v = r[iE].replace(",", "")
        w = r[iW].replace(",", "")
        if v.isdigit() and int(v) > 0:
            res[(fname, int(r[0]))] = (int(v), r[1].strip()[:90], int(w) if w.isdigit() else 0)
    return res


ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--kernel", required=True)
ap.add_argument("--units", type=float, default=1.0)
ap.add_argument("--base")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--stalls", action="store_true", help="rank lines by warp stall samples instead")
a = ap.parse_args()
cur = lines(a.rep, a.kernel)
base = lines(a.base, a.kernel) if a.base else {}
keys = set(cur) | set(base)
if a.stalls:
    tot = sum(v[2] for v in cur.values()) or 1
    for k, v in sorted(cur.items(), key=lambda kv: -kv[1][2])[:a.top]:
        print(f"{100 * v[2] / tot:6.2f}% {v[0] / a.units:9.2f}  {k[0]}:{k[1]:<5d} {v[1]}")
    raise SystemExit
rows = []
for k in keys:
    c = cur.get(k, (0, ""))[0] / a.units
    b = base.get(k, (0, ""))[0] / a.units
    rows.append((c - b if a.base else c, c, b, k, (cur.get(k) or base.get(k))[1]))
rows.sort(key=lambda r: -abs(r[0]))
print(f"total {sum(r[1] for r in rows):.1f}" + (f"  base {sum(r[2] for r in rows):.1f}" if a.base else ""))
for d, c, b, (f, ln), src in rows[:a.top]:
    print(f"{d:9.2f} {c:9.2f} {b:9.2f}  {f}:{ln:<5d} {src}")
