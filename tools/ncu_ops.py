#!/usr/bin/env python3
"""Per-opcode executed-instruction and stall-sample breakdown of one kernel from an
ncu --set full capture (--page source, SASS), normalised per unit of work.

    python tools/ncu_ops.py gpurun_out/x.ncu-rep --kernel k_cdc64_tc --units 16777220
"""
import argparse
import collections
import csv
import io
import re
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--kernel", required=True)
ap.add_argument("--units", type=float, default=1.0, help="work units per launch (e.g. blocks)")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--lines", type=int, default=0, help="also list the N SASS lines with most stall samples")
a = ap.parse_args()

raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--kernel-name", "regex:" + a.kernel],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "launch__occupancy_limit_registers",
          "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.per_cycle_active",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"):
    print(f"{k:70s} {d.get(k)}")
st = [(float(d[k].replace(",", "")), k) for k in rows[0]
      if k.startswith("smsp__pcsamp_warps_issue_stalled") and d[k] and not k.endswith("_not_issued")]
st.sort(reverse=True)
tot = sum(v for v, _ in st) or 1
print("stalls:", [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), round(v / tot, 3)) for v, k in st[:10]])

src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + a.kernel], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
iA, iS = hdr.index("Address"), hdr.index("Source")
iE, iW = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[2:]:
    if len(r) <= iE or not r[iE].replace(",", "").isdigit():
        break
    lines.append((r[iA], r[iS].strip(), int(r[iE].replace(",", "")), int(r[iW].replace(",", "") or 0)))
cnt, stall = collections.Counter(), collections.Counter()
for _, s, e, w in lines:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", s)
    if m:
        cnt[m.group(2)] += e
        stall[m.group(2)] += w
tw = sum(stall.values()) or 1
print(f"instructions per unit: {sum(cnt.values()) / a.units:.2f}")
for op, n in cnt.most_common(a.top):
    print(f"  {op:26s} {n / a.units:8.2f}   stall% {100 * stall[op] / tw:5.1f}")
if a.lines:
    idx = sorted(range(len(lines)), key=lambda i: -lines[i][3])[:a.lines]
    for i in sorted(idx):
        print(f"  {i:5d} {lines[i][1][:64]:64s} exec={lines[i][2]:10d} stall%={100 * lines[i][3] / tw:5.2f}")
