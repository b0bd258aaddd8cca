"""Summarize an ncu report: key SOL metrics, opcode mix and stall hot spots."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "Issued Instructions",
        "SM Frequency", "Dynamic Shared Memory Per Block", "Local Memory Spilling Requests"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in keys:
        print(f"  {d['Metric Name']:40s} {d['Metric Unit']:14s} {d['Metric Value']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hh = rr[0]
    vals = dict(zip(hh, rr[2]))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "sm__warps_active.avg.pct_of_peak_sustained_active"):
        if k in vals:
            print(f"  {k:40s} {rr[1][hh.index(k)]:14s} {vals[k]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
tot = sum(int(d["Instructions Executed"] or 0) for d in data)
samp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
op = collections.Counter()
ops = collections.Counter()
for d in data:
    s = d["Source"].strip().split()
    if not s:
        continue
    o = s[1] if s[0].startswith("@") else s[0]
    o = o.split(".")[0]
    op[o] += int(d["Instructions Executed"] or 0)
    ops[o] += int(d["Warp Stall Sampling (All Samples)"] or 0)
print(f"  warp instructions {tot}, stall samples {samp}")
for o, c in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 22):
    print(f"    {o:10s} {c:12d} {100*c/tot:6.2f}%   stall {100*ops[o]/samp:6.2f}%")
