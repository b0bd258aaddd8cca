"""Stall reasons, shared-memory wavefronts and instruction counts of an ncu
report, overall and per code region (regions split at RET instructions, i.e.
per non-inlined device function; the kernel body is region 0)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]


def num(x):
    try:
        return float(x)
    except Exception:
        return 0.0


regions = []
cur = {"start": data[0]["Address"] if data else "", "rows": []}
for d in data:
    cur["rows"].append(d)
    s = d["Source"].strip()
    if s.startswith("RET") or " RET" in s[:12]:
        regions.append(cur)
        cur = {"start": None, "rows": []}
    elif cur["start"] is None:
        cur["start"] = d["Address"]
if cur["rows"]:
    regions.append(cur)


def summarize(rows, label):
    inst = sum(num(d["Instructions Executed"]) for d in rows)
    samp = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in rows)
    wf = sum(num(d["L1 Wavefronts Shared"]) for d in rows)
    wfi = sum(num(d["L1 Wavefronts Shared Ideal"]) for d in rows)
    st = collections.Counter()
    for d in rows:
        for c in stall_cols:
            st[c] += num(d[c])
    tot = sum(st.values()) or 1
    top = ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in st.most_common(7))
    print(f"{label}: inst {inst:.3e}  samples {samp:.0f}  smem wavefronts {wf:.3e} "
          f"(ideal {wfi:.3e})\n    {top}")
    return samp


total = summarize(data, "ALL")
ranked = sorted(regions, key=lambda r: -sum(num(d["Warp Stall Sampling (All Samples)"])
                                          for d in r["rows"]))
for r in ranked[: int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    summarize(r["rows"], f"region @{r['start']} ({len(r['rows'])} instr)")
