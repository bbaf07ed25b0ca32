"""Aggregate an ncu '--page source --print-source cuda,sass --csv' dump per CUDA source line.

usage: python tools/ncu_lines.py dump.csv [top] [cells]
Prints, per source line: warp-instructions (per cell if `cells` is given),
share of stall samples, active threads per instruction, excess shared-memory
wavefronts (bank conflicts)."""
import collections
import csv
import sys

import gzip
rows = list(csv.reader(gzip.open(sys.argv[1], "rt") if sys.argv[1].endswith(".gz") else open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cells = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
agg = collections.defaultdict(lambda: [0, 0, 0, 0, ""])
hdr = None
fname = ""
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        cur = f"{fname}:{r[0]}"
        agg[cur][4] = r[1].strip()[:80]
        continue
    if len(r) < len(hdr) or cur is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ie = int(d.get("Instructions Executed") or 0)
        st = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        ti = int(d.get("Thread Instructions Executed") or 0)
        ex = d.get("L1 Wavefronts Shared Excessive") or "0"
        ex = int(ex) if ex.isdigit() else 0
    except ValueError:
        continue
    a = agg[cur]
    a[0] += ie
    a[1] += st
    a[2] += ti
    a[3] += ex
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr {ti}" + (f" ({ti / cells:.2f} per cell)" if cells else "") + f"  stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    per = f"{v[0] / cells:5.2f}/cell" if cells else f"{v[0] / ti * 100:5.1f}%"
    print(f"{per} {v[1] / ts * 100:5.1f}% stall thr {v[2] / max(v[0], 1):4.1f} xs-wav {v[3]:9d}  {k:18s} {v[4]}")
