"""Aggregate an ncu '--page source --print-source cuda,sass --csv' dump per CUDA source line."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
hdr = None; cur_line = None; cur_src = ""; fname = ""
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0]:
        cur_line = f"{fname}:{r[0]}"; cur_src = r[1]
    if len(r) < len(hdr) or not r[2]: continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ie = int(d.get("Instructions Executed") or 0); st = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        ti = int(d.get("Thread Instructions Executed") or 0)
    except ValueError:
        continue
    a = agg[cur_line]; a[0] += ie; a[1] += st; a[2] += ti; a[3] = cur_src.strip()[:90]
ti = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr {ti}  stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[0]/ti*100:5.1f}% inst {v[1]/ts*100:5.1f}% stall thr/inst {v[2]/max(v[0],1):4.1f}  {k:16s} {v[3]}")
