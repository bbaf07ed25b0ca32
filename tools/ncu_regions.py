"""Sum an ncu source-page dump (cuda,sass) over line ranges of one file.
usage: python tools/ncu_regions.py dump.csv cells name:a-b name:a-b ..."""
import collections, csv, sys
import gzip
rows = list(csv.reader(gzip.open(sys.argv[1], "rt") if sys.argv[1].endswith(".gz") else open(sys.argv[1])))
cells = float(sys.argv[2])
regs = [(x.split(":")[0], *map(int, x.split(":")[1].split("-"))) for x in sys.argv[3:]]
hdr = None; fname = ""; cur = None
ins = collections.Counter(); stl = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0]:
        cur = (fname, int(r[0])) if r[0].isdigit() else None
        continue
    if len(r) < len(hdr) or cur is None: continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ins[cur] += int(d.get("Instructions Executed") or 0); stl[cur] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError: pass
ti = sum(ins.values()); ts = sum(stl.values())
print(f"total {ti/cells:.2f} warp-instr/cell")
seen = set()
for name, a, b in regs:
    ks = [k for k in ins if k[0] == "block.cu" and a <= k[1] <= b]
    seen.update(ks)
    print(f"{name:12s} {sum(ins[k] for k in ks)/cells:5.2f}/cell  {sum(stl[k] for k in ks)/ts*100:5.1f}% stall")
by = collections.Counter(); bs = collections.Counter()
for k in ins:
    if k not in seen: by[k[0]] += ins[k]; bs[k[0]] += stl[k]
for f, v in by.most_common(): print(f"{'other:'+f:12s} {v/cells:5.2f}/cell  {bs[f]/ts*100:5.1f}% stall")
