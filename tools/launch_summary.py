"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
usage: python tools/launch_summary.py launches.csv [skip_first_n_launches]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ii = hdr.index("ID")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    n = r[ki].split("(")[0].replace("void ", "")[:60]
    agg[n][0] += 1; agg[n][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:60s} {c:5d} {v / 1e6:9.3f} ms {100 * v / tot:5.1f}%")
