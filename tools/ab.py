"""A/B timing of context options on the bench workloads (device-resident
inputs, library CUDA events): python tools/ab.py [rows]
Prints, per workload and option set, the median ms_total and ms_block."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
VARIANTS = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{"values": "l2"}, {"values": "smem"}]
NAMES = sys.argv[3].split(",") if len(sys.argv) > 3 else ["cfg1", "cfg2", "cfg3"]


def run(ctx, kw, n=5, strips=0):
    ts = []
    for i in range(n + 2):
        if strips:
            ctx.accumulate_strips(strips, **kw)
        else:
            ctx.accumulate(**kw)
        s = ctx.stats()
        if i >= 2:
            ts.append((s["ms_total"], s["ms_block"], s["ms_d8"], s["ms_graph"], s["ms_pass2"]))
    return np.median(np.array(ts), axis=0)


out = {}
for name in NAMES:
    r = rows if name != "cfg2" else min(rows, 4096)
    cfg = inputs.make_config(name, r, r)
    kw = {"atype": cfg.atype}
    if cfg.dem is not None:
        kw["dem"] = torch.from_numpy(cfg.dem).cuda()
    else:
        kw["dirs"] = torch.from_numpy(cfg.dirs).cuda()
    if cfg.w is not None:
        kw["w"] = torch.from_numpy(cfg.w).cuda()
    for v in VARIANTS:
        with fa.Context(0, tile=cfg.tile) as ctx:
            for k, x in v.items():
                if k != "strips":
                    ctx.set_option(k, x)
            t = run(ctx, kw, strips=int(v.get("strips", 0)))
        key = f"{name}:{','.join(f'{k}={x}' for k, x in v.items())}"
        out[key] = [round(float(x), 3) for x in t]
        print(key, "total %.3f block %.3f d8 %.3f graph %.3f pass2 %.3f" % tuple(t), flush=True)
print(json.dumps(out))
