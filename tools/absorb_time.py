"""Time fa_accumulate_absorb on a config (tuning/measurement tool, not the benchmark).
usage: python tools/absorb_time.py cfg3 [rows]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = inputs.make_config(name, rows, rows)
rng = np.random.default_rng(5)
al = torch.from_numpy((0.9 + 0.1 * rng.random((cfg.rows, cfg.cols))).astype(np.float32)).cuda()
dz = torch.from_numpy(cfg.dem).cuda()
dw = torch.from_numpy(cfg.w).cuda() if cfg.w is not None else None
out = torch.empty((cfg.rows, cfg.cols), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
with fa.Context(0, stream=st) as ctx:
    for _ in range(2):
        ctx.accumulate_absorb(al, dem=dz, w=dw, out=out)
    ts = []
    for _ in range(4):
        ctx.accumulate_absorb(al, dem=dz, w=dw, out=out)
        ts.append(ctx.stats())
s = {k: float(np.median([t[k] for t in ts])) for k in ("ms_total", "ms_pass1", "ms_graph", "ms_pass2", "ms_block")}
print(f"absorb {name} {cfg.rows}x{cfg.cols}: total {s['ms_total']:.2f} ms (pass1 {s['ms_pass1']:.2f} "
      f"[block {s['ms_block']:.2f}] graph {s['ms_graph']:.2f} finalize {s['ms_pass2']:.2f}) -> "
      f"{cfg.rows * cfg.cols / s['ms_total'] / 1e6:.1f} Gcells/s")
