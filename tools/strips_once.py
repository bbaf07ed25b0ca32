"""One warm fa_accumulate_strips call on cfg3 (for an ncu launch list of the
strip pipeline): python tools/strips_once.py [nstrips] [rows]"""
import sys

import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
cfg = inputs.make_config("cfg3", rows, rows)
z = torch.from_numpy(cfg.dem).cuda()
w = torch.from_numpy(cfg.w).cuda()
out = torch.empty(z.shape, dtype=torch.float64, device="cuda")
with fa.Context(0, tile=cfg.tile) as ctx:
    for i in range(4):
        torch.cuda.nvtx.range_push(f"call{i}")
        ctx.accumulate_strips(ns, dem=z, w=w, atype="f64", out=out)
        torch.cuda.nvtx.range_pop()
        s = ctx.stats()
        print(i, {k: round(v, 3) if isinstance(v, float) else v for k, v in s.items()}, flush=True)
