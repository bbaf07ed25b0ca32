"""Four warm fa_accumulate calls on a config (for ncu launch lists): python tools/cfg_once.py cfg2"""
import sys
sys.path.insert(0, ".")
import torch, inputs
from paper_1608_04431_b200 import fa
name = sys.argv[1]
cfg = inputs.make_config(name, None, None)
kw = {"atype": cfg.atype}
if cfg.dem is not None: kw["dem"] = torch.from_numpy(cfg.dem).cuda()
else: kw["dirs"] = torch.from_numpy(cfg.dirs).cuda()
if cfg.w is not None: kw["w"] = torch.from_numpy(cfg.w).cuda()
with fa.Context(0, tile=cfg.tile) as ctx:
    for i in range(4):
        ctx.accumulate(**kw)
        s = ctx.stats(); print(i, {k: round(v, 3) if isinstance(v, float) else v for k, v in s.items()}, flush=True)
