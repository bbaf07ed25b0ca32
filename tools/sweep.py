"""Tuning sweep (not the benchmark): time fa_accumulate on a config for several
kernel variants and print per-phase device times.

usage: python tools/sweep.py cfg rows "BR=32,WARPS=2,EVICT=0;BR=16,WARPS=4" [tile]
each variant is a ';'-separated list of FA_* environment settings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    rows = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
    shapes = sys.argv[3].split(";") if len(sys.argv) > 3 else ["BR=32"]
    tiles = sys.argv[4] if len(sys.argv) > 4 else None
    t0 = time.time()
    cfg = inputs.make_config(name, rows, rows)
    print(f"{name} {cfg.rows}x{cfg.cols} gen {time.time() - t0:.1f}s", flush=True)
    tile = cfg.tile if tiles is None else tuple(int(v) for v in tiles.split("x"))
    st = torch.cuda.Stream()
    src = torch.from_numpy(cfg.dem if cfg.dem is not None else cfg.dirs).cuda()
    w = torch.from_numpy(cfg.w).cuda() if cfg.w is not None else None
    out = torch.empty((cfg.rows, cfg.cols), dtype=fa.TORCH_ACC[fa.ATYPES[cfg.atype]], device="cuda")
    kw = dict(dem=src) if cfg.dem is not None else dict(dirs=src)
    for shape in shapes:
        for kv in shape.split(","):
            k, v = kv.split("=")
            os.environ["FA_" + k] = v
        nstrips = int(os.environ.get("FA_STRIPS", "0"))  # STRIPS=G: the multi-GPU strip pipeline, G strips on one device

        def call(ctx):
            if nstrips > 0:
                ctx.accumulate_strips(nstrips, w=w, atype=cfg.atype, out=out, **kw)
            else:
                ctx.accumulate(w=w, atype=cfg.atype, out=out, **kw)

        with fa.Context(0, stream=st, tile=tile) as ctx:
            for _ in range(2):
                call(ctx)
            res = []
            for _ in range(4):
                t0 = time.perf_counter()
                call(ctx)
                st.synchronize()
                r = ctx.stats()
                r["wall_ms"] = (time.perf_counter() - t0) * 1e3
                res.append(r)
        p = {k: float(np.median([r[k] for r in res]))
             for k in ("ms_pass1", "ms_graph", "ms_pass2", "ms_total", "ms_d8", "ms_block", "wall_ms")}
        r = res[-1]
        print(f"{shape}: total {p['ms_total']:.2f} ms  pass1 {p['ms_pass1']:.2f}  graph {p['ms_graph']:.2f}  "
              f"pass2 {p['ms_pass2']:.2f} [d8 {p['ms_d8']:.2f} block {p['ms_block']:.2f} wall {p['wall_ms']:.2f}]  -> {cfg.cells / p['ms_total'] / 1e6:.1f} Gcells/s  "
              f"nodes {r['graph_nodes']} launches {r['launches']} peel {r['peel_rounds']} "
              f"contract {r['contract_levels']} jumps {r['jump_rounds']}", flush=True)


if __name__ == "__main__":
    main()
