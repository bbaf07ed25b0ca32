"""Time the multi-rank path through the loopback transport on one GPU:
python tools/loopback_time.py [rows] [ranks] -- per record granularity,
the call's wall time and rank 0's phase times, graph nodes and exchanged
bytes (the ranks share one GPU here, so only relative numbers mean much)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402
from paper_1608_04431_b200.dist import strip_bounds  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = inputs.make_config("cfg3", rows, rows)
tile = (min(4096, rows // N), 4096)
bounds = [strip_bounds(rows, tile[0], q, N) for q in range(N)]
dem = [torch.from_numpy(np.ascontiguousarray(cfg.dem[r0:r0 + n])).cuda() for r0, n in bounds]
w = [torch.from_numpy(np.ascontiguousarray(cfg.w[r0:r0 + n])).cuda() for r0, n in bounds]
for rec in ("strips", "tiles"):
    ctxs = [fa.Context(0, stream=torch.cuda.Stream(), tile=tile) for _ in range(N)]
    for c in ctxs:
        c.set_option("dist_records", rec)
    out = None
    ts = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fa.accumulate_dist_loopback(ctxs, rows, [b[0] for b in bounds], dem=dem, w=w, atype="f64", out=out)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    s = ctxs[0].stats()
    print(f"{rec}: {np.median(ts[1:]):.2f} ms per call (8 ranks on one GPU); rank 0: pass1 {s['ms_pass1']:.2f} "
          f"graph {s['ms_graph']:.2f} pass2 {s['ms_pass2']:.2f} exchange {s['ms_exchange']:.3f} ms, "
          f"tile slots {s['tile_nodes']}, bytes exchanged {s['bytes_exchanged']}", flush=True)
    for c in ctxs:
        c.close()
