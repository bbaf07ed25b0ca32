"""cfg4's per-rank share on ONE GPU: python tools/cfg4_strip.py [rows] [cols] [steps]

BASELINE.json config 4 (131072^2, w = 1 -> u64, 30 % NoData) runs as 8 row
strips of 16384 x 131072 cells, one per B200.  This pool has one GPU per
call, so the 8-rank number cannot be measured here; this tool times what ONE
rank's kernels do at that size: a 16384 x 131072 raster of the cfg4 recipe
(seed 5, G2 + G3 30 % + G4; its own fractal, not a crop of the 131072^2 one,
whose fill is global) through fa_accumulate, device-resident, CUDA events
around `steps` calls.  No halo exchange and no record all-gather are in it
(DESIGN.md §8 gives their sizes); parity at this width is
tests/test_gpu_fullsize.py::test_cfg4_recipe_full_width_certified.
Prints one JSON line with Gcells/s and the HBM fractions (k_pass1<u64> at
9 B/cell: dirs 1 + A 8; whole path at 12 B/cell: z 4 + A 8)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5

try:
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    peak_src = "measured"
except Exception:
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"

t0 = time.time()
cfg = inputs.make_config("cfg4", rows, cols)
gen_s = time.time() - t0
cells = rows * cols
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    dz = torch.from_numpy(cfg.dem).cuda()
    acc = torch.empty((rows, cols), dtype=torch.uint64, device="cuda")
stream.synchronize()
with fa.Context(0, stream=stream, tile=cfg.tile) as ctx:
    for _ in range(3):
        ctx.accumulate(dem=dz, atype="u64", out=acc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = []
    e0.record(stream)
    for _ in range(steps):
        ctx.accumulate(dem=dz, atype="u64", out=acc)
        st.append(ctx.stats())
    e1.record(stream)
    e1.synchronize()
ms = e0.elapsed_time(e1) / steps


def med(k):
    return float(np.median([s[k] for s in st]))


blk, d8 = med("ms_block"), med("ms_d8")
print(json.dumps({
    "workload": f"cfg4 recipe, one rank's strip of 8: {rows}x{cols} f32 DEM seed 5, 30% NoData, filled, "
                f"w = 1 -> u64, {cfg.tile[0]}x{cfg.tile[1]} tiles",
    "value": cells / (ms * 1e-3) / 1e9, "unit": "Gcells/s", "ms_per_step": ms, "steps": steps, "n_gpus": 1,
    "nodata_frac": round(float(cfg.meta["nodata_frac"]), 4),
    "roofline": {"bound": "hbm", "kernel": "k_pass1", "bytes_per_cell": 9,
                 "achieved": cells * 9 / (blk * 1e-3) / 1e9, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                 "frac": cells * 9 / (blk * 1e-3) / 1e9 / peak,
                 "whole_path": {"bytes_per_cell": 12, "achieved": cells * 12 / (ms * 1e-3) / 1e9,
                                "frac": cells * 12 / (ms * 1e-3) / 1e9 / peak}},
    "kernels_ms": {"k_d8": d8, "k_pass1": blk},
    "phases_ms": {"pass1": med("ms_pass1"), "graph": med("ms_graph"), "pass2": med("ms_pass2")},
    "graph_nodes": int(st[-1]["graph_nodes"]), "launches": int(st[-1]["launches"]),
    "input_gen_s": round(gen_s, 1)}), flush=True)
