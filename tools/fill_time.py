"""Time fa_fill on the cfg1 / cfg3 terrains (measurement tool, not the benchmark)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402

for name, n, seed, frac in (("cfg1", 8192, 2, 0.05), ("cfg3", 32768, 4, 0.10))[: int(sys.argv[1]) if len(sys.argv) > 1 else 2]:
    z = inputs.terrain(seed, n, n)
    inputs.coast(z, seed, frac)
    dz = torch.from_numpy(z).cuda()
    out = torch.empty_like(dz)
    with fa.Context(0) as ctx:
        ctx.fill(dz, out=out)
        ts = []
        for _ in range(2):
            ctx.fill(dz, out=out)
            ts.append(ctx.stats())
    s = ts[-1]
    print(f"fill {name} {n}x{n}: {s['ms_total']:.1f} ms, {s['launches']} launches, {z.size / s['ms_total'] / 1e6:.2f} Gcells/s")
