"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of libfa on small rasters, each
result checked against the CPU oracle.  usage: python tools/sanitize_cases.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import oracle  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402
from paper_1608_04431_b200.dist import strip_bounds  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(d):
    e = oracle.accumulate(d).astype(np.uint32)
    e[d == 255] = np.uint32(0xFFFFFFFF)
    return e


z = inputs.filled_dem(3, 200, 171, coast_frac=0.1)
d = oracle.d8(z)
dr = inputs.random_dirs(4, 150, 133, p_nodata=0.1, p_noflow=0.02)
w = inputs.weights_f32(4, dr.shape)
ok = True
for opts in ({}, {"retention": "evict"}, {"d8": "fused"}, {"block_rows": 16}, {"values": "smem"},
             {"values": "smem", "retention": "evict"}):
    with fa.Context(0, tile=(64, 64)) as ctx:
        for k, v in opts.items():
            ctx.set_option(k, v)
        ok &= bool((ctx.flowdirs(cu(z)).cpu().numpy() == d).all())
        ok &= bool((ctx.accumulate(dem=cu(z), atype="u32").cpu().numpy() == u32(d)).all())
        ok &= bool((ctx.accumulate_strips(3, dem=cu(z), atype="u32").cpu().numpy() == u32(d)).all())
        got = ctx.accumulate(dirs=cu(dr), w=cu(w), atype="f64").cpu().numpy()
        exp = oracle.accumulate(dr, w, kind="f64")
        m = dr != 255
        ok &= bool((np.abs(got[m] - exp[m]) <= 1e-9 * exp[m]).all())
        links, at, xo, acc = ctx.perimeter_records(dirs=cu(dr), atype="u64")
        ok &= bool((links.cpu().numpy() == oracle.links(dr, 64, 64)).all())
    print("options", opts, "ok" if ok else "FAIL", flush=True)
with fa.Context(0, tile=(64, 64)) as ctx:
    ok &= bool((ctx.accumulate_streamed(dem=z, atype="u32", strip_rows=64) == u32(d)).all())
    al = np.random.default_rng(1).random(dr.shape).astype(np.float32)
    got = ctx.accumulate_absorb(cu(al), dirs=cu(dr), w=cu(w)).cpu().numpy()
    exp = oracle.accumulate_alpha(dr, al, w)
    ok &= bool((np.abs(got[m] - exp[m]) <= 1e-9 * np.abs(exp[m]) + 1e-300).all())
    zf = ctx.fill(cu(inputs.terrain(5, 128, 96))).cpu().numpy()
    ok &= bool(np.array_equal(zf.view(np.uint32), oracle.fill(inputs.terrain(5, 128, 96)).view(np.uint32)))
print("streamed / absorb / fill", "ok" if ok else "FAIL", flush=True)
N = 3
bounds = [strip_bounds(200, 64, q, N) for q in range(N)]
ctxs = [fa.Context(0, stream=torch.cuda.Stream(), tile=(64, 64)) for _ in range(N)]
out = fa.accumulate_dist_loopback(ctxs, 200, [b[0] for b in bounds],
                                  dem=[cu(z[r0:r0 + n]) for r0, n in bounds], atype="u32")
torch.cuda.synchronize()
ok &= bool((np.concatenate([o.cpu().numpy() for o in out]) == u32(d)).all())
for c in ctxs:
    c.close()
print("loopback", "ok" if ok else "FAIL", flush=True)
print("ALL OK" if ok else "SOME FAILED")
sys.exit(0 if ok else 1)
