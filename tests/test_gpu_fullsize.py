"""GPU parity at the benchmark's full size and launch configuration.

cfg3 (32768^2 f32 DEM, 10 % NoData, f32 weights -> f64, 4096^2 tiles) is the
workload bench.py times at N=1; it is checked element by element against the
oracle (f64 Kahn accumulation, relative error <= 1e-9, D13) and against the
oracle's exact fixed-point sum (P11), both through the single-device path
bench.py calls and through the row-strip path of the multi-GPU launch
(8 strips of 4096 rows, the N=8 configuration, on one device).  cfg4's recipe
(30 % NoData, w = 1, u64) is checked bit-exactly at a one-GPU size with the
N=8 strip layout, and certified (P8) on one tile row at cfg4's full width
of 131072 columns.  The oracle needs ~4 minutes of one host core for cfg3.
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def cfg3_full():
    cfg = inputs.make_config("cfg3")
    d = oracle.d8(cfg.dem)
    exp = oracle.accumulate(d, cfg.w, kind="f64")
    ex = oracle.accumulate(d, cfg.w, kind="fix23")
    return cfg, d, exp, ex


def _check_f64(got, d, exp, ex):
    data = d != 255
    assert np.isnan(got[~data]).all()
    g, e = got[data], exp[data]
    rel = np.abs(g - e) / e
    assert rel.max() <= 1e-9, rel.max()
    exact = ex[data].astype(np.float64) * 2.0 ** -23
    assert (np.abs(g - exact) / exact).max() <= 1e-9
    # Σw ≈ 9.7e8 < 2^30: every fp64 partial sum of grid weights is exact (P11),
    # so the result is the exact sum bit for bit, in any summation order
    assert (g == exact).all()


def test_cfg3_full_single_device(fa_lib, cfg3_full):
    cfg, d, exp, ex = cfg3_full
    with fa_lib.Context(0, tile=cfg.tile) as ctx:
        dz, dw = _cuda(cfg.dem), _cuda(cfg.w)
        dirs = ctx.flowdirs(dz).cpu().numpy()
        assert (dirs == d).all()
        got = ctx.accumulate(dem=dz, w=dw, atype="f64").cpu().numpy()
    _check_f64(got, d, exp, ex)


def test_cfg3_full_eight_strips(fa_lib, cfg3_full):
    cfg, d, exp, ex = cfg3_full
    with fa_lib.Context(0, tile=cfg.tile) as ctx:
        got = ctx.accumulate_strips(8, dem=_cuda(cfg.dem), w=_cuda(cfg.w), atype="f64").cpu().numpy()
    _check_f64(got, d, exp, ex)


def test_cfg4_recipe_eight_strips_u64(fa_lib):
    cfg = inputs.make_config("cfg4", 16384, 16384)
    d = oracle.d8(cfg.dem)
    exp = oracle.accumulate(d)
    with fa_lib.Context(0, tile=(4096, 4096)) as ctx:
        got = ctx.accumulate_strips(8, dem=_cuda(cfg.dem), atype="u64").cpu().numpy()
        one = ctx.accumulate(dem=_cuda(cfg.dem), atype="u64").cpu().numpy()
    assert (got == exp).all()
    assert (one == exp).all()


def test_cfg4_recipe_full_width_certified(fa_lib):
    """One tile row of cfg4 at its full width (4096 x 131072 cells, 30 %
    NoData, w = 1, u64, 4096^2 tiles): the column indices, the 4096 block
    columns and the 32 tile columns a rank of the 8-GPU run works with.  The
    oracle's own D8 codes must match byte for byte and its donor-identity
    certificate (P8: identity + mass balance on an acyclic D8 field is a
    complete certificate) must hold on every cell."""
    H, W = 4096, 131072
    cfg = inputs.make_config("cfg4", H, W)
    d = oracle.d8(cfg.dem)
    with fa_lib.Context(0, tile=(4096, 4096)) as ctx:
        dz = _cuda(cfg.dem)
        assert (ctx.flowdirs(dz).cpu().numpy() == d).all()
        got = ctx.accumulate(dem=dz, atype="u64").cpu().numpy()
    assert oracle.certify(d, got) == 0


@pytest.mark.slow
def test_serpentine_beyond_2_31_cells(fa_lib):
    """49152^2 = 2.42e9 cells on one GPU (more than 2^31, as a cfg4 strip of
    8 ranks holds 2^31): every cell index, block id and slot crosses 32-bit
    signed ranges, and the river is ONE chain of 2.4e9 cells through ~75 M
    block exits (the graph's chain contraction at its deepest).  Closed
    form P6: A = W*y + (y even ? x : W-1-x) + 1, up to 2.42e9 (fits u32)."""
    n = 49152
    d = inputs.serpentine(n, n)
    with fa_lib.Context(0) as ctx:
        got = ctx.accumulate(dirs=torch.from_numpy(d).cuda(), atype="u32")
        torch.cuda.synchronize()
    del d
    x = np.arange(n, dtype=np.uint64)
    for y0 in range(0, n, 4096):
        rows = got[y0:y0 + 4096].cpu().numpy().astype(np.uint64)
        y = np.arange(y0, y0 + rows.shape[0], dtype=np.uint64)[:, None]
        exp = n * y + np.where(y % 2 == 0, x[None, :], n - 1 - x[None, :]) + 1
        assert (rows == exp).all(), y0
