"""GPU parity at the benchmark's full size and launch configuration.

cfg3 (32768^2 f32 DEM, 10 % NoData, f32 weights -> f64, 4096^2 tiles) is the
workload bench.py times at N=1; it is checked element by element against the
oracle (f64 Kahn accumulation, relative error <= 1e-9, D13) and against the
oracle's exact fixed-point sum (P11), both through the single-device path
bench.py calls and through the row-strip path of the multi-GPU launch
(8 strips of 4096 rows, the N=8 configuration, on one device).  cfg4's recipe
(30 % NoData, w = 1, u64) is checked bit-exactly at a one-GPU size with the
N=8 strip layout.  The oracle needs ~4 minutes of one host core for cfg3.
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
