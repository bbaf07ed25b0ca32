"""fp64 accumulation under inexact sums (D13: per data cell |A_gpu - A_orc| <=
1e-9 |A_orc|), on the plain single-device path and the strip pipeline.

The cfg3 recipe's weights lie on a 2^-23 grid, so its sums are exact in any
order (test_gpu_parity.py); these cases use weights off that grid and over a
wide dynamic range, and a 16.7M-cell chain, so the GPU's summation order
(block-local sums, then the offsets) and the oracle's (chain order) round
differently.  The largest relative error seen is printed (pytest -s).
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rel(got, d, exp):
    data = d != 255
    assert np.isnan(got[~data]).all()
    return float((np.abs(got[data] - exp[data]) / np.abs(exp[data])).max())


def _wide(seed, shape):
    rng = np.random.default_rng(seed)
    return (rng.random(shape) * 10.0 ** (6 * rng.random(shape) - 3)).astype(np.float32)  # 1e-3 .. 1e3, off grid


@pytest.mark.parametrize("tile,G", [((0, 0), 1), ((256, 256), 1), ((256, 256), 3)])
def test_f64_wide_range_weights_dem(fa_lib, tile, G):
    cfg = inputs.make_config("cfg1", 1024, 1024)
    d = oracle.d8(cfg.dem)
    w = _wide(5, d.shape)
    with fa_lib.Context(0, tile=tile) as ctx:
        if G == 1:
            got = ctx.accumulate(dem=_cuda(cfg.dem), w=_cuda(w), atype="f64").cpu().numpy()
        else:
            got = ctx.accumulate_strips(G, dem=_cuda(cfg.dem), w=_cuda(w), atype="f64").cpu().numpy()
    r = _rel(got, d, oracle.accumulate(d, w, kind="f64"))
    print(f"wide-range weights tile={tile} G={G}: max rel err {r:.3e}")
    assert r <= 1e-9


def test_f64_uniform_off_grid_weights_random_dirs(fa_lib):
    d = inputs.random_dirs(8, 777, 555, p_nodata=0.1, p_noflow=0.01)
    w = np.random.default_rng(8).uniform(0.5, 1.5, d.shape).astype(np.float32)
    with fa_lib.Context(0, tile=(128, 256)) as ctx:
        got = ctx.accumulate(dirs=_cuda(d), w=_cuda(w), atype="f64").cpu().numpy()
    r = _rel(got, d, oracle.accumulate(d, w, kind="f64"))
    print(f"U(0.5,1.5) off-grid weights: max rel err {r:.3e}")
    assert r <= 1e-9


@pytest.mark.slow
def test_f64_serpentine_4096_deep_chain(fa_lib):
    """cfg2's serpentine (one chain of 16,777,216 cells) with off-grid f64
    weights: the longest possible fp64 chain at this size (SURVEY P11 bound
    ~n u = 1.9e-9 worst case; random rounding gives ~sqrt(n) u)."""
    d = inputs.serpentine(4096, 4096)
    w = np.random.default_rng(2).uniform(0.5, 1.5, d.shape).astype(np.float32)
    with fa_lib.Context(0) as ctx:
        got = ctx.accumulate(dirs=_cuda(d), w=_cuda(w), atype="f64").cpu().numpy()
    r = _rel(got, d, oracle.accumulate(d, w, kind="f64"))
    print(f"4096^2 serpentine, U(0.5,1.5) weights: max rel err {r:.3e}")
    assert r <= 1e-9
