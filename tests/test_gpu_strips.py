"""GPU parity of the multi-GPU data path (H4-H7).

`fa_accumulate_strips` runs the exact per-strip phases of fa_accumulate_dist
(pass 1 with halo rows, tile records, the producer graph over all tile
perimeter slots, injection, pass 2) for G strips on one device, exchanging the
records by device copies instead of NCCL.  `fa_accumulate_dist` itself is run
with one rank (NCCL, single-member communicator).
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("seed,H,W,tile,G", [(1, 300, 257, (64, 50), 2), (2, 300, 257, (64, 50), 5),
                                             (3, 129, 333, (32, 64), 4), (4, 513, 200, (100, 37), 3),
                                             (5, 64, 64, (1, 64), 7)])
def test_strips_random_dirs(fa_lib, seed, H, W, tile, G):
    d = inputs.random_dirs(seed, H, W, p_nodata=0.12, p_noflow=0.02)
    w = inputs.weights_u32(seed, (H, W), 0, 50)
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate_strips(G, dirs=_cuda(d), w=_cuda(w), atype="u64").cpu().numpy()
    assert (got == oracle.accumulate(d, w)).all()


def test_strips_transposed_serpentine_crosses_every_strip(fa_lib):
    """Columns snake top<->bottom: the river crosses every strip boundary 2W times."""
    d = inputs.serpentine(512, 384, transposed=True)
    with fa_lib.Context(0, tile=(64, 64)) as ctx:
        got = ctx.accumulate_strips(8, dirs=_cuda(d), atype="u32").cpu().numpy()
    exp = oracle.accumulate(d).astype(np.uint32)
    assert (got == exp).all()
    assert got.max() == 512 * 384


@pytest.mark.parametrize("G", [1, 2, 4])
def test_strips_dem_f64_cfg3_recipe(fa_lib, G):
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        got = ctx.accumulate_strips(G, dem=_cuda(cfg.dem), w=_cuda(cfg.w), atype="f64").cpu().numpy()
    exp = oracle.accumulate(d, cfg.w, kind="f64")
    data = d != 255
    assert np.isnan(got[~data]).all()
    assert (np.abs(got[data] - exp[data]) / exp[data]).max() <= 1e-9


def test_strips_dem_u32_cfg1_recipe(fa_lib):
    cfg = inputs.make_config("cfg1", 2048, 2048)
    d = oracle.d8(cfg.dem)
    with fa_lib.Context(0, tile=(512, 512)) as ctx:
        got = ctx.accumulate_strips(4, dem=_cuda(cfg.dem), atype="u32").cpu().numpy()
    exp = oracle.accumulate(d).astype(np.uint32)
    exp[d == 255] = np.uint32(0xFFFFFFFF)
    assert (got == exp).all()


def test_dist_single_rank_nccl(fa_lib):
    cfg = inputs.make_config("cfg1", 1024, 1024)
    d = oracle.d8(cfg.dem)
    nid = fa_lib.nccl_unique_id()
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        got = ctx.accumulate_dist(nid, 0, 1, 1024, 0, dem=_cuda(cfg.dem), atype="u64").cpu().numpy()
        st = ctx.stats()
    exp = oracle.accumulate(d)
    assert (got == exp).all()
    assert st["bytes_exchanged"] > 0
