"""GPU parity of absorption (Eq. 1 with a per-cell alpha,
P:L49-57) against the absorption oracle: fp64 within 1e-9 relative (D13),
on random D8 rasters (ragged blocks, NoData, NoFlow), the DEM recipes, the
alpha = 1 and alpha = 0 special cases, the transposed serpentine (deep
block-exit chains), host buffers and the alpha validation error."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check(got, d, exp, rtol=1e-9):
    data = d != 255
    assert np.isnan(got[~data]).all()
    g, e = got[data], exp[data]
    assert (np.abs(g - e) <= rtol * np.abs(e)).all(), np.max(np.abs(g - e) / np.maximum(np.abs(e), 1e-300))


@pytest.mark.parametrize("seed,H,W", [(1, 300, 257), (2, 129, 333), (3, 64, 64), (4, 513, 200), (5, 1, 100)])
def test_absorb_random_dirs(fa_lib, seed, H, W):
    rng = np.random.default_rng(seed)
    d = inputs.random_dirs(seed, H, W, p_nodata=0.12, p_noflow=0.02)
    al = rng.random((H, W)).astype(np.float32)
    al[rng.random((H, W)) < 0.3] = 1.0
    w = inputs.weights_f32(seed, (H, W))
    with fa_lib.Context(0) as ctx:
        got = ctx.accumulate_absorb(_cuda(al), dirs=_cuda(d), w=_cuda(w)).cpu().numpy()
    _check(got, d, oracle.accumulate_alpha(d, al, w))


def test_absorb_dem_recipe_and_special_cases(fa_lib):
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    rng = np.random.default_rng(9)
    al = (0.9 + 0.1 * rng.random(d.shape)).astype(np.float32)
    with fa_lib.Context(0) as ctx:
        got = ctx.accumulate_absorb(_cuda(al), dem=_cuda(cfg.dem), w=_cuda(cfg.w)).cpu().numpy()
        one = ctx.accumulate_absorb(_cuda(np.ones(d.shape, np.float32)), dem=_cuda(cfg.dem),
                                    w=_cuda(cfg.w)).cpu().numpy()
        zero = ctx.accumulate_absorb(_cuda(np.zeros(d.shape, np.float32)), dirs=_cuda(d)).cpu().numpy()
    _check(got, d, oracle.accumulate_alpha(d, al, cfg.w))
    data = d != 255
    # alpha = 1 is plain accumulation: exact on the grid weights (D13)
    ex = oracle.accumulate(d, cfg.w, kind="fix23")
    assert (one[data] == ex[data].astype(np.float64) * 2.0 ** -23).all()
    assert (zero[data] == 1.0).all() and np.isnan(zero[~data]).all()


def test_absorb_transposed_serpentine_host_buffers(fa_lib):
    d = inputs.serpentine(256, 192, transposed=True)
    al = np.full(d.shape, 0.999, np.float32)
    with fa_lib.Context(0) as ctx:
        got = ctx.accumulate_absorb(al, dirs=d)  # numpy in / out
    _check(got, d, oracle.accumulate_alpha(d, al))


def test_absorb_rejects_bad_alpha(fa_lib):
    d = inputs.random_dirs(11, 64, 64, p_nodata=0.1)
    al = np.full(d.shape, 0.5, np.float32)
    ys, xs = np.nonzero(d != 255)
    al[ys[0], xs[0]] = 1.5
    with fa_lib.Context(0) as ctx:
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate_absorb(_cuda(al), dirs=_cuda(d))
        assert e.value.status == fa_lib.FA_E_ARG
        al[ys[0], xs[0]] = 0.5
        al[d == 255] = np.nan  # ignored at NoData cells
        got = ctx.accumulate_absorb(_cuda(al), dirs=_cuda(d)).cpu().numpy()
    _check(got, d, oracle.accumulate_alpha(d, al))


@pytest.mark.parametrize("cap", ["1", "4", "128"])
def test_absorb_weighted_contraction(fa_lib, cap):
    """Deep block-exit chains: the serpentine's river crosses every block row
    (~32K chained nodes at 1024^2), so the weighted solver contracts chains
    with affine (acc, mul) pointer jumping; small walk caps force contraction
    on a random raster's forest too (context option FA_OPT_WALK_CAP)."""
    rng = np.random.default_rng(int(cap))
    d = inputs.serpentine(1024, 1024)
    al = (0.999 + 0.001 * rng.random(d.shape)).astype(np.float32)
    r = inputs.random_dirs(17, 300, 257, p_nodata=0.1, p_noflow=0.02)
    ar = rng.random(r.shape).astype(np.float32)
    w = inputs.weights_f32(17, r.shape)
    with fa_lib.Context(0) as ctx:
        ctx.set_option("walk_cap", int(cap))
        assert ctx.get_option("walk_cap") == int(cap)
        got = ctx.accumulate_absorb(_cuda(al), dirs=_cuda(d)).cpu().numpy()
        assert ctx.stats()["contract_levels"] > 0  # the weighted chain contraction ran
        gr = ctx.accumulate_absorb(_cuda(ar), dirs=_cuda(r), w=_cuda(w)).cpu().numpy()
    _check(got, d, oracle.accumulate_alpha(d, al))
    _check(gr, r, oracle.accumulate_alpha(r, ar, w))


@pytest.mark.parametrize("seed,H,W,tile,G", [(1, 300, 257, (64, 64), 2), (2, 300, 257, (64, 96), 5),
                                             (3, 129, 333, (32, 64), 4), (4, 513, 200, (96, 64), 3)])
def test_absorb_strips_random_dirs(fa_lib, seed, H, W, tile, G):
    """The multi-GPU strip pipeline with weighted tile links: tile records
    carry each slot's alpha path factor, G2 and the offsets are weighted."""
    rng = np.random.default_rng(seed)
    d = inputs.random_dirs(seed, H, W, p_nodata=0.12, p_noflow=0.02)
    al = rng.random((H, W)).astype(np.float32)
    al[rng.random((H, W)) < 0.3] = 1.0
    w = inputs.weights_f32(seed, (H, W))
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate_absorb(_cuda(al), dirs=_cuda(d), w=_cuda(w), nstrips=G).cpu().numpy()
    _check(got, d, oracle.accumulate_alpha(d, al, w))


def test_absorb_strips_dem_and_serpentine(fa_lib):
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    rng = np.random.default_rng(3)
    al = (0.9 + 0.1 * rng.random(d.shape)).astype(np.float32)
    s = inputs.serpentine(512, 384, transposed=True)
    als = (0.999 + 0.001 * rng.random(s.shape)).astype(np.float32)
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        got = ctx.accumulate_absorb(_cuda(al), dem=_cuda(cfg.dem), w=_cuda(cfg.w), nstrips=4).cpu().numpy()
    with fa_lib.Context(0, tile=(64, 64)) as ctx:
        gs = ctx.accumulate_absorb(_cuda(als), dirs=_cuda(s), nstrips=8).cpu().numpy()
    _check(got, d, oracle.accumulate_alpha(d, al, cfg.w))
    _check(gs, s, oracle.accumulate_alpha(s, als))


def test_absorb_dist_single_rank_nccl(fa_lib):
    """fa_accumulate_absorb_dist (NCCL, one rank): the records all-gather
    carries the alpha path factors; same result as the oracle."""
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    rng = np.random.default_rng(13)
    al = (0.9 + 0.1 * rng.random(d.shape)).astype(np.float32)
    nid = fa_lib.nccl_unique_id()
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        got = ctx.accumulate_absorb_dist(nid, 0, 1, 1024, 0, _cuda(al), dem=_cuda(cfg.dem),
                                         w=_cuda(cfg.w)).cpu().numpy()
        st = ctx.stats()
    _check(got, d, oracle.accumulate_alpha(d, al, cfg.w))
    assert st["bytes_exchanged"] > 0


@pytest.mark.parametrize("strip_rows", [64, 250, 0])
def test_absorb_streamed(fa_lib, strip_rows):
    """Out of core with absorption: alpha streamed with the strips (host buffers)."""
    rng = np.random.default_rng(strip_rows + 1)
    d = inputs.random_dirs(21, 513, 200, p_nodata=0.1, p_noflow=0.02)
    al = rng.random(d.shape).astype(np.float32)
    w = inputs.weights_f32(21, d.shape)
    with fa_lib.Context(0, tile=(64, 64)) as ctx:
        got = ctx.accumulate_absorb_streamed(al, dirs=d, w=w, strip_rows=strip_rows)
    _check(got, d, oracle.accumulate_alpha(d, al, w))
    cfg = inputs.make_config("cfg3", 512, 512)
    dd = oracle.d8(cfg.dem)
    a2 = (0.9 + 0.1 * rng.random(dd.shape)).astype(np.float32)
    with fa_lib.Context(0, tile=(128, 128)) as ctx:
        g2 = ctx.accumulate_absorb_streamed(a2, dem=cfg.dem, w=cfg.w, strip_rows=strip_rows)
    _check(g2, dd, oracle.accumulate_alpha(dd, a2, cfg.w))
