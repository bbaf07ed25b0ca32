"""GPU parity of the multi-rank path itself (H7): fa_accumulate_dist's per-rank
code run for N ranks at once through the loopback transport (ranks = host
threads, one context and stream each, exchange by device copies and events).

Every rank gets its OWN copy of its strip (no pointer into the whole raster),
so the halo rows it needs can only come from the exchange (C1), the records
of the other strips only from the all-gather (C2), and the slot ranges of the
other ranks only from the argument agreement (C0).  Results are compared
with the CPU oracle on the whole raster: bit-exact for integers, D13 (1e-9
relative) for f64.  P:L215 (global graph from the tiles' edges).
"""
import numpy as np
import pytest
import torch

import inputs
import oracle
from paper_1608_04431_b200.dist import strip_bounds

pytestmark = pytest.mark.gpu

U32M = np.uint32(0xFFFFFFFF)


def _split(a, bounds):
    if a is None:
        return None
    return [torch.from_numpy(np.ascontiguousarray(a[r0:r0 + n])).cuda() for r0, n in bounds]


def _run(fa_lib, N, tile, dem=None, dirs=None, w=None, alpha=None, atype="u32", bounds=None, options=None):
    src = dem if dem is not None else dirs
    H = src.shape[0]
    if bounds is None:
        bounds = [strip_bounds(H, tile[0], q, N) for q in range(N)]
    ctxs = [fa_lib.Context(0, stream=torch.cuda.Stream(), tile=tile) for _ in range(N)]
    try:
        for c in ctxs:
            for k, v in (options or {}).items():
                c.set_option(k, v)
        out = fa_lib.accumulate_dist_loopback(ctxs, H, [b[0] for b in bounds], dem=_split(dem, bounds),
                                              dirs=_split(dirs, bounds), w=_split(w, bounds),
                                              alpha=_split(alpha, bounds), atype=atype)
        torch.cuda.synchronize()
        stats = [c.stats() for c in ctxs]
        return np.concatenate([o.cpu().numpy() for o in out]), stats
    finally:
        for c in ctxs:
            c.close()


def _exp_u32(d, w=None):
    e = oracle.accumulate(d, w).astype(np.uint32)
    e[d == 255] = U32M
    return e


def _check_f64(got, d, exp):
    data = d != 255
    assert np.isnan(got[~data]).all()
    rel = np.abs(got[data] - exp[data]) / np.abs(exp[data])
    assert rel.max() <= 1e-9, rel.max()


@pytest.mark.parametrize("N", [2, 3, 8])
def test_loopback_dem_u32_cfg1_recipe(fa_lib, N):
    cfg = inputs.make_config("cfg1", 1024, 1024)
    d = oracle.d8(cfg.dem)
    got, st = _run(fa_lib, N, (128, 128), dem=cfg.dem)
    assert (got == _exp_u32(d)).all()
    assert all(s["bytes_exchanged"] > 0 for s in st)


@pytest.mark.parametrize("records", ["strips", "tiles"])
@pytest.mark.parametrize("N", [2, 5])
def test_loopback_dirs_ragged_tiles_and_strips(fa_lib, N, records):
    # 300 rows in 64-row tiles: the last tile row (and strip) is 44 rows; 257 cols in 50-col tiles
    # (5 ranks: equal 64-row strips + a 44-row last one -> strip-level records; 2 ranks: 128 + 172
    # rows, unequal -> the tiles are exchanged)
    d = inputs.random_dirs(11, 300, 257, p_nodata=0.12, p_noflow=0.02)
    w = inputs.weights_u32(11, d.shape, 0, 50)
    got, st = _run(fa_lib, N, (64, 50), dirs=d, w=w, atype="u64", options={"dist_records": records})
    assert (got == oracle.accumulate(d, w)).all()


def test_loopback_dem_one_row_last_strip(fa_lib):
    # 129 rows in 64-row tiles on 3 ranks: the last rank owns ONE row, so its
    # neighbour receives a single halo row and row H+1 is off the raster
    z = inputs.filled_dem(21, 129, 200, coast_frac=0.1)
    d = oracle.d8(z)
    got, _ = _run(fa_lib, 3, (64, 64), dem=z)
    assert (got == _exp_u32(d)).all()


@pytest.mark.parametrize("records", ["strips", "tiles"])
def test_loopback_transposed_serpentine_crosses_every_strip(fa_lib, records):
    d = inputs.serpentine(512, 384, transposed=True)
    got, _ = _run(fa_lib, 8, (64, 64), dirs=d, options={"dist_records": records})
    assert (got == oracle.accumulate(d).astype(np.uint32)).all()
    assert got.max() == 512 * 384


@pytest.mark.parametrize("records", ["strips", "tiles"])
@pytest.mark.parametrize("N", [2, 4, 8])
def test_loopback_cfg3_recipe_f64(fa_lib, N, records):
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    got, st = _run(fa_lib, N, (128, 128), dem=cfg.dem, w=cfg.w, atype="f64", options={"dist_records": records})
    _check_f64(got, d, oracle.accumulate(d, cfg.w, kind="f64"))
    # strip-level records: the producer graph holds each strip's perimeter (N
    # tiles of 1024/N x 1024), else the perimeters of the 8 x 8 tiles
    slots = N * (2 * (1024 // N + 1024) - 4) if records == "strips" else 64 * (4 * 128 - 4)
    assert all(s["tile_nodes"] == slots for s in st)


def test_loopback_f64_off_grid_weights_deep_chains(fa_lib):
    # weights off the 2^-23 grid over six decades (partial sums inexact), on the
    # transposed serpentine (one 196K-cell chain through all strips): D13
    d = inputs.serpentine(512, 384, transposed=True)
    rng = np.random.default_rng(3)
    w = (rng.random(d.shape) * 10.0 ** (6 * rng.random(d.shape) - 3)).astype(np.float32)
    got, _ = _run(fa_lib, 4, (64, 64), dirs=d, w=w, atype="f64")
    _check_f64(got, d, oracle.accumulate(d, w, kind="f64"))


@pytest.mark.parametrize("opts", [{"retention": "evict"}, {"d8": "fused"}, {"block_rows": 16}])
def test_loopback_options(fa_lib, opts):
    z = inputs.filled_dem(23, 384, 320, coast_frac=0.1)
    d = oracle.d8(z)
    got, _ = _run(fa_lib, 3, (128, 64), dem=z, options=opts)
    assert (got == _exp_u32(d)).all()


def test_loopback_absorption(fa_lib):
    d = inputs.random_dirs(31, 256, 200, p_nodata=0.1, p_noflow=0.02)
    rng = np.random.default_rng(31)
    al = rng.random(d.shape).astype(np.float32)
    w = inputs.weights_f32(31, d.shape)
    got, _ = _run(fa_lib, 4, (64, 64), dirs=d, w=w, alpha=al)
    _check_f64(got, d, oracle.accumulate_alpha(d, al, w))


def test_loopback_cycle_across_strips_all_ranks_fail(fa_lib):
    d = np.zeros((128, 64), np.uint8)
    d[63, 10], d[64, 10] = 5, 1  # a 2-cycle across the strip boundary (row 63 | 64)
    with pytest.raises(fa_lib.FaError) as e:
        _run(fa_lib, 2, (64, 64), dirs=d)
    assert e.value.status == fa_lib.FA_E_CYCLE


def test_loopback_u32_overflow_summed_over_ranks(fa_lib):
    # each rank's weights sum to 2^31 (fine alone); the whole raster reaches 2^32
    d = np.zeros((64, 64), np.uint8)
    w = np.full((64, 64), 2 ** 20, np.uint32)
    with pytest.raises(fa_lib.FaError) as e:
        _run(fa_lib, 2, (32, 64), dirs=d, w=w, atype="u32")
    assert e.value.status == fa_lib.FA_E_OVERFLOW
    got, _ = _run(fa_lib, 2, (32, 64), dirs=d, w=w, atype="u64")  # u64 holds it
    assert (got == 2 ** 20).all()


def test_loopback_bad_partition_rejected_by_every_rank(fa_lib):
    d = inputs.random_dirs(5, 128, 64)
    for bounds in ([(0, 64), (32, 96)], [(0, 32), (32, 96)]):  # overlapping / not whole tile rows
        with pytest.raises(fa_lib.FaError) as e:
            _run(fa_lib, 2, (64, 64), dirs=d, bounds=bounds)
        assert e.value.status == fa_lib.FA_E_STATE
        assert str(e.value).count("rank") >= 2  # every rank reported


@pytest.mark.slow
def test_loopback_cfg4_recipe_u64_8_ranks(fa_lib):
    # the cfg4 recipe (30 % NoData ocean, w = 1, u64) at 16384^2 on 8 ranks of 2048 rows
    cfg = inputs.make_config("cfg4", 16384, 16384)
    d = oracle.d8(cfg.dem)
    got, st = _run(fa_lib, 8, (2048, 2048), dem=cfg.dem, atype="u64")
    exp = oracle.accumulate(d)
    exp[d == 255] = np.uint64(0xFFFFFFFFFFFFFFFF)
    assert (got == exp).all()


@pytest.mark.slow
def test_loopback_cfg4_recipe_32768_streamed_certificate(fa_lib):
    """The cfg4 recipe (30 % NoData ocean, w = 1, u64, 4096^2 tiles) at 1/16
    of cfg4's cells (32768^2) on 8 ranks, one tile row each -- the parity
    plan of the 8-GPU run, where the host cannot hold the whole-raster
    oracle: the streamed donor-identity certificate (P8) checks every cell
    strip by strip (the identity with acyclicity is a complete certificate,
    SURVEY §8(c)), with the oracle's own D8 codes."""
    cfg = inputs.make_config("cfg4", 32768, 32768)
    H, W = cfg.rows, cfg.cols
    N, tile = 8, (4096, 4096)
    bounds = [strip_bounds(H, tile[0], q, N) for q in range(N)]
    ctxs = [fa_lib.Context(0, stream=torch.cuda.Stream(), tile=tile) for _ in range(N)]
    try:
        out = fa_lib.accumulate_dist_loopback(ctxs, H, [b[0] for b in bounds], dem=_split(cfg.dem, bounds),
                                              atype="u64")
        torch.cuda.synchronize()
    finally:
        for c in ctxs:
            c.close()

    def acc_rows(a, b):
        parts = []
        for (r0, n), o in zip(bounds, out):
            lo, hi = max(a, r0), min(b, r0 + n)
            if lo < hi:
                parts.append(o[lo - r0:hi - r0].cpu().numpy())
        return np.concatenate(parts)

    def dirs_rows(a, b):
        lo, hi = max(0, a - 1), min(H, b + 1)
        return oracle.d8(cfg.dem[lo:hi])[a - lo:a - lo + (b - a)]

    assert oracle.certify_strips(dirs_rows, acc_rows, H, W, 4096) == 0
