"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bar: D8 codes and integer accumulations bit-exact;
f64 per data cell |A_gpu - A_orc| <= 1e-9 |A_orc|; NoData markers exact.
"""
import math

import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

ND = -9999.0
U32M = np.uint32(0xFFFFFFFF)
U64M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _oracle_acc(d, w=None, atype="u32"):
    if atype == "f64":
        return oracle.accumulate(d, w, kind="f64")
    A = oracle.accumulate(d, w)
    if atype == "u32":
        A = A.astype(np.uint32)
        A[d == 255] = U32M
    return A


def _check(got, d, exp, atype):
    if atype == "f64":
        data = d != 255
        assert np.isnan(got[~data]).all()
        rel = np.abs(got[data] - exp[data]) / np.abs(exp[data])
        assert rel.max(initial=0.0) <= 1e-9, rel.max()
        return float(rel.max(initial=0.0))
    bad = np.flatnonzero(got.ravel() != exp.ravel())
    assert bad.size == 0, (bad.size, bad[:10], got.ravel()[bad[:5]], exp.ravel()[bad[:5]])
    return 0.0


# ---------------------------------------------------------------- H1 D8
@pytest.mark.parametrize("H,W", [(1, 1), (1, 200), (200, 1), (63, 65), (300, 517), (512, 512)])
def test_d8_fractal(fa_lib, H, W):
    z = inputs.filled_dem(7, H, W, coast_frac=0.1 if W > 2 else 0.0)
    with fa_lib.Context(0) as ctx:
        got = ctx.flowdirs(_cuda(z), ND).cpu().numpy()
    assert (got == oracle.d8(z, ND)).all()


@pytest.mark.parametrize("seed,levels,pnd", [(1, 2, 0.0), (2, 3, 0.1), (3, 5, 0.3), (4, 8, 0.05)])
def test_d8_ties_and_nodata(fa_lib, seed, levels, pnd):
    z = inputs.quantized_dem(seed, 257, 190, levels=levels, p_nodata=pnd)
    z[::3] = (z[::3] * np.float32(math.sqrt(2.0))).astype(np.float32)
    z[z < -1000] = np.float32(ND)
    z[5, 5] = np.nan
    z[6, 9] = np.inf
    with fa_lib.Context(0) as ctx:
        got = ctx.flowdirs(_cuda(z), ND).cpu().numpy()
    assert (got == oracle.d8(z, ND)).all()


@pytest.mark.parametrize("seed,H,W,levels,pnd", [(11, 257, 192, 3, 0.1), (12, 64, 512, 2, 0.0), (13, 33, 132, 5, 0.3),
                                                 (14, 1, 640, 4, 0.05), (15, 300, 4, 3, 0.2)])
def test_d8_vectorised_kernel_ties(fa_lib, seed, H, W, levels, pnd):
    """W % 4 == 0 takes the 4-columns-per-lane kernel with shared drops."""
    z = inputs.quantized_dem(seed, H, W, levels=levels, p_nodata=pnd)
    z[::5] = (z[::5] * np.float32(math.sqrt(2.0))).astype(np.float32)
    with fa_lib.Context(0) as ctx:
        got = ctx.flowdirs(_cuda(z), ND).cpu().numpy()
    assert (got == oracle.d8(z, ND)).all()


def test_d8_exact_sqrt2_pin(fa_lib):
    s2 = np.float32(math.sqrt(2.0))
    z = np.full((5, 5), 3.0, np.float32)
    z[2, 2] = 2.0
    z[2, 3] = 1.0
    z[1, 3] = np.float32(2.0) - s2
    with fa_lib.Context(0) as ctx:
        assert ctx.flowdirs(_cuda(z), ND).cpu().numpy()[2, 2] == 3


def test_d8_host_buffers(fa_lib):
    z = inputs.filled_dem(3, 100, 90)
    with fa_lib.Context(0) as ctx:
        got = ctx.flowdirs(z, ND)  # numpy in, numpy out: staged through the device
    assert (got == oracle.d8(z, ND)).all()


# ---------------------------------------------------------------- accumulation from dirs
RANDOM_CASES = [
    # seed, H, W, tile, p_nodata, p_noflow
    (0, 1, 1, (0, 0), 0.0, 0.0),
    (1, 1, 300, (0, 0), 0.0, 0.1),
    (2, 300, 1, (7, 1), 0.1, 0.0),
    (3, 64, 64, (0, 0), 0.0, 0.0),
    (4, 65, 63, (0, 0), 0.1, 0.02),
    (5, 200, 333, (0, 0), 0.3, 0.05),
    (6, 200, 333, (64, 64), 0.1, 0.02),
    (7, 257, 129, (100, 37), 0.15, 0.0),
    (8, 513, 700, (128, 256), 0.05, 0.01),
    (9, 130, 130, (1, 130), 0.1, 0.0),
    (10, 1024, 1024, (256, 256), 0.1, 0.01),
    (11, 777, 555, (65, 129), 0.2, 0.03),
]


@pytest.mark.parametrize("case", RANDOM_CASES, ids=lambda c: f"s{c[0]}_{c[1]}x{c[2]}_t{c[3][0]}x{c[3][1]}")
def test_acc_random_dirs_u32(fa_lib, case):
    seed, H, W, tile, pnd, pnf = case
    d = inputs.random_dirs(seed, H, W, p_nodata=pnd, p_noflow=pnf)
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate(dirs=_cuda(d), atype="u32").cpu().numpy()
    _check(got, d, _oracle_acc(d), "u32")


@pytest.mark.parametrize("case", RANDOM_CASES[4:9], ids=lambda c: f"s{c[0]}")
def test_acc_random_dirs_weighted_u64(fa_lib, case):
    seed, H, W, tile, pnd, pnf = case
    d = inputs.random_dirs(seed, H, W, p_nodata=pnd, p_noflow=pnf)
    w = inputs.weights_u32(seed, (H, W), 0, 1000)
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate(dirs=_cuda(d), w=_cuda(w), atype="u64").cpu().numpy()
    exp = oracle.accumulate(d, w)
    _check(got, d, exp, "u64")


@pytest.mark.parametrize("tile", [(0, 0), (64, 64), (1000, 129), (2048, 2048)])
def test_acc_serpentine_cfg2(fa_lib, tile):
    """cfg2: 4096^2 boustrophedon river, depth 16.7M (closed form P6)."""
    d = inputs.serpentine(4096, 4096)
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate(dirs=_cuda(d), atype="u32").cpu().numpy()
    y, x = np.mgrid[0:4096, 0:4096].astype(np.uint64)
    exp = (4096 * y + np.where(y % 2 == 0, x, 4095 - x) + 1).astype(np.uint32)
    _check(got, d, exp, "u32")


def test_acc_transposed_serpentine(fa_lib):
    d = inputs.serpentine(1024, 768, transposed=True)
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        got = ctx.accumulate(dirs=_cuda(d), atype="u64").cpu().numpy()
    _check(got, d, oracle.accumulate(d), "u64")


def test_acc_all_nodata_and_noflow(fa_lib):
    d = np.full((70, 90), 255, np.uint8)
    with fa_lib.Context(0) as ctx:
        got = ctx.accumulate(dirs=_cuda(d), atype="u32").cpu().numpy()
        assert (got == U32M).all()
        d0 = np.zeros((70, 90), np.uint8)
        got = ctx.accumulate(dirs=_cuda(d0), atype="u64").cpu().numpy()
        assert (got == 1).all()


# ---------------------------------------------------------------- from DEM (configs)
@pytest.mark.parametrize("name,size,tile", [("cfg0", None, (0, 0)), ("cfg0", None, (128, 128)),
                                            ("cfg1", 2048, (512, 512))])
def test_acc_dem_configs_u32(fa_lib, name, size, tile):
    cfg = inputs.make_config(name, size, size)
    d = oracle.d8(cfg.dem)
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate(dem=_cuda(cfg.dem), atype="u32").cpu().numpy()
    _check(got, d, _oracle_acc(d), "u32")


@pytest.mark.slow
def test_acc_cfg1_full(fa_lib):
    """cfg1 at its full size and tiling (8192^2, 2048^2 tiles), bit-exact."""
    cfg = inputs.make_config("cfg1")
    d = oracle.d8(cfg.dem)
    with fa_lib.Context(0, tile=cfg.tile) as ctx:
        dirs = ctx.flowdirs(_cuda(cfg.dem)).cpu().numpy()
        assert (dirs == d).all()
        got = ctx.accumulate(dem=_cuda(cfg.dem), atype="u32").cpu().numpy()
    _check(got, d, _oracle_acc(d), "u32")


@pytest.mark.parametrize("size,tile", [(1024, (0, 0)), (1536, (512, 512)), (1000, (333, 250))])
def test_acc_dem_weighted_f64_cfg3_recipe(fa_lib, size, tile):
    cfg = inputs.make_config("cfg3", size, size)
    d = oracle.d8(cfg.dem)
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate(dem=_cuda(cfg.dem), w=_cuda(cfg.w), atype="f64").cpu().numpy()
    _check(got, d, _oracle_acc(d, cfg.w, "f64"), "f64")
    # against the exact fixed-point sum too (P11)
    Ax = oracle.accumulate(d, cfg.w, kind="fix23")
    data = d != 255
    ex = Ax[data].astype(np.float64) * 2.0 ** -23
    assert (np.abs(got[data] - ex) / ex).max() <= 1e-9


@pytest.mark.parametrize("path", ["single", "strips", "streamed"])
def test_f64_grid_weights_bit_exact(fa_lib, path):
    """cfg3's weights lie on the grid 0.5 + k*2^-23 (P11): every partial sum
    is a multiple of 2^-23 below 2^30 (here Σw ≈ 1e6; cfg3 ≈ 9.7e8), so each
    fp64 addition is exact in any order and all three paths must equal the
    oracle's exact fixed-point sum bit for bit -- the D13 tolerance is not
    needed for this recipe (deterministic fp64)."""
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    ex = oracle.accumulate(d, cfg.w, kind="fix23")
    assert ex.max() < 2 ** 53
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        if path == "single":
            got = ctx.accumulate(dem=_cuda(cfg.dem), w=_cuda(cfg.w), atype="f64").cpu().numpy()
        elif path == "strips":
            got = ctx.accumulate_strips(4, dem=_cuda(cfg.dem), w=_cuda(cfg.w), atype="f64").cpu().numpy()
        else:
            got = ctx.accumulate_streamed(dem=cfg.dem, w=cfg.w, atype="f64", strip_rows=256)
    data = d != 255
    assert np.isnan(got[~data]).all()
    assert (got[data] == ex[data].astype(np.float64) * 2.0 ** -23).all()


def test_acc_host_buffers(fa_lib):
    d = inputs.random_dirs(21, 300, 200, p_nodata=0.1)
    with fa_lib.Context(0, tile=(64, 100)) as ctx:
        got = ctx.accumulate(dirs=d, atype="u64")  # numpy in / out
    _check(got, d, oracle.accumulate(d), "u64")


# ---------------------------------------------------------------- H4/H5 intermediates
@pytest.mark.parametrize("seed,H,W,th,tw", [(1, 200, 300, 64, 64), (2, 257, 129, 100, 37),
                                            (3, 128, 128, 128, 128), (4, 300, 300, 1, 300)])
def test_perimeter_records_match_oracle(fa_lib, seed, H, W, th, tw):
    d = inputs.random_dirs(seed, H, W, p_nodata=0.1, p_noflow=0.02)
    w = inputs.weights_u32(seed, (H, W), 0, 9)
    with fa_lib.Context(0, tile=(th, tw)) as ctx:
        links, at, xo, acc = ctx.perimeter_records(dirs=_cuda(d), w=_cuda(w), atype="u64")
    L = oracle.links(d, th, tw)
    assert (links.cpu().numpy() == L).all()
    A = oracle.accumulate(d, w)
    AT = oracle.tile_accumulate(d, th, tw, w)
    base = oracle.tiles_perim_base(H, W, th, tw)
    TC = (W + tw - 1) // tw
    at_exp = np.zeros(base[-1], np.uint64)
    for t in range(len(base) - 1):
        ty, tx = divmod(t, TC)
        y0, x0 = ty * th, tx * tw
        h, ww = min(th, H - y0), min(tw, W - x0)
        for p in range(base[t + 1] - base[t]):
            px, py = oracle.perim_xy(p, h, ww)
            if L[base[t] + p] == oracle.FLOW_EXTERNAL:
                at_exp[base[t] + p] = AT[y0 + py, x0 + px]
    assert (at.cpu().numpy() == at_exp).all()
    assert (xo.cpu().numpy() == oracle.offsets(d, th, tw, A)).all()
    _check(acc.cpu().numpy(), d, A, "u64")


def test_fig2_fixture_records(fa_lib):
    from golden_io import load_fig2

    f = load_fig2()
    d, w, (th, tw) = f["dirs"], f["w"], f["tile"]
    with fa_lib.Context(0, tile=(th, tw)) as ctx:
        links, at, xo, acc = ctx.perimeter_records(dirs=_cuda(d), w=_cuda(w), atype="u32")
    acc = acc.cpu().numpy()
    for x, y, v in f["expect_A"]:
        assert acc[y, x] == v == 100
    base = oracle.tiles_perim_base(14, 14, th, tw)
    for x, y, v in f["expect_X"]:
        t = (y // th) * 2 + x // tw
        assert xo.cpu().numpy()[base[t] + oracle.perim_index(x % tw, y % th, th, tw)] == v


# ---------------------------------------------------------------- errors
def test_errors(fa_lib):
    with fa_lib.Context(0) as ctx:
        d = np.full((10, 10), 3, np.uint8)
        d[4, 4] = 9
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate(dirs=_cuda(d))
        assert e.value.status == fa_lib.FA_E_DIRCODE
        d = np.full((10, 10), 0, np.uint8)
        d[3, 3], d[3, 4] = 3, 7  # 2-cycle inside a block
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate(dirs=_cuda(d))
        assert e.value.status == fa_lib.FA_E_CYCLE
        z = np.ones((10, 10), np.float32)
        w = np.ones((10, 10), np.float32)
        w[2, 2] = -1.0
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate(dem=_cuda(z), w=_cuda(w), atype="f64")
        assert e.value.status == fa_lib.FA_E_ARG
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate(dirs=_cuda(np.zeros((4, 4), np.uint8)), w=_cuda(w[:4, :4].copy()), atype="u32")
        assert e.value.status == fa_lib.FA_E_ARG
        wbig = np.full((64, 64), 2 ** 21, np.uint32)
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate(dirs=_cuda(np.zeros((64, 64), np.uint8)), w=_cuda(wbig), atype="u32")
        assert e.value.status == fa_lib.FA_E_OVERFLOW
        for shape in ((0, 16), (16, 0)):  # empty rasters are rejected, not run
            with pytest.raises(fa_lib.FaError) as e:
                ctx.accumulate(dirs=torch.zeros(shape, dtype=torch.uint8, device="cuda"), atype="u32")
            assert e.value.status == fa_lib.FA_E_ARG
        with pytest.raises(fa_lib.FaError) as e:  # dem and dirs together
            ctx.accumulate(dem=_cuda(z), dirs=_cuda(np.zeros((10, 10), np.uint8)), atype="u32")
        assert e.value.status == fa_lib.FA_E_ARG


def test_cycle_across_blocks(fa_lib):
    # a 2-cycle straddling a block boundary (cols 63|64) and a long loop of 4 blocks
    d = np.zeros((128, 128), np.uint8)
    d[10, 63], d[10, 64] = 3, 7
    with fa_lib.Context(0) as ctx:
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate(dirs=_cuda(d))
        assert e.value.status == fa_lib.FA_E_CYCLE
        d = np.zeros((128, 128), np.uint8)
        d[60, 60:70] = 3
        d[60:70, 70] = 5
        d[70, 61:71] = 7
        d[61:71, 60] = 1
        d[60, 70] = 5
        d[70, 70] = 7
        d[70, 60] = 1
        d[60, 60] = 3
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate(dirs=_cuda(d))
        assert e.value.status == fa_lib.FA_E_CYCLE
