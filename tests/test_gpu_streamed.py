"""GPU parity of the out-of-core path (the paper's EVICT
strategy): `fa_accumulate_streamed` keeps the raster in
host memory and only strips of whole tile rows on the device.  Phase A
(upload, D8, pass 1, tile records) and phase B (upload again, pass 1,
injected offsets, finalize, download) must give exactly the oracle's
integers, and the f64 result within D13, for every strip height -- one tile
row per strip (the most strips), ragged last strips, one strip holding the
whole raster -- and from a DEM (2-row z halos) or a D8 raster (1-row halos).
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,H,W,tile,strip_rows", [(1, 300, 257, (64, 50), 64), (2, 300, 257, (64, 50), 100),
                                                      (3, 129, 333, (32, 64), 1), (4, 513, 200, (100, 37), 250),
                                                      (5, 64, 64, (1, 64), 3), (6, 200, 180, (50, 60), 10**6)])
def test_streamed_random_dirs_u64(fa_lib, seed, H, W, tile, strip_rows):
    d = inputs.random_dirs(seed, H, W, p_nodata=0.12, p_noflow=0.02)
    w = inputs.weights_u32(seed, (H, W), 0, 50)
    with fa_lib.Context(0, tile=tile) as ctx:
        got = ctx.accumulate_streamed(dirs=d, w=w, atype="u64", strip_rows=strip_rows)
    assert (got == oracle.accumulate(d, w)).all()


def test_streamed_transposed_serpentine_crosses_every_strip(fa_lib):
    d = inputs.serpentine(512, 384, transposed=True)
    with fa_lib.Context(0, tile=(64, 64)) as ctx:
        got = ctx.accumulate_streamed(dirs=d, atype="u32", strip_rows=64)
    assert (got == oracle.accumulate(d).astype(np.uint32)).all()
    assert got.max() == 512 * 384


@pytest.mark.parametrize("strip_rows", [256, 384, 0])
def test_streamed_dem_f64_cfg3_recipe(fa_lib, strip_rows):
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        got = ctx.accumulate_streamed(dem=cfg.dem, w=cfg.w, atype="f64", strip_rows=strip_rows)
        st = ctx.stats()
    exp = oracle.accumulate(d, cfg.w, kind="f64")
    data = d != 255
    assert np.isnan(got[~data]).all()
    assert (np.abs(got[data] - exp[data]) / exp[data]).max() <= 1e-9
    # PCIe bytes: z and w uploaded twice, A downloaded once
    assert st["bytes_exchanged"] == 2 * 1024 * 1024 * 8 + 1024 * 1024 * 8


def test_streamed_dem_u32_pinned_torch(fa_lib):
    cfg = inputs.make_config("cfg1", 2048, 2048)
    d = oracle.d8(cfg.dem)
    dem = torch.from_numpy(cfg.dem).pin_memory()
    with fa_lib.Context(0, tile=(512, 512)) as ctx:
        got = ctx.accumulate_streamed(dem=dem, atype="u32", strip_rows=512)
        one = ctx.accumulate(dem=dem.cuda(), atype="u32").cpu()
    assert got.is_pinned()
    exp = oracle.accumulate(d).astype(np.uint32)
    assert (got.numpy() == exp).all()
    assert (one.numpy() == exp).all()


def test_streamed_rejects_device_buffers_and_reports_cycles(fa_lib):
    d = np.full((8, 8), 3, np.uint8)
    d[:, 7] = 5
    d[7, :] = 7
    d[7, 0] = 1  # the last column / row loop: a cycle
    with fa_lib.Context(0, tile=(4, 4)) as ctx:
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate_streamed(dirs=torch.from_numpy(d).cuda(), atype="u32", strip_rows=4,
                                    out=np.empty((8, 8), np.uint32))
        assert e.value.status == fa_lib.FA_E_ARG
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate_streamed(dirs=d, atype="u32", strip_rows=4)
        assert e.value.status == fa_lib.FA_E_CYCLE
