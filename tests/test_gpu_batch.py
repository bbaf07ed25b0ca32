"""GPU parity of fa_accumulate_batch: a queue of independent host rasters,
each accumulated as fa_accumulate does it (P:L49-57 per raster), with the
uploads / downloads of neighbouring rasters overlapping the device work.
Every raster is compared with the CPU oracle: bit-exact for integers, D13
(1e-9 relative) for f64."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

U32M = np.uint32(0xFFFFFFFF)


def _exp_u32(d, w=None):
    e = oracle.accumulate(d, w).astype(np.uint32)
    e[d == 255] = U32M
    return e


def test_batch_dem_u32_distinct_rasters(fa_lib):
    dems = [inputs.filled_dem(40 + k, 300, 260, coast_frac=0.1) for k in range(5)]
    with fa_lib.Context(0, tile=(128, 128)) as ctx:
        outs = ctx.accumulate_batch(dems=dems, atype="u32")
        st = ctx.stats()
    for z, o in zip(dems, outs):
        assert (o == _exp_u32(oracle.d8(z))).all()
    assert st["cells"] == 5 * 300 * 260 and st["ms_total"] > 0 and st["ms_compute"] > 0
    assert st["bytes_exchanged"] == 5 * 300 * 260 * (4 + 4)


def test_batch_f64_pinned_repeated_inputs(fa_lib):
    cfg = inputs.make_config("cfg3", 640, 512)
    z = torch.from_numpy(cfg.dem).pin_memory()
    w = torch.from_numpy(cfg.w).pin_memory()
    z2 = torch.from_numpy(inputs.filled_dem(9, 640, 512, coast_frac=0.1)).pin_memory()
    dems = [z, z2, z, z2]
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        outs = ctx.accumulate_batch(dems=dems, ws=[w, w, w, w], atype="f64")
    for zz, o in zip(dems, outs):
        assert o.is_pinned()
        d = oracle.d8(zz.numpy())
        exp = oracle.accumulate(d, cfg.w, kind="f64")
        got = o.numpy()
        data = d != 255
        assert np.isnan(got[~data]).all()
        assert (np.abs(got[data] - exp[data]) / np.abs(exp[data])).max() <= 1e-9
    # the same input twice: equal within D13 (f64 REDs land in any order, so not bit-equal)
    a, b = outs[0].numpy(), outs[2].numpy()
    m = ~np.isnan(a)
    assert (np.abs(a[m] - b[m]) <= 1e-9 * np.abs(a[m])).all()


def test_batch_dirs_u64_u32_weights_ragged(fa_lib):
    ds = [inputs.random_dirs(50 + k, 333, 129, p_nodata=0.1, p_noflow=0.03) for k in range(3)]
    ws = [inputs.weights_u32(50 + k, (333, 129), 0, 1000) for k in range(3)]
    with fa_lib.Context(0, tile=(100, 64)) as ctx:
        ctx.set_option("block_rows", 16)
        outs = ctx.accumulate_batch(dirs=ds, ws=ws, atype="u64")
    for d, w, o in zip(ds, ws, outs):
        assert (o == oracle.accumulate(d, w)).all()


def test_batch_one_raster_and_empty(fa_lib):
    d = inputs.serpentine(256, 192)
    with fa_lib.Context(0) as ctx:
        assert ctx.accumulate_batch(dirs=[]) == []
        (o,) = ctx.accumulate_batch(dirs=[d])
    assert (o == oracle.accumulate(d).astype(np.uint32)).all()


def test_batch_errors(fa_lib):
    good = inputs.random_dirs(61, 128, 64)
    bad = np.zeros((128, 64), np.uint8)
    bad[63, 10], bad[64, 10] = 5, 1  # a 2-cycle
    with fa_lib.Context(0, tile=(64, 64)) as ctx:
        outs = [np.zeros((128, 64), np.uint32) for _ in range(3)]
        with pytest.raises(fa_lib.FaError) as e:
            ctx.accumulate_batch(dirs=[good, bad, good], outs=outs)
        assert e.value.status == fa_lib.FA_E_CYCLE and "raster 1" in str(e.value)
        assert (outs[0] == oracle.accumulate(good).astype(np.uint32)).all()  # rasters before it are complete
        with pytest.raises(fa_lib.FaError) as e:  # device buffers are rejected
            ctx.accumulate_batch(dirs=[torch.from_numpy(good).cuda()])
        assert e.value.status == fa_lib.FA_E_ARG
        with pytest.raises(ValueError):
            ctx.accumulate_batch(dirs=[good, good], ws=[np.ones((128, 64), np.uint32)])
        # the context stays usable
        (o,) = ctx.accumulate_batch(dirs=[good])
        assert (o == oracle.accumulate(good).astype(np.uint32)).all()
