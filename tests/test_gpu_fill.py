"""GPU parity of depression filling (D15) against the
Priority-Flood+epsilon oracle: bit-exact f32 on the terrain recipes with and
without NoData coasts, ragged tile edges, negative elevations with NoData
blobs and non-finite cells, deep pits (long propagation across tiles), host
buffers, and the full DEM -> fill -> D8 -> accumulation pipeline."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu
NODATA = np.float32(-9999.0)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("seed,H,W,coast", [(1, 256, 256, 0.0), (2, 300, 257, 0.1), (3, 129, 333, 0.3),
                                            (4, 1, 50, 0.0), (5, 517, 1030, 0.05)])
def test_fill_terrain_bit_exact(fa_lib, seed, H, W, coast):
    z = inputs.terrain(seed, H, W)
    if coast > 0:
        inputs.coast(z, seed, coast)
    exp = oracle.fill(z)
    with fa_lib.Context(0) as ctx:
        got = ctx.fill(_cuda(z)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_fill_negative_nodata_blobs_and_host_buffers(fa_lib):
    rng = np.random.default_rng(4)
    z = (rng.random((200, 180)) * 40 - 20).astype(np.float32)
    z[rng.random(z.shape) < 0.05] = NODATA
    z[10, 10] = np.inf
    z[20, 30] = np.nan
    exp = oracle.fill(z)
    with fa_lib.Context(0) as ctx:
        got = ctx.fill(z)  # numpy in / out
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("tile", ["32", "64"])
def test_fill_deep_bowl_crosses_many_tiles(fa_lib, tile):
    # an L1 bowl: every interior cell is raised, the fill propagates inwards
    # across 8-16 tiles from the edge (FA_OPT_FILL_TILE: the 32x32 default
    # and the 64x64 tile kernel)
    H = W = 1024
    y, x = np.mgrid[0:H, 0:W]
    z = (np.abs(x - W // 2) + np.abs(y - H // 2)).astype(np.float32) * 0.01
    exp = oracle.fill(z)
    with fa_lib.Context(0) as ctx:
        ctx.set_option("fill_tile", int(tile))
        got = ctx.fill(_cuda(z)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    assert (exp > z).mean() > 0.4  # the inner diamond is raised to the rim level


def test_fill_then_accumulate_pipeline(fa_lib):
    z = inputs.terrain(7, 512, 512)
    inputs.coast(z, 7, 0.1)
    F = oracle.fill(z)
    d = oracle.d8(F)
    with fa_lib.Context(0, tile=(128, 128)) as ctx:
        zf = ctx.fill(_cuda(z))
        A = ctx.accumulate(dem=zf, atype="u64").cpu().numpy()
    assert (A == oracle.accumulate(d)).all()


def test_fill_serpentine_corridor_needs_many_launches(fa_lib):
    """A 1-cell corridor snaking through the whole raster, walls 1000 m high,
    its only outlet on the west edge: the filled surface rises one ulp per
    corridor cell from the outlet (~512K cells), so the fill front must travel
    the whole path -- far more launches than the old 4(H+W) guard allowed
    (a winding depression needs ~ path length / tile side launches)."""
    H = W = 1024
    z = np.full((H, W), 1000.0, np.float32)
    for y in range(1, H - 1, 2):
        z[y, 1:W - 1] = 0.0                      # corridor rows
        if y + 2 < H - 1:
            x = W - 2 if (y // 2) % 2 == 0 else 1
            z[y + 1, x] = 0.0                    # the bend to the next corridor row
    z[1, 0] = 0.0                                # the outlet (an edge seed)
    exp = oracle.fill(z)
    with fa_lib.Context(0) as ctx:
        got = ctx.fill(_cuda(z)).cpu().numpy()
        launches = ctx.stats()["launches"]
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    assert launches > 4 * (H + W) + 64
    assert (exp[z == 0.0] > 0).sum() >= (z == 0.0).sum() - 1  # every corridor cell but the outlet was raised
