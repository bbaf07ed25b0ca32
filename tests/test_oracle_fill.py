"""Pins of the depression-filling oracle (P:L59 Priority-Flood,
D15 with the epsilon step nextafterf): a hand-built pit, the fixed-point
certificate W(s) = z(s) at seeds and W(p) = max(z(p), nextafter(min W of
data neighbours)) elsewhere (its unique solution, a shortest-path fixpoint),
idempotence, no NoFlow cell after D8, and agreement with the independent
tiled label-correcting implementation of the input generator (G4)."""
import numpy as np
import pytest

import inputs
import oracle

NODATA = np.float32(-9999.0)


def _certify(z, W):
    H, Wd = z.shape
    nd = (z == NODATA) | ~np.isfinite(z)
    assert (W[nd] == z[nd]).all()
    zp = np.pad(z, 1, constant_values=NODATA)
    Wp = np.pad(W, 1, constant_values=np.inf)
    ndp = np.pad(nd, 1, constant_values=True)
    mins = np.full(z.shape, np.inf, np.float32)
    seed = np.zeros(z.shape, bool)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            if dy == 0 and dx == 0:
                continue
            nb_nd = ndp[1 + dy:1 + dy + H, 1 + dx:1 + dx + Wd]
            seed |= nb_nd
            w = np.where(nb_nd, np.inf, Wp[1 + dy:1 + dy + H, 1 + dx:1 + dx + Wd])
            mins = np.minimum(mins, w)
    data = ~nd
    assert (W[data & seed] == z[data & seed]).all()
    ns = data & ~seed
    exp = np.maximum(z[ns], np.nextafter(mins[ns], np.float32(np.inf)))
    assert (W[ns] == exp).all()


def test_hand_built_pit():
    z = np.full((5, 5), 10.0, np.float32)
    z[1:4, 1:4] = 1.0
    W = oracle.fill(z)
    e1 = np.nextafter(np.float32(10.0), np.float32(np.inf))
    e2 = np.nextafter(e1, np.float32(np.inf))
    exp = np.full((5, 5), 10.0, np.float32)
    exp[1:4, 1:4] = e1
    exp[2, 2] = e2
    assert (W == exp).all()


@pytest.mark.parametrize("seed,H,W,coast", [(1, 64, 64, 0.0), (2, 100, 77, 0.2), (3, 128, 128, 0.1)])
def test_fixed_point_certificate_and_generator_agreement(seed, H, W, coast):
    z = inputs.terrain(seed, H, W)
    if coast > 0:
        inputs.coast(z, seed, coast)
    F = oracle.fill(z)
    _certify(z, F)
    assert (F >= z).all()
    G = z.copy()
    inputs.fill(G)
    assert (F == G).all()
    assert (oracle.fill(F) == F).all()  # idempotent
    d = oracle.d8(F)
    assert not (d == 0).any()  # every data cell drains (P14)


def test_negative_elevations_and_nodata_blobs():
    rng = np.random.default_rng(4)
    z = (rng.random((60, 50)) * 40 - 20).astype(np.float32)  # below and above zero
    z[rng.random(z.shape) < 0.05] = NODATA
    z[10, 10] = np.inf  # non-finite counts as NoData
    F = oracle.fill(z)
    _certify(z, F)
