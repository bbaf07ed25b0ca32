"""Pins for the shared input generators (P14) -- determinism and structural invariants."""
import numpy as np
import pytest

import inputs
import oracle


def test_g1_rng_counter_based():
    # splitmix64 reference values (Vigna's published constants; x=0 -> 0xE220A8397B1DCDAF)
    assert inputs.splitmix64(0) == 0xE220A8397B1DCDAF
    u = inputs.u01(1, 0, 5)
    assert 0.0 <= u < 1.0 and u == inputs.u01(1, 0, 5)
    assert inputs.u01(1, 0, 5) != inputs.u01(1, 1, 5)


def test_g2_terrain_range_and_determinism():
    a = inputs.terrain(1, 256, 256)
    b = inputs.terrain(1, 256, 256)
    assert a.tobytes() == b.tobytes()
    assert a.min() == 0.0 and a.max() == 1000.0
    c = inputs.terrain(2, 256, 256)
    assert a.tobytes() != c.tobytes()
    r = inputs.terrain(3, 100, 37)
    assert r.shape == (100, 37) and r.min() == 0.0 and r.max() == 1000.0


def test_g3_coast_connected_touches_west():
    z = inputs.terrain(2, 300, 200)
    n = inputs.coast(z, 2, 0.1)
    nd = z == inputs.NODATA
    assert nd.sum() == n and nd[:, 0].all()
    # each row's NoData is a prefix -> connected through column 0
    for row in nd:
        k = row.sum()
        assert row[:k].all() and not row[k:].any()
    assert 0.05 < n / z.size < 0.15


@pytest.mark.parametrize("seed,H,W,frac", [(1, 64, 64, 0.0), (2, 80, 120, 0.1), (3, 129, 67, 0.3)])
def test_g4_fill_unique_descending_and_raised(seed, H, W, frac):
    z0 = inputs.terrain(seed, H, W)
    if frac:
        inputs.coast(z0, seed, frac)
    outs = []
    for tile in (0, 7, 32):
        z = z0.copy()
        inputs.fill(z, tile=tile)
        outs.append(z)
    # unique fixpoint: any tiling gives the same bits
    assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()
    z = outs[0]
    data = z != inputs.NODATA
    assert (z[data] >= z0[data]).all()
    # every data cell that is not a seed has a strictly lower data neighbour
    Hh, Ww = z.shape
    for y in range(Hh):
        for x in range(Ww):
            if not data[y, x]:
                continue
            nbrs = [(y + dy, x + dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if dy or dx]
            seed_cell = any(not (0 <= yy < Hh and 0 <= xx < Ww) or not data[yy, xx] for yy, xx in nbrs)
            if not seed_cell:
                assert any(z[yy, xx] < z[y, x] for yy, xx in nbrs), (y, x)
    # hence D8 on the filled surface has no NoFlow cell (D3) and is acyclic
    d = oracle.d8(z)
    assert not (d == 0).any()
    oracle.accumulate(d)


def test_g4_fill_brute_relaxation_small():
    """Independent check of the least-epsilon-cost definition by Bellman-Ford sweeps."""
    z0 = inputs.terrain(5, 24, 20)
    inputs.coast(z0, 5, 0.2)
    z = z0.copy()
    inputs.fill(z, tile=0)
    H, W = z0.shape
    data = z0 != inputs.NODATA
    Wv = np.where(data, np.float32(np.inf), z0).astype(np.float32)
    for y in range(H):
        for x in range(W):
            if data[y, x]:
                nb = [(y + dy, x + dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if dy or dx]
                if any(not (0 <= a < H and 0 <= b < W) or not data[a, b] for a, b in nb):
                    Wv[y, x] = z0[y, x]
    changed = True
    while changed:
        changed = False
        for y in range(H):
            for x in range(W):
                if not data[y, x]:
                    continue
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        a, b = y + dy, x + dx
                        if (dy or dx) and 0 <= a < H and 0 <= b < W and data[a, b] and np.isfinite(Wv[a, b]):
                            cand = max(z0[y, x], np.nextafter(Wv[a, b], np.float32(np.inf)))
                            if cand < Wv[y, x]:
                                Wv[y, x] = cand
                                changed = True
    assert (Wv[data] == z[data]).all()


def test_g5_weights_grid():
    w = inputs.weights_f32(4, (50, 50))
    assert w.min() >= 0.5 and w.max() < 1.5
    k = (w.astype(np.float64) - 0.5) * 2 ** 23
    assert (k == np.floor(k)).all()
    assert inputs.weights_f32(4, (50, 50)).tobytes() == w.tobytes()


def test_g6_serpentine_structure():
    d = inputs.serpentine(6, 5)
    assert list(d[0]) == [3, 3, 3, 3, 5] and list(d[1]) == [5, 7, 7, 7, 7]
    assert d[5, 0] == 5  # last row end steps S off the grid


def test_random_dirs_acyclic_and_valid():
    d = inputs.random_dirs(3, 40, 50, p_nodata=0.2, p_noflow=0.05)
    assert oracle.validate(d) == -1
    oracle.accumulate(d)  # raises on a cycle
    assert 0.1 < (d == 255).mean() < 0.3
