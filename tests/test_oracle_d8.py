"""Pins for the oracle's D8 stencil (O-D8) -- DESIGN.md pins P1-P4.

Nothing here compares the oracle with itself: each check is a spec table,
a hand-derived worked example, a closed form, or an independent brute-force
implementation (slopes compared as exact squared values).
"""
import math

import numpy as np
import pytest

import inputs
import oracle

ND = np.float32(-9999.0)


def _single_lower(k):
    """3x3 interior patch inside a 5x5 raster: only neighbour k of the centre is lower."""
    z = np.full((5, 5), 100.0, np.float32)
    z[2, 2] = 50.0
    z[2 + oracle.DY[k], 2 + oracle.DX[k]] = 10.0
    return z


def test_p1_offsets_table_and_bijection():
    # 1=N(0,-1) 2=NE(+1,-1) 3=E(+1,0) 4=SE(+1,+1) 5=S(0,+1) 6=SW(-1,+1) 7=W(-1,0) 8=NW(-1,-1)
    table = {1: (0, -1), 2: (1, -1), 3: (1, 0), 4: (1, 1), 5: (0, 1), 6: (-1, 1), 7: (-1, 0), 8: (-1, -1)}
    seen = set()
    for k, (dx, dy) in table.items():
        assert (oracle.DX[k], oracle.DY[k]) == (dx, dy)
        seen.add((dx, dy))
        # the stencil points at the unique lower neighbour
        assert oracle.d8(_single_lower(k))[2, 2] == k
    assert len(seen) == 8 and (0, 0) not in seen


def test_p2_exact_sqrt2_worked_example():
    # centre 2.0, E neighbour 1.0 (drop 1), NE neighbour 2 - fl32(sqrt2) (exact subtraction):
    # exact reading: NE slope (sqrt2 rounded)/sqrt2 < 1  -> E wins (code 3).
    # A naive fl32(d/fl32(sqrt2)) gives exactly 1.0 -> tie -> NE (2) would win.
    s2 = np.float32(math.sqrt(2.0))
    ne = np.float32(2.0) - s2
    assert float(ne) == 0.58578646183013916015625
    assert np.float32(np.float32(2.0) - ne) == s2  # the drop is exactly fl32(sqrt2)
    assert np.float32(s2 / s2) == np.float32(1.0)  # the naive rule ties
    z = np.full((5, 5), 3.0, np.float32)
    z[2, 2] = 2.0
    z[2, 3] = 1.0  # E
    z[1, 3] = ne   # NE
    assert oracle.d8(z)[2, 2] == 3
    # centre 10, N 9 (drop 1), NE 8.5 (1.5/sqrt2 = 1.06) -> NE; NE 8.6 (1.4/sqrt2 = 0.99) -> N
    for ne_z, want in ((8.5, 2), (8.6, 1)):
        z = np.full((5, 5), 20.0, np.float32)
        z[2, 2] = 10.0
        z[1, 2] = 9.0
        z[1, 3] = ne_z
        assert oracle.d8(z)[2, 2] == want


def test_p3_plane_ridge_bowl_closed_forms():
    H, W = 9, 11
    y, x = np.mgrid[0:H, 0:W].astype(np.float32)
    # plane z = x: every cell with x >= 1 flows W (7); column x = 0 has no lower data
    # neighbour -> outlet through its lowest off-grid code (D3): N(1) for the corner
    # (0,0), SE(4) for the bottom-left corner (SE,S,SW,W,NW off-grid), SW(6) otherwise.
    d = oracle.d8(x.copy())
    assert (d[:, 1:] == 7).all()
    assert d[0, 0] == 1 and d[H - 1, 0] == 4 and (d[1:H - 1, 0] == 6).all()
    # ridge z = -|x - c|: ridge cells tie E/W at equal drops -> lowest code E (3)
    c = 5
    d = oracle.d8(-np.abs(x - c))
    assert (d[:, c] == 3).all()
    assert (d[:, c + 1:-1] == 3).all() and (d[:, 1:c] == 7).all()
    # L1 bowl: quadrant cells flow diagonally to the centre, axis cells cardinally,
    # the interior centre is NoFlow (0)
    cy, cx = 4, 5
    z = (np.abs(x - cx) + np.abs(y - cy)).astype(np.float32)
    d = oracle.d8(z)
    assert d[cy, cx] == 0
    assert d[cy - 2, cx + 2] == 6 and d[cy + 2, cx + 2] == 8  # SW / NW toward the centre
    assert d[cy + 3, cx - 1] == 2 and d[cy - 1, cx - 4] == 4   # NE / SE
    assert d[cy, cx + 3] == 7 and d[cy, cx - 2] == 3 and d[cy - 3, cx] == 5 and d[cy + 2, cx] == 1


def _brute_d8(z, nodata):
    """Independent D8: exact squared slopes (cardinal d^2, diagonal d^2/2) in fp64,
    argmax with lowest code on ties, then the off-grid/NoData fallback."""
    H, W = z.shape
    out = np.zeros((H, W), np.uint8)
    for r in range(H):
        for c in range(W):
            zc = z[r, c]
            if not np.isfinite(zc) or zc == nodata:
                out[r, c] = 255
                continue
            best, code, first_out = -1.0, 0, 0
            for k in range(1, 9):
                rr, cc = r + oracle.DY[k], c + oracle.DX[k]
                if not (0 <= rr < H and 0 <= cc < W) or not np.isfinite(z[rr, cc]) or z[rr, cc] == nodata:
                    first_out = first_out or k
                    continue
                d = float(np.float32(zc - z[rr, cc]))
                if d <= 0:
                    continue
                s = d * d if k % 2 == 1 else d * d / 2.0
                if s > best:
                    best, code = s, k
            out[r, c] = code if code else first_out
    return out


@pytest.mark.parametrize("seed,levels,pnd", [(1, 3, 0.0), (2, 4, 0.1), (3, 6, 0.3), (4, 2, 0.05)])
def test_p4_brute_d8_on_tied_dems(seed, levels, pnd):
    z = inputs.quantized_dem(seed, 23, 31, levels=levels, p_nodata=pnd)
    # add exact-sqrt2 stress: scale some rows by fl32(sqrt2) so cardinal/diagonal drops nearly tie
    z[::3] = (z[::3] * np.float32(math.sqrt(2.0))).astype(np.float32)
    z[z < -1000] = ND
    got = oracle.d8(z, nodata=ND)
    assert (got == _brute_d8(z, ND)).all()


def test_p4_brute_d8_nonfinite_is_nodata():
    z = inputs.quantized_dem(9, 12, 13, levels=5)
    z[3, 4] = np.nan
    z[5, 6] = np.inf
    z[7, 1] = -np.inf
    got = oracle.d8(z)
    assert got[3, 4] == got[5, 6] == got[7, 1] == 255
    assert (got == _brute_d8(z, ND)).all()


def test_p4_brute_d8_on_fractal_filled_dem():
    z = inputs.filled_dem(11, 48, 40, coast_frac=0.2)
    assert (oracle.d8(z) == _brute_d8(z, ND)).all()
