"""Pins for the oracle accumulation (O-ACC, O-BRUTE, O-TILE, O-PAPER) -- DESIGN.md P5-P11."""
import numpy as np
import pytest

import inputs
import oracle
from golden_io import load_fig2, load_perimeter_sizes, load_spec_examples

U64MAX = np.uint64(0xFFFFFFFFFFFFFFFF)


# ---------------------------------------------------------------- P5 worked examples
@pytest.mark.parametrize("case", load_spec_examples(), ids=lambda c: c[0])
def test_p5_spec_examples(case):
    name, dirs, exp = case
    for A in (oracle.accumulate(dirs), oracle.brute(dirs)):
        for r, row in enumerate(exp):
            for c, v in enumerate(row):
                assert A[r, c] == (U64MAX if v is None else v), (name, r, c)


# ---------------------------------------------------------------- P6 closed forms
@pytest.mark.parametrize("H,W", [(64, 64), (7, 13), (4096, 4096)])
def test_p6_serpentine_closed_form(H, W):
    d = inputs.serpentine(H, W)
    A = oracle.accumulate(d)
    y, x = np.mgrid[0:H, 0:W].astype(np.uint64)
    exp = np.uint64(W) * y + np.where(y % 2 == 0, x, np.uint64(W - 1) - x) + np.uint64(1)
    assert (A == exp).all()
    last = (H - 1, 0) if (H - 1) % 2 else (H - 1, W - 1)
    assert A[last] == H * W


def test_p6_plane_and_bowl_closed_forms():
    H, W = 17, 23
    y, x = np.mgrid[0:H, 0:W].astype(np.float32)
    A = oracle.accumulate(oracle.d8(x.copy()))          # plane z = x
    assert (A == (W - x).astype(np.uint64)).all()
    z = (np.abs(x - 11) + np.abs(y - 8)).astype(np.float32)  # L1 bowl
    A = oracle.accumulate(oracle.d8(z))
    assert A[8, 11] == H * W


def test_p6_transposed_serpentine():
    H, W = 12, 9
    d = inputs.serpentine(H, W, transposed=True)
    A = oracle.accumulate(d)
    assert A.max() == H * W


# ---------------------------------------------------------------- P7 brute force
@pytest.mark.parametrize("seed", range(40))
def test_p7_brute_equals_kahn_random(seed):
    rng = np.random.default_rng(seed)
    H, W = int(rng.integers(1, 65)), int(rng.integers(1, 65))
    d = inputs.random_dirs(seed, H, W, p_nodata=[0, 0.1, 0.3][seed % 3], p_noflow=[0, 0.05][seed % 2])
    w = inputs.weights_u32(seed, (H, W), 0, 9) if seed % 4 == 0 else None
    A = oracle.accumulate(d, w)
    assert (A == oracle.brute(d, w)).all()


def test_p7_cycle_detected():
    d = np.array([[3, 7]], np.uint8)  # E then W: 2-cycle
    with pytest.raises(oracle.OracleError) as e:
        oracle.accumulate(d)
    assert e.value.code == 3
    with pytest.raises(oracle.OracleError):
        oracle.brute(d)


def test_p7_bad_code_detected():
    d = np.array([[3, 9]], np.uint8)
    assert oracle.validate(d) == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.accumulate(d)
    assert e.value.code == 2


# ---------------------------------------------------------------- P7 tiles (O-TILE / O-PAPER)
TILE_CASES = [(0, 40, 40, 8, 8), (1, 50, 37, 16, 9), (2, 64, 64, 64, 1), (3, 33, 65, 1, 65),
              (4, 100, 100, 7, 13), (5, 96, 128, 32, 32), (6, 17, 19, 5, 5), (7, 1, 50, 1, 7)]


@pytest.mark.parametrize("seed,H,W,th,tw", TILE_CASES)
def test_p7_paper_tiled_equals_untiled(seed, H, W, th, tw):
    # the paper's own correctness test: tiled result == authoritative
    d = inputs.random_dirs(seed, H, W, p_nodata=0.15, p_noflow=0.03)
    A = oracle.accumulate(d)
    assert (oracle.paper(d, th, tw) == A).all()
    w = inputs.weights_u32(seed, (H, W), 0, 5)
    assert (oracle.paper(d, th, tw, w) == oracle.accumulate(d, w)).all()


@pytest.mark.parametrize("seed,H,W,th,tw", TILE_CASES[:5])
def test_p7_tile_linearity_identity(seed, H, W, th, tw):
    """A_global restricted to tile T == A_T + Acc_T(x injected at perimeter cells) (D12)."""
    d = inputs.random_dirs(seed, H, W, p_nodata=0.1, p_noflow=0.02)
    A = oracle.accumulate(d)
    AT = oracle.tile_accumulate(d, th, tw)
    X = oracle.offsets(d, th, tw, A)
    base = oracle.tiles_perim_base(H, W, th, tw)
    inj = np.zeros((H, W), np.uint64)
    TC = (W + tw - 1) // tw
    for t in range(len(base) - 1):
        ty, tx = divmod(t, TC)
        y0, x0 = ty * th, tx * tw
        h, ww = min(th, H - y0), min(tw, W - x0)
        for p in range(base[t + 1] - base[t]):
            px, py = oracle.perim_xy(p, h, ww)
            inj[y0 + py, x0 + px] = X[base[t] + p]
    # Acc_T(inj): per tile, weights = injection (u32 suffices at these sizes)
    acc_inj = np.zeros((H, W), np.uint64)
    for t in range(len(base) - 1):
        ty, tx = divmod(t, TC)
        y0, x0 = ty * th, tx * tw
        h, ww = min(th, H - y0), min(tw, W - x0)
        part = oracle.accumulate(d, inj.astype(np.uint32), region=(y0, x0, h, ww))
        acc_inj[y0:y0 + h, x0:x0 + ww] = part[y0:y0 + h, x0:x0 + ww]
    data = d != 255
    inj_w = acc_inj - inj  # Acc_T(inj) includes inj itself as the weight; subtract the w term
    total = AT + acc_inj
    assert (total[data] == A[data]).all()
    assert (inj_w[data] <= acc_inj[data]).all()


def test_p9_fig2_exit_receives_99_finalizes_to_100():
    f = load_fig2()
    d, w, (th, tw) = f["dirs"], f["w"], f["tile"]
    A = oracle.accumulate(d, w)
    assert (A == oracle.brute(d, w)).all()
    assert (oracle.paper(d, th, tw, w) == A).all()
    for x, y, v in f["expect_A"]:
        assert A[y, x] == v
    AT = oracle.tile_accumulate(d, th, tw, w)
    for x, y, v in f["expect_AT"]:
        assert AT[y, x] == v
    X = oracle.offsets(d, th, tw, A)
    H, W = d.shape
    base = oracle.tiles_perim_base(H, W, th, tw)
    TC = (W + tw - 1) // tw
    for x, y, v in f["expect_X"]:
        t = (y // th) * TC + x // tw
        p = oracle.perim_index(x - (x // tw) * tw, y - (y // th) * th, th, tw)
        assert X[base[t] + p] == v


def test_p9_fig2_links():
    """Alg. 2 links on the Fig. 2 fixture: E (10,6) is an entry whose path leaves
    tile (0,1) at its top edge; the donors are FlowExternal."""
    f = load_fig2()
    d, (th, tw) = f["dirs"], f["tile"]
    L = oracle.links(d, th, tw)
    base = oracle.tiles_perim_base(14, 14, th, tw)

    def slot(x, y):
        t = (y // th) * 2 + x // tw
        return base[t] + oracle.perim_index(x % tw, y % th, th, tw)

    assert L[slot(9, 7)] == oracle.FLOW_EXTERNAL
    assert L[slot(10, 7)] == oracle.FLOW_EXTERNAL
    assert L[slot(11, 7)] == oracle.FLOW_EXTERNAL
    assert L[slot(10, 6)] == oracle.perim_index(3, 0, 7, 7)     # exits at (10,0), top edge
    assert L[slot(7, 9)] == oracle.perim_index(2, 0, 7, 7)      # -> (9,7) = d1's slot
    assert L[slot(3, 0)] == oracle.FLOW_TERMINATES               # NoData cell


# ---------------------------------------------------------------- P8 invariants
@pytest.mark.parametrize("name,size", [("cfg0", None), ("cfg1", 1024), ("cfg3", 1024)])
def test_p8_invariants_on_config_recipes(name, size):
    cfg = inputs.make_config(name, size, size)
    d = oracle.d8(cfg.dem)
    A = oracle.accumulate(d)
    assert oracle.certify(d, A) == 0   # donor identity + sum over terminals == sum w
    data = d != 255
    assert (A[data] >= 1).all()
    st = oracle.stats(d)
    assert st["noflow"] == 0           # filled DEMs have no NoFlow cells (D3)
    assert int(A[data].max()) == st["max_acc"]


def test_p8_certificate_detects_a_wrong_cell():
    d = inputs.random_dirs(5, 30, 30, p_nodata=0.1)
    A = oracle.accumulate(d)
    B = A.copy()
    i = np.flatnonzero(d.ravel() != 255)[17]
    B.ravel()[i] += 1
    assert oracle.certify(d, B) > 0


# ---------------------------------------------------------------- P10 perimeter sizes
def test_p10_perimeter_sizes_and_payload_bytes():
    for side, P, up, down, tx, *_ in load_perimeter_sizes():
        assert oracle.perim_count(side, side) == P
        assert P * (1 + 8 + 2) == up and P * 8 == down and P * 19 == tx
    assert 100 * oracle.perim_count(4000, 4000) == 1_599_600
    assert 100 * oracle.perim_count(4000, 4000) * 11 + 7_200 == 17_602_800
    assert oracle.perim_count(16384, 16384) == 65532                   # u16 limit
    assert oracle.perim_count(1, 5) == 5 and oracle.perim_count(1, 1) == 1


@pytest.mark.parametrize("h,w", [(7, 7), (1, 1), (1, 9), (6, 1), (2, 2), (3, 8), (13, 5)])
def test_p10_perimeter_bijection(h, w):
    P = oracle.perim_count(h, w)
    seen = set()
    for p in range(P):
        x, y = oracle.perim_xy(p, h, w)
        assert oracle.perim_index(x, y, h, w) == p
        assert x in (0, w - 1) or y in (0, h - 1)
        seen.add((x, y))
    assert len(seen) == P
    if h == w == 7:  # S:L62-66 examples
        assert oracle.perim_xy(6, 7, 7) == (6, 0) and oracle.perim_xy(23, 7, 7) == (0, 1)
        assert oracle.perim_index(6, 6, 7, 7) == 12 and oracle.perim_index(3, 3, 7, 7) == -1


# ---------------------------------------------------------------- P11 fp64 vs exact
def test_p11_f64_within_bound_of_exact_fixed_point():
    cfg = inputs.make_config("cfg3", 512, 512)
    d = oracle.d8(cfg.dem)
    Af = oracle.accumulate(d, cfg.w, kind="f64")
    Ax = oracle.accumulate(d, cfg.w, kind="fix23")
    data = d != 255
    exact = Ax[data].astype(np.float64) * 2.0 ** -23  # exact: < 2^53 units
    assert (Ax[data] < 2 ** 53).all()
    h = oracle.stats(d)["max_height"] + 8
    rel = np.abs(Af[data] - exact) / exact
    assert rel.max() <= h * 2.0 ** -53
    assert np.isnan(Af[~data]).all()


# ---------------------------------------------------------------- or_stats pins
# Workload characterisation: the height of a cell is its
# longest upstream path (edges); an outlet is a data cell whose flow leaves
# the grid or enters NoData (D3, D8); NoFlow cells are counted apart.  Closed
# forms and a brute-force walk pin every output of oracle.stats.
def _brute_stats(d):
    """Heights by walking every cell's downstream path (height(t) = max over
    cells upstream of t of their distance to t); outlets / NoFlow by
    definition.  Independent of the oracle's chain-following schedule."""
    H, W = d.shape
    dx = [0, 0, 1, 1, 1, 0, -1, -1, -1]
    dy = [0, -1, -1, 0, 1, 1, 1, 0, -1]
    ht = np.zeros((H, W), np.int64)
    outlets = noflow = 0
    for y in range(H):
        for x in range(W):
            c = int(d[y, x])
            if c == 255:
                continue
            if c == 0:
                noflow += 1
            else:
                ty, tx = y + dy[c], x + dx[c]
                if not (0 <= ty < H and 0 <= tx < W) or d[ty, tx] == 255:
                    outlets += 1
            # walk downstream: cell at distance k gets height >= k
            cy, cx, k = y, x, 0
            while True:
                cc = int(d[cy, cx])
                if cc == 0:
                    break
                ty, tx = cy + dy[cc], cx + dx[cc]
                if not (0 <= ty < H and 0 <= tx < W) or d[ty, tx] == 255:
                    break
                cy, cx, k = ty, tx, k + 1
                ht[cy, cx] = max(ht[cy, cx], k)
    data = d != 255
    return ht, data, outlets, noflow


def test_stats_serpentine_closed_form():
    H, W = 6, 9
    st = oracle.stats(inputs.serpentine(H, W), nbins=8)
    assert st["max_height"] == H * W - 1            # one chain through every cell
    assert st["outlets"] == 1 and st["noflow"] == 0  # the last row end steps off the grid
    assert st["max_acc"] == H * W
    assert list(st["height_hist"][:7]) == [1] * 7 and st["height_hist"][7] == H * W - 7


def test_stats_plane_closed_form():
    H, W = 5, 12
    d = np.full((H, W), 7, np.uint8)  # every cell drains west: column 0 leaves the grid
    st = oracle.stats(d, nbins=W + 3)
    assert st["max_height"] == W - 1 and st["outlets"] == H and st["noflow"] == 0
    assert st["max_acc"] == W
    assert list(st["height_hist"]) == [H] * W + [0, 0, 0]  # height of column x is W-1-x


def test_stats_bowl_closed_form():
    k = 6
    n = 2 * k + 1
    y, x = np.mgrid[0:n, 0:n]
    d = oracle.d8((np.abs(x - k) + np.abs(y - k)).astype(np.float32))
    st = oracle.stats(d)
    assert st["noflow"] == 1 and st["outlets"] == 0  # everything drains into the interior centre
    assert st["max_acc"] == n * n
    assert st["max_height"] == k                      # diagonal steps from a corner reach the centre in k


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_stats_random_rasters_match_brute_force(seed):
    d = inputs.random_dirs(seed, 23, 31, p_nodata=0.1, p_noflow=0.05)  # acyclic by construction
    assert oracle.validate(d) == -1
    ht, data, outlets, noflow = _brute_stats(d)
    st = oracle.stats(d, nbins=16)
    assert st["max_height"] == int(ht[data].max())
    assert st["outlets"] == outlets and st["noflow"] == noflow
    hist = np.bincount(np.minimum(ht[data], 15), minlength=16)
    assert list(st["height_hist"]) == list(hist)
    assert st["max_acc"] == int(oracle.brute(d)[data].max())


# ---------------------------------------------------------------- P8 streamed certificate
@pytest.mark.parametrize("strip", [1, 7, 64, 1000])
def test_p8_streamed_certificate_equals_whole_raster(strip):
    """The strip-by-strip certificate (the cfg4 parity plan when the host holds
    only strips) gives the whole-raster verdict, and catches a wrong cell in
    any strip, including next to a strip boundary."""
    d = inputs.random_dirs(9, 131, 77, p_nodata=0.1, p_noflow=0.02)
    w = inputs.weights_u32(9, d.shape, 0, 9)
    A = oracle.accumulate(d, w)
    rows = lambda arr: (lambda a, b: arr[a:b])
    assert oracle.certify(d, A, w) == 0
    assert oracle.certify_strips(rows(d), rows(A), 131, 77, strip, rows(w)) == 0
    for y in (0, strip - 1 if strip < 131 else 5, 130):
        B = A.copy()
        x = int(np.flatnonzero(d[y] != 255)[0])
        B[y, x] += 1
        assert oracle.certify(d, B, w) > 0
        assert oracle.certify_strips(rows(d), rows(B), 131, 77, strip, rows(w)) > 0


def test_p8_streamed_certificate_mass_balance():
    d = inputs.serpentine(40, 30)
    A = oracle.accumulate(d)
    rows = lambda arr: (lambda a, b: arr[a:b])
    assert oracle.certify_strips(rows(d), rows(A), 40, 30, 9) == 0
    B = A.copy()
    B[39, 0] -= 1  # the outlet: donor identity AND mass balance break
    assert oracle.certify_strips(rows(d), rows(B), 40, 30, 9) >= 2
