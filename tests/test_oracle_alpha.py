"""Pins of the absorption oracle (Eq. 1 with a per-cell alpha,
P:L49-57): A(p) = w(p) + sum_{target(n)=p} alpha(n) A(n).  Checked against
closed forms, the alpha = 1 / alpha = 0 special cases, a hand-built star,
linearity, and the independent path-walk form on random rasters."""
import numpy as np
import pytest

import inputs
import oracle


def test_chain_geometric_closed_form():
    # 1 x n chain flowing east into a NoFlow end: A_k = sum_j alpha^j = (1 - a^(k+1)) / (1 - a)
    n = 40
    d = np.full((1, n), 3, np.uint8)
    d[0, -1] = 0
    for a in (0.5, 0.25, 0.75):
        A = oracle.accumulate_alpha(d, np.full((1, n), a, np.float32))
        k = np.arange(n)
        exp = (1.0 - a ** (k + 1)) / (1.0 - a)
        assert np.allclose(A[0], exp, rtol=1e-15, atol=0)
    A = oracle.accumulate_alpha(d, np.full((1, n), 0.5, np.float32))
    assert (A[0] == 2.0 - 2.0 ** -np.arange(n)).all()  # exact in binary


def test_alpha_one_is_plain_accumulation_and_zero_is_w():
    d = inputs.random_dirs(3, 50, 40, p_nodata=0.1, p_noflow=0.05)
    w = inputs.weights_f32(3, d.shape)
    A1 = oracle.accumulate_alpha(d, np.ones(d.shape, np.float32), w)
    Aref = oracle.accumulate(d, w, kind="f64")
    data = d != 255
    assert (A1[data] == Aref[data]).all() and np.isnan(A1[~data]).all()
    A0 = oracle.accumulate_alpha(d, np.zeros(d.shape, np.float32), w)
    assert (A0[data] == w[data].astype(np.float64)).all()


def test_star_by_hand():
    # 3x3: the 8 ring cells drain into the NoFlow centre (codes pointing inwards)
    d = np.array([[4, 5, 6], [3, 0, 7], [2, 1, 8]], np.uint8)
    al = np.array([[0.5, 0.25, 1.0], [0.0, 0.9, 0.75], [0.125, 1.0, 0.5]], np.float32)
    w = np.arange(1, 10, dtype=np.float32).reshape(3, 3)
    A = oracle.accumulate_alpha(d, al, w)
    ring = [(0, 0), (0, 1), (0, 2), (1, 2), (2, 2), (2, 1), (2, 0), (1, 0)]
    exp = 5.0 + sum(float(al[y, x]) * float(w[y, x]) for y, x in ring)
    assert A[1, 1] == exp
    for y, x in ring:
        assert A[y, x] == w[y, x]


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_kahn_equals_path_walk(seed):
    rng = np.random.default_rng(seed)
    d = inputs.random_dirs(seed, 48, 37, p_nodata=0.1, p_noflow=0.03)
    al = rng.random(d.shape).astype(np.float32)
    al[rng.random(d.shape) < 0.2] = 1.0
    w = inputs.weights_f32(seed, d.shape)
    A = oracle.accumulate_alpha(d, al, w)
    B = oracle.accumulate_alpha(d, al, w, brute_force=True)
    data = d != 255
    assert np.allclose(A[data], B[data], rtol=1e-12, atol=0)
    assert np.isnan(A[~data]).all()


def test_linear_in_w_and_alpha_validation():
    rng = np.random.default_rng(7)
    d = inputs.random_dirs(7, 40, 40, p_nodata=0.1)
    al = rng.random(d.shape).astype(np.float32)
    w1 = inputs.weights_f32(1, d.shape)
    w2 = inputs.weights_f32(2, d.shape)
    data = d != 255
    Aa = oracle.accumulate_alpha(d, al, w1) + oracle.accumulate_alpha(d, al, w2)
    Ab = oracle.accumulate_alpha(d, al, (w1.astype(np.float64) + w2).astype(np.float32))
    assert np.allclose(Aa[data], Ab[data], rtol=1e-6)
    bad = al.copy()
    bad[data.nonzero()[0][0], data.nonzero()[1][0]] = 1.5
    with pytest.raises(oracle.OracleError):
        oracle.accumulate_alpha(d, bad)
    ok = al.copy()
    ok[~data] = np.nan  # NoData cells' alpha is ignored
    oracle.accumulate_alpha(d, ok)
