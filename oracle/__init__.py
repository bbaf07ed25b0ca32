"""TEST INFRASTRUCTURE ONLY -- the CPU oracle (plain C, single-threaded).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA path and the CUDA path never imports it.

Thin numpy/ctypes marshalling over ``oracle.c``; every arithmetic step lives
in the C file, which cites PAPER.md for each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NODATA = 255
NOFLOW = 0
FLOW_EXTERNAL = 0xFFFFFFFE
FLOW_TERMINATES = 0xFFFFFFFF
LINK_CYCLE = 0xFFFFFFFD
# (dx, dy) of codes 1..8; index 0 unused
DX = (0, 0, 1, 1, 1, 0, -1, -1, -1)
DY = (0, -1, -1, 0, 1, 1, 1, 0, -1)

STATUS = {0: "ok", 1: "bad argument", 2: "illegal direction byte", 3: "cycle", 5: "out of memory"}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {STATUS.get(code, code)}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so: plain -O2, no fast-math, no FP contraction."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off",
                               "-fno-fast-math", _SRC, "-o", _LIB, "-lm"])
    return _LIB


_lib = None
_P = ctypes.c_void_p
_I = ctypes.c_int64


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        sig = {
            "or_d8": ([_P, _I, _I, ctypes.c_float, _P], None),
            "or_validate": ([_P, _I], _I),
            "or_acc_region_u64": ([_P, _I, _I, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_acc_region_f64": ([_P, _I, _I, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_acc_region_fix": ([_P, _I, _I, _I, _I, _I, _I, _P, ctypes.c_int, _P], ctypes.c_int),
            "or_brute_u64": ([_P, _I, _I, _P, _P], ctypes.c_int),
            "or_acc_alpha_f64": ([_P, _I, _I, _P, _P, _P], ctypes.c_int),
            "or_fill": ([_P, _I, _I, ctypes.c_float, _P], ctypes.c_int),
            "or_brute_alpha_f64": ([_P, _I, _I, _P, _P, _P], ctypes.c_int),
            "or_perim_count": ([_I, _I], _I),
            "or_perim_xy": ([_I, _I, _I, _P, _P], ctypes.c_int),
            "or_perim_index": ([_I, _I, _I, _I], _I),
            "or_tiles_perim_total": ([_I, _I, _I, _I, _P], _I),
            "or_links": ([_P, _I, _I, _I, _I, _P], ctypes.c_int),
            "or_tile_acc_u64": ([_P, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_tile_acc_f64": ([_P, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_offsets_u64": ([_P, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_offsets_f64": ([_P, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_paper_u64": ([_P, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_paper_f64": ([_P, _I, _I, _I, _I, _P, _P], ctypes.c_int),
            "or_certify_u64": ([_P, _I, _I, _P, _P], _I),
            "or_certify_f64": ([_P, _I, _I, _P, _P, ctypes.c_double, _P], _I),
            "or_certify_rows_u64": ([_P, _I, _I, _P, _P, _I, _I, _P], _I),
            "or_stats": ([_P, _I, _I, _P, _I, _P], _I),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return a.ctypes.data_as(_P)


def _chk(rc, what):
    if rc:
        raise OracleError(rc, what)


# ---------------------------------------------------------------- D8
def d8(z: np.ndarray, nodata=-9999.0) -> np.ndarray:
    """O-D8 (oracle.c or_d8)."""
    z = np.ascontiguousarray(z, np.float32)
    H, W = z.shape
    d = np.empty((H, W), np.uint8)
    _L().or_d8(_p(z), H, W, float(np.float32(nodata)), _p(d))
    return d


def validate(dirs: np.ndarray) -> int:
    return int(_L().or_validate(_p(np.ascontiguousarray(dirs)), dirs.size))


# ---------------------------------------------------------------- accumulation
def _w_u32(w):
    return None if w is None else np.ascontiguousarray(w, np.uint32)


def accumulate(dirs: np.ndarray, w: np.ndarray | None = None, kind: str = "u64",
               region=None) -> np.ndarray:
    """O-ACC.  kind: "u64" (w None or u32) | "f64" (w None or f32) |
    "fix23" (exact int64 in units of 2^-23; w f32 on that grid).
    region=(y0, x0, h, w) treats a sub-rectangle as the whole raster (A_T);
    cells outside the region are left 0."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    y0, x0, h, ww = region if region is not None else (0, 0, H, W)
    if kind == "u64":
        A = np.zeros((H, W), np.uint64)
        rc = _L().or_acc_region_u64(_p(dirs), H, W, y0, x0, h, ww, _p(_w_u32(w)), _p(A))
    elif kind == "f64":
        A = np.zeros((H, W), np.float64)
        wf = None if w is None else np.ascontiguousarray(w, np.float32)
        rc = _L().or_acc_region_f64(_p(dirs), H, W, y0, x0, h, ww, _p(wf), _p(A))
    elif kind == "fix23":
        A = np.zeros((H, W), np.int64)
        wf = np.ones((H, W), np.float32) if w is None else np.ascontiguousarray(w, np.float32)
        rc = _L().or_acc_region_fix(_p(dirs), H, W, y0, x0, h, ww, _p(wf), 23, _p(A))
    else:
        raise ValueError(kind)
    _chk(rc, "or_acc")
    return A


def brute(dirs: np.ndarray, w: np.ndarray | None = None) -> np.ndarray:
    """O-BRUTE: every cell adds w along its downstream path (small rasters)."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    A = np.zeros((H, W), np.uint64)
    _chk(_L().or_brute_u64(_p(dirs), H, W, _p(_w_u32(w)), _p(A)), "or_brute")
    return A


def fill(z: np.ndarray, nodata: float = -9999.0) -> np.ndarray:
    """O-FILL: Priority-Flood + epsilon (D15), literally; returns the filled copy."""
    z = np.ascontiguousarray(z, np.float32)
    H, W = z.shape
    out = np.empty_like(z)
    _chk(_L().or_fill(_p(z), H, W, float(nodata), _p(out)), "or_fill")
    return out


def accumulate_alpha(dirs: np.ndarray, alpha: np.ndarray, w: np.ndarray | None = None,
                     brute_force: bool = False) -> np.ndarray:
    """O-ACC with absorption (Eq. 1 with a per-cell alpha in [0,1]):
    A(p) = w(p) + sum_{target(n)=p} alpha(n) A(n); fp64; NoData -> NaN.
    brute_force=True: the independent path-walk form (small rasters)."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    al = np.ascontiguousarray(alpha, np.float32)
    wf = None if w is None else np.ascontiguousarray(w, np.float32)
    A = np.zeros((H, W), np.float64)
    fn = _L().or_brute_alpha_f64 if brute_force else _L().or_acc_alpha_f64
    _chk(fn(_p(dirs), H, W, _p(wf), _p(al), _p(A)), "or_acc_alpha")
    return A


# ---------------------------------------------------------------- perimeters / tiles
def perim_count(h: int, w: int) -> int:
    return int(_L().or_perim_count(h, w))


def perim_xy(p: int, h: int, w: int):
    x, y = ctypes.c_int64(), ctypes.c_int64()
    _chk(_L().or_perim_xy(p, h, w, ctypes.byref(x), ctypes.byref(y)), "or_perim_xy")
    return x.value, y.value


def perim_index(x: int, y: int, h: int, w: int) -> int:
    return int(_L().or_perim_index(x, y, h, w))


def tiles_perim_base(H: int, W: int, th: int, tw: int) -> np.ndarray:
    """Slot base per tile (row-major tiles, ragged last row/col); last entry = total."""
    nt = ((H + th - 1) // th) * ((W + tw - 1) // tw)
    base = np.zeros(nt + 1, np.int64)
    _L().or_tiles_perim_total(H, W, th, tw, _p(base))
    return base


def links(dirs: np.ndarray, th: int, tw: int) -> np.ndarray:
    """Alg. 2 FollowPath for every tile perimeter slot (u32, sentinels)."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    L = np.zeros(int(tiles_perim_base(H, W, th, tw)[-1]), np.uint32)
    _chk(_L().or_links(_p(dirs), H, W, th, tw, _p(L)), "or_links")
    return L


def tile_accumulate(dirs: np.ndarray, th: int, tw: int, w=None, kind: str = "u64") -> np.ndarray:
    """A_T: Alg. 1 on every tile separately (raster-shaped output)."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    if kind == "u64":
        A = np.zeros((H, W), np.uint64)
        rc = _L().or_tile_acc_u64(_p(dirs), H, W, th, tw, _p(_w_u32(w)), _p(A))
    else:
        A = np.zeros((H, W), np.float64)
        wf = None if w is None else np.ascontiguousarray(w, np.float32)
        rc = _L().or_tile_acc_f64(_p(dirs), H, W, th, tw, _p(wf), _p(A))
    _chk(rc, "or_tile_acc")
    return A


def offsets(dirs: np.ndarray, th: int, tw: int, A: np.ndarray) -> np.ndarray:
    """x(v) per tile perimeter slot: external inbound flow from a global A."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    n = int(tiles_perim_base(H, W, th, tw)[-1])
    if A.dtype == np.float64:
        X = np.zeros(n, np.float64)
        rc = _L().or_offsets_f64(_p(dirs), H, W, th, tw, _p(np.ascontiguousarray(A)), _p(X))
    else:
        X = np.zeros(n, np.uint64)
        rc = _L().or_offsets_u64(_p(dirs), H, W, th, tw, _p(np.ascontiguousarray(A, np.uint64)), _p(X))
    _chk(rc, "or_offsets")
    return X


def paper(dirs: np.ndarray, th: int, tw: int, w=None, kind: str = "u64") -> np.ndarray:
    """O-PAPER: literal tiled method (Alg. 1 FIFO, Alg. 2, producer graph, EVICT finalize)."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    if kind == "u64":
        A = np.zeros((H, W), np.uint64)
        rc = _L().or_paper_u64(_p(dirs), H, W, th, tw, _p(_w_u32(w)), _p(A))
    else:
        A = np.zeros((H, W), np.float64)
        wf = None if w is None else np.ascontiguousarray(w, np.float32)
        rc = _L().or_paper_f64(_p(dirs), H, W, th, tw, _p(wf), _p(A))
    _chk(rc, "or_paper")
    return A


# ---------------------------------------------------------------- certificates / stats
def certify(dirs: np.ndarray, A: np.ndarray, w=None, rtol: float = 1e-9):
    """Donor identity + mass balance.  u64/u32 A: exact -> #violations.
    f64 A: -> (#violations, max relative residual)."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    if A.dtype == np.float64:
        mr = ctypes.c_double()
        wf = None if w is None else np.ascontiguousarray(w, np.float32)
        bad = _L().or_certify_f64(_p(dirs), H, W, _p(wf), _p(np.ascontiguousarray(A)), rtol,
                                  ctypes.byref(mr))
        return int(bad), mr.value
    A64 = A.astype(np.uint64)
    if A.dtype == np.uint32:  # widen the NoData marker consistently
        A64[A == np.uint32(0xFFFFFFFF)] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return int(_L().or_certify_u64(_p(dirs), H, W, _p(_w_u32(w)), _p(np.ascontiguousarray(A64))))


def stats(dirs: np.ndarray, nbins: int = 64) -> dict:
    """Workload characterisation: max height, height histogram, #outlets, #NoFlow, max A."""
    dirs = np.ascontiguousarray(dirs, np.uint8)
    H, W = dirs.shape
    hist = np.zeros(nbins, np.int64)
    out = np.zeros(3, np.int64)
    mh = _L().or_stats(_p(dirs), H, W, _p(hist), nbins, _p(out))
    if mh < 0:
        raise OracleError(5, "or_stats")
    return dict(max_height=int(mh), height_hist=hist, outlets=int(out[0]), noflow=int(out[1]),
                max_acc=int(out[2]))


def certify_strips(dirs_rows, acc_rows, H: int, W: int, strip: int, w_rows=None):
    """P8 donor identity + mass balance, streamed: the raster is visited in
    strips of `strip` rows, each with its halo rows, so host memory holds
    O(strip * W) cells.  dirs_rows(a, b) / acc_rows(a, b) / w_rows(a, b)
    return rows [a, b) as arrays (u8 codes; u64 or u32 accumulation; u32
    weights or None).  Returns the number of violating cells (+1 if the mass
    balance fails) -- equal to certify() on the whole raster."""
    bad = 0
    acc = np.zeros(2, np.uint64)
    for r0 in range(0, H, strip):
        r1 = min(H, r0 + strip)
        a, b = max(0, r0 - 1), min(H, r1 + 1)
        d = np.ascontiguousarray(dirs_rows(a, b), np.uint8)
        A = np.asarray(acc_rows(a, b))
        if A.dtype == np.uint32:
            A64 = A.astype(np.uint64)
            A64[A == np.uint32(0xFFFFFFFF)] = np.uint64(0xFFFFFFFFFFFFFFFF)
        else:
            A64 = np.ascontiguousarray(A, np.uint64)
        wv = None if w_rows is None else np.ascontiguousarray(w_rows(a, b), np.uint32)
        bad += int(_L().or_certify_rows_u64(_p(d), b - a, W, _p(wv), _p(A64), r0 - a, r1 - a, _p(acc)))
    return bad + int(acc[0] != acc[1])
