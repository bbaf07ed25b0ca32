"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no D8 rule, no accumulation,
no stitching).  It wraps ``fa_inputs.c`` (recipes G1..G6, DESIGN.md "Input
recipe") through ctypes and builds the five BASELINE.json configurations.
The synthetic rasters stand in for the paper's SRTM / NED / PAMAP datasets
(Table 1), which are not available here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fa_inputs.c")
_LIB = os.path.join(_HERE, "libfa_inputs.so")

NODATA = np.float32(-9999.0)
ROUGHNESS = 0.6

_c_i64 = ctypes.c_int64
_c_u64 = ctypes.c_uint64
_c_f32 = ctypes.c_float
_c_dbl = ctypes.c_double
_c_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile libfa_inputs.so (gcc, OpenMP, -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", "-std=c11", _SRC, "-o", _LIB, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.fa_in_terrain.argtypes = [_c_u64, _c_i64, _c_i64, _c_dbl, _c_p]
        lib.fa_in_terrain.restype = ctypes.c_int
        lib.fa_in_coast.argtypes = [_c_u64, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_f32, _c_p]
        lib.fa_in_coast.restype = _c_i64
        lib.fa_in_fill.argtypes = [_c_i64, _c_i64, _c_f32, _c_p]
        lib.fa_in_fill.restype = _c_i64
        lib.fa_in_fill_tiled.argtypes = [_c_i64, _c_i64, _c_f32, _c_p, _c_i64]
        lib.fa_in_fill_tiled.restype = _c_i64
        lib.fa_in_weights.argtypes = [_c_u64, _c_i64, _c_p]
        lib.fa_in_weights.restype = None
        lib.fa_in_weights_u32.argtypes = [_c_u64, _c_i64, ctypes.c_uint32, ctypes.c_uint32, _c_p]
        lib.fa_in_weights_u32.restype = None
        lib.fa_in_serpentine.argtypes = [_c_i64, _c_i64, ctypes.c_int, _c_p]
        lib.fa_in_serpentine.restype = None
        lib.fa_in_random_dirs.argtypes = [_c_u64, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_p]
        lib.fa_in_random_dirs.restype = None
        lib.fa_in_quantized_dem.argtypes = [_c_u64, _c_i64, _c_i64, ctypes.c_int, _c_dbl, _c_f32, _c_p]
        lib.fa_in_quantized_dem.restype = None
        lib.fa_in_u01.argtypes = [_c_u64, _c_u64, _c_u64]
        lib.fa_in_u01.restype = _c_dbl
        lib.fa_in_splitmix64.argtypes = [_c_u64]
        lib.fa_in_splitmix64.restype = _c_u64
        lib.fa_in_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_c_p)


def u01(seed: int, stream: int, i: int) -> float:
    return _L().fa_in_u01(seed, stream, i)


def splitmix64(x: int) -> int:
    return _L().fa_in_splitmix64(x)


def terrain(seed: int, H: int, W: int, rough: float = ROUGHNESS) -> np.ndarray:
    """G2: diamond-square fractal terrain, range exactly [0, 1000]."""
    z = np.empty((H, W), np.float32)
    rc = _L().fa_in_terrain(seed, H, W, rough, _ptr(z))
    if rc:
        raise RuntimeError(f"fa_in_terrain failed ({rc})")
    return z


def coast(z: np.ndarray, seed: int, frac: float, rough: float = ROUGHNESS,
          nodata: np.float32 = NODATA) -> int:
    """G3: in-place NoData ocean on the west side; returns #NoData cells."""
    H, W = z.shape
    n = _L().fa_in_coast(seed, H, W, frac, rough, nodata, _ptr(z))
    if n < 0:
        raise RuntimeError("fa_in_coast failed")
    return int(n)


def fill(z: np.ndarray, nodata: np.float32 = NODATA, tile: int = 256) -> int:
    """G4: in-place least-epsilon-cost fill (Priority-Flood+epsilon); returns #raised cells.

    The result is unique, so `tile` (the parallel decomposition) never changes it."""
    H, W = z.shape
    n = _L().fa_in_fill_tiled(H, W, nodata, _ptr(z), tile)
    if n < 0:
        raise RuntimeError(f"fa_in_fill failed ({n})")
    return int(n)


def weights_f32(seed: int, shape) -> np.ndarray:
    """G5: f32 weights 0.5 + k*2^-23 in [0.5, 1.5)."""
    w = np.empty(shape, np.float32)
    _L().fa_in_weights(seed, w.size, _ptr(w))
    return w


def weights_u32(seed: int, shape, lo: int = 0, hi: int = 7) -> np.ndarray:
    w = np.empty(shape, np.uint32)
    _L().fa_in_weights_u32(seed, w.size, lo, hi, _ptr(w))
    return w


def serpentine(H: int, W: int, transposed: bool = False) -> np.ndarray:
    """G6: boustrophedon river (depth H*W)."""
    d = np.empty((H, W), np.uint8)
    _L().fa_in_serpentine(H, W, int(transposed), _ptr(d))
    return d


def random_dirs(seed: int, H: int, W: int, p_nodata: float = 0.0, p_noflow: float = 0.0) -> np.ndarray:
    """Random acyclic D8 raster (potential-descending choices)."""
    d = np.empty((H, W), np.uint8)
    _L().fa_in_random_dirs(seed, H, W, p_nodata, p_noflow, _ptr(d))
    return d


def quantized_dem(seed: int, H: int, W: int, levels: int = 4, p_nodata: float = 0.0,
                  nodata: np.float32 = NODATA) -> np.ndarray:
    z = np.empty((H, W), np.float32)
    _L().fa_in_quantized_dem(seed, H, W, levels, p_nodata, nodata, _ptr(z))
    return z


def num_threads() -> int:
    return _L().fa_in_num_threads()


def filled_dem(seed: int, H: int, W: int, coast_frac: float = 0.0) -> np.ndarray:
    """G2 (+G3) + G4: the DEM recipe of configs 0, 1, 3, 4."""
    z = terrain(seed, H, W)
    if coast_frac > 0:
        coast(z, seed, coast_frac)
    fill(z)
    return z


@dataclass
class Config:
    """One BASELINE.json configuration (inputs as host numpy arrays)."""
    name: str
    rows: int
    cols: int
    tile: tuple            # (tile_rows, tile_cols); (0, 0) = one tile
    atype: str             # "u32" | "u64" | "f64"
    dem: np.ndarray | None = None
    dirs: np.ndarray | None = None
    w: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def cells(self) -> int:
        return self.rows * self.cols


CONFIG_SPECS = {
    # name: (rows, cols, seed, coast_frac, kind, tile, atype, weights)
    "cfg0": (512, 512, 1, 0.0, "dem", (0, 0), "u32", False),
    "cfg1": (8192, 8192, 2, 0.05, "dem", (2048, 2048), "u32", False),
    "cfg2": (4096, 4096, 3, 0.0, "serpentine", (0, 0), "u32", False),
    "cfg3": (32768, 32768, 4, 0.10, "dem", (4096, 4096), "f64", True),
    "cfg4": (131072, 131072, 5, 0.30, "dem", (4096, 4096), "u64", False),
}


def make_config(name: str, rows: int | None = None, cols: int | None = None) -> Config:
    """Build config `name`; rows/cols override gives a same-recipe crop-size variant."""
    R, C, seed, frac, kind, tile, atype, weighted = CONFIG_SPECS[name]
    R = rows or R
    C = cols or C
    cfg = Config(name=name, rows=R, cols=C, tile=tile, atype=atype)
    if kind == "dem":
        z = terrain(seed, R, C)
        nd = coast(z, seed, frac) if frac > 0 else 0
        raised = fill(z)
        cfg.dem = z
        cfg.meta.update(nodata_cells=nd, nodata_frac=nd / (R * C), raised_cells=raised)
    else:
        cfg.dirs = serpentine(R, C)
    if weighted:
        cfg.w = weights_f32(seed, (R, C))
    return cfg
