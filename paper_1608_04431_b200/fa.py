"""Thin ctypes binding over libfa.so (include/fa.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; torch is
used for device memory, streams and process groups.  There is no CPU
fallback: importing this module on a box without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FA_LIB") or os.path.join(_HERE, "libfa.so")  # FA_LIB: tuning builds only

FA_OK, FA_E_ARG, FA_E_DIRCODE, FA_E_CYCLE, FA_E_OVERFLOW, FA_E_NOMEM, FA_E_CUDA, FA_E_NCCL, FA_E_STATE = range(9)
STATUS_NAMES = {0: "FA_OK", 1: "FA_E_ARG", 2: "FA_E_DIRCODE", 3: "FA_E_CYCLE", 4: "FA_E_OVERFLOW",
                5: "FA_E_NOMEM", 6: "FA_E_CUDA", 7: "FA_E_NCCL", 8: "FA_E_STATE"}
W_NONE, W_U32, W_F32 = 0, 1, 2
A_U32, A_U64, A_F64 = 0, 1, 2
ATYPES = {"u32": A_U32, "u64": A_U64, "f64": A_F64}
TORCH_ACC = {A_U32: torch.uint32, A_U64: torch.uint64, A_F64: torch.float64}
FLOW_EXTERNAL = 0xFFFFFFFE
FLOW_TERMINATES = 0xFFFFFFFF

EXPORTS = ["fa_create", "fa_destroy", "fa_last_error", "fa_flowdirs", "fa_accumulate",
           "fa_accumulate_strips", "fa_perimeter_slots", "fa_perimeter_records", "fa_nccl_unique_id",
           "fa_accumulate_dist", "fa_get_stats", "fa_accumulate_streamed",
           "fa_accumulate_absorb", "fa_accumulate_absorb_dist", "fa_accumulate_absorb_streamed", "fa_fill",
           "fa_set_option", "fa_get_option", "fa_accumulate_dist_loopback", "fa_accumulate_batch"]
# context options (fa.h fa_option); values: RETAIN / EVICT, D8_SPLIT / D8_FUSED, block rows 32 / 16,
# graph walk cap, fill tile 32 / 64
OPT_RETENTION, OPT_D8, OPT_BLOCK_ROWS, OPT_WALK_CAP, OPT_FILL_TILE, OPT_VALUES, OPT_GRAPH, OPT_DIST_RECORDS = range(1, 9)
RETAIN, EVICT = 0, 1
D8_SPLIT, D8_FUSED = 0, 1
OPTIONS = {"retention": OPT_RETENTION, "d8": OPT_D8, "block_rows": OPT_BLOCK_ROWS, "walk_cap": OPT_WALK_CAP,
           "fill_tile": OPT_FILL_TILE, "values": OPT_VALUES, "graph": OPT_GRAPH, "dist_records": OPT_DIST_RECORDS}
VALUES_L2, VALUES_SMEM = 0, 1
GRAPH_HOST, GRAPH_DEVICE, GRAPH_AUTO = 0, 1, 2
DIST_TILES, DIST_STRIPS = 0, 1
OPTION_VALUES = {"retain": RETAIN, "evict": EVICT, "split": D8_SPLIT, "fused": D8_FUSED, "l2": VALUES_L2,
                 "smem": VALUES_SMEM, "host": GRAPH_HOST, "device": GRAPH_DEVICE, "auto": GRAPH_AUTO, "tiles": DIST_TILES,
                 "strips": DIST_STRIPS}


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for fa_accumulate_dist (rank 0 creates, all ranks receive)."""
    lib = load()
    buf = ctypes.create_string_buffer(128)
    st = lib.fa_nccl_unique_id(buf)
    if st != FA_OK:
        raise FaError(st, "fa_nccl_unique_id failed")
    return buf.raw


class FaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Stats(ctypes.Structure):
    _fields_ = [("ms_total", ctypes.c_double), ("ms_pass1", ctypes.c_double), ("ms_graph", ctypes.c_double),
                ("ms_pass2", ctypes.c_double), ("ms_exchange", ctypes.c_double),
                ("cells", ctypes.c_int64), ("blocks", ctypes.c_int64), ("graph_nodes", ctypes.c_int64),
                ("tile_nodes", ctypes.c_int64), ("peel_rounds", ctypes.c_int64),
                ("contract_levels", ctypes.c_int64), ("jump_rounds", ctypes.c_int64),
                ("bytes_exchanged", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("ms_d8", ctypes.c_double), ("ms_block", ctypes.c_double), ("ms_compute", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load libfa.so (must have been built: __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libfa.so not built at {LIB_PATH}; run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_float
    lib.fa_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, P, I, I]
    lib.fa_destroy.argtypes = [P]
    lib.fa_last_error.argtypes = [P]
    lib.fa_last_error.restype = ctypes.c_char_p
    lib.fa_flowdirs.argtypes = [P, P, I, I, F, P]
    lib.fa_accumulate.argtypes = [P, I, I, P, F, P, P, ctypes.c_int, P, ctypes.c_int]
    lib.fa_accumulate_strips.argtypes = [P, ctypes.c_int, I, I, P, F, P, P, ctypes.c_int, P, ctypes.c_int]
    lib.fa_accumulate_streamed.argtypes = [P, I, I, P, F, P, P, ctypes.c_int, P, ctypes.c_int, I]
    lib.fa_accumulate_absorb.argtypes = [P, ctypes.c_int, I, I, P, F, P, P, ctypes.c_int, P, P]
    lib.fa_fill.argtypes = [P, P, I, I, F, P]
    lib.fa_accumulate_absorb_streamed.argtypes = [P, I, I, P, F, P, P, ctypes.c_int, P, P, I]
    lib.fa_accumulate_absorb_dist.argtypes = [P, P, ctypes.c_int, ctypes.c_int, I, I, I, I, P, F, P, P,
                                              ctypes.c_int, P, P]
    lib.fa_perimeter_slots.argtypes = [P, I, I]
    lib.fa_perimeter_slots.restype = I
    lib.fa_perimeter_records.argtypes = [P, I, I, P, F, P, P, ctypes.c_int, ctypes.c_int, P, P, P, P]
    lib.fa_nccl_unique_id.argtypes = [P]
    lib.fa_accumulate_dist.argtypes = [P, P, ctypes.c_int, ctypes.c_int, I, I, I, I, P, F, P, P,
                                       ctypes.c_int, P, ctypes.c_int]
    lib.fa_get_stats.argtypes = [P, P, I]
    lib.fa_set_option.argtypes = [P, ctypes.c_int, I]
    lib.fa_get_option.argtypes = [P, ctypes.c_int, ctypes.POINTER(I)]
    PP = ctypes.POINTER(P)
    lib.fa_accumulate_dist_loopback.argtypes = [PP, ctypes.c_int, I, I, ctypes.POINTER(I), ctypes.POINTER(I), PP, F,
                                                PP, PP, ctypes.c_int, PP, PP, ctypes.c_int]
    lib.fa_accumulate_batch.argtypes = [P, ctypes.c_int, I, I, PP, F, PP, PP, ctypes.c_int, PP, ctypes.c_int]
    for fn in EXPORTS:
        if fn not in ("fa_last_error", "fa_perimeter_slots"):
            getattr(lib, fn).restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return ctypes.c_void_p(t.data_ptr())
    import numpy as np

    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return t.ctypes.data_as(ctypes.c_void_p)
    raise TypeError(type(t))


def _dtype_name(t) -> str:
    return str(t.dtype).replace("torch.", "")


def _check(t, name: str, dtypes: tuple, shape=None):
    """Reject a wrong dtype or shape before the C call (the library reads raw
    pointers: a float64 DEM or a short `out` would be misread / overrun)."""
    if t is None:
        return
    dn = _dtype_name(t)
    if dn not in dtypes:
        raise TypeError(f"{name} must be {' or '.join(dtypes)}, got {dn}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


ACC_DTYPE = {A_U32: "uint32", A_U64: "uint64", A_F64: "float64"}


def _check_inputs(dem, dirs, w, shape, alpha=None):
    # "exactly one of dem / dirs" is the library's own FA_E_ARG check (tested through the ABI)
    if len(shape) != 2:
        raise ValueError("rasters are 2-D (rows, cols)")
    _check(dem, "dem", ("float32",), shape)
    _check(dirs, "dirs", ("uint8",), shape)
    _check(w, "w", ("uint32", "float32"), shape)
    _check(alpha, "alpha", ("float32",), shape)


def _wtype(w):
    if w is None:
        return W_NONE
    dn = _dtype_name(w)
    if dn == "uint32":
        return W_U32
    if dn == "float32":
        return W_F32
    raise TypeError(f"weights must be uint32 or float32, got {dn}")


class Context:
    """One fa_ctx: bound to a device and a CUDA stream, with a tile size."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None,
                 tile: tuple[int, int] = (0, 0)):
        self.lib = load()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.tile = tuple(tile)
        h = ctypes.c_void_p()
        st = self.lib.fa_create(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream),
                                int(tile[0]), int(tile[1]))
        if st != FA_OK:
            raise FaError(st, "fa_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.fa_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st):
        if st != FA_OK:
            raise FaError(st, self.lib.fa_last_error(self.h).decode())

    def stats(self) -> dict:
        s = Stats()
        self._check(self.lib.fa_get_stats(self.h, ctypes.byref(s), ctypes.sizeof(s)))
        return s.as_dict()

    def set_option(self, name: str, value) -> None:
        """fa_set_option: retention 'retain'|'evict', d8 'split'|'fused', block_rows 32|16,
        walk_cap int, fill_tile 32|64."""
        v = OPTION_VALUES.get(value, value) if isinstance(value, str) else value
        self._check(self.lib.fa_set_option(self.h, OPTIONS[name], int(v)))

    def get_option(self, name: str) -> int:
        v = ctypes.c_int64()
        self._check(self.lib.fa_get_option(self.h, OPTIONS[name], ctypes.byref(v)))
        return int(v.value)

    # ---------------------------------------------------------------- H1
    def flowdirs(self, dem, nodata: float = -9999.0, out=None):
        rows, cols = dem.shape
        _check(dem, "dem", ("float32",))
        _check(out, "out", ("uint8",), (rows, cols))
        if out is None:
            out = torch.empty((rows, cols), dtype=torch.uint8, device=dem.device) if isinstance(
                dem, torch.Tensor) else __import__("numpy").empty((rows, cols), "uint8")
        self._check(self.lib.fa_flowdirs(self.h, _ptr(dem), rows, cols, float(nodata), _ptr(out)))
        return out

    # ---------------------------------------------------------------- N4
    def fill(self, dem, nodata: float = -9999.0, out=None):
        """Depression filling (Priority-Flood+epsilon surface) of a f32 DEM; device or host."""
        rows, cols = dem.shape
        _check(dem, "dem", ("float32",))
        _check(out, "out", ("float32",), (rows, cols))
        if out is None:
            out = torch.empty_like(dem) if isinstance(dem, torch.Tensor) else __import__("numpy").empty_like(dem)
        self._check(self.lib.fa_fill(self.h, _ptr(dem), rows, cols, float(nodata), _ptr(out)))
        return out

    # ---------------------------------------------------------------- H1-H6
    def accumulate(self, dem=None, dirs=None, w=None, atype: str = "u32", nodata: float = -9999.0,
                   out=None):
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        _check_inputs(dem, dirs, w, (rows, cols))
        a = ATYPES[atype]
        _check(out, "out", (ACC_DTYPE[a],), (rows, cols))
        if out is None:
            if isinstance(src, torch.Tensor):
                out = torch.empty((rows, cols), dtype=TORCH_ACC[a], device=src.device)
            else:
                import numpy as np

                out = np.empty((rows, cols), {A_U32: np.uint32, A_U64: np.uint64, A_F64: np.float64}[a])
        self._check(self.lib.fa_accumulate(self.h, rows, cols, _ptr(dem), float(nodata), _ptr(dirs),
                                           _ptr(w), _wtype(w), _ptr(out), a))
        return out

    def accumulate_strips(self, nstrips: int, dem=None, dirs=None, w=None, atype: str = "u32",
                          nodata: float = -9999.0, out=None):
        """The multi-GPU strip pipeline (H4-H7) run as `nstrips` strips on this device."""
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        _check_inputs(dem, dirs, w, (rows, cols))
        a = ATYPES[atype]
        _check(out, "out", (ACC_DTYPE[a],), (rows, cols))
        if out is None:
            out = torch.empty((rows, cols), dtype=TORCH_ACC[a], device=src.device)
        self._check(self.lib.fa_accumulate_strips(self.h, int(nstrips), rows, cols, _ptr(dem), float(nodata),
                                                  _ptr(dirs), _ptr(w), _wtype(w), _ptr(out), a))
        return out

    def accumulate_batch(self, dems=None, dirs=None, ws=None, atype: str = "u32", nodata: float = -9999.0,
                         outs=None):
        """fa_accumulate_batch: a list of independent host rasters (numpy, or CPU / pinned
        torch tensors) of one shape; uploads, device work and downloads of neighbouring
        rasters overlap.  Returns the list of outputs (host, pinned when the inputs are)."""
        srcs = dems if dems is not None else dirs
        if srcs is None or (dems is not None and dirs is not None):
            raise ValueError("give exactly one of dems, dirs")
        n = len(srcs)
        if ws is not None and len(ws) != n:
            raise ValueError("ws must have one entry per raster")
        if n == 0:
            return []
        rows, cols = srcs[0].shape
        for i in range(n):
            _check_inputs(dems[i] if dems is not None else None, dirs[i] if dirs is not None else None,
                          ws[i] if ws is not None else None, (rows, cols))
        wt = _wtype(ws[0]) if ws is not None else W_NONE
        if ws is not None and any(_wtype(x) != wt for x in ws):
            raise TypeError("all weights must have one dtype")
        a = ATYPES[atype]
        if outs is None:
            outs = []
            for s in srcs:
                if isinstance(s, torch.Tensor):
                    outs.append(torch.empty((rows, cols), dtype=TORCH_ACC[a], pin_memory=s.is_pinned()))
                else:
                    import numpy as np

                    outs.append(np.empty((rows, cols), {A_U32: np.uint32, A_U64: np.uint64, A_F64: np.float64}[a]))
        if len(outs) != n:
            raise ValueError("outs must have one entry per raster")
        for o in outs:
            _check(o, "out", (ACC_DTYPE[a],), (rows, cols))

        def arr(lst):
            if lst is None:
                return None
            return (ctypes.c_void_p * n)(*[_ptr(x) for x in lst])

        self._check(self.lib.fa_accumulate_batch(self.h, n, rows, cols, arr(dems), float(nodata), arr(dirs),
                                                 arr(ws), wt, arr(outs), a))
        return outs

    def accumulate_streamed(self, dem=None, dirs=None, w=None, atype: str = "u32", nodata: float = -9999.0,
                            strip_rows: int = 0, out=None):
        """Out-of-core accumulation (N2): host arrays in and out (numpy, or CPU / pinned torch
        tensors); only `strip_rows`-row strips are resident on the device (0: sized from free
        device memory)."""
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        _check_inputs(dem, dirs, w, (rows, cols))
        a = ATYPES[atype]
        _check(out, "out", (ACC_DTYPE[a],), (rows, cols))
        if out is None:
            if isinstance(src, torch.Tensor):
                out = torch.empty((rows, cols), dtype=TORCH_ACC[a], pin_memory=src.is_pinned())
            else:
                import numpy as np

                out = np.empty((rows, cols), {A_U32: np.uint32, A_U64: np.uint64, A_F64: np.float64}[a])
        self._check(self.lib.fa_accumulate_streamed(self.h, rows, cols, _ptr(dem), float(nodata), _ptr(dirs),
                                                    _ptr(w), _wtype(w), _ptr(out), a, int(strip_rows)))
        return out

    def accumulate_absorb(self, alpha, dem=None, dirs=None, w=None, nodata: float = -9999.0, out=None,
                          nstrips: int = 1):
        """Absorption (N3): A(p) = w(p) + sum alpha(n) A(n) over donors n; f64 output.
        alpha: f32 raster in [0,1] (device or host, like the other inputs)."""
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        _check_inputs(dem, dirs, w, (rows, cols), alpha)
        _check(out, "out", ("float64",), (rows, cols))
        if out is None:
            if isinstance(src, torch.Tensor):
                out = torch.empty((rows, cols), dtype=torch.float64, device=src.device)
            else:
                import numpy as np

                out = np.empty((rows, cols), np.float64)
        self._check(self.lib.fa_accumulate_absorb(self.h, int(nstrips), rows, cols, _ptr(dem), float(nodata),
                                                  _ptr(dirs),
                                                  _ptr(w), _wtype(w), _ptr(alpha), _ptr(out)))
        return out

    def accumulate_dist(self, nccl_id: bytes, rank: int, nranks: int, global_rows: int, row_begin: int,
                        dem=None, dirs=None, w=None, atype: str = "u32", nodata: float = -9999.0, out=None):
        """One rank's strip of the multi-GPU accumulation (collective over all ranks)."""
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        _check_inputs(dem, dirs, w, (rows, cols))
        a = ATYPES[atype]
        _check(out, "out", (ACC_DTYPE[a],), (rows, cols))
        if out is None:
            out = torch.empty((rows, cols), dtype=TORCH_ACC[a], device=src.device)
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        self._check(self.lib.fa_accumulate_dist(self.h, buf, rank, nranks, global_rows, cols, row_begin, rows,
                                                _ptr(dem), float(nodata), _ptr(dirs), _ptr(w), _wtype(w),
                                                _ptr(out), a))
        return out

    def accumulate_absorb_streamed(self, alpha, dem=None, dirs=None, w=None, nodata: float = -9999.0,
                                   strip_rows: int = 0, out=None):
        """Out-of-core absorption: host arrays in and out (numpy / CPU or pinned tensors)."""
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        _check_inputs(dem, dirs, w, (rows, cols), alpha)
        _check(out, "out", ("float64",), (rows, cols))
        if out is None:
            if isinstance(src, torch.Tensor):
                out = torch.empty((rows, cols), dtype=torch.float64, pin_memory=src.is_pinned())
            else:
                import numpy as np

                out = np.empty((rows, cols), np.float64)
        self._check(self.lib.fa_accumulate_absorb_streamed(self.h, rows, cols, _ptr(dem), float(nodata), _ptr(dirs),
                                                           _ptr(w), _wtype(w), _ptr(alpha), _ptr(out),
                                                           int(strip_rows)))
        return out

    def accumulate_absorb_dist(self, nccl_id: bytes, rank: int, nranks: int, global_rows: int, row_begin: int,
                               alpha, dem=None, dirs=None, w=None, nodata: float = -9999.0, out=None):
        """One rank's strip of the multi-GPU absorption accumulation (collective; f64 output)."""
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        _check_inputs(dem, dirs, w, (rows, cols), alpha)
        _check(out, "out", ("float64",), (rows, cols))
        if out is None:
            out = torch.empty((rows, cols), dtype=torch.float64, device=src.device)
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        self._check(self.lib.fa_accumulate_absorb_dist(self.h, buf, rank, nranks, global_rows, cols, row_begin,
                                                       rows, _ptr(dem), float(nodata), _ptr(dirs), _ptr(w),
                                                       _wtype(w), _ptr(alpha), _ptr(out)))
        return out

    def perimeter_slots(self, rows: int, cols: int) -> int:
        return int(self.lib.fa_perimeter_slots(self.h, rows, cols))

    def perimeter_records(self, dem=None, dirs=None, w=None, atype: str = "u32", nodata: float = -9999.0):
        """(links u32, A_T, x, A) per tile perimeter slot (H4/H5), as device tensors."""
        src = dem if dem is not None else dirs
        rows, cols = src.shape
        a = ATYPES[atype]
        ns = self.perimeter_slots(rows, cols)
        dev = src.device
        links = torch.empty(ns, dtype=torch.uint32, device=dev)
        at = torch.empty(ns, dtype=TORCH_ACC[a], device=dev)
        xo = torch.empty(ns, dtype=TORCH_ACC[a], device=dev)
        acc = torch.empty((rows, cols), dtype=TORCH_ACC[a], device=dev)
        self._check(self.lib.fa_perimeter_records(self.h, rows, cols, _ptr(dem), float(nodata), _ptr(dirs),
                                                  _ptr(w), _wtype(w), a, _ptr(links), _ptr(at), _ptr(xo),
                                                  _ptr(acc)))
        return links, at, xo, acc


def accumulate_dist_loopback(ctxs, global_rows: int, row_begin, dem=None, dirs=None, w=None, alpha=None,
                             atype: str = "u32", nodata: float = -9999.0, out=None):
    """fa_accumulate_dist_loopback: the multi-GPU path with len(ctxs) ranks run as
    threads inside one call (one Context per rank, each with its own stream),
    exchanging through device copies instead of NCCL.  dem / dirs / w / alpha /
    out are per-rank lists of the ranks' strips (device tensors) or None;
    row_begin is the per-rank list of first global rows.  Returns the list of
    per-rank accumulation strips."""
    lib = load()
    n = len(ctxs)
    per = [x for x in (dem, dirs) if x is not None][0]
    if alpha is not None:
        atype = "f64"
    a = ATYPES[atype]
    rows = [int(t.shape[0]) for t in per]
    cols = int(per[0].shape[1])
    for q in range(n):
        _check_inputs(dem[q] if dem else None, dirs[q] if dirs else None, w[q] if w else None, (rows[q], cols),
                      alpha[q] if alpha else None)
    if out is None:
        out = [torch.empty((rows[q], cols), dtype=TORCH_ACC[a], device=per[q].device) for q in range(n)]
    for q in range(n):
        _check(out[q], "out", (ACC_DTYPE[a],), (rows[q], cols))
    P = ctypes.c_void_p

    def arr(lst):
        if lst is None:
            return None
        return (P * n)(*[P(t.data_ptr()) if t is not None else None for t in lst])

    for lst in (dem, dirs, w, alpha, out):
        if lst is not None:
            for t in lst:
                if t is not None and not t.is_contiguous():
                    raise ValueError("tensors must be contiguous")
    hs = (P * n)(*[c.h for c in ctxs])
    I64 = ctypes.c_int64 * n
    st = lib.fa_accumulate_dist_loopback(hs, n, int(global_rows), cols, I64(*[int(r) for r in row_begin]),
                                         I64(*rows), arr(dem), float(nodata), arr(dirs), arr(w),
                                         _wtype(w[0] if w else None), arr(alpha), arr(out), a)
    if st != FA_OK:
        msgs = [c.lib.fa_last_error(c.h).decode() for c in ctxs]
        raise FaError(st, "; ".join(f"rank {q}: {m}" for q, m in enumerate(msgs) if m))
    return out
