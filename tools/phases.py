"""Per-phase cycle breakdown of the block kernels (profiling build libfa_prof.so).

usage: FA_LIB=paper_1608_04431_b200/libfa_prof.so python tools/phases.py [cfg] [rows] [shapes]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1608_04431_b200 import fa  # noqa: E402

NAMES = ["stage dirs", "masks", "init w", "inject x", "walks", "write A"]
NAMES1 = ["stage z", "D8", "masks+init", "walks", "exit nodes", "perim walks"]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    rows = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
    shapes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["32x32"]
    cfg = inputs.make_config(name, rows, rows)
    lib = fa.load()
    dbg = lib.fa_debug_phase_clocks
    dbg.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 16)()
    src = torch.from_numpy(cfg.dem if cfg.dem is not None else cfg.dirs).cuda()
    w = torch.from_numpy(cfg.w).cuda() if cfg.w is not None else None
    kw = dict(dem=src) if cfg.dem is not None else dict(dirs=src)
    for shape in shapes:
        os.environ["FA_BLOCK"] = shape
        with fa.Context(0, tile=cfg.tile) as ctx:
            ctx.accumulate(w=w, atype=cfg.atype, **kw)
            dbg(buf, 1)
            ctx.accumulate(w=w, atype=cfg.atype, **kw)
            st = ctx.stats()
            dbg(buf, 1)
        nb = st["blocks"]
        for title, idx, names, ms in (("pass1", range(8, 14), NAMES1, st["ms_pass1"]),
                                      ("pass2", range(0, 6), NAMES, st["ms_pass2"])):
            tot = sum(buf[i] for i in idx) or 1
            print(f"{shape}: {title} {ms:.2f} ms, {nb} blocks; mean cycles/block per phase:")
            for i, n in zip(idx, names):
                print(f"   {n:12s} {buf[i] / nb:10.0f}  ({buf[i] / tot * 100:4.1f}%)")
        print(f"   walk loop: sum over warps of max lane iterations {buf[14]}, lane-steps {buf[15]}"
              f" -> lane efficiency {buf[15] / max(1, 32 * buf[14]) * 100:.1f}%")


if __name__ == "__main__":
    main()
