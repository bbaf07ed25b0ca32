"""Build libfa.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

Flags: -gencode arch=compute_100a,code=sm_100a, -lineinfo for ncu source
mapping, and IEEE-exact float semantics (no --use_fast_math; -ftz=false,
-prec-div=true, -prec-sqrt=true) so the D8 stencil matches the oracle bit for
bit.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfa.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared",
    "-Xptxas", "-v",
]


def nccl_include() -> str:
    """The torch-bundled NCCL headers (libnccl itself is dlopen'ed at run time,
    so the process never holds two NCCL copies)."""
    import nvidia.nccl

    return os.path.join(list(nvidia.nccl.__path__)[0], "include")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "fa.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """variant "prof": -DFA_PHASE_CLOCKS per-phase cycle counters -> libfa_prof.so;
    other variants build libfa_<variant>.so with the given -D defines (tuning
    builds loaded through FA_LIB; never the product library)."""
    lib = LIB if not variant else os.path.join(HERE, f"libfa_{variant}.so")
    if not force and not variant and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    extra = (["-DFA_PHASE_CLOCKS"] if variant == "prof" else []) + [f"-D{d}" for d in defines]
    inc = ["-I", os.path.join(ROOT, "include"), "-I", nccl_include()]
    import shutil
    import tempfile

    # objects in a scratch directory: only the linked .so stays in the tree
    # (it travels to the GPU box; 300 MB of objects would too)
    objdir = tempfile.mkdtemp(prefix="libfa_build_")
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        r = subprocess.run([nvcc, *compile_flags, *extra, *inc, "-c", src, "-o", obj],
                           capture_output=True, text=True)
        return src, obj, r

    # one nvcc per translation unit, in parallel (the units only call each
    # other's host-side launchers, so no device link step is needed)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    log = "".join(r.stdout + r.stderr for _, _, r in results)
    bad = [src for src, _, r in results if r.returncode != 0]
    if bad:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed building libfa.so: " + ", ".join(bad))
    res = subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                          *[o for _, o, _ in results], "-o", lib + ".tmp", "-ldl"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libfa.so")
    os.replace(lib + ".tmp", lib)
    shutil.rmtree(objdir, ignore_errors=True)
    res.stdout, res.stderr = log, ""
    if variant:
        return lib
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(res.stdout + res.stderr)
    if verbose:
        sys.stdout.write(res.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
