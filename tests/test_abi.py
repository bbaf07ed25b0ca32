"""CPU-side checks of the boundary: libfa.so loads and exports every symbol
include/fa.h declares (no compute calls without a GPU); the oracle is not
reachable from the product package."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fa.h")).read()
    return sorted(set(re.findall(r"\b(fa_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1608_04431_b200 import build_native

    return build_native.build()


def test_header_symbols_exported(lib_path):
    declared = _declared()
    assert "fa_accumulate" in declared and "fa_accumulate_dist" in declared
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fa_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # nothing else leaks out of the library (hidden visibility)
    assert not [s for s in re.findall(r"\bT (\w+)", out) if not s.startswith("fa_")]


def test_library_loads_without_gpu(lib_path):
    lib = ctypes.CDLL(lib_path)
    for s in _declared():
        assert hasattr(lib, s)


def test_sm100a_cubin(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_has_no_oracle_or_cpu_fallback():
    pkg = os.path.join(ROOT, "paper_1608_04431_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle.c" not in txt, f


def test_binding_fails_loudly_when_library_missing(tmp_path, monkeypatch):
    from paper_1608_04431_b200 import fa

    monkeypatch.setattr(fa, "_lib", None)
    monkeypatch.setattr(fa, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        fa.load()
