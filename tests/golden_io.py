"""Parsers for the paper-cited text fixtures under tests/golden/."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_TOK = {".": 255, "o": 0}


def _dir_tok(t):
    return _TOK[t] if t in _TOK else int(t)


def load_fig2():
    """tests/golden/fig2_exit_100.txt -> dict(dirs, w, tile, expect_A, expect_AT, expect_X)."""
    lines = [ln.strip() for ln in open(os.path.join(GOLDEN, "fig2_exit_100.txt")) if ln.strip()
             and not ln.startswith("#")]
    hdr = lines[0].split()
    H, W, th, tw = int(hdr[1]), int(hdr[3]), int(hdr[5]), int(hdr[6])
    i = lines.index("dirs") + 1
    dirs = np.array([[_dir_tok(t) for t in lines[i + r].split()] for r in range(H)], np.uint8)
    i = lines.index("weights") + 1
    w = np.array([[int(t) for t in lines[i + r].split()] for r in range(H)], np.uint32)
    out = dict(dirs=dirs, w=w, tile=(th, tw), expect_A=[], expect_AT=[], expect_X=[])
    for ln in lines:
        p = ln.split()
        if p[0] in ("expect_A", "expect_AT", "expect_X"):
            out[p[0]].append((int(p[1]), int(p[2]), int(p[3])))
    return out


def load_spec_examples():
    """tests/golden/spec_examples.txt -> list of (name, dirs, expected A with NoData=None mask)."""
    lines = [ln.rstrip() for ln in open(os.path.join(GOLDEN, "spec_examples.txt"))
             if ln.strip() and not ln.startswith("#")]
    cases, i = [], 0
    while i < len(lines):
        _, name, H, W = lines[i].split()
        H, W = int(H), int(W)
        dirs = np.array([[_dir_tok(t) for t in lines[i + 1 + r].split()] for r in range(H)], np.uint8)
        assert lines[i + 1 + H] == "A"
        exp = [[None if t == "." else int(t) for t in lines[i + 2 + H + r].split()] for r in range(H)]
        cases.append((name, dirs, exp))
        i += 2 + 2 * H
    return cases


def load_perimeter_sizes():
    rows = []
    for ln in open(os.path.join(GOLDEN, "perimeter_sizes.txt")):
        if ln.startswith("#") or not ln.strip():
            continue
        p = ln.split()
        rows.append(tuple(int(v) for v in p[:5]))
    return rows
