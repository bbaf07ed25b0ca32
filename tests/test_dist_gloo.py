"""Multi-process (world size 2, gloo, CPU) tests of the row-strip protocol (H7).

No GPU here, so libfa's kernels cannot run; these tests cover the host logic
the multi-GPU path relies on, in real separate processes:
  * strip partition (whole tile rows, contiguous, ordered by rank);
  * the NCCL-id rendezvous through torch.distributed;
  * the decomposition itself: every rank computes its strip's tile perimeter
    records (F, A_T, L -- the paper's payload) with the CPU oracle,
    the records are all-gathered, every rank solves the producer's global
    graph redundantly and finalises its strip with the offsets
    injected (EVICT rerun); the gathered result must equal the
    oracle on the whole raster.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    port = _free_port()
    mp.start_processes(_entry, args=(fn, world, port, args), nprocs=world, join=True, start_method="spawn")


def _entry(rank, fn, world, port, args):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------- strip partition
def test_strip_bounds_cover_rows_in_order():
    from paper_1608_04431_b200.dist import strip_bounds

    for H, th, n in [(1000, 128, 2), (1000, 128, 8), (4096, 4096, 1), (32768, 4096, 8), (77, 10, 3)]:
        nxt = 0
        for r in range(n):
            r0, nr = strip_bounds(H, th, r, n)
            assert r0 == nxt and nr > 0 and r0 % th == 0
            nxt = r0 + nr
        assert nxt == H
    with pytest.raises(ValueError):
        strip_bounds(100, 50, 0, 3)


# ---------------------------------------------------------------- rendezvous
def _id_worker(rank, world):
    from paper_1608_04431_b200 import dist as fdist
    from paper_1608_04431_b200 import fa

    fa.nccl_unique_id = lambda: bytes(range(128))  # no GPU/NCCL needed for the mechanics
    nid = fdist.broadcast_nccl_id()
    assert nid == bytes(range(128)), rank


def test_nccl_id_broadcast_gloo():
    _run(_id_worker, 2)


# ---------------------------------------------------------------- protocol emulation
def _producer(H, W, th, tw, F, L, AT, base):
    """The producer's global graph over all tile perimeter slots:
    returns the offsets x (a_in) per slot.  Plain topological pass (small rasters)."""
    import oracle

    n = len(L)
    TC = (W + tw - 1) // tw
    parent = np.full(n, -1, np.int64)
    ext = np.zeros(n, bool)
    for t in range(len(base) - 1):
        ty, tx = divmod(t, TC)
        y0, x0 = ty * th, tx * tw
        h, w = min(th, H - y0), min(tw, W - x0)
        for p in range(base[t + 1] - base[t]):
            s = base[t] + p
            if L[s] == oracle.FLOW_EXTERNAL:
                ext[s] = True
                px, py = oracle.perim_xy(p, h, w)
                ny, nx = y0 + py + oracle.DY[F[s]], x0 + px + oracle.DX[F[s]]
                if 0 <= ny < H and 0 <= nx < W:
                    t2 = (ny // th) * TC + nx // tw
                    y2, x2 = (t2 // TC) * th, (t2 % TC) * tw
                    s2 = base[t2] + oracle.perim_index(nx - x2, ny - y2, min(th, H - y2), min(tw, W - x2))
                    if F[s2] != 255:
                        parent[s] = s2
            elif L[s] != oracle.FLOW_TERMINATES:
                parent[s] = base[t] + L[s]
    S = np.where(ext, AT, 0).astype(np.uint64)
    indeg = np.zeros(n, np.int64)
    for s in range(n):
        if parent[s] >= 0:
            indeg[parent[s]] += 1
    stack = [s for s in range(n) if indeg[s] == 0]
    while stack:
        s = stack.pop()
        p = parent[s]
        if p >= 0:
            S[p] += S[s]
            indeg[p] -= 1
            if indeg[p] == 0:
                stack.append(p)
    x = np.zeros(n, np.uint64)
    for s in range(n):
        if ext[s] and parent[s] >= 0:
            x[parent[s]] += S[s]
    return x


def _protocol_worker(rank, world, H, W, th, tw, seed):
    import inputs
    import oracle
    from paper_1608_04431_b200.dist import strip_bounds

    d = inputs.random_dirs(seed, H, W, p_nodata=0.1, p_noflow=0.02)  # every rank regenerates (seeded)
    w = inputs.weights_u32(seed, (H, W), 0, 9)
    base = oracle.tiles_perim_base(H, W, th, tw)
    TC = (W + tw - 1) // tw
    r0, nr = strip_bounds(H, th, rank, world)
    t0, t1 = (r0 // th) * TC, ((r0 + nr + th - 1) // th) * TC
    s0, s1 = base[t0], base[t1]
    # phase A on this strip only: records of its tiles (Alg. 1 + Alg. 2 per tile)
    strip = np.ascontiguousarray(d[r0:r0 + nr])
    sw = np.ascontiguousarray(w[r0:r0 + nr])
    Lloc = oracle.links(strip, th, tw)
    ATloc = oracle.tile_accumulate(strip, th, tw, sw)
    bl = oracle.tiles_perim_base(nr, W, th, tw)
    Floc = np.zeros(len(Lloc), np.uint8)
    ATs = np.zeros(len(Lloc), np.uint64)
    for t in range(len(bl) - 1):
        ty, tx = divmod(t, TC)
        y0, x0 = ty * th, tx * tw
        h, ww = min(th, nr - y0), min(tw, W - x0)
        for p in range(bl[t + 1] - bl[t]):
            px, py = oracle.perim_xy(p, h, ww)
            Floc[bl[t] + p] = strip[y0 + py, x0 + px]
            ATs[bl[t] + p] = ATloc[y0 + py, x0 + px]
    assert len(Lloc) == s1 - s0
    # C2: all-gather of the records (padded to the largest strip)
    n_max = torch.tensor([len(Lloc)])
    dist.all_reduce(n_max, op=dist.ReduceOp.MAX)
    pad = int(n_max)
    rec = torch.zeros((pad, 3), dtype=torch.int64)
    rec[:len(Lloc), 0] = torch.from_numpy(Lloc.astype(np.int64))
    rec[:len(Lloc), 1] = torch.from_numpy(Floc.astype(np.int64))
    rec[:len(Lloc), 2] = torch.from_numpy(ATs.astype(np.int64))
    parts = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(parts, rec)
    L = np.zeros(base[-1], np.uint32)
    F = np.zeros(base[-1], np.uint8)
    AT = np.zeros(base[-1], np.uint64)
    for q in range(world):
        q0, qn = strip_bounds(H, th, q, world)
        a0 = base[(q0 // th) * TC]
        a1 = base[((q0 + qn + th - 1) // th) * TC]
        L[a0:a1] = parts[q][:a1 - a0, 0].numpy().astype(np.uint32)
        F[a0:a1] = parts[q][:a1 - a0, 1].numpy().astype(np.uint8)
        AT[a0:a1] = parts[q][:a1 - a0, 2].numpy().astype(np.uint64)
    # phase B: redundant producer solve, then finalise this strip (EVICT rerun with w + x)
    x = _producer(H, W, th, tw, F, L, AT, base)
    inj = sw.astype(np.uint64)
    for t in range(len(bl) - 1):
        ty, tx = divmod(t, TC)
        y0, x0 = ty * th, tx * tw
        h, ww = min(th, nr - y0), min(tw, W - x0)
        for p in range(bl[t + 1] - bl[t]):
            px, py = oracle.perim_xy(p, h, ww)
            inj[y0 + py, x0 + px] += x[s0 + bl[t] + p]
    A = oracle.tile_accumulate(strip, th, tw, inj.astype(np.uint32))
    out = [torch.zeros((pad * 0 + H, W), dtype=torch.int64) for _ in range(world)] if rank == 0 else None
    full = torch.zeros((H, W), dtype=torch.int64)
    full[r0:r0 + nr] = torch.from_numpy(A.astype(np.int64))
    dist.all_reduce(full)  # strips are disjoint: the sum assembles the raster
    if rank == 0:
        exp = oracle.accumulate(d, w).astype(np.int64)
        got = full.numpy()
        data = d != 255
        assert (got[data] == exp[data]).all()
    del out


@pytest.mark.parametrize("H,W,th,tw,seed", [(60, 50, 16, 16, 1), (45, 37, 10, 13, 2)])
def test_strip_protocol_equals_oracle_gloo(H, W, th, tw, seed):
    _run(_protocol_worker, 2, H, W, th, tw, seed)
