"""Multi-GPU plumbing (H7): row strips over the ranks of a torch.distributed
process group, one rank per GPU.

torch.distributed carries only the rendezvous (the 128-byte NCCL id is
broadcast from rank 0); the data path -- halo rows, the all-gather of tile
perimeter records, the status all-reduce -- runs inside libfa over NCCL
(fa_accumulate_dist), and the perimeter graph is solved redundantly on every
rank ("producer" work, replicated instead of centralised).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def strip_bounds(global_rows: int, tile_rows: int, rank: int, nranks: int) -> tuple[int, int]:
    """(row_begin, local_rows) of `rank`: whole tile rows, as even as possible,
    contiguous and ordered by rank (the layout fa_accumulate_dist requires)."""
    th = tile_rows if 0 < tile_rows < global_rows else global_rows
    n_tile_rows = (global_rows + th - 1) // th
    if nranks > n_tile_rows:
        raise ValueError(f"{nranks} ranks but only {n_tile_rows} tile rows")
    t0 = n_tile_rows * rank // nranks
    t1 = n_tile_rows * (rank + 1) // nranks
    r0 = t0 * th
    r1 = min(t1 * th, global_rows)
    return r0, r1 - r0


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0 creates the NCCL id (fa_nccl_unique_id); every rank returns it."""
    rank = dist.get_rank(group)
    obj = [None]
    if rank == 0:
        from . import fa

        obj[0] = fa.nccl_unique_id()
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def accumulate(ctx, global_rows: int, dem=None, dirs=None, w=None, atype: str = "u32",
               nodata: float = -9999.0, out=None, nccl_id: bytes | None = None):
    """Collective: this rank's strip (device tensors of the strip only) ->
    its strip of the global accumulation."""
    rank, nranks = dist.get_rank(), dist.get_world_size()
    src = dem if dem is not None else dirs
    r0, nrows = strip_bounds(global_rows, ctx.tile[0], rank, nranks)
    if src.shape[0] != nrows:
        raise ValueError(f"rank {rank}: strip has {src.shape[0]} rows, expected {nrows}")
    if nccl_id is None:
        nccl_id = broadcast_nccl_id()
    return ctx.accumulate_dist(nccl_id, rank, nranks, global_rows, r0, dem=dem, dirs=dirs, w=w,
                               atype=atype, nodata=nodata, out=out)


def local_device() -> torch.device:
    import os

    return torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
