"""Multi-GPU ROW_DIV plumbing: nnz-balanced bands (as_dist_row_cuts, reading
A35) and the y all-gather (uneven bands -> one broadcast per rank over the process group:
NCCL on GPUs, gloo in the CPU tests).  The SpMV itself needs no communication when x is
replicated; the gather runs only when the next iterate needs the whole y (north_star)."""
from __future__ import annotations


def band(matrix, rank: int, world: int):
    """(r0, r1, band_matrix) of this rank: nnz-balanced cuts of the row range."""
    cuts = matrix.row_cuts(world)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    return r0, r1, (matrix if world == 1 else matrix.row_slice(r0, r1)), cuts


def allgather_rows(y_local, y_full, cuts, group=None):
    """In-place AllGatherV: y_full[cuts[r]:cuts[r+1]] <- rank r's y_local on every rank."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    y_full[int(cuts[rank]):int(cuts[rank + 1])] = y_local
    for r in range(world):
        a, b = int(cuts[r]), int(cuts[r + 1])
        if b > a:
            dist.broadcast(y_full[a:b], src=r, group=group)
    return y_full
