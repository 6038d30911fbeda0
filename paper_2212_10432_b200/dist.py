"""Multi-GPU ROW_DIV plumbing: nnz-balanced bands
(as_dist_row_cuts, reading A35), the y all-gather (uneven bands -> one broadcast per rank
over the process group: NCCL on GPUs, gloo in the CPU tests), and the halo exchange that
replaces it for banded matrices.

The SpMV itself needs no communication when x is replicated; an exchange runs only when the
next iterate needs y as its x (north_star).  All-gather: every rank receives all of y
((m - rows_r)*sv bytes).  Halo: rank r receives only the part of y inside its band's column
span [lo_r, hi_r] that other ranks own (C5, band +-4096: 2*4096 rows per rank instead of
the whole vector).

The C-ABI path (as_dist_*, class Dist) runs the band SpMV and the exchange inside the library:
"nccl" = AllGatherV as grouped ncclBroadcasts, "peer" = one push kernel storing the band
into every peer's y_full over peer memory + release/acquire flags.  init_dist and
register_peers below only carry the 128-byte NCCL id and the 256-byte IPC blobs over the
torch process group."""
from __future__ import annotations


def band(matrix, rank: int, world: int):
    """(r0, r1, band_matrix, cuts) of this rank: nnz-balanced cuts of the row range."""
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


def halo_plan(spans, cuts):
    """spans[r] = (lo, hi) column span of rank r's band (hi < lo: empty).  Returns the list
    of transfers (src, dst, a, b): rank src sends y[a:b] (global rows it owns) to rank dst."""
    world = len(cuts) - 1
    moves = []
    for dst in range(world):
        lo, hi = spans[dst]
        if hi < lo:
            continue
        for src in range(world):
            if src == dst:
                continue
            a, b = max(lo, int(cuts[src])), min(hi + 1, int(cuts[src + 1]))
            if b > a:
                moves.append((src, dst, a, b))
    return moves


def gather_spans(span, group=None):
    """All ranks' (lo, hi) column spans (one small all-gather at plan time)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([span[0], span[1]], dtype=torch.int64, device=dev)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [(int(o[0]), int(o[1])) for o in out]


def halo_exchange(y_local, x_full, cuts, moves, group=None):
    """x_full[own rows] <- y_local, then point-to-point transfers of the halo: after the
    call x_full holds the new y on every row this rank's band references."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    x_full[int(cuts[rank]):int(cuts[rank + 1])] = y_local
    ops = []
    for src, dst, a, b in moves:
        if src == rank:
            ops.append(dist.P2POp(dist.isend, x_full[a:b].contiguous(), dst, group))
        elif dst == rank:
            ops.append(dist.P2POp(dist.irecv, x_full[a:b], src, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return x_full


def init_dist(rank: int, world: int, device: int, cuts, nccl: bool = True, group=None):
    """Dist of this rank: rank 0's ncclUniqueId is broadcast over the process group (nccl=False:
    peer-memory mode only); the row cuts are installed."""
    import torch.distributed as dist
    from . import Dist
    obj = [Dist.unique_id() if (nccl and rank == 0) else None]
    if nccl and world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    d = Dist(rank, world, device, obj[0] if nccl else None)
    d.set_cuts(cuts)
    return d


def register_peers(d, y_full, group=None):
    """All-gather the IPC blobs of every rank's y_full and map the peers' buffers (collective)."""
    import torch.distributed as dist
    handles = [None] * d.world
    dist.all_gather_object(handles, d.ipc_handle(y_full), group=group)
    d.open_peers(y_full, handles)
