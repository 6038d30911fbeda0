"""World-size-2 gloo tests of the ROW_DIV multi-GPU host path (CPU only): nnz-balanced cuts,
band slicing, per-band plans, and the y all-gather reproduce the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

asp = pytest.importorskip("paper_2212_10432_b200")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import spmv as S
    import paper_2212_10432_b200 as asp
    from paper_2212_10432_b200 import dist as D
    coo = synth.random_powerlaw(997, 900, 4, 300, int_mode=True)
    x, _ = synth.vectors(coo.n, coo.m, 4, int_mode=True)
    A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
    r0, r1, Ab, cuts = D.band(A, rank, world)
    # each band gets its own plan (host-only here: the metadata path), then its y slice
    P = asp.Plan(Ab, Ab.random_graph(rank + 11), device=-1)
    assert P.info()["nnz_real"] == Ab.nnz
    rp, col, val = Ab.export_csr()
    y_loc, _ = S.spmv_csr(rp, col, val, x)
    y_full = torch.zeros(coo.m, dtype=torch.float64)
    D.allgather_rows(torch.from_numpy(y_loc.astype(np.float64)), y_full, cuts)
    nnz_band = torch.tensor([float(Ab.nnz)])
    dist.all_reduce(nnz_band)
    q.put((rank, y_full.numpy().copy(), cuts.tolist(), float(nnz_band.item())))
    dist.destroy_process_group()


def _halo_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import spmv as S
    import paper_2212_10432_b200 as asp
    from paper_2212_10432_b200 import dist as D
    c = synth.c5_band_csr(m=4096, nnz=4096 * 12, band=64, int_mode=True)
    x, _ = synth.vectors(c.n, c.m, 9, int_mode=True)
    A = asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)
    r0, r1, Ab, cuts = D.band(A, rank, world)
    rp, col, val = Ab.export_csr()
    y_loc, _ = S.spmv_csr(rp, col, val, x)
    spans = D.gather_spans(Ab.col_span())
    moves = D.halo_plan(spans, cuts)
    x_next = torch.full((c.m,), float("nan"), dtype=torch.float64)
    D.halo_exchange(torch.from_numpy(y_loc.astype(np.float64)), x_next, cuts, moves)
    lo, hi = spans[rank]
    halo_rows = sum(b - a for s, d, a, b in moves if d == rank)
    q.put((rank, lo, hi, x_next[lo:hi + 1].numpy().copy(), halo_rows))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    """NEXT-1: after the halo exchange every rank holds y on its band's whole column span,
    receiving only ~2*band rows instead of the full vector."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import spmv as S
    c = synth.c5_band_csr(m=4096, nnz=4096 * 12, band=64, int_mode=True)
    x, _ = synth.vectors(c.n, c.m, 9, int_mode=True)
    yref, _ = S.spmv_csr(c.row_ptr, c.col.astype(np.int64), c.val, x)
    for rank, lo, hi, got, halo in res:
        assert np.array_equal(got, yref[lo:hi + 1].astype(np.float64))
        assert halo <= 2 * 64 * (world - 1)        # only the band halo crosses ranks


@pytest.mark.parametrize("world", [2, 3])
def test_rowdiv_allgather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import spmv as S
    from oracle import builder_ref as B
    coo = synth.random_powerlaw(997, 900, 4, 300, int_mode=True)
    x, _ = synth.vectors(coo.n, coo.m, 4, int_mode=True)
    yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x)
    rp = np.zeros(coo.m + 1, np.int64)
    np.add.at(rp, coo.row + 1, 1)
    rp = np.cumsum(rp)
    for rank, y, cuts, nnz in res:
        assert cuts == B.row_cuts(rp, world).tolist()
        assert np.array_equal(y, yref.astype(np.float64))     # integer mode: bit-identical
        assert nnz == coo.nnz
