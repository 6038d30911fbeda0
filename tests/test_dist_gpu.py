"""GPU tests of the C-ABI multi-GPU path (as_dist_*, as_spmv_dist) and the allocator hooks.

Only one GPU is available to the tests, so: NCCL AllGatherV at world 1; the peer-memory
push (AS_EXCH_PEER) with TWO processes sharing cuda:0 (CUDA IPC mappings work between
processes on one device; the push kernel, release/acquire flags and epoch logic are the
same as across NVLink peers).  Integer-exact mode: bit-identical to the oracle."""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import spmv as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
asp = pytest.importorskip("paper_2212_10432_b200")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _band_case():
    c = synth.c5_band_csr(m=6000, nnz=6000 * 12, band=96, int_mode=True)
    x, _ = synth.vectors(c.n, c.m, 5, int_mode=True)
    return c, x


def _oracle_power(c, x, k):
    v = x.astype(np.float64)
    for _ in range(k):
        v, _ = S.spmv_csr(c.row_ptr, c.col.astype(np.int64), c.val, v)
        v = v.astype(np.float64)
    return v


@pytest.mark.parametrize("exchange", ["none", "nccl", "peer"])
def test_dist_world1(exchange):
    c, x = _band_case()
    A = asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)
    P = asp.Plan(A, "COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED", device=0)
    d = asp.Dist(0, 1, 0, asp.Dist.unique_id() if exchange == "nccl" else None)
    d.set_cuts([0, c.m])
    xs = torch.from_numpy(x).cuda()
    y = torch.full((c.m,), 7.0, dtype=torch.float64, device="cuda")
    if exchange == "peer":
        d.open_peers(y, [d.ipc_handle(y)])
    d.spmv(P, 1.0, xs, 0.0, y, exchange)
    d.check()
    assert np.array_equal(y.cpu().numpy(), _oracle_power(c, x, 1))
    with pytest.raises(asp.AsError):
        d.spmv(P, 1.0, xs, 0.0, y[1:], "peer")            # unregistered buffer
    with pytest.raises(asp.AsError):
        d.spmv(P, 1.0, y, 0.0, y, "none")                 # x aliases y
    if exchange != "nccl":
        with pytest.raises(asp.AsError):
            d.spmv(P, 1.0, xs, 0.0, y, "nccl")            # no communicator
    d.close()


PEER_GRAPHS = {
    # straddling rows (atomics): separate push kernel after the SpMV
    "push": "COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    # single-writer (one STORE per row): peer stores fused into the SpMV epilogue
    "fused": "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "fused_warp": "COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED",
}


def _peer_worker(rank, world, port, iters, q, graph="push", no_fuse=False, halo=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if no_fuse:
        os.environ["AS_DIST_NO_FUSE"] = "1"
    import torch
    import torch.distributed as dist
    import paper_2212_10432_b200 as asp
    from paper_2212_10432_b200 import dist as D
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        c, x = _band_case()
        A = asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)
        r0, r1, Ab, cuts = D.band(A, rank, world)
        P = asp.Plan(Ab, PEER_GRAPHS[graph], device=0)
        assert P.info()["single_writer"] == (graph != "push"), P.info()
        d = D.init_dist(rank, world, 0, cuts, nccl=False)
        span = Ab.col_span()
        if halo:  # each peer receives only the rows of this band inside its column span
            d.set_windows(D.gather_spans(span))
        Y = [torch.from_numpy(x).cuda(), torch.full((c.m,), float("nan"), dtype=torch.float64, device="cuda")]
        for y in Y:
            D.register_peers(d, y)
        for k in range(iters):                                   # ping-pong: x_{k+1} = A x_k
            d.spmv(P, 1.0, Y[k % 2], 0.0, Y[(k + 1) % 2], "peer")
        d.check()
        q.put((rank, (Y[iters % 2].cpu().numpy().copy(), span, (r0, r1)), None))
        dist.barrier()
        d.close()
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("world,graph,no_fuse,halo", [(2, "push", False, False), (3, "push", False, False),
                                                     (2, "fused", False, False), (3, "fused", False, False),
                                                     (3, "fused_warp", False, False), (2, "fused", True, False),
                                                     (3, "push", False, True), (3, "fused", False, True),
                                                     (2, "fused_warp", False, True)])
def test_dist_peer_push_multiprocess(world, graph, no_fuse, halo):
    """x_{k+1} = A x_k over peer memory: separate push kernel, or (single-writer plans) peer
    stores fused into the SpMV epilogue; with halo windows each rank receives only the rows
    its band reads.  Bit-identical to the oracle on every row a rank owns or reads."""
    import torch.multiprocessing as mp
    iters = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, iters, q, graph, no_fuse, halo))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=240) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    c, x = _band_case()
    ref = _oracle_power(c, x, iters)
    for rank, out, err in res:
        assert err is None, (rank, err)
        y, (lo, hi), (r0, r1) = out
        if halo:  # rows outside the band and the window are never sent: compare the rest
            keep = np.zeros(c.m, bool)
            keep[r0:r1] = True
            keep[lo:hi + 1] = True
            assert 0 < keep.sum() < c.m
            y, ref_r = y[keep], ref[keep]
        else:
            ref_r = ref
        assert np.array_equal(y, ref_r), (rank, np.nonzero(y != ref_r)[0][:10])


def test_torch_allocator_hooks():
    """as_set_allocator: every plan allocation goes through the hooks and is released on
    destroy; results unchanged."""
    live = {}

    def alloc(n, s):
        p = torch.cuda.caching_allocator_alloc(n, torch.cuda.current_device(), s)
        live[p] = n
        return p

    def release(p, s):
        assert p in live
        del live[p]
        torch.cuda.caching_allocator_delete(p)

    asp.set_allocator(alloc, release)
    try:
        c, x = _band_case()
        A = asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)
        P = asp.Plan(A, "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
                        "GMEM_ATOM_RED", device=0)
        assert live and sum(live.values()) > c.nnz * 12
        y = np.zeros(c.m)
        P.spmv_host(1.0, x, 0.0, y)
        assert np.array_equal(y, _oracle_power(c, x, 1))
        del P, A  # the matrix owns the device copy of its CSR made by the on-device Designer
        assert not live
    finally:
        asp.set_allocator()
