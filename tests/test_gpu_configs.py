"""GPU parity on the BASELINE configs C3 / C4 / C5 (shape-preserving scaled instances by
default; full size with AS_FULL=1), their named graphs, searched graphs, the committed bench
winners at full size (C2, C3, C4; C5 at 1/4 scale), and the ROW_DIV multi-band (multi-GPU)
decomposition emulated on one device.  EVERY row is checked against the long-double oracle
(all host cores) per DESIGN.md §3 O2; integer-exact variants must be bit-identical."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import spmv as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
asp = pytest.importorskip("paper_2212_10432_b200")

FULL = os.environ.get("AS_FULL") == "1"


def _mat(c):
    return asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)


def _sample_rows(m, seed=0, row_ptr=None):
    """first/last 4096 rows, 20,000 random rows, and the 256 longest rows (hub rows carry
    the longest accumulation / atomic chains)."""
    parts = [np.arange(0, min(m, 4096)), np.arange(max(0, m - 4096), m),
             np.random.default_rng(seed).integers(0, m, 20000)]
    if row_ptr is not None:
        parts.append(np.argsort(-np.diff(row_ptr), kind="stable")[:256])
    return np.unique(np.concatenate(parts))


def run_sampled(c, P, alpha, beta, seed, int_mode=False):
    """Every row of y against the oracle (the name is historical: round 1 sampled rows)."""
    x, y0 = synth.vectors(c.n, c.m, seed, c.val.dtype, int_mode)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
    P.spmv(alpha, dx, beta, dy)
    torch.cuda.synchronize()
    y = dy.cpu().numpy()
    yref, bound = S.spmv_csr(c.row_ptr, c.col, c.val.astype(np.float64), x.astype(np.float64), alpha, beta,
                             y0.astype(np.float64), nthreads=os.cpu_count() or 1)
    if int_mode:
        bad = np.nonzero(y.astype(np.float64) != yref.astype(np.float64))[0]
        assert bad.shape[0] == 0, (bad[:10], y[bad[:10]], yref[bad[:10]])
    ok, ratio = S.check(y, yref, bound, c.val.dtype)
    assert ok, ratio
    return y


@pytest.fixture(scope="module")
def c3():
    return synth.c3_rmat_csr() if FULL else synth.c3_rmat_csr(scale=20, nnz=1 << 24)


@pytest.fixture(scope="module")
def c4():
    if FULL:
        return synth.c4_blockdense_csr()
    return synth.c4_blockdense_csr(m=1 << 20, b=64, n_tiles=3072, nnz=25_000_000)


@pytest.fixture(scope="module")
def c5():
    return synth.c5_band_csr() if FULL else synth.c5_band_csr(m=1 << 22, nnz=1 << 26)


C3_GRAPHS = [
    # SURVEY §8(d) C3 seed graph; hub rows (> 2048 nnz) are cut into 2048-nonzero warp
    # chunks inside one-row BMTBs (a top-level BMTB_NNZ_BLOCK would mix rows, failing P1)
    "BIN(t=[32,2048]) { COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED"
    " | COMPRESS; BMTB_NNZ_BLOCK(2048); SHMEM_OFFSET_RED; GMEM_ATOM_RED"
    " | COMPRESS; BMTB_ROW_BLOCK(1); BMW_NNZ_BLOCK(2048); WARP_TOTAL_RED; GMEM_ATOM_RED }",
    "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,1); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL,1); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "SORT; COMPRESS; BMTB_ROW_BLOCK(1); SHMEM_TOTAL_RED; GMEM_ATOM_RED",
    # hub rows span thousands of BMTs: fp32 atomic chains beyond the A25 bound go through
    # the fp64 heavy-row accumulator
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16); GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
]


@pytest.mark.parametrize("graph", C3_GRAPHS)
def test_c3_graphs(c3, graph):
    P = asp.Plan(_mat(c3), graph, device=0)
    run_sampled(c3, P, 1.0, 0.0, 3)
    run_sampled(c3, P, 1.5, -0.5, 4)


def test_c3_search(c3):
    A = _mat(c3)
    best, text = asp.search(A, device=0, seed=3, max_candidates=10, budget_seconds=60, warmup=2, reps=5,
                            seed_graphs=C3_GRAPHS[:2])
    run_sampled(c3, best, 1.0, 0.0, 5)


C4_GRAPHS = [
    "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "DENSE_DECOM(b=64,theta=0.5) { DENSE | COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED }",
    "COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
]


@pytest.mark.parametrize("graph", C4_GRAPHS)
def test_c4_graphs(c4, graph):
    c, tiles = c4
    P = asp.Plan(_mat(c), graph, device=0, keep_host=graph.startswith("DENSE") and not FULL)
    run_sampled(c, P, 1.0, 0.0, 4)
    run_sampled(c, P, 2.0, 1.0, 6)
    if graph.startswith("DENSE") and not FULL:
        rid, rptr, tc = P.export("p0.tile.row_id"), P.export("p0.tile.row_ptr"), P.export("p0.tile.col")
        got = [(int(rid[t]), int(tc[k])) for t in range(rid.shape[0]) for k in range(rptr[t], rptr[t + 1])]
        assert got == [tuple(map(int, t)) for t in tiles]          # A13 pin: planted tiles extracted


C5_GRAPHS = [
    "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    # x-window staging form (banded): 32-nonzero BMTs, CSR5-like slot-major pad, 1024 threads
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024); GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(16); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512); GMEM_ATOM_RED",
    # SELL-C-sigma: sort inside 256-row BMTBs, pad per 32-row BMW (P:279 SORT_BMTB "decrease the padding rate")
    "COMPRESS; BMTB_ROW_BLOCK(256); SORT_BMTB; BMW_ROW_BLOCK(32); BMT_ROW_BLOCK(1); BMT_PAD(BMW); THREAD_TOTAL_RED; GMEM_ATOM_RED",
]


@pytest.mark.parametrize("graph", C5_GRAPHS)
def test_c5_graphs(c5, graph):
    P = asp.Plan(_mat(c5), graph, device=0)
    if "THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=" in graph:
        assert P.info()["kernels"].endswith("_xwin"), P.info()["kernels"]   # banded -> x window
    run_sampled(c5, P, 1.0, 0.0, 5)
    run_sampled(c5, P, -1.5, 0.5, 6)


def test_c5_xwin_integer_exact():
    c = synth.c5_band_csr(m=1 << 21, nnz=1 << 25, band=4096, int_mode=True)
    P = asp.Plan(_mat(c), C5_GRAPHS[2], device=0)
    assert P.info()["kernels"].endswith("_xwin")
    run_sampled(c, P, 2.0, -1.0, 8, int_mode=True)


@pytest.mark.parametrize("world", [2, 8])
def test_c5_rowdiv_bands_equal_single(world):
    """§8(e): each ROW_DIV band planned alone (as on its own GPU) writes its slice of y;
    the concatenation equals the single-device result bit for bit (integer mode)."""
    c = synth.c5_band_csr(m=1 << 20, nnz=1 << 24, band=4096, int_mode=True)
    A = _mat(c)
    x, _ = synth.vectors(c.n, c.m, 7, np.float64, True)
    dx = torch.from_numpy(x).cuda()
    y1 = torch.zeros(c.m, dtype=torch.float64, device="cuda")
    g = C5_GRAPHS[0]
    asp.Plan(A, g, device=0).spmv(1.0, dx, 0.0, y1)
    cuts = A.row_cuts(world)
    nnz = np.diff(c.row_ptr[cuts])
    assert nnz.max() - nnz.min() <= 2 * int(np.diff(c.row_ptr).max())   # nnz-balanced (A35)
    yb = torch.zeros(c.m, dtype=torch.float64, device="cuda")
    for r in range(world):
        band = A.row_slice(int(cuts[r]), int(cuts[r + 1]))
        try:  # each band may get its own design ("different designs for different parts")
            P = asp.Plan(band, band.random_graph(r) if r % 2 else g, device=0)
        except asp.AsError:
            P = asp.Plan(band, g, device=0)
        P.spmv(1.0, dx, 0.0, yb[int(cuts[r]):int(cuts[r + 1])])
    torch.cuda.synchronize()
    assert torch.equal(y1, yb)



BEST = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                   "best_graphs.json")))


def _int_twin(c, seed):
    """The integer-exact twin of a config: same structure, values from the integer stream."""
    return synth.Csr(c.m, c.n, c.row_ptr, c.col, synth._fast_values(seed, c.nnz, c.val.dtype, True), c.name)


@pytest.mark.parametrize("wl", ["lap2d-2048", "rmat-24", "blockdense-8m", "band-irreg-64m"])
def test_committed_winner_full_size(wl):
    """The exact graph the bench times for each config (profiles/best_graphs.json), planned
    on the full-size matrix (C5: a 1/4-scale instance of the same shape, 2^28 nonzeros, to
    stay within the GPU test budget): every row against the oracle in real mode, and the
    integer-exact twin bit-identical."""
    if wl == "lap2d-2048":
        coo = synth.c2_lap2d(2048)
        rp = np.zeros(coo.m + 1, np.int64)
        np.add.at(rp, coo.row + 1, 1)
        c, seed = synth.Csr(coo.m, coo.n, np.cumsum(rp), coo.col.astype(np.int32), coo.val, coo.name), 2
    elif wl == "rmat-24":
        c, seed = synth.c3_rmat_csr(), 3
    elif wl == "blockdense-8m":
        c, seed = synth.c4_blockdense_csr()[0], 4
    else:
        c, seed = synth.c5_band_csr(m=1 << 24, nnz=1 << 28), 5
    g = BEST[wl]["graph"]
    P = asp.Plan(_mat(c), g, device=0)
    run_sampled(c, P, 1.0, 0.0, 11)
    run_sampled(c, P, 1.5, -0.5, 12)
    del P
    ci = _int_twin(c, seed)
    del c
    P = asp.Plan(_mat(ci), g, device=0)
    run_sampled(ci, P, 2.0, -1.0, 13, int_mode=True)
