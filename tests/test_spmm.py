"""SpMM (NEXT-4): Y = alpha*A*X + beta*Y with k right-hand sides through the C-ABI
(as_spmm) against the long-double oracle applied column by column (the plain definition:
column c of Y is the SpMV of column c of X).  Integer-exact inputs -> bit-identical;
real inputs -> the SpMV tolerance per element (O2)."""
import numpy as np
import pytest

import synth
from oracle import spmv as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
asp = pytest.importorskip("paper_2212_10432_b200")

from test_host import COMPOSE_GRAPHS, CONC_GRAPHS, FAMILY_GRAPHS, assert_infeasible_justified  # noqa: E402

EXTRA = [
    "DIA_DECOM(theta=0.2,max=6) { DIA | COMPRESS; BMT_NNZ_BLOCK(5); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "DENSE_DECOM(b=8,theta=0.3) { DENSE | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED }",
    "DENSE_DECOM(b=64,theta=0.05) { DENSE | COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "HYB_DECOM(w=3) { COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED | "
    "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
]


def oracle_spmm(coo, X, alpha, beta, Y0):
    k = X.shape[1]
    out = np.empty((coo.m, k))
    bound = np.empty((coo.m, k))
    for c in range(k):
        out[:, c], bound[:, c] = S.spmv_coo(coo.m, coo.row, coo.col, coo.val.astype(np.float64),
                                            X[:, c].astype(np.float64), alpha, beta, Y0[:, c].astype(np.float64))
    return out, bound


def run(coo, graph, k, alpha, beta, int_mode, seed, pad=0):
    dt = coo.val.dtype
    g = np.random.default_rng(seed)
    if int_mode:
        X = g.integers(-4, 5, (coo.n, k)).astype(dt)
        Y0 = g.integers(-4, 5, (coo.m, k)).astype(dt)
    else:
        X = g.uniform(-1, 1, (coo.n, k)).astype(dt)
        Y0 = g.uniform(-1, 1, (coo.m, k)).astype(dt)
    P = asp.Plan(asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val), graph, device=0, spmm=True)
    tdt = torch.float64 if dt == np.float64 else torch.float32
    Xd = torch.zeros((coo.n, k + pad), dtype=tdt, device="cuda")
    Yd = torch.zeros((coo.m, k + pad), dtype=tdt, device="cuda")
    Xd[:, :k] = torch.from_numpy(X)
    Yd[:, :k] = torch.from_numpy(Y0)
    P.spmm(alpha, Xd[:, :k], beta, Yd[:, :k])
    torch.cuda.synchronize()
    Y = Yd[:, :k].cpu().numpy().astype(np.float64)
    ref, bound = oracle_spmm(coo, X, alpha, beta, Y0)
    if int_mode:
        assert np.array_equal(Y, ref), (graph, k, np.argwhere(Y != ref)[:5])
    tol = 1e-12 if dt == np.float64 else 1e-5
    assert np.all(np.abs(Y - ref) <= tol * bound), (graph, k, np.max(np.abs(Y - ref) / (bound + 1e-300)))
    if pad:
        assert torch.count_nonzero(Yd[:, k:]) == 0  # columns beyond k untouched


@pytest.mark.parametrize("graph", FAMILY_GRAPHS + EXTRA + CONC_GRAPHS)
@pytest.mark.parametrize("k", [1, 8, 19])
def test_spmm_integer_exact(graph, k):
    coo = synth.random_matrix(130, 120, 0.15, 3, int_mode=True, dense_rows=1)
    try:
        run(coo, graph, k, 2.0, -1.0, True, k)
    except asp.AsError as e:
        assert_infeasible_justified(coo, graph, e)


@pytest.mark.parametrize("graph", EXTRA + FAMILY_GRAPHS[::5])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("k,beta", [(64, 0.0), (70, 0.5), (3, 0.0)])
def test_spmm_real(graph, dtype, k, beta):
    coo = synth.random_powerlaw(700, 650, 3, 300).astype(dtype)
    try:
        run(coo, graph, k, 1.5, beta, False, 7, pad=5)
    except asp.AsError as e:
        assert_infeasible_justified(coo, graph, e)


def test_spmm_dense_tensor_core_blocks():
    """C4-shaped: planted dense 64x64 tiles go through the DMMA kernel; k = 64 (one column
    chunk) and 136 (three chunks, ragged)."""
    c, tiles = synth.c4_blockdense_csr(m=4096, b=64, n_tiles=24, nnz=200_000, int_mode=True)
    coo = c.to_coo()
    g = "DENSE_DECOM(b=64,theta=0.5) { DENSE | COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }"
    P = asp.Plan(asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val), g, device=0, spmm=True)
    assert "dense" in P.info()["kernels"]
    for k in (64, 136):
        run(coo, g, k, 1.0, 0.0, True, k)


def test_spmm_preconditions():
    coo = synth.random_matrix(20, 20, 0.3, 1)
    A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
    X = torch.zeros((20, 4), dtype=torch.float64, device="cuda")
    Y = torch.zeros((20, 4), dtype=torch.float64, device="cuda")
    P = asp.Plan(A, FAMILY_GRAPHS[0], device=0)
    with pytest.raises(asp.AsError):
        P.spmm(1.0, X, 0.0, Y)              # plan built without spmm=True
    P = asp.Plan(A, FAMILY_GRAPHS[0], device=0, spmm=True)
    with pytest.raises(asp.AsError):
        P.spmm(1.0, X, 0.0, X)              # X and Y alias
