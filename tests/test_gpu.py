"""GPU parity tests: the CUDA path (through the C-ABI) against the long-double oracle.

Tolerance (north_star, reading A2/O2): |y - yref| <= tol * (|alpha| sum_j |a_ij x_j| +
|beta y0_i|) per row, tol = 1e-12 (fp64) / 1e-5 (fp32).  Integer-exact mode: bit-identical.
Metadata of device plans (AS_PLAN_KEEP_HOST) equals the oracle's byte for byte."""
import os

import numpy as np
import pytest

import synth
from oracle import builder_ref as B
from oracle import graph_ref as G
from oracle import spmv as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
asp = pytest.importorskip("paper_2212_10432_b200")

from test_host import COMPOSE_GRAPHS, CONC_GRAPHS, FAMILY_GRAPHS, assert_infeasible_justified, compare_export  # noqa: E402


def _mat(coo):
    return asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)


def run_check(coo, graph, alpha=1.0, beta=0.0, int_mode=False, seed=0, keep_host=False, y_nan=False, plan=None):
    dt = coo.val.dtype
    x, y0 = synth.vectors(coo.n, coo.m, seed, dt, int_mode)
    if y_nan:
        y0[:] = np.nan
    P = plan or asp.Plan(_mat(coo), graph, device=0, keep_host=keep_host)
    dx = torch.from_numpy(x).cuda()
    dy = torch.from_numpy(y0.copy()).cuda()
    P.spmv(alpha, dx, beta, dy)
    torch.cuda.synchronize()
    y = dy.cpu().numpy()
    yref, bound = S.spmv_coo(coo.m, coo.row, coo.col, coo.val.astype(np.float64), x.astype(np.float64),
                             alpha, beta, y0.astype(np.float64))
    if int_mode:
        assert np.array_equal(y.astype(np.float64), yref.astype(np.float64)), \
            (graph, np.nonzero(y.astype(np.float64) != yref.astype(np.float64))[0][:10])
    ok, ratio = S.check(y, yref, bound, dt)
    assert ok, (graph, ratio)
    return P, ratio


@pytest.mark.parametrize("graph", FAMILY_GRAPHS + COMPOSE_GRAPHS + CONC_GRAPHS)
@pytest.mark.parametrize("seed", range(3))
def test_family_integer_exact(graph, seed):
    coo = synth.random_matrix(33 + 40 * seed, 29 + 17 * seed, 0.12 + 0.06 * seed, seed, int_mode=True,
                              dense_rows=seed % 2)
    ab = [(1.0, 0.0), (2.0, -1.0), (-0.5, 0.5)][seed]
    try:
        P, _ = run_check(coo, graph, *ab, int_mode=True, seed=seed, keep_host=True)
    except asp.AsError as e:
        assert_infeasible_justified(coo, graph, e)
        return
    compare_export(P, coo, graph)


@pytest.mark.parametrize("graph", FAMILY_GRAPHS + COMPOSE_GRAPHS + CONC_GRAPHS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_family_real(graph, dtype):
    coo = synth.random_powerlaw(700, 650, 3, 300).astype(dtype)
    try:
        run_check(coo, graph, 1.5, -0.5, seed=3)
    except asp.AsError as e:
        assert_infeasible_justified(coo, graph, e)


@pytest.mark.parametrize("seed", range(30))
def test_random_graphs(seed):
    """as_search's random legal graphs on ragged matrices spanning many tiles."""
    dt = np.float64 if seed % 2 == 0 else np.float32
    coo = synth.random_powerlaw(3000 + 37 * seed, 2500, seed, 1500, int_mode=seed % 3 == 0).astype(dt)
    text = _mat(coo).random_graph(seed)
    try:
        run_check(coo, text, 1.0 if seed % 4 else 2.0, 0.0 if seed % 3 else 1.0, int_mode=seed % 3 == 0, seed=seed)
    except asp.AsError as e:
        assert_infeasible_justified(coo, text, e)


@pytest.mark.parametrize("graph", [
    "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(32); SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COL_DIV(cuts=[5000,10000,20000]) { COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    # R-conc: the hub row's partials come from side-stream parts too (their atomic rows go to
    # the fp64 heavy-row scratch, their stores to their own scratch vectors)
    "COL_DIV(cuts=[5000,10000,20000]) { COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED"
    " | COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(stream=1); GMEM_ATOM_RED"
    " | COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(stream=2); GMEM_ATOM_RED"
    " | COMPRESS; BMTB_NNZ_BLOCK(32); SHMEM_OFFSET_RED; SET_RESOURCE(stream=3); GMEM_ATOM_RED }",
])
def test_fp32_heavy_rows(graph):
    """A25: an fp32 hub row split over thousands of writer units must stay within 1e-5 of
    sum|a x|: its partials go to the fp64 heavy-row accumulator."""
    g = np.random.default_rng(5)
    m, n = 2000, 60000
    rows = [np.full(n, 7)]                       # one dense hub row of 60,000 nonzeros
    cols = [np.arange(n)]
    for r in range(m):
        if r != 7:
            c = np.sort(g.choice(n, 5, replace=False))
            rows.append(np.full(5, r))
            cols.append(c)
    row = np.concatenate(rows).astype(np.int64)
    col = np.concatenate(cols).astype(np.int64)
    order = np.lexsort((col, row))
    coo = synth.Coo(m, n, row[order], col[order], g.uniform(-1, 1, row.shape[0]).astype(np.float32))
    P, ratio = run_check(coo, graph, 1.0, 0.5, seed=2)
    assert "k_heavy_epilogue" in P.info()["kernels"]


def test_beta_zero_ignores_nan():
    coo = synth.random_matrix(50, 40, 0.2, 1)
    for g in FAMILY_GRAPHS[:4]:
        run_check(coo, g, 1.0, 0.0, y_nan=True)


def test_empty_and_degenerate():
    # all rows empty
    coo = synth.Coo(5, 5, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    run_check(coo, "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED", 1.0, 0.5)
    # single dense row, single column
    coo = synth.random_matrix(1, 300, 1.0, 2)
    for g in FAMILY_GRAPHS:
        try:
            run_check(coo, g, 1.0, -1.0)
        except asp.AsError as e:
            assert_infeasible_justified(coo, g, e)
    coo = synth.random_matrix(300, 1, 1.0, 2)
    run_check(coo, "COMPRESS; BMT_NNZ_BLOCK(7); THREAD_BITMAP_RED_G; GMEM_ATOM_RED", 1.0, -1.0)


def test_preconditions():
    coo = synth.random_matrix(8, 8, 0.5, 1)
    P = asp.Plan(_mat(coo), FAMILY_GRAPHS[0], device=0)
    buf = torch.zeros(64, dtype=torch.float64, device="cuda")
    with pytest.raises(asp.AsError):
        P.spmv(1.0, buf[0:8], 0.0, buf[4:12])       # alias
    with pytest.raises(asp.AsError):
        P.spmv(1.0, buf.data_ptr() + 4, 0.0, buf[32:40])  # x not aligned to 8 bytes
    hp = asp.Plan(_mat(coo), FAMILY_GRAPHS[0], device=-1)
    with pytest.raises(asp.AsError):
        hp.spmv(1.0, buf[0:8], 0.0, buf[32:40])     # host-only plan
    # the binding checks dtype, length, contiguity and device before the C-ABI call
    with pytest.raises(asp.AsError):
        P.spmv(1.0, buf[0:8].float(), 0.0, buf[32:40])  # fp32 x on an fp64 plan
    with pytest.raises(asp.AsError):
        P.spmv(1.0, buf[0:7], 0.0, buf[32:40])          # x too short
    with pytest.raises(asp.AsError):
        P.spmv(1.0, buf[0:16:2], 0.0, buf[32:40])       # strided x
    with pytest.raises(asp.AsError):
        P.spmv(1.0, buf[0:8].cpu(), 0.0, buf[32:40])    # host tensor


def test_spmv_host_path():
    coo = synth.c1_uniform()
    x, y0 = synth.vectors(coo.n, coo.m, 1)
    P = asp.Plan(_mat(coo), "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; GMEM_ATOM_RED", device=0)
    y = y0.copy()
    P.spmv_host(2.0, x, 0.5, y)
    yref, bound = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, 2.0, 0.5, y0)
    assert S.check(y, yref, bound, np.float64)[0]


@pytest.mark.parametrize("graph", FAMILY_GRAPHS[::4] + [
    "COL_DIV(cuts=[500]) { COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }"])
def test_graph_replay(graph):
    """AS_PLAN_GRAPH: the captured launch sequence replays to the same y; a new (x, y, alpha,
    beta) triggers a re-capture."""
    coo = synth.c1_uniform(int_mode=True)
    A = _mat(coo)
    P = asp.Plan(A, graph, device=0, graph_replay=True)
    for seed, (al, be) in enumerate([(1.0, 0.0), (1.0, 0.0), (2.0, -1.0), (2.0, -1.0)]):
        x, y0 = synth.vectors(coo.n, coo.m, seed // 2, np.float64, True)
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
        P.spmv(al, dx, be, dy)
        torch.cuda.synchronize()
        yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, al, be, y0)
        assert np.array_equal(dy.cpu().numpy(), yref), (graph, seed)


@pytest.mark.parametrize("graph", [
    "DIA_DECOM(theta=0.5) { DIA }",
    "COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "BIN(t=[4]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }"])
def test_plan_profile(graph):
    """as_plan_profile: one entry per kernel of as_plan_info.kernels, positive times, and
    per-launch bytes that add up to the plan's bytes model when the parts' column sets are
    disjoint (one part) -- the bench's dominant-kernel roofline rests on it."""
    coo = synth.c2_lap2d(256)
    P = asp.Plan(_mat(coo), graph, device=0)
    x = torch.rand(coo.n, dtype=torch.float64, device="cuda")
    y = torch.zeros(coo.m, dtype=torch.float64, device="cuda")
    prof = P.profile(x, y, reps=3)
    info = P.info()
    assert [p[0] for p in prof] == info["kernels"].split(";")
    assert all(p[1] > 0 for p in prof)
    if info["n_parts"] == 1:
        assert sum(p[2] for p in prof) == pytest.approx(info["bytes_model"], rel=1e-12)
    P.spmv(1.0, x, 0.0, y)  # the plan still runs normally afterwards
    torch.cuda.synchronize()


LAP_CUTS = "cuts=[262144,524288,786432]"
PIPE_GRAPHS = [
    f"ROW_DIV({LAP_CUTS}) {{ DIA_DECOM(theta=0.5) {{ DIA }} }}",
    f"ROW_DIV({LAP_CUTS}) {{ COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }}",
    "COL_DIV(cuts=[500000]) { COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "DIA_DECOM(theta=0.9995) { DIA | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED }",
]


@pytest.mark.parametrize("graph", PIPE_GRAPHS)
@pytest.mark.parametrize("beta", [0.0, -2.0])
def test_spmv_host_pipelined(graph, beta):
    """as_spmv_host with several launches: chunked H2D of x / D2H of y on copy streams,
    overlapped with the kernels (integer-exact inputs -> bit-identical to the oracle)."""
    coo = synth.c2_lap2d(1024)
    x, y0 = synth.vectors(coo.n, coo.m, 4, np.float64, True)
    P = asp.Plan(_mat(coo), graph, device=0)
    assert P.info()["n_launches"] >= 2
    yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, 3.0, beta, y0)
    xh = torch.from_numpy(x).pin_memory().numpy()
    for _ in range(2):  # twice: the plan's copy streams and events are reused
        yh = torch.from_numpy(y0.copy()).pin_memory().numpy()
        P.spmv_host(3.0, xh, beta, yh)
        assert np.array_equal(yh, yref), np.nonzero(yh != yref)[0][:10]


def test_spmv_host_pipelined_bin():
    """BIN: launch order is not monotone in rows or columns."""
    coo = synth.random_powerlaw(20_000, 20_000, 7, 400, int_mode=True)
    x, y0 = synth.vectors(coo.n, coo.m, 5, np.float64, True)
    g = ("BIN(t=[4,64]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED | "
         "COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED | "
         "COMPRESS; BMTB_ROW_BLOCK(1); SHMEM_TOTAL_RED; GMEM_ATOM_RED }")
    P = asp.Plan(_mat(coo), g, device=0)
    yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, 1.0, 1.0, y0)
    yh = y0.copy()
    P.spmv_host(1.0, x, 1.0, yh)
    assert np.array_equal(yh, yref)


# ------------------------------------------------------------------ BASELINE configs
C1_GRAPH = "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; SET_RESOURCE(128); GMEM_ATOM_RED"


@pytest.mark.parametrize("int_mode", [False, True])
def test_c1_full(int_mode):
    coo = synth.c1_uniform(int_mode=int_mode)
    P, ratio = run_check(coo, C1_GRAPH, 1.5, -0.5, int_mode=int_mode, seed=1, keep_host=True)
    compare_export(P, coo, C1_GRAPH)


C2_GRAPHS = [
    "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(256) }",
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(128); SHMEM_OFFSET_RED; GMEM_ATOM_RED",
]


@pytest.fixture(scope="module")
def c2():
    return synth.c2_lap2d(2048)


@pytest.mark.parametrize("graph", C2_GRAPHS)
def test_c2_closed_form(c2, graph):
    """Full-size C2 (4,194,304 rows): A*1 = number of missing neighbours, exact in fp64."""
    P = asp.Plan(_mat(c2), graph, device=0)
    dx = torch.ones(c2.n, dtype=torch.float64, device="cuda")
    dy = torch.full((c2.m,), 7.0, dtype=torch.float64, device="cuda")
    P.spmv(1.0, dx, 0.0, dy)
    torch.cuda.synchronize()
    g = 2048
    i = np.arange(c2.m)
    gx, gy = i % g, i // g
    want = (gx == 0).astype(float) + (gx == g - 1) + (gy == 0) + (gy == g - 1)
    assert np.array_equal(dy.cpu().numpy(), want)


@pytest.mark.parametrize("graph", C2_GRAPHS)
def test_c2_real_sampled(c2, graph):
    """Full-size C2 in real mode, alpha/beta != trivial: sampled rows vs the oracle row by row."""
    x, y0 = synth.vectors(c2.n, c2.m, 2)
    P = asp.Plan(_mat(c2), graph, device=0)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
    P.spmv(1.5, dx, -0.5, dy)
    torch.cuda.synchronize()
    y = dy.cpu().numpy()
    rows = np.unique(np.concatenate([np.arange(0, 4096), np.arange(c2.m - 4096, c2.m),
                                     np.random.default_rng(0).integers(0, c2.m, 20000)]))
    rp = np.searchsorted(c2.row, np.arange(c2.m + 1))
    sel = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    srp = np.concatenate([[0], np.cumsum(rp[rows + 1] - rp[rows])])
    yref, bound = S.spmv_csr(srp, c2.col[sel], c2.val[sel], x, 1.5, -0.5, y0[rows])
    ok, ratio = S.check(y[rows], yref, bound, np.float64)
    assert ok, ratio


def test_c2_dia_metadata_closed_form(c2):
    P = asp.Plan(_mat(c2), C2_GRAPHS[0], device=0, keep_host=True)
    assert P.export("p0.dia.off").tolist() == [-2048, -1, 0, 1, 2048]
    dv = P.export("p0.dia.val")
    assert dv.shape[0] == 5 * c2.m and int((dv == 0).sum()) == 8192
    info = P.info()
    assert info["pads"] == 8192 and info["prepass_rows"] == 0


def test_search_small():
    coo = synth.random_powerlaw(4000, 4000, 5, 2000)
    A = _mat(coo)
    best, text = asp.search(A, device=0, seed=7, max_candidates=12, budget_seconds=60, warmup=2, reps=5,
                            seed_graphs=["COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED"])
    assert G.is_legal(text), text
    run_check(coo, text, 1.0, 0.0, plan=best)


def test_search_verifies_and_beats_seed(tmp_path):
    """a7 pins (SURVEY §8(c) search row): the CSR-Scalar seed is timed
    first, no candidate's y fails the search's own verification, the winner validates and
    passes O2, and its confirmed median is no slower than the seed's (within the 1 % tie
    band of A29)."""
    import json
    coo = synth.random_powerlaw(20000, 20000, 6, 3000).astype(np.float32)
    A = _mat(coo)
    log = str(tmp_path / "search.jsonl")
    seed = "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED"
    best, text = asp.search(A, device=0, seed=11, max_candidates=16, budget_seconds=60, warmup=2, reps=7,
                            seed_graphs=[seed], log_path=log)
    rows = [json.loads(l) for l in open(log)]
    assert rows[0]["graph"] == str(asp.Graph(seed)) and rows[0]["median_ms"] > 0
    assert not any(r["status"].endswith("wrong_result") for r in rows)
    assert G.is_legal(text), text
    run_check(coo, text, 1.5, -0.5, plan=best)
    seed_t = rows[0]["median_ms"]
    best_t = min(r["median_ms"] for r in rows if r["median_ms"] > 0 and r["graph"] == text)
    assert best_t <= seed_t * 1.01, (best_t, seed_t)


XCACHE_GRAPHS = [
    "COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=1,xcache=512); GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,xcache=1000); GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(5); BMT_PAD(GLOBAL,1); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=128,xcache=3000); GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
    "SET_RESOURCE(tpb=1024,grid=2,xcache=4096); GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(128); BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; "
    "SET_RESOURCE(tpb=256,xcache=65536); GMEM_ATOM_RED",
    "SORT; COMPRESS; BMW_NNZ_BLOCK(96); BMT_NNZ_BLOCK(3); BMT_PAD(BMW,1); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
    "SET_RESOURCE(tpb=512,xcache=2048); GMEM_ATOM_RED",
]


@pytest.mark.parametrize("graph", XCACHE_GRAPHS)
@pytest.mark.parametrize("dtype,int_mode", [(np.float64, True), (np.float32, True), (np.float64, False),
                                            (np.float32, False)])
def test_xcache_parity(graph, dtype, int_mode):
    """R-xcache: staging the most referenced x entries in shared memory (columns re-encoded as
    ~slot on the device) changes no result: bit-identical in integer mode, O2 otherwise, and
    the logical (exported) columns are the original ones."""
    coo = synth.random_powerlaw(9000, 7000, 4, 2500, int_mode=int_mode).astype(dtype)
    P, _ = run_check(coo, graph, 1.5 if not int_mode else 2.0, -0.5, int_mode=int_mode, seed=4, keep_host=True)
    assert "_xh" in P.info()["kernels"], P.info()["kernels"]
    if int_mode:
        compare_export(P, coo, graph)


@pytest.mark.parametrize("graph", FAMILY_GRAPHS + COMPOSE_GRAPHS + XCACHE_GRAPHS)
def test_device_readback_matches_oracle(graph):
    """The uploaded device format, read back from device memory ("dev." export keys: implicit
    arrays and fitted models evaluated, the xcache column encoding undone) equals the oracle's
    logical Matrix Metadata Set byte for byte -- a check of the arrays the kernels read, not
    of the host copy they were built from."""
    coo = synth.random_powerlaw(3000, 2600, 2, 900, int_mode=True)
    try:
        P = asp.Plan(_mat(coo), graph, device=0)
    except asp.AsError as e:
        assert_infeasible_justified(coo, graph, e)
        return
    csr = B.Csr(coo.m, coo.n, coo.row, coo.col, coo.val)
    parts, w = B.build(csr, G.parse(graph), coo.val.dtype)
    ref = B.export(parts, w)
    keys = P.device_keys()
    assert keys, graph
    for i, p in enumerate(parts):
        if p.kind == "csr" and (p.excl_rows.shape[0] or p.atom_rows.shape[0]):
            have = {k.split(".", 2)[2] for k in keys if k.startswith(f"dev.p{i}.")}
            assert "col" in have or "pad.col" in have, (graph, i, have)
    for k in keys:
        lk = k[len("dev."):]
        assert lk in ref, (graph, k)
        got, want = P.export(k), ref[lk]
        assert got.shape == want.shape and np.array_equal(got.astype(want.dtype), want), (graph, k)


def test_smem_optin_not_lowered_by_later_plans():
    """The dynamic shared-memory opt-in is a per-function attribute shared by all plans: a
    plan built later with a smaller need must not break an earlier plan's launches (the
    search builds and keeps plans in any order)."""
    coo = synth.random_powerlaw(9000, 7000, 4, 2500, int_mode=True).astype(np.float32)
    big = "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=1,xcache=20000); GMEM_ATOM_RED"
    small = big.replace("xcache=20000", "xcache=2000")
    P_big = asp.Plan(_mat(coo), big, device=0)
    P_small = asp.Plan(_mat(coo), small, device=0)
    run_check(coo, big, 2.0, -0.5, int_mode=True, seed=1, plan=P_big)
    run_check(coo, small, 2.0, -0.5, int_mode=True, seed=1, plan=P_small)
    cs_big = "COMPRESS; BMTB_NNZ_BLOCK(6000); SHMEM_OFFSET_RED; SET_RESOURCE(tpb=256,stages=0); GMEM_ATOM_RED"
    cs_small = cs_big.replace("6000", "64")
    Q_big = asp.Plan(_mat(coo), cs_big, device=0)
    Q_small = asp.Plan(_mat(coo), cs_small, device=0)
    run_check(coo, cs_big, 1.0, 0.0, int_mode=True, seed=2, plan=Q_big)
    run_check(coo, cs_small, 1.0, 0.0, int_mode=True, seed=2, plan=Q_small)


@pytest.mark.parametrize("graph", [
    "COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(stages=0); GMEM_ATOM_RED",
    "ROW_DIV(cuts=[700,1500]) { COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
    "GMEM_ATOM_RED }",
])
@pytest.mark.parametrize("beta", [0.0, -1.0])
def test_spmv_host_batch(graph, beta):
    """as_spmv_host_batch: k independent host-buffer SpMVs pipelined over two device buffer
    pairs; every y_i equals the oracle's (integer-exact: bit-identical), including k = 1, 2
    and odd k (buffer reuse across the pair)."""
    coo = synth.random_powerlaw(2500, 2300, 8, 700, int_mode=True)
    P = asp.Plan(_mat(coo), graph, device=0)
    for k in (1, 2, 5):
        xs, ys, refs = [], [], []
        for i in range(k):
            x, y0 = synth.vectors(coo.n, coo.m, 40 + i, np.float64, True)
            yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, 2.0, beta, y0)
            xs.append(torch.from_numpy(x).pin_memory().numpy())
            ys.append(torch.from_numpy(y0.copy()).pin_memory().numpy())
            refs.append(yref)
        P.spmv_host_batch(2.0, xs, beta, ys)
        for i in range(k):
            assert np.array_equal(ys[i], refs[i].astype(np.float64)), (graph, k, i)


def test_search_with_history(tmp_path):
    """as_search with a cost-model history (graph + matrix features -> log time per nonzero,
    NEXT-3): the model stage runs on history + own candidates, the winner validates and passes
    O2."""
    import json
    other = synth.random_powerlaw(6000, 5000, 3, 800)
    B_ = _mat(other)
    hist = [(B_.random_graph(s), B_.features(), 0.01 + 0.001 * (s % 7), other.row.shape[0]) for s in range(40)]
    hist = [h for h in hist if G.is_legal(h[0])]
    coo = synth.random_powerlaw(8000, 7000, 5, 1500)
    log = str(tmp_path / "s.jsonl")
    best, text = asp.search(_mat(coo), device=0, seed=3, max_candidates=20, budget_seconds=40, warmup=1, reps=3,
                            log_path=log, history=hist)
    rows = [json.loads(l) for l in open(log)]
    assert any("pred_ms" in r for r in rows)  # the model stage ran with the history
    assert G.is_legal(text), text
    run_check(coo, text, 1.0, 0.5, plan=best)


def test_search_large_matrix_mode(tmp_path):
    """Above the large-matrix threshold (here lowered with AS_SEARCH_BIG_NNZ) the search times
    candidates at full size over the on-device Designer's family: every timed candidate but the
    seed graphs is device-buildable, and the winner validates and passes O2."""
    import json
    import subprocess
    import sys
    log = str(tmp_path / "s.jsonl")
    code = f'''
import sys, json
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import synth, paper_2212_10432_b200 as asp
coo = synth.random_powerlaw(20000, 18000, 6, 3000)
A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
seed = "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED"
P, g = asp.search(A, device=0, seed=5, max_candidates=14, budget_seconds=40, warmup=1, reps=3,
                  seed_graphs=[seed], log_path={log!r})
rows = [json.loads(l) for l in open({log!r})]
timed = [r for r in rows if r["median_ms"] > 0 and r["i"] >= 1]
assert timed, rows
assert all(A.device_buildable(r["graph"]) for r in timed), [r["graph"] for r in timed if not A.device_buildable(r["graph"])]
print("WINNER", g)
'''
    env = dict(os.environ, AS_SEARCH_BIG_NNZ="100000")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    winner = [l for l in r.stdout.splitlines() if l.startswith("WINNER")][0][7:]
    assert G.is_legal(winner), winner


@pytest.mark.parametrize("graph", CONC_GRAPHS)
def test_concurrent_branches_every_entry_point(graph):
    """R-conc (SET_RESOURCE stream): side-stream parts write their own scratch, added after the
    join -- checked bit-exact in integer mode through as_spmv (also repeated, so the side
    streams and events are reused), CUDA-graph replay (the fork/join captured), the host
    path, a batch, and the serialised as_plan_profile; every row against the oracle."""
    coo = synth.random_matrix(900, 700, 0.02, 5, int_mode=True, dense_rows=1).astype(np.float64)
    x, y0 = synth.vectors(coo.n, coo.m, 5, np.float64, True)
    yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, 2.0, -1.0, y0)
    A = _mat(coo)
    try:
        P = asp.Plan(A, graph, device=0, keep_host=True)
    except asp.AsError as e:
        assert_infeasible_justified(coo, graph, e)
        return
    modes = P.export("mode").tolist()
    # a part runs beside the main stream (DIA / DENSE parts may be empty on a random matrix)
    assert 3 in modes or graph.startswith(("DIA", "DENSE")), modes
    dx = torch.from_numpy(x).cuda()
    for _ in range(3):
        dy = torch.from_numpy(y0.copy()).cuda()
        P.spmv(2.0, dx, -1.0, dy)
        torch.cuda.synchronize()
        assert np.array_equal(dy.cpu().numpy(), yref), graph
    G = asp.Plan(A, graph, device=0, graph_replay=True)
    for _ in range(2):
        dy = torch.from_numpy(y0.copy()).cuda()
        G.spmv(2.0, dx, -1.0, dy)
        torch.cuda.synchronize()
        assert np.array_equal(dy.cpu().numpy(), yref), graph
    yh = y0.copy()
    P.spmv_host(2.0, x, -1.0, yh)
    assert np.array_equal(yh, yref)
    ys = [y0.copy() for _ in range(3)]
    P.spmv_host_batch(2.0, [x, x, x], -1.0, ys)
    assert all(np.array_equal(v, yref) for v in ys)
    dy = torch.from_numpy(y0.copy()).cuda()
    prof = P.profile(dx, dy, reps=2)
    assert len(prof) >= 2 and all(ms >= 0 for _, ms, _ in prof)
    run_check(coo.astype(np.float32), graph, 1.5, -0.5, seed=7)   # fp32, north_star tolerance


def test_concurrent_dense_beside_residual_c4_shape():
    """R-conc on a C4-shaped matrix (planted 64x64 tiles + diagonal + scatter): the DENSE part
    on a side stream, the NNZ residual on the main stream -- bit-identical to the same graph on
    one stream and to the oracle (integer mode), fp64 and fp32."""
    A, _ = synth.c4_blockdense(m=65536, b=64, n_tiles=192, nnz=1_500_000, seed=9, int_mode=True)
    res = ("COMPRESS; BMW_NNZ_BLOCK(nnz=1024); BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=BMW,vec=1); "
           "THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED")
    seq = f"DENSE_DECOM(b=64,theta=0.5) {{ DENSE; SET_RESOURCE(tpb=256) | {res} }}"
    conc = f"DENSE_DECOM(b=64,theta=0.5) {{ DENSE; SET_RESOURCE(tpb=256,stream=1) | {res} }}"
    for dt in (np.float64, np.float32):
        coo = A.astype(dt)
        x, y0 = synth.vectors(coo.n, coo.m, 9, dt, True)
        out = []
        for g in (seq, conc):
            P = asp.Plan(_mat(coo), g, device=0, keep_host=True)
            dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
            P.spmv(1.0, dx, 1.0, dy)
            torch.cuda.synchronize()
            out.append(dy.cpu().numpy())
        assert P.export("mode").tolist() == [3, 0]          # DENSE beside the residual
        yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val.astype(np.float64), x.astype(np.float64), 1.0, 1.0,
                             y0.astype(np.float64))
        assert np.array_equal(out[0], out[1]) and np.array_equal(out[1].astype(np.float64), yref)


def test_concurrent_dia_side_part():
    """R-conc with a DIA part on the side stream: ROW_DIV puts the DIA band (1024 rows) beside
    the larger CSR band, which leads the launch order and so is the main stream; the DIA rows
    are pre-passed and added from the DIA part's scratch after the join (integer mode,
    bit-identical to the oracle)."""
    coo = synth.c2_lap2d(64)
    ints = np.where(coo.val > 0, 4.0, -1.0)
    coo = synth.Coo(coo.m, coo.n, coo.row, coo.col, ints)
    g = ("ROW_DIV(cuts=[1024]) { DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(stream=1) } | "
         "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }")
    P, _ = run_check(coo, g, 2.0, -1.0, int_mode=True, seed=4, keep_host=True)
    assert P.export("mode").tolist() == [3, 0]
    assert P.export("prepass").tolist() == list(range(1024))
