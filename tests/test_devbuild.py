"""On-device Designer (csrc/devbuild.cu): for the NNZ-blocked graph family the
format is built on the GPU.  Its arrays, read back from device memory and decoded ("dev."
keys), must equal the oracle's logical Matrix Metadata Set byte for byte (A6-A22: COMPRESS,
SORT/SORT_SUB, nested NNZ cutting A15, first_row, bitmaps A20, BMT_PAD A18, the writer
rule's pre-pass A22), y must match the oracle (integer-exact inputs: bit-identical), and the
plan must describe the same kernels and slots as the host-built plan of the same graph."""
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

DEV_GRAPHS = [
    "COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,stages=0); GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(40); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; "
    "SET_RESOURCE(tpb=128,grid=1,stages=0,xcache=300); GMEM_ATOM_RED",
    "SORT; COMPRESS; BMW_NNZ_BLOCK(100); BMT_NNZ_BLOCK(7); BMT_PAD(BMW,1); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
    "GMEM_ATOM_RED",
    "SORT_SUB(g=64); COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; "
    "SET_RESOURCE(tpb=512,grid=1,xcache=1000); GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(8192); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
    "SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=2048); GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(100); THREAD_BITMAP_RED_G; SET_RESOURCE(stages=0); GMEM_ATOM_RED",
    "SORT; COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; "
    "SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=0); GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(96); BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(5); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; "
    "GMEM_ATOM_RED",
    "SORT_SUB(g=7); COMPRESS; BMW_NNZ_BLOCK(33); BMT_NNZ_BLOCK(10); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; "
    "WARP_SEG_ADD_RED; SET_RESOURCE(tpb=64,grid=2,xcache=50); GMEM_ATOM_RED",
]

NOT_DEV = [  # shapes the host Designer keeps (tile kernel, x windows, composed levels, ROW blocks)
    "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "ROW_DIV(cuts=[100]) { COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(stages=0); GMEM_ATOM_RED }",
]


def _matrices():
    """int-exact fp64 and fp32 matrices with empty rows, a ragged tail and a hub row that
    spans more than 167 BMTs (A25 heavy row under fp32)."""
    a = synth.random_powerlaw(3000, 2600, 2, 900, int_mode=True)
    b = synth.random_matrix(257, 300, 0.03, 5, int_mode=True, dense_rows=2)
    hub = synth.random_powerlaw(1500, 4000, 9, 50, int_mode=True)
    r = np.full(3000, 700, np.int64)
    c = np.arange(3000, dtype=np.int64)
    keep = ~np.isin(r * 4000 + c, hub.row * 4000 + hub.col)
    row = np.concatenate([hub.row, r[keep]])
    col = np.concatenate([hub.col, c[keep]])
    val = np.concatenate([hub.val, np.full(int(keep.sum()), 3.0)])
    o = np.lexsort((col, row))
    hubm = synth.Coo(1500, 4000, row[o], col[o], val[o], "hub")
    return [a, b, hubm]


def _mat(coo):
    return asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)


@pytest.mark.parametrize("graph", DEV_GRAPHS)
@pytest.mark.parametrize("mi", range(3))
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_device_build_matches_oracle(graph, mi, dt):
    coo = _matrices()[mi].astype(dt)
    A = _mat(coo)
    P = asp.Plan(A, graph, device=0)
    info = P.info()
    assert info["device_built"] == 1, graph
    # metadata: every device array, decoded, equals the oracle's logical array
    csr = B.Csr(coo.m, coo.n, coo.row, coo.col, coo.val)
    parts, w = B.build(csr, G.parse(graph), coo.val.dtype)
    ref = B.export(parts, w)
    keys = P.device_keys()
    assert "dev.prepass" in keys
    assert any(k.endswith(".col") or k.endswith("pad.col") for k in keys)
    for k in keys:
        lk = k[len("dev."):]
        assert lk in ref, (graph, k)
        got, want = P.export(k), ref[lk]
        assert got.shape == want.shape and np.array_equal(got.astype(want.dtype), want), (graph, k)
    # y: integer-exact inputs -> bit-identical to the long-double oracle
    for alpha, beta, seed in [(1.0, 0.0, 1), (2.0, -1.0, 2)]:
        x, y0 = synth.vectors(coo.n, coo.m, seed, dt, True)
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
        P.spmv(alpha, dx, beta, dy)
        torch.cuda.synchronize()
        yref, bound = S.spmv_coo(coo.m, coo.row, coo.col, coo.val.astype(np.float64), x.astype(np.float64), alpha,
                                 beta, y0.astype(np.float64))
        y = dy.cpu().numpy().astype(np.float64)
        assert np.array_equal(y, yref), (graph, np.nonzero(y != yref)[0][:8])
    # the host-built plan of the same graph: same kernels, slots, pre-pass, writer class
    H = asp.Plan(A, graph, device=0, host_build=True)
    hi = H.info()
    assert hi["device_built"] == 0
    for k in ("kernels", "stored_slots", "pads", "prepass_rows", "n_launches", "single_writer", "n_parts",
              "modeled_arrays", "bytes_model", "bytes_model_beta", "bytes_floor"):
        assert info[k] == hi[k], (graph, k, info[k], hi[k])


@pytest.mark.parametrize("graph", NOT_DEV)
def test_host_designer_keeps_other_shapes(graph):
    coo = _matrices()[0]
    P = asp.Plan(_mat(coo), graph, device=0)
    assert P.info()["device_built"] == 0, graph


def test_device_build_real_values_and_cache_reuse():
    """Real-valued fp32 (O2 tolerance) on a matrix planned several times: the cached device
    CSR serves every plan, and a destroyed plan does not invalidate the others."""
    coo = synth.random_powerlaw(20000, 18000, 4, 3000, dtype=np.float32)
    A = _mat(coo)
    plans = [asp.Plan(A, g, device=0) for g in DEV_GRAPHS[:5]]
    del plans[2]
    x, y0 = synth.vectors(coo.n, coo.m, 3, np.float32)
    yref, bound = S.spmv_coo(coo.m, coo.row, coo.col, coo.val.astype(np.float64), x.astype(np.float64), 1.5, 0.5,
                             y0.astype(np.float64))
    for P in plans:
        assert P.info()["device_built"] == 1
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
        P.spmv(1.5, dx, 0.5, dy)
        torch.cuda.synchronize()
        ok, ratio = S.check(dy.cpu().numpy(), yref, bound, np.float32)
        assert ok, ratio


def _random_dev_graph(rng):
    """A random graph of the on-device Designer's family."""
    parts = []
    r = rng.integers(0, 3)
    if r == 1:
        parts.append("SORT")
    elif r == 2:
        parts.append(f"SORT_SUB(g={int(rng.choice([2, 5, 64, 1000]))})")
    parts.append("COMPRESS")
    k = int(rng.choice([1, 3, 4, 8, 13, 32, 40, 64, 100]))
    K = int(rng.choice([0, 5, 32, 96, 100, 256, 1000])) if rng.random() < 0.7 else 0
    if K:
        parts.append(f"BMW_NNZ_BLOCK({K})")
    parts.append(f"BMT_NNZ_BLOCK({k})")
    if rng.random() < 0.6:
        scope = "BMW" if K and rng.random() < 0.5 else "GLOBAL"
        parts.append(f"BMT_PAD({scope},{int(rng.choice([0, 1, 2, 4]))})")
    parts.append("THREAD_BITMAP_RED_G")
    if K:
        parts.append(str(rng.choice(["WARP_SEG_ADD_RED", "WARP_BITMAP_RED"])))
    xc = int(rng.choice([0, 0, 17, 500]))
    parts.append(f"SET_RESOURCE(tpb={int(rng.choice([64, 256, 1024]))},grid={int(rng.choice([0, 1, 2]))},"
                 f"stages=0,xcache={xc})")
    parts.append("GMEM_ATOM_RED")
    return "; ".join(parts)


@pytest.mark.parametrize("seed", range(24))
def test_device_build_fuzz(seed):
    """Random graphs of the family on random matrices: device-built arrays = oracle arrays,
    y bit-identical in integer mode, and the host build reports the same plan."""
    rng = np.random.default_rng(1000 + seed)
    dt = np.float32 if seed % 2 else np.float64
    coo = (synth.random_powerlaw(int(rng.integers(50, 3000)), int(rng.integers(40, 2500)), seed, 400, int_mode=True)
           if seed % 3 else synth.random_matrix(int(rng.integers(20, 400)), int(rng.integers(20, 300)), 0.05, seed,
                                                int_mode=True, dense_rows=1)).astype(dt)
    if coo.row.shape[0] == 0:
        return
    A = _mat(coo)
    for _ in range(3):
        graph = _random_dev_graph(rng)
        if not A.device_buildable(graph):  # the tile-kernel shapes stay on the host Designer
            continue
        try:
            P = asp.Plan(A, graph, device=0)
        except asp.AsError as e:
            H = None
            try:
                H = asp.Plan(A, graph, device=0, host_build=True)
            except asp.AsError:
                pass
            assert H is None, (graph, str(e))  # infeasible for both Designers or neither
            continue
        assert P.info()["device_built"] == 1
        csr = B.Csr(coo.m, coo.n, coo.row, coo.col, coo.val)
        parts, w = B.build(csr, G.parse(graph), coo.val.dtype)
        ref = B.export(parts, w)
        for k in P.device_keys():
            got, want = P.export(k), ref[k[len("dev."):]]
            assert got.shape == want.shape and np.array_equal(got.astype(want.dtype), want), (graph, k)
        x, y0 = synth.vectors(coo.n, coo.m, seed, dt, True)
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
        P.spmv(-1.5, dx, 0.5, dy)
        torch.cuda.synchronize()
        yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val.astype(np.float64), x.astype(np.float64), -1.5, 0.5,
                             y0.astype(np.float64))
        assert np.array_equal(dy.cpu().numpy().astype(np.float64), yref), graph
        hi = asp.Plan(A, graph, device=0, host_build=True).info()
        for key in ("kernels", "stored_slots", "prepass_rows", "bytes_model", "modeled_arrays"):
            assert P.info()[key] == hi[key], (graph, key)
