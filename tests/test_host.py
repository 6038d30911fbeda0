"""CPU tests of the native library's host logic against the oracle (no GPU needed):
the C-ABI loads and exports every declared symbol; the C++ graph validator agrees with the
oracle's; host-only plans (device = -1) reproduce the oracle's logical metadata byte for
byte (bit-exact integer/index arrays, value arrays copied exactly)."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import builder_ref as B
from oracle import graph_ref as G
from oracle import mtx_ref as M

asp = pytest.importorskip("paper_2212_10432_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "as.h")).read()
    declared = set(re.findall(r"\b(as_[a-z_0-9]+)\s*\(", hdr))
    declared -= {"as_status_t"}
    assert declared, "no declarations found"
    import ctypes
    lib = ctypes.CDLL(asp.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(asp.EXPORTED) == declared


def _mat(coo):
    return asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)


def test_ingest_errors_and_stats():
    with pytest.raises(asp.AsError) as e:
        asp.Matrix.from_coo(2, 2, [0, 0], [1, 1], np.array([1.0, 2.0]))
    assert e.value.status == "AS_ERR_DUPLICATE"
    with pytest.raises(asp.AsError) as e:
        asp.Matrix.from_coo(2, 2, [0, 2], [1, 1], np.array([1.0, 2.0]))
    assert e.value.status == "AS_ERR_INDEX_OUT_OF_RANGE"
    # unsorted input, 1-based, empty rows accepted (A6)
    A = asp.Matrix.from_coo(3, 3, [3, 1, 1], [1, 3, 1], np.array([5.0, 2.0, 1.0]), index_base=1)
    rp, col, val = A.export_csr()
    assert rp.tolist() == [0, 2, 2, 3] and col.tolist() == [0, 2, 0] and val.tolist() == [1.0, 2.0, 5.0]
    for seed in range(4):
        coo = synth.random_matrix(30, 20, 0.1 * (seed + 1), seed)
        st = _mat(coo).stats()
        ref = M.stats(coo.m, coo.n, coo.row)
        for k, v in ref.items():
            assert st[k] == pytest.approx(v, rel=1e-12, abs=1e-12), k


def test_mtx_ingest(tmp_path):
    p = tmp_path / "a.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 2.0\n3 1 -1.5\n2 2 4\n")
    A = asp.Matrix.from_mtx(p)
    m, n, r, c, v = M.parse_mtx(p.read_text())
    rp, col, val = A.export_csr()
    assert col.tolist() == c.tolist() and val.tolist() == v.tolist()
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n")
    with pytest.raises(asp.AsError) as e:
        asp.Matrix.from_mtx(p)
    assert e.value.status == "AS_ERR_DUPLICATE"


def test_row_cuts_from_ptr_match_oracle():
    """as_dist_row_cuts_ptr (band-local ranks) gives the oracle's A35 cuts from row_ptr alone."""
    for seed in range(4):
        coo = synth.random_powerlaw(500 + 77 * seed, 400, seed, 150)
        rp = np.zeros(coo.m + 1, np.int64)
        np.add.at(rp, coo.row + 1, 1)
        rp = np.cumsum(rp)
        for world in (1, 2, 3, 8):
            assert asp.row_cuts_from_ptr(rp, world).tolist() == B.row_cuts(rp, world).tolist()


def test_row_cuts_match_oracle():
    for seed in range(5):
        coo = synth.random_powerlaw(200, 200, seed, 80)
        A = _mat(coo)
        rp = np.zeros(coo.m + 1, np.int64)
        np.add.at(rp, coo.row + 1, 1)
        rp = np.cumsum(rp)
        for P in (1, 2, 3, 8):
            assert A.row_cuts(P).tolist() == B.row_cuts(rp, P).tolist()


GRAPH_CASES = [
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; SET_RESOURCE(128); GMEM_ATOM_RED",
    "SORT; COMPRESS; BMTB_ROW_BLOCK(2); BMT_ROW_BLOCK(1); BMT_PAD(BMTB); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(2); BMT_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED",
    "ROW_DIV(cuts=[1,2]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED | SORT; COMPRESS; BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED }",
    "DIA_DECOM(0.7) { DIA; SET_RESOURCE(tpb=64) | COMPRESS; BMTB_NNZ_BLOCK(8); SHMEM_OFFSET_RED; GMEM_ATOM_RED }",
    "COMPRESS; BMT_NNZ_BLOCK(4); BMT_PAD(GLOBAL); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(4); BMW_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "SORT; SORT_SUB(4); COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; SORT_BMTB; BMTB_ROW_BLOCK(4); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(4); BMT_ROW_BLOCK(1); BMT_PAD(scope=BMW); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "BIN(t=[3,1]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "COL_DIV(cuts=[2]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "COL_DIV(cuts=[2]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; GMEM_ATOM_RED | COMPRESS }",
    "DENSE_DECOM(b=2,theta=0.5) { DENSE; SET_RESOURCE(64); SET_RESOURCE(64) }",
    "DENSE_DECOM(b=2,theta=0.5) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "ROW_DIV(cuts=[2]) { DIA | COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED; SET_RESOURCE(256)",
    "COMPRESS; BMTB_ROW_BLOCK(1); BMW_ROW_BLOCK(1); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; WARP_TOTAL_RED; SHMEM_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(rows=1, rows=2); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(0); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "ROW_DIV(cuts=[3,2]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "SET_RESOURCE(tpb=100); COMPRESS",
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; SET_RESOURCE(tpb=100); GMEM_ATOM_RED",
    "DIA_DECOM(theta=1.5) { DIA }",
    "COMPRESS; BMTB_ROW_BLOCK(8); BMT_NNZ_BLOCK(2); BMT_PAD(scope=BMTB, vec=3); THREAD_TOTAL_RED; GMEM_ATOM_RED",
]


def _oracle_verdict(text):
    try:
        return "ok", G.to_string(G.parse(text))
    except G.GraphParseError:
        return "parse", None
    except G.GraphIllegal:
        return "illegal", None


def _product_verdict(text):
    try:
        return "ok", str(asp.Graph(text))
    except asp.AsError as e:
        return {"AS_ERR_GRAPH_PARSE": "parse", "AS_ERR_GRAPH_ILLEGAL": "illegal"}[e.status], None


@pytest.mark.parametrize("text", GRAPH_CASES + [c["graph"] for c in __import__("json").load(
    open(os.path.join(ROOT, "tests", "golden", "canonical_4x4.json")))["validator"]])
def test_validator_agrees_with_oracle(text):
    assert _product_verdict(text) == _oracle_verdict(text)


def _mutations(rng, text):
    """Random token-level mutations of legal graphs: swap two ops, drop one, duplicate one."""
    ops = [o.strip() for o in text.split(";")]
    k = rng.integers(0, 4)
    if k == 0 and len(ops) > 1:
        i, j = rng.choice(len(ops), 2, replace=False)
        ops[i], ops[j] = ops[j], ops[i]
    elif k == 1 and len(ops) > 1:
        ops.pop(int(rng.integers(0, len(ops))))
    elif k == 2:
        i = int(rng.integers(0, len(ops)))
        ops.insert(i, ops[i])
    else:
        pool = ["SORT", "COMPRESS", "BMTB_ROW_BLOCK(4)", "BMW_NNZ_BLOCK(64)", "BMT_NNZ_BLOCK(2)", "BMT_PAD(BMW)",
                "SORT_BMTB", "WARP_SEG_ADD_RED", "SHMEM_TOTAL_RED", "THREAD_TOTAL_RED", "SET_RESOURCE(64)"]
        ops.insert(int(rng.integers(0, len(ops) + 1)), pool[int(rng.integers(0, len(pool)))])
    return "; ".join(ops)


def test_validator_fuzz_agreement():
    rng = np.random.default_rng(0)
    A = _mat(synth.random_powerlaw(500, 500, 1, 100))
    n_ok = 0
    for i in range(400):
        base = A.random_graph(i)
        text = base if i % 3 == 0 else _mutations(rng, base)
        pv, ov = _product_verdict(text), _oracle_verdict(text)
        assert pv == ov, text
        n_ok += pv[0] == "ok"
    assert n_ok > 100


def _golden_coo(name):
    import json
    a = json.load(open(os.path.join(ROOT, "tests", "golden", "canonical_4x4.json")))[name]
    return synth.Coo(a["m"], a["n"], np.array(a["row"], np.int64), np.array(a["col"], np.int64),
                     np.array(a["val"], np.float64), name)


# export dtypes (DESIGN.md §3 Indices): indices int64, bitmaps uint32, values in the plan dtype
def _export_dtype(key, plan_dtype):
    if key.endswith(".bitmap"):
        return np.dtype(np.uint32)
    if key.endswith((".val", "dia.val", "tile.val", "pad.val")) or key.split(".")[-1] == "val":
        return np.dtype(plan_dtype)
    return np.dtype(np.int64)


def compare_export(P, coo, graph_text, dtype=None):
    """The product planned the graph: the oracle must plan it too (in the plan's dtype, which
    fixes BMT_PAD's default vec) and export the same logical arrays byte for byte."""
    csr = B.Csr(coo.m, coo.n, coo.row, coo.col, coo.val)
    parts, w = B.build(csr, G.parse(graph_text), dtype or coo.val.dtype)
    ex = B.export(parts, w)
    keys = set(P.keys())
    assert set(ex) == keys, (set(ex) ^ keys)
    for k, ref in ex.items():
        got = P.export(k)
        assert got.dtype == _export_dtype(k, coo.val.dtype), (k, got.dtype)
        assert np.array_equal(got.astype(ref.dtype), ref), (graph_text, k, got[:20], ref[:20])
        assert got.shape == ref.shape
    return True


@pytest.mark.parametrize("case", __import__("json").load(open(os.path.join(ROOT, "tests", "golden", "canonical_4x4.json")))["graphs"],
                         ids=lambda c: c["graph"][:40])
def test_host_plan_golden(case):
    coo = _golden_coo(case.get("matrix", "matrix"))
    P = asp.Plan(_mat(coo), case["graph"], device=-1)
    for k, want in case["expect"].items():
        assert P.export(k).tolist() == want, k
    assert compare_export(P, coo, case["graph"])


FAMILY_GRAPHS = [
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(37); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(5); BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(50); BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_ROW_BLOCK(3); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(32); BMT_NNZ_BLOCK(1); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(96); BMT_NNZ_BLOCK(1); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(5); BMT_PAD(GLOBAL,1); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(40); BMT_NNZ_BLOCK(4); BMT_PAD(BMTB,2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(96); BMT_NNZ_BLOCK(3); BMT_PAD(BMW,1); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_ROW_BLOCK(5); BMT_NNZ_BLOCK(2); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(7); BMW_ROW_BLOCK(1); BMT_NNZ_BLOCK(2); THREAD_TOTAL_RED; WARP_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(1); SHMEM_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(6); SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(13); SHMEM_OFFSET_RED; SET_RESOURCE(64); GMEM_ATOM_RED",
    "SORT; COMPRESS; BMTB_ROW_BLOCK(4); BMT_ROW_BLOCK(1); BMT_PAD(scope=BMTB,vec=2); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(8); SORT_BMTB; BMW_ROW_BLOCK(3); BMT_ROW_BLOCK(2); BMT_PAD(scope=BMW,vec=1); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "SORT_SUB(g=6); COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL,4); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "BIN(t=[2,5]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMTB_ROW_BLOCK(1); SHMEM_TOTAL_RED; GMEM_ATOM_RED }",
    "ROW_DIV(cuts=[5, 17]) { COMPRESS; BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "COL_DIV(cuts=[7, 15]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED | COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED }",
    "DIA_DECOM(theta=0.2,max=3) { DIA | COMPRESS; BMT_NNZ_BLOCK(5); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "DENSE_DECOM(b=4,theta=0.25) { DENSE | DIA_DECOM(0.3) { DIA | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED } }",
    "ROW_DIV(cuts=[9]) { DENSE_DECOM(b=3,theta=0.3) { DENSE | COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED } | DIA_DECOM(0.25, 2) { DIA; SET_RESOURCE(64) | SORT; COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED } }",
    "HYB_DECOM(w=3) { COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "SORT; HYB_DECOM(w=2) { COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL,1); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED }",
    "DIA_DECOM(theta=0.2,max=3) { DIA | HYB_DECOM(w=1) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED } }",
]


# Cross-level compositions (Fig. 5, P:322 Adapter) that no specialised
# family covers: they lower to the composed kernel (compose.cu).  Each row of the verdict's
# list of formerly infeasible graphs is here, plus every (thread, warp, block) reduction
# combination over ROW and NNZ levels, BMT_PAD, and the no-reduction (per-nonzero) form.
COMPOSE_GRAPHS = [
    "COMPRESS; BMTB_ROW_BLOCK(4); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(64); BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(3); BMT_ROW_BLOCK(2); THREAD_BITMAP_RED_G; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(1); BMW_NNZ_BLOCK(32); WARP_TOTAL_RED; SHMEM_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(1); BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(4); THREAD_TOTAL_RED; WARP_TOTAL_RED; SHMEM_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(1); BMT_NNZ_BLOCK(3); THREAD_TOTAL_RED; SHMEM_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(8); BMW_ROW_BLOCK(2); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; WARP_SEG_ADD_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(4); BMW_ROW_BLOCK(1); WARP_TOTAL_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(128); BMW_NNZ_BLOCK(32); WARP_SEG_ADD_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(128); BMW_NNZ_BLOCK(32); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(100); BMW_NNZ_BLOCK(37); BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_ROW_BLOCK(4); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_ROW_BLOCK(3); BMT_ROW_BLOCK(2); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(16); WARP_SEG_ADD_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(40); BMT_NNZ_BLOCK(2); WARP_BITMAP_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_ROW_BLOCK(2); BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(5); BMT_ROW_BLOCK(2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(6); BMT_ROW_BLOCK(1); GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); GMEM_ATOM_RED",
    "COMPRESS; GMEM_ATOM_RED",
    "COMPRESS; BMTB_NNZ_BLOCK(40); BMT_NNZ_BLOCK(4); BMT_PAD(BMTB,1); THREAD_BITMAP_RED_G; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(8); BMW_ROW_BLOCK(4); BMT_ROW_BLOCK(1); BMT_PAD(BMW,2); THREAD_TOTAL_RED; WARP_SEG_ADD_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "COMPRESS; BMW_ROW_BLOCK(1); BMT_NNZ_BLOCK(2); BMT_PAD(BMW,1); THREAD_TOTAL_RED; WARP_TOTAL_RED; GMEM_ATOM_RED",
    "SORT; COMPRESS; BMTB_ROW_BLOCK(16); SORT_BMTB; BMW_ROW_BLOCK(4); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; WARP_SEG_ADD_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED",
    "ROW_DIV(cuts=[11]) { COMPRESS; BMTB_ROW_BLOCK(4); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; SHMEM_OFFSET_RED; GMEM_ATOM_RED | COMPRESS; BMW_ROW_BLOCK(4); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; WARP_SEG_ADD_RED; GMEM_ATOM_RED }",
    "COL_DIV(cuts=[14]) { COMPRESS; BMTB_NNZ_BLOCK(64); BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; SHMEM_OFFSET_RED; GMEM_ATOM_RED }",
]

# R-conc: branches whose SET_RESOURCE names different launch streams run concurrently;
# every part then adds atomically onto a fully pre-passed y (writer_rule, mode 2)
CONC_GRAPHS = [
    "DENSE_DECOM(b=4,theta=0.25) { DENSE; SET_RESOURCE(tpb=128,stream=1) | COMPRESS; BMW_NNZ_BLOCK(64); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=256,grid=1); GMEM_ATOM_RED }",
    "DIA_DECOM(theta=0.2,max=3) { DIA; SET_RESOURCE(stream=2) | COMPRESS; BMT_NNZ_BLOCK(5); BMT_PAD(GLOBAL,1); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "COL_DIV(cuts=[7, 15]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; SET_RESOURCE(stream=1); GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED | COMPRESS; BMTB_ROW_BLOCK(4); BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; SHMEM_OFFSET_RED; SET_RESOURCE(64,stream=3); GMEM_ATOM_RED }",
    "ROW_DIV(cuts=[9]) { COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; SET_RESOURCE(stream=1); GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "HYB_DECOM(w=2) { COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; SET_RESOURCE(stream=1); GMEM_ATOM_RED }",
]

# Product-only infeasibility: device resource limits the oracle does not model:
# shared memory (P2), the padded-slot cap (P4b), int32 device indices (A36), > 64 DIA
# diagonals, DENSE tiles > 128.  Any other AS_ERR_PLAN_INFEASIBLE must be infeasible for the
# oracle too (P1, ROW_DIV/COL_DIV cuts out of range, DIA/DENSE on permuted rows, a residual
# without a branch) -- a regression that rejects a plannable graph fails here.
RESOURCE_LIMITS = ("P2:", "P4b:", "exceeds int32", "more than 64 diagonals", "DENSE tiles larger than 128")


def assert_infeasible_justified(coo, graph, err):
    assert err.status == "AS_ERR_PLAN_INFEASIBLE", err
    if any(k in str(err) for k in RESOURCE_LIMITS):
        return
    csr = B.Csr(coo.m, coo.n, coo.row, coo.col, coo.val)
    with pytest.raises(B.Infeasible):
        B.build(csr, G.parse(graph), coo.val.dtype)


@pytest.mark.parametrize("graph", FAMILY_GRAPHS + COMPOSE_GRAPHS + CONC_GRAPHS)
@pytest.mark.parametrize("seed", range(3))
def test_host_plan_matches_oracle(graph, seed):
    coo = synth.random_matrix(33 + seed, 29, 0.12 + 0.06 * seed, seed, int_mode=True, dense_rows=seed % 2)
    try:
        P = asp.Plan(_mat(coo), graph, device=-1)
    except asp.AsError as e:
        assert_infeasible_justified(coo, graph, e)
        return
    assert compare_export(P, coo, graph)


def test_compose_graphs_plan():
    """Every composition plans (no 'no kernel' rejection) on a matrix where P1 holds."""
    coo = synth.random_matrix(40, 40, 0.1, 4, int_mode=True)
    for g in COMPOSE_GRAPHS:
        if "TOTAL_RED" in g and ("NNZ" in g or "BMT_ROW_BLOCK(2)" in g or "BMW_ROW_BLOCK(4)" in g):
            continue  # P1 may legitimately reject multi-row TOTAL blocks
        P = asp.Plan(_mat(coo), g, device=-1)  # raises on a missing kernel
        assert P.info()["kernels"], g


@pytest.mark.parametrize("seed", range(40))
def test_random_graphs_match_oracle(seed):
    """The search's random graphs (as_random_graph) are legal for the oracle and their
    metadata matches it bit for bit."""
    coo = synth.random_powerlaw(300, 280, seed % 5, 120, int_mode=True)
    A = _mat(coo)
    text = A.random_graph(seed)
    assert _oracle_verdict(text)[0] == "ok", text
    try:
        P = asp.Plan(A, text, device=-1)
    except asp.AsError as e:
        assert_infeasible_justified(coo, text, e)
        return
    compare_export(P, coo, text)


def test_fp32_plan_values():
    coo = synth.random_matrix(20, 20, 0.3, 3).astype(np.float32)
    P = asp.Plan(_mat(coo), "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED", device=-1)
    assert P.export("p0.val").dtype == np.float32
    assert compare_export(P, coo, "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED", np.float32)


def test_dist_host_validation():
    """as_dist_* host logic without a GPU: rank/world ranges, cut validation, NCCL id needs a
    device, spmv before cuts; as_set_allocator rejects half-installed hooks."""
    with pytest.raises(asp.AsError) as e:
        asp.Dist(2, 2, -1)
    assert e.value.status == "AS_ERR_INVALID_ARG"
    with pytest.raises(asp.AsError):
        asp.Dist(0, asp.AS_DIST_HANDLE_BYTES, -1)  # world > AS_DIST_MAX_WORLD
    d = asp.Dist(1, 3, -1)
    d.set_cuts([0, 4, 4, 9])                      # an empty band is legal (A35)
    for bad in ([1, 4, 6, 9], [0, 5, 4, 9]):
        with pytest.raises(asp.AsError) as e:
            d.set_cuts(bad)
        assert e.value.status == "AS_ERR_INVALID_ARG"
    with pytest.raises(asp.AsError) as e:
        asp.Dist(0, 2, -1, b"\0" * asp.AS_DIST_ID_BYTES)
    assert e.value.status == "AS_ERR_INVALID_ARG"
    with pytest.raises(asp.AsError):
        d.ipc_handle(1 << 20)                     # host-only dist
    d.close()
    import ctypes
    with pytest.raises(asp.AsError):
        asp._ck(asp._lib.as_set_allocator(asp._ALLOC_T(lambda n, s, c: None), asp._FREE_T(), None))
    asp.set_allocator()                           # restore defaults: OK


def test_dist_unique_id():
    """ncclGetUniqueId through the runtime-loaded NCCL (no device needed)."""
    try:
        a = asp.Dist.unique_id()
    except asp.AsError as e:
        assert e.status == "AS_ERR_NCCL"
        pytest.skip("NCCL not loadable here")
    assert len(a) == asp.AS_DIST_ID_BYTES and a != asp.Dist.unique_id()


def test_binding_checks_host_arrays():
    """Plan.spmv_host refuses arrays of the wrong dtype / length before the C-ABI call
    (a float32 or short y would otherwise be overrun by the device-to-host copy)."""
    coo = synth.random_matrix(20, 16, 0.3, 3)
    P = asp.Plan(_mat(coo), "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED", device=-1)
    x, y = np.zeros(16), np.zeros(20)
    for bad in [(x.astype(np.float32), y), (x, y.astype(np.float32)), (x[:15], y), (x, y[:19]), (x, y[::2])]:
        with pytest.raises(asp.AsError):
            P.spmv_host(1.0, bad[0], 0.0, bad[1])
    y.flags.writeable = False
    with pytest.raises(asp.AsError):
        P.spmv_host(1.0, x, 0.0, y)


def test_device_buildable_query():
    """as_graph_device_buildable: the NNZ-blocked family goes to the on-device Designer
    (devbuild.cu); ROW blocks, converting branches, the tile kernel's shapes, x windows and
    AS_PLAN_HOST_BUILD stay on the host Designer."""
    coo = synth.random_powerlaw(500, 400, 2, 90)
    A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
    yes = ["COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(stages=0); GMEM_ATOM_RED",
           "SORT; COMPRESS; BMW_NNZ_BLOCK(100); BMT_NNZ_BLOCK(7); BMT_PAD(BMW,1); THREAD_BITMAP_RED_G; "
           "WARP_SEG_ADD_RED; GMEM_ATOM_RED",
           "SORT_SUB(g=4); COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(2); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; "
           "WARP_BITMAP_RED; GMEM_ATOM_RED"]
    no = ["COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",  # x-window candidate (stages=2)
          "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
          "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
          "BIN(t=[4]) { COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(stages=0); GMEM_ATOM_RED }",
          "COMPRESS; BMTB_NNZ_BLOCK(64); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; SET_RESOURCE(stages=0); GMEM_ATOM_RED"]
    for g in yes:
        assert A.device_buildable(g), g
        assert not A.device_buildable(g, host_build=True), g
    for g in no:
        assert not A.device_buildable(g), g


def test_matrix_features():
    """as_matrix_features (the search cost model's matrix features) against a direct count."""
    coo = synth.random_powerlaw(700, 500, 3, 120).astype(np.float32)
    A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
    L = np.bincount(coo.row, minlength=coo.m).astype(np.float64)
    want = [np.log2(1 + coo.m), np.log2(1 + coo.n), np.log2(1 + L.sum()), L.mean(), np.log2(1 + L.var()),
            np.log2(1 + L.max()), float((L == 0).mean()), 4.0]
    assert np.allclose(A.features(), want, rtol=1e-12, atol=1e-12)


def test_conc_dia_side_part_export():
    """R-conc with the DIA part beside a CSR band (the CSR band leads the launch order): the
    C++ writer rule (modes, pre-pass) and every exported array equal the oracle's."""
    coo = synth.c2_lap2d(16)
    g = ("ROW_DIV(cuts=[64]) { DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(stream=1) } | "
         "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }")
    P = asp.Plan(_mat(coo), g, device=-1, keep_host=True)
    assert P.export("mode").tolist() == [3, 0] and P.export("prepass").tolist() == list(range(64))
    assert compare_export(P, coo, g)
