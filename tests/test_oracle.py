"""Pins for the oracle (CPU only).  Each pin checks the oracle against something other than
itself: hand-worked fixtures (tests/golden, cited), brute force on tiny inputs, closed
forms, and invariants (semantics preservation, permutation/graph independence)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import builder_ref as B
from oracle import graph_ref as G
from oracle import mtx_ref as M
from oracle import spmv as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "canonical_4x4.json")))


def _A(name="matrix"):
    a = GOLD[name]
    return a["m"], a["n"], np.array(a["row"]), np.array(a["col"]), np.array(a["val"], float)


# ------------------------------------------------------------------ O1 SpMV
@pytest.mark.parametrize("case", GOLD["spmv"], ids=lambda c: c["cite"][:30])
def test_spmv_hand_examples(case):
    m, n, r, c, v = _A()
    y0 = np.array(case["y0"], float) if case["y0"] is not None else None
    y, b = S.spmv_coo(m, r, c, v, np.array(case["x"], float), case["alpha"], case["beta"], y0)
    assert [float(t) for t in y] == case["y"]
    assert [float(t) for t in b] == case["bound"]


def _dense_exact(m, n, r, c, v, x, alpha, beta, y0):
    """Brute force in exact rationals over the dense matrix."""
    A = [[Fraction(0)] * n for _ in range(m)]
    for i, j, a in zip(r, c, v):
        A[i][j] = Fraction(float(a))
    out = []
    for i in range(m):
        s = sum(A[i][j] * Fraction(float(x[j])) for j in range(n))
        yi = Fraction(float(alpha)) * s
        if beta != 0:
            yi += Fraction(float(beta)) * Fraction(float(y0[i]))
        out.append(yi)
    return out


@pytest.mark.parametrize("seed", range(12))
def test_spmv_dense_bruteforce_integer_exact(seed):
    """S:71 property: agrees with the dense product for matrices <= 64x64 (exactly, in
    integer mode, since every partial sum is a small dyadic number)."""
    g = np.random.default_rng(seed)
    m, n = int(g.integers(1, 65)), int(g.integers(1, 65))
    A = synth.random_matrix(m, n, 0.2, seed, int_mode=True)
    x, y0 = synth.vectors(n, m, seed, int_mode=True)
    alpha, beta = [(1.0, 0.0), (2.0, 1.0), (-0.5, -1.0), (1.0, 0.5)][seed % 4]
    y, _ = S.spmv_coo(m, A.row, A.col, A.val, x, alpha, beta, y0)
    ref = _dense_exact(m, n, A.row, A.col, A.val, x, alpha, beta, y0)
    assert [Fraction(float(t)) for t in y] == ref


@pytest.mark.parametrize("seed", range(6))
def test_spmv_dense_bruteforce_real(seed):
    m, n = 40 + seed, 33
    A = synth.random_matrix(m, n, 0.3, seed)
    x, y0 = synth.vectors(n, m, seed)
    y, bnd = S.spmv_coo(m, A.row, A.col, A.val, x, 1.5, -0.5, y0)
    ref = _dense_exact(m, n, A.row, A.col, A.val, x, 1.5, -0.5, y0)
    for yi, ri, bi in zip(y, ref, bnd):
        assert abs(Fraction(float(yi)) - ri) <= Fraction(1e-15) * Fraction(float(bi)) + Fraction(1e-300)


def test_spmv_special_cases():
    # identity -> y = x
    n = 17
    x, _ = synth.vectors(n, n, 5)
    y, _ = S.spmv_coo(n, np.arange(n), np.arange(n), np.ones(n), x)
    assert np.array_equal(y.astype(float), x)
    # alpha = 0 -> y = beta*y0 exactly; beta = 0 -> NaN in y0 not propagated (A1)
    m, nn, r, c, v = _A()
    y0 = np.array([1.0, np.nan, 3.0, 4.0])
    y, _ = S.spmv_coo(m, r, c, v, np.ones(4), 1.0, 0.0, y0)
    assert np.all(np.isfinite(y.astype(float)))
    y, _ = S.spmv_coo(m, r, c, v, np.ones(4), 0.0, 2.0, np.array([1.0, 2.0, 3.0, 4.0]))
    assert list(y.astype(float)) == [2.0, 4.0, 6.0, 8.0]


def test_spmv_thread_count_independent():
    A = synth.c1_uniform()
    x, _ = synth.vectors(A.n, A.m, 1)
    y1, b1 = S.spmv_coo(A.m, A.row, A.col, A.val, x, nthreads=1)
    y8, b8 = S.spmv_coo(A.m, A.row, A.col, A.val, x, nthreads=7)
    assert np.array_equal(y1, y8) and np.array_equal(b1, b8)


def test_lap2d_closed_form():
    """C2 pin: 5-point Laplacian (4 / -1) times the ones vector = number of missing
    neighbours: 0 interior, 1 on edges, 2 on corners (exact)."""
    g = 64
    A = synth.c2_lap2d(g)
    assert A.nnz == 5 * g * g - 4 * g
    y, _ = S.spmv_coo(A.m, A.row, A.col, A.val, np.ones(A.n))
    gx, gy = np.arange(A.m) % g, np.arange(A.m) // g
    missing = (gx == 0).astype(int) + (gx == g - 1) + (gy == 0) + (gy == g - 1)
    assert np.array_equal(y.astype(float), missing.astype(float))


def test_check_tolerance():
    yref = np.array([1.0, 2.0], np.longdouble)
    bnd = np.array([1.0, 0.0], np.longdouble)
    assert S.check(np.array([1.0 + 5e-13, 2.0]), yref, bnd, np.float64)[0]
    assert not S.check(np.array([1.0 + 5e-12, 2.0]), yref, bnd, np.float64)[0]
    # a row whose bound is 0 (all its terms are 0) accepts only +-0, however small the error
    y1, b1 = np.array([1.0, 0.0], np.longdouble), np.array([1.0, 0.0], np.longdouble)
    assert not S.check(np.array([1.0, 1e-300]), y1, b1, np.float64)[0]
    assert S.check(np.array([1.0, -0.0]), y1, b1, np.float64)[0]
    z = np.array([0.0], np.longdouble)
    assert S.check(np.array([-0.0]), z, z, np.float64)[0]          # bound 0 => y must be +-0
    assert not S.check(np.array([1e-300]), z, z, np.float64)[0]


# ------------------------------------------------------------------ stats / MM
def test_stats_pins():
    m, n, r, c, v = _A()
    st = M.stats(m, n, r)
    for k in ("avg_row_len", "row_len_variance", "irregular", "max_row_len", "min_row_len", "empty_rows"):
        assert st[k] == GOLD["stats"][k], k
    # uniform rows -> variance 0; lengths [1, 21] -> variance exactly 100, regular
    assert M.stats(3, 3, np.array([0, 1, 2]))["row_len_variance"] == 0.0
    st = M.stats(2, 30, np.array([0] + [1] * 21))
    assert st["row_len_variance"] == 100.0 and st["irregular"] == 0


def test_mtx_parse():
    txt = "%%MatrixMarket matrix coordinate real symmetric\n% c\n2 2 2\n1 1 1.0\n2 1 3.0\n"
    m, n, r, c, v = M.parse_mtx(txt)
    assert (m, n) == (2, 2) and list(zip(r, c, v)) == [(0, 0, 1.0), (0, 1, 3.0), (1, 0, 3.0)]
    m, n, r, c, v = M.parse_mtx("%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n")
    assert list(v) == [1.0]
    with pytest.raises(M.MtxError) as e:
        M.parse_mtx("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n")
    assert e.value.kind == "DUPLICATE"
    with pytest.raises(M.MtxError) as e:
        M.parse_mtx("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n")
    assert e.value.kind == "INDEX_OUT_OF_RANGE"
    with pytest.raises(M.MtxError):
        M.parse_mtx("garbage\n")


# ------------------------------------------------------------------ validator
@pytest.mark.parametrize("case", GOLD["validator"], ids=lambda c: c["cite"][:30])
def test_validator_examples(case):
    if case["rule"] is None:
        g = G.parse(case["graph"])
        if "canonical" in case:
            assert G.to_string(g) == case["canonical"]
        assert G.to_string(G.parse(G.to_string(g))) == G.to_string(g)
    else:
        with pytest.raises(G.GraphIllegal) as e:
            G.parse(case["graph"])
        assert e.value.rule == case["rule"]


def test_parse_errors():
    for bad in ["FOO_RED", "COMPRESS;", "COMPRESS; BMT_NNZ_BLOCK()", "ROW_DIV(cuts=[2]) {",
                "COMPRESS; BMT_NNZ_BLOCK(nnz=4, nnz=5)"]:
        with pytest.raises((G.GraphParseError, G.GraphIllegal)):
            G.parse(bad)


# ------------------------------------------------------------------ builder
def _build(graph, coo=None, dtype=np.float64, matrix="matrix"):
    if coo is None:
        m, n, r, c, v = _A(matrix)
    else:
        m, n, r, c, v = coo.m, coo.n, coo.row, coo.col, coo.val
    csr = B.Csr(m, n, r, c, v)
    parts, w = B.build(csr, G.parse(graph), dtype)
    return B.export(parts, w), parts


@pytest.mark.parametrize("case", GOLD["graphs"], ids=lambda c: c["graph"][:40])
def test_builder_golden(case):
    ex, _ = _build(case["graph"], matrix=case.get("matrix", "matrix"))
    for k, want in case["expect"].items():
        assert k in ex, k
        got = ex[k]
        assert got.tolist() == want, (k, got.tolist(), want)


def _golden_failures():
    bad = 0
    for case in GOLD["graphs"]:
        try:
            ex, _ = _build(case["graph"], matrix=case.get("matrix", "matrix"))
        except Exception:
            bad += 1
            continue
        bad += any(k not in ex or ex[k].tolist() != w for k, w in case["expect"].items())
    return bad


@pytest.mark.parametrize("mutation", ["ascending", "unstable", "unrestarted_nnz", "unrestarted_row", "sort_sub_global"])
def test_golden_pins_catch_mutations(monkeypatch, mutation):
    """The hand-derived goldens must fail on plausible mistakes in the oracle's row
    permutations (A7, A8, A19) and block cutting (A15): a reversed sort, an unstable sort,
    children cut without restarting at their parent, SORT_SUB applied globally."""
    assert _golden_failures() == 0
    if mutation == "ascending":
        monkeypatch.setattr(B, "_stable_desc", lambda L: np.argsort(np.asarray(L), kind="stable"))
    elif mutation == "unstable":
        # ties broken by descending position (a valid descending sort, but not stable)
        monkeypatch.setattr(B, "_stable_desc", lambda L: np.lexsort((-np.arange(len(L)), -np.asarray(L))))
    elif mutation == "sort_sub_global":
        orig = B._stable_desc
        monkeypatch.setattr(B, "_run_seq", _patched_run_seq_sort_sub_global(B._run_seq))
    else:
        kind = "NNZ" if mutation == "unrestarted_nnz" else "ROW"
        orig_cut = B._cut

        def cut(row_ptr, parents, k, size):
            if k == kind and parents:   # ignore the parents: one global cut
                return orig_cut(row_ptr, [(parents[0][0], parents[-1][1])], k, size)
            return orig_cut(row_ptr, parents, k, size)
        monkeypatch.setattr(B, "_cut", cut)
    assert _golden_failures() > 0, mutation


def _patched_run_seq_sort_sub_global(run_seq):
    def patched(csr, seq, st, parts, dtype):
        seq = [G.Op("SORT", {}, []) if op.name == "SORT_SUB" else op for op in seq]
        return run_seq(csr, seq, st, parts, dtype)
    return patched


def reconstruct(ex, parts, m):
    """Semantics preservation (O5 iv): rebuild (row, col, val) from the exported
    metadata of every part, dropping pads; returns a dict (row, col) -> summed value."""
    acc = {}
    for i, p in enumerate(parts):
        pre = f"p{i}."
        if p.kind == "csr":
            org, rp, col, val = ex[pre + "origin_rows"], ex[pre + "row_ptr"], ex[pre + "col"], ex[pre + "val"]
            if pre + "bmt.bitmap" in ex:   # rows from first_row + bitmap (A20), not row_ptr
                nz, fr, bm = ex[pre + "bmt.nz_ptr"], ex[pre + "bmt.first_row"], ex[pre + "bmt.bitmap"]
                nw = bm.shape[0] // max(1, fr.shape[0])
                for t in range(fr.shape[0]):
                    bits = [(int(bm[t * nw + j // 32]) >> (j % 32)) & 1 for j in range(nz[t + 1] - nz[t])]
                    for j in range(len(bits)):
                        r = fr[t] + sum(bits[1:j + 1])
                        e = nz[t] + j
                        key = (int(org[r]), int(col[e]))
                        acc[key] = acc.get(key, 0.0) + float(val[e])
                continue
            if pre + "pad.col" in ex:      # rows from the padded slot layout (A18)
                pw, pc, pv = ex[pre + "pad.width"], ex[pre + "pad.col"], ex[pre + "pad.val"]
                nzb = ex[pre + "bmt.nz_ptr"]
                lens = np.diff(nzb)
                # recompute group membership from the scope's nz_ptr
                scope = next(o.params["scope"] for o in p.ops if o.name == "BMT_PAD")
                gptr = [0, rp[-1]] if scope == "GLOBAL" else list(ex[pre + scope.lower() + ".nz_ptr"])
                base, t = 0, 0
                for gi in range(len(gptr) - 1):
                    mine = []
                    while t < lens.shape[0] and nzb[t] >= gptr[gi] and nzb[t + 1] <= gptr[gi + 1]:
                        mine.append(t)
                        t += 1
                    nt, W = len(mine), int(pw[gi])
                    vec = next(o.params["vec"] for o in p.ops if o.name == "BMT_PAD") or (16 // val.itemsize)
                    for lt, bt in enumerate(mine):
                        for j in range(W):
                            slot = base + (j // vec) * nt * vec + lt * vec + j % vec
                            if j < lens[bt]:
                                e = nzb[bt] + j
                                r = np.searchsorted(rp, e, side="right") - 1
                                assert pc[slot] == col[e]
                                key = (int(org[r]), int(pc[slot]))
                                acc[key] = acc.get(key, 0.0) + float(pv[slot])
                            else:
                                assert pv[slot] == 0 and pc[slot] == col[nzb[bt + 1] - 1]
                    base += nt * W
                continue
            for r in range(org.shape[0]):
                for e in range(rp[r], rp[r + 1]):
                    key = (int(org[r]), int(col[e]))
                    acc[key] = acc.get(key, 0.0) + float(val[e])
        elif p.kind == "dia":
            off, dv, org = ex[pre + "dia.off"], ex[pre + "dia.val"], ex[pre + "origin_rows"]
            mb = org.shape[0]
            for d, o in enumerate(off):
                for i, r in enumerate(org):
                    if dv[d * mb + i] != 0:
                        key = (int(r), int(r + o))
                        acc[key] = acc.get(key, 0.0) + float(dv[d * mb + i])
        elif p.kind == "dense":
            rid, rptr, tc, tv = ex[pre + "tile.row_id"], ex[pre + "tile.row_ptr"], ex[pre + "tile.col"], ex[pre + "tile.val"]
            bb = int(round((tv.shape[0] // max(1, tc.shape[0])) ** 0.5)) if tc.shape[0] else 0
            for tr in range(rid.shape[0]):
                for t in range(rptr[tr], rptr[tr + 1]):
                    for j in range(bb):
                        for i in range(bb):
                            a = tv[t * bb * bb + j * bb + i]
                            if a != 0:
                                key = (int(rid[tr] * bb + i), int(tc[t] * bb + j))
                                acc[key] = acc.get(key, 0.0) + float(a)
    return acc


FUZZ_GRAPHS = [
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(40); THREAD_BITMAP_RED_G; GMEM_ATOM_RED",
    "SORT; COMPRESS; BMTB_ROW_BLOCK(4); BMT_ROW_BLOCK(1); BMT_PAD(scope=BMTB,vec=2); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "SORT_SUB(g=5); COMPRESS; BMTB_ROW_BLOCK(3); SORT_BMTB; BMW_ROW_BLOCK(2); BMT_ROW_BLOCK(1); BMT_PAD(scope=BMW,vec=1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "ROW_DIV(cuts=[7, 20]) { COMPRESS; BMW_NNZ_BLOCK(16); BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED }",
    "COL_DIV(cuts=[10]) { COMPRESS; BMTB_NNZ_BLOCK(11); SHMEM_OFFSET_RED; GMEM_ATOM_RED | COMPRESS; BMT_ROW_BLOCK(2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "BIN(t=[2, 6]) { COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "DIA_DECOM(theta=0.3,max=3) { DIA | COMPRESS; BMT_NNZ_BLOCK(5); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "DENSE_DECOM(b=4,theta=0.3) { DENSE | DIA_DECOM(0.5) { DIA | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED } }",
    "HYB_DECOM(w=2) { COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "BIN(t=[3]) { HYB_DECOM(w=1) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED } }",
    "DIA_DECOM(theta=0.3,max=3) { DIA; SET_RESOURCE(stream=1) | COMPRESS; BMT_NNZ_BLOCK(5); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "COL_DIV(cuts=[10]) { COMPRESS; BMTB_NNZ_BLOCK(11); SHMEM_OFFSET_RED; SET_RESOURCE(stream=2); GMEM_ATOM_RED | COMPRESS; BMT_ROW_BLOCK(2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
]


@pytest.mark.parametrize("w", [1, 2, 5])
def test_hyb_split_is_first_w_per_row(w):
    """R-hyb: the ELL branch of HYB_DECOM(w) holds exactly the first min(len, w) nonzeros of
    every row (column order), the COO branch the rest -- checked against a direct count."""
    A = synth.random_matrix(40, 30, 0.25, 7, int_mode=True, dense_rows=1)
    ex, parts = _build(f"HYB_DECOM(w={w}) {{ COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED"
                       " | COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }", A)
    rows = {}
    for r, c in zip(A.row.tolist(), A.col.tolist()):
        rows.setdefault(r, []).append(c)
    for b, part in enumerate(parts):
        orig, rp, col = ex[f"p{b}.origin_rows"], ex[f"p{b}.row_ptr"], ex[f"p{b}.col"]
        got = {int(orig[i]): col[rp[i]:rp[i + 1]].tolist() for i in range(len(orig))}
        want = {r: (cs[:w] if b == 0 else cs[w:]) for r, cs in rows.items() if (cs[:w] if b == 0 else cs[w:])}
        assert got == want


@pytest.mark.parametrize("graph", FUZZ_GRAPHS)
@pytest.mark.parametrize("seed", range(4))
def test_builder_semantics_preservation(graph, seed):
    """S:230 / O5(iv): the exported metadata of any graph rebuilds exactly the input
    triplets (pads dropped), and every input row is either written by a part or in the
    beta pre-pass (A22)."""
    A = synth.random_matrix(30 + seed, 28, 0.15 + 0.05 * seed, seed, int_mode=True, dense_rows=seed % 2)
    try:
        ex, parts = _build(graph, A)
    except B.Infeasible:
        pytest.skip("infeasible on this matrix")
    acc = reconstruct(ex, parts, A.m)
    want = {(int(r), int(c)): float(v) for r, c, v in zip(A.row, A.col, A.val)}
    assert acc == want
    written = set()
    for p in parts:
        written |= set(p.excl_rows.tolist()) | set(p.atom_rows.tolist())
    assert set(range(A.m)) == written | set(ex["prepass"].tolist())


@pytest.mark.parametrize("seed", range(3))
def test_sort_is_permutation_and_stable(seed):
    A = synth.random_matrix(50, 20, 0.2, seed, int_mode=True)
    for gr in ["SORT; COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
               "SORT_SUB(g=7); COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED"]:
        ex, _ = _build(gr, A)
        org = ex["p0.origin_rows"]
        nonempty = np.unique(A.row)
        assert sorted(org.tolist()) == nonempty.tolist()          # permutation of covered rows
        lens = np.diff(ex["p0.row_ptr"])
        if gr.startswith("SORT;"):
            assert np.all(np.diff(lens) <= 0)                     # descending
            for a in range(1, org.shape[0]):                     # stable: ties keep row order
                if lens[a] == lens[a - 1]:
                    assert org[a] > org[a - 1]


def test_dia_on_lap2d_closed_form():
    """A12 on C2 (grid g): offsets {-g,-1,0,1,g}, 5*g^2 slots, 4*g pads, empty residual."""
    g = 32
    A = synth.c2_lap2d(g)
    ex, parts = _build("DIA_DECOM(theta=0.5,max=8) { DIA }", A)
    assert ex["p0.dia.off"].tolist() == [-g, -1, 0, 1, g]
    dv = ex["p0.dia.val"]
    assert dv.shape[0] == 5 * g * g and int((dv == 0).sum()) == 4 * g
    assert ex["prepass"].tolist() == [] and ex["mode"].tolist() == [0]


def test_writer_rule_concurrent_pin():
    """R-conc on the canonical 4x4 (hand-derived).  DIA_DECOM(0.75) selects offset 0 (3 of 4
    band positions filled; every other offset fills <= 1/2), so the DIA part writes rows
    0-3 and the residual {(0,2), (2,0), (2,1), (2,3)} rows 0 and 2.  One stream: DIA STOREs
    first, the residual ADDs onto rows DIA wrote, no pre-pass (A22).  Residual on another
    stream: it runs beside DIA into its own scratch and is added after the join (mode 3);
    DIA already writes rows 0 and 2, so still no pre-pass.  ROW_DIV(2) bands on two
    streams: band 0 (first in launch order) is the main stream and STOREs rows 0-1; band 1
    runs beside it, and its rows 2-3, which no main-stream part writes, are pre-passed."""
    seq = "DIA_DECOM(theta=0.75,max=8) { DIA%s | COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED%s; GMEM_ATOM_RED }"
    ex, parts = _build(seq % ("", ""))
    assert ex["p0.dia.off"].tolist() == [0] and ex["p1.origin_rows"].tolist() == [0, 2]
    assert ex["launch_order"].tolist() == [0, 1] and ex["mode"].tolist() == [0, 1] and ex["prepass"].tolist() == []
    for a, b in [("; SET_RESOURCE(stream=1)", ""), ("", "; SET_RESOURCE(stream=2)")]:
        ex, parts = _build(seq % (a, b))
        assert ex["launch_order"].tolist() == [0, 1] and ex["mode"].tolist() == [0, 3], (a, b)
        assert ex["prepass"].tolist() == []
    assert [p.stream for p in parts] == [0, 2]
    # the same stream named on both branches is one stream: the sequential rule
    ex, _ = _build(seq % ("; SET_RESOURCE(stream=2)", "; SET_RESOURCE(stream=2)"))
    assert ex["mode"].tolist() == [0, 1] and ex["prepass"].tolist() == []
    band = "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED%s; GMEM_ATOM_RED"
    ex, _ = _build("ROW_DIV(cuts=[2]) { %s | %s }" % (band % "; SET_RESOURCE(stream=1)", band % ""))
    assert ex["launch_order"].tolist() == [0, 1] and ex["mode"].tolist() == [0, 3]
    assert ex["prepass"].tolist() == [2, 3]


def test_dense_extracts_planted_tiles():
    """A13 on a small C4: the extracted tile set equals the planted list."""
    A, tiles = synth.c4_blockdense(m=2048, b=16, n_tiles=24, nnz=12000, seed=7)
    ex, _ = _build("DENSE_DECOM(b=16,theta=0.5) { DENSE | COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }", A)
    rid, rptr, tc = ex["p0.tile.row_id"], ex["p0.tile.row_ptr"], ex["p0.tile.col"]
    got = [(int(rid[tr]), int(tc[t])) for tr in range(rid.shape[0]) for t in range(rptr[tr], rptr[tr + 1])]
    assert got == [tuple(map(int, t)) for t in tiles]


def test_every_graph_same_y_integer_mode():
    """O5(i): summing each part's contribution in the writer order gives the oracle y
    exactly in integer mode, for every fuzz graph (checks the writer rule end to end)."""
    A = synth.random_matrix(37, 31, 0.2, 11, int_mode=True, dense_rows=1)
    x, y0 = synth.vectors(A.n, A.m, 11, int_mode=True)
    yref, _ = S.spmv_coo(A.m, A.row, A.col, A.val, x, 2.0, -1.0, y0)
    for graph in FUZZ_GRAPHS:
        try:
            ex, parts = _build(graph, A)
        except B.Infeasible:
            continue
        acc = reconstruct(ex, parts, A.m)
        # simulate: pre-pass, then parts in launch order with their modes
        y = y0.astype(np.float64).copy()
        y[ex["prepass"]] *= -1.0
        rowsum = {}
        for (r, c), v in acc.items():
            rowsum[r] = rowsum.get(r, 0.0) + v * x[c]
        done = set()
        for i in ex["launch_order"]:
            p = parts[i]
            for r in p.excl_rows.tolist() + p.atom_rows.tolist():
                if r in done:
                    continue
                done.add(r)
                if r in set(ex["prepass"].tolist()):
                    y[r] += 2.0 * rowsum.get(r, 0.0)
                else:
                    y[r] = 2.0 * rowsum.get(r, 0.0) - 1.0 * y0[r]
        assert np.array_equal(y, yref.astype(float)), graph


def test_row_cuts_pin():
    """A35 on A with P=2 (hand: cuts [0,2,4])."""
    rp = np.array([0, 2, 3, 6, 7])
    assert B.row_cuts(rp, 2).tolist() == GOLD["row_cuts"]["cuts"]
    # balanced by construction on uniform rows; empty bands legal when P > m
    assert B.row_cuts(np.arange(0, 101, 10), 5).tolist() == [0, 2, 4, 6, 8, 10]
    assert B.row_cuts(np.array([0, 5]), 3).tolist() == [0, 0, 1, 1]
