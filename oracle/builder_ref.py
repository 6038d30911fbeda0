"""Oracle: reference Matrix Metadata Set builder.

Test infrastructure only (see oracle/__init__.py).  Executes an operator graph on a
canonical CSR matrix "by executing its operators in orders, which include logic to
modify Matrix Metadata Set" (draft §Operator Graph; §V-A) and returns every
LOGICAL array the product's `as_plan_export` must reproduce byte for byte.

Written for clarity, not speed: plain loops over rows/blocks with numpy only for
storage, stable sorts and prefix sums.  Each step follows one reading in DESIGN.md
§Readings (A-numbers refer to SURVEY.md §8(c), restated there):

  ROW_DIV / COL_DIV      P:20, "divides the whole matrix into striped sub-matrices"   A10, A11
  SORT / SORT_SUB / BIN  P:21, "reorder matrix rows according to their lengths";
                         P:802 "sorted in a decreasing order"                               A7, A8, A9
  DIA_DECOM / DENSE_DECOM P:21 "separate the locally dense parts or diagonal band parts"    A12, A13
  HYB_DECOM              P:583 "the matrix decomposition strategy of HYB" (NEXT-4)          R-hyb
  COMPRESS               P:22 "pushes non-zeros to the left of each row"                    A6, A14
  *_BLOCK                P:25 "cut adjacent non-zeros of the matrix into blocks"; P:33     A15
  BMT_PAD                P:279 "add zeros to specific positions"; "padded to the max"  A18
  SORT_BMTB              P:279 "reorders rows of each BMTB"                                  A19
  THREAD_BITMAP_RED_G    P:281 "using a bitmap to mark row boundaries"                       A20
  SHMEM_OFFSET_RED       P:281 "CSR-like row offset indices that record the position of the
                         first intermediate result of each row"                             A21
  writer rule / beta     P:281, P:335 (GMEM_ATOM_RED)                                        A22
"""
from __future__ import annotations

import dataclasses
import numpy as np

from . import graph_ref as G


class Infeasible(ValueError):
    """Matrix-dependent plan-time rejection (reading A16 P1-P4 / parameter ranges)."""


@dataclasses.dataclass
class State:
    """A branch of the converting stage: an ordered list of global rows, an entry mask."""
    rows: np.ndarray          # global row ids, current order
    mask: np.ndarray          # bool[nnz] over the canonical CSR entries still in this branch
    contiguous: bool          # rows are r0..r1-1 ascending (no permutation applied)


class Csr:
    """Canonical CSR of the whole matrix (rows ascending, cols ascending within a row)."""

    def __init__(self, m, n, row, col, val):
        self.m, self.n = int(m), int(n)
        order = np.lexsort((col, row))
        self.row = np.asarray(row, np.int64)[order]
        self.col = np.asarray(col, np.int64)[order]
        self.val = np.asarray(val)[order]
        self.row_ptr = np.zeros(self.m + 1, np.int64)
        np.add.at(self.row_ptr, self.row + 1, 1)
        self.row_ptr = np.cumsum(self.row_ptr)

    def entries(self, r, mask):
        a, e = self.row_ptr[r], self.row_ptr[r + 1]
        idx = np.arange(a, e)
        return idx[mask[a:e]]


def _row_len(csr: Csr, st: State) -> np.ndarray:
    """Number of entries of each branch row still present (empty rows count 0, A6)."""
    cs = np.concatenate([[0], np.cumsum(st.mask.astype(np.int64))])
    cnt = cs[csr.row_ptr[1:]] - cs[csr.row_ptr[:-1]]
    return cnt[st.rows]


def _stable_desc(lengths: np.ndarray) -> np.ndarray:
    """Stable permutation sorting by descending length (ties keep current order) (A7)."""
    return np.argsort(-lengths, kind="stable")


# =====================================================================================
# Parts
# =====================================================================================
@dataclasses.dataclass
class Part:
    kind: str                     # "csr" | "dia" | "dense"
    arrays: dict                  # logical arrays (export keys without the "p{i}." prefix)
    excl_rows: np.ndarray         # global rows written exclusively (one writer unit)
    atom_rows: np.ndarray         # global rows written by several units of this part (atomics)
    ops: list = None              # mapping + implementing ops (csr parts)
    stream: int = 0               # SET_RESOURCE stream of the part's branch (R-conc)


def _stream_of(seq):
    """The launch stream a branch's SET_RESOURCE names (R-conc; 0 when it names none)."""
    for op in seq:
        if op.name == "SET_RESOURCE":
            return op.params["stream"]
    return 0


def build(csr: Csr, graph, dtype=np.float64):
    """Execute the graph; returns (parts, writer) where writer holds launch order, modes
    and the beta pre-pass row list (A22)."""
    parts = []
    st = State(np.arange(csr.m, dtype=np.int64), np.ones(csr.row.shape[0], bool), True)
    _run_seq(csr, graph, st, parts, np.dtype(dtype))
    writer = writer_rule(csr.m, parts)
    return parts, writer


def _run_seq(csr, seq, st, parts, dtype):
    for k, op in enumerate(seq):
        nm = op.name
        if nm == "ROW_DIV":
            cuts = op.params["cuts"]
            mb = st.rows.shape[0]
            if cuts[-1] >= mb:
                raise Infeasible(f"ROW_DIV cut {cuts[-1]} >= rows {mb}")
            bounds = [0] + cuts + [mb]
            for b, sub in enumerate(op.branches):
                _run_seq(csr, sub, State(st.rows[bounds[b]:bounds[b + 1]], st.mask.copy(), st.contiguous), parts, dtype)
            return
        if nm == "COL_DIV":
            cuts = op.params["cuts"]
            if cuts[-1] >= csr.n:
                raise Infeasible(f"COL_DIV cut {cuts[-1]} >= cols {csr.n}")
            bounds = [0] + cuts + [csr.n]
            for b, sub in enumerate(op.branches):
                keep = (csr.col >= bounds[b]) & (csr.col < bounds[b + 1])
                _run_seq(csr, sub, State(st.rows, st.mask & keep, st.contiguous), parts, dtype)
            return
        if nm == "SORT":
            perm = _stable_desc(_row_len(csr, st))
            st = State(st.rows[perm], st.mask, False)
            continue
        if nm == "SORT_SUB":
            g = op.params["g"]
            lens = _row_len(csr, st)
            perm = []
            for a in range(0, lens.shape[0], g):
                perm.extend(a + _stable_desc(lens[a:a + g]))
            st = State(st.rows[np.asarray(perm, np.int64)], st.mask, False)
            continue
        if nm == "BIN":
            t = op.params["t"]
            lens = _row_len(csr, st)
            lo = [0] + t
            hi = t + [np.iinfo(np.int64).max]
            for b, sub in enumerate(op.branches):
                sel = (lens > lo[b]) & (lens <= hi[b])
                _run_seq(csr, sub, State(st.rows[sel], st.mask, False), parts, dtype)
            return
        if nm == "HYB_DECOM":
            # HYB split (reading R-hyb; the decomposition P:583 names as missing):
            # in every row of the branch, its first w live nonzeros (column order) go to
            # branch 0 (ELL part), the remaining live ones to branch 1 (COO part).
            w = op.params["w"]
            ell = np.zeros_like(st.mask)
            rest = np.zeros_like(st.mask)
            for r in st.rows:
                k = 0
                for e in range(csr.row_ptr[r], csr.row_ptr[r + 1]):
                    if st.mask[e]:
                        if k < w:
                            ell[e] = True
                        else:
                            rest[e] = True
                        k += 1
            _run_seq(csr, op.branches[0], State(st.rows, ell, st.contiguous), parts, dtype)
            _run_seq(csr, op.branches[1], State(st.rows, rest, st.contiguous), parts, dtype)
            return
        if nm == "DIA_DECOM":
            _dia_decom(csr, op, st, parts, dtype)
            return
        if nm == "DENSE_DECOM":
            _dense_decom(csr, op, st, parts, dtype)
            return
        if nm == "COMPRESS":
            parts.append(_compress_and_map(csr, st, seq[k + 1:], dtype))
            parts[-1].stream = _stream_of(seq[k + 1:])
            return
        raise AssertionError(nm)


# ------------------------------------------------------------------ DIA_DECOM (A12)
def _dia_decom(csr, op, st, parts, dtype):
    if not st.contiguous:
        raise Infeasible("DIA_DECOM needs contiguous unpermuted rows")
    theta, dmax = op.params["theta"], op.params["max"]
    rows = st.rows
    mb = rows.shape[0]
    r0 = int(rows[0]) if mb else 0
    count = {}
    for r in rows:
        for e in csr.entries(r, st.mask):
            o = int(csr.col[e] - r)
            count[o] = count.get(o, 0) + 1
    sel = []
    for o, c in count.items():
        ln = sum(1 for r in rows if 0 <= r + o < csr.n)
        if float(c) >= theta * float(ln):
            sel.append(o)
    if len(sel) > dmax:
        sel.sort(key=lambda o: (-count[o], abs(o), o))
        sel = sel[:dmax]
    sel.sort()
    D = len(sel)
    dia_val = np.zeros(D * mb, dtype)
    mask = st.mask.copy()
    pos = {o: d for d, o in enumerate(sel)}
    for i, r in enumerate(rows):
        for e in csr.entries(r, st.mask):
            o = int(csr.col[e] - r)
            if o in pos:
                dia_val[pos[o] * mb + i] = csr.val[e]
                mask[e] = False
    arrays = {"dia.off": np.asarray(sel, np.int64), "dia.val": dia_val,
              "origin_rows": np.arange(r0, r0 + mb, dtype=np.int64) if D else np.zeros(0, np.int64)}
    excl = arrays["origin_rows"].copy()
    parts.append(Part("dia", arrays, excl, np.zeros(0, np.int64), stream=_stream_of(op.branches[0])))
    _residual(csr, op, State(rows, mask, True), parts, dtype)


def _residual(csr, op, st, parts, dtype):
    if len(op.branches) == 2:
        _run_seq(csr, op.branches[1], st, parts, dtype)
    elif _row_len(csr, st).sum() > 0:
        raise Infeasible(f"{op.name}: residual is non-empty but the graph gives it no branch")


# ------------------------------------------------------------------ DENSE_DECOM (A13)
def _dense_decom(csr, op, st, parts, dtype):
    if not st.contiguous:
        raise Infeasible("DENSE_DECOM needs contiguous unpermuted rows")
    b, theta = op.params["b"], op.params["theta"]
    rows = st.rows
    mb = rows.shape[0]
    r0 = int(rows[0]) if mb else 0
    r1 = r0 + mb
    count = {}
    for r in rows:
        for e in csr.entries(r, st.mask):
            key = (int(r) // b, int(csr.col[e]) // b)
            count[key] = count.get(key, 0) + 1
    tiles = sorted(k for k, c in count.items() if float(c) >= theta * float(b * b))
    T = len(tiles)
    tile_val = np.zeros(T * b * b, dtype)
    tindex = {k: t for t, k in enumerate(tiles)}
    mask = st.mask.copy()
    for r in rows:
        for e in csr.entries(r, st.mask):
            I, J = int(r) // b, int(csr.col[e]) // b
            t = tindex.get((I, J))
            if t is not None:
                i, j = int(r) - I * b, int(csr.col[e]) - J * b
                tile_val[t * b * b + j * b + i] = csr.val[e]
                mask[e] = False
    row_id, row_ptr = [], [0]
    for t, (I, J) in enumerate(tiles):
        if not row_id or row_id[-1] != I:
            if row_id:
                row_ptr.append(t)
            row_id.append(I)
    row_ptr.append(T)
    if not T:
        row_ptr = [0]
    excl = sorted(r for I in row_id for r in range(I * b, I * b + b) if r0 <= r < r1)
    arrays = {"tile.row_id": np.asarray(row_id, np.int64), "tile.row_ptr": np.asarray(row_ptr, np.int64),
              "tile.col": np.asarray([J for _, J in tiles], np.int64), "tile.val": tile_val,
              "origin_rows": np.asarray(excl, np.int64)}
    parts.append(Part("dense", arrays, np.asarray(excl, np.int64), np.zeros(0, np.int64),
                      stream=_stream_of(op.branches[0])))
    _residual(csr, op, State(rows, mask, True), parts, dtype)


# ------------------------------------------------------------------ COMPRESS + mapping
def _compress_and_map(csr, st, rest, dtype):
    """COMPRESS (A6, A14): rows in current order, empty rows compacted away; then the
    mapping and implementing operators of `rest` in order."""
    origin, rp, cols, vals = [], [0], [], []
    for r in st.rows:
        es = csr.entries(r, st.mask)
        if es.shape[0] == 0:
            continue
        origin.append(int(r))
        cols.extend(csr.col[es].tolist())
        vals.extend(csr.val[es].tolist())
        rp.append(len(cols))
    origin = np.asarray(origin, np.int64)
    row_ptr = np.asarray(rp, np.int64)
    col = np.asarray(cols, np.int64)
    val = np.asarray(vals, dtype=dtype)

    levels = {}     # lvl -> (kind, size)
    order = []
    pad = None
    sort_bmtb = False
    reds = []
    for op in rest:
        if op.name.endswith("_BLOCK"):
            lvl, kind = op.name.split("_")[0], op.name.split("_")[1]
            levels[lvl] = (kind, op.params["rows"] if kind == "ROW" else op.params["nnz"])
            order.append(lvl)
        elif op.name == "BMT_PAD":
            pad = dict(op.params)
        elif op.name == "SORT_BMTB":
            sort_bmtb = True
        elif op.name in G.REDUCTIONS:
            reds.append(op.name)

    blocks = {}     # lvl -> list of (a, e) nz ranges
    parent = [(0, int(row_ptr[-1]))] if row_ptr[-1] > 0 else []
    for lvl in order:
        kind, size = levels[lvl]
        blocks[lvl] = _cut(row_ptr, parent, kind, size)
        if lvl == "BMTB" and sort_bmtb:
            origin, row_ptr, col, val = _sort_bmtb(row_ptr, col, val, origin, blocks["BMTB"])
        parent = blocks[lvl]

    arrays = {"origin_rows": origin, "row_ptr": row_ptr, "col": col, "val": val}
    for lvl in order:
        nz_ptr = np.asarray([a for a, _ in blocks[lvl]] + [int(row_ptr[-1])], np.int64) if blocks[lvl] else np.zeros(1, np.int64)
        first_row = np.asarray([_row_of(row_ptr, a) for a, _ in blocks[lvl]], np.int64)
        arrays[f"{lvl.lower()}.nz_ptr"] = nz_ptr
        arrays[f"{lvl.lower()}.first_row"] = first_row

    # P1 (A16): X_TOTAL_RED needs every level-X block inside one row
    for red in reds:
        lvl = G.REDUCTIONS[red]
        if red.endswith("_TOTAL_RED"):
            for a, e in blocks[lvl]:
                if _row_of(row_ptr, a) != _row_of(row_ptr, e - 1):
                    raise Infeasible(f"P1: {red} but a {lvl} block spans rows")

    if "THREAD_BITMAP_RED_G" in reds and levels.get("BMT", ("", 0))[0] == "NNZ":
        k = levels["BMT"][1]
        nw = (k + 31) // 32
        head = np.zeros(int(row_ptr[-1]), bool)
        head[row_ptr[:-1]] = True
        bm = np.zeros(len(blocks["BMT"]) * nw, np.uint32)
        for t, (a, e) in enumerate(blocks["BMT"]):
            for j in range(e - a):
                if head[a + j]:
                    bm[t * nw + j // 32] |= np.uint32(1 << (j % 32))
        arrays["bmt.bitmap"] = bm

    if pad is not None:
        vec = pad["vec"] or (16 // np.dtype(dtype).itemsize)
        groups = [(0, int(row_ptr[-1]))] if pad["scope"] == "GLOBAL" else blocks[pad["scope"]]
        widths, pcol, pval = [], [], []
        bmts = blocks["BMT"]
        ti = 0
        for ga, ge in groups:
            mine = []
            while ti < len(bmts) and bmts[ti][1] <= ge and bmts[ti][0] >= ga:
                mine.append(bmts[ti])
                ti += 1
            nt = len(mine)
            W = max((e - a) for a, e in mine) if mine else 0
            W = (W + vec - 1) // vec * vec
            gcol = np.zeros(nt * W, np.int64)
            gval = np.zeros(nt * W, dtype)
            for t, (a, e) in enumerate(mine):
                for j in range(W):
                    slot = (j // vec) * nt * vec + t * vec + (j % vec)
                    if a + j < e:
                        gcol[slot] = col[a + j]
                        gval[slot] = val[a + j]
                    else:
                        gcol[slot] = col[e - 1]   # pad col = last real col (A18)
            widths.append(W)
            pcol.append(gcol)
            pval.append(gval)
        arrays["pad.width"] = np.asarray(widths, np.int64)
        # padded slot offset of every group (nt * W slots each), plus the total
        arrays["pad.base"] = np.concatenate([[0], np.cumsum([p.shape[0] for p in pcol])]).astype(np.int64)
        arrays["pad.col"] = np.concatenate(pcol) if pcol else np.zeros(0, np.int64)
        arrays["pad.val"] = np.concatenate(pval) if pval else np.zeros(0, dtype)

    if "SHMEM_OFFSET_RED" in reds:
        ptr, offs = [0], []
        for a, e in blocks["BMTB"]:
            r = _row_of(row_ptr, a)
            loc = []
            while r < row_ptr.shape[0] - 1 and row_ptr[r] < e:
                loc.append(max(int(row_ptr[r]), a) - a)
                r += 1
            loc.append(e - a)
            offs.extend(loc)
            ptr.append(len(offs))
        arrays["bmtb.reduce_ptr"] = np.asarray(ptr, np.int64)
        arrays["bmtb.reduce_row_offsets"] = np.asarray(offs, np.int64)

    # writer units: blocks of the highest level that has a reduction (A21/A22)
    red_lvls = [G.REDUCTIONS[r] for r in reds if G.REDUCTIONS[r] != "GMEM"]
    excl, atom = [], []
    if red_lvls:
        top = max(red_lvls, key=lambda l: G.RED_ORDER[l])
        units = blocks[top]
    else:
        units = [(i, i + 1) for i in range(int(row_ptr[-1]))]  # every nonzero is a unit
    starts = np.asarray([a for a, _ in units], np.int64)
    for r in range(origin.shape[0]):
        a, e = int(row_ptr[r]), int(row_ptr[r + 1])
        ua = np.searchsorted(starts, a, side="right") - 1
        ue = np.searchsorted(starts, e - 1, side="right") - 1
        (excl if ua == ue else atom).append(int(origin[r]))
    return Part("csr", arrays, np.asarray(excl, np.int64), np.asarray(atom, np.int64), rest)


def _row_of(row_ptr, e):
    return int(np.searchsorted(row_ptr, e, side="right") - 1)


def _cut(row_ptr, parents, kind, size):
    """A15: children restart at each parent; under an NNZ parent the 'rows' are the row
    fragments inside it; the last child of each parent is ragged."""
    out = []
    for a, e in parents:
        if kind == "NNZ":
            for s in range(a, e, size):
                out.append((s, min(s + size, e)))
        else:
            frags = []
            r = _row_of(row_ptr, a)
            while r < row_ptr.shape[0] - 1 and row_ptr[r] < e:
                frags.append((max(int(row_ptr[r]), a), min(int(row_ptr[r + 1]), e)))
                r += 1
            for i in range(0, len(frags), size):
                grp = frags[i:i + size]
                out.append((grp[0][0], grp[-1][1]))
    return out


def _sort_bmtb(row_ptr, col, val, origin, bmtb):
    """A19: stable descending sort of the rows inside each BMTB (rows are whole here)."""
    lens = np.diff(row_ptr)
    perm = []
    for a, e in bmtb:
        r0, r1 = _row_of(row_ptr, a), _row_of(row_ptr, e - 1) + 1
        perm.extend(r0 + _stable_desc(lens[r0:r1]))
    perm = np.asarray(perm, np.int64)
    new_rp = np.zeros_like(row_ptr)
    new_rp[1:] = np.cumsum(lens[perm])
    idx = np.concatenate([np.arange(row_ptr[r], row_ptr[r + 1]) for r in perm]) if perm.shape[0] else np.zeros(0, np.int64)
    return origin[perm], new_rp, col[idx], val[idx]


# ------------------------------------------------------------------ writer rule (A22)
def writer_rule(m, parts):
    """Launch order = non-empty parts by descending count of exclusively written rows
    (stable).  Parts naming a SET_RESOURCE stream other than the first part's run beside
    it into scratch (mode 3, R-conc; below).  Walking that order: a part whose exclusive rows are all first writes
    STOREs alpha*s + beta*y; otherwise it ADDs and its first-written exclusive rows join
    the beta pre-pass.  Atomic rows first written by a part, and rows no part writes,
    join the pre-pass (y <- beta*y, or 0 when beta == 0)."""
    live = [i for i, p in enumerate(parts) if p.excl_rows.shape[0] + p.atom_rows.shape[0] > 0]
    live.sort(key=lambda i: -parts[i].excl_rows.shape[0])
    # R-conc: the main stream is the launch stream of the first part in launch order; parts
    # naming another stream run beside it (mode 3): each sums into a scratch vector of its
    # own, added into y after the streams join -- so the rule runs over the main-stream
    # parts only, and rows of side parts that no main part writes join the pre-pass
    main = parts[live[0]].stream if live else 0
    written = np.zeros(m, bool)
    prepass = np.zeros(m, bool)
    mode = {}
    for i in live:
        p = parts[i]
        if p.stream != main:
            continue
        first = ~written[p.excl_rows]
        if first.all():
            mode[i] = 0   # STORE
        else:
            mode[i] = 1   # ADD
            prepass[p.excl_rows[first]] = True
        prepass[p.atom_rows[~written[p.atom_rows]]] = True
        written[p.excl_rows] = True
        written[p.atom_rows] = True
    for i in live:
        p = parts[i]
        if p.stream == main:
            continue
        mode[i] = 3
        prepass[p.excl_rows[~written[p.excl_rows]]] = True
        prepass[p.atom_rows[~written[p.atom_rows]]] = True
    prepass |= ~written
    return {"launch_order": np.asarray(live, np.int64),
            "mode": np.asarray([mode.get(i, 0) for i in range(len(parts))], np.int64),
            "prepass": np.nonzero(prepass)[0].astype(np.int64)}


def export(parts, writer) -> dict:
    """Flatten to the export namespace used by as_plan_export ("p<i>.<key>")."""
    out = {}
    for i, p in enumerate(parts):
        for k, v in p.arrays.items():
            out[f"p{i}.{k}"] = v
    out["launch_order"] = writer["launch_order"]
    out["mode"] = writer["mode"]
    out["prepass"] = writer["prepass"]
    return out


# ------------------------------------------------------------------ multi-GPU cuts (A35)
def row_cuts(row_ptr, P):
    """cut_r = the i minimising |P*row_ptr[i] - r*nnz| (ties -> smaller i), r = 1..P-1,
    made non-decreasing; cut_0 = 0, cut_P = m.  ROW_DIV across ranks."""
    m = row_ptr.shape[0] - 1
    nnz = int(row_ptr[-1])
    cuts = [0]
    for r in range(1, P):
        best, bi = None, 0
        for i in range(m + 1):
            d = abs(P * int(row_ptr[i]) - r * nnz)
            if best is None or d < best:
                best, bi = d, i
        cuts.append(max(bi, cuts[-1]))
    cuts.append(m)
    return np.asarray(cuts, np.int64)
