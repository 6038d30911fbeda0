"""Oracle: Matrix Market parser, COO canonicaliser and row statistics.

Test infrastructure only (see oracle/__init__.py).

* input format: "takes a sparse matrix stored in the Matrix Market file format as input"
  (P:2, draft §Operator Graph); COO is "the universal source format".
  Reading A3: coordinate real/integer/pattern, general/symmetric; pattern -> 1.0;
  symmetric mirrored with the diagonal once; 1-based -> 0-based.  Reading A4:
  duplicates are an error.  Reading A6: empty rows are accepted.
* statistics: average row length nnz/n and row variance
  sum((row_len - nnz/n)^2)/n (§VII-C); "irregular" <=> variance > 100.
"""
from __future__ import annotations

import numpy as np


class MtxError(ValueError):
    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def parse_mtx(text: str):
    """Returns (m, n, row, col, val) canonical (sorted by (row, col)), 0-based."""
    lines = text.splitlines()
    if not lines or not lines[0].lower().startswith("%%matrixmarket"):
        raise MtxError("MALFORMED", "missing %%MatrixMarket header")
    hdr = lines[0].lower().split()
    if len(hdr) != 5 or hdr[1] != "matrix" or hdr[2] != "coordinate":
        raise MtxError("MALFORMED", "only 'matrix coordinate' is supported")
    field, sym = hdr[3], hdr[4]
    if field not in ("real", "integer", "pattern") or sym not in ("general", "symmetric"):
        raise MtxError("MALFORMED", f"unsupported field/symmetry {field}/{sym}")
    i = 1
    while i < len(lines) and (lines[i].startswith("%") or not lines[i].strip()):
        i += 1
    if i >= len(lines):
        raise MtxError("MALFORMED", "missing size line")
    size = lines[i].split()
    if len(size) != 3:
        raise MtxError("MALFORMED", "size line must be 'm n nnz'")
    m, n, nnz = (int(s) for s in size)
    rows, cols, vals = [], [], []
    for line in lines[i + 1:]:
        if not line.strip() or line.startswith("%"):
            continue
        t = line.split()
        if len(t) != (2 if field == "pattern" else 3):
            raise MtxError("MALFORMED", f"bad entry line {line!r}")
        r, c = int(t[0]) - 1, int(t[1]) - 1
        v = 1.0 if field == "pattern" else float(t[2])
        if not (0 <= r < m and 0 <= c < n):
            raise MtxError("INDEX_OUT_OF_RANGE", f"({r+1},{c+1})")
        rows.append(r)
        cols.append(c)
        vals.append(v)
        if sym == "symmetric" and r != c:
            rows.append(c)
            cols.append(r)
            vals.append(v)
    if len([1 for line in lines[i + 1:] if line.strip() and not line.startswith("%")]) != nnz:
        raise MtxError("MALFORMED", "entry count does not match the size line")
    return canonicalize(m, n, np.asarray(rows, np.int64), np.asarray(cols, np.int64),
                        np.asarray(vals, np.float64))


def canonicalize(m, n, row, col, val):
    if row.shape[0] and (row.min() < 0 or row.max() >= m or col.min() < 0 or col.max() >= n):
        raise MtxError("INDEX_OUT_OF_RANGE", "triplet outside the matrix")
    order = np.lexsort((col, row))
    row, col, val = row[order], col[order], val[order]
    if row.shape[0] > 1:
        dup = (row[1:] == row[:-1]) & (col[1:] == col[:-1])
        if dup.any():
            k = int(np.argmax(dup))
            raise MtxError("DUPLICATE", f"({row[k]},{col[k]})")
    return m, n, row, col, val


def stats(m, n, row):
    """P:437 avg = nnz/n (n = number of rows here, as in the paper's notation), population
    variance; P:111 irregular <=> variance > 100."""
    lens = np.bincount(np.asarray(row, np.int64), minlength=m).astype(np.int64)
    nnz = int(lens.sum())
    avg = nnz / m if m else 0.0
    var = float(sum((float(L) - avg) ** 2 for L in lens) / m) if m else 0.0
    return {"m": m, "n": n, "nnz": nnz, "max_row_len": int(lens.max()) if m else 0,
            "min_row_len": int(lens.min()) if m else 0, "empty_rows": int((lens == 0).sum()),
            "avg_row_len": avg, "row_len_variance": var, "irregular": int(var > 100.0)}
