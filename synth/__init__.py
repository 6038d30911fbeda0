"""Seeded synthetic inputs shared by the CUDA path, the oracle tests and bench.py.

This module holds NO arithmetic of the method (no SpMV, no format building): it only
draws matrices and vectors.  Both sides of every parity test read their inputs from
here and from nowhere else (task rule: "only the seeded input generators serve both").

RNG: numpy's Philox4x32-10 counter-based generator keyed by (config seed, stream id),
with disjoint streams: 0 = matrix structure, 1 = x, 2 = y0, 3 = integer-mode values,
4 = real-mode values (SURVEY.md §8(d) "Configs as concrete synthetic inputs").

Every generator returns a ``Coo`` whose triplets are sorted by (row, col) and unique.
Real mode draws values, x and y0 from U[-1, 1); integer-exact mode draws values from
{-4..4}\\{0} and x, y0 from {-4..4} (SURVEY.md §8(c) "Integer-exact mode").

Configs (BASELINE.json "configs"; recipe in DESIGN.md §Inputs):
  C1 uniform-1k       1000x1000, diagonal + 9,000 uniform off-diagonal, fp64
  C2 lap2d-2048       5-point Laplacian on a 2048^2 grid, fp64 (values 4 / -1)
  C3 rmat-24          Graph500 R-MAT scale 24, 2^28 nnz incl. diagonal, fp32
  C4 blockdense-8m    24,576 dense 64x64 tiles + diagonal + uniform scatter, 2e8 nnz, fp64
  C5 band-irreg-64m   64M rows, 2^30 nnz, banded irregular rows, fp64
Each has a ``scale`` knob so that tests can draw a small instance with the same shape.
"""
from __future__ import annotations

import dataclasses
import numpy as np

STREAM_MATRIX, STREAM_X, STREAM_Y, STREAM_INTVAL, STREAM_VAL = 0, 1, 2, 3, 4


def rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed), int(stream)]))


@dataclasses.dataclass
class Coo:
    m: int
    n: int
    row: np.ndarray  # int64, sorted by (row, col), unique
    col: np.ndarray  # int64
    val: np.ndarray  # float64 or float32
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row.shape[0])

    def astype(self, dtype) -> "Coo":
        return Coo(self.m, self.n, self.row, self.col, self.val.astype(dtype), self.name)


def _sorted_unique(m, n, row, col):
    key = row.astype(np.int64) * np.int64(n) + col.astype(np.int64)
    key = np.unique(key)
    return (key // n).astype(np.int64), (key % n).astype(np.int64)


def _values(seed, nnz, dtype, int_mode):
    if int_mode:
        v = rng(seed, STREAM_INTVAL).integers(1, 5, size=nnz) * \
            np.where(rng(seed, STREAM_INTVAL + 16).random(nnz) < 0.5, -1, 1)
        return v.astype(dtype)
    return rng(seed, STREAM_VAL).uniform(-1.0, 1.0, size=nnz).astype(dtype)


def vectors(n: int, m: int, seed: int, dtype=np.float64, int_mode: bool = False):
    """x[n], y0[m] for a config (streams 1 and 2)."""
    if int_mode:
        x = rng(seed, STREAM_X).integers(-4, 5, size=n).astype(dtype)
        y = rng(seed, STREAM_Y).integers(-4, 5, size=m).astype(dtype)
    else:
        x = rng(seed, STREAM_X).uniform(-1.0, 1.0, size=n).astype(dtype)
        y = rng(seed, STREAM_Y).uniform(-1.0, 1.0, size=m).astype(dtype)
    return x, y


# ----------------------------------------------------------------------------------
# Hand-worked canonical matrix
# ----------------------------------------------------------------------------------
def canonical_4x4() -> Coo:
    row = np.array([0, 0, 1, 2, 2, 2, 3], dtype=np.int64)
    col = np.array([0, 2, 1, 0, 1, 3, 3], dtype=np.int64)
    val = np.arange(1, 8, dtype=np.float64)
    return Coo(4, 4, row, col, val, "canonical-4x4")


# ----------------------------------------------------------------------------------
# Small fuzz matrices
# ----------------------------------------------------------------------------------
def random_matrix(m: int, n: int, density: float, seed: int, dtype=np.float64,
                  int_mode: bool = False, empty_rows: bool = True,
                  dense_rows: int = 0) -> Coo:
    """Uniform random pattern; optionally some empty rows and some fully dense rows."""
    g = rng(seed, STREAM_MATRIX)
    mask = g.random((m, n)) < density
    if dense_rows:
        mask[g.choice(m, size=min(dense_rows, m), replace=False)] = True
    if not empty_rows:
        for r in np.nonzero(~mask.any(axis=1))[0]:
            mask[r, g.integers(0, n)] = True
    row, col = np.nonzero(mask)
    row = row.astype(np.int64)
    col = col.astype(np.int64)
    return Coo(m, n, row, col, _values(seed, row.shape[0], dtype, int_mode), f"rand-{m}x{n}-{seed}")


def random_powerlaw(m: int, n: int, seed: int, max_len: int, dtype=np.float64,
                    int_mode: bool = False) -> Coo:
    """Rows with Zipf-like lengths (some empty, a few long): exercises ragged tails."""
    g = rng(seed, STREAM_MATRIX)
    lens = np.minimum((g.pareto(1.2, size=m) * 2).astype(np.int64), min(max_len, n))
    rows, cols = [], []
    for r in range(m):
        if lens[r]:
            c = np.sort(g.choice(n, size=int(lens[r]), replace=False))
            rows.append(np.full(c.shape[0], r, dtype=np.int64))
            cols.append(c.astype(np.int64))
    row = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    col = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    return Coo(m, n, row, col, _values(seed, row.shape[0], dtype, int_mode), f"powerlaw-{m}-{seed}")


# ----------------------------------------------------------------------------------
# C1 uniform-1k
# ----------------------------------------------------------------------------------
def c1_uniform(m: int = 1000, nnz: int = 10_000, seed: int = 1, dtype=np.float64,
               int_mode: bool = False) -> Coo:
    """Diagonal + (nnz - m) distinct off-diagonal positions uniform over the m^2 - m
    off-diagonal cells (BASELINE configs[0])."""
    g = rng(seed, STREAM_MATRIX)
    off = g.choice(m * m - m, size=nnz - m, replace=False).astype(np.int64)
    r = off // (m - 1)
    c = off % (m - 1)
    c = c + (c >= r)  # skip the diagonal cell of row r
    row = np.concatenate([r, np.arange(m, dtype=np.int64)])
    col = np.concatenate([c, np.arange(m, dtype=np.int64)])
    row, col = _sorted_unique(m, m, row, col)
    assert row.shape[0] == nnz
    return Coo(m, m, row, col, _values(seed, nnz, dtype, int_mode), "uniform-1k")


# ----------------------------------------------------------------------------------
# C2 lap2d-2048
# ----------------------------------------------------------------------------------
def c2_lap2d(grid: int = 2048, dtype=np.float64) -> Coo:
    """5-point stencil: row i = gx + grid*gy; (i,i)=4; (i,i+-1)=-1 in the same grid row;
    (i,i+-grid)=-1 when in range.  nnz = 5*grid^2 - 4*grid."""
    m = grid * grid
    i = np.arange(m, dtype=np.int64)
    gx = i % grid
    gy = i // grid
    parts_r, parts_c, parts_v = [], [], []
    for dc, ok, v in ((-grid, gy > 0, -1.0), (-1, gx > 0, -1.0), (0, np.ones(m, bool), 4.0),
                      (1, gx < grid - 1, -1.0), (grid, gy < grid - 1, -1.0)):
        rr = i[ok]
        parts_r.append(rr)
        parts_c.append(rr + dc)
        parts_v.append(np.full(rr.shape[0], v))
    row = np.concatenate(parts_r)
    col = np.concatenate(parts_c)
    val = np.concatenate(parts_v)
    order = np.lexsort((col, row))
    return Coo(m, m, row[order], col[order], val[order].astype(dtype), f"lap2d-{grid}")


def c2_lap2d_band(grid: int, ny: int, gy0: int, gy1: int, dtype=np.float64) -> "Csr":
    """Rows of the 5-point stencil on a grid x ny grid (row i = gx + grid*gy) whose grid row
    gy lies in [gy0, gy1), with GLOBAL column indices (n = grid*ny).  The ROW_DIV band of
    rank r in the weak-scaled C2 (ny = grid*P, band = grid rows [grid*r, grid*(r+1))).
    c2_lap2d_band(g, g, 0, g) has exactly the rows of c2_lap2d(g)."""
    r0, r1 = gy0 * grid, gy1 * grid
    i = np.arange(r0, r1, dtype=np.int64)
    gx, gy = i % grid, i // grid
    # per row, the 5 candidate columns in ascending order with their presence mask
    cand = np.stack([i - grid, i - 1, i, i + 1, i + grid], axis=1)
    ok = np.stack([gy > 0, gx > 0, np.ones_like(gx, bool), gx < grid - 1, gy < ny - 1], axis=1)
    vals = np.array([-1.0, -1.0, 4.0, -1.0, -1.0])
    rl = ok.sum(axis=1)
    rp = np.zeros(r1 - r0 + 1, np.int64)
    np.cumsum(rl, out=rp[1:])
    col = cand[ok].astype(np.int32)
    val = np.broadcast_to(vals, cand.shape)[ok].astype(dtype)
    return Csr(r1 - r0, grid * ny, rp, col, val, f"lap2d-{grid}x{ny}-band{gy0}")


# ----------------------------------------------------------------------------------
# C3 rmat
# ----------------------------------------------------------------------------------
def c3_rmat(scale: int = 24, nnz: int = 1 << 28, seed: int = 3, dtype=np.float32,
            int_mode: bool = False, abcd=(0.57, 0.19, 0.19, 0.05)) -> Coo:
    """Graph500 R-MAT (no noise), labels permuted, self-loops and duplicates dropped,
    diagonal added; edges drawn until nnz is reached exactly (first occurrences kept
    in draw order).  SURVEY §8(d) C3."""
    n = 1 << scale
    g = rng(seed, STREAM_MATRIX)
    a, b, c, _ = abcd
    perm = g.permutation(n).astype(np.int64)
    target_off = nnz - n
    keys = np.zeros(0, np.int64)
    order_idx = np.zeros(0, np.int64)
    drawn = 0
    batch = max(1 << 16, min(1 << 24, int(target_off * 1.3)))
    while True:
        r = np.zeros(batch, np.int64)
        cc = np.zeros(batch, np.int64)
        for _ in range(scale):
            u = g.random(batch)
            rbit = u >= a + b
            cbit = ((u >= a) & (u < a + b)) | (u >= a + b + c)
            r = (r << 1) | rbit
            cc = (cc << 1) | cbit
        r = perm[r]
        cc = perm[cc]
        keep = r != cc
        k = r[keep] * n + cc[keep]
        idx = drawn + np.nonzero(keep)[0].astype(np.int64)
        drawn += batch
        keys = np.concatenate([keys, k])
        order_idx = np.concatenate([order_idx, idx])
        uk, first = np.unique(keys, return_index=True)
        keys = uk
        order_idx = order_idx[first]
        if keys.shape[0] >= target_off:
            break
    sel = np.argsort(order_idx, kind="stable")[:target_off]
    k = np.sort(keys[sel])
    row = np.concatenate([k // n, np.arange(n, dtype=np.int64)])
    col = np.concatenate([k % n, np.arange(n, dtype=np.int64)])
    row, col = _sorted_unique(n, n, row, col)
    assert row.shape[0] == nnz
    return Coo(n, n, row, col, _values(seed, nnz, dtype, int_mode), f"rmat-{scale}")


# ----------------------------------------------------------------------------------
# C4 blockdense
# ----------------------------------------------------------------------------------
def c4_blockdense(m: int = 8_388_608, b: int = 64, n_tiles: int = 24_576,
                  nnz: int = 200_000_000, seed: int = 4, dtype=np.float64,
                  int_mode: bool = False):
    """Planted fully dense b x b tiles (tile rows without replacement, tile col uniform),
    + diagonal, + uniform scattered entries outside planted tiles (dedup) until nnz
    exactly.  Returns (Coo, planted_tiles[(I, J)] sorted).  SURVEY §8(d) C4."""
    g = rng(seed, STREAM_MATRIX)
    nt = m // b
    I = np.sort(g.choice(nt, size=n_tiles, replace=False)).astype(np.int64)
    J = g.integers(0, nt, size=n_tiles).astype(np.int64)
    ii, jj = np.meshgrid(np.arange(b, dtype=np.int64), np.arange(b, dtype=np.int64), indexing="ij")
    tr = (I[:, None, None] * b + ii[None]).reshape(-1)
    tc = (J[:, None, None] * b + jj[None]).reshape(-1)
    diag = np.arange(m, dtype=np.int64)
    base = np.unique(np.concatenate([tr * m + tc, diag * m + diag]))
    tile_key = np.sort(I * nt + J)
    need = nnz - base.shape[0]
    extra = np.zeros(0, np.int64)
    while extra.shape[0] < need:
        cnt = int((need - extra.shape[0]) * 1.05) + 1024
        r = g.integers(0, m, size=cnt).astype(np.int64)
        c = g.integers(0, m, size=cnt).astype(np.int64)
        tk = (r // b) * nt + (c // b)
        pos = np.searchsorted(tile_key, tk)
        pos = np.minimum(pos, tile_key.shape[0] - 1)
        in_tile = tile_key[pos] == tk
        k = (r * m + c)[~in_tile]
        k = k[~np.isin(k, base, assume_unique=False)]
        allk = np.concatenate([extra, k])
        _, first = np.unique(allk, return_index=True)
        extra = allk[np.sort(first)]
    extra = extra[:need]
    keys = np.sort(np.concatenate([base, extra]))
    row, col = keys // m, keys % m
    assert row.shape[0] == nnz
    tiles = np.stack([I, J], axis=1)
    tiles = tiles[np.lexsort((tiles[:, 1], tiles[:, 0]))]
    return Coo(m, m, row, col, _values(seed, nnz, dtype, int_mode), "blockdense"), tiles


# ----------------------------------------------------------------------------------
# C5 band-irregular
# ----------------------------------------------------------------------------------
def c5_band_irreg_csr(m: int = 67_108_864, nnz: int = 1 << 30, band: int = 4096, seed: int = 5,
                      dtype=np.float64, int_mode: bool = False):
    """Row lengths L_i ~ 0.9*U{4..16} + 0.1*U{17..123}, adjusted by a seeded round-robin
    +-1 until sum = nnz; columns = diagonal + (L_i - 1) distinct uniform in
    [i-band, i+band] \\cap [0, m) \\ {i}.  Returned as CSR (row_ptr int64, col int32,
    val) to keep the 1B-nnz instance within host memory.  SURVEY §8(d) C5."""
    g = rng(seed, STREAM_MATRIX)
    short = g.integers(4, 17, size=m)
    long_ = g.integers(17, 124, size=m)
    L = np.where(g.random(m) < 0.9, short, long_).astype(np.int64)
    lo = np.maximum(np.arange(m) - band, 0)
    hi = np.minimum(np.arange(m) + band, m - 1)
    cap = (hi - lo + 1).astype(np.int64)  # window size incl. diagonal
    L = np.minimum(L, cap)
    diff = int(nnz - L.sum())
    order = g.permutation(m)
    step = 1 if diff > 0 else -1
    pos = 0
    while diff != 0:
        k = min(abs(diff), m)
        idx = order[(pos + np.arange(k)) % m]
        ok = (L[idx] < cap[idx]) if step > 0 else (L[idx] > 1)
        idx = idx[ok]
        L[idx] += step
        diff -= step * idx.shape[0]
        pos += k
    row_ptr = np.zeros(m + 1, np.int64)
    np.cumsum(L, out=row_ptr[1:])
    col = np.empty(int(row_ptr[-1]), np.int32)
    chunk = 1 << 20
    for r0 in range(0, m, chunk):
        r1 = min(m, r0 + chunk)
        _fill_band_rows(g, r0, r1, L, lo, hi, row_ptr, col)
    val = _values(seed, col.shape[0], dtype, int_mode)
    return m, row_ptr, col, val


def _fill_band_rows(g, r0, r1, L, lo, hi, row_ptr, col):
    rows = np.arange(r0, r1, dtype=np.int64)
    need = L[r0:r1] - 1
    # draw with oversampling, dedup per row, redraw the few short rows
    out_keys = []
    pending = rows
    pneed = need
    over = 2
    while pending.shape[0]:
        cnt = pneed * over + 4
        rr = np.repeat(pending, cnt)
        width = (hi[pending] - lo[pending]).astype(np.int64)  # excludes diagonal
        u = g.integers(0, np.repeat(width, cnt))
        cc = np.repeat(lo[pending], cnt) + u
        cc = cc + (cc >= rr)
        key = rr * (1 << 32) + cc
        # first occurrence per (row, col) in draw order
        _, first = np.unique(key, return_index=True)
        first.sort()
        key = key[first]
        rk = key >> 32
        # rank within row in draw order
        order = np.argsort(rk, kind="stable")
        key = key[order]
        rk = rk[order]
        bounds = np.searchsorted(rk, pending)
        counts = np.diff(np.append(bounds, rk.shape[0]))
        ok = counts >= pneed
        rank = np.arange(rk.shape[0]) - np.repeat(bounds, counts)
        take = rank < np.repeat(pneed, counts)
        take &= np.repeat(ok, counts)
        out_keys.append(key[take])
        pending = pending[~ok]
        pneed = pneed[~ok]
        over *= 2
    keys = np.concatenate(out_keys + [rows * (1 << 32) + rows])
    keys.sort()
    col[row_ptr[r0]:row_ptr[r1]] = (keys & ((1 << 32) - 1)).astype(np.int32)


def csr_to_coo(m, n, row_ptr, col, val, name="") -> Coo:
    row = np.repeat(np.arange(m, dtype=np.int64), np.diff(row_ptr))
    return Coo(m, n, row, col.astype(np.int64), val, name)


# ----------------------------------------------------------------------------------
# Fast multithreaded C generators for the full-size configs (synth/gen.c)
# ----------------------------------------------------------------------------------
@dataclasses.dataclass
class Csr:
    m: int
    n: int
    row_ptr: np.ndarray  # int64[m+1]
    col: np.ndarray      # int32[nnz], ascending within a row
    val: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_coo(self) -> Coo:
        return csr_to_coo(self.m, self.n, self.row_ptr, self.col, self.val, self.name)

    def rows(self, rows):
        """Sub-CSR of the given rows (for sampled oracle checks)."""
        rows = np.asarray(rows, np.int64)
        a, e = self.row_ptr[rows], self.row_ptr[rows + 1]
        rp = np.concatenate([[0], np.cumsum(e - a)])
        idx = np.concatenate([np.arange(x, y) for x, y in zip(a, e)]) if rows.shape[0] else np.zeros(0, np.int64)
        return rp, self.col[idx].astype(np.int64), self.val[idx]


_GEN = None


def _gen():
    global _GEN
    if _GEN is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, lib = os.path.join(here, "gen.c"), os.path.join(here, "libsynth.so")
        if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
            subprocess.check_call(["gcc", "-O3", "-shared", "-fPIC", "-pthread", src, "-o", lib])
        L = ctypes.CDLL(lib)
        i64, vp, u64 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_uint64
        L.synth_values.argtypes = [u64, i64, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int]
        L.synth_c5.argtypes = [i64, i64, i64, u64, vp, vp, ctypes.c_int]
        L.synth_c5_rowptr.argtypes = [i64, i64, i64, u64, vp, ctypes.c_int]
        L.synth_c5_band.argtypes = [i64, i64, u64, vp, i64, i64, vp, ctypes.c_int]
        L.synth_values_range.argtypes = [u64, i64, i64, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int]
        L.synth_c4.argtypes = [i64, i64, i64, i64, u64, vp, vp, vp, ctypes.c_int]
        L.synth_c3.argtypes = [ctypes.c_int, i64, ctypes.c_double, ctypes.c_double, ctypes.c_double, u64, vp, vp,
                               ctypes.c_int]
        _GEN = L
    return _GEN


def _nth():
    import os
    return os.cpu_count() or 1


def _fast_values(seed, nnz, dtype, int_mode):
    val = np.empty(nnz, dtype)
    _gen().synth_values(seed, nnz, int(int_mode), int(np.dtype(dtype) == np.float32), val.ctypes.data, _nth())
    return val


def c5_band_csr(m: int = 67_108_864, nnz: int = 1 << 30, band: int = 4096, seed: int = 5,
                dtype=np.float64, int_mode: bool = False) -> Csr:
    """C5 band-irreg-64m (BASELINE configs[4]) via synth/gen.c."""
    rp = np.empty(m + 1, np.int64)
    col = np.empty(nnz, np.int32)
    rc = _gen().synth_c5(m, nnz, band, seed, rp.ctypes.data, col.ctypes.data, _nth())
    if rc:
        raise ValueError("C5 row-length adjustment failed (nnz not reachable)")
    return Csr(m, m, rp, col, _fast_values(seed, nnz, dtype, int_mode), "band-irreg")


def c5_row_ptr(m: int = 67_108_864, nnz: int = 1 << 30, band: int = 4096, seed: int = 5) -> np.ndarray:
    """row_ptr of C5 alone (row lengths + the seeded adjustment; 0.5 GB, no columns)."""
    rp = np.empty(m + 1, np.int64)
    if _gen().synth_c5_rowptr(m, nnz, band, seed, rp.ctypes.data, _nth()):
        raise ValueError("C5 row-length adjustment failed (nnz not reachable)")
    return rp


def c5_band_rows(row_ptr: np.ndarray, r0: int, r1: int, band: int = 4096, seed: int = 5, dtype=np.float64,
                 int_mode: bool = False) -> "Csr":
    """Rows [r0, r1) of C5 as a CSR band with global columns -- bit-identical to the same
    rows of c5_band_csr (counter-based per-row draws and per-nonzero values), generated
    without the rest of the matrix (a multi-GPU rank's ROW_DIV band)."""
    m = row_ptr.shape[0] - 1
    a, e = int(row_ptr[r0]), int(row_ptr[r1])
    col = np.empty(e - a, np.int32)
    _gen().synth_c5_band(m, band, seed, np.ascontiguousarray(row_ptr, np.int64).ctypes.data, r0, r1,
                         col.ctypes.data, _nth())
    val = np.empty(e - a, dtype)
    _gen().synth_values_range(seed, a, e - a, int(int_mode), int(np.dtype(dtype) == np.float32), val.ctypes.data,
                              _nth())
    return Csr(r1 - r0, m, (row_ptr[r0:r1 + 1] - a).astype(np.int64), col, val, "band-irreg")


def c4_blockdense_csr(m: int = 8_388_608, b: int = 64, n_tiles: int = 24_576, nnz: int = 200_000_000,
                      seed: int = 4, dtype=np.float64, int_mode: bool = False):
    """C4 blockdense-8m (BASELINE configs[3]) via synth/gen.c -> (Csr, tiles[(I, J)] sorted)."""
    rp = np.empty(m + 1, np.int64)
    col = np.empty(nnz, np.int32)
    tiles = np.empty((n_tiles, 2), np.int64)
    rc = _gen().synth_c4(m, b, n_tiles, nnz, seed, tiles.ctypes.data, rp.ctypes.data, col.ctypes.data, _nth())
    if rc:
        raise ValueError(f"C4 generation failed ({rc})")
    tiles = tiles[np.lexsort((tiles[:, 1], tiles[:, 0]))]
    return Csr(m, m, rp, col, _fast_values(seed, nnz, dtype, int_mode), "blockdense"), tiles


def c3_rmat_csr(scale: int = 24, nnz: int = 1 << 28, seed: int = 3, dtype=np.float32, int_mode: bool = False,
                abcd=(0.57, 0.19, 0.19, 0.05)) -> Csr:
    """C3 rmat-24 (BASELINE configs[2]) via synth/gen.c."""
    n = 1 << scale
    rp = np.empty(n + 1, np.int64)
    col = np.empty(nnz, np.int32)
    rc = _gen().synth_c3(scale, nnz, abcd[0], abcd[1], abcd[2], seed, rp.ctypes.data, col.ctypes.data, _nth())
    if rc:
        raise ValueError(f"C3 generation failed ({rc})")
    return Csr(n, n, rp, col, _fast_values(seed, nnz, dtype, int_mode), f"rmat-{scale}")
