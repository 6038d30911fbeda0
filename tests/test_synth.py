"""The seeded generators produce what DESIGN.md §5 says (structure only; no method arithmetic)."""
import numpy as np

import synth


def _check_csr(c):
    rp, col = c.row_ptr, c.col.astype(np.int64)
    assert rp[0] == 0 and rp[-1] == c.nnz and np.all(np.diff(rp) >= 0)
    r = np.repeat(np.arange(c.m), np.diff(rp))
    key = r * c.n + col
    assert np.all(np.diff(key) > 0)          # sorted, no duplicates
    assert col.min() >= 0 and col.max() < c.n
    return r, col


def test_c5_band_structure():
    c = synth.c5_band_csr(m=1 << 16, nnz=1 << 20, band=256)
    r, col = _check_csr(c)
    assert c.nnz == 1 << 20
    assert np.all(np.abs(col - r) <= 256)
    diag = np.zeros(c.m, bool)
    diag[r[col == r]] = True
    assert diag.all()                         # every row holds its diagonal (no empty rows)
    lens = np.diff(c.row_ptr)
    assert abs(lens.mean() - 16.0) < 1e-9
    # deterministic and thread-count independent
    c2 = synth.c5_band_csr(m=1 << 16, nnz=1 << 20, band=256)
    assert np.array_equal(c.col, c2.col) and np.array_equal(c.val, c2.val)


def test_c4_planted_tiles():
    c, tiles = synth.c4_blockdense_csr(m=1 << 16, b=64, n_tiles=200, nnz=1_200_000, seed=9)
    r, col = _check_csr(c)
    assert c.nnz == 1_200_000
    assert len(set(tiles[:, 0].tolist())) == 200
    present = set((r * c.n + col).tolist())
    for I, J in tiles[:5]:
        for i in (0, 17, 63):
            for j in (0, 31, 63):
                assert (I * 64 + i) * c.n + J * 64 + j in present
    assert all(i * c.n + i in present for i in range(0, c.m, 997))


def test_c3_rmat_structure():
    c = synth.c3_rmat_csr(scale=14, nnz=1 << 18, dtype=np.float32)
    r, col = _check_csr(c)
    assert c.nnz == 1 << 18 and c.val.dtype == np.float32
    lens = np.diff(c.row_ptr)
    assert lens.min() >= 1                    # diagonal added: no empty rows
    assert lens.max() > 20 * lens.mean()      # power-law hubs


def test_value_modes():
    v = synth._fast_values(3, 10000, np.float64, True)
    assert set(np.unique(v).tolist()) <= {-4, -3, -2, -1, 1, 2, 3, 4}
    v = synth._fast_values(3, 10000, np.float64, False)
    assert v.min() >= -1 and v.max() < 1 and abs(v.mean()) < 0.05


def test_lap2d_band_weak_scaling():
    """bench.py's weak-scaled C2: band r of the grid x (grid*P) Laplacian; one band of a square
    grid is C2 itself, and the P bands stacked are the whole taller Laplacian (nnz closed form
    5*g*ny - 2*g - 2*ny)."""
    import numpy as np
    import synth
    g = 32
    full = synth.c2_lap2d(g)
    b = synth.c2_lap2d_band(g, g, 0, g)
    rp = np.zeros(full.m + 1, np.int64)
    np.add.at(rp, full.row + 1, 1)
    assert np.array_equal(np.cumsum(rp), b.row_ptr) and np.array_equal(full.col, b.col)
    assert np.array_equal(full.val, b.val)
    P = 3
    bands = [synth.c2_lap2d_band(g, g * P, g * r, g * (r + 1)) for r in range(P)]
    tall = synth.c2_lap2d_band(g, g * P, 0, g * P)
    assert sum(x.nnz for x in bands) == tall.nnz == 5 * g * (g * P) - 2 * g - 2 * (g * P)
    assert np.array_equal(np.concatenate([x.col for x in bands]), tall.col)
    assert all(x.n == g * g * P for x in bands)


def test_c5_band_rows_equal_whole_matrix():
    """A rank's ROW_DIV band generated alone equals the same rows of the whole matrix."""
    m, nnz = 1 << 16, 1 << 20
    A = synth.c5_band_csr(m=m, nnz=nnz, band=512)
    rp = synth.c5_row_ptr(m=m, nnz=nnz, band=512)
    assert np.array_equal(rp, A.row_ptr)
    for r0, r1 in [(0, 1000), (12345, 40000), (m - 77, m)]:
        b = synth.c5_band_rows(rp, r0, r1, band=512)
        a, e = int(rp[r0]), int(rp[r1])
        assert b.m == r1 - r0 and b.n == m
        assert np.array_equal(b.row_ptr, rp[r0:r1 + 1] - a)
        assert np.array_equal(b.col, A.col[a:e])
        assert np.array_equal(b.val, A.val[a:e])
