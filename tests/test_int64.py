"""Index widths (A36: narrowest lossless per array, int32 below 2^31).  The device arrays that
hold row / column / BMT ids stay int32; element positions are computed in int64 by the
kernels (implicit NNZ block starts t*k, int64 BMT_PAD group bases), so a part with more
than 2^31 nonzeros runs, and a stored offset array that would overflow int32 is rejected with
an A36 message.  This test plans a banded matrix with 2^31 + 2^24 nonzeros (fp32) through
the on-device Designer and checks the rows around the 2^31 element boundary, the first and
last rows and random windows against the long-double oracle.  The int32 side of A36 is
every other GPU test."""
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

NNZ = (1 << 31) + (1 << 24)
M = NNZ // 16


def _mem_available_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return 0.0


@pytest.fixture(scope="module")
def big():
    if _mem_available_gb() < 160:
        pytest.skip(f"needs ~160 GB of host memory, {_mem_available_gb():.0f} GB available")
    free, _ = torch.cuda.mem_get_info()
    if free < 80 * 2**30:
        pytest.skip("needs ~80 GB of device memory")
    c = synth.c5_band_csr(m=M, nnz=NNZ, band=4096, seed=31, dtype=np.float32)
    assert c.row_ptr[-1] == NNZ > 2**31
    return c


def _windows(c):
    b = int(np.searchsorted(c.row_ptr, 2**31, side="right")) - 1  # row holding element 2^31
    rng = np.random.default_rng(5)
    wins = [(0, 20000), (max(0, b - 20000), min(c.m, b + 20000)), (c.m - 20000, c.m)]
    wins += [(int(r), min(c.m, int(r) + 5000)) for r in rng.integers(0, c.m - 5000, 12)]
    return wins


@pytest.mark.parametrize("graph", [
    "COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=0); THREAD_BITMAP_RED_G; "
    "SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=0); GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(nnz=8192); BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; "
    "WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=4096); GMEM_ATOM_RED",
])
def test_more_than_2pow31_nonzeros(big, graph):
    c = big
    A = asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)
    P = asp.Plan(A, graph, device=0)
    info = P.info()
    assert info["device_built"] == 1 and info["nnz_real"] == NNZ
    x, y0 = synth.vectors(c.n, c.m, 3, np.float32)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
    P.spmv(1.25, dx, -0.5, dy)
    torch.cuda.synchronize()
    y = dy.cpu().numpy()
    del P, A
    for r0, r1 in _windows(c):
        a, e = int(c.row_ptr[r0]), int(c.row_ptr[r1])
        rp = c.row_ptr[r0:r1 + 1] - a
        yref, bound = S.spmv_csr(rp, c.col[a:e], c.val[a:e].astype(np.float64), x.astype(np.float64), 1.25, -0.5,
                                 y0[r0:r1].astype(np.float64), nthreads=os.cpu_count() or 1)
        ok, ratio = S.check(y[r0:r1], yref, bound, np.float32)
        assert ok, (graph, r0, r1, ratio)


def test_stored_offsets_over_int32_rejected(big):
    """A stored offset array that would need int64 (explicit BMT starts: K % k != 0) is
    rejected naming A36 rather than truncated."""
    c = big
    A = asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)
    g = ("COMPRESS; BMW_NNZ_BLOCK(nnz=100); BMT_NNZ_BLOCK(nnz=7); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
         "SET_RESOURCE(stages=0); GMEM_ATOM_RED")
    with pytest.raises(asp.AsError, match="A36"):
        asp.Plan(A, g, device=0)
