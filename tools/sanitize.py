"""Run every kernel form once on small matrices (for compute-sanitizer memcheck / racecheck /
synccheck; developer tool).  Each graph is checked against the oracle as well."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2212_10432_b200 as asp  # noqa: E402
from oracle import spmv as S  # noqa: E402
from test_host import CONC_GRAPHS, FAMILY_GRAPHS  # noqa: E402

EXTRA = [
    "DIA_DECOM(theta=0.5,max=8) { DIA | COMPRESS; BMT_NNZ_BLOCK(3); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
    "DENSE_DECOM(b=64,theta=0.3) { DENSE | COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }",
    "COMPRESS; BMTB_NNZ_BLOCK(100); SHMEM_OFFSET_RED; SET_RESOURCE(tpb=128,grid=0,stages=2); GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024); GMEM_ATOM_RED",
    "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED",
    "COMPRESS; BMT_NNZ_BLOCK(64); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED",
]


def main():
    fails = 0
    cases = [(synth.random_powerlaw(900, 800, 3, 300), FAMILY_GRAPHS + EXTRA[:3] + CONC_GRAPHS),
             (synth.c5_band_csr(m=1 << 19, nnz=1 << 23, band=512).to_coo(), EXTRA[3:])]  # x-window form
    for coo, graphs in cases:
        A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
        x, y0 = synth.vectors(coo.n, coo.m, 1)
        for alpha, beta in ((1.5, -0.5), (1.0, 0.0)):  # generic and STORE/beta=0 epilogues
            yref, bnd = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, alpha, beta, y0)
            for g in graphs:
                try:
                    P = asp.Plan(A, g, device=0)
                except asp.AsError as e:
                    print("infeasible", g[:60], e)
                    continue
                dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda()
                P.spmv(alpha, dx, beta, dy)
                torch.cuda.synchronize()
                ok, ratio = S.check(dy.cpu().numpy(), yref, bnd, np.float64)
                fails += not ok
                print("ok " if ok else "BAD", beta, P.info()["kernels"], g[:70])
    # SpMM kernels (DMMA dense tiles, DIA, CSR parts), k = 70 (ragged column chunk)
    coo = synth.random_powerlaw(900, 800, 3, 300)
    A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
    for g in ["DENSE_DECOM(b=64,theta=0.02) { DENSE | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED }",
              "DIA_DECOM(theta=0.01,max=8) { DIA | COMPRESS; BMT_NNZ_BLOCK(5); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }"]:
        P = asp.Plan(A, g, device=0, spmm=True)
        X = torch.rand((coo.n, 70), dtype=torch.float64, device="cuda")
        Y = torch.rand((coo.m, 70), dtype=torch.float64, device="cuda")
        P.spmm(1.5, X, -0.5, Y)
        torch.cuda.synchronize()
        print("ok  spmm", P.info()["kernels"], g[:60])
    print("failures:", fails)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
