"""Run a few as_spmv calls per graph on a generated config (for ncu captures; developer tool).

    python tools/run_graphs.py c5s "G1" "G2" ...     (c5s = C5 shape at 1/16 scale)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2212_10432_b200 as asp  # noqa: E402

CONFIGS = {
    "c5s": lambda: synth.c5_band_csr(m=1 << 22, nnz=1 << 26),
    "c3s": lambda: synth.c3_rmat_csr(scale=22, nnz=1 << 26),
    "c4s": lambda: synth.c4_blockdense_csr(m=1 << 21, b=64, n_tiles=6144, nnz=50_000_000)[0],
}


def main():
    if sys.argv[1] in CONFIGS:
        c = CONFIGS[sys.argv[1]]()
    else:  # full-size BASELINE configs (c1..c5)
        import bench
        c = bench.to_csr(bench.load_config(sys.argv[1])[0])
    A = asp.Matrix.from_csr(c.m, c.n, c.row_ptr, c.col, c.val)
    tdt = torch.float64 if c.val.dtype.itemsize == 8 else torch.float32
    x = torch.rand(c.n, dtype=tdt, device="cuda")
    y = torch.zeros(c.m, dtype=tdt, device="cuda")
    for g in sys.argv[2:]:
        P = asp.Plan(A, g, device=0)
        for _ in range(3):
            P.spmv(1.0, x, 0.0, y)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
