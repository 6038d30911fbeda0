"""SpMM measurement (NEXT-4, developer tool): Y = A X on C4 (blockdense-8m, DENSE_DECOM tiles
on the fp64 DMMA tensor cores + CSR-family residual) for k right-hand sides; CUDA events,
L2 flushed before each rep; GFLOP/s = 2 * nnz * k / t.  One JSON line per (graph, k)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--k", type=int, nargs="+", default=[8, 16, 64])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--graphs", nargs="+", default=[
        "DENSE_DECOM(b=64,theta=0.5) { DENSE | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED }",
        "COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; GMEM_ATOM_RED"])
    args = ap.parse_args()
    import torch
    import bench
    import paper_2212_10432_b200 as asp
    coo, wl, _ = bench.load_config(args.config)
    coo = bench.to_csr(coo)
    A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
    tdt = torch.float64 if coo.val.dtype.itemsize == 8 else torch.float32
    flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
    for g in args.graphs:
        P = asp.Plan(A, g, device=0, spmm=True)
        for k in args.k:
            X = torch.rand((coo.n, k), dtype=tdt, device="cuda")
            Y = torch.zeros((coo.m, k), dtype=tdt, device="cuda")
            for _ in range(2):
                P.spmm(1.0, X, 0.0, Y)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                flush.view(torch.int64).sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                P.spmm(1.0, X, 0.0, Y)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            print(json.dumps({"workload": wl, "graph": g, "k": k, "ms": t, "gflops": 2 * coo.nnz * k / (t * 1e-3) / 1e9,
                              "kernels": P.info()["kernels"]}), flush=True)
            del X, Y


if __name__ == "__main__":
    main()
