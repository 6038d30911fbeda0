"""Kernel sweep (developer tool): time a list of graphs on one config, L2 flushed before each
rep, CUDA events around each as_spmv; prints one JSON line per graph.

    python tools/sweep.py --config c2 --graphs "G1" "G2" ...   [--env AS_DIA_VARIANT=1]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--graphs", nargs="+", required=True)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--beta", type=float, default=0.0)
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import synth
    import paper_2212_10432_b200 as asp
    coo, wl, _ = bench.load_config(args.config)
    coo = bench.to_csr(coo)
    A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
    x, y0 = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y0).cuda()
    flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
    for g in args.graphs:
        try:
            P = asp.Plan(A, g, device=0)
        except asp.AsError as e:
            print(json.dumps({"graph": g, "error": str(e)}))
            continue
        info = P.info()
        for _ in range(3):
            P.spmv(1.0, dx, args.beta, dy)
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            flush.view(torch.int64).sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P.spmv(1.0, dx, args.beta, dy)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        med = statistics.median(ts)
        P.spmv(1.0, dx, 0.0, dy)
        ysum = float(dy.double().abs().sum())  # cross-variant sanity (same y up to rounding)
        bm = info["bytes_model"] if args.beta == 0 else info["bytes_model_beta"]
        print(json.dumps({"config": wl, "graph": g, "env": {k: v for k, v in os.environ.items() if k.startswith("AS_")},
                          "median_us": med * 1e3, "min_us": min(ts) * 1e3, "gflops": 2 * coo.nnz / (med * 1e-3) / 1e9,
                          "model_gbs": bm / (med * 1e-3) / 1e9, "kernels": info["kernels"], "bytes_model": bm,
                          "y_abs_sum": ysum, "lib": os.environ.get("AS_LIB_AB", "")}))
        del P


if __name__ == "__main__":
    main()
