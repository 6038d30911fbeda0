"""A/B of as_search with and without the cost-model stage (developer tool): same seed,
same budget, no seed graphs; prints the best graph and its re-timed median per run.

    python tools/search_ab.py --config c5s --budget 30 [--no-surrogate]
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
    ap.add_argument("--config", default="c5s")
    ap.add_argument("--budget", type=float, default=30.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-surrogate", action="store_true")
    args = ap.parse_args()
    if args.no_surrogate:
        os.environ["AS_SEARCH_NO_SURROGATE"] = "1"
    import torch
    import bench
    import synth
    import paper_2212_10432_b200 as asp
    coo, wl, _ = bench.load_config(args.config)
    coo = bench.to_csr(coo)
    A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
    log = os.path.join(ROOT, "gpurun_out", f"search_ab_{args.config}_{'base' if args.no_surrogate else 'model'}.jsonl")
    P, g = asp.search(A, device=0, seed=args.seed, max_candidates=64, budget_seconds=args.budget, warmup=2, reps=5,
                      log_path=log)
    x, _ = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    dx = torch.from_numpy(x).cuda()
    dy = torch.zeros(coo.m, dtype=dx.dtype, device="cuda")
    flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        P.spmv(1.0, dx, 0.0, dy)
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.spmv(1.0, dx, 0.0, dy)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    n_eval = sum(1 for _ in open(log))
    print(json.dumps({"config": wl, "surrogate": not args.no_surrogate, "budget_s": args.budget, "candidates": n_eval,
                      "best_us": statistics.median(ts) * 1e3, "graph": g}))


if __name__ == "__main__":
    main()
