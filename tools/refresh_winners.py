"""Longer as_search runs on full-size configs to refresh profiles/best_graphs.json (developer
tool; the bench seeds its own searches with the committed winners).

    python tools/refresh_winners.py --configs c4 c5 --budget 240 > gpurun_out/refresh.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c4", "c5"])
    ap.add_argument("--budget", type=float, default=240.0)
    ap.add_argument("--candidates", type=int, default=160)
    args = ap.parse_args()
    import bench
    import paper_2212_10432_b200 as asp
    for cfg in args.configs:
        coo, wl, seeds = bench.load_config(cfg)
        coo = bench.to_csr(coo)
        A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
        t = time.perf_counter()
        log = os.path.join(ROOT, "gpurun_out", f"search_{wl}_refresh.jsonl")
        P, g = asp.search(A, device=0, seed=7, max_candidates=args.candidates, budget_seconds=args.budget, warmup=3,
                          reps=10, seed_graphs=seeds, log_path=log)
        rows = [json.loads(l) for l in open(log)]
        best = [r for r in rows if r["graph"] == g and r["median_ms"] > 0]
        print(json.dumps({"config": wl, "winner": g, "search_s": time.perf_counter() - t, "timed": len(rows),
                          "winner_ms": min(r["median_ms"] for r in best) if best else None,
                          "seed_ms": [r["median_ms"] for r in rows if r["i"] < len(seeds)]}), flush=True)
        del P, A


if __name__ == "__main__":
    main()
