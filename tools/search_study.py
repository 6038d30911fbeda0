"""NEXT-3 study of as_search on synthetic matrices (developer measurement tool):

  * surrogate accuracy: mean absolute deviation |pred - measured| / measured of the cost
    model's predictions for the candidates it nominated (the paper: ~5 %);
  * iterations to the best: the index (in evaluation order) of the first candidate within
    1 % of the search's final best time, regular (row-length variance <= 100, A39) vs
    irregular matrices (the paper: regular matrices need 3.5x fewer iterations).

    python tools/search_study.py --budget 60 --seeds 3 > gpurun_out/search_study.jsonl
"""
import argparse
import json
import os
import statistics
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def matrices():
    import synth
    yield "lap2d-1024 (regular)", synth.c2_lap2d(1024)
    yield "uniform-2m (regular)", synth.c1_uniform(m=1 << 21, nnz=1 << 24, seed=11)
    yield "band-irreg-4m", synth.c5_band_csr(m=1 << 22, nnz=1 << 26)
    yield "rmat-21", synth.c3_rmat_csr(scale=21, nnz=1 << 25)
    yield "powerlaw-1m", synth.random_powerlaw(1 << 20, 1 << 20, 3, 20000)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=60.0)
    ap.add_argument("--candidates", type=int, default=48)
    ap.add_argument("--seeds", type=int, default=2)
    args = ap.parse_args()
    import paper_2212_10432_b200 as asp
    for name, M in matrices():
        if hasattr(M, "row_ptr"):
            A = asp.Matrix.from_csr(M.m, M.n, M.row_ptr, M.col, M.val)
        else:
            A = asp.Matrix.from_coo(M.m, M.n, M.row, M.col, M.val)
        st = A.stats()
        for seed in range(1, args.seeds + 1):
            with tempfile.NamedTemporaryFile(suffix=".jsonl", delete=False) as f:
                log = f.name
            P, g = asp.search(A, device=0, seed=seed, max_candidates=args.candidates, budget_seconds=args.budget,
                              warmup=2, reps=7, log_path=log)
            rows = [json.loads(l) for l in open(log)]
            os.unlink(log)
            timed = [r for r in rows if r["median_ms"] > 0 and r["status"] in
                     ("ok", "model", "refine", "sample", "sample_model", "sample_refine")]
            best = min(r["median_ms"] for r in timed)
            first = next(k for k, r in enumerate(timed) if r["median_ms"] <= 1.01 * best)
            mad = [abs(r["pred_ms"] - r["median_ms"]) / r["median_ms"] for r in timed if "pred_ms" in r]
            print(json.dumps({"matrix": name, "seed": seed, "variance": st["row_len_variance"],
                              "irregular": bool(st["irregular"]), "timed": len(timed), "best_ms": best,
                              "iterations_to_best": first + 1, "model_candidates": len(mad),
                              "surrogate_mad": statistics.mean(mad) if mad else None, "winner": g}), flush=True)
            del P


if __name__ == "__main__":
    main()
