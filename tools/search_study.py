"""NEXT-3 study of as_search on synthetic matrices (developer measurement tool):

  * surrogate accuracy: mean absolute deviation |pred - measured| / measured of the cost
    model's predictions for the candidates it nominated (the paper: ~5 %), fitted
    online on the search's own candidates, and (--history) with a history of the OTHER
    matrices' searches (graph + matrix features -> log time per nonzero: the paper's model
    is trained on other matrices) -- leave-one-matrix-out;
  * iterations to the best: the index (in evaluation order) of the first candidate within
    1 % / 3 % / 5 % of the search's final best time, regular (row-length variance <= 100,
    A39) vs irregular matrices (the paper: regular matrices need 3.5x fewer iterations).

    python tools/search_study.py --budget 45 --seeds 2 [--history] > gpurun_out/search_study.jsonl
"""
import argparse
import json
import os
import statistics
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TIMED = ("ok", "model", "refine", "sample", "sample_model", "sample_refine")


def matrices():
    import synth
    yield "lap2d-1024 (regular)", synth.c2_lap2d(1024)
    yield "uniform-2m (regular)", synth.c1_uniform(m=1 << 21, nnz=1 << 24, seed=11)
    yield "band-irreg-4m", synth.c5_band_csr(m=1 << 22, nnz=1 << 26)
    yield "rmat-21", synth.c3_rmat_csr(scale=21, nnz=1 << 25)
    yield "powerlaw-1m", synth.random_powerlaw(1 << 20, 1 << 20, 3, 20000)


def run(asp, A, seed, args, history=()):
    with tempfile.NamedTemporaryFile(suffix=".jsonl", delete=False) as f:
        log = f.name
    P, g = asp.search(A, device=0, seed=seed, max_candidates=args.candidates, budget_seconds=args.budget, warmup=2,
                      reps=7, log_path=log, history=history)
    rows = [json.loads(l) for l in open(log)]
    os.unlink(log)
    del P
    return g, rows


def summary(rows):
    timed = [r for r in rows if r["median_ms"] > 0 and r["status"] in TIMED]
    best = min(r["median_ms"] for r in timed)
    it = {f"iterations_to_best_{b}pct": next(k for k, r in enumerate(timed) if r["median_ms"] <= (1 + b / 100) * best) + 1
          for b in (1, 3, 5)}
    mad = [abs(r["pred_ms"] - r["median_ms"]) / r["median_ms"] for r in timed if "pred_ms" in r]
    return {"timed": len(timed), "best_ms": best, **it, "model_candidates": len(mad),
            "surrogate_mad": statistics.mean(mad) if mad else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=60.0)
    ap.add_argument("--candidates", type=int, default=48)
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--history", action="store_true", help="leave-one-matrix-out runs with the others' history")
    args = ap.parse_args()
    import paper_2212_10432_b200 as asp
    mats = []
    for name, M in matrices():
        if hasattr(M, "row_ptr"):
            A = asp.Matrix.from_csr(M.m, M.n, M.row_ptr, M.col, M.val)
        else:
            A = asp.Matrix.from_coo(M.m, M.n, M.row, M.col, M.val)
        mats.append((name, A))
    records = {}  # matrix -> history records (graph, matrix features, ms, nnz) of its own searches
    for name, A in mats:
        st = A.stats()
        feats = A.features()
        records[name] = []
        for seed in range(1, args.seeds + 1):
            g, rows = run(asp, A, seed, args)
            records[name] += [(r["graph"], feats, r["median_ms"], st["nnz"]) for r in rows
                              if r["median_ms"] > 0 and r["status"] in TIMED]
            print(json.dumps({"matrix": name, "seed": seed, "history": False, "variance": st["row_len_variance"],
                              "irregular": bool(st["irregular"]), **summary(rows), "winner": g}), flush=True)
    if args.history:
        for name, A in mats:
            st = A.stats()
            hist = [h for other, recs in records.items() if other != name for h in recs]
            for seed in range(1, args.seeds + 1):
                g, rows = run(asp, A, seed, args, history=hist)
                print(json.dumps({"matrix": name, "seed": seed, "history": True, "history_records": len(hist),
                                  "variance": st["row_len_variance"], "irregular": bool(st["irregular"]),
                                  **summary(rows), "winner": g}), flush=True)


if __name__ == "__main__":
    main()
