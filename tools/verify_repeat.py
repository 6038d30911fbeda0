"""Repeat-verification of one plan on a BASELINE config (developer tool): run as_spmv R times
with alpha = 1, beta = 0.5 on a known y0 and check every run against the long-double oracle
(O2 tolerance).  Prints one JSON line per run: failing rows, max err/bound, and details of
the worst rows (length, heavy-row class).  Used to chase nondeterministic results.

    python tools/verify_repeat.py --config c3 --graph "..." --reps 20
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--graph", nargs="+", required=True)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import bench
    import synth
    import paper_2212_10432_b200 as asp
    from oracle import spmv as S
    coo, wl, _ = bench.load_config(args.config)
    coo = bench.to_csr(coo)
    A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
    x, y0 = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    yref, bound = S.spmv_csr(coo.row_ptr, coo.col, coo.val.astype(np.float64), x.astype(np.float64), 1.0, 0.5,
                             y0.astype(np.float64), nthreads=os.cpu_count())
    lens = np.diff(coo.row_ptr)
    dx = torch.from_numpy(x).cuda()
    for g in args.graph:
        P = asp.Plan(A, g, device=0)
        for r in range(args.reps):
            dy = torch.from_numpy(y0.copy()).cuda()
            P.spmv(1.0, dx, 0.5, dy)
            torch.cuda.synchronize()
            y = dy.cpu().numpy()
            err = np.abs(y.astype(np.longdouble) - yref)
            lim = np.longdouble(1e-5 if coo.val.dtype == np.float32 else 1e-12) * bound
            bad = np.nonzero(~(err <= lim))[0]
            ratio = np.where(bound > 0, err / np.where(bound > 0, bound, 1), 0)
            worst = np.argsort(-ratio)[:5]
            print(json.dumps({"config": wl, "graph": g, "rep": r, "kernels": P.info()["kernels"], "bad_rows": int(bad.shape[0]),
                              "max_ratio": float(ratio.max()),
                              "worst": [{"row": int(i), "len": int(lens[i]), "ratio": float(ratio[i]),
                                         "y": float(y[i]), "ref": float(yref[i])} for i in worst]}), flush=True)
        del P


if __name__ == "__main__":
    main()
