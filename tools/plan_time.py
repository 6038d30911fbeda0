"""as_plan wall time, on-device Designer vs host Designer (developer measurement tool).

    python tools/plan_time.py --configs c3 c5 > gpurun_out/plan_time.jsonl

For each config: the first device build (includes the one-time upload of the canonical CSR),
a second device build of another graph (cache hit), and the host build of the same graphs;
each plan's y is compared between the two builds (same arithmetic -> bit-identical)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GRAPHS = {
    "c3": ["COMPRESS; BMW_NNZ_BLOCK(nnz=8192); BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; "
           "WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=24576); GMEM_ATOM_RED",
           "SORT; COMPRESS; BMW_NNZ_BLOCK(nnz=4096); BMT_NNZ_BLOCK(nnz=32); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
           "SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"],
    "c5": ["COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=2); THREAD_BITMAP_RED_G; "
           "SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=0); GMEM_ATOM_RED",
           "SORT_SUB(g=65536); COMPRESS; BMW_NNZ_BLOCK(nnz=1024); BMT_NNZ_BLOCK(nnz=16); THREAD_BITMAP_RED_G; "
           "WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=1,stages=0); GMEM_ATOM_RED"],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c3", "c5"])
    args = ap.parse_args()
    import torch
    import bench
    import synth
    import paper_2212_10432_b200 as asp
    for cfg in args.configs:
        coo, wl, _ = bench.load_config(cfg)
        coo = bench.to_csr(coo)
        A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
        x, _ = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
        dx = torch.from_numpy(x).cuda()
        for i, g in enumerate(GRAPHS[cfg]):
            ys = {}
            for mode in ("device", "host"):
                torch.cuda.synchronize()
                t = time.perf_counter()
                P = asp.Plan(A, g, device=0, host_build=(mode == "host"))
                torch.cuda.synchronize()
                dt = time.perf_counter() - t
                dy = torch.zeros(coo.m, dtype=dx.dtype, device="cuda")
                P.spmv(1.0, dx, 0.0, dy)
                torch.cuda.synchronize()
                ys[mode] = dy
                print(json.dumps({"config": wl, "graph": g, "build": mode, "first": i == 0, "plan_s": dt,
                                  "device_built": P.info()["device_built"], "kernels": P.info()["kernels"]}),
                      flush=True)
                del P
            # real-valued data: atomics of straddling rows may add in another order
            diff = float(((ys["device"].double() - ys["host"].double()).abs().max()
                          / ys["host"].double().abs().max().clamp_min(1e-300)))
            print(json.dumps({"config": wl, "graph": g, "y_max_rel_diff": diff}), flush=True)
        del A


if __name__ == "__main__":
    main()
