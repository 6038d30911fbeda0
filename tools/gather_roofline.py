"""Gather roofline of the irregular configs (developer measurement tool; see gather_roofline.cu).

    python tools/gather_roofline.py [--configs c3 c4] [--reps 15] > gpurun_out/gather.jsonl

For each matrix: time (CUDA events, L2 flushed before every rep, median) of
  stream   : read val + col once (no x)                      -> streaming floor
  gather   : read val + col + x[col] in CSR order            -> the matrix's gather roofline
  hot K    : gather with the K most referenced columns read from a shared-memory copy
and of random-sector gathers from the same x (hash indices, no index stream).  Prints one JSON
line per measurement with GB/s of algorithmic bytes (val + col + x + y as in the plan bytes
model) and gathers/s.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libgather_roofline.so")


def build():
    src = os.path.join(HERE, "gather_roofline.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-o", SO, src])
    lib = ctypes.CDLL(SO)
    lib.gr_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                              ctypes.c_int, ctypes.c_void_p]
    lib.gr_launch_async.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_void_p]
    lib.gr_launch_dsm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_void_p]
    lib.gr_launch_x.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    lib.gr_launch_unr.argtypes = lib.gr_launch_x.argtypes[:1] + lib.gr_launch_x.argtypes[2:]
    lib.gr_launch_hash.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return lib


def timeit(fn, reps, flush):
    import torch
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts)


def load(name):
    import synth
    if name == "c3":
        A = synth.c3_rmat_csr()
        return "rmat-24", A.m, A.n, A.col, A.val
    if name == "c4":
        A, tiles = synth.c4_blockdense_csr()
        b = 64
        rows = np.repeat(np.arange(A.m, dtype=np.int64), np.diff(A.row_ptr))
        key = (rows // b) * ((A.n + b - 1) // b) + A.col.astype(np.int64) // b
        planted = tiles[:, 0] * ((A.n + b - 1) // b) + tiles[:, 1]
        resid = ~np.isin(key, planted)
        return "blockdense-8m residual", A.m, A.n, np.ascontiguousarray(A.col[resid]), np.ascontiguousarray(A.val[resid])
    if name == "c5":
        A = synth.c5_band_csr()
        return "band-irreg-64m", A.m, A.n, A.col, A.val
    raise ValueError(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c3", "c4"])
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--hot", nargs="+", type=int, default=[8192, 16384, 32768, 49152])
    ap.add_argument("--dsm", action="store_true",
                    help="also time the hot-x copy distributed over a thread-block cluster (DSMEM)")
    ap.add_argument("--async-gather", action="store_true",
                    help="also time cp.async-staged gathers (relabeled columns, hot prefix in smem)")
    ap.add_argument("--relabel", action="store_true",
                    help="also time the gathers with columns relabeled by descending reference count")
    ap.add_argument("--xld", nargs="+", type=int, default=[],
                    help="also time gather / hot K with x-load variants (0 L1-allocating, 1 L1::no_allocate, "
                         "2 .cg, 3 L1::evict_first, 4 .nc without L2 policy) and hot-x copies up to --xld-hot-max")
    ap.add_argument("--xld-hot", nargs="+", type=int, default=[0, 24576, 32768, 40960, 49152])
    ap.add_argument("--xld-tpb", nargs="+", type=int, default=[1024])
    ap.add_argument("--unr", nargs="+", type=int, default=[],
                    help="also time hot-x .cg gathers with 1/2/4/8 vectors in flight per thread (--xld-hot sizes)")
    args = ap.parse_args()
    import torch
    lib = build()
    dev = torch.device("cuda:0")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    flush_buf = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device=dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)

    def flush():
        flush_buf.zero_()
        flush_buf.view(torch.int64).sum()

    for cfg in args.configs:
        wl, m, n, col, val = load(cfg)
        nnz = col.shape[0]
        dt = 0 if val.dtype == np.float32 else 1
        sv = val.itemsize
        dcol = torch.from_numpy(col).to(dev)
        dval = torch.from_numpy(val).to(dev)
        x = torch.rand(n, dtype=torch.float32 if dt == 0 else torch.float64, device=dev)
        s = torch.cuda.current_stream().cuda_stream
        model = nnz * (sv + 4) + n * sv + m * sv  # plan bytes model (beta = 0) without metadata
        base = {"config": wl, "nnz": nnz, "n": n, "dtype": "f32" if dt == 0 else "f64", "bytes_model": model}

        def run(mode, colp, xh=None, nh=0, grid=2 * nsm, tpb=1024):
            rc = lib.gr_launch(dt, mode, dval.data_ptr(), colp.data_ptr(), x.data_ptr(),
                               xh.data_ptr() if xh is not None else 0, nh, nnz, out.data_ptr(), grid, tpb, s)
            assert rc == 0, rc

        for mode, name in [(0, "stream"), (1, "gather")]:
            med, mn = timeit(lambda: run(mode, dcol), args.reps, flush)
            print(json.dumps({**base, "kernel": name, "median_us": med * 1e3, "min_us": mn * 1e3,
                              "model_gbs": model / (med * 1e-3) / 1e9, "gathers_per_s": nnz / (med * 1e-3)}), flush=True)
        cnt = np.bincount(col, minlength=n)
        order = np.argsort(-cnt, kind="stable")
        for K in args.hot:
            if K * sv > 200 * 1024:
                continue
            hot = order[:K]
            slot = np.full(n, -1, np.int64)
            slot[hot] = np.arange(K)
            enc = np.where(slot[col] >= 0, ~slot[col], col).astype(np.int32)
            cover = float(cnt[hot].sum()) / nnz
            denc = torch.from_numpy(enc).to(dev)
            xh = x[torch.from_numpy(hot).to(dev)].contiguous()
            med, mn = timeit(lambda: run(2, denc, xh, K, grid=nsm, tpb=1024), args.reps, flush)
            print(json.dumps({**base, "kernel": f"gather_hot{K}", "hot_cover": cover, "median_us": med * 1e3,
                              "min_us": mn * 1e3, "model_gbs": model / (med * 1e-3) / 1e9,
                              "gathers_per_s": nnz / (med * 1e-3)}), flush=True)
            del denc
        for xld in args.xld:
            for K in args.xld_hot:
                if K * sv > 220 * 1024:
                    continue
                if K:
                    hot = order[:K]
                    slot = np.full(n, -1, np.int64)
                    slot[hot] = np.arange(K)
                    enc = np.where(slot[col] >= 0, ~slot[col], col).astype(np.int32)
                    cover = float(cnt[hot].sum()) / nnz
                    denc = torch.from_numpy(enc).to(dev)
                    xh = x[torch.from_numpy(hot).to(dev)].contiguous()
                else:
                    cover, denc, xh = 0.0, dcol, x
                for tpb in args.xld_tpb:
                    grid = nsm * max(1, 1024 // tpb) if K else 2 * nsm * max(1, 1024 // tpb)

                    def runx():
                        rc = lib.gr_launch_x(dt, 2 if K else 1, xld, dval.data_ptr(), denc.data_ptr(), x.data_ptr(),
                                             xh.data_ptr(), K, nnz, out.data_ptr(), grid, tpb, s)
                        assert rc == 0, rc
                    med, mn = timeit(runx, args.reps, flush)
                    print(json.dumps({**base, "kernel": f"gather_xld{xld}_hot{K}", "xld": xld, "hot": K,
                                      "tpb": tpb, "grid": grid, "hot_cover": cover, "median_us": med * 1e3,
                                      "min_us": mn * 1e3, "model_gbs": model / (med * 1e-3) / 1e9,
                                      "gathers_per_s": nnz / (med * 1e-3)}), flush=True)
                del denc
        for unr in args.unr:
            for K in [k for k in args.xld_hot if k]:
                hot = order[:K]
                slot = np.full(n, -1, np.int64)
                slot[hot] = np.arange(K)
                denc = torch.from_numpy(np.where(slot[col] >= 0, ~slot[col], col).astype(np.int32)).to(dev)
                xh = x[torch.from_numpy(hot).to(dev)].contiguous()

                def runu():
                    rc = lib.gr_launch_unr(dt, unr, dval.data_ptr(), denc.data_ptr(), x.data_ptr(), xh.data_ptr(), K,
                                           nnz, out.data_ptr(), nsm, 1024, s)
                    assert rc == 0, rc
                med, mn = timeit(runu, args.reps, flush)
                print(json.dumps({**base, "kernel": f"gather_cg_unr{unr}_hot{K}", "unr": unr, "hot": K,
                                  "in_flight_per_thread": unr * (4 if dt == 0 else 2), "median_us": med * 1e3,
                                  "min_us": mn * 1e3, "gathers_per_s": nnz / (med * 1e-3)}), flush=True)
                del denc
        if args.dsm:
            for (csize, kl) in [(1, 24576), (2, 24576), (4, 24576), (8, 24576), (2, 16384), (4, 16384), (8, 16384),
                                (16, 12288)]:
                if kl * sv > 200 * 1024:
                    continue
                K = csize * kl
                hot = order[:K]
                slot = np.full(n, -1, np.int64)
                slot[hot] = np.arange(K)
                enc = np.where(slot[col] >= 0, ~slot[col], col).astype(np.int32)
                denc = torch.from_numpy(enc).to(dev)
                xh = x[torch.from_numpy(hot).to(dev)].contiguous()
                cover = float(cnt[hot].sum()) / nnz

                def rund():
                    rc = lib.gr_launch_dsm(dt, csize, dval.data_ptr(), denc.data_ptr(), x.data_ptr(), xh.data_ptr(), kl,
                                           nnz, out.data_ptr(), (nsm // csize) * csize, 1024, s)
                    assert rc == 0, rc
                try:
                    med, mn = timeit(rund, args.reps, flush)
                    print(json.dumps({**base, "kernel": f"dsm_c{csize}_kl{kl}", "hot_cover": cover,
                                      "median_us": med * 1e3, "min_us": mn * 1e3,
                                      "gathers_per_s": nnz / (med * 1e-3)}), flush=True)
                except AssertionError as e:
                    print(json.dumps({**base, "kernel": f"dsm_c{csize}_kl{kl}", "error": str(e)}), flush=True)
                del denc, xh
        if args.async_gather:
            rank = np.empty(n, np.int64)
            rank[order] = np.arange(n)
            rcol = torch.from_numpy(rank[col].astype(np.int32)).to(dev)
            xr = x[torch.from_numpy(order).to(dev)].contiguous()
            for (ch, K, tpb) in [(8, 0, 1024), (16, 0, 512), (8, 16384, 1024), (16, 16384, 512), (8, 8192, 1024)]:
                def runa():
                    rc = lib.gr_launch_async(dt, ch, dval.data_ptr(), rcol.data_ptr(), xr.data_ptr(), xr.data_ptr(), K,
                                             nnz, out.data_ptr(), (2048 // tpb) * nsm if K == 0 else nsm, tpb, s)
                    assert rc == 0, rc
                try:
                    med, mn = timeit(runa, args.reps, flush)
                except AssertionError as e:
                    print(json.dumps({**base, "kernel": f"async_ch{ch}_hot{K}_t{tpb}", "error": str(e)}), flush=True)
                    continue
                print(json.dumps({**base, "kernel": f"async_ch{ch}_hot{K}_t{tpb}", "median_us": med * 1e3,
                                  "min_us": mn * 1e3, "model_gbs": model / (med * 1e-3) / 1e9,
                                  "gathers_per_s": nnz / (med * 1e-3)}), flush=True)
            # the register-gather reference on the same relabeled columns
            for K in (0, 16384):
                def runr():
                    rc = lib.gr_launch(dt, 3 if K else 1, dval.data_ptr(), rcol.data_ptr(), xr.data_ptr(), xr.data_ptr(),
                                       K, nnz, out.data_ptr(), nsm if K else 2 * nsm, 1024, s)
                    assert rc == 0, rc
                med, mn = timeit(runr, args.reps, flush)
                print(json.dumps({**base, "kernel": f"reg_relabel_hot{K}", "median_us": med * 1e3}), flush=True)
            del rcol, xr
        if args.relabel:
            # column relabeling: rank[c] = position of c in the descending-count order; x permuted to match
            rank = np.empty(n, np.int64)
            rank[order] = np.arange(n)
            rcol = torch.from_numpy(rank[col].astype(np.int32)).to(dev)
            xr = x[torch.from_numpy(order).to(dev)].contiguous()
            xsave = x

            def runr(mode, nh, grid, tpb):
                rc = lib.gr_launch(dt, mode, dval.data_ptr(), rcol.data_ptr(), xr.data_ptr(), xr.data_ptr(), nh, nnz,
                                   out.data_ptr(), grid, tpb, s)
                assert rc == 0, rc
            for (mode, K, grid, tpb) in [(1, 0, 2 * nsm, 1024), (1, 0, nsm, 1024), (1, 0, 4 * nsm, 512)] + \
                    [(3, K, nsm, 1024) for K in args.hot if K * sv <= 200 * 1024]:
                med, mn = timeit(lambda: runr(mode, K, grid, tpb), args.reps, flush)
                cover = float(cnt[order[:K]].sum()) / nnz
                print(json.dumps({**base, "kernel": f"relabel_gather_hot{K}_g{grid}_t{tpb}", "hot_cover": cover,
                                  "median_us": med * 1e3, "min_us": mn * 1e3, "model_gbs": model / (med * 1e-3) / 1e9,
                                  "gathers_per_s": nnz / (med * 1e-3)}), flush=True)
            # cost of permuting x per call (x'[i] = x[order[i]])
            dorder = torch.from_numpy(order).to(dev)
            med, mn = timeit(lambda: torch.index_select(xsave, 0, dorder, out=xr), args.reps, flush)
            print(json.dumps({**base, "kernel": "permute_x_index_select", "median_us": med * 1e3}), flush=True)
            del rcol, xr, dorder
        # random sectors alone: the same number of gathers, hashed indices, no index stream
        med, mn = timeit(lambda: lib.gr_launch_hash(dt, x.data_ptr(), n, nnz, out.data_ptr(), 2 * nsm, 1024, s),
                         args.reps, flush)
        print(json.dumps({**base, "kernel": "hash_gather", "median_us": med * 1e3, "min_us": mn * 1e3,
                          "gathers_per_s": nnz / (med * 1e-3), "sector_gbs": nnz * 32 / (med * 1e-3) / 1e9}), flush=True)
        del dcol, dval, x


if __name__ == "__main__":
    main()
