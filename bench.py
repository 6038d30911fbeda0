"""bench.py — SpMV GFLOP/s and HBM GB/s (% of roofline) of the searched operator graph.

Headline (N=1): BASELINE configs[2] = C3 `rmat-24`, the largest single-GPU configuration
(Graph500 R-MAT, 16,777,216 rows, 268,435,456 nnz, fp32), alpha = 1, beta = 0, the graph
found by as_search (seeded with the committed best design, profiles/best_graphs.json).  One
step = one as_spmv call (the whole hot loop a5 + a6; the plan a1-a4 and the search a7 run
before the timed region, as the paper times the generated SpMV program) with the
inputs resident in HBM; L2 is flushed (write + read back of 2 x L2) before every timed step,
outside the CUDA events.  ms_per_step is the MEDIAN of the timed steps (A27).

The same JSON line carries the other BASELINE configs measured in the same run under
"configs" (C2 lap2d-2048, C4 blockdense-8m, C5 band-irreg-64m: their committed best graphs,
same timing protocol, each with its dominant-kernel roofline), the gather roofline of the
headline matrix (tools/gather_roofline.cu: stream every (val, col) pair once and gather
x[col], no reduction, no y -- the floor any SpMV over these nonzeros has on this GPU),
cpu_baseline (the oracle on the host cores), and e2e (as_spmv_host, host buffers).

Multi-GPU (torchrun, one rank per GPU): default C5 `band-irreg-64m` (BASELINE configs[4])
ROW_DIV across ranks with nnz-balanced cuts (reading A35, as_dist_row_cuts_ptr on the row
pointer alone); every rank GENERATES ONLY ITS BAND (synth.c5_band_rows) and plans it; x is
replicated.  value = total nnz of all ranks / the max-over-ranks SpMV step time (strong
scaling).  The y exchange the next iterate needs is timed separately: as_spmv_dist with the
NCCL AllGatherV (SpMV + exchange per step) and the all-gather alone.
`--impl reference` times the oracle (long-double CPU SpMV) on the host, full config.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import re
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "SpMV GFLOP/s and achieved HBM GB/s (% of roofline) per matrix at 1/2/4/8 B200"
C2_SEEDS = [
    "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=128,grid=16) }",
    "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=512,grid=4) }",
    "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(128); SHMEM_OFFSET_RED; GMEM_ATOM_RED",
]
WORKLOAD = {"c1": "uniform-1k", "c2": "lap2d-2048", "c3": "rmat-24", "c4": "blockdense-8m", "c5": "band-irreg-64m"}


def best_graph(wl):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "best_graphs.json")))[wl]["graph"]
    except Exception:
        return None


def peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx):
        self.idx, self.samples, self.stop = idx, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_config(name, int_mode=False):
    """(csr, workload name, seed graphs); the committed best graph (if any) seeds first."""
    if name == "c2":
        coo, seeds = synth.c2_lap2d(2048), list(C2_SEEDS)
    elif name == "c1":
        coo, seeds = synth.c1_uniform(int_mode=int_mode), [
            "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; SET_RESOURCE(128); GMEM_ATOM_RED"]
    elif name == "c4":
        coo, _ = synth.c4_blockdense_csr()
        seeds = [
            "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMTB_ROW_BLOCK(32); BMT_ROW_BLOCK(1); BMT_PAD(BMTB); THREAD_TOTAL_RED; SET_RESOURCE(64); GMEM_ATOM_RED }",
            "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }"]
    elif name == "c3":
        coo = synth.c3_rmat_csr()
        seeds = [
            "COMPRESS; BMW_NNZ_BLOCK(4096); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=1,xcache=32768); GMEM_ATOM_RED",
            "COMPRESS; BMW_NNZ_BLOCK(4096); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED",
            "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=1,xcache=16384); GMEM_ATOM_RED",
            "BIN(t=[32,2048]) { COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED"
            " | COMPRESS; BMTB_NNZ_BLOCK(2048); SHMEM_OFFSET_RED; GMEM_ATOM_RED"
            " | COMPRESS; BMTB_ROW_BLOCK(1); BMW_NNZ_BLOCK(2048); WARP_TOTAL_RED; GMEM_ATOM_RED }"]
    elif name in ("c3s", "c4s", "c5s"):  # shape-preserving 1/4..1/16-scale instances (dev sweeps)
        c = {"c3s": lambda: synth.c3_rmat_csr(scale=22, nnz=1 << 26),
             "c4s": lambda: synth.c4_blockdense_csr(m=1 << 21, b=64, n_tiles=6144, nnz=50_000_000)[0],
             "c5s": lambda: synth.c5_band_csr(m=1 << 22, nnz=1 << 26)}[name]()
        return c, c.name + "-scaled", []
    elif name == "c5":
        coo = synth.c5_band_csr()
        seeds = [
            "COMPRESS; BMT_NNZ_BLOCK(64); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED",
            "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED"]
    else:
        raise SystemExit(f"unknown config {name}")
    wl = WORKLOAD[name]
    b = best_graph(wl)
    if b:
        seeds = [b] + [s for s in seeds if s != b]
    return coo, wl, seeds


def csr_of(coo):
    """row_ptr of a synth.Coo or synth.Csr."""
    if isinstance(coo, synth.Csr):
        return coo.row_ptr
    rp = np.zeros(coo.m + 1, np.int64)
    np.add.at(rp, coo.row + 1, 1)
    return np.cumsum(rp)


def to_csr(obj):
    if isinstance(obj, synth.Csr):
        return obj
    return synth.Csr(obj.m, obj.n, csr_of(obj), obj.col.astype(np.int32), obj.val, obj.name)


def reference_arm(args, coo, wl):
    """The oracle (long-double CSR SpMV, oracle/spmv_ref.c) on the host cores: every step one
    full pass over the same matrix as our arm (same config); median of the steps."""
    from oracle import spmv as S
    rp = csr_of(coo)
    x, _ = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    cores = os.cpu_count() or 1
    col, val = coo.col, coo.val.astype(np.float64)
    for _ in range(max(1, min(args.warmup, 2))):
        S.spmv_csr(rp, col, val, x, nthreads=cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        S.spmv_csr(rp, col, val, x, nthreads=cores)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    v = 2.0 * coo.nnz / t / 1e9
    sample = f"{args.steps} full passes over {wl} ({coo.nnz} nnz), long double, {cores} threads"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64x", "data": "synthetic",
            "config": {"workload": wl, "nnz": coo.nnz, "rows": coo.m, "same_config": True},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(coo, wl, budget_s=10.0, y_gpu=None):
    """The oracle timed on the host cores; its first pass also checks the timed GPU y of the
    same (A, x) row by row (north_star tolerance O2), at full size."""
    from oracle import spmv as S
    rp = csr_of(coo)
    x, _ = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    cores = os.cpu_count() or 1
    col, val = coo.col, coo.val.astype(np.float64)
    yref, bound = S.spmv_csr(rp, col, val, x.astype(np.float64), nthreads=cores)
    parity = None
    if y_gpu is not None:
        ok, ratio = S.check(y_gpu, yref, bound, coo.val.dtype)
        parity = {"rows_checked": int(coo.m), "max_err_over_bound": float(ratio), "ok": bool(ok),
                  "tol": 1e-12 if coo.val.dtype == np.float64 else 1e-5,
                  "what": "every row of the last timed y vs the long-double oracle, |y - yref| <= tol * sum|a_ij x_j|"}
    del yref, bound
    n, t_tot = 0, 0.0
    while t_tot < budget_s and n < 5000:
        t0 = time.perf_counter()
        S.spmv_csr(rp, col, val, x, nthreads=cores)
        t_tot += time.perf_counter() - t0
        n += 1
    # single-threaded beside all cores, on the first rows holding <= 2e7 nonzeros
    r1 = int(np.searchsorted(rp, min(int(rp[-1]), 20_000_000), side="right")) - 1
    nz1 = int(rp[r1])
    t0 = time.perf_counter()
    S.spmv_csr(rp[:r1 + 1], col[:nz1], val[:nz1], x, nthreads=1)
    t1 = max(time.perf_counter() - t0, 1e-9)
    cpu = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    import platform
    return {"value": 2.0 * coo.nnz * n / t_tot / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "parity": parity,
            "sample": f"{n} full passes over {wl} ({coo.nnz} nnz), long double, {cores} threads, {t_tot:.1f} s",
            "value_1thread": 2.0 * nz1 / t1 / 1e9, "sample_1thread": f"first {r1} rows ({nz1} nnz)", "cpu": cpu,
            "long_double": "x87 80-bit extended" if platform.machine() in ("x86_64", "AMD64") else platform.machine()}


E2E_BANDS = 4  # ROW_DIV bands of the pipelined e2e plan (C2 sweep: 4 -> 0.94 ms, 8 -> 0.98, 16 -> 1.10)


def cdev():
    """Device of control-plane tensors: cuda under nccl, cpu under gloo."""
    return "cpu" if os.environ.get("AS_BENCH_BACKEND") == "gloo" else "cuda"


class Timer:
    """CUDA-event timing on the launching stream with an L2 flush (write + read back of 2 x
    L2, outside the events) before every timed call."""

    def __init__(self, torch, stream, local, no_flush):
        self.torch, self.stream, self.no_flush = torch, stream, no_flush
        l2 = torch.cuda.get_device_properties(local).L2_cache_size
        self.flush_buf = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")

    def flush(self):
        if not self.no_flush:
            self.flush_buf.zero_()
            self.flush_buf.view(self.torch.int64).sum()

    def steps(self, fn, n):
        torch = self.torch
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for e0, e1 in evs:
            self.flush()
            e0.record(self.stream)
            fn()
            e1.record(self.stream)
        torch.cuda.synchronize()
        return [e0.elapsed_time(e1) for e0, e1 in evs]


def dominant_of(P, dx, dy, timer, npass):
    """Per-launch device times (as_plan_profile, CUDA events between the launches, L2 flushed
    before each pass) and per-launch algorithmic bytes; the dominant launch."""
    acc = None
    for _ in range(npass):
        timer.flush()
        prof = P.profile(dx, dy, reps=1, stream=timer.stream)
        acc = [[n, ms, by] for n, ms, by in prof] if acc is None else [[a[0], a[1] + p_[1], a[2]] for a, p_ in zip(acc, prof)]
    per = [(n, ms / npass, by) for n, ms, by in acc]
    name, dms, dby = max(per, key=lambda e: e[1])
    return {"kernel": name, "ms": dms, "bytes": dby, "launches": [{"kernel": n, "ms": ms, "bytes": by} for n, ms, by in per]}


def gather_roofline(torch, coo, dx, timer, reps, hot_k=0):
    """tools/gather_roofline.cu on this matrix's own (val, col) arrays in CSR order: stream
    every pair once and gather x[col] (no reduction, no y).  Returns the median time."""
    here = os.path.join(ROOT, "tools")
    so = os.path.join(here, "libgather_roofline.so")
    src = os.path.join(here, "gather_roofline.cu")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", so, src])
    lib = ctypes.CDLL(so)
    lib.gr_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                              ctypes.c_int, ctypes.c_void_p]
    dcol = torch.from_numpy(np.ascontiguousarray(coo.col, np.int32)).cuda()
    dval = torch.from_numpy(np.ascontiguousarray(coo.val)).cuda()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    dt = 0 if coo.val.dtype == np.float32 else 1
    s = timer.stream.cuda_stream

    def run():
        rc = lib.gr_launch(dt, 1, dval.data_ptr(), dcol.data_ptr(), dx.data_ptr(), None, 0, coo.nnz, out.data_ptr(),
                           2 * nsm, 1024, s)
        assert rc == 0, rc
    for _ in range(3):
        run()
    ms = statistics.median(timer.steps(run, reps))
    hot = None
    if hot_k:
        # the same gathers with the plan's hot-x copy in shared memory and the rest read at L2
        # only (.cg), the kernel's own access pattern without the reduction: the request-rate
        # ceiling of this matrix
        lib.gr_launch_x.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        cnt = np.bincount(coo.col, minlength=coo.n)
        order = np.argsort(-cnt, kind="stable")[:hot_k]
        slot = np.full(coo.n, -1, np.int64)
        slot[order] = np.arange(hot_k)
        sl = slot[coo.col]
        denc = torch.from_numpy(np.where(sl >= 0, ~sl, coo.col).astype(np.int32)).cuda()
        del sl
        xh = dx[torch.from_numpy(order).cuda()].contiguous()

        def run_hot():
            rc = lib.gr_launch_x(dt, 2, 2, dval.data_ptr(), denc.data_ptr(), dx.data_ptr(), xh.data_ptr(), hot_k,
                                 coo.nnz, out.data_ptr(), nsm, 1024, s)
            assert rc == 0, rc
        for _ in range(3):
            run_hot()
        hot = {"ms": statistics.median(timer.steps(run_hot, reps)), "hot": hot_k,
               "cover": float(cnt[order].sum()) / coo.nnz}
        del denc, xh
    del dcol, dval
    return ms, hot


def run_config(args, torch, asp, name, A, coo, wl, seeds, graph, search, local, timer, with_e2e, budget):
    """Plan (search or fixed graph), then time args.steps steps (median) and profile the
    dominant launch.  Returns (result dict, plan, dx, dy)."""
    stream = timer.stream
    t_plan = time.perf_counter()
    if graph:
        P = asp.Plan(A, graph, device=local)
        graph = str(asp.Graph(graph))
        searched = False
    else:
        P, graph = asp.search(A, device=local, seed=1, max_candidates=args.search_candidates,
                              budget_seconds=budget, warmup=3, reps=10, seed_graphs=seeds,
                              log_path=os.path.join(ROOT, "gpurun_out", f"search_{wl}.jsonl")
                              if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else None)
        searched = True
    plan_s = time.perf_counter() - t_plan
    info = P.info()
    dt = coo.val.dtype
    x, _ = synth.vectors(coo.n, coo.m, 2, dt)
    dx = torch.from_numpy(x).cuda()
    dy = torch.zeros(coo.m, dtype=torch.float64 if dt == np.float64 else torch.float32, device="cuda")

    def step():
        P.spmv(1.0, dx, 0.0, dy, stream)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ms = timer.steps(step, args.steps)
    t_ms = statistics.median(ms)
    hbm, hbm_kind = peaks()
    dom = dominant_of(P, dx, dy, timer, max(3, args.steps // 3))
    dom["share_of_step"] = dom["ms"] / t_ms if t_ms else None
    achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9 if dom["ms"] > 0 else 0.0
    achieved_step = info["bytes_model"] / (t_ms * 1e-3) / 1e9
    launches = int(info["n_launches"])
    r = {"workload": wl, "rows": coo.m, "nnz": coo.nnz, "dtype": "f64" if dt == np.float64 else "f32",
         "graph": graph, "searched": searched, "plan_and_search_s": round(plan_s, 2), "kernels": info["kernels"],
         "ms_per_step": t_ms, "ms_min": min(ms), "ms_mean": statistics.mean(ms), "steps": args.steps,
         "gflops": 2.0 * coo.nnz / (t_ms * 1e-3) / 1e9, "bytes_model": info["bytes_model"],
         "bytes_floor": info["bytes_floor"], "launches": launches, "clocks": clk.summary(),
         "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                      "peak_kind": hbm_kind, "frac_of_8tbs": achieved / 8000.0, "achieved_step": achieved_step,
                      "frac_step": achieved_step / hbm, "dominant": dom}}
    # traffic: the committed ncu capture of this workload's dominant kernel, when it is the
    # same kernel form (profiles/traffic_<workload>.json)
    prof = os.path.join(ROOT, "profiles", f"traffic_{wl}.json")
    r["roofline"]["traffic"] = None
    if os.path.exists(prof):
        try:
            tjs = json.load(open(prof))
            for tj in (tjs if isinstance(tjs, list) else [tjs]):  # one capture per graph shape
                same = tj.get("graph", graph) == graph or ("bytes_model" in tj and tj["bytes_model"] == info["bytes_model"])
                if tj.get("kernels") == info["kernels"] and same:
                    r["roofline"]["traffic"] = tj["dram_bytes_per_launch"]
                    r["roofline"]["traffic_src"] = tj.get("src")
                    break
        except Exception:
            pass
    if with_e2e:
        r["e2e"] = e2e_of(args, torch, asp, P, A, coo, graph, local, timer)
        nw = 100 if t_ms < 1.0 else 20
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0.record(stream)
        for _ in range(nw):
            step()
        w1.record(stream)
        torch.cuda.synchronize()
        wm = w0.elapsed_time(w1) / nw
        r["warm"] = {"ms_per_step": wm, "gflops": 2.0 * coo.nnz / (wm * 1e-3) / 1e9, "calls": nw}
    return r, P, dx, dy


def e2e_of(args, torch, asp, P, A, coo, graph, local, timer):
    """e2e through the C-ABI with pinned host buffers, copies inside the timed region: the
    searched plan (copies, kernels, copies back to back) and the same graph under ROW_DIV into
    E2E_BANDS bands, which as_spmv_host pipelines; the faster is reported."""
    x, _ = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.zeros(coo.m, dtype=torch.float64 if coo.val.dtype == np.float64 else torch.float32).pin_memory()
    xn, yn = xh.numpy(), yh.numpy()
    cands = [(graph, P)]
    if "ROW_DIV" not in graph and coo.m >= 8 * E2E_BANDS:
        cut = ",".join(str(coo.m * i // E2E_BANDS) for i in range(1, E2E_BANDS))
        g_pipe = f"ROW_DIV(cuts=[{cut}]) {{ {graph} }}"
        try:
            cands.append((g_pipe, asp.Plan(A, g_pipe, device=local)))
        except asp.AsError:
            pass
    res = []
    for g_e, P_e in cands:
        for _ in range(2):
            P_e.spmv_host(1.0, xn, 0.0, yn, timer.stream)
        ms = timer.steps(lambda: P_e.spmv_host(1.0, xn, 0.0, yn, timer.stream), max(3, args.steps // 3))
        res.append((statistics.median(ms), g_e, int(P_e.info()["n_launches"])))
    names = ["searched", "pipelined"][:len(res)]
    # a batch of K steps through as_spmv_host_batch: step i+1's x goes up and step i-1's y
    # comes down while SpMV i runs (every step still copies its x up and its y back); timed
    # as one event window over the K steps, L2 flushed before it
    K = max(4, args.steps // 2)
    try:
        ys = [torch.zeros_like(yh).pin_memory().numpy() for _ in range(K)]
        xs = [xn] * K
        P.spmv_host_batch(1.0, xs[:2], 0.0, ys[:2], timer.stream)
        bms = [t / K for t in timer.steps(lambda: P.spmv_host_batch(1.0, xs, 0.0, ys, timer.stream), 3)]
        res.append((statistics.median(bms), graph, int(P.info()["n_launches"])))
        names.append(f"batch{K}")
        del ys
    except Exception as e:  # the per-call numbers stand
        names.append(f"batch_error: {str(e)[:120]}")
    best = min(range(len(res)), key=lambda i: res[i][0])
    tm, g_e, l_e = res[best]
    sv = xn.itemsize
    return {"value": 2.0 * coo.nnz / (tm * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": tm,
            "h2d_bytes_per_step": int(coo.n * sv), "d2h_bytes_per_step": int(coo.m * sv), "graph": g_e,
            "launches_per_step": l_e, "how": names[best],
            "candidates_ms": {names[i]: r[0] for i, r in enumerate(res)}}


def single_gpu(args, torch, asp):
    t0 = time.perf_counter()
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    timer = Timer(torch, stream, 0, args.no_flush)
    name = args.config or "c3"
    coo, wl, seeds = load_config(name)
    coo = to_csr(coo)
    A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
    graph = args.graph or (seeds[0] if name == "c1" else None)
    if args.no_search and not graph:
        graph = seeds[0]
    head, P, dx, dy = run_config(args, torch, asp, name, A, coo, wl, seeds, graph, not graph, 0, timer, True,
                                 args.search_budget)
    # the gather roofline of this matrix (tools/gather_roofline.cu, timed live)
    gr = None
    if not args.no_gather and name in ("c3", "c4", "c5", "c3s", "c5s"):
        try:
            m_hot = re.search(r"xcache=(\d+)", head["graph"])
            gms, hot = gather_roofline(torch, coo, dx, timer, max(5, args.steps // 2),
                                       int(m_hot.group(1)) if m_hot else 0)
            dk = head["roofline"]["dominant"]
            gr = {"ms": gms, "achieved_gbs": head["bytes_model"] / (gms * 1e-3) / 1e9,
                  "frac_step": gms / head["ms_per_step"], "frac_dominant": gms / dk["ms"] if dk["ms"] else None,
                  "note": "time to stream every (val, col) pair once and gather x[col] (no reduction, no y), "
                          "CSR order, same x, L2 flushed: frac = gather time / SpMV time"}
            if hot:
                gr["hot_cg"] = {**hot, "frac_step": hot["ms"] / head["ms_per_step"],
                                "note": "same stream and gathers with the plan's xcache hot columns read from shared "
                                        "memory and the rest at L2 only (.cg): the L1->L2 request-rate ceiling of "
                                        "this access pattern (DESIGN.md section 4)"}
        except Exception as e:  # the measurement tool is optional; the SpMV numbers stand
            gr = {"error": str(e)[:200]}
    head["roofline"]["gather"] = gr
    y_gpu = dy.cpu().numpy()  # y of the last timed step (alpha 1, beta 0): checked by the oracle leg
    cpu = None if args.no_cpu_baseline else cpu_baseline(coo, wl, y_gpu=y_gpu)
    del y_gpu
    launches = head["launches"] * args.steps
    del P, dx, dy, A, coo
    torch.cuda.empty_cache()
    extras = []
    for cfg in [c for c in args.extra.split(",") if c and c != name]:
        if time.perf_counter() - t0 > args.max_seconds:
            extras.append({"workload": WORKLOAD.get(cfg, cfg), "skipped": "time budget"})
            continue
        try:
            c2, wl2, seeds2 = load_config(cfg)
            c2 = to_csr(c2)
            A2 = asp.Matrix.from_csr(c2.m, c2.n, c2.row_ptr, c2.col, c2.val)
            r2, P2, dx2, dy2 = run_config(args, torch, asp, cfg, A2, c2, wl2, seeds2, seeds2[0], False, 0, timer,
                                          False, 0)
            extras.append(r2)
            del P2, dx2, dy2, A2, c2
        except Exception as e:
            extras.append({"workload": WORKLOAD.get(cfg, cfg), "error": str(e)[:300]})
        torch.cuda.empty_cache()
    hr = head["roofline"]
    line = {
        "metric": METRIC, "value": head["gflops"], "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": head["dtype"], "data": "synthetic",
        "config": {"workload": wl, "rows": head["rows"], "nnz": head["nnz"], "graph": head["graph"],
                   "searched": head["searched"], "alpha": 1.0, "beta": 0.0,
                   "l2": "flushed before every step (inputs 2.4 GB > L2 as well)" if not args.no_flush else "not flushed",
                   "timing": f"median of {args.steps} steps, CUDA events on the launch stream",
                   "parallelism": "row_div1", "plan_and_search_s": head["plan_and_search_s"],
                   "kernels": head["kernels"], "bytes_model": head["bytes_model"], "bytes_floor": head["bytes_floor"]},
        "hbm_gbs_model": hr["achieved"],
        "roofline": {k: hr[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
        "roofline_detail": {k: v for k, v in hr.items() if k not in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
        "gpu_launches": launches,
        "clocks": head["clocks"],
        "e2e": head["e2e"],
        "warm": head.get("warm"),
        "configs": extras,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def multi_gpu(args, torch, asp, world, rank, local):
    """ROW_DIV across ranks: rank-local band generation (C5) or bands of a shared config."""
    import torch.distributed as dist
    if os.environ.get("AS_BENCH_BACKEND") == "gloo":
        local = 0
    torch.cuda.set_device(local)
    if os.environ.get("AS_BENCH_BACKEND") == "gloo":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    timer = Timer(torch, stream, local, args.no_flush)
    name = args.config or "c5"
    small = os.environ.get("AS_BENCH_C5_SCALE")  # tests: a shape-preserving small C5
    if name == "c5":
        m, nnz = (1 << 26, 1 << 30) if not small else (1 << int(small), 1 << (int(small) + 4))
        rp = synth.c5_row_ptr(m=m, nnz=nnz)
        cuts = asp.row_cuts_from_ptr(rp, world)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        band = synth.c5_band_rows(rp, r0, r1)
        wl = WORKLOAD["c5"] + (f"-2^{small}" if small else "")
        seeds = [best_graph(WORKLOAD["c5"])] if best_graph(WORKLOAD["c5"]) else []
        m_global, n_global = m, m
        scaling = "strong"
    else:
        coo, wl, seeds = load_config(name)
        coo = to_csr(coo)
        cuts = asp.row_cuts_from_ptr(coo.row_ptr, world)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        a, e = int(coo.row_ptr[r0]), int(coo.row_ptr[r1])
        band = synth.Csr(r1 - r0, coo.n, coo.row_ptr[r0:r1 + 1] - a, coo.col[a:e], coo.val[a:e], coo.name)
        m_global, n_global = coo.m, coo.n
        scaling = "strong"
    A = asp.Matrix.from_csr(band.m, band.n, band.row_ptr, band.col, band.val)
    graph = args.graph or (seeds[0] if seeds else None)
    t_plan = time.perf_counter()
    if graph and (args.no_search or not args.search_budget):
        P = asp.Plan(A, graph, device=local)
        graph = str(asp.Graph(graph))
    else:
        P, graph = asp.search(A, device=local, seed=1 + rank, max_candidates=args.search_candidates,
                              budget_seconds=args.search_budget, warmup=3, reps=10, seed_graphs=[graph] if graph else [])
    plan_s = time.perf_counter() - t_plan
    info = P.info()
    dt = band.val.dtype
    tdt = torch.float64 if dt == np.float64 else torch.float32
    # replicated x (every rank holds the whole vector, north_star); deterministic per index
    x = torch.from_numpy(synth.vectors(n_global, 1, 2, dt)[0]).cuda()
    dy = torch.zeros(band.m, dtype=tdt, device="cuda")

    def step():
        P.spmv(1.0, x, 0.0, dy, stream)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    with Clocks(local) as clk:
        ms = timer.steps(step, args.steps)
    t_ms = statistics.median(ms)
    tt = torch.tensor([t_ms], device=cdev(), dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())
    tot = torch.tensor([float(band.nnz), float(info["bytes_model"])], device=cdev(), dtype=torch.float64)
    dist.all_reduce(tot)
    nnz_total, bytes_total = int(tot[0].item()), float(tot[1].item())
    # y exchange for the next iterate, timed separately: the all-gather alone
    # (uneven bands: one NCCL broadcast per rank), and as_spmv_dist (SpMV + NCCL AllGatherV
    # inside the library) per step; a watchdog keeps a failing exchange from hiding the line
    exch = {}
    done = threading.Event()

    def watchdog():
        if not done.wait(args.exchange_timeout):
            if rank == 0:
                exch["error"] = "exchange timed out"
                emit()
            os._exit(0)
    line_box = {}

    def emit():
        line = line_box["line"]
        line["exchange"] = exch
        print(json.dumps(line), flush=True)
    hbm, hbm_kind = peaks()
    line_box["line"] = {
        "metric": METRIC, "value": 2.0 * nnz_total / (t_max * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64" if dt == np.float64 else "f32", "data": "synthetic",
        "config": {"workload": wl, "rows": m_global, "nnz": nnz_total, "graph": graph, "parallelism": f"row_div{world}",
                   "band_generation": "rank-local" if name == "c5" else "sliced", "plan_and_search_s": round(plan_s, 2),
                   "kernels": info["kernels"], "l2": "flushed before every step" if not args.no_flush else "not flushed",
                   "timing": f"median of {args.steps} steps per rank, max over ranks"},
        "roofline": {"bound": "hbm", "achieved": bytes_total / (t_max * 1e-3) / 1e9 / world, "peak": hbm,
                     "unit": "GB/s", "frac": bytes_total / (t_max * 1e-3) / 1e9 / world / hbm, "traffic": None,
                     "peak_kind": hbm_kind, "note": "per-GPU: sum of the ranks' plan bytes models / max step / N"},
        "gpu_launches": int(info["n_launches"]) * args.steps,
        "clocks": clk.summary(),
        "e2e": None,
    }
    if args.exchange != "none":
        threading.Thread(target=watchdog, daemon=True).start()
        try:
            from paper_2212_10432_b200 import dist as D
            y_full = torch.zeros(m_global, dtype=tdt, device="cuda")
            dist.barrier()
            ag = timer.steps(lambda: D.allgather_rows(dy, y_full, cuts), max(3, args.steps // 3))
            t_ag = torch.tensor([statistics.median(ag)], device=cdev(), dtype=torch.float64)
            dist.all_reduce(t_ag, op=dist.ReduceOp.MAX)
            exch["allgather_ms"] = float(t_ag.item())
            exch["allgather_bytes_per_rank"] = int((m_global - band.m) * dy.element_size())
            if args.exchange in ("nccl", "peer", "peer_halo") and cdev() == "cuda":
                d = D.init_dist(rank, world, local, cuts, nccl=args.exchange == "nccl")
                kind = "peer" if args.exchange == "peer_halo" else args.exchange
                if kind == "peer":
                    D.register_peers(d, y_full)
                if args.exchange == "peer_halo":
                    d.set_windows(D.gather_spans(A.col_span()))
                for _ in range(3):
                    d.spmv(P, 1.0, x, 0.0, y_full, kind, stream)
                torch.cuda.synchronize()
                dist.barrier()
                sd = timer.steps(lambda: d.spmv(P, 1.0, x, 0.0, y_full, kind, stream), args.steps)
                d.check()
                t_sd = torch.tensor([statistics.median(sd)], device=cdev(), dtype=torch.float64)
                dist.all_reduce(t_sd, op=dist.ReduceOp.MAX)
                exch["kind"] = args.exchange
                exch["spmv_plus_exchange_ms"] = float(t_sd.item())
                exch["spmv_plus_exchange_gflops"] = 2.0 * nnz_total / (float(t_sd.item()) * 1e-3) / 1e9
                d.close()
        except Exception as e:
            exch["error"] = str(e)[:300]
        done.set()
    if rank == 0:
        emit()
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c1..c5 (default: c3 at N=1, c5 at N>1)")
    ap.add_argument("--graph", default=None, help="skip the search and time this graph")
    ap.add_argument("--no-search", action="store_true", help="time the committed best graph")
    ap.add_argument("--search-budget", type=float, default=60.0)
    ap.add_argument("--search-candidates", type=int, default=24)
    ap.add_argument("--extra", default="c2,c4,c5", help="other configs timed in the same run (N=1)")
    ap.add_argument("--max-seconds", type=float, default=900.0, help="skip remaining extras after this")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gather", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["none", "allgather", "nccl", "peer", "peer_halo"],
                    help="N > 1: y exchange timed after the SpMV (allgather alone, plus as_spmv_dist "
                         "SpMV + exchange for nccl / peer / peer_halo)")
    ap.add_argument("--exchange-timeout", type=float, default=300.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:  # the oracle on the host; under torchrun only rank 0 runs it
            coo, wl, _ = load_config(args.config or ("c3" if world == 1 else "c5"))
            reference_arm(args, to_csr(coo), wl)
        return

    import torch
    import paper_2212_10432_b200 as asp
    if world > 1:
        multi_gpu(args, torch, asp, world, rank, local)
    else:
        single_gpu(args, torch, asp)


if __name__ == "__main__":
    main()
