"""bench.py — SpMV GFLOP/s and HBM GB/s (% of roofline) of the searched operator graph.

Default workload (N=1): BASELINE configs[1] = C2 `lap2d-2048`, the 5-point Laplacian on a
2048x2048 grid (4,194,304 rows, 20,963,328 nnz, fp64), alpha=1, beta=0.  One step = one
as_spmv call (the whole hot loop a5+a6; the plan a1-a4 and the search a7 run before the
timed region, as in the paper, which times the generated SpMV program) with the
inputs resident in HBM.  L2 is flushed (memset of 2 x L2 bytes) before every timed step,
outside the timed events.

Multi-GPU (torchrun, one rank per GPU): ROW_DIV bands with nnz-balanced cuts (reading A35),
each rank plans/searches its own band; the y -> x exchange (all-gather over NCCL, or the
halo of banded matrices) runs only with --exchange allgather|halo|nccl|peer.
`--impl reference` times the oracle (long-double CPU SpMV) on the host instead.
"""
from __future__ import annotations

import argparse
import json
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
    "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(128) }",
    "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); BMT_PAD(GLOBAL,1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED",
    "COMPRESS; BMTB_ROW_BLOCK(128); SHMEM_OFFSET_RED; GMEM_ATOM_RED",
]


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
    if name == "c2":
        return synth.c2_lap2d(2048), "lap2d-2048", C2_SEEDS
    if name == "c1":
        return synth.c1_uniform(int_mode=int_mode), "uniform-1k", [
            "COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; SET_RESOURCE(128); GMEM_ATOM_RED"]
    if name == "c4":
        coo, _ = synth.c4_blockdense_csr()
        return coo, "blockdense-8m", [
            "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMTB_ROW_BLOCK(32); BMT_ROW_BLOCK(1); BMT_PAD(BMTB); THREAD_TOTAL_RED; SET_RESOURCE(64); GMEM_ATOM_RED }",
            "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMW_NNZ_BLOCK(1024); BMT_NNZ_BLOCK(32); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED }",
            "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED }",
            "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }",
            "DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMTB_ROW_BLOCK(64); BMT_ROW_BLOCK(1); BMT_PAD(BMTB); THREAD_TOTAL_RED; SET_RESOURCE(128); GMEM_ATOM_RED }",
            "COMPRESS; BMTB_ROW_BLOCK(64); BMT_ROW_BLOCK(1); BMT_PAD(BMTB); THREAD_TOTAL_RED; SET_RESOURCE(128); GMEM_ATOM_RED"]
    if name == "c3":
        return synth.c3_rmat_csr(), "rmat-24", [
            "BIN(t=[32,2048]) { COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED"
            " | COMPRESS; BMTB_NNZ_BLOCK(2048); SHMEM_OFFSET_RED; GMEM_ATOM_RED"
            " | COMPRESS; BMTB_ROW_BLOCK(1); BMW_NNZ_BLOCK(2048); WARP_TOTAL_RED; GMEM_ATOM_RED }",
            "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED",
            "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,1); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
            "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16); GMEM_ATOM_RED"]
    if name in ("c3s", "c4s", "c5s"):  # shape-preserving 1/4..1/16-scale instances (dev sweeps)
        c = {"c3s": lambda: synth.c3_rmat_csr(scale=22, nnz=1 << 26),
             "c4s": lambda: synth.c4_blockdense_csr(m=1 << 21, b=64, n_tiles=6144, nnz=50_000_000)[0],
             "c5s": lambda: synth.c5_band_csr(m=1 << 22, nnz=1 << 26)}[name]()
        return c, c.name + "-scaled", []
    if name == "c5":
        return synth.c5_band_csr(), "band-irreg-64m", [
            "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0); GMEM_ATOM_RED",
            "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED",
            "COMPRESS; BMT_NNZ_BLOCK(64); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED",
            "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED",
            "COMPRESS; BMTB_ROW_BLOCK(256); SORT_BMTB; BMW_ROW_BLOCK(32); BMT_ROW_BLOCK(1); BMT_PAD(BMW); THREAD_TOTAL_RED; GMEM_ATOM_RED",
            "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"]
    raise SystemExit(f"unknown config {name}")


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


def reference_arm(args, coo, wl, scaling="strong"):
    """The oracle (long-double CSR SpMV, oracle/spmv_ref.c) on the host cores."""
    from oracle import spmv as S
    rp = csr_of(coo)
    x, _ = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    cores = os.cpu_count() or 1
    # bounded sample: the first rows covering ~1/8 of the nonzeros (C2: ~2.6M nnz) per step
    frac_rows = max(1, coo.m // 8)
    srp = rp[:frac_rows + 1]
    nnz_s = int(srp[-1])
    col, val = coo.col[:nnz_s], coo.val[:nnz_s].astype(np.float64)
    for _ in range(max(1, args.warmup)):
        S.spmv_csr(srp, col, val, x, nthreads=cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        S.spmv_csr(srp, col, val, x, nthreads=cores)
        ts.append(time.perf_counter() - t0)
    t = statistics.mean(ts)
    v = 2.0 * nnz_s / t / 1e9
    sample = f"first {frac_rows} rows ({nnz_s} nnz) of {wl} per step, long double, {cores} threads"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64x", "data": "synthetic",
            "config": {"workload": wl, "nnz": coo.nnz, "rows": coo.m},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_baseline(coo, wl, budget_s=10.0):
    from oracle import spmv as S
    rp = csr_of(coo)
    x, _ = synth.vectors(coo.n, coo.m, 2, coo.val.dtype)
    cores = os.cpu_count() or 1
    col, val = coo.col, coo.val.astype(np.float64)
    S.spmv_csr(rp, col, val, x, nthreads=cores)
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
            "sample": f"{n} full passes over {wl} ({coo.nnz} nnz), long double, {cores} threads, {t_tot:.1f} s",
            "value_1thread": 2.0 * nz1 / t1 / 1e9, "sample_1thread": f"first {r1} rows ({nz1} nnz)", "cpu": cpu,
            "long_double": "x87 80-bit extended" if platform.machine() in ("x86_64", "AMD64") else platform.machine()}


E2E_BANDS = 4  # ROW_DIV bands of the pipelined e2e plan (C2 sweep: 4 -> 0.94 ms, 8 -> 0.98, 16 -> 1.10)


def cdev():
    """Device of control-plane tensors: cuda under nccl, cpu under gloo."""
    return "cpu" if os.environ.get("AS_BENCH_BACKEND") == "gloo" else "cuda"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--graph", default=None, help="skip the search and time this graph")
    ap.add_argument("--search-budget", type=float, default=20.0)
    ap.add_argument("--search-candidates", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--exchange", default="none", choices=["none", "allgather", "halo", "nccl", "peer", "peer_halo"],
                    help="y -> next x exchange after the SpMV (N > 1), timed separately: allgather/halo "
                         "over torch.distributed; nccl/peer = as_spmv_dist (C-ABI: SpMV + AllGatherV, or "
                         "SpMV + peer-memory push; peer_halo: only the rows each peer's band reads), "
                         "timed as whole steps")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no search/baseline/e2e)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1 on c2: weak = the Laplacian grows to 2048 x 2048N and each rank owns one "
                         "2048 x 2048 ROW_DIV band (per-GPU work fixed); strong = C2 itself cut into N bands")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    weak = world > 1 and args.config == "c2" and args.scaling == "weak"
    if weak:
        # weak scaling of the ROW_DIV path: global grid 2048 x 2048*world, rank r generates
        # only its band (grid rows [2048r, 2048(r+1)), global columns)
        g = 2048
        coo = synth.c2_lap2d_band(g, g * world, g * rank, g * (rank + 1))
        wl, seeds = f"lap2d-{g}x{g * world}", C2_SEEDS
    else:
        coo, wl, seeds = load_config(args.config)
        coo = to_csr(coo)
    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, coo, wl, "weak" if args.config == "c2" and args.scaling == "weak" else "strong")
        return

    import torch
    import paper_2212_10432_b200 as asp

    if os.environ.get("AS_BENCH_BACKEND") == "gloo":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # AS_BENCH_BACKEND=gloo: control plane over gloo so that N ranks can share one GPU
        # (single-GPU validation of the N > 1 code path; the exchange kinds need nccl)
        if os.environ.get("AS_BENCH_BACKEND") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if weak:
        A = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
        cuts = np.arange(world + 1, dtype=np.int64) * coo.m
        m_global = coo.m * world
    else:
        A_full = asp.Matrix.from_csr(coo.m, coo.n, coo.row_ptr, coo.col, coo.val)
        cuts = A_full.row_cuts(world)
        m_global = coo.m
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    A = A if weak else (A_full if world == 1 else A_full.row_slice(r0, r1))
    nnz_local = A.nnz
    stream = torch.cuda.current_stream()

    t_plan = time.perf_counter()
    if args.config == "c1" and not args.graph:
        # BASELINE configs[0] names a single graph (COMPRESS + BMT_NNZ_BLOCK(4) + thread reduction)
        args.graph = seeds[0]
    if args.graph:
        P = asp.Plan(A, args.graph, device=local)
        graph = str(asp.Graph(args.graph))
        searched = False
    elif args.profile:
        P = asp.Plan(A, seeds[0], device=local)
        graph = str(asp.Graph(seeds[0]))
        searched = False
    else:
        P, graph = asp.search(A, device=local, seed=1, max_candidates=args.search_candidates,
                              budget_seconds=args.search_budget, warmup=3, reps=10, seed_graphs=seeds,
                              log_path=os.path.join(ROOT, "gpurun_out", f"search_{wl}_r{rank}.jsonl")
                              if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else None)
        searched = True
    plan_s = time.perf_counter() - t_plan
    info = P.info()
    dt = coo.val.dtype
    x, _ = synth.vectors(coo.n, coo.m, 2, dt)
    dx = torch.from_numpy(x).cuda()
    m_local = r1 - r0
    dy = torch.zeros(m_local, dtype=torch.float64 if dt == np.float64 else torch.float32, device="cuda")
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")

    def step():
        P.spmv(1.0, dx, 0.0, dy, stream)

    def flush_l2():
        # write 2x L2 (the flush), then read it back so the dirty lines are written back to
        # HBM before the timed region rather than during it
        flush.zero_()
        flush.view(torch.int64).sum()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        for e0, e1 in evs:
            if not args.no_flush:
                flush_l2()
            e0.record(stream)
            step()
            e1.record(stream)
        torch.cuda.synchronize()
        gather_ms = None
        if args.exchange in ("nccl", "peer", "peer_halo") and dist:
            # as_spmv_dist: band SpMV into y_full + the exchange inside the library
            from paper_2212_10432_b200 import dist as D
            d = D.init_dist(rank, world, local, cuts, nccl=args.exchange == "nccl")
            y_full = torch.zeros(m_global, dtype=dy.dtype, device="cuda")
            kind = "peer" if args.exchange == "peer_halo" else args.exchange
            if kind == "peer":
                D.register_peers(d, y_full)
            if args.exchange == "peer_halo":
                d.set_windows(D.gather_spans(A.col_span()))
            for _ in range(3):
                d.spmv(P, 1.0, dx, 0.0, y_full, kind, stream)
            torch.cuda.synchronize()
            dist.barrier()
            gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for g0, g1 in gev:
                if not args.no_flush:
                    flush_l2()
                g0.record(stream)
                d.spmv(P, 1.0, dx, 0.0, y_full, kind, stream)
                g1.record(stream)
            torch.cuda.synchronize()
            d.check()
            gather_ms = statistics.mean(g0.elapsed_time(g1) for g0, g1 in gev)
            dist.barrier()
            d.close()
        elif args.exchange != "none" and dist:
            # y -> next x: all-gather (uneven bands, NCCL broadcasts) or halo (P2P of the
            # band's column span only, NEXT-1), timed separately from the SpMV
            from paper_2212_10432_b200 import dist as D
            x_next = torch.zeros(m_global, dtype=dy.dtype, device="cuda")
            moves = D.halo_plan(D.gather_spans(A.col_span()), cuts) if args.exchange == "halo" else None
            dist.barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            if args.exchange == "halo":
                D.halo_exchange(dy, x_next, cuts, moves)
            else:
                D.allgather_rows(dy, x_next, cuts)
            g1.record(stream)
            torch.cuda.synchronize()
            gather_ms = g0.elapsed_time(g1)
    if gather_ms is not None:
        gm = torch.tensor([gather_ms], device=cdev(), dtype=torch.float64)
        dist.all_reduce(gm, op=dist.ReduceOp.MAX)
        gather_ms = float(gm.item())
    ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    t_ms = statistics.mean(ms)
    if dist:
        tt = torch.tensor([t_ms], device=cdev(), dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        tot = torch.tensor([float(nnz_local)], device=cdev(), dtype=torch.float64)
        dist.all_reduce(tot)
        nnz_total = int(tot.item())
    else:
        nnz_total = nnz_local
    gflops = 2.0 * nnz_total / (t_ms * 1e-3) / 1e9
    hbm, hbm_kind = peaks()
    achieved_step = info["bytes_model"] / (t_ms * 1e-3) / 1e9
    launches = int(info["n_launches"])
    # dominant kernel: per-launch device times (as_plan_profile, CUDA events between the
    # launches, L2 flushed before each pass) and per-launch algorithmic bytes
    dominant = None
    if not args.profile:
        acc = None
        for _ in range(max(3, args.steps // 3)):
            if not args.no_flush:
                flush_l2()
            prof = P.profile(dx, dy, reps=1, stream=stream)
            acc = [[n, ms, by] for n, ms, by in prof] if acc is None else [[a[0], a[1] + p_[1], a[2]] for a, p_ in zip(acc, prof)]
        npass = max(3, args.steps // 3)
        per = [(n, ms / npass, by) for n, ms, by in acc]
        name, dms, dby = max(per, key=lambda e: e[1])
        dominant = {"kernel": name, "ms": dms, "bytes": dby, "share_of_step": dms / t_ms if t_ms else None,
                    "launches": [{"kernel": n, "ms": ms, "bytes": by} for n, ms, by in per]}
    achieved_gbs = (dominant["bytes"] / (dominant["ms"] * 1e-3) / 1e9) if dominant and dominant["ms"] > 0 else achieved_step

    # e2e through the C-ABI with host buffers (pinned), copies inside the timed region.  Two
    # plans: the searched one (copies, kernels, copies back to back) and the same graph under
    # ROW_DIV into E2E_BANDS bands, which as_spmv_host pipelines (chunked H2D of x and D2H of
    # y on copy streams overlapping the band kernels); the faster is reported.
    e2e = None
    if not args.profile:
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.zeros(m_local, dtype=dy.dtype).pin_memory()
        xn, yn = xh.numpy(), yh.numpy()
        cands = [(graph, P)]
        if "ROW_DIV" not in graph and m_local >= 8 * E2E_BANDS:
            cut = ",".join(str(m_local * i // E2E_BANDS) for i in range(1, E2E_BANDS))
            g_pipe = f"ROW_DIV(cuts=[{cut}]) {{ {graph} }}"
            try:
                cands.append((g_pipe, asp.Plan(A, g_pipe, device=local)))
            except asp.AsError:
                pass
        res = []
        for g_e, P_e in cands:
            for _ in range(2):
                P_e.spmv_host(1.0, xn, 0.0, yn, stream)
            e2e_ms = []
            for _ in range(max(3, args.steps // 3)):
                if not args.no_flush:
                    flush_l2()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                P_e.spmv_host(1.0, xn, 0.0, yn, stream)
                e1.record(stream)
                torch.cuda.synchronize()
                e2e_ms.append(e0.elapsed_time(e1))
            res.append((statistics.mean(e2e_ms), g_e, int(P_e.info()["n_launches"])))
        tm, g_e, l_e = min(res)
        if dist:
            tt = torch.tensor([tm], device=cdev(), dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tm = float(tt.item())
        sv = dx.element_size()
        e2e = {"value": 2.0 * nnz_total / (tm * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": tm,
               "h2d_bytes_per_step": int(coo.n * sv), "d2h_bytes_per_step": int(m_local * sv),
               "graph": g_e, "launches_per_step": l_e,
               "candidates_ms": {("pipelined" if i else "searched"): r[0] for i, r in enumerate(res)}}

    # warm steady state: back-to-back calls in one event window, no
    # flush -- for C2 the working set is a small multiple of L2
    warm = None
    if not args.profile:
        nw = 100 if t_ms < 1.0 else 20
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0.record(stream)
        for _ in range(nw):
            step()
        w1.record(stream)
        torch.cuda.synchronize()
        wm = w0.elapsed_time(w1) / nw
        warm = {"ms_per_step": wm, "gflops": 2.0 * nnz_local / (wm * 1e-3) / 1e9, "calls": nw}

    # CUDA-graph replay of the same plan (AS_PLAN_GRAPH): the launch-latency floor of small
    # matrices ("C1 also reports CUDA-Graph replay time"); small workloads only
    graph_replay = None
    if not args.profile and nnz_local < 50_000_000:
        Pg = asp.Plan(A, graph, device=local, graph_replay=True)
        for _ in range(3):
            Pg.spmv(1.0, dx, 0.0, dy, stream)
        gts = []
        for _ in range(args.steps):
            if not args.no_flush:
                flush_l2()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            Pg.spmv(1.0, dx, 0.0, dy, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            gts.append(e0.elapsed_time(e1))
        graph_replay = {"ms_per_step": statistics.mean(gts), "gflops": 2.0 * nnz_local / (statistics.mean(gts) * 1e-3) / 1e9}
        del Pg

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    traffic = None
    # weak-scaled C2 bands run the same per-rank kernel as C2 itself
    prof = os.path.join(ROOT, "profiles", f"traffic_{'lap2d-2048' if weak else wl}.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            if tj.get("kernels") == info["kernels"]:
                traffic = tj["dram_bytes_per_launch"]
        except Exception:
            pass
    line = {
        "metric": METRIC, "value": gflops, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
        "scaling": "weak" if (weak or world == 1) and args.config == "c2" and args.scaling == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64" if dt == np.float64 else "f32", "data": "synthetic",
        "config": {"workload": wl, "rows": m_global, "nnz": nnz_total, "graph": graph, "searched": searched,
                   "alpha": 1.0, "beta": 0.0, "l2": "flushed before every step" if not args.no_flush else "not flushed",
                   "parallelism": f"row_div{world}", "plan_and_search_s": round(plan_s, 2),
                   "kernels": info["kernels"], "bytes_model": info["bytes_model"], "bytes_floor": info["bytes_floor"]},
        "hbm_gbs_model": achieved_gbs,
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": achieved_gbs / hbm, "traffic": traffic, "peak_kind": hbm_kind,
                     "frac_of_8tbs": achieved_gbs / 8000.0,
                     # measured DRAM bytes of the dominant kernel (ncu, committed) over the same
                     # time: the model counts x and y in full although part of them stays in
                     # L2, and a read-dominated stream can beat the copy peak, so frac may
                     # exceed 1 where frac_dram does not
                     "achieved_dram": (traffic / (t_ms * 1e-3) / 1e9) if traffic else None,
                     "frac_dram": (traffic / (t_ms * 1e-3) / 1e9 / hbm) if traffic else None,
                     "achieved_step": achieved_step, "frac_step": achieved_step / hbm,
                     "dominant": dominant,
                     "note": "achieved = algorithmic bytes of the dominant kernel / its mean launch duration "
                             "(CUDA events between launches, as_plan_profile); achieved_step = the plan's "
                             "bytes model / the step time" + (" (single launch)" if launches == 1 else
                                                              f" ({launches} launches)")},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if graph_replay is not None:
        line["graph_replay"] = graph_replay
    if warm is not None:
        line["warm"] = warm
    if gather_ms is not None:
        line["exchange"] = {"kind": args.exchange, "ms": gather_ms,
                            "timed": "spmv + exchange per step (as_spmv_dist)" if args.exchange in ("nccl", "peer", "peer_halo")
                            else "exchange only"}
    if not args.no_cpu_baseline and not args.profile and world == 1:
        line["cpu_baseline"] = cpu_baseline(coo, wl)
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
