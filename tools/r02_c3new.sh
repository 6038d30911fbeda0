#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out /tmp/prof
OLD="COMPRESS; BMW_NNZ_BLOCK(nnz=8192); BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=0,stages=2,xcache=24576); GMEM_ATOM_RED"
NEW="COMPRESS; BMW_NNZ_BLOCK(nnz=4096); BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=8,stages=2,xcache=24576); GMEM_ATOM_RED"
timeout 600 python tools/sweep.py --config c3 --reps 30 --graphs "$OLD" "$NEW" "$OLD" "$NEW" > gpurun_out/c3new.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/c3new.jsonl'):
    try: d=json.loads(l); print(round(d['median_us'],1), d['bytes_model'], d['kernels'], d['graph'][:60])
    except Exception: pass
"
timeout 900 ncu --set full --clock-control none -k regex:k_nnz_warp_pe -s 3 -c 1 -o /tmp/prof/c3new \
  python tools/sweep.py --config c3 --reps 2 --graphs "$NEW" > gpurun_out/prof_c3new.log 2>&1
ncu -i /tmp/prof/c3new.ncu-rep --page raw --csv > gpurun_out/prof_c3new_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/prof_c3new_raw.csv")))
h, u, v = rows[0], rows[1], rows[2]
for a, b, c in zip(h, u, v):
    if a in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"):
        print(a, b, c)
PY
