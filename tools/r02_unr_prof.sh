#!/bin/bash
# gather rate vs loads in flight per thread (hot-x .cg microbenchmark) + ncu --set full of the C3 winner (.cg build)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out /tmp/prof
timeout 900 python tools/gather_roofline.py --configs c3 --reps 9 --hot 24576 --unr 1 2 4 8 --xld-hot 24576 \
  > gpurun_out/gather_unr.jsonl 2> gpurun_out/gather_unr.err
python -c "
import json
for l in open('gpurun_out/gather_unr.jsonl'):
    d=json.loads(l); print(d['kernel'], round(d['median_us'],1))
"
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nnz_warp_pe -s 3 -c 1 -o /tmp/prof/c3cg \
  python tools/sweep.py --config c3 --reps 2 --graphs "$C3" > gpurun_out/prof_c3cg.log 2>&1
ncu -i /tmp/prof/c3cg.ncu-rep --page raw --csv > gpurun_out/prof_c3cg_raw.csv 2>/dev/null
ncu -i /tmp/prof/c3cg.ncu-rep --page details --csv > gpurun_out/prof_c3cg_details.csv 2>/dev/null
ncu -i /tmp/prof/c3cg.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_c3cg_sass.csv 2>/dev/null
ls -la gpurun_out/prof_c3cg_*
