#!/bin/bash
# Round-2 profiles of the current winners: the bench command's launch list (committed winner,
# no search) and ncu --set full of C3's and C4's dominant kernels, reduced to CSV pages.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out /tmp/prof
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_c3_r02b.csv \
  python bench.py --no-search --steps 5 --warmup 3 --extra "" --no-cpu-baseline --no-gather > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nnz_warp_pe -s 3 -c 1 -o /tmp/prof/c3 \
  python tools/sweep.py --config c3 --reps 2 --graphs "$C3" > gpurun_out/prof_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_nnz_warp_pe|k_dense64" -s 6 -c 2 -o /tmp/prof/c4 \
  python tools/sweep.py --config c4 --reps 2 --graphs "$C4" > gpurun_out/prof_c4.log 2>&1
for r in c3 c4; do
  ncu -i /tmp/prof/$r.ncu-rep --page raw --csv > gpurun_out/prof_${r}_r02b_raw.csv 2>/dev/null
  ncu -i /tmp/prof/$r.ncu-rep --page details --csv > gpurun_out/prof_${r}_r02b_details.csv 2>/dev/null
  ncu -i /tmp/prof/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${r}_r02b_sass.csv 2>/dev/null
  ncu -i /tmp/prof/$r.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_${r}_r02b_src.csv 2>/dev/null
done
ls -la gpurun_out/prof_*_r02b_* gpurun_out/launches_bench_c3_r02b.csv; echo done
# A/B: L2 persisting set-aside for the evict_last x gathers
for sa in 0 50331648 83886080; do
  AS_L2_SETASIDE=$sa timeout 600 python tools/sweep.py --config c3 --reps 20 --graphs "$C3" >> gpurun_out/ab_setaside.jsonl 2>> gpurun_out/ab_setaside.err
done
cut -c1-40,300-520 gpurun_out/ab_setaside.jsonl
