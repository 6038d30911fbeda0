#!/bin/bash
# ncu --set full of the C3 and C4 winners' dominant kernels (run under gpurun, repo root).
# The reports are reduced to CSV pages on the box (gpurun brings back <= 64 MiB).
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
mkdir -p /tmp/prof
ncu --set full --clock-control none --import-source on -k regex:k_nnz_warp_pe -s 3 -c 1 -o /tmp/prof/c3 \
  python tools/sweep.py --config c3 --reps 2 --graphs "$C3" > gpurun_out/prof_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_nnz_warp_pe|k_dense64" -s 6 -c 2 -o /tmp/prof/c4 \
  python tools/sweep.py --config c4 --reps 2 --graphs "$C4" > gpurun_out/prof_c4.log 2>&1
for r in c3 c4; do
  ncu -i /tmp/prof/$r.ncu-rep --page raw --csv > gpurun_out/prof_${r}_r02_raw.csv 2>/dev/null
  ncu -i /tmp/prof/$r.ncu-rep --page details --csv > gpurun_out/prof_${r}_r02_details.csv 2>/dev/null
  ncu -i /tmp/prof/$r.ncu-rep --page source --csv > gpurun_out/prof_${r}_r02_source.csv 2>/dev/null
done
ls -la gpurun_out/prof_*_r02_* ; echo done
