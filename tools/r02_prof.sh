#!/bin/bash
# ncu --set full of the C3 and C4 winners' dominant kernels (run under gpurun, repo root)
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
ncu --set full --clock-control none --import-source on -k regex:k_nnz_warp_pe -s 3 -c 1 -o gpurun_out/prof_c3_r02 \
  python tools/sweep.py --config c3 --reps 2 --graphs "$C3" > gpurun_out/prof_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_nnz_warp_pe|k_dense64" -s 6 -c 2 -o gpurun_out/prof_c4_r02 \
  python tools/sweep.py --config c4 --reps 2 --graphs "$C4" > gpurun_out/prof_c4.log 2>&1
echo done
