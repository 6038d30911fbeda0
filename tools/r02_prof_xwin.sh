#!/bin/bash
# ncu --set full of C5's x-window kernel and of the committed C5 kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out /tmp/prof
GX="COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=2); GMEM_ATOM_RED"
G0="COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0); GMEM_ATOM_RED"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o /tmp/prof/c5x \
  python tools/sweep.py --config c5 --reps 1 --graphs "$GX" > gpurun_out/prof_c5x.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o /tmp/prof/c50 \
  python tools/sweep.py --config c5 --reps 1 --graphs "$G0" > gpurun_out/prof_c50.log 2>&1
for r in c5x c50; do
  ncu -i /tmp/prof/$r.ncu-rep --page details --csv > gpurun_out/prof_${r}_details.csv 2>/dev/null
  ncu -i /tmp/prof/$r.ncu-rep --page raw --csv > gpurun_out/prof_${r}_raw.csv 2>/dev/null
  ncu -i /tmp/prof/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${r}_sass.csv 2>/dev/null
done
ls -la gpurun_out/prof_c5*
