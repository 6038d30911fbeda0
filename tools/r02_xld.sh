#!/bin/bash
# x-gather load variants x hot-x copy size on C3 / C4 residual (gather microbenchmark)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python tools/gather_roofline.py --configs c3 c4 --reps 9 --hot 32768 --xld 0 1 2 3 4 \
  --xld-hot 0 24576 32768 40960 49152 --xld-tpb 1024 512 > gpurun_out/gather_xld.jsonl 2> gpurun_out/gather_xld.err
echo "rc=$?"; tail -3 gpurun_out/gather_xld.err
