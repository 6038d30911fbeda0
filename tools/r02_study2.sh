#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider -k "history or search" > gpurun_out/t_hist.log 2>&1; echo "rc=$?" >> gpurun_out/t_hist.log; tail -3 gpurun_out/t_hist.log
timeout 2400 python tools/search_study.py --budget 45 --seeds 2 --history > gpurun_out/search_study2.jsonl 2> gpurun_out/search_study2.err
cut -c1-330 gpurun_out/search_study2.jsonl; tail -3 gpurun_out/search_study2.err
