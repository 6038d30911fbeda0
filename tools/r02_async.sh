#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/gather_roofline.py --configs c3 c4 --async-gather --hot 16384 --reps 10 > gpurun_out/gather_async.jsonl 2> gpurun_out/gather_async.err
cut -c1-40,120-260 gpurun_out/gather_async.jsonl
timeout 900 python tools/plan_time.py --configs c3 c5 > gpurun_out/plan_time2.jsonl 2> gpurun_out/plan_time2.err
timeout 1800 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?" >> gpurun_out/bench2.err
tail -c 300 gpurun_out/bench2.json
