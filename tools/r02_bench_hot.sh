#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --no-search --extra "" --no-cpu-baseline > gpurun_out/bench_hot.json 2> gpurun_out/bench_hot.err; echo "rc=$?"
tail -3 gpurun_out/bench_hot.err
python -c "
import json; d=json.load(open('gpurun_out/bench_hot.json')); print(d['ms_per_step'], json.dumps(d['roofline_detail']['gather']))"
