#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -m gpu -x -q -p no:cacheprovider -k "batch or concurrent or host" > gpurun_out/e2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_tests.log; tail -2 gpurun_out/e2e_tests.log
timeout 900 python bench.py --no-search --extra "" --no-cpu-baseline --no-gather > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['ms_per_step'], json.dumps(d['e2e']))"
