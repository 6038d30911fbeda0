#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_final3.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest_final3.log
tail -3 gpurun_out/gputest_final3.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final3.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final3.log; cat gpurun_out/smoke_final3.log
timeout 1500 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo "bench rc=$?" >> gpurun_out/bench_final3.err
tail -c 400 gpurun_out/bench_final3.json
