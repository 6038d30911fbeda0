#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest4.log 2>&1; echo "rc=$?" >> gpurun_out/gputest4.log
tail -4 gpurun_out/gputest4.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log; cat gpurun_out/smoke2.log
timeout 1800 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?" >> gpurun_out/bench3.err
tail -2 gpurun_out/bench3.err
