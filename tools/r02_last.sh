#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_spmm.py tests/test_bench_contract.py tests/test_dist_gpu.py -m gpu -x -q -p no:cacheprovider -k "concurrent or heavy or family or spmm or contract or batch or dist or peer" > gpurun_out/last.log 2>&1; echo "rc=$?" >> gpurun_out/last.log
tail -3 gpurun_out/last.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
