#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bench_contract.py tests/test_gpu.py -m gpu -x -q -p no:cacheprovider -k "contract or concurrent or heavy" > gpurun_out/contract.log 2>&1; echo "rc=$?" >> gpurun_out/contract.log
tail -15 gpurun_out/contract.log
