#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_devbuild.py -m gpu -x -q -p no:cacheprovider -k "search" > gpurun_out/search_check.log 2>&1; echo "rc=$?" >> gpurun_out/search_check.log
tail -3 gpurun_out/search_check.log
