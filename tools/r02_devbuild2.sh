#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 900 python -m pytest tests/test_devbuild.py -x -q -p no:cacheprovider > gpurun_out/devbuild_tests.log 2>&1; echo "rc=$?" >> gpurun_out/devbuild_tests.log
tail -5 gpurun_out/devbuild_tests.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gputest3.log 2>&1; echo "rc=$?" >> gpurun_out/gputest3.log
tail -40 gpurun_out/gputest3.log
timeout 900 python tools/plan_time.py --configs c3 c5 > gpurun_out/plan_time.jsonl 2> gpurun_out/plan_time.err
cat gpurun_out/free.txt
