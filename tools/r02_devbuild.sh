#!/bin/bash
# On-device Designer: its tests, the whole GPU suite (make_plan routes eligible graphs to it), plan times
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_devbuild.py -x -q -p no:cacheprovider > gpurun_out/devbuild_tests.log 2>&1; echo "rc=$?" >> gpurun_out/devbuild_tests.log
tail -30 gpurun_out/devbuild_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest2.log 2>&1; echo "rc=$?" >> gpurun_out/gputest2.log
tail -15 gpurun_out/gputest2.log
timeout 1200 python tools/plan_time.py --configs c3 c5 > gpurun_out/plan_time.jsonl 2> gpurun_out/plan_time.err
cat gpurun_out/plan_time.jsonl | cut -c1-60,200-400; tail -3 gpurun_out/plan_time.err
