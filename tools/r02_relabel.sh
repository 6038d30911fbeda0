#!/bin/bash
# Column-relabel gather experiment + quick GPU regression of the split kernel build.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider > gpurun_out/gputest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_quick.log
timeout 1200 python tools/gather_roofline.py --configs c3 --relabel --hot 16384 24576 32768 49152 > gpurun_out/gather_relabel.jsonl 2> gpurun_out/gather_relabel.err
tail -2 gpurun_out/gputest_quick.log; cat gpurun_out/gather_relabel.jsonl | cut -c1-220
