#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_spmm.py tests/test_bench_contract.py -m gpu -x -q -p no:cacheprovider -k "concurrent or heavy or family or spmm or contract or batch" > gpurun_out/conc_check.log 2>&1; echo "rc=$?" >> gpurun_out/conc_check.log
tail -3 gpurun_out/conc_check.log
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
timeout 600 python tools/sweep.py --config c4 --reps 20 --graphs "$C4" > gpurun_out/conc_check_c4.jsonl 2>&1; cut -c1-60,400-700 gpurun_out/conc_check_c4.jsonl | head -3
