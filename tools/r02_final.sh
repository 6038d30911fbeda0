#!/bin/bash
# Round-2 final state on the B200: default bench line, PCIe copy bandwidth, the bench's ncu
# launch list (committed winners, no search), GPU suite, smoke.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_final.txt 2>&1
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?" >> gpurun_out/bench_final.err
tail -c 300 gpurun_out/bench_final.json; echo
timeout 120 python tools/pcie_bw.py > gpurun_out/pcie.json 2>&1; cat gpurun_out/pcie.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_final.csv \
  python bench.py --no-search --steps 5 --warmup 3 --no-cpu-baseline --no-gather > gpurun_out/launches_bench_final.log 2>&1
echo "ncu rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest_final.log
tail -3 gpurun_out/gputest_final.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log; cat gpurun_out/smoke_final.log
