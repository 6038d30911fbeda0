#!/bin/bash
# A/B: fp32 per-lane segment accumulation (AS_F32_ACC) on C3; parity of the fp32 family
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
AS_LIB_AB=paper_2212_10432_b200/libalphasparse_f32acc.so timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -k "family or xcache or c3 or heavy" > gpurun_out/f32acc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f32acc_tests.log
tail -3 gpurun_out/f32acc_tests.log
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
for lib in "" f32acc; do
  export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
  timeout 600 python tools/sweep.py --config c3 --reps 20 --graphs "$C3" >> gpurun_out/ab_f32acc.jsonl 2>> gpurun_out/ab_f32acc.err
done
unset AS_LIB_AB
python - <<'PY'
import json
for l in open("gpurun_out/ab_f32acc.jsonl"):
    d = json.loads(l)
    print(d["config"], (d.get("lib") or "main")[-14:], round(d.get("median_us", -1), 1), d.get("y_abs_sum"))
PY
