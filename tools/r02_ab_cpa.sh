#!/bin/bash
# A/B: cp.async-staged stream (AS_CPA) in the xcache warp kernel; parity first
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
AS_LIB_AB=paper_2212_10432_b200/libalphasparse_cpa.so timeout 900 python -m pytest tests/test_gpu.py tests/test_devbuild.py -m gpu -x -q -p no:cacheprovider -k "xcache or family_real or committed" > gpurun_out/cpa_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cpa_tests.log
tail -3 gpurun_out/cpa_tests.log
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
G=("$C3" "${C3/xcache=24576/xcache=16384}" "${C3/xcache=24576/xcache=20480}")
for lib in "" cpa; do
  export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
  timeout 600 python tools/sweep.py --config c3 --reps 20 --graphs "${G[@]}" >> gpurun_out/ab_cpa.jsonl 2>> gpurun_out/ab_cpa.err
done
unset AS_LIB_AB
python - <<'PY'
import json, re
for l in open("gpurun_out/ab_cpa.jsonl"):
    d = json.loads(l)
    m = re.search(r"xcache=(\d+)", d.get("graph", ""))
    print(d["config"], (d.get("lib") or "main")[-12:], m.group(1) if m else "-", round(d.get("median_us", -1), 1), d.get("y_abs_sum"), d.get("error", "")[:80])
PY
