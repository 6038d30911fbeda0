#!/bin/bash
# R-conc: GPU parity of the concurrent-branch graphs + C4 / C2 timings with the DENSE / DIA branch on a side stream
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_spmm.py -m gpu -x -q -p no:cacheprovider -k "family or spmm or random_graphs or concurrent" > gpurun_out/conc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/conc_tests.log
tail -3 gpurun_out/conc_tests.log
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
C2="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['lap2d-2048']['graph'])")"
C4S="${C4/xcache=0) |/xcache=0,stream=1) |}"
G=("$C4" "$C4S")
for r in "tpb=256,grid=3" "tpb=384,grid=2" "tpb=1024,grid=1" "tpb=256,grid=4" "tpb=512,grid=1"; do
  G+=("${C4S/tpb=512,grid=2/$r}")
done
timeout 900 python tools/sweep.py --config c4 --reps 20 --graphs "${G[@]}" > gpurun_out/conc3_c4.jsonl 2> gpurun_out/conc2.err
timeout 300 python tools/sweep.py --config c2 --reps 20 --graphs "$C2" "${C2/\{ DIA |/\{ DIA; SET_RESOURCE(stream=1) |}" > gpurun_out/conc3_c2.jsonl 2>> gpurun_out/conc2.err
python - <<'PY'
import json, re
for f in ["gpurun_out/conc3_c4.jsonl", "gpurun_out/conc3_c2.jsonl"]:
    for l in open(f):
        d = json.loads(l)
        m = re.findall(r"SET_RESOURCE\(([^)]*)\)", d.get("graph", ""))
        print(d.get("config"), m, round(d.get("median_us", -1), 1), d.get("y_abs_sum"), d.get("error", ""))
PY
