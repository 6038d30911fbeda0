#!/bin/bash
# timing experiment: DENSE part concurrent with the gather-bound residual (AS_CONC_EXP, y not checked)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
G=("$C4")
for r in "tpb=512,grid=1" "tpb=256,grid=2" "tpb=256,grid=3" "tpb=384,grid=2" "tpb=1024,grid=1"; do
  G+=("${C4/tpb=512,grid=2/$r}")
done
for m in 0 1 3 2; do
  AS_CONC_EXP=$m timeout 900 python tools/sweep.py --config c4 --reps 15 --graphs "${G[@]}" | sed "s/^{/{\"conc\": $m, /" >> gpurun_out/conc.jsonl 2>> gpurun_out/conc.err
done
python - <<'PY'
import json, re
for l in open("gpurun_out/conc.jsonl"):
    d = json.loads(l)
    m = re.findall(r"SET_RESOURCE\(([^)]*)\)", d.get("graph", ""))
    print(d["conc"], m[-1] if m else "-", round(d.get("median_us", -1), 1))
PY
