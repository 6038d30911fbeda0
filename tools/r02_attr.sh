#!/bin/bash
# Attribution of the C3 kernel time (experiment builds: no y stores / no bitmap / neither)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
for lib in "" xny xnb xnbny; do
  export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
  timeout 600 python tools/sweep.py --config c3 --reps 20 --graphs "$C3" >> gpurun_out/attr.jsonl 2>> gpurun_out/attr.err
done
unset AS_LIB_AB
python - <<'PY'
import json
for l in open("gpurun_out/attr.jsonl"):
    d = json.loads(l)
    print(d["config"], (d["lib"] or "main")[-14:], round(d.get("median_us", -1), 1))
PY
