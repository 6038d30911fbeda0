#!/bin/bash
# A/B of the x-gather L1 behaviour (AS_X_LD) x hot-x copy size on the C3 / C4 winners
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
G3=()
for K in 24576 32768 40960 49152; do G3+=("${C3/xcache=24576/xcache=$K}"); done
for lib in "" xld1 xld2 xld3; do
  export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
  timeout 600 python tools/sweep.py --config c3 --reps 15 --graphs "${G3[@]}" >> gpurun_out/ab_xld.jsonl 2>> gpurun_out/ab_xld.err
  timeout 600 python tools/sweep.py --config c4 --reps 15 --graphs "$C4" >> gpurun_out/ab_xld.jsonl 2>> gpurun_out/ab_xld.err
done
unset AS_LIB_AB
python - <<'PY'
import json, re
for l in open("gpurun_out/ab_xld.jsonl"):
    d = json.loads(l)
    m = re.search(r"xcache=(\d+)", d.get("graph", ""))
    print(d["config"], (d.get("lib") or "main")[-12:], m.group(1) if m else "-", round(d.get("median_us", -1), 1))
PY
