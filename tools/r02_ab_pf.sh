#!/bin/bash
# A/B: column look-ahead + predicated EM0 stores + shared-window hot-x loads (main) vs the
# same without look-ahead (nola) vs the previous commit (head)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
C4="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['blockdense-8m']['graph'])")"
C5="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['band-irreg-64m']['graph'])")"
for cfg in c3 c4 c5; do
  G=$C3; [ $cfg = c4 ] && G=$C4; [ $cfg = c5 ] && G=$C5
  for lib in "" pf; do
    export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
    timeout 600 python tools/sweep.py --config $cfg --reps 20 --graphs "$G" >> gpurun_out/ab_pf.jsonl 2>> gpurun_out/ab_pf.err
  done
done
unset AS_LIB_AB
python - <<'PY'
import json
for l in open("gpurun_out/ab_pf.jsonl"):
    d = json.loads(l)
    print(d["config"], (d["lib"] or "main")[-12:], round(d.get("median_us", -1), 1), d.get("y_abs_sum"))
PY
