#!/bin/bash
# A/B: k_nnz_warp_pe launch bound 768 with 16-element fp32 batches (more registers per thread)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
G768="${C3/tpb=1024/tpb=768}"
G512="${C3/tpb=1024/tpb=512}"
timeout 600 python tools/sweep.py --config c3 --reps 20 --graphs "$C3" "$G768" "$G512" >> gpurun_out/ab_lb.jsonl 2>> gpurun_out/ab_lb.err
AS_LIB_AB=paper_2212_10432_b200/libalphasparse_lb768.so timeout 600 python tools/sweep.py --config c3 --reps 20 --graphs "$G768" "$G512" >> gpurun_out/ab_lb.jsonl 2>> gpurun_out/ab_lb.err
python - <<'PY'
import json, re
for l in open("gpurun_out/ab_lb.jsonl"):
    d = json.loads(l)
    m = re.search(r"tpb=(\d+)", d.get("graph", ""))
    print(d["config"], (d.get("lib") or "main")[-12:], m.group(1) if m else "-", round(d.get("median_us", -1), 1), d.get("y_abs_sum"), d.get("error", "")[:80])
PY
