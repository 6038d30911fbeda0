#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
C3="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['rmat-24']['graph'])")"
C5="$(python -c "import json;print(json.load(open('profiles/best_graphs.json'))['band-irreg-64m']['graph'])")"
timeout 600 python tools/sweep.py --config c3 --reps 20 --graphs "$C3" "${C3/xcache=24576/xcache=32768}" "${C3/xcache=24576/xcache=16384}" > gpurun_out/cg_c3.jsonl 2>&1
timeout 600 python tools/sweep.py --config c5 --reps 10 --graphs "$C5" > gpurun_out/cg_c5.jsonl 2>&1
python -c "
import json
for f in ['gpurun_out/cg_c3.jsonl','gpurun_out/cg_c5.jsonl']:
    for l in open(f):
        try: d=json.loads(l); print(d['config'], d['graph'][-60:], round(d['median_us'],1))
        except Exception: pass
"
bash tools/r02_conc.sh
