#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/refresh_winners.py --configs c4 --budget 600 --candidates 400 > gpurun_out/refresh_c4.jsonl 2> gpurun_out/refresh_c4.err
tail -2 gpurun_out/refresh_c4.jsonl
python - <<'PY'
import json
rows = [json.loads(l) for l in open("gpurun_out/search_blockdense-8m_refresh.jsonl")]
rows = [r for r in rows if r.get("median_ms", -1) > 0]
rows.sort(key=lambda r: r["median_ms"])
for r in rows[:8]:
    print(round(r["median_ms"] * 1e3, 1), r["graph"][:400])
PY
