#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"
done
for f in gpurun_out/san_*.log; do echo "$f: $(grep -c '^ok' $f) ok, $(grep 'ERROR SUMMARY' $f)"; done
