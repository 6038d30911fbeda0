# as_search with vs without the cost-model stage on the scaled irregular configs (developer tool)
for c in c5s c3s c4s; do
  for s in 1 2; do
    python tools/search_ab.py --config $c --budget 40 --seed $s --no-surrogate >> gpurun_out/search_ab.jsonl 2>> gpurun_out/search_ab.err
    python tools/search_ab.py --config $c --budget 40 --seed $s >> gpurun_out/search_ab.jsonl 2>> gpurun_out/search_ab.err
  done
done
cat gpurun_out/search_ab.jsonl
