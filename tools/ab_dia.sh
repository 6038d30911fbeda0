# A/B of the DIA kernel forms on C2 (developer tool): direct 16-B loads (0), 32-B loads (1), TMA-staged (2)
G=("DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=512,grid=4) }"
   "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=128,grid=16) }")
for v in 0 2 1 0 2; do
  AS_DIA_VARIANT=$v python tools/sweep.py --config c2 --reps 30 --graphs "${G[@]}" | sed "s/^/{\"variant\": $v, \"r\": /; s/\$/}/" >> gpurun_out/ab_dia.jsonl 2>> gpurun_out/ab_dia.err
done
python -c "
import json
for l in open('gpurun_out/ab_dia.jsonl'):
    d=json.loads(l); r=d['r']; print(d['variant'], round(r['median_us'],2), round(r['min_us'],2), round(r['model_gbs']), r['graph'][:70])"
