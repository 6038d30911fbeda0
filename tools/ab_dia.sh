# A/B of the DIA kernel forms on C2 (developer tool): 16-B loads, 2 rows/thread (0) vs 8-B loads, 1 row/thread, <= 32 regs (3)
G=("DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=512,grid=4) }"
   "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=256,grid=8) }"
   "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=1024,grid=2) }"
   "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=128,grid=0) }")
for v in 0 3 0 3; do
  AS_DIA_VARIANT=$v python tools/sweep.py --config c2 --reps 30 --graphs "${G[@]}" | sed "s/^/{\"variant\": $v, \"r\": /; s/\$/}/" >> gpurun_out/ab_dia3.jsonl 2>> gpurun_out/ab_dia.err
done
python -c "
import json
for l in open('gpurun_out/ab_dia3.jsonl'):
    d=json.loads(l); r=d['r']; print(d['variant'], round(r['median_us'],2), round(r['min_us'],2), round(r['model_gbs']), r['graph'][:70])"
