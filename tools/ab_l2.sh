# A/B: x in an L2 persisting access-policy window during as_spmv (AS_L2_PERSIST=1) vs evict_last hints only
G3=("COMPRESS; BMW_NNZ_BLOCK(4096); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED")
G4=("DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMW_NNZ_BLOCK(1024); BMT_NNZ_BLOCK(16); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED }")
for v in "" 1 "" 1; do
  env ${v:+AS_L2_PERSIST=1} python tools/sweep.py --config ${1:-c3} --reps 10 --graphs "${G3[@]}" | sed "s/^/{\"persist\": \"$v\", \"r\": /; s/\$/}/" >> gpurun_out/ab_l2.jsonl 2>> gpurun_out/ab_l2.err
  env ${v:+AS_L2_PERSIST=1} python tools/sweep.py --config ${2:-c4} --reps 10 --graphs "${G4[@]}" | sed "s/^/{\"persist\": \"$v\", \"r\": /; s/\$/}/" >> gpurun_out/ab_l2.jsonl 2>> gpurun_out/ab_l2.err
done
python -c "
import json
for l in open('gpurun_out/ab_l2.jsonl'):
    d=json.loads(l); r=d['r']; print(d['persist'] or '-', r['config'], round(r['median_us'],1))"
