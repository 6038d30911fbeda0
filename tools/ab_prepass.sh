# A/B on full C5: beta=0 pre-pass as an indexed list (AS_PREPASS=1) vs a fill of y (2) (developer tool)
G=("COMPRESS; BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=GLOBAL,vec=4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED"
   "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED"
   "COMPRESS; BMW_NNZ_BLOCK(4096); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED")
for m in 1 2 1 2; do
  AS_PREPASS=$m python tools/sweep.py --config ${1:-c5} --reps 10 --graphs "${G[@]}" | sed "s/^/{\"prepass\": $m, \"r\": /; s/\$/}/" >> gpurun_out/ab_prepass.jsonl 2>> gpurun_out/ab_prepass.err
done
python -c "
import json
for l in open('gpurun_out/ab_prepass.jsonl'):
    d=json.loads(l); r=d['r']; print(d['prepass'], round(r['median_us'],1), round(r['gflops'],1), r['graph'][:90])"
