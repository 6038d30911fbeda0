# A/B on c5s: x-window staging (stages=2 -> k_nnz_thread_xw, now predicated-emit) vs direct gathers (stages=0)
G=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0); GMEM_ATOM_RED"
   "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=2); GMEM_ATOM_RED"
   "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=1,stages=2); GMEM_ATOM_RED"
   "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=1,stages=2); GMEM_ATOM_RED")
for v in "" 1; do
  env ${v:+AS_NT_LEGACY=1} python tools/sweep.py --config ${1:-c5s} --reps 20 --graphs "${G[@]}" | sed "s/^/{\"legacy\": \"$v\", \"r\": /; s/\$/}/" >> gpurun_out/ab_xw.jsonl 2>> gpurun_out/ab_xw.err
done
python -c "
import json
for l in open('gpurun_out/ab_xw.jsonl'):
    d=json.loads(l); r=d['r']; print(d['legacy'] or 'pe', round(r['median_us'],1), r['kernels'], r['graph'][70:125])"
