# A/B: k_nnz_thread branching form (AS_NT_LEGACY=1) vs predicated-emit form (developer tool)
G5=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(16); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=8,stages=0); GMEM_ATOM_RED")
G3=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(16); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED")
CFG5=${1:-c5s}; CFG3=${2:-c3s}
for leg in 1 ""; do
  tag=${leg:+legacy}; tag=${tag:-pe}
  env ${leg:+AS_NT_LEGACY=1} python tools/sweep.py --config $CFG5 --reps 20 --graphs "${G5[@]}" > gpurun_out/ab_pe_${CFG5}_$tag.jsonl 2>> gpurun_out/ab_pe.err
  env ${leg:+AS_NT_LEGACY=1} python tools/sweep.py --config $CFG3 --reps 20 --graphs "${G3[@]}" > gpurun_out/ab_pe_${CFG3}_$tag.jsonl 2>> gpurun_out/ab_pe.err
done
for f in gpurun_out/ab_pe_*.jsonl; do echo "== $f"; python -c "
import json,sys
for l in open('$f'): d=json.loads(l); print(round(d.get('median_us',0),1), round(d.get('gflops',0),1), d['graph'][:90])"; done
