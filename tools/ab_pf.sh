# A/B: L2 bulk prefetch distance of k_nnz_thread_pe (AS_NT_PF = 0 / 1 / 2 CTA rounds ahead)
G5=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=4,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED")
G3=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED")
CFG5=${1:-c5s}; CFG3=${2:-c3s}
for pf in 0 1 2; do
  AS_NT_PF=$pf python tools/sweep.py --config $CFG5 --reps 20 --graphs "${G5[@]}" > gpurun_out/ab_pf_${CFG5}_$pf.jsonl 2>> gpurun_out/ab_pf.err
  AS_NT_PF=$pf python tools/sweep.py --config $CFG3 --reps 20 --graphs "${G3[@]}" > gpurun_out/ab_pf_${CFG3}_$pf.jsonl 2>> gpurun_out/ab_pf.err
done
for f in gpurun_out/ab_pf_*.jsonl; do echo "== $f"; python -c "
import json,sys
for l in open('$f'): d=json.loads(l); print(round(d.get('median_us',0),1), round(d.get('gflops',0),1), d['graph'][:100])"; done
