# A/B: k_nnz_thread_pe default (1024 threads/SM) vs lean (AS_NT_LEAN=1: <= 42 regs, 3 x 512 threads/SM)
G5=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=3,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=3,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0); GMEM_ATOM_RED")
G3=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=3,stages=2); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED")
for v in 0 1; do
  AS_NT_LEAN=$v python tools/sweep.py --config c5s --reps 20 --graphs "${G5[@]}" | sed "s/^/{\"lean\": $v, \"r\": /; s/\$/}/" >> gpurun_out/ab_lean.jsonl 2>> gpurun_out/ab_lean.err
  AS_NT_LEAN=$v python tools/sweep.py --config c3s --reps 20 --graphs "${G3[@]}" | sed "s/^/{\"lean\": $v, \"r\": /; s/\$/}/" >> gpurun_out/ab_lean.jsonl 2>> gpurun_out/ab_lean.err
done
python -c "
import json
for l in open('gpurun_out/ab_lean.jsonl'):
    d=json.loads(l); r=d['r']; print(d['lean'], r['config'], round(r['median_us'],1), r['graph'][:100])"
