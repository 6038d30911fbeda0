# A/B: k_nnz_thread_pe with one batch of load look-ahead (AS_NT_PIPE=1, KB 4) vs without (developer tool)
G5=("COMPRESS; BMT_NNZ_BLOCK(64); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(64); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=4,stages=0); GMEM_ATOM_RED")
G3=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED")
for pp in 0 1; do
  AS_NT_PIPE=$pp python tools/sweep.py --config ${1:-c5s} --reps 20 --graphs "${G5[@]}" > gpurun_out/ab_pipe_c5_$pp.jsonl 2>> gpurun_out/ab_pipe.err
  AS_NT_PIPE=$pp python tools/sweep.py --config ${2:-c3s} --reps 20 --graphs "${G3[@]}" > gpurun_out/ab_pipe_c3_$pp.jsonl 2>> gpurun_out/ab_pipe.err
done
for f in gpurun_out/ab_pipe_*.jsonl; do echo "== $f"; python -c "
import json,sys
for l in open('$f'): d=json.loads(l); print(round(d.get('median_us',0),1), round(d.get('gflops',0),1), d['graph'][:100])"; done
