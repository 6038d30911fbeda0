# A/B: k_nnz_warp branching vs predicated-emit form (CSR5-like warp tiles) on c5s / c3s (developer tool)
G5=("COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED"
    "COMPRESS; BMW_NNZ_BLOCK(4096); BMT_NNZ_BLOCK(32); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED"
    "COMPRESS; BMW_NNZ_BLOCK(8192); BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; WARP_BITMAP_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED"
    "COMPRESS; BMW_NNZ_BLOCK(1024); BMT_NNZ_BLOCK(32); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=256,grid=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(64); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED")
G3=("COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED"
    "COMPRESS; BMW_NNZ_BLOCK(1024); BMT_NNZ_BLOCK(32); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=256,grid=16); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED")
for leg in 1 ""; do
  tag=${leg:+legacy}; tag=${tag:-pe}
  env ${leg:+AS_NT_LEGACY=1} python tools/sweep.py --config c5s --reps 20 --graphs "${G5[@]}" > gpurun_out/ab_warp_c5s_$tag.jsonl 2>> gpurun_out/ab_warp.err
  env ${leg:+AS_NT_LEGACY=1} python tools/sweep.py --config c3s --reps 20 --graphs "${G3[@]}" > gpurun_out/ab_warp_c3s_$tag.jsonl 2>> gpurun_out/ab_warp.err
done
for f in gpurun_out/ab_warp_*.jsonl; do echo "== $f"; python -c "
import json,sys
for l in open('$f'): d=json.loads(l); print(round(d.get('median_us',0),1), round(d.get('gflops',0),1), d.get('kernels','')[:40], d['graph'][:110])"; done
