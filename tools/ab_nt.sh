# nnz_thread kernel variants (AS_NT_EXP) on the irregular configs (developer tool)
G5=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=3,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED")
G3=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED")
for e in 0 1 2 3; do
  AS_NT_EXP=$e python tools/sweep.py --config c5s --graphs "${G5[@]}" > gpurun_out/nt_c5s_$e.jsonl 2>> gpurun_out/nt.err
  AS_NT_EXP=$e python tools/sweep.py --config c3s --graphs "${G3[@]}" > gpurun_out/nt_c3s_$e.jsonl 2>> gpurun_out/nt.err
done
