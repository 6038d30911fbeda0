# A/B of two in-tree builds (AS_LIB_AB=ab/lib_old.so vs default) on the irregular configs (developer tool)
G5=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED")
G3=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(16); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=0,stages=0); GMEM_ATOM_RED")
for lib in ab/lib_old.so ""; do
  tag=${lib:+old}; tag=${tag:-new}
  AS_LIB_AB=$lib python tools/sweep.py --config c5s --graphs "${G5[@]}" > gpurun_out/ab_c5s_$tag.jsonl 2>> gpurun_out/ab.err
  AS_LIB_AB=$lib python tools/sweep.py --config c3s --graphs "${G3[@]}" > gpurun_out/ab_c3s_$tag.jsonl 2>> gpurun_out/ab.err
  AS_LIB_AB=$lib python tools/sweep.py --config c5s --graphs "${G5[0]}" --beta 1.0 >> gpurun_out/ab_c5s_$tag.jsonl 2>> gpurun_out/ab.err
done
