# ncu captures of k_nnz_thread on the C3/C5-shaped matrices (developer tool)
G3="COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o gpurun_out/prof_nt_c3s python tools/run_graphs.py c3s "$G3" > gpurun_out/prof_nt_c3s.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o gpurun_out/prof_nt_c5s python tools/run_graphs.py c5s "$G3" > gpurun_out/prof_nt_c5s.log 2>&1
