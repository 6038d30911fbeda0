# ncu captures of the irregular-matrix kernels on a C5-shaped matrix (developer tool)
G1="COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; GMEM_ATOM_RED"
G2="COMPRESS; BMTB_ROW_BLOCK(256); SORT_BMTB; BMW_ROW_BLOCK(32); BMT_ROW_BLOCK(1); BMT_PAD(BMW); THREAD_TOTAL_RED; GMEM_ATOM_RED"
G3="COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED"
ncu --set full --clock-control none --import-source on -k regex:k_nnz_warp -s 2 -c 1 -o gpurun_out/prof_c5_nnzwarp python tools/run_graphs.py c5s "$G1" > gpurun_out/prof_c5a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_thread_row_pad -s 2 -c 1 -o gpurun_out/prof_c5_sell python tools/run_graphs.py c5s "$G2" > gpurun_out/prof_c5b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o gpurun_out/prof_c5_nnzthr python tools/run_graphs.py c5s "$G3" > gpurun_out/prof_c5c.log 2>&1
