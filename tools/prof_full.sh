# ncu --set full of the dominant kernel of each full-size winner (C3, C4, C5), one launch each
G3="COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
G4="DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(tpb=256,grid=0,stages=2) | COMPRESS; BMTB_ROW_BLOCK(rows=64); BMT_ROW_BLOCK(rows=1); BMT_PAD(scope=BMTB,vec=0); THREAD_TOTAL_RED; SET_RESOURCE(tpb=128,grid=0,stages=2); GMEM_ATOM_RED }"
G5="COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED"
ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o gpurun_out/prof_c3_full python tools/run_graphs.py c3 "$G3" > gpurun_out/prof_c3.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/parts_c4.csv python tools/run_graphs.py c4 "$G4" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_thread_row_pad -s 2 -c 1 -o gpurun_out/prof_c4_sell python tools/run_graphs.py c4 "$G4" > gpurun_out/prof_c4a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dense -s 2 -c 1 -o gpurun_out/prof_c4_dense python tools/run_graphs.py c4 "$G4" > gpurun_out/prof_c4b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o gpurun_out/prof_c5_full python tools/run_graphs.py c5 "$G5" > gpurun_out/prof_c5.log 2>&1
