# Round-1 winners at full size: launch lists + one ncu --set full capture of each dominant kernel
G3="COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
G4="DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(tpb=256,grid=0,stages=2) | COMPRESS; BMTB_ROW_BLOCK(rows=32); BMT_ROW_BLOCK(rows=1); BMT_PAD(scope=BMTB,vec=0); THREAD_TOTAL_RED; SET_RESOURCE(tpb=64,grid=0,stages=2); GMEM_ATOM_RED }"
G5="COMPRESS; BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=GLOBAL,vec=4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/run_graphs.py c3 "$G3" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o gpurun_out/prof2_c3 python tools/run_graphs.py c3 "$G3" > gpurun_out/prof2_c3.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/run_graphs.py c4 "$G4" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_thread_row_pad -s 2 -c 1 -o gpurun_out/prof2_c4 python tools/run_graphs.py c4 "$G4" > gpurun_out/prof2_c4.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/run_graphs.py c5 "$G5" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nnz_thread -s 2 -c 1 -o gpurun_out/prof2_c5 python tools/run_graphs.py c5 "$G5" > gpurun_out/prof2_c5.log 2>&1
