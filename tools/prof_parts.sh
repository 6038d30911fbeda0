# per-kernel device times (ncu launch list) of the current best graphs on scaled configs
for spec in \
 "c4s|DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMTB_ROW_BLOCK(64); BMT_ROW_BLOCK(1); BMT_PAD(BMTB); THREAD_TOTAL_RED; SET_RESOURCE(128); GMEM_ATOM_RED }" \
 "c5s|COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED" \
 "c3s|COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16); GMEM_ATOM_RED"; do
  cfg="${spec%%|*}"; g="${spec#*|}"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/parts_$cfg.csv python tools/run_graphs.py $cfg "$g" > /dev/null 2>&1
done
