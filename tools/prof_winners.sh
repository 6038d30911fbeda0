# Final round-1 winners at full size: launch lists + one ncu --set full capture of each dominant kernel
G3="COMPRESS; BMW_NNZ_BLOCK(nnz=2048); BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2,stages=2); GMEM_ATOM_RED"
G4="DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(tpb=256,grid=0,stages=2) | COMPRESS; BMW_NNZ_BLOCK(nnz=1024); BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=BMW,vec=2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2,stages=2); GMEM_ATOM_RED }"
G5="COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0); GMEM_ATOM_RED"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 3 4 5; do
  eval G=\$G$c
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches3_c$c.csv python tools/run_graphs.py c$c "$G" > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_nnz -s 2 -c 1 -o gpurun_out/prof3_c$c python tools/run_graphs.py c$c "$G" > gpurun_out/prof3_c$c.log 2>&1
done
# export the summaries on the box and drop the large reports (gpurun_out is capped at 64 MiB)
for c in 3 4 5; do
  ncu -i gpurun_out/prof3_c$c.ncu-rep --page raw --csv > gpurun_out/prof3_c$c.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof3_c$c.ncu-rep --page details --csv > gpurun_out/prof3_c$c.details.csv 2>/dev/null
done
rm -f gpurun_out/prof3_c*.ncu-rep
