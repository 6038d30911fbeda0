# A/B of two in-tree builds: x gathers with L1::evict_last (ab/lib_xl1.so) vs default (developer tool)
G3=("COMPRESS; BMW_NNZ_BLOCK(4096); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED")
G4=("DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMW_NNZ_BLOCK(1024); BMT_NNZ_BLOCK(16); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED }")
G5=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0); GMEM_ATOM_RED")
G2=("DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=512,grid=4) }")
for lib in "" ab/lib_xl1.so "" ab/lib_xl1.so; do
  for c in c3s:G3 c4s:G4 c5s:G5 c2:G2; do
    cfg=${c%%:*}; eval "gs=(\"\${${c#*:}[@]}\")"
    AS_LIB_AB=$lib python tools/sweep.py --config $cfg --reps 20 --graphs "${gs[@]}" | sed "s|^|{\"lib\": \"${lib:-default}\", \"r\": |; s|\$|}|" >> gpurun_out/ab_xl1.jsonl 2>> gpurun_out/ab_xl1.err
  done
done
python -c "
import json
for l in open('gpurun_out/ab_xl1.jsonl'):
    d=json.loads(l); r=d['r']; print(d['lib'], r['config'], round(r['median_us'],1))"
