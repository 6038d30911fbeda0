# A/B: x gathers through L1 (ld.global.nc, default) vs L2 only (AS_X_CG=1) (developer tool)
G3=("COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=1024,grid=2); GMEM_ATOM_RED"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,0); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED")
G4=("DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(256) | COMPRESS; BMW_NNZ_BLOCK(1024); BMT_NNZ_BLOCK(32); BMT_PAD(BMW,2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED }")
G5=("COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0); GMEM_ATOM_RED")
for v in 0 1; do
  AS_X_CG=$v python tools/sweep.py --config c3s --reps 20 --graphs "${G3[@]}" | sed "s/^/{\"xcg\": $v, \"r\": /; s/\$/}/" >> gpurun_out/ab_xcg.jsonl 2>> gpurun_out/ab_xcg.err
  AS_X_CG=$v python tools/sweep.py --config c4s --reps 20 --graphs "${G4[@]}" | sed "s/^/{\"xcg\": $v, \"r\": /; s/\$/}/" >> gpurun_out/ab_xcg.jsonl 2>> gpurun_out/ab_xcg.err
  AS_X_CG=$v python tools/sweep.py --config c5s --reps 20 --graphs "${G5[@]}" | sed "s/^/{\"xcg\": $v, \"r\": /; s/\$/}/" >> gpurun_out/ab_xcg.jsonl 2>> gpurun_out/ab_xcg.err
done
python -c "
import json
for l in open('gpurun_out/ab_xcg.jsonl'):
    d=json.loads(l); r=d['r']; print(d['xcg'], r['config'], round(r['median_us'],1), r['graph'][:80])"
