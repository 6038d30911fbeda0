# HYB_DECOM graphs on the C5/C3 shapes (developer tool)
G5=("HYB_DECOM(w=16) { COMPRESS; BMTB_ROW_BLOCK(64); BMT_ROW_BLOCK(1); BMT_PAD(BMTB,2); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED }"
    "HYB_DECOM(w=12) { COMPRESS; BMTB_ROW_BLOCK(256); SORT_BMTB; BMW_ROW_BLOCK(32); BMT_ROW_BLOCK(1); BMT_PAD(BMW,2); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED }"
    "COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL,4); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=512,grid=2,stages=0); GMEM_ATOM_RED")
G3=("HYB_DECOM(w=16) { COMPRESS; BMTB_ROW_BLOCK(64); BMT_ROW_BLOCK(1); BMT_PAD(BMTB,4); THREAD_TOTAL_RED; GMEM_ATOM_RED | COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED }"
    "COMPRESS; BMW_NNZ_BLOCK(2048); BMT_NNZ_BLOCK(64); BMT_PAD(BMW,4); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2); GMEM_ATOM_RED")
python tools/sweep.py --config c5s --reps 20 --graphs "${G5[@]}" > gpurun_out/sweep_hyb_c5s.jsonl 2>> gpurun_out/sweep_hyb.err
python tools/sweep.py --config c3s --reps 20 --graphs "${G3[@]}" > gpurun_out/sweep_hyb_c3s.jsonl 2>> gpurun_out/sweep_hyb.err
for f in gpurun_out/sweep_hyb_*.jsonl; do echo "== $f"; python -c "
import json
for l in open('$f'): d=json.loads(l); print(round(d.get('median_us',0),1), round(d.get('gflops',0),1), d.get('kernels','')[:50], d['graph'][:90])"; done
