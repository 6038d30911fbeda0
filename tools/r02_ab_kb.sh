#!/bin/bash
# A/B of the nnz-kernel load scheduling: non-volatile loads (main), volatile (vol), fp32
# warp batches of 8 / 16 (kb8, kb16); C3 winner family with xcache, C5 and C4 winners.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="COMPRESS; BMW_NNZ_BLOCK(nnz=8192); BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED"
for lib in "" vol kb8 kb16; do
  export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
  timeout 900 python tools/sweep.py --config c3 --reps 20 --graphs \
    "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=16384); GMEM_ATOM_RED" \
    "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=24576); GMEM_ATOM_RED" \
    "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=32768); GMEM_ATOM_RED" \
    "$B; SET_RESOURCE(tpb=1024,grid=2,stages=0); GMEM_ATOM_RED" >> gpurun_out/ab_kb.jsonl 2>> gpurun_out/ab_kb.err
done
for lib in "" vol; do
  export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
  timeout 900 python tools/sweep.py --config c5 --reps 10 --graphs \
    "COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=2); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=0); GMEM_ATOM_RED" >> gpurun_out/ab_kb.jsonl 2>> gpurun_out/ab_kb.err
done
export AS_LIB_AB=paper_2212_10432_b200/libalphasparse_kb8.so
timeout 600 python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider -k "nnz or xcache or warp" > gpurun_out/ab_kb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_kb_tests.log
unset AS_LIB_AB
tail -2 gpurun_out/ab_kb_tests.log; cut -c1-100,300-520 gpurun_out/ab_kb.jsonl
