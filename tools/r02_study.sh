#!/bin/bash
# NEXT-3 study (surrogate MAD vs P:371's 5 %, iterations to the best vs row variance)
# and the N=2 bench path on one GPU (gloo control plane, peer-memory exchange, rank-local C5 bands)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
AS_BENCH_BACKEND=gloo AS_BENCH_C5_SCALE=24 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 --exchange peer --search-budget 20 \
  > gpurun_out/bench_w2.json 2> gpurun_out/bench_w2.err; echo "rc=$?" >> gpurun_out/bench_w2.err
tail -c 1500 gpurun_out/bench_w2.json
timeout 1500 python tools/search_study.py --budget 45 --seeds 2 > gpurun_out/search_study.jsonl 2> gpurun_out/search_study.err
cut -c1-400 gpurun_out/search_study.jsonl
G4='DENSE_DECOM(b=64,theta=0.5) { DENSE; SET_RESOURCE(tpb=256,grid=0,stages=2,xcache=0) | COMPRESS; BMW_NNZ_BLOCK(nnz=1024); BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=BMW,vec=2); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; SET_RESOURCE(tpb=512,grid=2,stages=2); GMEM_ATOM_RED }'
for lib in "" kb8d; do
  export AS_LIB_AB=${lib:+paper_2212_10432_b200/libalphasparse_$lib.so}
  timeout 600 python tools/sweep.py --config c4 --reps 20 --graphs "$G4" >> gpurun_out/ab_kb8d.jsonl 2>> gpurun_out/ab_kb8d.err
done
unset AS_LIB_AB
cut -c1-60,400-600 gpurun_out/ab_kb8d.jsonl
