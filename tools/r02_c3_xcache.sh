#!/bin/bash
# Round-2 C3 hot-x cache sweep (run under gpurun from the repo root)
W="COMPRESS; BMW_NNZ_BLOCK(nnz=4096); BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED"
T="COMPRESS; BMT_NNZ_BLOCK(nnz=32); BMT_PAD(scope=GLOBAL,vec=0); THREAD_BITMAP_RED_G"
python tools/sweep.py --config c3 --reps 20 --graphs \
  "$W; SET_RESOURCE(tpb=1024,grid=2,stages=2); GMEM_ATOM_RED" \
  "$W; SET_RESOURCE(tpb=1024,grid=1,stages=2,xcache=16384); GMEM_ATOM_RED" \
  "$W; SET_RESOURCE(tpb=1024,grid=1,stages=2,xcache=32768); GMEM_ATOM_RED" \
  "$W; SET_RESOURCE(tpb=1024,grid=1,stages=2,xcache=49152); GMEM_ATOM_RED" \
  "$W; SET_RESOURCE(tpb=512,grid=0,stages=2,xcache=24576); GMEM_ATOM_RED" \
  "$T; SET_RESOURCE(tpb=1024,grid=2,stages=2); GMEM_ATOM_RED" \
  "$T; SET_RESOURCE(tpb=1024,grid=1,stages=2,xcache=32768); GMEM_ATOM_RED" \
  "$T; SET_RESOURCE(tpb=512,grid=0,stages=2,xcache=24576); GMEM_ATOM_RED"
