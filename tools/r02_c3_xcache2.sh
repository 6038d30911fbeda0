#!/bin/bash
# C3 xcache sweep after the batched fill; A/B of short-array fusion (AS_NO_FUSE)
B="COMPRESS; BMW_NNZ_BLOCK(nnz=8192); BMT_NNZ_BLOCK(nnz=64); BMT_PAD(scope=BMW,vec=0); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED"
python tools/sweep.py --config c3 --reps 20 --graphs \
  "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=16384); GMEM_ATOM_RED" \
  "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=24576); GMEM_ATOM_RED" \
  "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=32768); GMEM_ATOM_RED" \
  "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=40960); GMEM_ATOM_RED" \
  "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=49152); GMEM_ATOM_RED" \
  "$B; SET_RESOURCE(tpb=512,grid=2,stages=0,xcache=16384); GMEM_ATOM_RED" \
  "$B; SET_RESOURCE(tpb=768,grid=1,stages=0,xcache=32768); GMEM_ATOM_RED"
AS_NO_FUSE=1 python tools/sweep.py --config c3 --reps 20 --graphs "$B; SET_RESOURCE(tpb=1024,grid=1,stages=0,xcache=24576); GMEM_ATOM_RED"
