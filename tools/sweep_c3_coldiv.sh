# C3 (rmat-24 fp32): COL_DIV stripes so that each stripe's x slice stays L2-resident (developer tool)
B="COMPRESS; BMT_NNZ_BLOCK(32); BMT_PAD(GLOBAL); THREAD_BITMAP_RED_G; SET_RESOURCE(tpb=256,grid=16,stages=2); GMEM_ATOM_RED"
C=${1:-c3}
N=$((1<<24)); [ "$C" = c3s ] && N=$((1<<22))
python tools/sweep.py --config $C --reps 20 --graphs "$B" \
  "COL_DIV(cuts=[$((N/2))]) { $B }" \
  "COL_DIV(cuts=[$((N/4)),$((N/2)),$((3*N/4))]) { $B }" \
  "COL_DIV(cuts=[$((N/8)),$((N/4)),$((3*N/8)),$((N/2)),$((5*N/8)),$((3*N/4)),$((7*N/8))]) { $B }"
