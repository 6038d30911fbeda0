#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_devbuild.py -q -p no:cacheprovider -k "large_matrix or history or fuzz or batch" > gpurun_out/t_new.log 2>&1; echo "rc=$?" >> gpurun_out/t_new.log
tail -5 gpurun_out/t_new.log
# NVTX ranges: profile only kernels inside as_spmv (ncu --nvtx-include)
C1G="COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; GMEM_ATOM_RED"
timeout 300 ncu --nvtx --nvtx-include "as_spmv/" --metrics gpu__time_duration.sum --csv --log-file gpurun_out/nvtx_as_spmv.csv \
  python tools/sweep.py --config c1 --reps 3 --graphs "$C1G" > gpurun_out/nvtx.log 2>&1
grep -c "k_nnz_thread\|k_prepass" gpurun_out/nvtx_as_spmv.csv; grep -o '"[a-z_:<>A-Za-z0-9, ]*k_[a-z_]*[^"]*"' gpurun_out/nvtx_as_spmv.csv | sort | uniq -c | head
