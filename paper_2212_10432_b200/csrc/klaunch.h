// Launch groups of the SpMV kernel family (kernels_impl.cuh), one translation unit per
// (group, value type): kernels_nt_f32.cu, kernels_nt_f64.cu, kernels_nw_f32.cu,
// kernels_nw_f64.cu, kernels_other.cu.  kernels.cu dispatches on the family and dtype.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "devpart.h"

namespace as {
template <class V>
int launch_grp_nnz_thread(const DevPart& p, const V* x, V* y, cudaStream_t s);
template <class V>
int launch_grp_nnz_warp(const DevPart& p, const V* x, V* y, cudaStream_t s);
template <class V>
int launch_grp_other(const DevPart& p, const V* x, V* y, cudaStream_t s);
template <class V>
int prep_grp_nnz_thread_xh(const DevPart& p, size_t smem, int tpb);
template <class V>
int prep_grp_nnz_warp_xh(const DevPart& p, size_t smem, int tpb);
template <class V>
int xw_occ_t(int pad, int vec, int tpb, size_t smem);
template <class V>
int prep_grp_block_offset(DevPart& p);
}  // namespace as
