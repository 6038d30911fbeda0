// Dispatch of the sm_100a SpMV kernel family (kernels_impl.cuh) by family and value type,
// the writer rule's beta pre-pass and fp32 heavy-row epilogue (A22, A25), and the L2 flush
// used by timing.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "devpart.h"
#include "kcommon.cuh"
#include "klaunch.h"

namespace as {

namespace {

// =====================================================================================
// beta pre-pass of the writer rule (A22): y[r] = beta * y[r] (0 when beta == 0)
// =====================================================================================
template <class V>
__global__ void k_prepass(const int32_t* __restrict__ rows, int64_t n, double beta, V* __restrict__ y) {
  for (int64_t i = gtid(); i < n; i += gthreads()) {
    int64_t r = ldm(rows + i);
    y[r] = beta == 0.0 ? (V)0 : (V)(beta * (double)y[r]);
  }
}
// R-conc: a side-stream part's scratch rows added into y after the streams join
template <class V>
__global__ void k_side_add(const int32_t* __restrict__ rows, int64_t n, const V* __restrict__ ys, V* __restrict__ y) {
  for (int64_t i = gtid(); i < n; i += gthreads()) {
    const int64_t r = ldm(rows + i);
    y[r] = (V)((double)y[r] + (double)ys[r]);
  }
}
// heavy rows of fp32 plans: y[r] += (float)acc (one rounding of the fp64 sum)
__global__ void k_heavy_epilogue(const int32_t* __restrict__ rows, const double* __restrict__ acc, int64_t n,
                                 float* __restrict__ y) {
  for (int64_t i = gtid(); i < n; i += gthreads()) {
    const int64_t r = rows[i];
    y[r] = (float)((double)y[r] + acc[i]);
  }
}

template <class V>
int launch_typed(const DevPart& p, const V* x, V* y, cudaStream_t s) {
  if (p.fam == FAM_NNZ_THREAD) return launch_grp_nnz_thread<V>(p, x, y, s);
  if (p.fam == FAM_NNZ_WARP) return launch_grp_nnz_warp<V>(p, x, y, s);
  return launch_grp_other<V>(p, x, y, s);
}

}  // namespace


int launch_part(const DevPart& p, const void* x, void* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (p.fam == FAM_COMPOSE) return launch_compose(p, x, y, stream);
  if (p.dtype == 1) return launch_typed<double>(p, (const double*)x, (double*)y, s);
  return launch_typed<float>(p, (const float*)x, (float*)y, s);
}

int launch_prepass(const int32_t* rows, int64_t n, double beta, void* y, int dtype, void* stream) {
  if (n <= 0) return 0;
  int64_t g = std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (dtype == 1) k_prepass<double><<<g, 256, 0, (cudaStream_t)stream>>>(rows, n, beta, (double*)y);
  else k_prepass<float><<<g, 256, 0, (cudaStream_t)stream>>>(rows, n, beta, (float*)y);
  return (int)cudaGetLastError();
}

int launch_side_add(const int32_t* rows, int64_t n, const void* ys, void* y, int dtype, void* stream) {
  if (n <= 0) return 0;
  int64_t g = std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (dtype == 1) k_side_add<double><<<g, 256, 0, (cudaStream_t)stream>>>(rows, n, (const double*)ys, (double*)y);
  else k_side_add<float><<<g, 256, 0, (cudaStream_t)stream>>>(rows, n, (const float*)ys, (float*)y);
  return (int)cudaGetLastError();
}

int launch_heavy_epilogue(const int32_t* rows, const double* acc, int64_t n, void* y, void* stream) {
  if (n <= 0) return 0;
  int64_t g = std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_heavy_epilogue<<<g, 256, 0, (cudaStream_t)stream>>>(rows, acc, n, (float*)y);
  return (int)cudaGetLastError();
}

// L2 flush for timing (as_search): after a memset of the 2x-L2 buffer, read it back so the
// dirty lines are written back here, not inside the next timed SpMV.
__global__ void k_read_back(const uint4* __restrict__ p, int64_t n, unsigned* sink) {
  unsigned acc = 0;
  for (int64_t i = gtid(); i < n; i += gthreads()) {
    const uint4 v = __ldcg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u && sink) *sink = acc;  // keeps the loads; practically never taken
}
int launch_l2_flush(void* buf, size_t bytes, int pattern, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(buf, pattern, bytes, s);
  if (e != cudaSuccess) return (int)e;
  k_read_back<<<148 * 8, 512, 0, s>>>((const uint4*)buf, (int64_t)(bytes / 16), nullptr);
  return (int)cudaGetLastError();
}


template <class V>
static int xh_prep(const DevPart& p, size_t smem, int tpb) {
  return p.fam == FAM_NNZ_THREAD ? prep_grp_nnz_thread_xh<V>(p, smem, tpb) : prep_grp_nnz_warp_xh<V>(p, smem, tpb);
}

int prepare_part(DevPart& p) {
  if (p.fam == FAM_COMPOSE) return prepare_compose(p);
  if (p.xh_n > 0 && (p.fam == FAM_NNZ_THREAD || p.fam == FAM_NNZ_WARP)) {
    const int tpb = p.tpb > 0 ? p.tpb : 256;
    p.smem = (size_t)p.xh_n * (p.dtype == 1 ? 8 : 4);
    const int per = p.dtype == 1 ? xh_prep<double>(p, p.smem, tpb) : xh_prep<float>(p, p.smem, tpb);
    cudaGetLastError();
    if (per < 1) return (int)cudaErrorInvalidConfiguration;
    p.xh_ctas = p.grid > 0 ? std::min(p.grid, per) : per;
    return 0;
  }
  if (p.fam == FAM_BLOCK_OFFSET) {
    const size_t sv = p.dtype == 1 ? 8 : 4;
    if (p.variant == 1)  // TMA-staged CSR-stream: 2 stages of values, columns, row offsets
      p.smem = 2 * ((size_t)p.smem_cap * (sv + 4) + (size_t)p.smem_rcap * 4) + (size_t)p.smem_cap * 8 + 16;
    else
      p.smem = (size_t)p.max_block_nnz * sizeof(double);
    return p.dtype == 1 ? prep_grp_block_offset<double>(p) : prep_grp_block_offset<float>(p);
  }
  return 0;
}

int xw_ctas_per_sm(int dtype, int pad, int vec, int tpb, size_t smem) {
  int n = dtype == 1 ? xw_occ_t<double>(pad, vec, tpb, smem) : xw_occ_t<float>(pad, vec, tpb, smem);
  cudaGetLastError();
  return n;
}
int device_sm_count(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

int device_max_smem_optin(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return v;
}

const char* fam_kernel_name(const DevPart& p) {
  switch (p.fam) {
    case FAM_THREAD_ROW: return p.pad ? "k_thread_row_pad" : "k_thread_row";
    case FAM_NNZ_THREAD: return "k_nnz_thread";
    case FAM_NNZ_WARP: return (p.variant & 7) == 1 ? "k_nnz_warp<seg>" : "k_nnz_warp<bitmap>";
    case FAM_WARP_ROW: return "k_warp_row";
    case FAM_BLOCK_TOTAL: return "k_block_total";
    case FAM_BLOCK_OFFSET: return "k_block_offset";
    case FAM_DIA: return "k_dia";
    case FAM_DENSE: return "k_dense";
    case FAM_COMPOSE: return "k_compose";
    default: return "?";
  }
}

}  // namespace as
