// Dispatch of the composed-level kernel k_compose (compose_impl.cuh; Fig. 5)
// over the (value type, BMT_PAD) groups compiled in compose_{f32,f64}{,_pad}.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "devpart.h"

namespace as {
template <class V, bool PAD>
int compose_launch_grp(const DevPart& p, const V* x, V* y, cudaStream_t s, int64_t g, int tpb);
template <class V, bool PAD>
cudaError_t compose_optin_grp(size_t bytes);

int launch_compose(const DevPart& p, const void* x, void* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int tpb = p.tpb > 0 ? p.tpb : 256;
  const int64_t per = p.has_w ? tpb / 32 : tpb;
  const int64_t units = p.has_b ? p.n_bmtb : ((p.has_w ? p.n_bmw : p.n_bmt) + per - 1) / per;
  int64_t g = units > 0 ? units : 1;
  if (p.grid > 0) {  // SET_RESOURCE grid = k -> k * #SM persistent CTAs
    int dev = 0;
    cudaGetDevice(&dev);
    g = std::min<int64_t>(g, (int64_t)p.grid * device_sm_count(dev));
  }
  if (g > (int64_t(1) << 31) - 1) g = (int64_t(1) << 31) - 1;
  if (p.dtype == 1) {
    if (p.pad) compose_launch_grp<double, true>(p, (const double*)x, (double*)y, s, g, tpb);
    else compose_launch_grp<double, false>(p, (const double*)x, (double*)y, s, g, tpb);
  } else {
    if (p.pad) compose_launch_grp<float, true>(p, (const float*)x, (float*)y, s, g, tpb);
    else compose_launch_grp<float, false>(p, (const float*)x, (float*)y, s, g, tpb);
  }
  return (int)cudaGetLastError();
}

int prepare_compose(DevPart& p) {
  if (p.bred != RED_OFFSET) return 0;
  p.smem = (size_t)std::max<int64_t>(p.max_block_nnz, 1) * sizeof(double);
  if (p.smem <= 48 * 1024) return 0;
  cudaError_t e0 = p.dtype == 1 ? compose_optin_grp<double, false>(p.smem) : compose_optin_grp<float, false>(p.smem);
  cudaError_t e1 = p.dtype == 1 ? compose_optin_grp<double, true>(p.smem) : compose_optin_grp<float, true>(p.smem);
  return (int)(e0 != cudaSuccess ? e0 : e1);
}

}  // namespace as
