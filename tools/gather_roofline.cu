// Gather roofline (developer measurement tool, not part of the product path).
//
// The irregular configs (C3 rmat-24, the C4 residual) are bound by the x gathers, not by
// HBM: each nonzero reads one 32-byte L2 sector of x for 4 (fp32) or 8 (fp64) useful bytes.
// These kernels measure the ceiling any SpMV over the same nonzeros must respect: stream
// every (val, col) pair once and gather x[col] for it, with no reduction by row and no y
// traffic.  Loads use the same cache policies as the product kernels (matrix streams
// L1::no_allocate + L2 evict_first; x gathers through L1 with L2 evict_last), so the time
// of k_gather on a matrix's own column array is the gather roofline of that matrix.
//
//   k_stream      : val + col only (no gather)            -> streaming floor
//   k_gather      : val + col + x[col]                    -> gather roofline
//   k_gather_hash : x[hash(i) % n], no col stream         -> random-sector L2 rate alone
//   k_gather_hot  : as k_gather, columns < 0 read a shared-memory copy of the hot x entries
//                   (~col), the rest x[col]               -> the hot-x cache's ceiling
//   mode 3        : columns relabeled by descending reference count (x permuted to match),
//                   col < K read the shared-memory prefix -> what a column relabeling buys
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t pol_ef() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_el() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_s4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ double2 ld_s2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ int4 ld_si4(const int32_t* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ int2 ld_si2(const int32_t* p) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ double ldx(const float* x, int64_t c) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  return (double)v;
}
__device__ __forceinline__ double ldx(const double* x, int64_t c) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pol_el()));
  return v;
}

// x-gather load variants (A/B of the L1 behaviour of the gathers): 0 = L1-allocating .nc with
// an L2 evict_last policy (the product's ldx), 1 = L1::no_allocate, 2 = .cg (L2 only),
// 3 = L1::evict_first, 4 = plain .nc without an L2 policy
template <int XLD>
__device__ __forceinline__ double ldxv_(const float* x, int64_t c) {
  float v;
  if (XLD == 0) asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  else if (XLD == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  else if (XLD == 2) asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  else if (XLD == 3)
    asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  else asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(x + c));
  return (double)v;
}
template <int XLD>
__device__ __forceinline__ double ldxv_(const double* x, int64_t c) {
  double v;
  if (XLD == 0) asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pol_el()));
  else if (XLD == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pol_el()));
  else if (XLD == 2) asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pol_el()));
  else if (XLD == 3)
    asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pol_el()));
  else asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(x + c));
  return v;
}

// 4 (fp32) / 2 (fp64) elements per vector, UNR vectors in flight per thread
template <class V>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int W = 4;
  static __device__ __forceinline__ void ld(const float* v, const int32_t* c, double* vo, int32_t* co) {
    float4 a = ld_s4(v);
    int4 b = ld_si4(c);
    vo[0] = a.x, vo[1] = a.y, vo[2] = a.z, vo[3] = a.w;
    co[0] = b.x, co[1] = b.y, co[2] = b.z, co[3] = b.w;
  }
};
template <>
struct Vec<double> {
  static constexpr int W = 2;
  static __device__ __forceinline__ void ld(const double* v, const int32_t* c, double* vo, int32_t* co) {
    double2 a = ld_s2(v);
    int2 b = ld_si2(c);
    vo[0] = a.x, vo[1] = a.y;
    co[0] = b.x, co[1] = b.y;
  }
};


constexpr int UNR = 4;  // vectors in flight per thread (other kernels)

template <class V, int MODE, int XLD = 0, int UNR = 4>  // MODE 0 stream, 1 gather, 2 gather with hot smem (~slot), 3 hot = col < nh (relabeled)
__global__ void __launch_bounds__(1024) k_gather(const V* __restrict__ val, const int32_t* __restrict__ col,
                                                 const V* __restrict__ x, const V* __restrict__ xh, int nh,
                                                 int64_t nnz, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  V* sh = (V*)smem;
  if (MODE >= 2) {
    for (int i = threadIdx.x; i < nh; i += blockDim.x) sh[i] = xh[i];
    __syncthreads();
  }
  constexpr int W = Vec<V>::W;
  const int64_t nv = nnz / W;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (UNR - 1) * T < nv; i += UNR * T) {
    double v[UNR * W];
    int32_t c[UNR * W];
#pragma unroll
    for (int u = 0; u < UNR; ++u) Vec<V>::ld(val + (i + u * T) * W, col + (i + u * T) * W, v + u * W, c + u * W);
    double xv[UNR * W];
#pragma unroll
    for (int q = 0; q < UNR * W; ++q) {
      if (MODE == 0) xv[q] = (double)c[q];
      else if (MODE == 1) xv[q] = ldxv_<XLD>(x, c[q]);
      else if (MODE == 2) xv[q] = c[q] < 0 ? (double)sh[~c[q]] : ldxv_<XLD>(x, c[q]);
      else xv[q] = c[q] < nh ? (double)sh[c[q]] : ldxv_<XLD>(x, c[q]);
    }
#pragma unroll
    for (int q = 0; q < UNR * W; ++q) acc += v[q] * xv[q];
  }
  for (; i < nv; i += T) {
    double v[W];
    int32_t c[W];
    Vec<V>::ld(val + i * W, col + i * W, v, c);
#pragma unroll
    for (int q = 0; q < W; ++q) {
      double xv = MODE == 0   ? (double)c[q]
                  : MODE == 1 ? ldxv_<XLD>(x, c[q])
                  : MODE == 2 ? (c[q] < 0 ? (double)sh[~c[q]] : ldxv_<XLD>(x, c[q]))
                              : (c[q] < nh ? (double)sh[c[q]] : ldxv_<XLD>(x, c[q]));
      acc += v[q] * xv;
    }
  }
  if (acc == 1234.5678) out[0] = acc;  // keeps the loads live; practically never stores
}

// mode 5: x gathers issued as cp.async (LDGSTS) into a per-thread shared-memory staging
// ring (no registers held while in flight), CH elements per chunk, 2 chunks in flight, the
// first nh columns (relabeled / encoded hot set) read from a shared-memory copy.  Measures
// whether register-free gathers raise the sustainable gather rate.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <class V>
__device__ __forceinline__ void cp_async_x(V* dst, const V* src) {
  if constexpr (sizeof(V) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <class V, int CH>
__global__ void __launch_bounds__(1024) k_gather_async(const V* __restrict__ val, const int32_t* __restrict__ col,
                                                        const V* __restrict__ x, const V* __restrict__ xh, int nh,
                                                        int64_t nnz, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  V* sh = (V*)smem;
  for (int i = threadIdx.x; i < nh; i += blockDim.x) sh[i] = xh[i];
  V* ring = sh + ((nh + 3) & ~3) + threadIdx.x * (2 * CH + 1);
  __syncthreads();
  constexpr int W = Vec<V>::W;
  static_assert(CH % W == 0, "chunk = whole vectors");
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t nch = nnz / ((int64_t)CH * T);  // full chunk rounds (tail ignored: microbench)
  double acc = 0.0;
  V vprev[CH];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto chunk_base = [&](int64_t r) { return (r * T + tid) * CH; };
  auto issue = [&](int64_t r, int buf, V* vv) {
    const int64_t b = chunk_base(r);
#pragma unroll
    for (int q = 0; q < CH; q += W) {
      double v[W];
      int32_t c[W];
      Vec<V>::ld(val + b + q, col + b + q, v, c);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        vv[q + w] = (V)v[w];
        V* d = ring + buf * CH + q + w;
        if (c[w] < nh) *d = sh[c[w]];
        else cp_async_x(d, x + c[w]);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (nch > 0) issue(0, 0, vprev);
  for (int64_t r = 0; r < nch; ++r) {
    V vcur[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) vcur[q] = vprev[q];
    if (r + 1 < nch) {
      issue(r + 1, (int)((r + 1) & 1), vprev);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    const V* xs = ring + (r & 1) * CH;
#pragma unroll
    for (int q = 0; q < CH; ++q) acc += (double)vcur[q] * (double)xs[q];
  }
  if (acc == 1234.5678) out[0] = acc;
}

// mode 6: the hot-x copy distributed over a thread-block cluster of C CTAs (DSMEM): CTA r of
// the cluster holds hot slots [r*Kl, (r+1)*Kl); a gather of hot slot s reads CTA s/Kl's
// shared memory through mapa + ld.shared::cluster.  C times the hot set of one CTA at the same
// shared-memory (and L1) footprint per SM.
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class V>
__device__ __forceinline__ double ld_dsm(const V* local_base, int64_t s, int kl) {
  const unsigned owner = (unsigned)(s / kl), off = (unsigned)(s - (int64_t)owner * kl);
  const unsigned a = smem_u32(local_base + off);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(owner));
  if constexpr (sizeof(V) == 4) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra));
    return (double)v;
  } else {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
    return v;
  }
}
template <class V>
__global__ void __launch_bounds__(1024) k_gather_dsm(const V* __restrict__ val, const int32_t* __restrict__ col,
                                                      const V* __restrict__ x, const V* __restrict__ xh, int kl,
                                                      int64_t nnz, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  V* sh = (V*)smem;
  const unsigned rk = cluster_rank();
  for (int i = threadIdx.x; i < kl; i += blockDim.x) sh[i] = xh[(int64_t)rk * kl + i];
  cluster_sync();
  constexpr int W = Vec<V>::W;
  const int64_t nv = nnz / W;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (UNR - 1) * T < nv; i += UNR * T) {
    double v[UNR * W];
    int32_t c[UNR * W];
#pragma unroll
    for (int u = 0; u < UNR; ++u) Vec<V>::ld(val + (i + u * T) * W, col + (i + u * T) * W, v + u * W, c + u * W);
    double xv[UNR * W];
#pragma unroll
    for (int q = 0; q < UNR * W; ++q) xv[q] = c[q] < 0 ? ld_dsm(sh, ~c[q], kl) : ldx(x, c[q]);
#pragma unroll
    for (int q = 0; q < UNR * W; ++q) acc += v[q] * xv[q];
  }
  cluster_sync();  // no CTA leaves while a partner may still read its shared memory
  if (acc == 1234.5678) out[0] = acc;
}

__device__ __forceinline__ uint32_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return (uint32_t)(z ^ (z >> 31));
}
template <class V>
__global__ void __launch_bounds__(1024) k_gather_hash(const V* __restrict__ x, int64_t n, int64_t count, double* out) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * T < count; i += 8 * T) {
    double xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = ldx(x, (int64_t)(mix(i + u * T) % (uint64_t)n));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += xv[u];
  }
  for (; i < count; i += T) acc += ldx(x, (int64_t)(mix(i) % (uint64_t)n));
  if (acc == 1234.5678) out[0] = acc;
}

}  // namespace

extern "C" {
// dtype 0 = fp32, 1 = fp64; mode 0 stream, 1 gather, 2 hot smem; returns cudaError_t
int gr_launch(int dtype, int mode, const void* val, const int32_t* col, const void* x, const void* xh, int nh,
              int64_t nnz, double* out, int grid, int tpb, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  size_t sm = mode >= 2 ? (size_t)nh * (dtype ? 8 : 4) : 0;
#define L(V, M)                                                                                           \
  do {                                                                                                    \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_gather<V, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)sm);                                                    \
    k_gather<V, M><<<grid, tpb, sm, s>>>((const V*)val, col, (const V*)x, (const V*)xh, nh, nnz, out);    \
  } while (0)
  if (dtype == 0) {
    if (mode == 0) L(float, 0);
    else if (mode == 1) L(float, 1);
    else if (mode == 2) L(float, 2);
    else L(float, 3);
  } else {
    if (mode == 0) L(double, 0);
    else if (mode == 1) L(double, 1);
    else if (mode == 2) L(double, 2);
    else L(double, 3);
  }
#undef L
  return (int)cudaGetLastError();
}
// mode 1 / 2 with the x-gather load variant xld (0..4, see ldxv_)
int gr_launch_x(int dtype, int mode, int xld, const void* val, const int32_t* col, const void* x, const void* xh,
                int nh, int64_t nnz, double* out, int grid, int tpb, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  size_t sm = mode >= 2 ? (size_t)nh * (dtype ? 8 : 4) : 0;
#define LX(V, M, X)                                                                                          \
  do {                                                                                                       \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_gather<V, M, X>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)sm);                                                       \
    k_gather<V, M, X><<<grid, tpb, sm, s>>>((const V*)val, col, (const V*)x, (const V*)xh, nh, nnz, out);    \
  } while (0)
#define LXM(V, X)            \
  do {                       \
    if (mode == 1) LX(V, 1, X); \
    else LX(V, 2, X);        \
  } while (0)
#define LXV(V)                  \
  do {                          \
    if (xld == 0) LXM(V, 0);    \
    else if (xld == 1) LXM(V, 1); \
    else if (xld == 2) LXM(V, 2); \
    else if (xld == 3) LXM(V, 3); \
    else LXM(V, 4);             \
  } while (0)
  if (dtype == 0) LXV(float);
  else LXV(double);
#undef LXV
#undef LXM
#undef LX
  return (int)cudaGetLastError();
}
// hot-x gathers (mode 2, .cg) with UNR vectors in flight per thread (1, 2, 4, 8): how the
// gather rate depends on the loads a thread keeps in flight
int gr_launch_unr(int dtype, int unr, const void* val, const int32_t* col, const void* x, const void* xh, int nh,
                  int64_t nnz, double* out, int grid, int tpb, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  size_t sm = (size_t)nh * (dtype ? 8 : 4);
#define LU(V, U)                                                                                                \
  do {                                                                                                          \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_gather<V, 2, 2, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)sm);                                                          \
    k_gather<V, 2, 2, U><<<grid, tpb, sm, s>>>((const V*)val, col, (const V*)x, (const V*)xh, nh, nnz, out);    \
  } while (0)
  if (dtype == 0) {
    if (unr == 1) LU(float, 1);
    else if (unr == 2) LU(float, 2);
    else if (unr == 8) LU(float, 8);
    else LU(float, 4);
  } else {
    if (unr == 1) LU(double, 1);
    else if (unr == 2) LU(double, 2);
    else if (unr == 8) LU(double, 8);
    else LU(double, 4);
  }
#undef LU
  return (int)cudaGetLastError();
}
// cp.async-staged gathers (mode 5): ch = chunk elements (8 or 16), nh hot columns in smem
int gr_launch_async(int dtype, int ch, const void* val, const int32_t* col, const void* x, const void* xh, int nh,
                    int64_t nnz, double* out, int grid, int tpb, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sv = dtype ? 8 : 4;
  size_t sm = ((size_t)((nh + 3) & ~3) + (size_t)tpb * (2 * ch + 1)) * sv;
#define LA(V, C)                                                                                                    \
  do {                                                                                                              \
    cudaFuncSetAttribute(k_gather_async<V, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);               \
    k_gather_async<V, C><<<grid, tpb, sm, s>>>((const V*)val, col, (const V*)x, (const V*)xh, nh, nnz, out);         \
  } while (0)
  if (dtype == 0) {
    if (ch == 8) LA(float, 8);
    else LA(float, 16);
  } else {
    if (ch == 8) LA(double, 8);
    else LA(double, 16);
  }
#undef LA
  return (int)cudaGetLastError();
}
// cluster-distributed hot-x gathers (mode 6): csize CTAs per cluster, kl hot entries per CTA
int gr_launch_dsm(int dtype, int csize, const void* val, const int32_t* col, const void* x, const void* xh, int kl,
                  int64_t nnz, double* out, int grid, int tpb, void* stream) {
  const size_t sm = (size_t)kl * (dtype ? 8 : 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)tpb);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (dtype == 0) {
    cudaFuncSetAttribute(k_gather_dsm<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (csize > 8) cudaFuncSetAttribute(k_gather_dsm<float>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    e = cudaLaunchKernelEx(&cfg, k_gather_dsm<float>, (const float*)val, col, (const float*)x, (const float*)xh, kl, nnz,
                           out);
  } else {
    cudaFuncSetAttribute(k_gather_dsm<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (csize > 8) cudaFuncSetAttribute(k_gather_dsm<double>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    e = cudaLaunchKernelEx(&cfg, k_gather_dsm<double>, (const double*)val, col, (const double*)x, (const double*)xh,
                           kl, nnz, out);
  }
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}
int gr_launch_hash(int dtype, const void* x, int64_t n, int64_t count, double* out, int grid, int tpb, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == 0) k_gather_hash<float><<<grid, tpb, 0, s>>>((const float*)x, n, count, out);
  else k_gather_hash<double><<<grid, tpb, 0, s>>>((const double*)x, n, count, out);
  return (int)cudaGetLastError();
}
}
