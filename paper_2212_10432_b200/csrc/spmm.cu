// SpMM on an Operator-Graph plan (NEXT-4): Y = alpha * A * X + beta * Y with k right-hand
// sides (X: n x k, Y: m x k, row-major with leading dimensions ldx, ldy).  The plan's parts
// run in the same writer-rule order as the SpMV (reading A22): the beta pre-pass, then
// every part STOREs (first writer) or ADDs its partial rows.
//
// * DENSE parts (DENSE_DECOM tiles): with k right-hand sides each b x b tile times the
//   b x k panel of X is a real contraction, so it runs on the tensor cores -- fp64 DMMA
//   (mma.sync.aligned.m8n8k4.row.col.f64; tcgen05 has no fp64 kind and TF32 would break the
//   1e-5 fp32 tolerance, so fp32 tiles are widened exactly to fp64 in shared memory).
// * DIA parts: one thread per (row, column), diagonals streamed, x rows read coalesced.
// * every CSR-family part: a row-parallel CSR SpMM over the part's COMPRESS arrays (uploaded
//   with AS_PLAN_SPMM): a group of g = pow2 >= min(k, 32) lanes per row, lane c owning
//   columns c, c+g, ...; each nonzero's X row is read coalesced.  Rows are summed in fp64
//   by one group (no split rows), so no atomics and no fp32 heavy-row scratch are needed.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "devpart.h"
#include "optin.h"

namespace as {
namespace {

__device__ __forceinline__ int64_t gtid_s() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gthreads_s() { return (int64_t)gridDim.x * blockDim.x; }

template <class V>
__device__ __forceinline__ void put(V* y, double s, double alpha, double beta, bool add) {
  double v = alpha * s;
  if (add) v += (double)*y;
  else if (beta != 0.0) v += beta * (double)*y;
  *y = (V)v;
}

template <class V>
__global__ void k_spmm_prepass(const int32_t* __restrict__ rows, int64_t n, double beta, V* __restrict__ Y,
                               int64_t ldy, int64_t k) {
  for (int64_t i = gtid_s(); i < n * k; i += gthreads_s()) {
    V* p = Y + (int64_t)__ldg(rows + i / k) * ldy + i % k;
    *p = beta == 0.0 ? (V)0 : (V)(beta * (double)*p);
  }
}

template <class V>
__global__ void k_spmm_scale(int64_t m, double beta, V* __restrict__ Y, int64_t ldy, int64_t k) {
  for (int64_t i = gtid_s(); i < m * k; i += gthreads_s()) {
    V* p = Y + (i / k) * ldy + i % k;
    *p = beta == 0.0 ? (V)0 : (V)(beta * (double)*p);
  }
}

// CSR part: G lanes per row (G = power of two <= 32)
template <class V, int G>
__global__ void __launch_bounds__(256) k_spmm_csr(SpmmPart s, double alpha, double beta, const V* __restrict__ X,
                                                  int64_t ldx, V* __restrict__ Y, int64_t ldy, int64_t k) {
  const int64_t grp = gtid_s() / G, ngrp = gthreads_s() / G;
  const int lane = threadIdx.x % G;
  const V* val = (const V*)s.val;
  for (int64_t i = grp; i < s.m_p; i += ngrp) {
    const int64_t a = __ldg(s.rp + i), e = __ldg(s.rp + i + 1);
    const int64_t r = __ldg(s.rows + i);
    const bool add = s.add[i] != 0;
    for (int64_t c0 = 0; c0 < k; c0 += 4 * G) {  // 4 columns per lane in flight
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int64_t j = a;
      // 4 nonzeros per step: their column indices / values first, then 4 x 4 X loads in
      // flight (the X rows are scattered, so the gathers' latency is what bounds this loop)
      for (; j + 4 <= e; j += 4) {
        double v[4];
        const V* xr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = (double)__ldg(val + j + u);
          xr[u] = X + (int64_t)__ldg(s.col + j + u) * ldx;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t c = c0 + lane + q * G;
          if (c < k) {
            double xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u] = (double)__ldg(xr[u] + c);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[q] += v[u] * xv[u];
          }
        }
      }
      for (; j < e; ++j) {
        const double v = (double)__ldg(val + j);
        const V* xr = X + (int64_t)__ldg(s.col + j) * ldx;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t c = c0 + lane + q * G;
          if (c < k) acc[q] += v * (double)__ldg(xr + c);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t c = c0 + lane + q * G;
        if (c < k) put(Y + r * ldy + c, acc[q], alpha, beta, add);
      }
    }
  }
}

// CSR part, fp64 with 16-byte aligned X / Y rows and even k: lane pairs of columns read as
// one double2 (half the load instructions of k_spmm_csr), G lanes per row cover 2G columns
// per pass, 4 nonzeros in flight
template <int G>
__global__ void __launch_bounds__(256) k_spmm_csr2(SpmmPart s, double alpha, double beta, const double* __restrict__ X,
                                                   int64_t ldx, double* __restrict__ Y, int64_t ldy, int64_t k) {
  const int64_t grp = gtid_s() / G, ngrp = gthreads_s() / G;
  const int lane = threadIdx.x % G;
  const double* val = (const double*)s.val;
  for (int64_t i = grp; i < s.m_p; i += ngrp) {
    const int64_t a = __ldg(s.rp + i), e = __ldg(s.rp + i + 1);
    const int64_t r = __ldg(s.rows + i);
    const bool add = s.add[i] != 0;
    for (int64_t c0 = 2 * lane; c0 < k; c0 += 2 * G) {
      double2 acc = make_double2(0.0, 0.0);
      int64_t j = a;
      for (; j + 4 <= e; j += 4) {
        double v[4];
        double2 xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = __ldg(val + j + u);
          xv[u] = __ldg((const double2*)(X + (int64_t)__ldg(s.col + j + u) * ldx + c0));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc.x += v[u] * xv[u].x;
          acc.y += v[u] * xv[u].y;
        }
      }
      for (; j < e; ++j) {
        const double v = __ldg(val + j);
        const double2 xv = __ldg((const double2*)(X + (int64_t)__ldg(s.col + j) * ldx + c0));
        acc.x += v * xv.x;
        acc.y += v * xv.y;
      }
      put(Y + r * ldy + c0, acc.x, alpha, beta, add);
      put(Y + r * ldy + c0 + 1, acc.y, alpha, beta, add);
    }
  }
}

// DIA part: one thread per (row, column)
template <class V>
__global__ void k_spmm_dia(DevPart p, double alpha, double beta, const V* __restrict__ X, int64_t ldx,
                           V* __restrict__ Y, int64_t ldy, int64_t k) {
  const V* dv = (const V*)p.dia_val;
  for (int64_t t = gtid_s(); t < p.mb * k; t += gthreads_s()) {
    const int64_t i = t / k, c = t % k, r = p.r0 + i;
    double acc = 0.0;
    for (int d = 0; d < p.D; ++d) {
      const int64_t col = r + p.dia_off[d];
      if (col >= 0 && col < p.n) acc += (double)__ldg(dv + d * p.dia_stride + i) * (double)__ldg(X + col * ldx + c);
    }
    put(Y + r * ldy + c, acc, alpha, beta, p.mode != 0);
  }
}

// DENSE part on the tensor cores: one CTA (8 warps) per tile row; per tile, the b x b tile
// (column-major in HBM) and the b x 64 panel of X are staged in shared memory as fp64, and
// warp w computes a 16-row x 32-column block of Y with m8n8k4 DMMA (2 x 4 accumulator
// blocks), for b <= 64 (tile rows/cols beyond b are zero-filled).  Columns are processed in
// chunks of 64.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}
constexpr int kTB = 64;
constexpr int kLd = kTB + 8;  // padded row stride: the 4 k-rows a DMMA fragment reads hit 2 bank halves
constexpr size_t kDenseSmem = 2 * (size_t)kTB * kLd * sizeof(double);
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
template <class V>
__global__ void __launch_bounds__(256) k_spmm_dense_dmma(DevPart p, double alpha, double beta, const V* __restrict__ X,
                                                         int64_t ldx, V* __restrict__ Y, int64_t ldy, int64_t k) {
  extern __shared__ double smem_d[];
  double* sT = smem_d;                // tile, column-major: (i, j) at j*kLd + i
  double* sX = smem_d + kTB * kLd;    // panel: (j, c) at j*kLd + c
  const int b = (int)p.b;
  const V* tv = (const V*)p.tile_val;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  const bool async16 = sizeof(V) == 8 && b == kTB && !(((uintptr_t)X | (uintptr_t)(ldx * 8)) & 15);
  for (int64_t tr = blockIdx.x; tr < p.n_tile_rows; tr += gridDim.x) {
    const int64_t I = __ldg(p.tile_row_id + tr);
    const int64_t t0 = __ldg(p.tile_row_ptr + tr), t1 = __ldg(p.tile_row_ptr + tr + 1);
    for (int64_t c0 = 0; c0 < k; c0 += kTB) {
      // warp w: rows [16*rp, 16*rp + 16) (two 8-row fragments) x columns [32*ch, 32*ch + 32)
      // (four 8-column blocks): 2 A + 4 B fragment loads per 8 DMMAs
      const int rp = warp >> 1, ch = warp & 1;
      double acc[2][4][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) acc[h][nb][0] = acc[h][nb][1] = 0.0;
      for (int64_t t = t0; t < t1; ++t) {
        const int64_t J = __ldg(p.tile_col + t);
        __syncthreads();  // previous tile consumed
        if (async16) {
          // fp64, b = 64, 16-byte aligned X rows: 16-byte cp.async chunks (zero-filled past k
          // and n), all 16 per thread in flight at once
          for (int q = threadIdx.x; q < kTB * kTB / 2; q += blockDim.x) {
            const int j = q >> 5, i2 = (q & 31) * 2;
            cp_async16(sT + j * kLd + i2, (const double*)tv + t * kTB * kTB + j * kTB + i2, 16);
            const int64_t xr = J * kTB + j, c = c0 + i2;
            const int nb = (xr < p.n && c < k) ? (c + 1 < k ? 16 : 8) : 0;
            cp_async16(sX + j * kLd + i2, nb ? (const void*)(X + xr * ldx + c) : (const void*)X, nb);
          }
          asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
        } else {
          for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) {
            const int i = e & 63, j = e >> 6;
            sT[j * kLd + i] = (i < b && j < b) ? (double)__ldg(tv + t * b * b + (int64_t)j * b + i) : 0.0;
            const int64_t xr = J * b + j, c = c0 + i;  // panel element (j, c0 + i)
            sX[j * kLd + i] = (j < b && xr < p.n && c < k) ? (double)__ldg(X + xr * ldx + c) : 0.0;
          }
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kTB; kk += 4) {
          const double* tk = sT + (kk + tig) * kLd + rp * 16 + g;  // A[16rp + 8h + g][kk + tig]
          const double a0 = tk[0], a1 = tk[8];
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) {
            const double bb = sX[(kk + tig) * kLd + ch * 32 + nb * 8 + g];  // B[kk + tig][32ch + 8nb + g]
            dmma_8x8x4(acc[0][nb][0], acc[0][nb][1], a0, bb);
            dmma_8x8x4(acc[1][nb][0], acc[1][nb][1], a1, bb);
          }
        }
      }
      // D[g][2*tig + e] of (row fragment h, column block nb) -> Y row 16rp + 8h + g,
      // column c0 + 32ch + 8nb + 2tig + e
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = rp * 16 + h * 8 + g;
        const int64_t row = I * b + lr;
        if (lr < b && row >= p.row_lo && row < p.row_hi) {
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int64_t c = c0 + ch * 32 + nb * 8 + 2 * tig + e;
              if (c < k) put(Y + row * ldy + c, acc[h][nb][e], alpha, beta, p.mode != 0);
            }
        }
      }
    }
  }
}

int grid_of(int64_t work, int tpb) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = (work + tpb - 1) / tpb;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 16));
}

template <class V>
int spmm_part_t(const DevPart& p, const SpmmPart& s, double alpha, double beta, const V* X, int64_t ldx, V* Y,
                int64_t ldy, int64_t k, cudaStream_t st) {
  if (p.fam == FAM_DIA) {
    k_spmm_dia<V><<<grid_of(p.mb * k, 256), 256, 0, st>>>(p, alpha, beta, X, ldx, Y, ldy, k);
  } else if (p.fam == FAM_DENSE) {
    if (p.b > kTB) return (int)cudaErrorInvalidValue;
    // the shared-memory opt-in is a per-device function attribute: set it for the device
    // this launch runs on (idempotent and cheap; no process-wide cache to go stale or race)
    cudaError_t e = smem_optin(k_spmm_dense_dmma<V>, kDenseSmem);
    if (e != cudaSuccess) return (int)e;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(p.n_tile_rows, 148 * 8));
    k_spmm_dense_dmma<V><<<g, 256, kDenseSmem, st>>>(p, alpha, beta, X, ldx, Y, ldy, k);
  } else {
    if (!s.m_p) return 0;
    if constexpr (sizeof(V) == 8) {
      if (!(k & 1) && !(((uintptr_t)X | (uintptr_t)(ldx * 8)) & 15)) {  // double2 form
        const int64_t half = std::min<int64_t>(k / 2, 32);
        const int G = half <= 1 ? 1 : half <= 2 ? 2 : half <= 4 ? 4 : half <= 8 ? 8 : half <= 16 ? 16 : 32;
        const int g = grid_of(s.m_p * G, 256);
        const double* Xd = (const double*)X;
        double* Yd = (double*)Y;
        switch (G) {
          case 1: k_spmm_csr2<1><<<g, 256, 0, st>>>(s, alpha, beta, Xd, ldx, Yd, ldy, k); break;
          case 2: k_spmm_csr2<2><<<g, 256, 0, st>>>(s, alpha, beta, Xd, ldx, Yd, ldy, k); break;
          case 4: k_spmm_csr2<4><<<g, 256, 0, st>>>(s, alpha, beta, Xd, ldx, Yd, ldy, k); break;
          case 8: k_spmm_csr2<8><<<g, 256, 0, st>>>(s, alpha, beta, Xd, ldx, Yd, ldy, k); break;
          case 16: k_spmm_csr2<16><<<g, 256, 0, st>>>(s, alpha, beta, Xd, ldx, Yd, ldy, k); break;
          default: k_spmm_csr2<32><<<g, 256, 0, st>>>(s, alpha, beta, Xd, ldx, Yd, ldy, k); break;
        }
        return (int)cudaGetLastError();
      }
    }
    const int64_t kk = std::min<int64_t>(k, 32);
    const int G = kk <= 1 ? 1 : kk <= 2 ? 2 : kk <= 4 ? 4 : kk <= 8 ? 8 : kk <= 16 ? 16 : 32;
    const int g = grid_of(s.m_p * G, 256);
    switch (G) {
      case 1: k_spmm_csr<V, 1><<<g, 256, 0, st>>>(s, alpha, beta, X, ldx, Y, ldy, k); break;
      case 2: k_spmm_csr<V, 2><<<g, 256, 0, st>>>(s, alpha, beta, X, ldx, Y, ldy, k); break;
      case 4: k_spmm_csr<V, 4><<<g, 256, 0, st>>>(s, alpha, beta, X, ldx, Y, ldy, k); break;
      case 8: k_spmm_csr<V, 8><<<g, 256, 0, st>>>(s, alpha, beta, X, ldx, Y, ldy, k); break;
      case 16: k_spmm_csr<V, 16><<<g, 256, 0, st>>>(s, alpha, beta, X, ldx, Y, ldy, k); break;
      default: k_spmm_csr<V, 32><<<g, 256, 0, st>>>(s, alpha, beta, X, ldx, Y, ldy, k); break;
    }
  }
  return (int)cudaGetLastError();
}

}  // namespace

int launch_spmm_part(const DevPart& p, const SpmmPart& s, double alpha, double beta, const void* X, int64_t ldx,
                     void* Y, int64_t ldy, int64_t k, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (p.dtype == 1) return spmm_part_t<double>(p, s, alpha, beta, (const double*)X, ldx, (double*)Y, ldy, k, st);
  return spmm_part_t<float>(p, s, alpha, beta, (const float*)X, ldx, (float*)Y, ldy, k, st);
}

int launch_spmm_prepass(const int32_t* rows, int64_t n, int64_t m, double beta, void* Y, int64_t ldy, int64_t k,
                        int dtype, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (rows) {
    if (n <= 0) return 0;
    if (dtype == 1) k_spmm_prepass<double><<<grid_of(n * k, 256), 256, 0, st>>>(rows, n, beta, (double*)Y, ldy, k);
    else k_spmm_prepass<float><<<grid_of(n * k, 256), 256, 0, st>>>(rows, n, beta, (float*)Y, ldy, k);
  } else {
    if (m <= 0) return 0;
    if (dtype == 1) k_spmm_scale<double><<<grid_of(m * k, 256), 256, 0, st>>>(m, beta, (double*)Y, ldy, k);
    else k_spmm_scale<float><<<grid_of(m * k, 256), 256, 0, st>>>(m, beta, (float*)Y, ldy, k);
  }
  return (int)cudaGetLastError();
}

}  // namespace as
