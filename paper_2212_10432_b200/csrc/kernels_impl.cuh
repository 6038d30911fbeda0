// sm_100a SpMV kernel family: one kernel per (mapping level x reduction strategy) class of
// the implementing stage (§IV-A), plus the DIA / dense-tile kernels implied by
// DIA_DECOM / DENSE_DECOM (P:21 draft) and the beta pre-pass of the writer rule (A22).
//
// Every kernel computes, for its rows, acc = sum a_ij * x_j in double (fp64 accumulation
// for fp32 data too, reading A2) and writes
//   exclusive rows:  STORE y = alpha*acc + beta*y   |  ADD  y += alpha*acc
//   shared rows:     atomicAdd(y, alpha*partial)     (GMEM_ATOM_RED)
// The path is HBM-bound (0.12-0.25 flop/B), so the kernels are written for bytes in flight:
// streaming loads of values/indices through the non-coherent path with an evict-first L2
// hint (the matrix is touched once per call), gathers of x through L1/L2, and grid-stride
// loops so any SET_RESOURCE grid is legal.  No tensor cores: with one vector every dense
// block is a GEMV (2 flops per value loaded), not a contraction.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "devpart.h"
#include "kcommon.cuh"
#include "klaunch.h"

namespace as {

namespace {


// =====================================================================================
// FAM_THREAD_ROW: BMT_ROW_BLOCK(s) [+ROW parents] + THREAD_TOTAL / THREAD_BITMAP_RED_G.
// CSR-Scalar when unpadded; ELL / SELL-P (slot-major interleaved) with
// BMT_PAD: consecutive threads read consecutive vec-chunks -> fully coalesced 128-bit loads.
// =====================================================================================
template <class V>
__global__ void __launch_bounds__(1024) k_thread_row(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const V* val = (const V*)p.val;
  for (int64_t t = thread_units(p.n_bmt).begin, t_e = thread_units(p.n_bmt).end; t < t_e; t += blockDim.x) {
    int64_t r0 = bmt_rowp_at(p, t);
    int64_t r1 = bmt_rowp_at(p, t + 1);
    for (int64_t r = r0; r < r1; ++r) {
      int64_t a = ldm(p.row_ptr + r), e = ldm(p.row_ptr + r + 1);
      double acc0 = 0.0, acc1 = 0.0;
      int64_t i = a;
      for (; i + 1 < e; i += 2) {
        int32_t c0 = ld_stream(p.col + i), c1 = ld_stream(p.col + i + 1);
        double v0 = (double)ld_stream(val + i), v1 = (double)ld_stream(val + i + 1);
        acc0 += v0 * ldx(x, c0);
        acc1 += v1 * ldx(x, c1);
      }
      if (i < e) acc0 += (double)ld_stream(val + i) * ldx(x, ld_stream(p.col + i));
      write_excl(p, y, r, acc0 + acc1);
    }
  }
}


template <class V, int VEC>
__global__ void __launch_bounds__(1024) k_thread_row_pad(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const V* pval = (const V*)p.pad_val;
  for (int64_t t = thread_units(p.n_bmt).begin, t_e = thread_units(p.n_bmt).end; t < t_e; t += blockDim.x) {
    int64_t g, t0, t1;
    if (p.grp_regular) {
      g = t / p.grp_regular;
      t0 = g * p.grp_regular;
      t1 = min(t0 + p.grp_regular, p.n_bmt);
    } else {  // binary search the group of BMT t
      int64_t lo = 0, hi = p.n_grp - 1;
      while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (ldm(p.grp_first_bmt + mid) <= t) lo = mid;
        else hi = mid - 1;
      }
      g = lo;
      t0 = ldm(p.grp_first_bmt + g);
      t1 = ldm(p.grp_first_bmt + g + 1);
    }
    const int64_t nt = t1 - t0, lt = t - t0;
    const int64_t W = grp_width_at(p, g);
    const int64_t base = grp_base_at(p, g) + lt * VEC;
    const int64_t stride = nt * VEC;
    int64_t r0 = bmt_rowp_at(p, t);
    int64_t r1 = bmt_rowp_at(p, t + 1);
    if (r1 - r0 == 1) {
      // whole BMT is one row: read all W slots (pads have value 0, valid col)
      double acc[VEC];
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
      const int64_t nchunk = W / VEC;
#pragma unroll 4
      for (int64_t c = 0; c < nchunk; ++c) {
        double v[VEC];
        int32_t cc[VEC];
        PadLoad<V, VEC>::ld(pval + base + c * stride, p.pad_col + base + c * stride, v, cc);
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] += v[q] * ldx(x, cc[q]);
      }
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < VEC; ++q) s += acc[q];
      write_excl(p, y, r0, s);
    } else {
      // several rows in one padded BMT: row boundaries from row_ptr (local offsets)
      int64_t nz0 = ldm(p.row_ptr + r0);
      for (int64_t r = r0; r < r1; ++r) {
        int64_t ja = ldm(p.row_ptr + r) - nz0, je = ldm(p.row_ptr + r + 1) - nz0;
        double acc = 0.0;
        for (int64_t j = ja; j < je; ++j) {
          int64_t slot = base + (j / VEC) * stride + (j % VEC);
          acc += (double)ld_stream(pval + slot) * ldx(x, ld_stream(p.pad_col + slot));
        }
        write_excl(p, y, r, acc);
      }
    }
  }
}

// =====================================================================================
// BMT element source for the nonzero-split kernels.
//   PAD = false: the CSR order of COMPRESS; a thread walks k consecutive nonzeros, so the
//                loads allocate in L1 (the warp's 32*k-element window is reused across j).
//   PAD = true:  BMT_PAD slot-major layout (reading A18): element j of BMT t sits at
//                base_g + (j/VEC)*n_t*VEC + lt*VEC + j%VEC, so at every step the 32 lanes of
//                a warp read 32 consecutive VEC-chunks: fully coalesced streaming loads (the
//                CSR5 tile transpose expressed with the paper's own padding operator).
// =====================================================================================

// Serial pass over one BMT (THREAD_BITMAP_RED_G): calls seg(row, partial, head_inside) at
// every bitmap head after element 0; returns the open (last) segment in acc/row/inside.
// x accessors: straight from global memory (L1 / L2 evict_last), or from a shared-memory
// ring buffer holding the CTA's current x window (banded matrices, k_nnz_thread_xw).
// Elements per batch of the warp-level NNZ kernels: fp64 batches of 8 spill 100-180 bytes
// next to the warp-combine state; fp32 operands stay fp32 in registers until the FMA, so
// fp32 affords 8 gathers in flight per lane at 64 registers (C3 winner family: 924.7 ->
// 885.7 us; 16 spills 120-184 bytes and is slower, 949 us; profiles/r02/ab_kb.jsonl).
// AS_NWPE_LB (A/B build knob): launch bound of k_nnz_warp_pe (its register budget)
#ifndef AS_NWPE_LB
#define AS_NWPE_LB 1024
#endif
#ifndef AS_KBW_F32
#define AS_KBW_F32 8
#endif
#ifndef AS_KBW_F64
#define AS_KBW_F64 4
#endif
template <class V>
constexpr int kbw_of() {
  return sizeof(V) == 4 ? AS_KBW_F32 : AS_KBW_F64;
}

template <class V>
struct XGlobal {
  const V* __restrict__ x;
  __device__ __forceinline__ double operator()(int64_t c) const { return ldx(x, c); }
  __device__ __forceinline__ V v(int64_t c) const { return ldxv(x, c); }
};
// Hot-x cache (SET_RESOURCE xcache, reading R-xcache): the part's K most referenced x
// entries are staged in shared memory once per (persistent) CTA; their columns were
// re-encoded at plan time as ~slot (negative), so a gather reads shared memory instead of
// moving a 32-byte L1/L2 sector.  On power-law matrices (C3) the top 32K columns carry a
// third of the nonzeros; the rest are gathered from global memory as before.
template <class V>
struct XHot {
  const V* __restrict__ x;
  const V* sm;
  __device__ __forceinline__ double operator()(int64_t c) const { return c < 0 ? (double)sm[~c] : (double)ldxv_l2(x, c); }
  __device__ __forceinline__ V v(int64_t c) const { return c < 0 ? sm[~c] : ldxv_l2(x, c); }
};
// All CTAs fill at kernel start, so the fill's latency is exposed once per CTA: 8 column
// indices, then 8 gathers, are in flight per thread (a one-load-at-a-time loop cost ~25 us
// of start-up for 24K entries)
template <class V>
__device__ __forceinline__ void xhot_fill(const DevPart& p, const V* __restrict__ x, V* sm) {
  constexpr int U = 8;
  const int64_t n = p.xh_n, T = blockDim.x;
  int64_t i = threadIdx.x;
  for (; i + (U - 1) * T < n; i += U * T) {
    int32_t c[U];
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = ldm(p.xh_cols + i + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) sm[i + u * T] = v[u];
  }
  for (; i < n; i += T) sm[i] = __ldg(x + ldm(p.xh_cols + i));
  __syncthreads();
}

template <class V>
struct XRing {
  const V* ring;
  int64_t mask;
  __device__ __forceinline__ double operator()(int64_t c) const { return (double)ring[c & mask]; }
  __device__ __forceinline__ V v(int64_t c) const { return ring[c & mask]; }
};

// One batch of KB elements starting at j0.  FULL: j0 + KB <= len, so no bounds predicates
// (the common case: every batch but the BMT's last).
template <class V, bool PAD, int VEC, int KB, bool FULL, class XA, class Seg>
__device__ __forceinline__ void bmt_batch(XA xa, const uint32_t* bm, const V* pv, const int32_t* pc, int64_t stride,
                                          int j0, int len, int64_t& row, double& acc, bool& inside, Seg& seg) {
  double v[KB];
  int32_t c[KB];
  if constexpr (PAD) {
#pragma unroll
    for (int q = 0; q < KB; q += VEC) {
      if (FULL || j0 + q < len) {
        PadLoad<V, VEC>::ld(pv + ((j0 + q) / VEC) * stride, pc + ((j0 + q) / VEC) * stride, v + q, c + q);
      } else {
#pragma unroll
        for (int r = 0; r < VEC; ++r) {
          v[q + r] = (V)0;
          c[q + r] = 0;
        }
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      if (FULL || j0 + q < len) {
        v[q] = (double)ld_seq(pv + j0 + q);
        c[q] = ld_seq(pc + j0 + q);
      } else {
        v[q] = 0.0;
        c[q] = 0;
      }
    }
  }
  double xv[KB];
#pragma unroll
  for (int q = 0; q < KB; ++q) xv[q] = (FULL || j0 + q < len) ? xa(c[q]) : 0.0;
  // head bits of this batch; element 0 of the BMT never cuts (its head state is `inside`)
  const uint32_t wd = (ldm(bm + (j0 >> 5)) >> (j0 & 31)) & ~(uint32_t)(j0 == 0);
#pragma unroll
  for (int q = 0; q < KB; ++q) {
    if (!FULL && j0 + q >= len) break;
    if ((wd >> q) & 1u) {
      seg(row, acc, inside);
      ++row;
      acc = 0.0;
      inside = true;
    }
    acc += v[q] * xv[q];
  }
}

template <class V, bool PAD, int VEC, int KB, class XA, class Seg>
__device__ __forceinline__ void bmt_pass(const DevPart& p, XA xa, const uint32_t* bm, PadPos pp, int64_t a, int len,
                                         int64_t& row, double& acc, bool& inside, Seg seg) {
  // Batches of KB elements: all value/column loads of a batch are issued, then all x
  // gathers, then the bitmap-segmented accumulation -> KB independent loads in flight per
  // thread instead of one element behind each head test.  pp: slot base/stride of this
  // BMT in the padded layout, computed by the caller (no per-BMT division).
  static_assert(32 % KB == 0 && KB % VEC == 0, "KB divides 32 and is a multiple of VEC");
  inside = ldm(bm) & 1u;
  acc = 0.0;
  const V* pv = PAD ? (const V*)p.pad_val + pp.base : (const V*)p.val + a;
  const int32_t* pc = PAD ? p.pad_col + pp.base : p.col + a;
  const int full = len & ~(KB - 1);
  int j0 = 0;
  for (; j0 < full; j0 += KB)
    bmt_batch<V, PAD, VEC, KB, true>(xa, bm, pv, pc, pp.stride, j0, len, row, acc, inside, seg);
  if (j0 < len) bmt_batch<V, PAD, VEC, KB, false>(xa, bm, pv, pc, pp.stride, j0, len, row, acc, inside, seg);
}

// =====================================================================================
// FAM_NNZ_THREAD: BMT_NNZ_BLOCK(k) + THREAD_BITMAP_RED_G.  Each thread reduces its k
// nonzeros serially, cutting at bitmap heads (bit j = element j starts a row, A20); rows
// whose head and end lie in the BMT are exclusive, straddlers go to y by atomics ("_G").
// =====================================================================================
template <class V, bool PAD, int VEC, int KB, class XA>
__device__ __forceinline__ void nnz_thread_bmt(const DevPart& p, XA xa, V* __restrict__ y, int64_t t) {
  int64_t a = p.bmt_start ? ldm(p.bmt_start + t) : t * p.k;
  int64_t e = p.bmt_start ? ldm(p.bmt_start + t + 1) : min(a + p.k, p.nnz_p);
  int64_t row = bmt_row0(p, t);
  double acc;
  bool inside;
  PadPos pp{0, 0};
  if constexpr (PAD) pp = p.n_grp == 1 ? PadPos{t * VEC, p.n_bmt * VEC} : pad_pos<VEC>(p, t);
  bmt_pass<V, PAD, VEC, KB>(p, xa, bmt_bits(p, t), pp, a, (int)(e - a), row, acc, inside,
                            [&](int64_t r, double s, bool in) {
                              if (in) write_excl(p, y, r, s);
                              else write_atom(p, y, r, s);
                            });
  bool ends = (t + 1 >= p.n_bmt) ? true : (ldm(bmt_bits(p, t + 1)) & 1u);
  if (inside && ends) write_excl(p, y, row, acc);
  else write_atom(p, y, row, acc);
}

template <class V, bool PAD, int VEC, int KB>
__global__ void __launch_bounds__(1024) k_nnz_thread(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  for (int64_t t = thread_units(p.n_bmt).begin, t_e = thread_units(p.n_bmt).end; t < t_e; t += blockDim.x)
    nnz_thread_bmt<V, PAD, VEC, KB>(p, XGlobal<V>{x}, y, t);
}

// -------------------------------------------------------------------------------------
// k_nnz_thread, predicated-emit form (all plans but fp32 ADD-mode parts with heavy rows).  The per-element
// head test of the form above branches around a writer call, and the 32 lanes of a warp
// hit their heads at different elements, so ncu saw 12 of 32 threads active on average
// (C5: 1.35 warp instructions per nonzero).  Here the loop body is branch-free: rows that
// close inside the BMT (the only ones a head can close, apart from the BMT's first
// segment) are written by one predicated store; the straddling first segment is kept in
// a register and, with the open last segment, written after the loop (atomically when
// it straddles, A22) -- the same writes as THREAD_BITMAP_RED_G above, in the same order
// per row.
//   EM 0: STORE mode, beta == 0, affine origin_rows (y[base + r] = alpha * s)
//   EM 1: any mode / beta / origin_rows
// -------------------------------------------------------------------------------------
template <class V, int EM>
__device__ __forceinline__ void emit_excl(const DevPart& p, V* y, bool pred, int64_t r, double s) {
  if constexpr (EM == 0) {
    if (pred) {
      y[p.origin_base + r] = (V)(p.alpha * s);
      if (p.n_peer) peer_store(p, p.origin_base + r, (V)(p.alpha * s));
    }
  } else {
    if (pred) {
      const int64_t g = out_row(p, r);
      double v = p.alpha * s;
      if (p.mode == 1) v += (double)y[g];
      else if (p.beta != 0.0) v += p.beta * (double)y[g];
      y[g] = (V)v;
      if (p.mode == 0 && p.n_peer) peer_store(p, g, (V)v);
    }
  }
}

// Loads of one batch (values, columns) ...
template <class V, bool PAD, int VEC, int KB, bool FULL>
__device__ __forceinline__ void batch_load(const V* pv, const int32_t* pc, int64_t stride, int j0, int len, V* v,
                                           int32_t* c) {
  if constexpr (PAD) {
#pragma unroll
    for (int q = 0; q < KB; q += VEC) {
      if (FULL || j0 + q < len) {
        PadLoad<V, VEC>::ld(pv + (q / VEC) * stride, pc + (q / VEC) * stride, v + q, c + q);
      } else {
#pragma unroll
        for (int r = 0; r < VEC; ++r) {
          v[q + r] = (V)0;
          c[q + r] = 0;
        }
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      if (FULL || j0 + q < len) {
        v[q] = ld_seq(pv + q);
        c[q] = ld_seq(pc + q);
      } else {
        v[q] = (V)0;
        c[q] = 0;
      }
    }
  }
}

// ... and their use: x gathers, then the branch-free bitmap-segmented accumulation.
// Bitmap words of one BMT.  BMO: the first two words are loaded once per BMT (k <= 64: every
// batch's word) instead of once per batch -- the thread-level kernel gains (C5 2632 -> 2468
// us), the register-bound warp-level kernel loses (C3 886 -> 904 us), so it is a template
// choice of the kernel (profiles/r02/ab_pe.jsonl; a one-batch load prefetch spilled and lost
// everywhere: C3 1277, C5 6459 us).
template <bool BMO>
struct BmWords {
  const uint32_t* bm;
  uint32_t w0, w1;
  __device__ __forceinline__ uint32_t at(int j0) const {
    if constexpr (BMO) {
      const int w = j0 >> 5;
      return w == 0 ? w0 : w == 1 ? w1 : ldm(bm + w);
    } else {
      return ldm(bm + (j0 >> 5));
    }
  }
};

// AS_F32_ACC (A/B build knob): fp32 data accumulate each lane's BMT segment in fp32 (FFMA)
// instead of fp64; a segment holds at most k products, so its rounding error is at most
// k * 2^-24 * sum|a x| (k = 32: 1.9e-6, inside the north_star fp32 tolerance of 1e-5)
#ifndef AS_F32_ACC
#define AS_F32_ACC 0
#endif
template <class V>
using AccOf = std::conditional_t<AS_F32_ACC && sizeof(V) == 4, float, double>;
template <class V, int KB, int EM, bool FULL, class XA, class BW, class A>
__device__ __forceinline__ void batch_use(const DevPart& p, V* y, XA xa, const BW& bm, int j0, int len,
                                          const V* v, const int32_t* c, int32_t& row, A& acc, bool& inside,
                                          A& first) {
  V xv[KB];
#pragma unroll
  for (int q = 0; q < KB; ++q) xv[q] = (FULL || j0 + q < len) ? xa.v(c[q]) : (V)0;
  const uint32_t wd = (bm.at(j0) >> (j0 & 31)) & ~(uint32_t)(j0 == 0);
#pragma unroll
  for (int q = 0; q < KB; ++q) {
    const bool h = (FULL || j0 + q < len) && ((wd >> q) & 1u);
    emit_excl<V, EM>(p, y, h && inside, row, (double)acc);
    first = (h && !inside) ? acc : first;
    row += h ? 1 : 0;
    inside = inside || h;
    acc = (h ? (A)0 : acc) + (A)v[q] * (A)xv[q];
  }
}

// AS_L1_PREFETCH (A/B build knob): request the next batch's value / column lines into L1
// while the current batch waits on its gathers, so the batch's loads hit L1 instead of
// exposing the HBM latency (the prefetch issues the same L1->L2 requests the loads would).
#ifndef AS_L1_PREFETCH
#define AS_L1_PREFETCH 0
#endif
template <class V, bool PAD, int VEC, int KB>
__device__ __forceinline__ void batch_prefetch_l1(const V* pv, const int32_t* pc, int64_t stride) {
  if constexpr (PAD) {
#pragma unroll
    for (int q = 0; q < KB; q += VEC) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(pv + (q / VEC) * stride));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(pc + (q / VEC) * stride));
    }
  } else {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(pv));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(pc));
  }
}

// One BMT in predicated-emit form: rows closed inside the BMT are stored in the loop; the
// caller gets the straddling first segment (`first`, valid when !s0 && inside), the open last
// segment (`acc`, of row `row`), and whether the BMT starts at a row head (s0) / holds a
// head anywhere (inside).
struct ScanPE {
  double first, acc;
  int32_t row;
  bool s0, inside;
};
template <class V, bool PAD, int VEC, int KB, int EM, bool BMO, class XA>
__device__ __forceinline__ ScanPE bmt_scan_pe(const DevPart& p, V* y, XA xa, int64_t t, PadPos pp) {
  static_assert(32 % KB == 0 && KB % VEC == 0, "KB divides 32 and is a multiple of VEC");
  const int64_t a = p.bmt_start ? ldm(p.bmt_start + t) : t * p.k;
  const int64_t e = p.bmt_start ? ldm(p.bmt_start + t + 1) : min(a + p.k, p.nnz_p);
  const int len = (int)(e - a);
  const uint32_t* bmp = bmt_bits(p, t);
  const V* pv = PAD ? (const V*)p.pad_val + pp.base : (const V*)p.val + a;  // batch base
  const int32_t* pc = PAD ? p.pad_col + pp.base : p.col + a;
  BmWords<BMO> bm{bmp, 0u, 0u};
  if constexpr (BMO) {
    bm.w0 = ldm(bmp);
    bm.w1 = p.bm_words > 1 ? ldm(bmp + 1) : 0u;
  }
  ScanPE o;
  o.s0 = (BMO ? bm.w0 : ldm(bmp)) & 1u;
  o.inside = o.s0;
  o.row = (int32_t)bmt_row0(p, t);  // device row indices are int32 (A36)
  AccOf<V> acc = 0, first = 0;
  const int full = len & ~(KB - 1);
  int j0 = 0;
  // pv / pc advance to the batch's first element (slot-major: KB/VEC chunk rows per batch)
  const int64_t adv = PAD ? (KB / VEC) * pp.stride : KB;
  V v[KB];
  int32_t c[KB];
  for (; j0 < full; j0 += KB, pv += adv, pc += adv) {
    batch_load<V, PAD, VEC, KB, true>(pv, pc, pp.stride, j0, len, v, c);
    if constexpr (AS_L1_PREFETCH)
      if (j0 + KB < len) batch_prefetch_l1<V, PAD, VEC, KB>(pv + adv, pc + adv, pp.stride);
    batch_use<V, KB, EM, true>(p, y, xa, bm, j0, len, v, c, o.row, acc, o.inside, first);
  }
  if (j0 < len) {
    batch_load<V, PAD, VEC, KB, false>(pv, pc, pp.stride, j0, len, v, c);
    batch_use<V, KB, EM, false>(p, y, xa, bm, j0, len, v, c, o.row, acc, o.inside, first);
  }
  o.acc = (double)acc;
  o.first = (double)first;
  return o;
}

// one BMT of THREAD_BITMAP_RED_G in predicated-emit form, with the BMT's two boundary writes
template <class V, bool PAD, int VEC, int KB, int EM, class XA>
__device__ __forceinline__ void nnz_thread_bmt_pe(const DevPart& p, XA xa, V* __restrict__ y, int64_t t) {
  PadPos pp{0, 0};
  if constexpr (PAD) pp = p.n_grp == 1 ? PadPos{t * VEC, p.n_bmt * VEC} : pad_pos<VEC>(p, t);
  const ScanPE o = bmt_scan_pe<V, PAD, VEC, KB, EM, true>(p, y, xa, t, pp);
  // first segment closed inside the BMT but begun before it: straddler
  if (!o.s0 && o.inside) write_atom(p, y, bmt_row0(p, t), o.first);
  // open last segment: exclusive iff it began at a head here and the next BMT starts a row
  const bool ends = (t + 1 >= p.n_bmt) ? true : (ldm(bmt_bits(p, t + 1)) & 1u);
  if (o.inside && ends) write_excl(p, y, o.row, o.acc);
  else write_atom(p, y, o.row, o.acc);
}

template <class V, bool PAD, int VEC, int KB, int EM, bool XH>
__global__ void __launch_bounds__(1024) k_nnz_thread_pe(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const Units u = thread_units(p.n_bmt);
  if constexpr (XH) {
    extern __shared__ __align__(128) unsigned char xh_smem[];
    V* xs = (V*)xh_smem;
    xhot_fill(p, x, xs);
    for (int64_t t = u.begin, t_e = u.end; t < t_e; t += blockDim.x)
      nnz_thread_bmt_pe<V, PAD, VEC, KB, EM>(p, XHot<V>{x, xs}, y, t);
  } else {
    for (int64_t t = u.begin, t_e = u.end; t < t_e; t += blockDim.x)
      nnz_thread_bmt_pe<V, PAD, VEC, KB, EM>(p, XGlobal<V>{x}, y, t);
  }
}

// =====================================================================================
// k_nnz_thread, x-window form (banded matrices): persistent CTAs own contiguous BMT ranges
// processed in rounds of blockDim BMTs; round i of CTA c needs x[lo, hi] (computed at plan
// time, lo made non-decreasing, span < ring size).  The CTA keeps x in a shared-memory ring
// buffer, loading only the part of each window beyond what it already holds, so the
// gathers read shared memory instead of moving a 32-byte L1/L2 sector per nonzero.
// =====================================================================================
// EM >= 0: predicated-emit scan (bmt_scan_pe) on the ring; EM < 0: branching form
template <class V, bool PAD, int VEC, int EM>
__global__ void __launch_bounds__(1024) k_nnz_thread_xw(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* ring = (V*)smem_raw;
  const int64_t mask = p.xw_size - 1;
  const int64_t per = (p.n_bmt + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(b0 + per, p.n_bmt);
  const int64_t rounds = b1 > b0 ? (b1 - b0 + blockDim.x - 1) / blockDim.x : 0;
  int64_t have_hi = -1;
  for (int64_t i = 0; i < rounds; ++i) {
    const int64_t w = (int64_t)blockIdx.x * p.xw_rpc + i;
    const int64_t lo = ldm(p.xwin + 2 * w), hi = ldm(p.xwin + 2 * w + 1);
    for (int64_t c = max(have_hi + 1, lo) + threadIdx.x; c <= hi; c += blockDim.x) ring[c & mask] = __ldg(x + c);
    if (hi > have_hi) have_hi = hi;
    __syncthreads();
    const int64_t t = b0 + i * blockDim.x + threadIdx.x;
    if (t < b1) {
      if constexpr (EM >= 0) nnz_thread_bmt_pe<V, PAD, VEC, (sizeof(V) == 4 ? 4 : 8), EM>(p, XRing<V>{ring, mask}, y, t);
      else nnz_thread_bmt<V, PAD, VEC, 8>(p, XRing<V>{ring, mask}, y, t);
    }
    __syncthreads();  // the next window update overwrites entries this round may read
  }
}

// =====================================================================================
// FAM_NNZ_WARP: BMW blocks of BMT_NNZ(k) tiles; lanes take BMTs in rounds of 32.
// Per lane: c_in (partial before its first head), c_out (partial from its last head),
// interior rows stored directly.  Warp level:
//   WRED == 1  WARP_SEG_ADD_RED: segmented inclusive scan over lanes (shfl_up + head flags,
//              the "segment sum" of P:281)
//   WRED == 2  WARP_BITMAP_RED: ballot of per-lane head flags (the lane bitmap) locates each
//              segment's previous head lane; plain prefix sums give the segment totals.
// Rows closed inside the BMW are exclusive; rows entering from before the BMW or leaving
// after it are added atomically.
// =====================================================================================

// Vector load of KL consecutive values / columns (one chunk per lane; adjacent lanes read
// adjacent chunks, so a warp reads 32*KL contiguous elements per instruction).
template <class V, int KL>
__device__ __forceinline__ void ld_chunk(const V* v, const int32_t* c, double* vo, int32_t* co) {
  if constexpr (KL == 1) {
    vo[0] = (double)ld_stream(v);
    co[0] = ld_stream(c);
  } else {
    PadLoad<V, KL>::ld(v, c, vo, co);
  }
}

// =====================================================================================
// FAM_NNZ_WARP, tile form (BMT_NNZ_BLOCK(k) with k in {1,2,4}, uniform BMW_NNZ_BLOCK of a
// multiple of 32k, no padding): a round is 32*k contiguous nonzeros read with one vector
// load per lane (coalesced, no per-BMT metadata).  Row heads come from a packed bitmap (1
// bit per nonzero: the per-BMT bitmaps of A20 concatenated in lane order) and the row of
// every lane from the BMW's first row plus a warp prefix count of heads (the first_row of
// each BMT is linear in the head count, so it is computed, not stored; reading A17).
// =====================================================================================
template <class V, int KL, int WRED>
__global__ void __launch_bounds__(512) k_warp_tile(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const V* val = (const V*)p.val;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = gthreads() >> 5;
  const int64_t k2 = p.bmts_per_bmw * KL;  // nonzeros per BMW
  for (int64_t w = warp_units(p.n_bmw).begin, w_e = warp_units(p.n_bmw).end; w < w_e; w += blockDim.x >> 5) {
    const int64_t a = w * k2, e = min(a + k2, p.nnz_p);
    const uint32_t w0 = ldm(p.bits + (a >> 5));
    const bool head_a = w0 & (1u << (a & 31));
    int64_t rb = (int64_t)ldm(p.bmw_first_row + w) - (head_a ? 1 : 0);  // row before the round
    double carry = 0.0;
    bool carry_inside = false, carry_live = false;
    int64_t carry_row = 0;
    // 2-stage software pipeline: the vector loads of round r+1 are in flight while round r
    // gathers x and runs its segmented combine.
    auto load_round = [&](int64_t eb, double* v, int32_t* c, uint32_t& hb) {
      const int64_t i0 = eb + lane * KL;
      const bool active = i0 < e;
      if (active && i0 + KL <= e) {
        ld_chunk<V, KL>(val + i0, p.col + i0, v, c);
      } else {
#pragma unroll
        for (int q = 0; q < KL; ++q) {
          v[q] = (active && i0 + q < e) ? (double)ld_stream(val + i0 + q) : 0.0;
          c[q] = (active && i0 + q < e) ? ld_stream(p.col + i0 + q) : 0;
        }
      }
      hb = 0;
      if (active) {
        hb = (ldm(p.bits + (i0 >> 5)) >> (i0 & 31)) & ((1u << KL) - 1u);
        if (e - i0 < KL) hb &= (1u << (e - i0)) - 1u;
      }
    };
    double vn[KL];
    int32_t cn[KL];
    uint32_t hbn;
    load_round(a, vn, cn, hbn);
    for (int64_t eb = a; eb < e; eb += 32 * KL) {
      const int64_t i0 = eb + lane * KL;
      const bool active = i0 < e;
      const int nact = (int)min((int64_t)32, (e - eb + KL - 1) / KL);
      double v[KL];
      int32_t c[KL];
#pragma unroll
      for (int q = 0; q < KL; ++q) {
        v[q] = vn[q];
        c[q] = cn[q];
      }
      const uint32_t hb = hbn;
      if (eb + 32 * KL < e) load_round(eb + 32 * KL, vn, cn, hbn);
      double xv[KL];
#pragma unroll
      for (int q = 0; q < KL; ++q) xv[q] = (active && i0 + q < e) ? ldx(x, c[q]) : 0.0;
      // exclusive prefix of head counts over lanes -> this lane's starting row
      int cnt = __popc(hb), pre = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, pre, d);
        if (lane >= d) pre += n;
      }
      const int total = __shfl_sync(0xffffffffu, pre, 31);
      int64_t row = rb + (pre - cnt);  // row of the element before this lane's chunk
      // serial pass over the lane's KL elements
      double cin = 0.0, cout = 0.0, cur = 0.0;
      bool hh = false;
      int64_t head_row = row + 1;
#pragma unroll
      for (int q = 0; q < KL; ++q) {
        if (hb & (1u << q)) {
          if (!hh) {
            cin = cur;
            hh = true;
          } else {
            write_excl(p, y, row, cur);  // row wholly inside this lane's chunk
          }
          ++row;
          cur = 0.0;
        }
        cur += v[q] * xv[q];
      }
      if (hh) cout = cur;
      else cin = cur;
      double v_end, closing;
      bool inside_end, closing_inside;
      warp_combine<WRED>(lane, hh, cin, cout, carry, carry_inside, closing, closing_inside, v_end, inside_end);
      if (active && hh) {
        bool exists = !(lane == 0 && !carry_live && (hb & 1u));
        if (exists) {
          if (closing_inside) write_excl(p, y, head_row - 1, closing);
          else write_atom(p, y, head_row - 1, closing);
        }
      }
      carry = __shfl_sync(0xffffffffu, v_end, nact - 1);
      carry_inside = __shfl_sync(0xffffffffu, (int)inside_end, nact - 1);
      carry_row = __shfl_sync(0xffffffffu, row, nact - 1);
      carry_live = true;
      rb += total;
    }
    if (lane == 0 && carry_live) {
      bool ends = e >= p.nnz_p ? true : ((ldm(p.bits + (e >> 5)) >> (e & 31)) & 1u);
      if (carry_inside && ends) write_excl(p, y, carry_row, carry);
      else write_atom(p, y, carry_row, carry);
    }
  }
}

template <class V, int WRED, bool PAD, int VEC>
__global__ void __launch_bounds__(1024) k_nnz_warp(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = gthreads() >> 5;
  for (int64_t w = warp_units(p.n_bmw).begin, w_e = warp_units(p.n_bmw).end; w < w_e; w += blockDim.x >> 5) {
    int64_t tb0 = bmw_bmt_at(p, w);
    int64_t tb1 = bmw_bmt_at(p, w + 1);
    double carry = 0.0;
    bool carry_inside = false;  // open segment's row started at a head inside this BMW
    bool carry_live = false;    // an open segment exists (false only before the first element)
    int64_t carry_row = 0;
    for (int64_t base = tb0; base < tb1; base += 32) {
      const int64_t t = base + lane;
      const bool active = t < tb1;
      const int nact = (int)min((int64_t)32, tb1 - base);
      double cin = 0.0, cout = 0.0;
      bool hh = false, b0 = false;
      int64_t head_row = 0;  // row of the first head in this lane
      int64_t last_row = 0;  // row of this lane's last element
      if (active) {
        int64_t a = p.bmt_start ? ldm(p.bmt_start + t) : t * p.k;
        int64_t e = p.bmt_start ? ldm(p.bmt_start + t + 1) : min(a + p.k, p.nnz_p);
        int64_t row = bmt_row0(p, t);
        head_row = row;
        double cur;
        bool in;
        bool first_open = true;
        PadPos pp{0, 0};
        if constexpr (PAD) {
          if (p.pad_grp_bmw) pp = PadPos{grp_base_at(p, w) + (t - tb0) * VEC, (tb1 - tb0) * VEC};
          else if (p.n_grp == 1) pp = PadPos{t * VEC, p.n_bmt * VEC};
          else pp = pad_pos<VEC>(p, t);
        }
        bmt_pass<V, PAD, VEC, 8>(p, XGlobal<V>{x}, bmt_bits(p, t), pp, a, (int)(e - a), row, cur, in,
                              [&](int64_t r, double s, bool inside) {
          if (!inside && first_open) {  // continuation of a row begun in an earlier lane
            cin = s;
            head_row = r + 1;
          } else {
            write_excl(p, y, r, s);  // row wholly inside this lane's BMT
          }
          first_open = false;
        });
        b0 = ldm(bmt_bits(p, t)) & 1u;
        hh = in;
        if (hh) cout = cur;
        else cin = cur;
        last_row = row;
      }
      double v_end, closing;
      bool inside_end, closing_inside;
      warp_combine<WRED>(lane, hh, cin, cout, carry, carry_inside, closing, closing_inside, v_end, inside_end);
      if (active && hh) {
        // the row closed at this lane's first head; none only when the BMW itself starts
        // with a head (lane 0 of the first round, element 0 is a row start)
        bool exists = !(lane == 0 && !carry_live && b0);
        if (exists) {
          if (closing_inside) write_excl(p, y, head_row - 1, closing);
          else write_atom(p, y, head_row - 1, closing);
        }
      }
      carry = __shfl_sync(0xffffffffu, v_end, nact - 1);
      carry_inside = __shfl_sync(0xffffffffu, (int)inside_end, nact - 1);
      carry_row = __shfl_sync(0xffffffffu, last_row, nact - 1);
      carry_live = true;
    }
    if (lane == 0 && carry_live) {
      // final open segment: the row of the BMW's last element
      bool ends = (tb1 >= p.n_bmt) ? true : (ldm(bmt_bits(p, tb1)) & 1u);
      if (carry_inside && ends) write_excl(p, y, carry_row, carry);
      else write_atom(p, y, carry_row, carry);
    }
  }
}

// k_nnz_warp, predicated-emit form: each lane scans its BMT with bmt_scan_pe (rows closed
// inside the BMT stored by one predicated store, no divergent writer calls), then the same
// warp combine of (cin, cout, head flag) as above.  Same writes as k_nnz_warp.
template <class V, int WRED, bool PAD, int VEC, int KB, int EM, bool XH>
__global__ void __launch_bounds__(AS_NWPE_LB) k_nnz_warp_pe(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  extern __shared__ __align__(128) unsigned char xh_smem[];
  if constexpr (XH) xhot_fill(p, x, (V*)xh_smem);
  using XA = std::conditional_t<XH, XHot<V>, XGlobal<V>>;
  XA xa;
  if constexpr (XH) xa = XHot<V>{x, (const V*)xh_smem};
  else xa = XGlobal<V>{x};
  for (int64_t w = warp_units(p.n_bmw).begin, w_e = warp_units(p.n_bmw).end; w < w_e; w += blockDim.x >> 5) {
    const int64_t tb0 = bmw_bmt_at(p, w);
    const int64_t tb1 = bmw_bmt_at(p, w + 1);
    double carry = 0.0;
    bool carry_inside = false;  // open segment's row started at a head inside this BMW
    bool carry_live = false;    // an open segment exists (false only before the first element)
    int64_t carry_row = 0;
    for (int64_t base = tb0; base < tb1; base += 32) {
      const int64_t t = base + lane;
      const bool active = t < tb1;
      const int nact = (int)min((int64_t)32, tb1 - base);
      double cin = 0.0, cout = 0.0;
      bool hh = false, b0 = false;
      int64_t head_row = 0;  // row of the first head in this lane
      int64_t last_row = 0;  // row of this lane's last element
      if (active) {
        PadPos pp{0, 0};
        if constexpr (PAD) {
          if (p.pad_grp_bmw) pp = PadPos{grp_base_at(p, w) + (t - tb0) * VEC, (tb1 - tb0) * VEC};
          else if (p.n_grp == 1) pp = PadPos{t * VEC, p.n_bmt * VEC};
          else pp = pad_pos<VEC>(p, t);
        }
        const ScanPE o = bmt_scan_pe<V, PAD, VEC, KB, EM, false>(p, y, xa, t, pp);
        b0 = o.s0;
        hh = o.inside;
        const int64_t row0 = bmt_row0(p, t);
        if (!o.s0) {
          cin = o.inside ? o.first : o.acc;  // continuation of a row begun in an earlier lane
          head_row = row0 + 1;
        } else {
          head_row = row0;
        }
        if (hh) cout = o.acc;
        last_row = o.row;
      }
      double v_end, closing;
      bool inside_end, closing_inside;
      warp_combine<WRED>(lane, hh, cin, cout, carry, carry_inside, closing, closing_inside, v_end, inside_end);
      if (active && hh) {
        // the row closed at this lane's first head; none only when the BMW itself starts
        // with a head (lane 0 of the first round, element 0 is a row start)
        const bool exists = !(lane == 0 && !carry_live && b0);
        if (exists) {
          if (closing_inside) write_excl(p, y, head_row - 1, closing);
          else write_atom(p, y, head_row - 1, closing);
        }
      }
      carry = __shfl_sync(0xffffffffu, v_end, nact - 1);
      carry_inside = __shfl_sync(0xffffffffu, (int)inside_end, nact - 1);
      carry_row = __shfl_sync(0xffffffffu, last_row, nact - 1);
      carry_live = true;
    }
    if (lane == 0 && carry_live) {
      // final open segment: the row of the BMW's last element
      const bool ends = (tb1 >= p.n_bmt) ? true : (ldm(bmt_bits(p, tb1)) & 1u);
      if (carry_inside && ends) write_excl(p, y, carry_row, carry);
      else write_atom(p, y, carry_row, carry);
    }
  }
}

// =====================================================================================
// FAM_WARP_ROW: single-row BMWs + WARP_TOTAL_RED (CSR-Vector).  Lanes stride over
// the BMW's nonzeros (coalesced), or over its BMT_NNZ(k) chunks with THREAD_TOTAL_RED;
// butterfly shuffle reduction; lane 0 writes.
// =====================================================================================
template <class V>
__global__ void __launch_bounds__(1024) k_warp_row(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const V* val = (const V*)p.val;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = gthreads() >> 5;
  for (int64_t w = warp_units(p.n_bmw).begin, w_e = warp_units(p.n_bmw).end; w < w_e; w += blockDim.x >> 5) {
    int64_t a = ldm(p.bmw_start + w), e = ldm(p.bmw_start + w + 1);
    int64_t row = p.bmw_first_row ? ldm(p.bmw_first_row + w) : w;
    double acc = 0.0;
    if (p.k <= 0) {
      for (int64_t i = a + lane; i < e; i += 32) acc += (double)ld_stream(val + i) * ldx(x, ld_stream(p.col + i));
    } else {
      for (int64_t c = a + lane * p.k; c < e; c += 32 * p.k) {
        int64_t ce = min(c + p.k, e);
        for (int64_t i = c; i < ce; ++i) acc += (double)ld_stream(val + i) * ldx(x, ld_stream(p.col + i));
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      bool excl = p.bmw_all_excl || (a == ldm(p.row_ptr + row) && e == ldm(p.row_ptr + row + 1));
      if (excl) write_excl(p, y, row, acc);
      else write_atom(p, y, row, acc);
    }
  }
}

// =====================================================================================
// FAM_BLOCK_TOTAL: single-row BMTBs + SHMEM_TOTAL_RED ("adds up all intermediate results
// of a thread block to a result"): CTA-wide sum, one store/atomic per CTA.
// =====================================================================================
template <class V>
__global__ void __launch_bounds__(1024) k_block_total(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  __shared__ double red[32];
  const V* val = (const V*)p.val;
  for (int64_t b = blockIdx.x; b < p.n_bmtb; b += gridDim.x) {
    int64_t a = p.bmtb_start ? ldm(p.bmtb_start + b) : b * p.k1;
    int64_t e = p.bmtb_start ? ldm(p.bmtb_start + b + 1) : min(a + p.k1, p.nnz_p);
    double acc = 0.0;
    for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x)
      acc += (double)ld_stream(val + i) * ldx(x, ld_stream(p.col + i));
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      s = warp_sum(s);
      if (threadIdx.x == 0) {
        int64_t row = ldm(p.bmtb_first_row + b);
        if (a == ldm(p.row_ptr + row) && e == ldm(p.row_ptr + row + 1)) write_excl(p, y, row, s);
        else write_atom(p, y, row, s);
      }
    }
    __syncthreads();
  }
}

// =====================================================================================
// FAM_BLOCK_OFFSET, TMA form: BMTB + SHMEM_OFFSET_RED with the block's values, columns and
// CSR row offsets ("reduce_row_offsets") staged into shared memory by bulk
// asynchronous copies (cp.async.bulk, SASS UBLKCP) that complete on an mbarrier.  Two
// stages: while the CTA reduces block b, the copies of its next block are in flight.
// Persistent grid; CTA c owns a contiguous range of BMTBs.
// =====================================================================================
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

template <class V>
__global__ void __launch_bounds__(1024) k_block_offset_tma(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  // smem per stage: val[cap] | col[cap] | rp[rcap]; then prod[cap] (double); then 2 mbarriers
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t cap = p.smem_cap, rcap = p.smem_rcap;  // elements (multiples of 4, +4 slack)
  const size_t stage_bytes = (size_t)cap * (sizeof(V) + 4) + (size_t)rcap * 4;
  double* prod = (double*)(smem_raw + 2 * stage_bytes);
  uint64_t* bars = (uint64_t*)(prod + cap);
  const V* val = (const V*)p.val;
  const int64_t per = (p.n_bmtb + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(b0 + per, p.n_bmtb);
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // block geometry: nonzeros [a, e), rows [r0, r1) intersecting it
  auto geom = [&](int64_t b, int64_t& a, int64_t& e, int64_t& r0, int64_t& r1) {
    a = p.bmtb_start ? ldm(p.bmtb_start + b) : b * p.k1;
    e = p.bmtb_start ? ldm(p.bmtb_start + b + 1) : min(a + p.k1, p.nnz_p);
    r0 = ldm(p.bmtb_first_row + b);
    r1 = b + 1 < p.n_bmtb ? ldm(p.bmtb_first_row + b + 1) + 1 : p.m_p;  // conservative (+1)
    if (r1 > p.m_p) r1 = p.m_p;
  };
  auto issue = [&](int64_t b, int st) {  // thread 0: copies of block b into stage st
    int64_t a, e, r0, r1;
    geom(b, a, e, r0, r1);
    const int64_t aa = a & ~int64_t(3), ea = (e + 3) & ~int64_t(3);
    const int64_t ra = r0 & ~int64_t(3), re = (r1 + 1 + 3) & ~int64_t(3);
    unsigned char* base = smem_raw + st * stage_bytes;
    const uint32_t bv = (uint32_t)((ea - aa) * sizeof(V)), bc = (uint32_t)((ea - aa) * 4), br = (uint32_t)((re - ra) * 4);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of this stage
    mbar_expect_tx(&bars[st], bv + bc + br);
    bulk_g2s(base, val + aa, bv, &bars[st]);
    bulk_g2s(base + cap * sizeof(V), p.col + aa, bc, &bars[st]);
    bulk_g2s(base + cap * (sizeof(V) + 4), p.row_ptr + ra, br, &bars[st]);
  };
  if (threadIdx.x == 0 && b0 < b1) issue(b0, 0);
  uint32_t phase[2] = {0, 0};
  for (int64_t b = b0; b < b1; ++b) {
    const int st = (int)((b - b0) & 1);
    if (threadIdx.x == 0 && b + 1 < b1) issue(b + 1, st ^ 1);
    int64_t a, e, r0, r1;
    geom(b, a, e, r0, r1);
    const int64_t aa = a & ~int64_t(3), ra = r0 & ~int64_t(3);
    const unsigned char* base = smem_raw + st * stage_bytes;
    const V* sv = (const V*)base;
    const int32_t* sc = (const int32_t*)(base + cap * sizeof(V));
    const int32_t* srp = (const int32_t*)(base + cap * (sizeof(V) + 4));
    mbar_wait(&bars[st], phase[st]);
    phase[st] ^= 1;
    for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x)
      prod[i - a] = (double)sv[i - aa] * ldx(x, sc[i - aa]);
    __syncthreads();
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      const int64_t ra_ = srp[r - ra];
      if (ra_ >= e) continue;
      const int64_t re_ = srp[r + 1 - ra];
      const int64_t fa = max(ra_, a), fe = min(re_, e);
      if (fe <= fa) continue;
      double s = 0.0;
      for (int64_t i = fa; i < fe; ++i) s += prod[i - a];
      if (fa == ra_ && fe == re_) write_excl(p, y, r, s);
      else write_atom(p, y, r, s);
    }
    __syncthreads();  // stage st and prod are free for reuse
  }
}

// =====================================================================================
// FAM_BLOCK_OFFSET: BMTB + SHMEM_OFFSET_RED (CSR-Stream).  The CTA stages the products of
// its nonzeros in shared memory (coalesced pass; the "adapter" of P:322 copying register
// results to shared memory), then reduces its row fragments in parallel using the CSR-like
// row offsets ("reduce_row_offsets") = the block's slice of row_ptr.
// =====================================================================================
template <class V>
__global__ void __launch_bounds__(1024) k_block_offset(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* prod = (double*)smem_raw;  // max_block_nnz products
  const V* val = (const V*)p.val;
  for (int64_t b = blockIdx.x; b < p.n_bmtb; b += gridDim.x) {
    int64_t a = p.bmtb_start ? ldm(p.bmtb_start + b) : b * p.k1;
    int64_t e = p.bmtb_start ? ldm(p.bmtb_start + b + 1) : min(a + p.k1, p.nnz_p);
    for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x)
      prod[i - a] = (double)ld_stream(val + i) * ldx(x, ld_stream(p.col + i));
    __syncthreads();
    int64_t r0 = ldm(p.bmtb_first_row + b);
    for (int64_t r = r0 + threadIdx.x; r < p.m_p; r += blockDim.x) {
      int64_t ra = ldm(p.row_ptr + r);
      if (ra >= e) break;
      int64_t re = ldm(p.row_ptr + r + 1);
      int64_t fa = max(ra, a), fe = min(re, e);
      double s = 0.0;
      for (int64_t i = fa; i < fe; ++i) s += prod[i - a];
      if (fa == ra && fe == re) write_excl(p, y, r, s);
      else write_atom(p, y, r, s);
    }
    __syncthreads();
  }
}

// =====================================================================================
// FAM_DIA: y_r = sum_d dia_val[d*stride + i] * x[r + off_d]  (DIA root format).
// Each thread owns R = 32 B / sizeof(V) consecutive rows: one 256-bit load per diagonal
// (sm_100 `ld.global.nc.L2::evict_first.v4.b64` / `.v8.b32`), all D diagonals issued before
// the first FMA (D templated for D <= 8) so 32*D bytes per thread are in flight; offsets
// live in the kernel parameter space (constant bank); x gathers hit L1 (the +-1 diagonals
// reuse the lines of the main diagonal).
// =====================================================================================
template <class V>
struct Ld32;
template <>
struct Ld32<double> {
  static constexpr int R = 4;
  static __device__ __forceinline__ void ld(const double* p, double* o) {
    unsigned long long a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
    o[0] = __longlong_as_double((long long)a);
    o[1] = __longlong_as_double((long long)b);
    o[2] = __longlong_as_double((long long)c);
    o[3] = __longlong_as_double((long long)d);
  }
};
template <>
struct Ld32<float> {
  static constexpr int R = 8;
  static __device__ __forceinline__ void ld(const float* p, double* o) {
    unsigned r[8];
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = (double)__int_as_float((int)r[q]);
  }
};

template <class V, int R>
__device__ __forceinline__ void dia_rows_fma(const DevPart& p, const V* __restrict__ x, int64_t r, int64_t o,
                                             const double* v, double* acc) {
  if (r + o >= 0 && r + o + R <= p.n) {  // interior: no bounds checks
#pragma unroll
    for (int q = 0; q < R; ++q) acc[q] += v[q] * ldx(x, r + q + o);
  } else {
#pragma unroll
    for (int q = 0; q < R; ++q) {
      int64_t c = r + q + o;
      if (c >= 0 && c < p.n) acc[q] += v[q] * ldx(x, c);
    }
  }
}

template <class V, int BYTES>
struct LdN;
template <class V>
struct LdN<V, 32> {
  static constexpr int R = Ld32<V>::R;
  static __device__ __forceinline__ void ld(const V* p, double* o) { Ld32<V>::ld(p, o); }
};
template <>
struct LdN<double, 16> {
  static constexpr int R = 2;
  static __device__ __forceinline__ void ld(const double* p, double* o) {
    double2 t = ld_stream2(p);
    o[0] = t.x;
    o[1] = t.y;
  }
};
template <class V>
struct LdN<V, 8> {  // one row per thread (variant 3: <= 32 registers, 2048 resident threads/SM)
  static constexpr int R = sizeof(V) == 8 ? 1 : 2;
  static __device__ __forceinline__ void ld(const V* p, double* o) {
    if constexpr (sizeof(V) == 8) {
      o[0] = ld_stream(p);
    } else {
      float2 t = ld_stream2(p);
      o[0] = t.x;
      o[1] = t.y;
    }
  }
};
template <>
struct LdN<float, 16> {
  static constexpr int R = 4;
  static __device__ __forceinline__ void ld(const float* p, double* o) {
    float4 t = ld_stream4(p);
    o[0] = t.x;
    o[1] = t.y;
    o[2] = t.z;
    o[3] = t.w;
  }
};

template <class V, int DT, int BYTES>
__global__ void __launch_bounds__(1024, BYTES == 8 ? 2 : 1) k_dia(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  constexpr int R = LdN<V, BYTES>::R;
  const V* dv = (const V*)p.dia_val;
  for (int64_t i0 = gtid() * R; i0 < p.mb; i0 += gthreads() * R) {
    double acc[R];
#pragma unroll
    for (int q = 0; q < R; ++q) acc[q] = 0.0;
    const int64_t r = p.r0 + i0;
    if constexpr (DT > 0) {
      double v[DT][R];
#pragma unroll
      for (int d = 0; d < DT; ++d) LdN<V, BYTES>::ld(dv + d * p.dia_stride + i0, v[d]);
#pragma unroll
      for (int d = 0; d < DT; ++d) dia_rows_fma<V, R>(p, x, r, p.dia_off[d], v[d], acc);
    } else {
#pragma unroll 2
      for (int d = 0; d < p.D; ++d) {
        double v[R];
        LdN<V, BYTES>::ld(dv + d * p.dia_stride + i0, v);
        dia_rows_fma<V, R>(p, x, r, p.dia_off[d], v, acc);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (i0 + q < p.mb) write_excl(p, y, i0 + q, acc[q]);
  }
}

// =====================================================================================
// FAM_DENSE, b = 64, fp64: one warp per tile row; half-warp h takes tile columns j = h,
// h+2, ...; lane owns 4 consecutive tile rows and reads them with one 256-bit load per
// column (a half-warp reads one whole 512-byte column), 4 columns in flight; the halves
// combine with one shuffle.
// =====================================================================================
template <class V>
__global__ void __launch_bounds__(1024) k_dense64(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const double* tv = (const double*)p.tile_val;
  const int lane = threadIdx.x & 31, half = lane >> 4, r4 = (lane & 15) * 4;
  for (int64_t tr = warp_units(p.n_tile_rows).begin, tr_e = warp_units(p.n_tile_rows).end; tr < tr_e;
       tr += blockDim.x >> 5) {
    const int64_t I = ldm(p.tile_row_id + tr);
    const int64_t t0 = ldm(p.tile_row_ptr + tr), t1 = ldm(p.tile_row_ptr + tr + 1);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t J = ldm(p.tile_col + t);
      const double* tile = tv + t * 4096 + r4;
      const bool full = J * 64 + 64 <= p.n;
#pragma unroll 4
      for (int j = half; j < 64; j += 2) {
        double v[4];
        Ld32<double>::ld(tile + j * 64, v);
        const int64_t c = J * 64 + j;
        const double xj = (full || c < p.n) ? ldx((const V*)x, c) : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += v[q] * xj;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 16);
    if (half == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t row = I * 64 + r4 + q;
        if (row >= p.row_lo && row < p.row_hi) write_excl(p, y, row, acc[q]);
      }
    }
  }
}

// =====================================================================================
// FAM_DENSE: BSR-like b x b tiles (column-major) of DENSE_DECOM.  One warp per tile row;
// lane owns rows i = lane + 32q; for each tile column j the warp reads b contiguous values
// (coalesced) and one broadcast x element.  CUDA cores: a single right-hand side makes
// every tile a GEMV, not a contraction.
// =====================================================================================
template <class V, int RPL>
__global__ void __launch_bounds__(1024) k_dense(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  const V* tv = (const V*)p.tile_val;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = gthreads() >> 5;
  const int64_t b = p.b, bb = b * b;
  for (int64_t tr = gtid() >> 5; tr < p.n_tile_rows; tr += nwarps) {
    int64_t I = ldm(p.tile_row_id + tr);
    int64_t t0 = ldm(p.tile_row_ptr + tr), t1 = ldm(p.tile_row_ptr + tr + 1);
    double acc[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) acc[q] = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
      int64_t J = ldm(p.tile_col + t);
      const V* tile = tv + t * bb;
#pragma unroll 4
      for (int64_t j = 0; j < b; ++j) {
        int64_t c = J * b + j;
        double xj = c < p.n ? ldx(x, c) : 0.0;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          int64_t i = lane + 32 * q;
          if (i < b) acc[q] += (double)ld_stream(tile + j * b + i) * xj;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      int64_t i = lane + 32 * q;
      int64_t row = I * b + i;
      if (i < b && row >= p.row_lo && row < p.row_hi) write_excl(p, y, row, acc[q]);
    }
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int64_t grid_for(const DevPart& p, int64_t units, int64_t units_per_cta) {
  int64_t g = (units + units_per_cta - 1) / units_per_cta;
  if (p.grid > 0) return std::min<int64_t>((int64_t)p.grid * sm_count(), std::max<int64_t>(g, 1));
  // grid = 0 (auto): streaming DIA runs persistent, 2048 resident threads per SM (C2 sweep:
  // 40.0 us persistent vs 42.0 us one-pass grid)
  if (p.fam == FAM_DIA) g = std::min<int64_t>(g, (int64_t)sm_count() * (2048 / p.tpb));
  if (g < 1) g = 1;
  if (g > (int64_t(1) << 31) - 1) g = (int64_t(1) << 31) - 1;
  return g;
}

}  // namespace

// Launch groups: each is explicitly instantiated per value type in its own translation unit
// (kernels_*.cu), so the kernel family compiles in parallel.
template <class V>
int launch_grp_nnz_thread(const DevPart& p, const V* x, V* y, cudaStream_t s) {
  const int tpb = p.tpb > 0 ? p.tpb : 256;
  (void)tpb;
  switch (p.fam) {
    case FAM_NNZ_THREAD: {
      if (p.xwin) {
        const int64_t g = p.xw_grid;
        const bool pex = p.variant != 9 && !(sizeof(V) == 4 && p.n_heavy && p.mode == 1);
#define AS_XW(PADV, VECV)                                                          \
  {                                                                                \
    if (!pex) k_nnz_thread_xw<V, PADV, VECV, -1><<<g, tpb, p.smem, s>>>(p, x, y);  \
    else k_nnz_thread_xw<V, PADV, VECV, 1><<<g, tpb, p.smem, s>>>(p, x, y);        \
  }
        if (!p.pad) AS_XW(false, 1)
        else if (p.vec == 1) AS_XW(true, 1)
        else if (p.vec == 2) AS_XW(true, 2)
        else AS_XW(true, 4)
#undef AS_XW
        break;
      }
      int64_t g = grid_for(p, p.n_bmt, tpb);
      const int tt = tpb;
      // batches of KB loads per thread: 8 for fp64, 4 for fp32 (A/B on c5s fp64: KB 4 633 vs
      // KB 8 646 GF/s; c3s fp32: 408 vs 394; KB 16 or 80 registers slower everywhere)
      // predicated-emit form unless exclusive rows may need the fp32 heavy-row scratch
      // (write_excl consults it in ADD mode only), or the legacy form is forced for A/B
      // timing (variant 9)
      const bool pe = p.variant != 9 && !(sizeof(V) == 4 && p.n_heavy && p.mode == 1);
      const bool em0 = p.mode == 0 && p.beta == 0.0 && !p.origin && !p.org_model.kind;
      const int64_t gx = std::min<int64_t>(g, (int64_t)std::max(1, p.xh_ctas) * sm_count());  // xcache: persistent
#define AS_NT(PADV, VECV)                                                                                 \
  {                                                                                                       \
    constexpr int KBV = sizeof(V) == 4 && VECV <= 4 ? 4 : 8;                                              \
    if (!pe) k_nnz_thread<V, PADV, VECV, KBV><<<g, tt, 0, s>>>(p, x, y);                                  \
    else if (p.xh_n && em0) k_nnz_thread_pe<V, PADV, VECV, KBV, 0, true><<<gx, tt, p.smem, s>>>(p, x, y);   \
    else if (p.xh_n) k_nnz_thread_pe<V, PADV, VECV, KBV, 1, true><<<gx, tt, p.smem, s>>>(p, x, y);          \
    else if (em0) k_nnz_thread_pe<V, PADV, VECV, KBV, 0, false><<<g, tt, 0, s>>>(p, x, y);                 \
    else k_nnz_thread_pe<V, PADV, VECV, KBV, 1, false><<<g, tt, 0, s>>>(p, x, y);                          \
  }
      if (!p.pad) {
        AS_NT(false, 1)
      } else if (p.vec == 1) {
        AS_NT(true, 1)
      } else if (p.vec == 2) {
        AS_NT(true, 2)
      } else {
        AS_NT(true, 4)
      }
#undef AS_NT
      break;
    }
    default:
      return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

template <class V>
int launch_grp_nnz_warp(const DevPart& p, const V* x, V* y, cudaStream_t s) {
  const int tpb = p.tpb > 0 ? p.tpb : 256;
  (void)tpb;
  switch (p.fam) {
    case FAM_NNZ_WARP: {
      int64_t g = grid_for(p, p.n_bmw, tpb / 32);
      if (p.tile) {
        const int tt = tpb > 512 ? 512 : tpb;  // launch bound of k_warp_tile
        g = grid_for(p, p.n_bmw, tt / 32);
#define AS_TILE(KL)                                                                 \
  if (p.variant == 1) k_warp_tile<V, KL, 1><<<g, tt, 0, s>>>(p, x, y);             \
  else k_warp_tile<V, KL, 2><<<g, tt, 0, s>>>(p, x, y);
        if (p.k == 1) {
          AS_TILE(1)
        } else if (p.k == 2) {
          AS_TILE(2)
        } else {
          AS_TILE(4)
        }
#undef AS_TILE
        break;
      }
      // predicated-emit form unless fp32 ADD-mode heavy rows need the scratch path, or the
      // legacy form is forced (variant + 8: AS_NT_LEGACY)
      const bool pe = p.variant < 8 && !(sizeof(V) == 4 && p.n_heavy && p.mode == 1);
      const bool em0 = p.mode == 0 && p.beta == 0.0 && !p.origin && !p.org_model.kind;
      const int64_t gx = std::min<int64_t>(g, (int64_t)std::max(1, p.xh_ctas) * sm_count());  // xcache: persistent
      constexpr int KBW = kbw_of<V>();
#define AS_NWPE(WR, PADV, VECV)                                                                  \
  {                                                                                              \
    if (p.xh_n && em0) k_nnz_warp_pe<V, WR, PADV, VECV, (KBW > VECV ? KBW : VECV), 0, true><<<gx, tpb, p.smem, s>>>(p, x, y); \
    else if (p.xh_n) k_nnz_warp_pe<V, WR, PADV, VECV, (KBW > VECV ? KBW : VECV), 1, true><<<gx, tpb, p.smem, s>>>(p, x, y);   \
    else if (em0) k_nnz_warp_pe<V, WR, PADV, VECV, (KBW > VECV ? KBW : VECV), 0, false><<<g, tpb, 0, s>>>(p, x, y);           \
    else k_nnz_warp_pe<V, WR, PADV, VECV, (KBW > VECV ? KBW : VECV), 1, false><<<g, tpb, 0, s>>>(p, x, y);                    \
  }
#define AS_NW(WR)                                                              \
  if (pe) {                                                                    \
    if (!p.pad) AS_NWPE(WR, false, 1)                                          \
    else if (p.vec == 1) AS_NWPE(WR, true, 1)                                  \
    else if (p.vec == 2) AS_NWPE(WR, true, 2)                                  \
    else AS_NWPE(WR, true, 4)                                                  \
  } else if (!p.pad) k_nnz_warp<V, WR, false, 1><<<g, tpb, 0, s>>>(p, x, y);   \
  else if (p.vec == 1) k_nnz_warp<V, WR, true, 1><<<g, tpb, 0, s>>>(p, x, y);  \
  else if (p.vec == 2) k_nnz_warp<V, WR, true, 2><<<g, tpb, 0, s>>>(p, x, y);  \
  else k_nnz_warp<V, WR, true, 4><<<g, tpb, 0, s>>>(p, x, y);
      if ((p.variant & 7) == 1) {
        AS_NW(1)
      } else {
        AS_NW(2)
      }
#undef AS_NW
#undef AS_NWPE
      break;
    }
    default:
      return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

template <class V>
int launch_grp_other(const DevPart& p, const V* x, V* y, cudaStream_t s) {
  const int tpb = p.tpb > 0 ? p.tpb : 256;
  (void)tpb;
  switch (p.fam) {
    case FAM_THREAD_ROW:
      if (!p.pad) {
        k_thread_row<V><<<grid_for(p, p.n_bmt, tpb), tpb, 0, s>>>(p, x, y);
      } else {
        int64_t g = grid_for(p, p.n_bmt, tpb);
        if (p.vec == 1) k_thread_row_pad<V, 1><<<g, tpb, 0, s>>>(p, x, y);
        else if (p.vec == 2) k_thread_row_pad<V, 2><<<g, tpb, 0, s>>>(p, x, y);
        else k_thread_row_pad<V, 4><<<g, tpb, 0, s>>>(p, x, y);
      }
      break;
    case FAM_WARP_ROW:
      k_warp_row<V><<<grid_for(p, p.n_bmw, tpb / 32), tpb, 0, s>>>(p, x, y);
      break;
    case FAM_BLOCK_TOTAL:
      k_block_total<V><<<grid_for(p, p.n_bmtb, 1), tpb, 0, s>>>(p, x, y);
      break;
    case FAM_BLOCK_OFFSET:
      if (p.variant == 1) k_block_offset_tma<V><<<grid_for(p, p.n_bmtb, 1), tpb, p.smem, s>>>(p, x, y);
      else k_block_offset<V><<<grid_for(p, p.n_bmtb, 1), tpb, p.smem, s>>>(p, x, y);
      break;
    case FAM_DIA: {
      // variant 3 (default): 8-byte loads, one fp64 row per thread, <= 32 registers -> 2048
      // resident threads per SM (C2: 35.9 us); 0: 16-byte row pairs, 64 registers (42.0 us);
      // 1: 32-byte (sm_100 256-bit loads, 46-48 us)
      const int R = p.variant == 1 ? LdN<V, 32>::R : LdN<V, 16>::R;
      int64_t g = grid_for(p, (p.mb + R - 1) / R, tpb);
      const int64_t g3 = grid_for(p, (p.mb + LdN<V, 8>::R - 1) / LdN<V, 8>::R, tpb);
#define AS_DIA_CASE(K)                                                          \
  case K:                                                                       \
    if (p.variant == 1) k_dia<V, K, 32><<<g, tpb, 0, s>>>(p, x, y);            \
    else if (p.variant == 3) k_dia<V, K, 8><<<g3, tpb, 0, s>>>(p, x, y);       \
    else k_dia<V, K, 16><<<g, tpb, 0, s>>>(p, x, y);                           \
    break;
      switch (p.D) {
        AS_DIA_CASE(1) AS_DIA_CASE(2) AS_DIA_CASE(3) AS_DIA_CASE(4)
        AS_DIA_CASE(5) AS_DIA_CASE(6) AS_DIA_CASE(7) AS_DIA_CASE(8)
        default:
          if (p.variant == 1) k_dia<V, 0, 32><<<g, tpb, 0, s>>>(p, x, y);
          else k_dia<V, 0, 16><<<g, tpb, 0, s>>>(p, x, y);
      }
#undef AS_DIA_CASE
      break;
    }
    case FAM_DENSE: {
      int64_t g = grid_for(p, p.n_tile_rows, tpb / 32);
      int rpl = (int)((p.b + 31) / 32);
      if constexpr (sizeof(V) == 8) {
        if (p.b == 64) {
          k_dense64<V><<<g, tpb, 0, s>>>(p, x, y);
          break;
        }
      }
      if (rpl <= 1) k_dense<V, 1><<<g, tpb, 0, s>>>(p, x, y);
      else if (rpl == 2) k_dense<V, 2><<<g, tpb, 0, s>>>(p, x, y);
      else if (rpl <= 4) k_dense<V, 4><<<g, tpb, 0, s>>>(p, x, y);
      else return (int)cudaErrorInvalidValue;
      break;
    }
    default:
      return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

namespace {
// xcache (R-xcache): opt the XH instantiations the launch may pick (EM 0 / 1) in to `smem`
// bytes of dynamic shared memory; returns the CTAs per SM they reach (0 on failure)
template <class K>
int xh_optin(K kern, size_t smem, int tpb) {
  if (smem_optin(kern, smem) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, tpb, smem) != cudaSuccess) return 0;
  return n;
}
template <class V, bool PAD, int VEC>
int xh_prep_thread(size_t smem, int tpb) {
  constexpr int KB = sizeof(V) == 4 && VEC <= 4 ? 4 : 8;
  return std::min(xh_optin(k_nnz_thread_pe<V, PAD, VEC, KB, 0, true>, smem, tpb),
                  xh_optin(k_nnz_thread_pe<V, PAD, VEC, KB, 1, true>, smem, tpb));
}
template <class V, int WR, bool PAD, int VEC>
int xh_prep_warp(size_t smem, int tpb) {
  constexpr int KB = kbw_of<V>() > VEC ? kbw_of<V>() : VEC;
  return std::min(xh_optin(k_nnz_warp_pe<V, WR, PAD, VEC, KB, 0, true>, smem, tpb),
                  xh_optin(k_nnz_warp_pe<V, WR, PAD, VEC, KB, 1, true>, smem, tpb));
}
}  // namespace

// xcache opt-in of the group's XH instantiations (R-xcache); CTAs per SM they reach (0 = fail)
template <class V>
int prep_grp_nnz_thread_xh(const DevPart& p, size_t smem, int tpb) {
  if (!p.pad) return xh_prep_thread<V, false, 1>(smem, tpb);
  if (p.vec == 1) return xh_prep_thread<V, true, 1>(smem, tpb);
  if (p.vec == 2) return xh_prep_thread<V, true, 2>(smem, tpb);
  return xh_prep_thread<V, true, 4>(smem, tpb);
}
template <class V>
int prep_grp_nnz_warp_xh(const DevPart& p, size_t smem, int tpb) {
  if ((p.variant & 7) == 1) {
    if (!p.pad) return xh_prep_warp<V, 1, false, 1>(smem, tpb);
    if (p.vec == 1) return xh_prep_warp<V, 1, true, 1>(smem, tpb);
    if (p.vec == 2) return xh_prep_warp<V, 1, true, 2>(smem, tpb);
    return xh_prep_warp<V, 1, true, 4>(smem, tpb);
  }
  if (!p.pad) return xh_prep_warp<V, 2, false, 1>(smem, tpb);
  if (p.vec == 1) return xh_prep_warp<V, 2, true, 1>(smem, tpb);
  if (p.vec == 2) return xh_prep_warp<V, 2, true, 2>(smem, tpb);
  return xh_prep_warp<V, 2, true, 4>(smem, tpb);
}

// x-window kernel: opt in to `smem` bytes of dynamic shared memory and return how many
// CTAs of `tpb` threads fit per SM (0 on failure).
template <class V>
int xw_occ_t(int pad, int vec, int tpb, size_t smem) {
  auto occ = [&](auto kern) {
    if (smem_optin(kern, smem) != cudaSuccess) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, tpb, smem) != cudaSuccess) return 0;
    return n;
  };
  // both forms (branching -1, predicated-emit 1) get the shared-memory opt-in; the smaller
  // occupancy of the two decides the grid
  auto both = [&](auto k0, auto k1) { return std::min(occ(k0), occ(k1)); };
  if (!pad) return both(k_nnz_thread_xw<V, false, 1, -1>, k_nnz_thread_xw<V, false, 1, 1>);
  if (vec == 1) return both(k_nnz_thread_xw<V, true, 1, -1>, k_nnz_thread_xw<V, true, 1, 1>);
  if (vec == 2) return both(k_nnz_thread_xw<V, true, 2, -1>, k_nnz_thread_xw<V, true, 2, 1>);
  return both(k_nnz_thread_xw<V, true, 4, -1>, k_nnz_thread_xw<V, true, 4, 1>);
}
// CSR-stream shared-memory opt-in (FAM_BLOCK_OFFSET); returns cudaError_t, sets p.grid for TMA
template <class V>
int prep_grp_block_offset(DevPart& p) {
  if (p.variant == 1) {  // TMA-staged CSR-stream
    cudaError_t e = smem_optin(k_block_offset_tma<V>, p.smem);
    if (e != cudaSuccess) return (int)e;
    int per_sm = 0;
    const int tpb = p.tpb > 0 ? p.tpb : 256;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_block_offset_tma<V>, tpb, p.smem);
    if (e != cudaSuccess) return (int)e;
    if (per_sm < 1) return (int)cudaErrorInvalidConfiguration;
    if (p.grid <= 0) p.grid = per_sm;  // persistent: every resident CTA slot, CTA-blocked ranges
    else if (p.grid > per_sm) p.grid = per_sm;
    return 0;
  }
  return p.smem > 48 * 1024 ? (int)smem_optin(k_block_offset<V>, p.smem) : 0;
}

#define AS_KERNELS_INSTANTIATE_NNZ_THREAD(V)                                                   \
  template int launch_grp_nnz_thread<V>(const DevPart&, const V*, V*, cudaStream_t);           \
  template int prep_grp_nnz_thread_xh<V>(const DevPart&, size_t, int);                         \
  template int xw_occ_t<V>(int, int, int, size_t);
#define AS_KERNELS_INSTANTIATE_NNZ_WARP(V)                                                     \
  template int launch_grp_nnz_warp<V>(const DevPart&, const V*, V*, cudaStream_t);             \
  template int prep_grp_nnz_warp_xh<V>(const DevPart&, size_t, int);
#define AS_KERNELS_INSTANTIATE_OTHER(V)                                                        \
  template int launch_grp_other<V>(const DevPart&, const V*, V*, cudaStream_t);                \
  template int prep_grp_block_offset<V>(DevPart&);

}  // namespace as
