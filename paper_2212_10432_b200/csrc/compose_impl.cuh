// FAM_COMPOSE: every mapping/reduction combination the implementing stage admits that no
// specialised family of kernels.cu covers -- the paper's Kernel Builder splicing one code
// fragment per level (Fig. 5, §V-C).  Levels (BMTB, BMW, BMT) are optional,
// each ROW or NNZ blocked with children restarting at every parent (A15); each may carry its
// reduction or none:
//   thread  THREAD_TOTAL_RED | THREAD_BITMAP_RED_G | none   -> a serial pass over the BMT
//           cutting at row heads (TOTAL is the single-row case, P1); rows that close inside
//           the BMT are complete
//   warp    WARP_TOTAL_RED (butterfly) | WARP_SEG_ADD_RED / WARP_BITMAP_RED (segmented
//           combine of the lanes' boundary partials, warp_combine) | none
//   block   SHMEM_TOTAL_RED (CTA-wide sum) | SHMEM_OFFSET_RED | none
// SHMEM_OFFSET_RED over child levels uses the Adapter of P:322 ("copies register results
// into shared memory"): every partial a lower level produces -- a thread's complete rows,
// its boundary partials, a warp's combined rows -- is stored at the shared-memory slot of
// the partial's LAST nonzero (slots of distinct segments never collide), the other slots
// stay 0, and the block then sums each row's slot range (its CSR-like row offsets)
// and writes it once.  Without a block reduction a level's partials go to y under the
// writer rule (A22): rows complete inside a unit of the coarsest reduction level are stored
// (STORE / ADD mode), the others added atomically (GMEM_ATOM_RED).  A level without its own
// reduction forwards its children's partials; the kernel pre-adds one thread's consecutive
// same-row products in registers (a re-association of the same sum, reading R-compose).
// With no reduction below GMEM at all every nonzero is written on its own (per_elem).
//
// Row heads come from a packed bitmap (bit e = nonzero e starts its row), rows from the
// BMT's first row plus the heads seen, so ROW and NNZ blocks are handled alike.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "devpart.h"
#include "kcommon.cuh"

namespace as {
namespace {

__device__ __forceinline__ bool is_head(const DevPart& p, int64_t e) {
  return e >= p.nnz_p ? true : ((ldm(p.bits + (e >> 5)) >> (e & 31)) & 1u);
}
__device__ __forceinline__ int64_t c_bmt_start(const DevPart& p, int64_t t) {
  return p.bmt_start ? (int64_t)ldm(p.bmt_start + t) : min(t * p.k, p.nnz_p);
}

// runtime-vec slot position of BMT t in the BMT_PAD layout (A18)
__device__ __forceinline__ PadPos pad_pos_rt(const DevPart& p, int64_t t) {
  int64_t g, t0, t1;
  if (p.grp_regular) {
    g = t / p.grp_regular;
    t0 = g * p.grp_regular;
    t1 = min(t0 + p.grp_regular, p.n_bmt);
  } else {
    int64_t lo = 0, hi = p.n_grp - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (ldm(p.grp_first_bmt + mid) <= t) lo = mid;
      else hi = mid - 1;
    }
    g = lo;
    t0 = ldm(p.grp_first_bmt + g);
    t1 = ldm(p.grp_first_bmt + g + 1);
  }
  return {grp_base_at(p, g) + (t - t0) * p.vec, (t1 - t0) * p.vec};
}

// One BMT's serial pass: summary of its boundary segments; rows closing strictly inside
// (between two heads of this BMT) go to emit(row, value, last_nonzero).
struct CSeg {
  double cin = 0.0, cout = 0.0;  // before the first head / from the last head
  int64_t fh = 0;                // first head (global nonzero index), valid when hh
  int32_t row0 = 0, row_last = 0;
  bool hh = false, h0 = false;   // any head in the BMT / element 0 is a head
};

template <class V, bool PAD, class Emit>
__device__ __forceinline__ CSeg scan_bmt(const DevPart& p, const V* __restrict__ x, int64_t t, int64_t a, int64_t e,
                                         PadPos pp, Emit emit) {
  constexpr int KB = 4;
  const V* val = PAD ? (const V*)p.pad_val : (const V*)p.val;
  const int32_t* col = PAD ? p.pad_col : p.col;
  CSeg o;
  o.row0 = (int32_t)bmt_row0(p, t);
  int32_t row = o.row0;
  double cur = 0.0;
  const int len = (int)(e - a);
  for (int j0 = 0; j0 < len; j0 += KB) {
    double v[KB], xv[KB];
    int32_t c[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int j = j0 + q;
      if (j < len) {
        const int64_t s = PAD ? pp.base + (int64_t)(j / p.vec) * pp.stride + (j % p.vec) : a + j;
        v[q] = (double)ld_seq(val + s);
        c[q] = ld_seq(col + s);
      } else {
        v[q] = 0.0;
        c[q] = 0;
      }
    }
#pragma unroll
    for (int q = 0; q < KB; ++q) xv[q] = j0 + q < len ? ldx(x, c[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int j = j0 + q;
      if (j >= len) break;
      if (is_head(p, a + j)) {
        if (!o.hh) {
          o.cin = cur;
          o.fh = a + j;
          o.hh = true;
        } else {
          emit(row, cur, a + j - 1);
        }
        if (j > 0) ++row;
        cur = 0.0;
      }
      cur += v[q] * xv[q];
    }
  }
  if (o.hh) o.cout = cur;
  else o.cin = cur;
  o.row_last = row;
  o.h0 = len > 0 && is_head(p, a);
  return o;
}

// per_elem: no reduction below GMEM -- every product is its own partial (A22: a nonzero is
// exclusive iff its row has length 1)
template <class V, bool PAD>
__device__ __forceinline__ void elems_bmt(const DevPart& p, const V* __restrict__ x, V* __restrict__ y, int64_t t,
                                          int64_t a, int64_t e, PadPos pp) {
  const V* val = PAD ? (const V*)p.pad_val : (const V*)p.val;
  const int32_t* col = PAD ? p.pad_col : p.col;
  int32_t row = (int32_t)bmt_row0(p, t);
  for (int64_t j = 0; j < e - a; ++j) {
    const int64_t s = PAD ? pp.base + (j / p.vec) * pp.stride + (j % p.vec) : a + j;
    const bool h = is_head(p, a + j);
    if (h && j > 0) ++row;
    const double prod = (double)ld_seq(val + s) * ldx(x, ld_seq(col + s));
    if (h && is_head(p, a + j + 1)) write_excl(p, y, row, prod);
    else write_atom(p, y, row, prod);
  }
}

// Where a partial goes: BR 0 = y (writer rule), 1 = CTA total, 2 = shared-memory slot of
// its last nonzero (the Adapter of P:322)
template <class V, int BR>
struct Sink {
  const DevPart& p;
  V* __restrict__ y;
  double* slots;  // BR == 2: slots of the current BMTB, relative to ua
  int64_t ua;
  double tot;
  __device__ __forceinline__ void row(int32_t r, double v, int64_t last) {  // a complete row
    if constexpr (BR == 2) slots[last - ua] = v;
    else if constexpr (BR == 1) tot += v;
    else write_excl(p, y, r, v);
  }
  __device__ __forceinline__ void bnd(int32_t r, double v, int64_t last, bool excl) {  // boundary partial
    if constexpr (BR == 2) slots[last - ua] = v;
    else if constexpr (BR == 1) tot += v;
    else if (excl) write_excl(p, y, r, v);
    else write_atom(p, y, r, v);
  }
};

template <class V, bool PAD>
__device__ __forceinline__ PadPos c_pad(const DevPart& p, int64_t t, int64_t w, int64_t tb0, int64_t tb1) {
  PadPos pp{0, 0};
  if constexpr (PAD) {
    if (p.pad_grp_bmw) pp = PadPos{grp_base_at(p, w) + (t - tb0) * p.vec, (tb1 - tb0) * p.vec};
    else if (p.n_grp == 1) pp = PadPos{t * p.vec, p.n_bmt * p.vec};
    else pp = pad_pos_rt(p, t);
  }
  return pp;
}

// A BMT whose partials leave the thread level directly (no warp reduction above it).
template <class V, bool PAD, int BR>
__device__ __forceinline__ void thread_bmt(const DevPart& p, const V* __restrict__ x, Sink<V, BR>& sk, int64_t t,
                                           PadPos pp) {
  const int64_t a = c_bmt_start(p, t), e = c_bmt_start(p, t + 1);
  if (p.per_elem) {
    elems_bmt<V, PAD>(p, x, sk.y, t, a, e, pp);
    return;
  }
  const CSeg o = scan_bmt<V, PAD>(p, x, t, a, e, pp, [&](int32_t r, double v, int64_t last) { sk.row(r, v, last); });
  if (o.hh && !o.h0) sk.bnd(o.row0, o.cin, o.fh - 1, false);  // row begun before the BMT
  // last segment: exclusive iff it began at a head here and the next nonzero starts a row
  sk.bnd(o.row_last, o.hh ? o.cout : o.cin, e - 1, o.hh && is_head(p, e));
}

template <class V, bool PAD, int WR, int BR>
__device__ __forceinline__ void warp_bmw(const DevPart& p, const V* __restrict__ x, Sink<V, BR>& sk, int64_t w,
                                         int lane) {
  const int64_t tb0 = bmw_bmt_at(p, w);
  const int64_t tb1 = bmw_bmt_at(p, w + 1);
  if (tb1 <= tb0) return;
  const int64_t wa = c_bmt_start(p, tb0), we = c_bmt_start(p, tb1);
  if constexpr (WR == RED_NONE) {
    for (int64_t t = tb0 + lane; t < tb1; t += 32) thread_bmt<V, PAD, BR>(p, x, sk, t, c_pad<V, PAD>(p, t, w, tb0, tb1));
    return;
  } else if constexpr (WR == RED_TOTAL) {
    // single-row BMW (P1): butterfly sum of every lane's partial (WARP_TOTAL_RED)
    double acc = 0.0;
    for (int64_t t = tb0 + lane; t < tb1; t += 32) {
      const int64_t a = c_bmt_start(p, t), e = c_bmt_start(p, t + 1);
      const CSeg o = scan_bmt<V, PAD>(p, x, t, a, e, c_pad<V, PAD>(p, t, w, tb0, tb1),
                                      [&](int32_t, double v, int64_t) { acc += v; });
      acc += o.cin + o.cout;
    }
    acc = warp_sum(acc);
    if (lane == 0) sk.bnd((int32_t)bmt_row0(p, tb0), acc, we - 1, is_head(p, wa) && is_head(p, we));
  } else {
    // WARP_SEG_ADD_RED / WARP_BITMAP_RED: lanes' boundary partials combined in lane order
    double carry = 0.0;
    bool carry_inside = false, carry_live = false;
    int32_t carry_row = 0;
    for (int64_t base = tb0; base < tb1; base += 32) {
      const int64_t t = base + lane;
      const bool active = t < tb1;
      const int nact = (int)min((int64_t)32, tb1 - base);
      CSeg o;
      if (active) {
        const int64_t a = c_bmt_start(p, t), e = c_bmt_start(p, t + 1);
        o = scan_bmt<V, PAD>(p, x, t, a, e, c_pad<V, PAD>(p, t, w, tb0, tb1),
                             [&](int32_t r, double v, int64_t last) { sk.row(r, v, last); });
      }
      double v_end, closing;
      bool inside_end, closing_inside;
      warp_combine<WR == RED_SEG ? 1 : 2>(lane, o.hh, o.cin, o.cout, carry, carry_inside, closing, closing_inside,
                                          v_end, inside_end);
      if (active && o.hh) {
        // the row closed at this lane's first head (none when the BMW starts with a head)
        const bool exists = !(lane == 0 && !carry_live && o.h0);
        if (exists) sk.bnd(o.h0 ? o.row0 - 1 : o.row0, closing, o.fh - 1, closing_inside);
      }
      carry = __shfl_sync(0xffffffffu, v_end, nact - 1);
      carry_inside = __shfl_sync(0xffffffffu, (int)inside_end, nact - 1);
      carry_row = __shfl_sync(0xffffffffu, o.row_last, nact - 1);
      carry_live = true;
    }
    if (lane == 0 && carry_live) sk.bnd(carry_row, carry, we - 1, carry_inside && is_head(p, we));
  }
}

template <class V, bool PAD, int WR, int BR>
__global__ void __launch_bounds__(1024) k_compose(DevPart p, const V* __restrict__ x, V* __restrict__ y) {
  extern __shared__ __align__(16) double csm[];  // BR 2: max_block_nnz slots; BR 1: 32 warp sums
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t n_child = p.has_w ? p.n_bmw : p.n_bmt;
  const int64_t per = p.has_w ? nw : blockDim.x;  // children per CTA unit without BMTB
  const int64_t n_units = p.has_b ? p.n_bmtb : (n_child + per - 1) / per;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    int64_t c0, c1, ua = 0, ue = 0;
    if (p.has_b) {
      c0 = ldm(p.bmtb_child + u);
      c1 = ldm(p.bmtb_child + u + 1);
      ua = p.bmtb_start ? ldm(p.bmtb_start + u) : u * p.k1;
      ue = p.bmtb_start ? ldm(p.bmtb_start + u + 1) : min(ua + p.k1, p.nnz_p);
    } else {
      c0 = u * per;
      c1 = min(c0 + per, n_child);
    }
    Sink<V, BR> sk{p, y, csm, ua, 0.0};
    if constexpr (BR == 2) {
      for (int64_t i = threadIdx.x; i < ue - ua; i += blockDim.x) csm[i] = 0.0;
      __syncthreads();
    }
    if (p.has_w) {
      for (int64_t w = c0 + wid; w < c1; w += nw) warp_bmw<V, PAD, WR, BR>(p, x, sk, w, lane);
    } else {
      for (int64_t t = c0 + threadIdx.x; t < c1; t += blockDim.x)
        thread_bmt<V, PAD, BR>(p, x, sk, t, c_pad<V, PAD>(p, t, 0, 0, 0));
    }
    if constexpr (BR == 2) {
      // SHMEM_OFFSET_RED: warp per row fragment of the BMTB, lanes over its slots
      __syncthreads();
      const int64_t r0 = ldm(p.bmtb_first_row + u);
      for (int64_t r = r0 + wid;; r += nw) {
        if (r >= p.m_p) break;
        const int64_t ra = ldm(p.row_ptr + r);
        if (ra >= ue) break;
        const int64_t re = ldm(p.row_ptr + r + 1);
        const int64_t fa = max(ra, ua), fe = min(re, ue);
        double s = 0.0;
        for (int64_t i = fa + lane; i < fe; i += 32) s += csm[i - ua];
        s = warp_sum(s);
        if (lane == 0) {
          if (fa == ra && fe == re) write_excl(p, y, (int32_t)r, s);
          else write_atom(p, y, (int32_t)r, s);
        }
      }
      __syncthreads();
    } else if constexpr (BR == 1) {
      // SHMEM_TOTAL_RED: single-row BMTB (P1), CTA-wide sum
      double s = warp_sum(sk.tot);
      if (lane == 0) csm[wid] = s;
      __syncthreads();
      if (wid == 0) {
        s = lane < nw ? csm[lane] : 0.0;
        s = warp_sum(s);
        if (lane == 0) {
          const int32_t row = (int32_t)ldm(p.bmtb_first_row + u);
          if (is_head(p, ua) && is_head(p, ue)) write_excl(p, y, row, s);
          else write_atom(p, y, row, s);
        }
      }
      __syncthreads();
    }
  }
}

template <class V, bool PAD, int WR>
int launch_wr(const DevPart& p, const V* x, V* y, cudaStream_t s, int64_t g, int tpb) {
  if (p.bred == RED_OFFSET) k_compose<V, PAD, WR, 2><<<g, tpb, p.smem, s>>>(p, x, y);
  else if (p.bred == RED_TOTAL) k_compose<V, PAD, WR, 1><<<g, tpb, 32 * sizeof(double), s>>>(p, x, y);
  else k_compose<V, PAD, WR, 0><<<g, tpb, 0, s>>>(p, x, y);
  return 0;
}
template <class V, bool PAD>
int launch_pad(const DevPart& p, const V* x, V* y, cudaStream_t s, int64_t g, int tpb) {
  switch (p.wred) {
    case RED_TOTAL: return launch_wr<V, PAD, RED_TOTAL>(p, x, y, s, g, tpb);
    case RED_SEG: return launch_wr<V, PAD, RED_SEG>(p, x, y, s, g, tpb);
    case RED_BITMAP: return launch_wr<V, PAD, RED_BITMAP>(p, x, y, s, g, tpb);
    default: return launch_wr<V, PAD, RED_NONE>(p, x, y, s, g, tpb);
  }
}

template <class V, bool PAD, int WR, int BR>
cudaError_t optin_one(size_t bytes) {
  return as::smem_optin(k_compose<V, PAD, WR, BR>, bytes);
}

}  // namespace

// One (value type, BMT_PAD) group of k_compose per translation unit (compose_*.cu)
template <class V, bool PAD>
int compose_launch_grp(const DevPart& p, const V* x, V* y, cudaStream_t s, int64_t g, int tpb) {
  return launch_pad<V, PAD>(p, x, y, s, g, tpb);
}
template <class V, bool PAD>
cudaError_t compose_optin_grp(size_t bytes) {
  cudaError_t e = cudaSuccess;
  auto f = [&](cudaError_t r) {
    if (r != cudaSuccess) e = r;
  };
  f(optin_one<V, PAD, RED_NONE, 2>(bytes));
  f(optin_one<V, PAD, RED_TOTAL, 2>(bytes));
  f(optin_one<V, PAD, RED_SEG, 2>(bytes));
  f(optin_one<V, PAD, RED_BITMAP, 2>(bytes));
  return e;
}

#define AS_COMPOSE_INSTANTIATE(V, PAD)                                                            \
  template int compose_launch_grp<V, PAD>(const DevPart&, const V*, V*, cudaStream_t, int64_t, int); \
  template cudaError_t compose_optin_grp<V, PAD>(size_t);

}  // namespace as
