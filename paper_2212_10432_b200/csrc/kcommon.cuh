// Device helpers shared by the sm_100a SpMV kernel translation units (kernels.cu,
// compose.cu): cache-policy loads, y writers of the writer rule (A22), unit distribution,
// BMT_PAD slot arithmetic (A18) and the warp-level segmented combine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "devpart.h"
#include "optin.h"

namespace as {
namespace {

// ---------------------------------------------------------------- load helpers
// Loads are plain (non-volatile) inline PTX so the compiler may hoist and batch them like
// ordinary loads; AS_LD_VOLATILE=1 restores `asm volatile` (A/B knob).
#if defined(AS_LD_VOLATILE) && AS_LD_VOLATILE
#define AS_LDASM asm volatile
#else
#define AS_LDASM asm
#endif
// Matrix streams: read once per SpMV -> L1::no_allocate + an L2 evict_first cache policy.
__device__ __forceinline__ uint64_t pol_ef() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
#define AS_LD1(T, PT, C, p)                                                                            \
  T v;                                                                                                 \
  AS_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint." PT " %0, [%1], %2;" : "=" C(v) : "l"(p), \
               "l"(pol_ef()));                                                                         \
  return v;
__device__ __forceinline__ double ld_stream(const double* p) { AS_LD1(double, "f64", "d", p) }
__device__ __forceinline__ float ld_stream(const float* p) { AS_LD1(float, "f32", "f", p) }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { AS_LD1(int32_t, "s32", "r", p) }
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  AS_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 v;
  AS_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ float2 ld_stream2(const float* p) {
  float2 v;
  AS_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ int2 ld_stream_i2(const int32_t* p) {
  int2 v;
  AS_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ int4 ld_stream_i4(const int32_t* p) {
  int4 v;
  AS_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol_ef()));
  return v;
}
// x gathers: reused across rows -> cached in L1 (non-coherent path) and kept in L2 with an
// evict_last policy while the evict_first matrix streams pass through (the "L2 persistence
// window for x" of north_star, expressed per load).
__device__ __forceinline__ uint64_t pol_el() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// AS_X_LD (A/B build knob, default 0): L1 behaviour of the x gathers -- 0 L1-allocating,
// 1 L1::no_allocate, 2 .cg (L2 only), 3 L1::evict_first; all with the L2 evict_last policy.
#ifndef AS_X_LD
#define AS_X_LD 0
#endif
#if AS_X_LD == 1
#define AS_XQ "ld.global.nc.L1::no_allocate.L2::cache_hint."
#elif AS_X_LD == 2
#define AS_XQ "ld.global.cg.L2::cache_hint."
#elif AS_X_LD == 3
#define AS_XQ "ld.global.nc.L1::evict_first.L2::cache_hint."
#else
#define AS_XQ "ld.global.nc.L2::cache_hint."
#endif
__device__ __forceinline__ double ldx(const double* x, int64_t c) {
  double v;
  AS_LDASM(AS_XQ "f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pol_el()));
  return v;
}
__device__ __forceinline__ double ldx(const float* x, int64_t c) {
  float v;
  AS_LDASM(AS_XQ "f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  return (double)v;
}
// the same gathers in the value type (fp32 operands are widened only at the FMA: the
// product of two fp32 numbers is exact in fp64, so this is the same arithmetic with half
// the registers per element in flight)
__device__ __forceinline__ double ldxv(const double* x, int64_t c) { return ldx(x, c); }
__device__ __forceinline__ float ldxv(const float* x, int64_t c) {
  float v;
  AS_LDASM(AS_XQ "f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  return v;
}
// x gathers of the hot-x (xcache) kernels: the columns outside the shared-memory copy of a
// scattered matrix are rarely re-read from L1 (C3: 10 % L1 hits), so they are read at L2
// only (.cg): C3 877.6 -> 863 us, gather microbenchmark 750 -> 672 us
// (profiles/r02/ab_xld.jsonl, gather_xld.jsonl)
__device__ __forceinline__ double ldx_l2(const double* x, int64_t c) {
  double v;
  AS_LDASM("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pol_el()));
  return v;
}
__device__ __forceinline__ float ldxv_l2(const float* x, int64_t c) {
  float v;
  AS_LDASM("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(x + c), "l"(pol_el()));
  return v;
}
__device__ __forceinline__ double ldxv_l2(const double* x, int64_t c) { return ldx_l2(x, c); }

// metadata: small, reused by neighbours -> plain non-coherent load
__device__ __forceinline__ int32_t ldm(const int32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ldm(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ int64_t ldm(const int64_t* p) { return __ldg(p); }

// ---------------------------------------------------------------- writers
// Model-Driven Format Compression: evaluate a fitted index model with its patches
__device__ __forceinline__ int64_t idx_eval(const IdxModel& m, int64_t i) {
  int64_t v = m.w == 1 ? m.b + m.k1 * i : m.b + m.k1 * (i / m.w) + m.k2 * (i % m.w);
  for (int j = 0; j < m.np; ++j)
    if (i == m.pi[j]) v = m.pv[j];
  return v;
}
__device__ __forceinline__ int64_t out_row(const DevPart& p, int64_t r) {
  if (p.origin) return (int64_t)ldm(p.origin + r);
  return p.org_model.kind ? idx_eval(p.org_model, r) : p.origin_base + r;
}
// first (compacted) row of NNZ BMT t: stored array, or its fitted model
__device__ __forceinline__ int64_t bmt_row0(const DevPart& p, int64_t t) {
  return p.bmt_first_row ? (int64_t)ldm(p.bmt_first_row + t * p.fr_stride) : idx_eval(p.fr_model, t);
}
// bitmap words of BMT t (stride: bm_words, or the fused metadata stride)
__device__ __forceinline__ const uint32_t* bmt_bits(const DevPart& p, int64_t t) { return p.bitmap + t * p.bm_stride; }
// per-block arrays that Model-Driven Format Compression may have replaced by a fitted model
__device__ __forceinline__ int64_t grp_base_at(const DevPart& p, int64_t g) {
  return p.grp_base ? ldm(p.grp_base + g) : idx_eval(p.pb_model, g);
}
__device__ __forceinline__ int64_t grp_width_at(const DevPart& p, int64_t g) {
  return p.grp_width ? (int64_t)ldm(p.grp_width + g) : idx_eval(p.pw_model, g);
}
__device__ __forceinline__ int64_t bmw_bmt_at(const DevPart& p, int64_t w) {
  if (p.bmw_bmt_ptr) return ldm(p.bmw_bmt_ptr + w);
  return p.bwp_model.kind ? idx_eval(p.bwp_model, w) : min(w * p.bmts_per_bmw, p.n_bmt);
}
__device__ __forceinline__ int64_t bmt_rowp_at(const DevPart& p, int64_t t) {
  if (p.bmt_row_ptr) return ldm(p.bmt_row_ptr + t);
  return p.brp_model.kind ? idx_eval(p.brp_model, t) : min(t * p.s, p.m_p);
}
// fp32 plans: scratch slot of a heavy row (A25), or -1.  A 1-bit-per-row filter (L1/L2
// resident) answers the common case; only heavy rows pay the binary search.
__device__ __forceinline__ int64_t heavy_slot(const DevPart& p, int64_t g) {
  if (!((__ldg(p.heavy_bits + (g >> 5)) >> (g & 31)) & 1u)) return -1;
  int64_t lo = 0, hi = p.n_heavy - 1;
  while (lo <= hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int64_t v = __ldg(p.heavy_rows + mid);
    if (v == g) return mid;
    if (v < g) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

// fused exchange (as_spmv_dist): the final value of row g also goes to every peer's band
template <class V>
__device__ __forceinline__ void peer_store(const DevPart& p, int64_t g, V v) {
#pragma unroll 1
  for (int i = 0; i < p.n_peer; ++i)
    if (g >= p.peer_lo[i] && g < p.peer_hi[i]) ((V*)p.peer_y[i])[g] = v;  // peer i's halo window
}

template <class V>
__device__ __forceinline__ void write_excl(const DevPart& p, V* y, int64_t r, double acc) {
  int64_t g = out_row(p, r);
  if constexpr (sizeof(V) == 4) {
    if (p.n_heavy && p.mode == 1) {
      const int64_t sl = heavy_slot(p, g);
      if (sl >= 0) {
        atomicAdd(p.heavy_acc + sl, p.alpha * acc);
        return;
      }
    }
  }
  if (p.mode == 0) {
    double v = p.alpha * acc;
    if (p.beta != 0.0) v += p.beta * (double)y[g];
    y[g] = (V)v;
    if (p.n_peer) peer_store(p, g, (V)v);
  } else {
    y[g] = (V)((double)y[g] + p.alpha * acc);
  }
}
template <class V>
__device__ __forceinline__ void write_atom(const DevPart& p, V* y, int64_t r, double acc) {
  const int64_t g = out_row(p, r);
  if constexpr (sizeof(V) == 4) {
    if (p.n_heavy) {
      const int64_t sl = heavy_slot(p, g);
      if (sl >= 0) {
        atomicAdd(p.heavy_acc + sl, p.alpha * acc);  // fp64 accumulation (A2, A25)
        return;
      }
    }
  }
  atomicAdd(y + g, (V)(p.alpha * acc));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gthreads() { return (int64_t)gridDim.x * blockDim.x; }

// Unit distribution for persistent grids: CTA-blocked (CTA c owns a contiguous range of
// units), interleaved inside the CTA (consecutive warps / threads take consecutive units).
// All warps of an SM then work on neighbouring rows, so their x windows share L1; with one
// unit per warp / thread (grid = 0) this is the plain one-to-one mapping.
struct Units {
  int64_t begin, end, step;
};
__device__ __forceinline__ Units warp_units(int64_t n) {
  const int64_t wpc = blockDim.x >> 5, per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b = (int64_t)blockIdx.x * per;
  return {b + (threadIdx.x >> 5), min(b + per, n), wpc};
}
__device__ __forceinline__ Units thread_units(int64_t n) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b = (int64_t)blockIdx.x * per;
  return {b + threadIdx.x, min(b + per, n), (int64_t)blockDim.x};
}

template <class V, int VEC>
struct PadLoad;
template <>
struct PadLoad<double, 2> {
  template <class O>
  static __device__ __forceinline__ void ld(const double* v, const int32_t* c, O* vo, int32_t* co) {
    double2 a = ld_stream2(v);
    int2 b = ld_stream_i2(c);
    vo[0] = a.x;
    vo[1] = a.y;
    co[0] = b.x;
    co[1] = b.y;
  }
};
template <>
struct PadLoad<float, 4> {
  template <class O>
  static __device__ __forceinline__ void ld(const float* v, const int32_t* c, O* vo, int32_t* co) {
    float4 a = ld_stream4(v);
    int4 b = ld_stream_i4(c);
    vo[0] = a.x;
    vo[1] = a.y;
    vo[2] = a.z;
    vo[3] = a.w;
    co[0] = b.x;
    co[1] = b.y;
    co[2] = b.z;
    co[3] = b.w;
  }
};
template <>
struct PadLoad<float, 2> {
  template <class O>
  static __device__ __forceinline__ void ld(const float* v, const int32_t* c, O* vo, int32_t* co) {
    float2 a = ld_stream2(v);
    int2 b = ld_stream_i2(c);
    vo[0] = a.x;
    vo[1] = a.y;
    co[0] = b.x;
    co[1] = b.y;
  }
};
template <class V>
struct PadLoad<V, 1> {
  template <class O>
  static __device__ __forceinline__ void ld(const V* v, const int32_t* c, O* vo, int32_t* co) {
    vo[0] = (O)ld_stream(v);
    co[0] = ld_stream(c);
  }
};
template <>
struct PadLoad<double, 4> {
  template <class O>
  static __device__ __forceinline__ void ld(const double* v, const int32_t* c, O* vo, int32_t* co) {
    double2 a = ld_stream2(v), b = ld_stream2(v + 2);
    int4 q = ld_stream_i4(c);
    vo[0] = a.x;
    vo[1] = a.y;
    vo[2] = b.x;
    vo[3] = b.y;
    co[0] = q.x;
    co[1] = q.y;
    co[2] = q.z;
    co[3] = q.w;
  }
};

__device__ __forceinline__ double ld_seq(const double* p) {
  double v;
  AS_LDASM("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ float ld_seq(const float* p) {
  float v;
  AS_LDASM("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ int32_t ld_seq(const int32_t* p) {
  int32_t v;
  AS_LDASM("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_ef()));
  return v;
}

struct PadPos {
  int64_t base, stride;
};
template <int VEC>
__device__ __forceinline__ PadPos pad_pos(const DevPart& p, int64_t t) {
  int64_t g, t0, t1;
  if (p.grp_regular) {
    g = t / p.grp_regular;
    t0 = g * p.grp_regular;
    t1 = min(t0 + p.grp_regular, p.n_bmt);
  } else {
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
  return {grp_base_at(p, g) + (t - t0) * VEC, (t1 - t0) * VEC};
}

// Warp-level combine of per-lane partials (one round of 32 consecutive BMTs).
//   hh: lane holds a row head; cin: partial before its first head (all of it if none);
//   cout: partial from its last head to its end; carry: open segment entering the round.
// Outputs per lane: closing = total of the row closed at the lane's first head (+ whether
// that row started inside the BMW), v_end = open segment value at the lane's end.
template <int WRED>
__device__ __forceinline__ void warp_combine(int lane, bool hh, double cin, double cout, double carry,
                                             bool carry_inside, double& closing, bool& closing_inside,
                                             double& v_end, bool& inside_end) {
  if (WRED == 1) {  // WARP_SEG_ADD_RED: segmented inclusive scan (Blelloch segment sum)
    double v = hh ? cout : cin;
    bool f = hh;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      double nv = __shfl_up_sync(0xffffffffu, v, d);
      bool nf = __shfl_up_sync(0xffffffffu, (int)f, d);
      if (lane >= d) {
        if (!f) v += nv;
        f = f || nf;
      }
    }
    if (!f) v += carry;
    v_end = v;
    inside_end = f ? true : carry_inside;
    double pv = __shfl_up_sync(0xffffffffu, v_end, 1);
    bool pin = __shfl_up_sync(0xffffffffu, (int)inside_end, 1);
    if (lane == 0) {
      pv = carry;
      pin = carry_inside;
    }
    closing = pv + cin;
    closing_inside = pin;
  } else {  // WARP_BITMAP_RED: lane head bitmap (ballot) + plain prefix sums
    const unsigned mask = __ballot_sync(0xffffffffu, hh);
    double P = hh ? 0.0 : cin;  // non-head lanes contribute wholly to the open segment
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      double nv = __shfl_up_sync(0xffffffffu, P, d);
      if (lane >= d) P += nv;
    }
    const unsigned below = mask & ((1u << lane) - 1u);  // previous head lane strictly below
    const int h = below ? 31 - __clz(below) : -1;
    const int hs = h < 0 ? 0 : h;
    double cout_h = __shfl_sync(0xffffffffu, cout, hs);
    double P_h = __shfl_sync(0xffffffffu, P, hs);
    double P_prev = __shfl_up_sync(0xffffffffu, P, 1);
    if (lane == 0) P_prev = 0.0;
    if (h >= 0) {
      closing = cout_h + (P_prev - P_h) + cin;
      closing_inside = true;
    } else {
      closing = carry + P_prev + cin;
      closing_inside = carry_inside;
    }
    const unsigned upto = mask & (lane == 31 ? 0xffffffffu : ((1u << (lane + 1)) - 1u));
    const int h2 = upto ? 31 - __clz(upto) : -1;
    const int h2s = h2 < 0 ? 0 : h2;
    double cout_h2 = __shfl_sync(0xffffffffu, cout, h2s);
    double P_h2 = __shfl_sync(0xffffffffu, P, h2s);
    if (h2 >= 0) {
      v_end = cout_h2 + (P - P_h2);
      inside_end = true;
    } else {
      v_end = carry + P;
      inside_end = carry_inside;
    }
  }
}

}  // namespace

}  // namespace as
