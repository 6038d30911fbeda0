// Plan = the built format made device-resident + its precomputed launch list.
// Uploads only the arrays the chosen kernel reads ("All arrays of a format are extracted
// from Matrix Metadata Set by choosing the metadata needed by the kernel") and
// replaces arrays that are linear by construction by arithmetic (A17).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "internal.h"
#include "plan.h"

namespace as {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      fail(AS_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    }
    fail(AS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <class T>
bool is_affine(const std::vector<T>& v, int64_t step, int64_t base = 0, int64_t cap = INT64_MAX) {
  for (size_t i = 0; i < v.size(); ++i)
    if ((int64_t)v[i] != std::min(base + (int64_t)i * step, cap)) return false;
  return true;
}

std::vector<int32_t> to_i32(const std::vector<int64_t>& v, const char* what) {
  std::vector<int32_t> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i] > INT32_MAX || v[i] < INT32_MIN) fail(AS_ERR_PLAN_INFEASIBLE, std::string(what) + " exceeds int32 (reading A36)");
    o[i] = (int32_t)v[i];
  }
  return o;
}

}  // namespace

void* Plan::up(const void* h, size_t bytes, cudaStream_t s, size_t pad_to) {
  // +64 bytes of zeroed tail: aligned bulk copies (cp.async.bulk, 16-B granules) and vector
  // loads may read up to 3 elements past the end of an array
  size_t alloc = std::max<size_t>(std::max(bytes, pad_to), 16) + 64;
  void* d = dev_alloc(alloc, s);
  allocs.push_back(d);
  dev_bytes += alloc;
  ck(cudaMemsetAsync((char*)d + bytes, 0, alloc - bytes, s), "cudaMemsetAsync");
  if (bytes) ck(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
  return d;
}

const int32_t* Plan::up_i32(const std::vector<int64_t>& v, cudaStream_t s, const char* what) {
  auto t = to_i32(v, what);
  const int32_t* d = (const int32_t*)up(t.data(), t.size() * 4, s);
  cudaStreamSynchronize(s);  // host temporary dies here
  return d;
}

const void* Plan::up_vals(const std::vector<double>& v, cudaStream_t s, size_t pad_elems) {
  size_t n = std::max(v.size(), pad_elems);
  if (dt == AS_R64F && n == v.size()) {
    const void* d = up(v.data(), n * 8, s);
    cudaStreamSynchronize(s);
    return d;
  }
  if (dt == AS_R64F) {
    std::vector<double> t(n, 0.0);
    std::copy(v.begin(), v.end(), t.begin());
    const void* d = up(t.data(), n * 8, s);
    cudaStreamSynchronize(s);
    return d;
  }
  std::vector<float> t(n, 0.0f);
  parallel_for((int64_t)v.size(), [&](int64_t a, int64_t e) {
    for (int64_t i = a; i < e; ++i) t[i] = (float)v[i];
  });
  const void* d = up(t.data(), n * 4, s);
  cudaStreamSynchronize(s);
  return d;
}

// BMT_PAD arrays (A18): slot-major values/columns + per-group first BMT, slot base, width.
void Plan::upload_pad(const HostPart& h, DevPart& d, cudaStream_t s, const std::vector<int32_t>* pad_col) {
  const int64_t sv = dt == AS_R64F ? 8 : 4;
  d.pad = 1;
  d.vec = h.vec;
  d.n_grp = (int64_t)h.pad_width.size();
  // regular groups: every group (but the last) holds the same number of BMTs
  int64_t per = d.n_grp ? h.grp_first_bmt[1] - h.grp_first_bmt[0] : 0;
  bool reg = per > 0;
  for (int64_t g = 0; g < d.n_grp && reg; ++g)
    if (h.grp_first_bmt[g] != g * per) reg = false;
  d.grp_regular = reg ? per : 0;
  d.grp_first_bmt = up_i32(h.grp_first_bmt, s, "grp_first_bmt");
  // Model-Driven Format Compression (NEXT-2) of the per-group slot base and pad_width (the
  // paper's bmt_sizes_of_bmtb): regular groups give linear / step models
  const bool mdc = !std::getenv("AS_NO_MDC");
  int64_t saved = 0;
  if (mdc && fit_array_model(h.grp_base, kMaxPatches, &d.pb_model)) {
    ++modeled_arrays;
    saved += (int64_t)h.grp_base.size() * 8;
  } else {
    d.grp_base = (const int64_t*)up(h.grp_base.data(), h.grp_base.size() * 8, s);
  }
  if (mdc && fit_array_model(h.pad_width, kMaxPatches, &d.pw_model)) {
    ++modeled_arrays;
    saved += (int64_t)h.pad_width.size() * 4;
  } else {
    d.grp_width = up_i32(h.pad_width, s, "pad_width");
  }
  bytes_model -= (double)saved;
  const std::vector<int32_t>& pc = (pad_col && !pad_col->empty()) ? *pad_col : h.pad_col;
  d.pad_col = (const int32_t*)up(pc.data(), pc.size() * 4, s);
  cudaStreamSynchronize(s);
  d.pad_val = up_vals(h.pad_val, s);
  bytes_model += (double)(h.pad_col.size() * 4 + h.pad_val.size() * sv + d.n_grp * (reg ? 12 : 16));
}

// Hot-x cache (SET_RESOURCE xcache = K, reading R-xcache): the K columns the part
// references most (ties: smaller column) are staged in shared memory by every persistent CTA;
// their entries in col / pad_col are re-encoded as ~slot (slots in column order).  Only the
// device copies change: the exported (logical) metadata keeps the original columns.
bool Plan::encode_xcache(const HostPart& h, DevPart& d, cudaStream_t s, std::vector<int32_t>& col_enc,
                         std::vector<int32_t>& pad_enc) {
  const int64_t sv = dt == AS_R64F ? 8 : 4;
  const int64_t cap = (device_max_smem_optin(device) - 1024) / sv;
  int64_t K = std::min<int64_t>(h.xcache, cap);
  if (K <= 0 || h.col.empty()) return false;
  const int64_t nn = host.n;
  std::vector<int32_t> cnt((size_t)nn, 0);
  parallel_for((int64_t)h.col.size(), [&](int64_t a, int64_t e) {
    for (int64_t i = a; i < e; ++i) __atomic_fetch_add(&cnt[(size_t)h.col[i]], 1, __ATOMIC_RELAXED);
  });
  std::vector<int32_t> cand;
  for (int64_t c = 0; c < nn; ++c)
    if (cnt[(size_t)c]) cand.push_back((int32_t)c);
  K = std::min<int64_t>(K, (int64_t)cand.size());
  if (K <= 0) return false;
  auto hotter = [&](int32_t a, int32_t b) { return cnt[a] != cnt[b] ? cnt[a] > cnt[b] : a < b; };
  std::nth_element(cand.begin(), cand.begin() + (K - 1), cand.end(), hotter);
  cand.resize((size_t)K);
  std::sort(cand.begin(), cand.end());
  std::vector<int32_t> slot((size_t)nn, -1);
  for (int64_t i = 0; i < K; ++i) slot[(size_t)cand[(size_t)i]] = (int32_t)i;
  auto enc = [&](const std::vector<int32_t>& in, std::vector<int32_t>& out) {
    out.resize(in.size());
    parallel_for((int64_t)in.size(), [&](int64_t a, int64_t e) {
      for (int64_t i = a; i < e; ++i) {
        const int32_t sl = slot[(size_t)in[i]];
        out[i] = sl >= 0 ? ~sl : in[i];
      }
    });
  };
  if (h.pad) enc(h.pad_col, pad_enc);
  else enc(h.col, col_enc);
  std::vector<int64_t> hot(cand.begin(), cand.end());
  d.xh_cols = up_i32(hot, s, "xcache columns");
  d.xh_n = K;
  bytes_model += (double)(K * 4);
  return true;
}

// x-window staging for k_nnz_thread (banded matrices): persistent CTAs, per (CTA, round)
// x range [lo, hi]; enabled only when every round's window fits the shared-memory ring.
void Plan::try_xwin(const HostPart& h, DevPart& d, cudaStream_t s) {
  const Level& T = h.lv[2];
  const int64_t sv = dt == AS_R64F ? 8 : 4;
  const int64_t max_smem = device_max_smem_optin(device);
  int64_t W = 1;
  while (W * 2 * sv <= std::min<int64_t>(max_smem, 128 * 1024)) W *= 2;
  if (W < 4096) return;
  const int tpb = d.tpb;
  const int per_sm = xw_ctas_per_sm(d.dtype, d.pad, d.vec, tpb, (size_t)(W * sv));
  const int64_t grid = (int64_t)per_sm * device_sm_count(device), nb = T.count();
  if (std::getenv("AS_TRACE"))
    std::fprintf(stderr, "[as_plan] x-window candidate: ring %lld, %d CTAs/SM, %lld BMTs\n", (long long)W, per_sm,
                 (long long)nb);
  if (per_sm < 1) return;
  if (nb < grid * tpb) return;  // too small to fill the persistent grid
  const int64_t per = (nb + grid - 1) / grid, rpc = (per + tpb - 1) / tpb;
  std::vector<int64_t> win((size_t)(grid * rpc * 2), 0);
  std::vector<uint8_t> ok((size_t)grid, 1);
  parallel_for(
      grid,
      [&](int64_t c0, int64_t c1) {
        for (int64_t c = c0; c < c1; ++c) {
          const int64_t b0 = c * per, b1 = std::min(b0 + per, nb);
          std::vector<int64_t> lo(rpc, INT64_MAX), hi(rpc, -1);
          for (int64_t i = 0; i < rpc; ++i) {
            const int64_t t0 = b0 + i * tpb, t1 = std::min(t0 + tpb, b1);
            if (t0 >= t1) continue;
            for (int64_t e = T.start[t0]; e < T.start[t1]; ++e) {
              lo[i] = std::min<int64_t>(lo[i], h.col[e]);
              hi[i] = std::max<int64_t>(hi[i], h.col[e]);
            }
          }
          // lo non-decreasing (suffix minimum), every window within the ring
          for (int64_t i = rpc - 2; i >= 0; --i) lo[i] = std::min(lo[i], lo[i + 1]);
          int64_t mh = -1;
          for (int64_t i = 0; i < rpc; ++i) {
            if (hi[i] < 0) {
              win[(c * rpc + i) * 2] = 0;
              win[(c * rpc + i) * 2 + 1] = -1;
              continue;
            }
            mh = std::max(mh, hi[i]);
            if (mh - lo[i] >= W) ok[c] = 0;
            win[(c * rpc + i) * 2] = lo[i];
            win[(c * rpc + i) * 2 + 1] = hi[i];
          }
        }
      },
      1);
  for (auto v : ok)
    if (!v) return;
  if (std::getenv("AS_TRACE"))
    std::fprintf(stderr, "[as_plan] x-window: ring %lld, grid %lld x %d, %lld rounds/CTA\n", (long long)W,
                 (long long)grid, tpb, (long long)rpc);
  d.xw_size = W;
  d.xw_grid = grid;
  d.xw_rpc = rpc;
  d.smem = (size_t)(W * sv);
  d.xwin = up_i32(win, s, "xwin");
  bytes_model += (double)(win.size() * 4);
}

// A25 for fp32 plans: a row whose value is assembled from more than 167 fp32 additions
// (1e-5 / 2^-24; atomic partials of the units it spans plus ADDs from other parts) could
// exceed the fp32 tolerance; such rows accumulate in an fp64 scratch instead and are added
// to y once by an epilogue (k_heavy_epilogue).
void Plan::mark_heavy_rows(cudaStream_t s) {
  const int64_t kBound = 167;
  std::vector<int32_t> cnt((size_t)m, 0);
  for (int64_t pi : host.launch_order) {
    const HostPart& h = host.parts[pi];
    for (int64_t r : h.excl) cnt[r] += 1;
    if (h.atom.empty()) continue;
    int top = -1;
    for (int l = 2; l >= 0; --l)
      if (h.red[l] != RED_NONE) top = l;
    const int64_t mp = (int64_t)h.origin.size();
    int64_t u = 0;
    for (int64_t r = 0; r < mp; ++r) {
      const int64_t a = h.row_ptr[r], e = h.row_ptr[r + 1];
      int64_t span;
      if (top < 0) {
        span = e - a;
      } else {
        const std::vector<int64_t>& st = h.lv[top].start;
        while (st[u + 1] <= a) ++u;
        int64_t v = u;
        while (st[v + 1] < e) ++v;
        span = v - u + 1;
      }
      if (span > 1) cnt[h.origin[r]] += (int32_t)std::min<int64_t>(span, INT32_MAX / 4);
    }
  }
  std::vector<int64_t> heavy;
  for (int64_t r = 0; r < m; ++r)
    if (cnt[r] > kBound) heavy.push_back(r);
  if (heavy.empty()) return;
  d_heavy_rows = up_i32(heavy, s, "heavy_rows");
  n_heavy = (int64_t)heavy.size();
  d_heavy_acc = (double*)up(nullptr, 0, s, (size_t)n_heavy * 8);
  std::vector<uint32_t> bits((size_t)(m / 32 + 1), 0u);
  for (int64_t r : heavy) bits[(size_t)(r >> 5)] |= 1u << (r & 31);
  const uint32_t* d_bits = (const uint32_t*)up(bits.data(), bits.size() * 4, s);
  cudaStreamSynchronize(s);
  for (auto& d : launches) {
    d.heavy_bits = d_bits;
    d.heavy_rows = d_heavy_rows;
    d.n_heavy = n_heavy;
    d.heavy_acc = d_heavy_acc;
  }
}

Plan::~Plan() {
  if (device >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    for (void* p : allocs) dev_free(p, stream);
    if (d_x) dev_free(d_x, stream);
    if (d_y) dev_free(d_y, stream);
    if (d_x1) dev_free(d_x1, stream);
    if (d_y1) dev_free(d_y1, stream);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    for (int k = 0; k < 4; ++k) {
      if (side[k]) cudaStreamDestroy(side[k]);
      if (ev_join[k]) cudaEventDestroy(ev_join[k]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    cudaSetDevice(cur);
  }
}

cudaEvent_t Plan::host_event(size_t i) {
  while (evs.size() <= i) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    evs.push_back(e);
  }
  return evs[i];
}

// Superset of the x columns a part reads and of the global y rows it writes.
static Plan::Span part_span(const HostPart& h, int64_t n) {
  Plan::Span sp{INT64_MAX, -1, INT64_MAX, -1};
  auto rows = [&](int64_t a, int64_t b) {  // [a, b]
    sp.rlo = std::min(sp.rlo, a);
    sp.rhi = std::max(sp.rhi, b);
  };
  auto cols = [&](int64_t a, int64_t b) {
    sp.clo = std::min(sp.clo, std::max<int64_t>(a, 0));
    sp.chi = std::max(sp.chi, std::min<int64_t>(b, n - 1));
  };
  if (h.kind == "dia") {
    if (h.mb > 0 && !h.dia_off.empty()) {
      rows(h.r0, h.r0 + h.mb - 1);
      auto mm = std::minmax_element(h.dia_off.begin(), h.dia_off.end());
      cols(h.r0 + *mm.first, h.r0 + h.mb - 1 + *mm.second);
    }
  } else if (h.kind == "dense") {
    if (h.mb > 0 && !h.tile_col.empty()) {
      rows(h.r0, h.r0 + h.mb - 1);
      auto mm = std::minmax_element(h.tile_col.begin(), h.tile_col.end());
      cols(*mm.first * h.b, *mm.second * h.b + h.b - 1);
    }
  } else {
    for (int32_t c : h.col) cols(c, c);
    for (int64_t r : h.origin) rows(r, r);
    for (int64_t r : h.excl) rows(r, r);
    for (int64_t r : h.atom) rows(r, r);
  }
  return sp;
}

void Plan::upload(cudaStream_t s) {
  const int64_t sv = dt == AS_R64F ? 8 : 4;
  const bool mdc = !std::getenv("AS_NO_MDC");  // Model-Driven Format Compression (A/B knob)
  const bool fuse = !std::getenv("AS_NO_FUSE");  // short-array fusion (A/B knob)
  int max_smem = device_max_smem_optin(device);
  for (int64_t pi : host.launch_order) {
    const HostPart& h = host.parts[pi];
    const double bytes_before = bytes_model;  // per-launch array bytes (as_plan_profile)
    DevPart d;
    d.fam = h.fam;
    d.dtype = dt == AS_R64F ? 1 : 0;
    d.mode = h.mode;
    d.tpb = h.tpb > 0 ? h.tpb : (h.kind == "dia" ? 128 : 256);  // family defaults (C2 sweep)
    d.grid = h.grid;
    d.n = host.n;
    if (h.kind == "dia") {
      d.D = (int)h.dia_off.size();
      if (d.D > kMaxDiags) fail(AS_ERR_PLAN_INFEASIBLE, "DIA part with more than 64 diagonals");
      for (int i = 0; i < d.D; ++i) d.dia_off[i] = (int32_t)h.dia_off[i];
      d.r0 = h.r0;
      d.mb = h.mb;
      d.origin_base = h.r0;
      d.variant = 3;  // 8-byte loads, one row (fp64) per thread, <= 32 registers: 35.9 vs 42.0 us on C2
      if (const char* v = std::getenv("AS_DIA_VARIANT")) d.variant = std::atoi(v);  // tuning knob
      const int64_t R = 32 / sv;  // k_dia reads 32-byte row groups
      d.dia_stride = (h.mb + R - 1) / R * R;
      std::vector<double> padded((size_t)(d.D * d.dia_stride), 0.0);
      for (int i = 0; i < d.D; ++i)
        std::copy(h.dia_val.begin() + (size_t)i * h.mb, h.dia_val.begin() + (size_t)(i + 1) * h.mb,
                  padded.begin() + (size_t)i * d.dia_stride);
      d.dia_val = up_vals(padded, s);
      bytes_model += (double)(d.D * h.mb * sv);
    } else if (h.kind == "dense") {
      d.b = h.b;
      d.n_tile_rows = (int64_t)h.tile_row_id.size();
      d.row_lo = h.r0;
      d.row_hi = h.r0 + h.mb;
      d.tile_row_id = up_i32(h.tile_row_id, s, "tile_row_id");
      d.tile_row_ptr = up_i32(h.tile_row_ptr, s, "tile_row_ptr");
      d.tile_col = up_i32(h.tile_col, s, "tile_col");
      d.tile_val = up_vals(h.tile_val, s);
      if (d.b > 128) fail(AS_ERR_PLAN_INFEASIBLE, "DENSE tiles larger than 128 are not implemented");
      bytes_model += (double)(h.tile_val.size() * sv + (h.tile_col.size() + 2 * h.tile_row_id.size() + 1) * 4);
    } else {
      const int64_t mp = (int64_t)h.origin.size(), nnz = h.row_ptr.back();
      // Index widths (A36, narrowest lossless per array): element positions are computed in
      // int64 by the kernels (implicit NNZ block starts t*k, int64 BMT_PAD group bases), so a
      // part may hold >= 2^31 nonzeros; every STORED index array is int32 and up_i32 rejects
      // one whose values do not fit (AS_ERR_PLAN_INFEASIBLE naming the array)
      d.m_p = mp;
      d.nnz_p = nnz;
      // origin_rows: implicit when affine (A17), else a fitted model (NEXT-2), else stored
      if (mp && is_affine(h.origin, 1, h.origin[0])) {
        d.origin_base = h.origin[0];
      } else if (mdc && fit_array_model(h.origin, kMaxPatches, &d.org_model)) {
        ++modeled_arrays;
      } else {
        d.origin = up_i32(h.origin, s, "origin_rows");
        bytes_model += (double)(mp * 4);
      }
      const Level &B = h.lv[0], &W = h.lv[1], &T = h.lv[2];
      bool need_rowptr = true, need_colval = true;
      std::vector<int32_t> col_enc, pad_enc;  // xcache-encoded device columns (empty: as built)
      switch (h.fam) {
        case FAM_THREAD_ROW: {
          d.n_bmt = T.count();
          d.s = T.size;
          if (!is_affine(T.first_row, T.size, 0)) {
            std::vector<int64_t> brp = T.first_row;
            brp.push_back(mp);
            if (mdc && fit_array_model(brp, kMaxPatches, &d.brp_model)) {
              ++modeled_arrays;  // ROW-block row offsets as a model (NEXT-2)
            } else {
              d.bmt_row_ptr = up_i32(brp, s, "bmt_row_ptr");
              bytes_model += (double)(brp.size() * 4);
            }
          }
          if (h.pad) {
            upload_pad(h, d, s);
            need_colval = false;
            // row_ptr only for multi-row padded BMTs
            bool multi = false;
            for (int64_t t = 0; t < T.count() && !multi; ++t)
              multi = (t + 1 < T.count() ? T.first_row[t + 1] : mp) - T.first_row[t] > 1;
            need_rowptr = multi;
          }
          break;
        }
        case FAM_NNZ_THREAD:
        case FAM_NNZ_WARP: {
          d.n_bmt = T.count();
          d.k = T.size;
          if (h.fam == FAM_NNZ_WARP && !h.pad && (T.size == 1 || T.size == 2 || T.size == 4) && W.nnz &&
              !B.present && W.size % (32 * T.size) == 0 && h.xcache == 0) {
            // tile form: packed 1-bit heads + BMW first rows; BMT starts and first rows
            // are computed from them (k_warp_tile)
            d.tile = 1;
            d.variant = h.red[1] == RED_SEG ? 1 : 2;
            d.n_bmw = W.count();
            d.bmts_per_bmw = W.size / T.size;
            std::vector<uint32_t> bits((size_t)(nnz / 32 + 2), 0u);
            for (int64_t r = 0; r < mp; ++r) bits[(size_t)(h.row_ptr[r] >> 5)] |= 1u << (h.row_ptr[r] & 31);
            d.bits = (const uint32_t*)up(bits.data(), bits.size() * 4, s);
            cudaStreamSynchronize(s);
            d.bmw_first_row = up_i32(W.first_row, s, "bmw_first_row");
            bytes_model += (double)(bits.size() * 4 + W.first_row.size() * 4);
            need_rowptr = false;
            break;
          }
          std::vector<int64_t> st(T.start.begin(), T.start.end() - 1);
          if (!is_affine(st, T.size, 0)) {
            d.bmt_start = up_i32(T.start, s, "bmt_start");
            bytes_model += (double)(T.start.size() * 4);
          }
          d.bm_words = h.bm_words;
          d.bm_stride = h.bm_words;
          if (mdc && fit_array_model(T.first_row, kMaxPatches, &d.fr_model)) {
            ++modeled_arrays;  // Model-Driven Format Compression (NEXT-2): computed, not loaded
            d.bitmap = (const uint32_t*)up(h.bitmap.data(), h.bitmap.size() * 4, s);
            bytes_model += (double)(h.bitmap.size() * 4);
          } else if (fuse && h.bm_words >= 1 && h.bm_words <= 3) {
            // short-array fusion: {first_row, bm0[, bm1[, bm2]]} per BMT, padded to a
            // power-of-two stride of int32 words
            const int S = h.bm_words + 1 <= 2 ? 2 : 4;
            const int64_t nb = T.count();
            std::vector<int32_t> fused((size_t)(nb * S), 0);
            for (int64_t t = 0; t < nb; ++t) {
              if (T.first_row[t] > INT32_MAX) fail(AS_ERR_PLAN_INFEASIBLE, "bmt_first_row exceeds int32 (reading A36)");
              fused[(size_t)(t * S)] = (int32_t)T.first_row[t];
              for (int w = 0; w < h.bm_words; ++w) fused[(size_t)(t * S + 1 + w)] = (int32_t)h.bitmap[(size_t)(t * h.bm_words + w)];
            }
            const int32_t* f = (const int32_t*)up(fused.data(), fused.size() * 4, s);
            cudaStreamSynchronize(s);
            d.bmt_first_row = f;
            d.bitmap = (const uint32_t*)(f + 1);
            d.fr_stride = d.bm_stride = S;
            ++fused_arrays;
            bytes_model += (double)(fused.size() * 4);
          } else {
            d.bmt_first_row = up_i32(T.first_row, s, "bmt_first_row");
            bytes_model += (double)(T.first_row.size() * 4);
            d.bitmap = (const uint32_t*)up(h.bitmap.data(), h.bitmap.size() * 4, s);
            bytes_model += (double)(h.bitmap.size() * 4);
          }
          if (h.xcache > 0) encode_xcache(h, d, s, col_enc, pad_enc);
          if (h.pad) {  // CSR5-like slot-major tiles (BMT_PAD over NNZ BMTs)
            upload_pad(h, d, s, &pad_enc);
            need_colval = false;
            d.pad_grp_bmw = (h.fam == FAM_NNZ_WARP && h.pad_scope == 1) ? 1 : 0;
          }
          if (h.fam == FAM_NNZ_THREAD && h.stages == 2 && !d.xh_n) try_xwin(h, d, s);
          if (h.fam == FAM_NNZ_WARP) {
            d.variant = h.red[1] == RED_SEG ? 1 : 2;
            d.n_bmw = W.count();
            // BMT index range of each BMW (BMTs restart at BMW boundaries)
            std::vector<int64_t> ptr(W.count() + 1, 0);
            int64_t t = 0;
            for (int64_t w = 0; w < W.count(); ++w) {
              ptr[w] = t;
              while (t < T.count() && T.start[t] < W.start[w + 1]) ++t;
            }
            ptr[W.count()] = t;
            int64_t per = W.count() ? ptr[1] - ptr[0] : 0;
            if (per > 0 && is_affine(ptr, per, 0, T.count())) {
              d.bmts_per_bmw = per;
            } else if (mdc && fit_array_model(ptr, kMaxPatches, &d.bwp_model)) {
              ++modeled_arrays;  // BMT range per BMW as a model (NEXT-2)
            } else {
              d.bmw_bmt_ptr = up_i32(ptr, s, "bmw_bmt_ptr");
              bytes_model += (double)(ptr.size() * 4);
            }
          }
          need_rowptr = false;
          break;
        }
        case FAM_WARP_ROW: {
          d.n_bmw = W.count();
          d.k = T.present ? T.size : 0;
          bool rowblocks = !W.nnz && (!B.present || !B.nnz);
          d.bmw_all_excl = rowblocks ? 1 : 0;
          if (rowblocks && W.size == 1 && is_affine(W.first_row, 1, 0)) {
            d.bmw_start = nullptr;  // == row_ptr
          } else {
            d.bmw_start = up_i32(W.start, s, "bmw_start");
            d.bmw_first_row = up_i32(W.first_row, s, "bmw_first_row");
            bytes_model += (double)((W.start.size() + W.first_row.size()) * 4);
          }
          break;
        }
        case FAM_BLOCK_TOTAL:
        case FAM_BLOCK_OFFSET: {
          d.n_bmtb = B.count();
          std::vector<int64_t> st(B.start.begin(), B.start.end() - 1);
          if (B.nnz && is_affine(st, B.size, 0)) {
            d.k1 = B.size;
          } else {
            d.bmtb_start = up_i32(B.start, s, "bmtb_start");
            bytes_model += (double)(B.start.size() * 4);
          }
          d.bmtb_first_row = up_i32(B.first_row, s, "bmtb_first_row");
          bytes_model += (double)(B.first_row.size() * 4);
          int64_t mx = 0;
          for (int64_t b = 0; b < B.count(); ++b) mx = std::max(mx, B.start[b + 1] - B.start[b]);
          d.max_block_nnz = mx;
          if (h.fam == FAM_BLOCK_OFFSET) {
            // TMA form when two staged blocks + the product buffer fit in shared memory:
            // per stage cap elements (aligned span + slack) and rcap row offsets
            int64_t cap = 0, rcap = 0;
            for (int64_t b = 0; b < B.count(); ++b) {
              int64_t a = B.start[b], e = B.start[b + 1];
              cap = std::max(cap, ((e + 3) & ~int64_t(3)) - (a & ~int64_t(3)));
              int64_t r0 = B.first_row[b], r1 = b + 1 < B.count() ? std::min(B.first_row[b + 1] + 1, mp) : mp;
              rcap = std::max(rcap, ((r1 + 1 + 3) & ~int64_t(3)) - (r0 & ~int64_t(3)));
            }
            d.smem_cap = cap + 4;
            d.smem_rcap = rcap + 4;
            int64_t need = 2 * (d.smem_cap * (sv + 4) + d.smem_rcap * 4) + d.smem_cap * 8 + 16;
            if (need <= max_smem && h.stages == 2) d.variant = 1;
            else if ((int64_t)mx * 8 > max_smem)
              fail(AS_ERR_PLAN_INFEASIBLE, "P2: SHMEM_OFFSET_RED block of " + std::to_string(mx) +
                                               " nonzeros exceeds the shared-memory opt-in limit");
          }
          break;
        }
        case FAM_COMPOSE: {
          // composed levels (compose.cu): packed row-head bits + each present level's block
          // starts / first rows / child ranges; a missing BMT level runs as NNZ_BLOCK(1)
          d.tred = h.red[2];
          d.wred = h.red[1];
          d.bred = h.red[0];
          d.has_w = W.present;
          d.has_b = B.present;
          d.per_elem = h.red[0] == RED_NONE && h.red[1] == RED_NONE && h.red[2] == RED_NONE;
          std::vector<uint32_t> bits((size_t)(nnz / 32 + 2), 0u);
          for (int64_t r = 0; r < mp; ++r) bits[(size_t)(h.row_ptr[r] >> 5)] |= 1u << (h.row_ptr[r] & 31);
          d.bits = (const uint32_t*)up(bits.data(), bits.size() * 4, s);
          cudaStreamSynchronize(s);
          bytes_model += (double)(bits.size() * 4);
          std::vector<int64_t> tstart, tfirst;
          const std::vector<int64_t>* ts = &T.start;
          const std::vector<int64_t>* tf = &T.first_row;
          if (!T.present) {
            d.t_synth = 1;
            tstart.resize((size_t)nnz + 1);
            tfirst.resize((size_t)nnz);
            for (int64_t e = 0; e <= nnz; ++e) tstart[(size_t)e] = e;
            for (int64_t r = 0; r < mp; ++r)
              for (int64_t e = h.row_ptr[r]; e < h.row_ptr[r + 1]; ++e) tfirst[(size_t)e] = r;
            ts = &tstart;
            tf = &tfirst;
          }
          const int64_t nt = (int64_t)ts->size() - 1;
          d.n_bmt = nt;
          d.k = T.present ? (T.nnz ? T.size : 0) : 1;
          std::vector<int64_t> st0(ts->begin(), ts->end() - 1);
          if (!(d.k > 0 && is_affine(st0, d.k, 0))) {
            d.k = 0;
            d.bmt_start = up_i32(*ts, s, "bmt_start");
            bytes_model += (double)(ts->size() * 4);
          }
          if (mdc && fit_array_model(*tf, kMaxPatches, &d.fr_model)) {
            ++modeled_arrays;
          } else {
            d.bmt_first_row = up_i32(*tf, s, "bmt_first_row");
            bytes_model += (double)(tf->size() * 4);
          }
          // child block range of every block of `lv` at the next present level
          auto child_ptr = [&](const Level& lv, const std::vector<int64_t>& cstart) {
            std::vector<int64_t> ptr((size_t)lv.count() + 1, 0);
            int64_t c = 0;
            const int64_t nc = (int64_t)cstart.size() - 1;
            for (int64_t b = 0; b < lv.count(); ++b) {
              ptr[(size_t)b] = c;
              while (c < nc && cstart[(size_t)c] < lv.start[(size_t)b + 1]) ++c;
            }
            ptr[(size_t)lv.count()] = c;
            return ptr;
          };
          if (W.present) {
            d.n_bmw = W.count();
            std::vector<int64_t> ptr = child_ptr(W, *ts);
            const int64_t per = W.count() ? ptr[1] - ptr[0] : 0;
            if (per > 0 && is_affine(ptr, per, 0, nt)) {
              d.bmts_per_bmw = per;
            } else if (mdc && fit_array_model(ptr, kMaxPatches, &d.bwp_model)) {
              ++modeled_arrays;
            } else {
              d.bmw_bmt_ptr = up_i32(ptr, s, "bmw_bmt_ptr");
              bytes_model += (double)(ptr.size() * 4);
            }
          }
          if (B.present) {
            d.n_bmtb = B.count();
            std::vector<int64_t> bst(B.start.begin(), B.start.end() - 1);
            if (B.nnz && is_affine(bst, B.size, 0)) {
              d.k1 = B.size;
            } else {
              d.bmtb_start = up_i32(B.start, s, "bmtb_start");
              bytes_model += (double)(B.start.size() * 4);
            }
            d.bmtb_first_row = up_i32(B.first_row, s, "bmtb_first_row");
            std::vector<int64_t> cp = child_ptr(B, W.present ? W.start : *ts);
            d.bmtb_child = up_i32(cp, s, "bmtb_child");
            bytes_model += (double)((B.first_row.size() + cp.size()) * 4);
            int64_t mx = 0;
            for (int64_t b = 0; b < B.count(); ++b) mx = std::max(mx, B.start[b + 1] - B.start[b]);
            d.max_block_nnz = mx;
            if (h.red[0] == RED_OFFSET && mx * 8 > max_smem)
              fail(AS_ERR_PLAN_INFEASIBLE, "P2: SHMEM_OFFSET_RED block of " + std::to_string(mx) +
                                               " nonzeros exceeds the shared-memory opt-in limit");
          }
          need_rowptr = h.red[0] == RED_OFFSET;
          if (h.pad) {
            upload_pad(h, d, s);
            need_colval = false;
            d.pad_grp_bmw = (W.present && h.pad_scope == 1) ? 1 : 0;
          }
          break;
        }
        default:
          fail(AS_ERR_PLAN_INFEASIBLE, "part without a kernel");
      }
      if (need_rowptr) {
        d.row_ptr = up_i32(h.row_ptr, s, "row_ptr");
        bytes_model += (double)((mp + 1) * 4);
      }
      if (h.fam == FAM_WARP_ROW && !d.bmw_start) d.bmw_start = d.row_ptr;
      if (need_colval) {
        const std::vector<int32_t>& cc = col_enc.empty() ? h.col : col_enc;
        d.col = (const int32_t*)up(cc.data(), cc.size() * 4, s);
        d.val = up_vals(h.val, s);
        bytes_model += (double)(nnz * (4 + sv));
      }
    }
    if (std::getenv("AS_NT_LEGACY")) {  // A/B knob: branching forms of the nnz kernels
      if (d.fam == FAM_NNZ_THREAD) d.variant = 9;
      if (d.fam == FAM_NNZ_WARP && !d.tile) d.variant += 8;
    }
    ck((cudaError_t)prepare_part(d), "kernel attributes");
    // name the kernel form actually chosen (as_plan_info.kernels)
    std::string& fn = host.parts[pi].fam_name;
    if (d.xwin) fn += "_xwin";
    if (d.xh_n) fn += "_xh";
    if (d.tile) fn += "_tile";
    if (d.fam == FAM_BLOCK_OFFSET && d.variant == 1) fn += "_tma";
    launches.push_back(d);
    launch_part.push_back(pi);
    launch_stream.push_back(h.stream);
    spans.push_back(part_span(h, host.n));
    launch_bytes.push_back(bytes_model - bytes_before);
  }
  if (!host.prepass.empty()) {
    d_prepass = up_i32(host.prepass, s, "prepass");
    n_prepass = (int64_t)host.prepass.size();
  }
  if (dt == AS_R32F) mark_heavy_rows(s);
  // xcache is implemented in the predicated-emit nnz kernels; parts that will run the
  // branching form (fp32 ADD-mode parts with heavy rows, or the AS_NT_LEGACY A/B knob) get
  // their columns back unencoded
  for (size_t i = 0; i < launches.size(); ++i) {
    DevPart& d = launches[i];
    if (!d.xh_n) continue;
    const bool legacy = (d.fam == FAM_NNZ_THREAD && d.variant == 9) || (d.fam == FAM_NNZ_WARP && d.variant >= 8) ||
                        (d.dtype == 0 && d.n_heavy && d.mode == 1);
    if (!legacy) continue;
    const HostPart& h = host.parts[host.launch_order[i]];
    if (d.pad) d.pad_col = (const int32_t*)up(h.pad_col.data(), h.pad_col.size() * 4, s);
    else d.col = (const int32_t*)up(h.col.data(), h.col.size() * 4, s);
    d.xh_n = 0;
    d.xh_cols = nullptr;
    d.smem = 0;
    std::string& fn = host.parts[host.launch_order[i]].fam_name;
    const size_t at = fn.find("_xh");
    if (at != std::string::npos) fn.erase(at, 3);
  }
  main_stream = launch_stream.empty() ? 0 : launch_stream[0];
  for (int k : launch_stream) concurrent = concurrent || k != main_stream;
  // side streams and fork/join events are created here, once, so concurrent as_spmv calls on
  // the plan never race on creating them
  if (concurrent) {
    for (int k : launch_stream)
      if (k != main_stream && !side[k]) {
        ck(cudaStreamCreateWithFlags(&side[k], cudaStreamNonBlocking), "side stream");
        ck(cudaEventCreateWithFlags(&ev_join[k], cudaEventDisableTiming), "join event");
      }
    ck(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "fork event");
  }
  const size_t L = launches.size();
  side_y.assign(L, nullptr);
  side_rows.assign(L, nullptr);
  side_zero.assign(L, nullptr);
  n_side_rows.assign(L, 0);
  n_side_zero.assign(L, 0);
  for (size_t i = 0; i < L; ++i) {
    const HostPart& h = host.parts[host.launch_order[i]];
    if (h.mode != 3) continue;
    side_y[i] = up(nullptr, 0, s, (size_t)m * (dt == AS_R64F ? 8 : 4));
    std::vector<int64_t> rows(h.excl);
    rows.insert(rows.end(), h.atom.begin(), h.atom.end());
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
    side_rows[i] = up_i32(rows, s, "side rows");
    n_side_rows[i] = (int64_t)rows.size();
    if (!h.atom.empty()) {
      std::vector<int64_t> z(h.atom);
      std::sort(z.begin(), z.end());
      side_zero[i] = up_i32(z, s, "side atomic rows");
      n_side_zero[i] = (int64_t)z.size();
    }
  }
  single_writer = host.prepass.empty() && n_heavy == 0;
  for (int64_t pi : host.launch_order)
    if (host.parts[pi].mode != 0 || !host.parts[pi].atom.empty()) single_writer = false;
  ck(cudaStreamSynchronize(s), "upload");
}

// SpMM (NEXT-4): the plain COMPRESS arrays of every CSR-family part plus a per-row "add"
// flag: the part is in ADD mode, or the row is one of ITS atomic rows (it straddles writer
// units of this part in the SpMV, so its value was initialised by the pre-pass or an earlier
// part; SpMM adds this part's whole-row partial).  Exclusive rows of a STORE part store.
void Plan::upload_spmm(cudaStream_t s) {
  // the SpMM DENSE kernel (k_spmm_dense_dmma) holds tiles of b <= 64; reject larger tiles at
  // plan time so as_spmm never launches a prefix of the parts and then fails on a later one
  for (int64_t pi : host.launch_order)
    if (host.parts[pi].kind == "dense" && host.parts[pi].b > 64)
      fail(AS_ERR_PLAN_INFEASIBLE, "AS_PLAN_SPMM: DENSE tiles larger than 64 are not implemented for SpMM");
  std::vector<uint8_t> atom((size_t)m, 0);
  for (int64_t pi : host.launch_order) {
    const HostPart& h = host.parts[pi];
    for (int64_t r : h.atom) atom[(size_t)r] = 1;  // this part's atomic rows (cleared below)
    SpmmPart sp;
    if (h.kind == "csr") {
      sp.m_p = (int64_t)h.origin.size();
      sp.rows = up_i32(h.origin, s, "spmm rows");
      sp.rp = up_i32(h.row_ptr, s, "spmm row_ptr");
      sp.col = (const int32_t*)up(h.col.data(), h.col.size() * 4, s);
      sp.val = up_vals(h.val, s);
      std::vector<uint8_t> add((size_t)sp.m_p);
      for (int64_t i = 0; i < sp.m_p; ++i) add[(size_t)i] = (h.mode != 0 || atom[(size_t)h.origin[i]]) ? 1 : 0;
      sp.add = (const uint8_t*)up(add.data(), add.size(), s);
      ck(cudaStreamSynchronize(s), "spmm upload");
    }
    for (int64_t r : h.atom) atom[(size_t)r] = 0;
    spmm_parts.push_back(sp);
  }
  spmm = true;
}

void Plan::compute_model() {
  const double sv = dt == AS_R64F ? 8 : 4;
  // x: compulsory distinct columns; y per writer rule
  double ybytes0 = 0, ybytes1 = 0;
  for (int64_t pi : host.launch_order) {
    const HostPart& h = host.parts[pi];
    double ex = (double)h.excl.size(), at = (double)h.atom.size();
    if (h.mode == 3) {
      // R-conc side part: STOREs (and atomics onto zeroed rows) into its scratch, then
      // k_side_add reads each written row's scratch value and updates y
      const double t = ex * sv + at * (4 + 3 * sv) + (ex + at) * (4 + 3 * sv);
      ybytes0 += t;
      ybytes1 += t;
      continue;
    }
    if (h.mode == 0) {
      ybytes0 += ex * sv;
      ybytes1 += 2 * ex * sv;
    } else {
      ybytes0 += 2 * ex * sv;
      ybytes1 += 2 * ex * sv;
    }
    ybytes0 += 2 * at * sv;
    ybytes1 += 2 * at * sv;
  }
  // per launch (as_plan_profile): + the x bytes of the part's distinct columns + its y traffic
  if (launch_bytes.size() == host.launch_order.size()) {
    std::vector<uint8_t> seen((size_t)host.n, 0);
    for (size_t i = 0; i < host.launch_order.size(); ++i) {
      const HostPart& h = host.parts[host.launch_order[i]];
      int64_t xc = 0;
      if (h.kind == "csr") {
        std::fill(seen.begin(), seen.end(), 0);
        for (int32_t c : h.col)
          if (!seen[(size_t)c]) {
            seen[(size_t)c] = 1;
            ++xc;
          }
      } else if (i < spans.size() && spans[i].chi >= spans[i].clo) {
        xc = spans[i].chi - spans[i].clo + 1;
      }
      const double ex = (double)h.excl.size(), at = (double)h.atom.size();
      launch_bytes[i] += (double)xc * sv + (h.mode == 0 || h.mode == 3 ? ex * sv : 2 * ex * sv) + 2 * at * sv;
    }
  }
  double pre = (double)host.prepass.size();
  // beta == 0: as_spmv fills all of y instead when that moves fewer bytes (api.cpp run_plan)
  double prebytes0 = (double)m * sv <= pre * (4 + 32) ? (double)m * sv : pre * (4 + sv);
  double prebytes1 = pre * (4 + 2 * sv);
  prepass_bytes = pre ? prebytes0 : 0;
  info.bytes_model = bytes_model + host.distinct_cols * sv + ybytes0 + (pre ? prebytes0 : 0);
  info.bytes_model_beta = bytes_model + host.distinct_cols * sv + ybytes1 + (pre ? prebytes1 : 0);
  info.bytes_floor = nnz_real * (sv + 4) + host.n * sv + host.m * sv;
}

}  // namespace as
