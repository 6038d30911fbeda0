// Device readback of a plan's format ("dev.<key>" export keys): the arrays the kernels
// actually read, copied back from device memory and decoded to the logical Matrix Metadata
// Set layout (§V-A) -- int32 -> int64 indices, arrays that are implicit (A17) or
// replaced by a fitted model (Model-Driven Format Compression) evaluated, the
// hot-x column encoding (~slot, R-xcache) undone, the DIA row stride padding dropped.  The
// tests compare these with the oracle's logical arrays byte for byte, so what is checked is
// the uploaded format itself, not the host copy it was built from.
#include <cuda_runtime.h>

#include <cstring>

#include "internal.h"
#include "plan.h"

namespace as {

namespace {

template <class T>
std::vector<T> d2h(const void* p, int64_t n) {
  std::vector<T> v((size_t)std::max<int64_t>(n, 0));
  if (n > 0) check_cuda(cudaMemcpy(v.data(), p, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost), "readback");
  return v;
}
std::vector<int64_t> widen(const std::vector<int32_t>& v) { return std::vector<int64_t>(v.begin(), v.end()); }
int64_t model_at(const IdxModel& m, int64_t i) {
  int64_t v = m.w == 1 ? m.b + m.k1 * i : m.b + m.k1 * (i / m.w) + m.k2 * (i % m.w);
  for (int j = 0; j < m.np; ++j)
    if (i == m.pi[j]) v = m.pv[j];
  return v;
}
template <class T>
std::vector<uint8_t> bytes(const std::vector<T>& v) {
  std::vector<uint8_t> b(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
  return b;
}

// the logical arrays of one uploaded part (key suffix -> bytes)
void part_arrays(const Plan& P, const DevPart& d, int64_t part, std::vector<std::pair<std::string, std::vector<uint8_t>>>& out) {
  const int64_t sv = d.dtype == 1 ? 8 : 4;
  auto put_i = [&](const std::string& k, const std::vector<int64_t>& v) { out.push_back({k, bytes(v)}); };
  auto put_raw = [&](const std::string& k, std::vector<uint8_t> b) { out.push_back({k, std::move(b)}); };
  if (d.fam == FAM_DIA) {
    std::vector<int64_t> off(d.dia_off, d.dia_off + d.D);
    put_i("dia.off", off);
    std::vector<uint8_t> all = d2h<uint8_t>(d.dia_val, d.D * d.dia_stride * sv), v((size_t)(d.D * d.mb * sv));
    for (int i = 0; i < d.D; ++i)
      std::memcpy(v.data() + (size_t)(i * d.mb * sv), all.data() + (size_t)(i * d.dia_stride * sv), (size_t)(d.mb * sv));
    put_raw("dia.val", std::move(v));
    return;
  }
  if (d.fam == FAM_DENSE) {
    std::vector<int64_t> rid = widen(d2h<int32_t>(d.tile_row_id, d.n_tile_rows));
    std::vector<int64_t> rptr = widen(d2h<int32_t>(d.tile_row_ptr, d.n_tile_rows + 1));
    const int64_t nt = rptr.empty() ? 0 : rptr.back();
    put_i("tile.row_id", rid);
    put_i("tile.row_ptr", rptr);
    put_i("tile.col", widen(d2h<int32_t>(d.tile_col, nt)));
    put_raw("tile.val", d2h<uint8_t>(d.tile_val, nt * d.b * d.b * sv));
    return;
  }
  // CSR-family parts
  std::vector<int64_t> org((size_t)d.m_p);
  if (d.origin) org = widen(d2h<int32_t>(d.origin, d.m_p));
  else
    for (int64_t i = 0; i < d.m_p; ++i) org[(size_t)i] = d.org_model.kind ? model_at(d.org_model, i) : d.origin_base + i;
  put_i("origin_rows", org);
  if (d.row_ptr) put_i("row_ptr", widen(d2h<int32_t>(d.row_ptr, d.m_p + 1)));
  std::vector<int32_t> hot;
  if (d.xh_n) hot = d2h<int32_t>(d.xh_cols, d.xh_n);
  auto decode = [&](std::vector<int32_t> c) {
    std::vector<int64_t> o(c.size());
    for (size_t i = 0; i < c.size(); ++i) o[i] = c[i] < 0 ? (int64_t)hot[(size_t)~c[i]] : (int64_t)c[i];
    return o;
  };
  if (d.col) put_i("col", decode(d2h<int32_t>(d.col, d.nnz_p)));
  if (d.val) put_raw("val", d2h<uint8_t>(d.val, d.nnz_p * sv));
  // BMT level of the NNZ families and of composed parts with a real BMT level
  const bool bmt_nnz = d.fam == FAM_NNZ_THREAD || d.fam == FAM_NNZ_WARP || (d.fam == FAM_COMPOSE && !d.t_synth);
  if (bmt_nnz && !d.tile) {
    std::vector<int64_t> st;
    if (d.bmt_start) st = widen(d2h<int32_t>(d.bmt_start, d.n_bmt + 1));
    else
      for (int64_t t = 0; t <= d.n_bmt; ++t) st.push_back(std::min(t * d.k, d.nnz_p));
    put_i("bmt.nz_ptr", st);
    std::vector<int64_t> fr((size_t)d.n_bmt);
    if (d.bmt_first_row) {  // plain, or fused with the bitmap words (stride fr_stride)
      std::vector<int32_t> raw = d2h<int32_t>(d.bmt_first_row, d.n_bmt * d.fr_stride);
      for (int64_t t = 0; t < d.n_bmt; ++t) fr[(size_t)t] = raw[(size_t)(t * d.fr_stride)];
    } else {
      for (int64_t t = 0; t < d.n_bmt; ++t) fr[(size_t)t] = model_at(d.fr_model, t);
    }
    put_i("bmt.first_row", fr);
  }
  if (d.bitmap && d.bm_words) {
    std::vector<uint32_t> raw = d2h<uint32_t>(d.bitmap, d.n_bmt * d.bm_stride), bm((size_t)(d.n_bmt * d.bm_words));
    for (int64_t t = 0; t < d.n_bmt; ++t)
      for (int w = 0; w < d.bm_words; ++w) bm[(size_t)(t * d.bm_words + w)] = raw[(size_t)(t * d.bm_stride + w)];
    put_raw("bmt.bitmap", bytes(bm));
  }
  if (d.fam == FAM_THREAD_ROW) {
    std::vector<int64_t> fr((size_t)d.n_bmt);
    if (d.bmt_row_ptr) fr = widen(d2h<int32_t>(d.bmt_row_ptr, d.n_bmt));
    else
      for (int64_t t = 0; t < d.n_bmt; ++t) fr[(size_t)t] = d.brp_model.kind ? model_at(d.brp_model, t) : t * d.s;
    put_i("bmt.first_row", fr);
  }
  if (d.pad) {
    std::vector<int64_t> w((size_t)d.n_grp), base((size_t)d.n_grp);
    if (d.grp_width) w = widen(d2h<int32_t>(d.grp_width, d.n_grp));
    else
      for (int64_t g = 0; g < d.n_grp; ++g) w[(size_t)g] = model_at(d.pw_model, g);
    if (d.grp_base) base = d2h<int64_t>(d.grp_base, d.n_grp);
    else
      for (int64_t g = 0; g < d.n_grp; ++g) base[(size_t)g] = model_at(d.pb_model, g);
    std::vector<int64_t> gf = widen(d2h<int32_t>(d.grp_first_bmt, d.n_grp + 1));
    const int64_t total = d.n_grp ? base.back() + (gf[(size_t)d.n_grp] - gf[(size_t)d.n_grp - 1]) * w.back() : 0;
    base.push_back(total);
    put_i("pad.width", w);
    put_i("pad.base", base);
    put_i("pad.col", decode(d2h<int32_t>(d.pad_col, total)));
    put_raw("pad.val", d2h<uint8_t>(d.pad_val, total * sv));
  }
  if ((d.fam == FAM_BLOCK_TOTAL || d.fam == FAM_BLOCK_OFFSET || (d.fam == FAM_COMPOSE && d.has_b)) && d.n_bmtb) {
    std::vector<int64_t> st;
    if (d.bmtb_start) st = widen(d2h<int32_t>(d.bmtb_start, d.n_bmtb + 1));
    else
      for (int64_t b = 0; b <= d.n_bmtb; ++b) st.push_back(std::min(b * d.k1, d.nnz_p));
    put_i("bmtb.nz_ptr", st);
    put_i("bmtb.first_row", widen(d2h<int32_t>(d.bmtb_first_row, d.n_bmtb)));
  }
  (void)P;
  (void)part;
}

}  // namespace

std::vector<std::pair<std::string, std::vector<uint8_t>>> device_arrays(const Plan& P) {
  std::vector<std::pair<std::string, std::vector<uint8_t>>> all;
  if (P.device < 0) return all;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(P.device);
  check_cuda(cudaDeviceSynchronize(), "readback sync");
  for (size_t i = 0; i < P.launches.size(); ++i) {
    std::vector<std::pair<std::string, std::vector<uint8_t>>> one;
    part_arrays(P, P.launches[i], P.launch_part[i], one);
    for (auto& kv : one) all.push_back({"dev.p" + std::to_string(P.launch_part[i]) + "." + kv.first, std::move(kv.second)});
  }
  // the writer rule's pre-pass rows (A22) as uploaded
  all.push_back({"dev.prepass", bytes(widen(d2h<int32_t>(P.d_prepass, P.n_prepass)))});
  cudaSetDevice(cur);
  return all;
}

}  // namespace as
