// On-device Designer for the NNZ-blocked graph family (SURVEY N10 / §7 hard parts: "must be
// on-device (CUB sort/scan)").  The host builder (builder.cpp) executes any Operator Graph on
// the Matrix Metadata Set (§V-A) with multithreaded loops over every nonzero; at
// 10^8-10^9 nonzeros that makes as_plan take seconds and starves as_search (the search
// should be dominated by running SpMV programs, not by building them).  This file builds the
// same format on the GPU for graphs of the shape
//
//   [SORT | SORT_SUB(g)]; COMPRESS; [BMW_NNZ_BLOCK(K)]; BMT_NNZ_BLOCK(k); [BMT_PAD(GLOBAL|BMW, vec)];
//   THREAD_BITMAP_RED_G; [WARP_SEG_ADD_RED | WARP_BITMAP_RED]; [SET_RESOURCE]; GMEM_ATOM_RED
//
// (CSR5-like tiles, the searched winners of C3 and C5), every step the reading the host
// builder implements:
//   SORT / SORT_SUB (A7, A8)   stable radix sort of (group, ~row length) keys (CUB)
//   COMPRESS (A14, A6)         flagged select of non-empty rows, exclusive scan of lengths,
//                              warp-per-row gather of columns and values
//   NNZ block cutting (A15)    arithmetic: BMW w = [wK, (w+1)K), BMT j of BMW w = [wK + jk, ...)
//                              (children restart at every parent)
//   first_row (A15)            binary search of every BMT start in the compacted row_ptr
//   bitmaps (A20)              atomicOr of every row head into its BMT's words
//   BMT_PAD (A18)              slot-major interleaved fill, pad col = the BMT's last column
//   writer rule (A22)          a row is exclusive iff its first and last nonzero fall in the
//                              same writer unit (BMW with a warp reduction, else BMT); the
//                              pre-pass lists atomic rows and rows no part writes
//   fp32 heavy rows (A25)      rows spanning more than 167 writer units
//   xcache (R-xcache)          column histogram, top-K by (count desc, column asc), ~slot code
// into device arrays laid out exactly as Plan::upload lays out the host build (short-array
// fusion included; Model-Driven Format Compression is not applied here: the arrays are
// stored).  The canonical CSR is uploaded once per (matrix, device) and cached, so every
// candidate of a search reuses it.  tests/test_gpu.py checks the device-built arrays ("dev."
// readback keys, decoded) against the oracle byte for byte and the y against the oracle;
// AS_HOST_BUILD=1 forces the host builder (A/B).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "plan.h"

namespace as {

// ------------------------------------------------------------------ canonical CSR cache
struct DevCsr {
  int device = -1;
  as_dtype_t dt = AS_R64F;
  int64_t* rp = nullptr;  // m + 1
  int32_t* col = nullptr;
  void* val = nullptr;
  ~DevCsr() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    dev_free(rp, nullptr);
    dev_free(col, nullptr);
    dev_free(val, nullptr);
    cudaSetDevice(cur);
  }
};

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? AS_ERR_OOM : AS_ERR_CUDA, std::string("device build: ") + what + ": " +
                                                                         cudaGetErrorString(e));
  }
}

// scratch owned by one build (freed on scope exit)
struct Scratch {
  std::vector<void*> p;
  cudaStream_t s;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <class T>
  T* get(size_t n) {
    void* d = dev_alloc(std::max<size_t>(n * sizeof(T), 16), s);
    p.push_back(d);
    return (T*)d;
  }
  ~Scratch() {
    cudaStreamSynchronize(s);
    for (void* d : p) dev_free(d, s);
  }
};

constexpr int TPB = 256;
inline unsigned blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + TPB - 1) / TPB, 148 * 32)); }
__device__ __forceinline__ int64_t gtid_() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gthr_() { return (int64_t)gridDim.x * blockDim.x; }

// NNZ block geometry (A15): BMW w = [wK, min((w+1)K, nnz)); its BMTs restart at wK in steps of k.
struct Geo {
  int64_t nnz, K, k, bpw;  // K = 0: no BMW level; bpw = BMTs per full BMW
  __host__ __device__ int64_t bmt_of(int64_t e) const { return K ? (e / K) * bpw + (e % K) / k : e / k; }
  __host__ __device__ int64_t start(int64_t t) const { return K ? (t / bpw) * K + (t % bpw) * k : t * k; }
  __host__ __device__ int64_t end(int64_t t) const {
    const int64_t s = start(t);
    int64_t be = K ? (t / bpw + 1) * K : nnz;
    if (be > nnz) be = nnz;
    return s + k < be ? s + k : be;
  }
};

__global__ void k_len(const int64_t* __restrict__ rp, int64_t m, uint32_t* __restrict__ len) {
  for (int64_t i = gtid_(); i < m; i += gthr_()) len[i] = (uint32_t)(rp[i + 1] - rp[i]);
}
// SORT / SORT_SUB key: group in the high word, ~length in the low word; an LSD radix sort is
// stable, so equal lengths keep their row order (A7, A8)
__global__ void k_sort_keys(const uint32_t* __restrict__ len, int64_t m, int64_t g, uint64_t* __restrict__ key,
                            int32_t* __restrict__ idx) {
  for (int64_t i = gtid_(); i < m; i += gthr_()) {
    key[i] = ((uint64_t)(i / g) << 32) | (uint64_t)(0xFFFFFFFFu - len[i]);
    idx[i] = (int32_t)i;
  }
}
__global__ void k_nonempty(const uint32_t* __restrict__ len, const int32_t* __restrict__ perm, int64_t m,
                           uint8_t* __restrict__ flag) {
  for (int64_t i = gtid_(); i < m; i += gthr_()) flag[i] = len[perm ? perm[i] : i] > 0;
}
__global__ void k_clen(const uint32_t* __restrict__ len, const int32_t* __restrict__ origin, int64_t mp,
                       int64_t* __restrict__ clen) {
  for (int64_t i = gtid_(); i <= mp; i += gthr_()) clen[i] = i < mp ? (int64_t)len[origin[i]] : 0;
}
// COMPRESS gather: warp per row
template <class V>
__global__ void k_gather_rows(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, const V* __restrict__ val,
                              const int32_t* __restrict__ origin, const int64_t* __restrict__ rpc, int64_t mp,
                              int32_t* __restrict__ col_c, V* __restrict__ val_c) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = gtid_() >> 5; i < mp; i += gthr_() >> 5) {
    const int64_t a = rp[origin[i]], o = rpc[i], n = rpc[i + 1] - o;
    for (int64_t j = lane; j < n; j += 32) {
      col_c[o + j] = col[a + j];
      val_c[o + j] = val[a + j];
    }
  }
}
__device__ __forceinline__ int64_t upper_row(const int64_t* __restrict__ rpc, int64_t mp, int64_t e) {
  int64_t lo = 0, hi = mp;  // last i with rpc[i] <= e
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (rpc[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
// first_row of every BMT + the bitmap words (fused: {first_row, bm0, ...} every S words)
__global__ void k_first_row(const int64_t* __restrict__ rpc, int64_t mp, Geo geo, int64_t n_bmt, int32_t* __restrict__ fr,
                            int64_t fstride) {
  for (int64_t t = gtid_(); t < n_bmt; t += gthr_()) fr[t * fstride] = (int32_t)upper_row(rpc, mp, geo.start(t));
}
__global__ void k_bitmap(const int64_t* __restrict__ rpc, int64_t mp, Geo geo, uint32_t* __restrict__ bm, int64_t bstride) {
  for (int64_t i = gtid_(); i < mp; i += gthr_()) {
    const int64_t h = rpc[i], t = geo.bmt_of(h), j = h - geo.start(t);
    atomicOr(bm + t * bstride + (j >> 5), 1u << (j & 31));
  }
}
__global__ void k_bmt_start(Geo geo, int64_t n_bmt, int32_t* __restrict__ st) {
  for (int64_t t = gtid_(); t <= n_bmt; t += gthr_()) st[t] = (int32_t)(t < n_bmt ? geo.start(t) : geo.nnz);
}
// column histogram (distinct columns of the bytes model; xcache ranking)
__global__ void k_hist(const int32_t* __restrict__ col, int64_t nnz, int32_t* __restrict__ cnt) {
  for (int64_t e = gtid_(); e < nnz; e += gthr_()) atomicAdd(cnt + col[e], 1);
}
__global__ void k_hot_keys(const int32_t* __restrict__ cnt, int64_t n, uint64_t* __restrict__ key,
                           unsigned long long* __restrict__ distinct) {
  unsigned long long d = 0;
  for (int64_t c = gtid_(); c < n; c += gthr_()) {
    key[c] = ((uint64_t)(0xFFFFFFFFu - (uint32_t)cnt[c]) << 32) | (uint64_t)c;
    d += cnt[c] > 0;
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if ((threadIdx.x & 31) == 0 && d) atomicAdd(distinct, d);
}
__global__ void k_low_word(const uint64_t* __restrict__ key, int64_t K, int32_t* __restrict__ out) {
  for (int64_t i = gtid_(); i < K; i += gthr_()) out[i] = (int32_t)(uint32_t)key[i];
}
__global__ void k_slot(const int32_t* __restrict__ hot, int64_t K, int32_t* __restrict__ slot) {
  for (int64_t i = gtid_(); i < K; i += gthr_()) slot[hot[i]] = (int32_t)i;
}
__device__ __forceinline__ int32_t enc(const int32_t* __restrict__ slot, int32_t c) {
  if (!slot) return c;
  const int32_t s = slot[c];
  return s >= 0 ? ~s : c;
}
template <class V>
__global__ void k_copy_cv(const int32_t* __restrict__ col, const V* __restrict__ val, int64_t nnz,
                          const int32_t* __restrict__ slot, int32_t* __restrict__ col_o, V* __restrict__ val_o) {
  for (int64_t e = gtid_(); e < nnz; e += gthr_()) {
    col_o[e] = enc(slot, col[e]);
    val_o[e] = val[e];
  }
}
// BMT_PAD fill (A18) in slot order (coalesced writes).  Groups: GLOBAL = one group of every
// BMT; BMW scope = the BMTs of each BMW.  Full groups hold bpw BMTs of width Wf; the last
// group may be smaller (nt_l BMTs of width W_l).
template <class V>
__global__ void k_pad_fill(Geo geo, int64_t n_grp, int64_t bpg, int64_t Wf, int64_t Wl, int64_t vec,
                           int64_t total, const int32_t* __restrict__ col, const V* __restrict__ val,
                           const int32_t* __restrict__ slot, int32_t* __restrict__ pcol, V* __restrict__ pval,
                           int64_t n_bmt) {
  const int64_t full = (n_grp - 1) * bpg * Wf;  // slots of the full groups
  for (int64_t s = gtid_(); s < total; s += gthr_()) {
    int64_t g, rel, nt, W;
    if (s < full) {
      g = s / (bpg * Wf);
      rel = s - g * bpg * Wf;
      nt = bpg;
      W = Wf;
    } else {
      g = n_grp - 1;
      rel = s - full;
      nt = n_bmt - g * bpg;
      W = Wl;
    }
    (void)W;
    const int64_t chunk = rel / (nt * vec), within = rel - chunk * nt * vec;
    const int64_t lt = within / vec, j = chunk * vec + within % vec;
    const int64_t t = g * bpg + lt;
    const int64_t a = geo.start(t), e = geo.end(t);
    if (a + j < e) {
      pcol[s] = enc(slot, col[a + j]);
      pval[s] = val[a + j];
    } else {
      pcol[s] = enc(slot, col[e - 1]);
      pval[s] = (V)0;
    }
  }
}
// writer rule (A22) of the single part: exclusive iff first and last nonzero in one unit;
// pre[r] = 1 for atomic rows and rows never written (empty); fp32: heavy = span > 167 (A25)
__global__ void k_writer(const int64_t* __restrict__ rpc, const int32_t* __restrict__ origin, int64_t base, int64_t mp,
                         Geo geo, int unit_bmw, uint8_t* __restrict__ pre, uint8_t* __restrict__ heavy,
                         unsigned long long* __restrict__ n_atom) {
  unsigned long long na = 0;
  for (int64_t i = gtid_(); i < mp; i += gthr_()) {
    const int64_t a = rpc[i], e = rpc[i + 1];
    const int64_t ua = unit_bmw ? a / geo.K : geo.bmt_of(a), ue = unit_bmw ? (e - 1) / geo.K : geo.bmt_of(e - 1);
    const int64_t r = origin ? origin[i] : base + i;
    const bool at = ua != ue;
    pre[r] = at;
    na += at;
    if (heavy && ue - ua + 1 > 167) heavy[r] = 1;
  }
  for (int o = 16; o; o >>= 1) na += __shfl_down_sync(0xffffffffu, na, o);
  if ((threadIdx.x & 31) == 0 && na) atomicAdd(n_atom, na);
}
__global__ void k_heavy_bits(const int32_t* __restrict__ rows, int64_t n, uint32_t* __restrict__ bits) {
  for (int64_t i = gtid_(); i < n; i += gthr_()) atomicOr(bits + (rows[i] >> 5), 1u << (rows[i] & 31));
}
__global__ void k_scatter_stride(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ out, int64_t stride) {
  for (int64_t i = gtid_(); i < n; i += gthr_()) out[i * stride] = in[i];
}
__global__ void k_widen_f32(const double* __restrict__ in, int64_t n, float* __restrict__ out) {
  for (int64_t i = gtid_(); i < n; i += gthr_()) out[i] = (float)in[i];
}

// Model-Driven Format Compression of a device int32 array (the host's fit_array_model on a
// copy; the fit rejects random data after a few elements)
bool fit_model_d2h(const int32_t* d, int64_t n, cudaStream_t s, IdxModel* out) {
  if (n < 2) return false;
  if (n > 8192) {  // probe: the first 4096 entries + the mid and last pairs decide most arrays
    std::vector<int32_t> pre(4096), q(4);
    ck(cudaMemcpyAsync(pre.data(), d, 4096 * 4, cudaMemcpyDeviceToHost, s), "model probe");
    ck(cudaMemcpyAsync(q.data(), d + n / 2, 8, cudaMemcpyDeviceToHost, s), "model probe");
    ck(cudaMemcpyAsync(q.data() + 2, d + n - 2, 8, cudaMemcpyDeviceToHost, s), "model probe");
    ck(cudaStreamSynchronize(s), "model probe sync");
    if (!model_may_fit(std::vector<int64_t>(pre.begin(), pre.end()), n, q[0], q[1], q[2], q[3], kMaxPatches))
      return false;
  }
  std::vector<int32_t> h((size_t)n);
  ck(cudaMemcpyAsync(h.data(), d, (size_t)n * 4, cudaMemcpyDeviceToHost, s), "model d2h");
  ck(cudaStreamSynchronize(s), "model d2h sync");
  return fit_array_model(std::vector<int64_t>(h.begin(), h.end()), kMaxPatches, out);
}

// select the indices i in [0, n) with flag[i] != 0 (ascending) into a new int32 array
int32_t* select_flagged(Scratch& S, const uint8_t* flag, int64_t n, int64_t* count, cudaStream_t s,
                        bool keep, Plan* P) {
  int64_t* d_cnt = S.get<int64_t>(1);
  thrust::counting_iterator<int32_t> it(0);
  size_t tmp = 0;
  ck(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag, (int32_t*)nullptr, d_cnt, n, s), "select size");
  void* t = S.get<uint8_t>(tmp);
  int32_t* out = keep ? (int32_t*)P->up(nullptr, 0, s, (size_t)n * 4) : S.get<int32_t>((size_t)n);
  ck(cub::DeviceSelect::Flagged(t, tmp, it, flag, out, d_cnt, n, s), "select");
  ck(cudaMemcpyAsync(count, d_cnt, 8, cudaMemcpyDeviceToHost, s), "select count");
  ck(cudaStreamSynchronize(s), "select sync");
  return out;
}

}  // namespace

// ------------------------------------------------------------------ eligibility
bool dev_build_spec(const Seq& g, const Matrix& A, int flags, DevSpec* sp) {
  if (std::getenv("AS_HOST_BUILD") || std::getenv("AS_NT_LEGACY")) return false;
  if (flags & (AS_PLAN_KEEP_HOST | AS_PLAN_SPMM | AS_PLAN_HOST_BUILD)) return false;
  if (A.nnz() == 0 || A.m >= INT32_MAX || A.n >= INT32_MAX) return false;
  DevSpec d;
  size_t i = 0;
  if (i < g.size() && g[i].name == "SORT") {
    d.sort = 1;
    ++i;
  } else if (i < g.size() && g[i].name == "SORT_SUB") {
    d.sort = 2;
    d.g = g[i].geti("g");
    ++i;
  }
  if (i >= g.size() || g[i].name != "COMPRESS") return false;
  ++i;
  if (i < g.size() && g[i].name == "BMW_NNZ_BLOCK") {
    d.K = g[i].params[0].second.i;
    ++i;
  }
  if (i >= g.size() || g[i].name != "BMT_NNZ_BLOCK") return false;
  d.k = g[i].params[0].second.i;
  ++i;
  if (i < g.size() && g[i].name == "BMT_PAD") {
    const std::string& sc = g[i].gets("scope");
    if (sc == "GLOBAL") d.pad_scope = -1;
    else if (sc == "BMW" && d.K) d.pad_scope = 1;
    else return false;
    d.pad = true;
    d.vec = g[i].geti("vec");
    if (d.vec == 0) d.vec = A.dt == AS_R64F ? 2 : 4;
    ++i;
  }
  bool tb = false, gm = false;
  for (; i < g.size(); ++i) {
    const std::string& nm = g[i].name;
    if (nm == "THREAD_BITMAP_RED_G") tb = true;
    else if (nm == "WARP_SEG_ADD_RED") d.wred = RED_SEG;
    else if (nm == "WARP_BITMAP_RED") d.wred = RED_BITMAP;
    else if (nm == "GMEM_ATOM_RED") gm = true;
    else if (nm == "SET_RESOURCE") {
      d.tpb = (int)g[i].geti("tpb");
      d.grid = (int)g[i].geti("grid");
      d.stages = (int)g[i].geti("stages");
      d.xcache = g[i].geti("xcache");
    } else {
      return false;
    }
  }
  if (!tb || !gm) return false;
  if (d.K && d.wred == RED_NONE) return false;  // composed kernel (host lowering)
  if (!d.K && d.wred != RED_NONE) return false;
  // forms the host upload derives from the host arrays: the warp tile kernel and x windows
  if (d.K && !d.pad && (d.k == 1 || d.k == 2 || d.k == 4) && d.K % (32 * d.k) == 0 && d.xcache == 0) return false;
  if (!d.K && d.stages == 2 && d.xcache == 0) return false;
  *sp = d;
  return true;
}

// ------------------------------------------------------------------ the build
void dev_build(Plan& P, const Matrix& A, const DevSpec& sp, cudaStream_t s) {
  const int64_t m = A.m, n = A.n, nnz = A.nnz();
  const bool f64 = A.dt == AS_R64F;
  const int64_t sv = f64 ? 8 : 4;
  // canonical CSR, uploaded once per (matrix, device); the cache slot is shared by threads
  // planning the same matrix, so it is read and replaced under a lock (the upload itself runs
  // outside it: two threads may both upload, the later one's copy is kept)
  static std::mutex cache_mu;
  std::shared_ptr<DevCsr> C;
  {
    std::lock_guard<std::mutex> lk(cache_mu);
    C = A.dcache;
  }
  if (!C || C->device != P.device) {
    C = std::make_shared<DevCsr>();
    C->device = P.device;
    C->dt = A.dt;
    C->rp = (int64_t*)dev_alloc((size_t)(m + 1) * 8, nullptr);
    C->col = (int32_t*)dev_alloc((size_t)nnz * 4 + 64, nullptr);
    C->val = dev_alloc((size_t)nnz * sv + 64, nullptr);
    ck(cudaMemcpyAsync(C->rp, A.row_ptr.data(), (size_t)(m + 1) * 8, cudaMemcpyHostToDevice, s), "upload row_ptr");
    ck(cudaMemcpyAsync(C->col, A.col.data(), (size_t)nnz * 4, cudaMemcpyHostToDevice, s), "upload col");
    if (f64) {
      ck(cudaMemcpyAsync(C->val, A.val.data(), (size_t)nnz * 8, cudaMemcpyHostToDevice, s), "upload val");
    } else {  // fp32: widened copies on the host are exact; narrow on the device in chunks
      Scratch S(s);
      const int64_t ch = int64_t(1) << 25;
      double* buf = S.get<double>((size_t)std::min(nnz, ch));
      for (int64_t a = 0; a < nnz; a += ch) {
        const int64_t c = std::min(ch, nnz - a);
        ck(cudaMemcpyAsync(buf, A.val.data() + a, (size_t)c * 8, cudaMemcpyHostToDevice, s), "upload val");
        k_widen_f32<<<blocks(c), TPB, 0, s>>>(buf, c, (float*)C->val + a);
      }
    }
    ck(cudaStreamSynchronize(s), "upload csr");
    if (!std::getenv("AS_NO_DEV_CACHE")) {
      std::lock_guard<std::mutex> lk(cache_mu);
      A.dcache = C;
    }
  }
  Scratch S(s);
  // row lengths, SORT / SORT_SUB permutation, COMPRESS
  uint32_t* len = S.get<uint32_t>((size_t)m);
  k_len<<<blocks(m), TPB, 0, s>>>(C->rp, m, len);
  int32_t* perm = nullptr;
  if (sp.sort) {
    const int64_t g = sp.sort == 1 ? m : std::max<int64_t>(sp.g, 1);
    const int64_t ng = (m + g - 1) / g;
    int hb = 0;
    while ((int64_t(1) << hb) < ng) ++hb;
    uint64_t *k0 = S.get<uint64_t>((size_t)m), *k1 = S.get<uint64_t>((size_t)m);
    int32_t *v0 = S.get<int32_t>((size_t)m);
    perm = S.get<int32_t>((size_t)m);
    k_sort_keys<<<blocks(m), TPB, 0, s>>>(len, m, g, k0, v0);
    size_t tmp = 0;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, perm, m, 0, 32 + hb, s), "sort size");
    void* t = S.get<uint8_t>(tmp);
    ck(cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, perm, m, 0, 32 + hb, s), "sort");
  }
  uint8_t* flag = S.get<uint8_t>((size_t)m);
  k_nonempty<<<blocks(m), TPB, 0, s>>>(len, perm, m, flag);
  int64_t mp = 0;
  int32_t* origin = nullptr;
  {
    int64_t* d_cnt = S.get<int64_t>(1);
    size_t tmp = 0;
    int32_t* out = S.get<int32_t>((size_t)m);
    if (perm) {
      ck(cub::DeviceSelect::Flagged(nullptr, tmp, perm, flag, out, d_cnt, m, s), "compress size");
      void* t = S.get<uint8_t>(tmp);
      ck(cub::DeviceSelect::Flagged(t, tmp, perm, flag, out, d_cnt, m, s), "compress");
    } else {
      thrust::counting_iterator<int32_t> it(0);
      ck(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag, out, d_cnt, m, s), "compress size");
      void* t = S.get<uint8_t>(tmp);
      ck(cub::DeviceSelect::Flagged(t, tmp, it, flag, out, d_cnt, m, s), "compress");
    }
    ck(cudaMemcpyAsync(&mp, d_cnt, 8, cudaMemcpyDeviceToHost, s), "compress count");
    ck(cudaStreamSynchronize(s), "compress sync");
    origin = out;
  }
  // origin_rows implicit when affine (no permutation, no empty row: origin = row)
  const bool affine = !perm && mp == m;
  int64_t* rpc = C->rp;
  if (!affine) {
    int64_t* clen = S.get<int64_t>((size_t)mp + 1);
    rpc = S.get<int64_t>((size_t)mp + 1);
    k_clen<<<blocks(mp + 1), TPB, 0, s>>>(len, origin, mp, clen);
    size_t tmp = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp, clen, rpc, mp + 1, s), "scan size");
    void* t = S.get<uint8_t>(tmp);
    ck(cub::DeviceScan::ExclusiveSum(t, tmp, clen, rpc, mp + 1, s), "scan");
  }
  // compacted columns / values: the canonical arrays unless rows were permuted
  const int32_t* col_c = C->col;
  const void* val_c = C->val;
  if (perm) {
    int32_t* cc = S.get<int32_t>((size_t)nnz);
    void* vc = S.get<uint8_t>((size_t)(nnz * sv));
    if (f64) k_gather_rows<double><<<blocks(mp * 32), TPB, 0, s>>>(C->rp, C->col, (const double*)C->val, origin, rpc, mp, cc, (double*)vc);
    else k_gather_rows<float><<<blocks(mp * 32), TPB, 0, s>>>(C->rp, C->col, (const float*)C->val, origin, rpc, mp, cc, (float*)vc);
    col_c = cc;
    val_c = vc;
  }

  // part descriptor (mirrors Plan::upload for FAM_NNZ_THREAD / FAM_NNZ_WARP)
  HostPart hp;
  hp.kind = "csr";
  hp.fam = sp.K ? FAM_NNZ_WARP : FAM_NNZ_THREAD;
  hp.fam_name = sp.K ? (sp.wred == RED_SEG ? "nnz_warp_seg" : "nnz_warp_bitmap") : "nnz_thread_bitmap";
  hp.mode = 0;
  hp.red[2] = RED_BITMAP;
  hp.red[1] = (Red)sp.wred;
  double bytes_model = 0;
  DevPart d;
  d.fam = hp.fam;
  d.dtype = f64 ? 1 : 0;
  d.mode = 0;
  d.tpb = sp.tpb > 0 ? sp.tpb : 256;
  d.grid = sp.grid;
  d.n = n;
  d.m_p = mp;
  d.nnz_p = nnz;
  const bool mdc = !std::getenv("AS_NO_MDC");  // Model-Driven Format Compression (as Plan::upload)
  if (affine) {
    d.origin_base = 0;
  } else if (mdc && fit_model_d2h(origin, mp, s, &d.org_model)) {
    ++P.modeled_arrays;
  } else {
    d.origin = (const int32_t*)P.up(nullptr, 0, s, (size_t)mp * 4);
    ck(cudaMemcpyAsync((void*)d.origin, origin, (size_t)mp * 4, cudaMemcpyDeviceToDevice, s), "origin");
    bytes_model += (double)(mp * 4);
  }
  Geo geo{nnz, sp.K, sp.k, sp.K ? (sp.K + sp.k - 1) / sp.k : 0};
  const int64_t nbmw = sp.K ? (nnz + sp.K - 1) / sp.K : 0;
  const int64_t n_bmt = sp.K ? (nnz / sp.K) * geo.bpw + ((nnz % sp.K) + sp.k - 1) / sp.k : (nnz + sp.k - 1) / sp.k;
  d.n_bmt = n_bmt;
  d.k = sp.k;
  const bool st_affine = !sp.K || sp.K % sp.k == 0 || nnz <= sp.K;
  if (!st_affine) {
    if (nnz >= INT32_MAX) fail(AS_ERR_PLAN_INFEASIBLE, "bmt_start exceeds int32 (reading A36)");
    int32_t* st = (int32_t*)P.up(nullptr, 0, s, (size_t)(n_bmt + 1) * 4);
    k_bmt_start<<<blocks(n_bmt + 1), TPB, 0, s>>>(geo, n_bmt, st);
    d.bmt_start = st;
    bytes_model += (double)((n_bmt + 1) * 4);
  }
  const int bmw_words = (int)((sp.k + 31) / 32);
  d.bm_words = bmw_words;
  const bool fuse = !std::getenv("AS_NO_FUSE") && bmw_words >= 1 && bmw_words <= 3;
  int32_t* fr_tmp = S.get<int32_t>((size_t)n_bmt);
  k_first_row<<<blocks(n_bmt), TPB, 0, s>>>(rpc, mp, geo, n_bmt, fr_tmp, 1);
  if (mdc && fit_model_d2h(fr_tmp, n_bmt, s, &d.fr_model)) {
    ++P.modeled_arrays;  // first rows computed, not loaded (NEXT-2); bitmap stored alone
    uint32_t* bm = (uint32_t*)P.up(nullptr, 0, s, (size_t)(n_bmt * bmw_words) * 4);
    k_bitmap<<<blocks(mp), TPB, 0, s>>>(rpc, mp, geo, bm, bmw_words);
    d.bitmap = bm;
    d.bm_stride = bmw_words;
    bytes_model += (double)(n_bmt * bmw_words * 4);
  } else if (fuse) {  // short-array fusion: {first_row, bm0[, bm1[, bm2]]} per BMT
    const int S4 = bmw_words + 1 <= 2 ? 2 : 4;
    int32_t* f = (int32_t*)P.up(nullptr, 0, s, (size_t)(n_bmt * S4) * 4);  // zero-filled
    k_scatter_stride<<<blocks(n_bmt), TPB, 0, s>>>(fr_tmp, n_bmt, f, S4);
    k_bitmap<<<blocks(mp), TPB, 0, s>>>(rpc, mp, geo, (uint32_t*)(f + 1), S4);
    d.bmt_first_row = f;
    d.bitmap = (const uint32_t*)(f + 1);
    d.fr_stride = d.bm_stride = S4;
    ++P.fused_arrays;
    bytes_model += (double)(n_bmt * S4 * 4);
  } else {
    int32_t* fr = (int32_t*)P.up(nullptr, 0, s, (size_t)n_bmt * 4);
    uint32_t* bm = (uint32_t*)P.up(nullptr, 0, s, (size_t)(n_bmt * bmw_words) * 4);
    ck(cudaMemcpyAsync(fr, fr_tmp, (size_t)n_bmt * 4, cudaMemcpyDeviceToDevice, s), "first_row");
    k_bitmap<<<blocks(mp), TPB, 0, s>>>(rpc, mp, geo, bm, bmw_words);
    d.bmt_first_row = fr;
    d.bitmap = bm;
    d.bm_stride = bmw_words;
    bytes_model += (double)(n_bmt * 4 + n_bmt * bmw_words * 4);
  }
  // column histogram: distinct columns (x bytes) and the xcache ranking
  int32_t* cnt = S.get<int32_t>((size_t)n);
  ck(cudaMemsetAsync(cnt, 0, (size_t)n * 4, s), "hist memset");
  k_hist<<<blocks(nnz), TPB, 0, s>>>(C->col, nnz, cnt);
  uint64_t* hkey = S.get<uint64_t>((size_t)n);
  unsigned long long* d_dist = S.get<unsigned long long>(2);
  ck(cudaMemsetAsync(d_dist, 0, 16, s), "memset");
  k_hot_keys<<<blocks(n), TPB, 0, s>>>(cnt, n, hkey, d_dist);
  unsigned long long distinct = 0;
  ck(cudaMemcpyAsync(&distinct, d_dist, 8, cudaMemcpyDeviceToHost, s), "distinct");
  ck(cudaStreamSynchronize(s), "hist sync");
  const int32_t* slot = nullptr;
  int64_t K = 0;
  if (sp.xcache > 0) {
    const int64_t cap = (device_max_smem_optin(P.device) - 1024) / sv;
    K = std::min<int64_t>({sp.xcache, cap, (int64_t)distinct});
  }
  if (K > 0) {
    uint64_t* hk2 = S.get<uint64_t>((size_t)n);
    size_t tmp = 0;
    ck(cub::DeviceRadixSort::SortKeys(nullptr, tmp, hkey, hk2, n, 0, 64, s), "hot sort size");
    void* t = S.get<uint8_t>(tmp);
    ck(cub::DeviceRadixSort::SortKeys(t, tmp, hkey, hk2, n, 0, 64, s), "hot sort");
    int32_t* hot = S.get<int32_t>((size_t)K);
    k_low_word<<<blocks(K), TPB, 0, s>>>(hk2, K, hot);
    int32_t* hot_sorted = (int32_t*)P.up(nullptr, 0, s, (size_t)K * 4);
    tmp = 0;
    ck(cub::DeviceRadixSort::SortKeys(nullptr, tmp, hot, hot_sorted, K, 0, 32, s), "hot cols size");
    void* t2 = S.get<uint8_t>(tmp);
    ck(cub::DeviceRadixSort::SortKeys(t2, tmp, hot, hot_sorted, K, 0, 32, s), "hot cols");
    int32_t* sl = S.get<int32_t>((size_t)n);
    ck(cudaMemsetAsync(sl, 0xFF, (size_t)n * 4, s), "slot memset");
    k_slot<<<blocks(K), TPB, 0, s>>>(hot_sorted, K, sl);
    slot = sl;
    d.xh_cols = hot_sorted;
    d.xh_n = K;
    bytes_model += (double)(K * 4);
  }
  // values / columns: BMT_PAD slot-major tiles, or the compacted arrays (xcache-encoded)
  int64_t slots = nnz;
  if (sp.pad) {
    const int64_t vec = sp.vec;
    auto rup = [&](int64_t w) { return (w + vec - 1) / vec * vec; };
    int64_t n_grp, bpg, Wf, Wl;
    if (sp.pad_scope < 0) {  // GLOBAL: one group, width = the longest BMT
      n_grp = 1;
      bpg = n_bmt;
      const int64_t full_len = sp.K ? std::min(sp.k, sp.K) : sp.k;
      int64_t mx = std::min(full_len, nnz);
      if (sp.K && nnz >= sp.K) mx = std::max(mx, std::min(sp.k, sp.K));
      Wf = Wl = rup(mx);
    } else {  // BMW scope: one group per BMW
      n_grp = nbmw;
      bpg = geo.bpw;
      Wf = rup(std::min(sp.k, sp.K));
      const int64_t rem = nnz - (nbmw - 1) * sp.K;
      Wl = rup(std::min(sp.k, rem));
      if (n_grp == 1) Wf = Wl;
    }
    const int64_t nt_last = n_bmt - (n_grp - 1) * bpg;
    const int64_t total = (n_grp - 1) * bpg * Wf + nt_last * Wl;
    if (total > 4 * nnz + (int64_t(1) << 20))
      fail(AS_ERR_PLAN_INFEASIBLE, "P4b: BMT_PAD would store " + std::to_string(total) + " slots");
    std::vector<int32_t> gfirst((size_t)n_grp + 1), gw((size_t)n_grp);
    std::vector<int64_t> gbase((size_t)n_grp);
    for (int64_t g = 0; g < n_grp; ++g) {
      gfirst[(size_t)g] = (int32_t)(g * bpg);
      gw[(size_t)g] = (int32_t)(g + 1 < n_grp ? Wf : Wl);
      gbase[(size_t)g] = g * bpg * Wf;
    }
    gfirst[(size_t)n_grp] = (int32_t)n_bmt;
    d.pad = 1;
    d.vec = (int)vec;
    d.n_grp = n_grp;
    d.grp_regular = bpg;
    d.grp_first_bmt = (const int32_t*)P.up(gfirst.data(), gfirst.size() * 4, s);
    double saved = 0;  // per-group slot base and pad_width as models (as Plan::upload_pad)
    if (mdc && fit_array_model(gbase, kMaxPatches, &d.pb_model)) {
      ++P.modeled_arrays;
      saved += (double)n_grp * 8;
    } else {
      d.grp_base = (const int64_t*)P.up(gbase.data(), gbase.size() * 8, s);
    }
    std::vector<int64_t> gw64(gw.begin(), gw.end());
    if (mdc && fit_array_model(gw64, kMaxPatches, &d.pw_model)) {
      ++P.modeled_arrays;
      saved += (double)n_grp * 4;
    } else {
      d.grp_width = (const int32_t*)P.up(gw.data(), gw.size() * 4, s);
    }
    bytes_model -= saved;
    int32_t* pcol = (int32_t*)P.up(nullptr, 0, s, (size_t)total * 4);
    void* pval = P.up(nullptr, 0, s, (size_t)(total * sv));
    if (f64) k_pad_fill<double><<<blocks(total), TPB, 0, s>>>(geo, n_grp, bpg, Wf, Wl, vec, total, col_c, (const double*)val_c, slot, pcol, (double*)pval, n_bmt);
    else k_pad_fill<float><<<blocks(total), TPB, 0, s>>>(geo, n_grp, bpg, Wf, Wl, vec, total, col_c, (const float*)val_c, slot, pcol, (float*)pval, n_bmt);
    ck(cudaStreamSynchronize(s), "pad fill");  // host vectors above die at scope exit
    d.pad_col = pcol;
    d.pad_val = pval;
    d.pad_grp_bmw = (hp.fam == FAM_NNZ_WARP && sp.pad_scope == 1) ? 1 : 0;
    bytes_model += (double)(total * 4 + total * sv + n_grp * 12);
    slots = total;
  } else {
    int32_t* co = (int32_t*)P.up(nullptr, 0, s, (size_t)nnz * 4);
    void* vo = P.up(nullptr, 0, s, (size_t)(nnz * sv));
    if (f64) k_copy_cv<double><<<blocks(nnz), TPB, 0, s>>>(col_c, (const double*)val_c, nnz, slot, co, (double*)vo);
    else k_copy_cv<float><<<blocks(nnz), TPB, 0, s>>>(col_c, (const float*)val_c, nnz, slot, co, (float*)vo);
    d.col = co;
    d.val = vo;
    bytes_model += (double)(nnz * (4 + sv));
  }
  if (hp.fam == FAM_NNZ_WARP) {
    d.variant = sp.wred == RED_SEG ? 1 : 2;
    d.n_bmw = nbmw;
    d.bmts_per_bmw = nbmw ? std::min(geo.bpw, n_bmt) : 0;
  }
  // writer rule: pre-pass rows, atomic count, fp32 heavy rows
  uint8_t* pre = S.get<uint8_t>((size_t)m);
  ck(cudaMemsetAsync(pre, 1, (size_t)m, s), "pre memset");
  uint8_t* heavy = nullptr;
  if (!f64) {
    heavy = S.get<uint8_t>((size_t)m);
    ck(cudaMemsetAsync(heavy, 0, (size_t)m, s), "heavy memset");
  }
  unsigned long long* d_na = S.get<unsigned long long>(1);
  ck(cudaMemsetAsync(d_na, 0, 8, s), "memset");
  k_writer<<<blocks(mp), TPB, 0, s>>>(rpc, affine ? nullptr : origin, 0, mp, geo, hp.fam == FAM_NNZ_WARP ? 1 : 0, pre,
                                      heavy, d_na);
  unsigned long long n_atom = 0;
  ck(cudaMemcpyAsync(&n_atom, d_na, 8, cudaMemcpyDeviceToHost, s), "atom count");
  int64_t n_pre = 0;
  int32_t* dpre = select_flagged(S, pre, m, &n_pre, s, true, &P);
  if (n_pre) {
    P.d_prepass = dpre;
    P.n_prepass = n_pre;
  }
  d.tpb = sp.tpb > 0 ? sp.tpb : 256;
  ck((cudaError_t)prepare_part(d), "kernel attributes");
  if (d.xh_n) hp.fam_name += "_xh";
  if (heavy) {
    int64_t nh = 0;
    int32_t* rows = select_flagged(S, heavy, m, &nh, s, true, &P);
    if (nh) {
      P.d_heavy_rows = rows;
      P.n_heavy = nh;
      P.d_heavy_acc = (double*)P.up(nullptr, 0, s, (size_t)nh * 8);
      uint32_t* bits = (uint32_t*)P.up(nullptr, 0, s, (size_t)(m / 32 + 1) * 4);
      k_heavy_bits<<<blocks(nh), TPB, 0, s>>>(rows, nh, bits);
      d.heavy_bits = bits;
      d.heavy_rows = rows;
      d.n_heavy = nh;
      d.heavy_acc = P.d_heavy_acc;
    }
  }
  // spans (as_spmv_host pipelining): columns and rows touched
  Plan::Span span{0, n - 1, 0, m - 1};
  {
    int32_t* mm = S.get<int32_t>(4);
    size_t tmp = 0, tmp2 = 0;
    ck(cub::DeviceReduce::Min(nullptr, tmp, C->col, mm, nnz, s), "min size");
    ck(cub::DeviceReduce::Max(nullptr, tmp2, C->col, mm + 1, nnz, s), "max size");
    void* t = S.get<uint8_t>(std::max(tmp, tmp2));
    ck(cub::DeviceReduce::Min(t, tmp, C->col, mm, nnz, s), "min");
    ck(cub::DeviceReduce::Max(t, tmp2, C->col, mm + 1, nnz, s), "max");
    if (origin) {
      ck(cub::DeviceReduce::Min(t, tmp, origin, mm + 2, mp, s), "rmin");
      ck(cub::DeviceReduce::Max(t, tmp2, origin, mm + 3, mp, s), "rmax");
    }
    int32_t h[4];
    ck(cudaMemcpyAsync(h, mm, 16, cudaMemcpyDeviceToHost, s), "span");
    ck(cudaStreamSynchronize(s), "span sync");
    span = Plan::Span{h[0], h[1], h[2], h[3]};
  }
  ck(cudaStreamSynchronize(s), "device build");

  // plan bookkeeping (Plan::upload + Plan::compute_model + make_plan's info, single part)
  const int64_t n_excl = mp - (int64_t)n_atom;
  P.bytes_model = bytes_model;
  P.launches.push_back(d);
  P.launch_part.push_back(0);
  P.launch_stream.push_back(0);  // one part: nothing runs beside it
  P.spans.push_back(span);
  P.launch_bytes.push_back(bytes_model + (double)distinct * sv + (double)n_excl * sv + 2.0 * (double)n_atom * sv);
  P.single_writer = n_pre == 0 && P.n_heavy == 0 && n_atom == 0;
  hp.pad = sp.pad;
  P.host = HostPlan();
  P.host.m = m;
  P.host.n = n;
  P.host.dt = A.dt;
  P.host.distinct_cols = (int64_t)distinct;
  P.host.launch_order = {0};
  P.host.parts.push_back(std::move(hp));
  const double y0 = (double)n_excl * sv + 2.0 * (double)n_atom * sv, y1 = 2.0 * (double)n_excl * sv + 2.0 * (double)n_atom * sv;
  const double pre_d = (double)n_pre;
  const double pb0 = (double)m * sv <= pre_d * (4 + 32) ? (double)m * sv : pre_d * (4 + sv);
  const double pb1 = pre_d * (4 + 2 * sv);
  P.prepass_bytes = n_pre ? pb0 : 0;
  auto& info = P.info;
  info.bytes_model = bytes_model + (double)distinct * sv + y0 + (n_pre ? pb0 : 0);
  info.bytes_model_beta = bytes_model + (double)distinct * sv + y1 + (n_pre ? pb1 : 0);
  info.bytes_floor = (double)(nnz * (sv + 4) + n * sv + m * sv);
  info.nnz_real = nnz;
  info.n_parts = 1;
  info.prepass_rows = n_pre;
  info.n_launches = 1 + (n_pre ? 1 : 0) + (P.n_heavy ? 1 : 0);
  info.stored_slots = slots;
  info.pads = slots - nnz;
  std::string kn = n_pre ? "k_prepass;" : "";
  kn += P.host.parts[0].fam_name;
  if (P.n_heavy) kn += ";k_heavy_epilogue";
  std::strncpy(info.kernels, kn.c_str(), sizeof(info.kernels) - 1);
}

}  // namespace as
