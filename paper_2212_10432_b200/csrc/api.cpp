// C-ABI entry points (include/as.h).  Every call converts internal exceptions to statuses.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "internal.h"
#include "plan.h"

namespace as {
Matrix matrix_from_coo(int64_t, int64_t, int64_t, const int64_t*, const int64_t*, const void*, as_dtype_t, int);
Matrix matrix_from_csr(int64_t, int64_t, const int64_t*, const int32_t*, const void*, as_dtype_t);
Matrix matrix_from_mtx(const char*, as_dtype_t);
as_stats_t matrix_stats(const Matrix&);
Matrix matrix_row_slice(const Matrix&, int64_t, int64_t);
as_status_t search_impl(const Matrix& A, const as_search_cfg_t* cfg, int device, void* stream, as_plan_t* best,
                        char* best_graph, size_t* len);
std::vector<double> matrix_features(const Matrix& A);

namespace {
thread_local std::string g_last_error;
struct AllocHooks {
  void* (*alloc)(size_t, void*, void*) = nullptr;
  void (*release)(void*, void*, void*) = nullptr;
  void* ctx = nullptr;
} g_hooks;
}
void set_last_error(const std::string& m) { g_last_error = m; }

// Every allocation remembers the hooks that made it, so it is released by the same allocator
// even after as_set_allocator changed them (a matrix's cached device CSR or a plan may
// outlive the hooks that were current when it was built).
std::mutex g_owner_mu;
std::unordered_map<void*, AllocHooks> g_owner;

void* dev_alloc(size_t bytes, void* stream) {
  void* d = nullptr;
  const AllocHooks h = g_hooks;
  if (h.alloc) {
    d = h.alloc(bytes, stream, h.ctx);
    if (!d) fail(AS_ERR_OOM, "allocator hook returned NULL for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMalloc(&d, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(e == cudaErrorMemoryAllocation ? AS_ERR_OOM : AS_ERR_CUDA,
           "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
  }
  std::lock_guard<std::mutex> lk(g_owner_mu);
  g_owner[d] = h;
  return d;
}

void dev_free(void* p, void* stream) {
  if (!p) return;
  AllocHooks h = g_hooks;
  {
    std::lock_guard<std::mutex> lk(g_owner_mu);
    auto it = g_owner.find(p);
    if (it != g_owner.end()) {
      h = it->second;
      g_owner.erase(it);
    }
  }
  if (h.release) h.release(p, stream, h.ctx);
  else cudaFree(p);
}

as_status_t copy_string(const std::string& s, char* buf, size_t* len) {
  if (!len) {
    set_last_error("len is NULL");
    return AS_ERR_INVALID_ARG;
  }
  size_t need = s.size() + 1;
  if (!buf || *len < need) {
    bool had = buf != nullptr;
    *len = need;
    if (had) {
      set_last_error("buffer too small");
      return AS_ERR_INVALID_ARG;
    }
    return AS_OK;
  }
  std::memcpy(buf, s.c_str(), need);
  *len = need;
  return AS_OK;
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(AS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Builds the plan object; device < 0 -> host-only.
Plan* make_plan(const Matrix& A, const Seq& g, const std::string& canon, int device, void* stream, int flags) {
  auto* P = new Plan();
  try {
    P->dt = A.dt;
    P->m = A.m;
    P->n = A.n;
    P->nnz_real = A.nnz();
    P->canon = canon;
    P->device = device;
    P->stream = stream;
    if (device >= 0) {
      // A/B knob: L2 set-aside for persisting lines (the x gathers carry an evict_last
      // policy; without a set-aside the L2 may treat them as normal lines)
      static const char* sa = std::getenv("AS_L2_SETASIDE");
      if (sa) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)std::atoll(sa));
        cudaGetLastError();
        cudaSetDevice(cur);
      }
    }
    DevSpec spec;
    if (device >= 0 && dev_build_spec(g, A, flags, &spec)) {
      // on-device Designer (devbuild.cu): the format is built on the GPU from the cached
      // canonical CSR; P->host keeps only the part skeleton
      int cur = 0;
      check_cuda(cudaGetDevice(&cur), "cudaGetDevice");
      check_cuda(cudaSetDevice(device), "cudaSetDevice");
      try {
        dev_build(*P, A, spec, (cudaStream_t)stream);
        P->graph_mode = (flags & AS_PLAN_GRAPH) != 0;
        P->dev_built = true;
      } catch (...) {
        cudaSetDevice(cur);
        throw;
      }
      cudaSetDevice(cur);
      P->host = HostPlan();
      return P;
    }
    P->host = build_plan(A, g);
    if (device >= 0) {
      int cur = 0;
      check_cuda(cudaGetDevice(&cur), "cudaGetDevice");
      check_cuda(cudaSetDevice(device), "cudaSetDevice");
      try {
        P->upload((cudaStream_t)stream);
        if (flags & AS_PLAN_SPMM) P->upload_spmm((cudaStream_t)stream);
        P->graph_mode = (flags & AS_PLAN_GRAPH) != 0;
      } catch (...) {
        cudaSetDevice(cur);
        throw;
      }
      cudaSetDevice(cur);
    }
    P->compute_model();
    auto& info = P->info;
    info.nnz_real = A.nnz();
    info.n_parts = (int64_t)P->host.parts.size();
    info.prepass_rows = (int64_t)P->host.prepass.size();
    int64_t side_adds = 0;  // R-conc: one k_side_add per side-stream part after the join
    for (void* ys : P->side_y) side_adds += ys != nullptr;
    info.n_launches = (int64_t)P->host.launch_order.size() + (P->host.prepass.empty() ? 0 : 1) +
                      (P->n_heavy ? 1 : 0) + side_adds;  // heavy-row epilogue (the scratch memset is a copy op)
    int64_t slots = 0;
    for (auto& p : P->host.parts) {
      if (p.kind == "csr") slots += p.pad ? (int64_t)p.pad_val.size() : (int64_t)p.val.size();
      else if (p.kind == "dia") slots += (int64_t)p.dia_val.size();
      else slots += (int64_t)p.tile_val.size();
    }
    info.stored_slots = slots;
    info.pads = slots - A.nnz();
    std::string k;
    if (!P->host.prepass.empty()) k = "k_prepass";
    for (int64_t pi : P->host.launch_order) {
      if (!k.empty()) k += ";";
      k += P->host.parts[pi].fam_name;
    }
    if (P->n_heavy) k += ";k_heavy_epilogue";
    std::strncpy(info.kernels, k.c_str(), sizeof(info.kernels) - 1);
    P->host_kept = device < 0 || (flags & AS_PLAN_KEEP_HOST);
    if (!P->host_kept) P->host = HostPlan();
    return P;
  } catch (...) {
    delete P;
    throw;
  }
}

// The launch sequence of one as_spmv call: beta pre-pass, fp32 heavy-row scratch reset, the
// parts in writer-rule order, the heavy-row epilogue.  before(i) runs on the host before
// launch i is enqueued, after(i) after it (as_spmv_host hooks its copy pipeline there).
template <class Before, class After>
int run_plan(Plan& P, const void* x, void* y, double a, double b, cudaStream_t s, Before before, After after,
             void* const* peer_y = nullptr, const int64_t* peer_lo = nullptr, const int64_t* peer_hi = nullptr,
             int n_peers = 0) {
  const size_t sv = P.dt == AS_R64F ? 8 : 4;
  int err = 0;
  if (P.n_prepass) {
    // beta == 0: y is write-only, so zeroing all of y is as correct as zeroing the listed
    // rows.  A listed row costs its 4-byte index plus a scattered 32-byte sector write (ncu,
    // C5: 16.7 M listed rows took 141 us, 418 MB read + 356 MB written), the fill m*sv bytes
    // streamed: fill when it moves fewer bytes
    static const int mode = std::getenv("AS_PREPASS") ? std::atoi(std::getenv("AS_PREPASS")) : 0;  // A/B: 1 list, 2 fill
    if (b == 0.0 && (mode == 2 || (mode == 0 && (double)P.m * sv <= (double)P.n_prepass * (4 + 32))))
      err = (int)cudaMemsetAsync(y, 0, (size_t)P.m * sv, s);
    else
      err = launch_prepass(P.d_prepass, P.n_prepass, b, y, P.dt == AS_R64F ? 1 : 0, s);
  }
  if (P.n_heavy && !err) err = (int)cudaMemsetAsync(P.d_heavy_acc, 0, (size_t)P.n_heavy * 8, s);
  // R-conc: launches naming another stream than the first launch's run on side streams,
  // forked here (after the pre-pass) and joined below; each writes its own scratch vector,
  // added into y after the join (writer mode 3)
  const int dtype = P.dt == AS_R64F ? 1 : 0;
  auto on = [&](size_t i) -> cudaStream_t {
    const int k = P.launch_stream[i];
    return (P.concurrent && k != P.main_stream) ? P.side[k] : s;
  };
  if (P.concurrent && !err) {  // side streams / events: created by Plan::upload
    err = (int)cudaEventRecord(P.ev_fork, s);
    for (int k = 0; k < 4 && !err; ++k)
      if (P.side[k]) err = (int)cudaStreamWaitEvent(P.side[k], P.ev_fork, 0);
  }
  for (size_t i = 0; i < P.launches.size() && !err; ++i) {
    before(i);
    DevPart d = P.launches[i];
    d.alpha = a;
    d.beta = b;
    d.n_peer = n_peers;
    for (int q = 0; q < n_peers; ++q) {
      d.peer_y[q] = peer_y[q];
      d.peer_lo[q] = peer_lo[q];
      d.peer_hi[q] = peer_hi[q];
    }
    void* yd = y;
    if (i < P.side_y.size() && P.side_y[i]) {  // side part: STOREs alpha*s into its scratch
      yd = P.side_y[i];
      d.beta = 0.0;
      d.mode = 0;
      d.n_peer = 0;
      if (P.n_side_zero[i]) err = launch_prepass(P.side_zero[i], P.n_side_zero[i], 0.0, yd, dtype, on(i));
    }
    if (!err) err = launch_part(d, x, yd, on(i));
    if (!err) after(i);
  }
  if (P.concurrent)  // joined even after a failed launch: nothing queued on a side stream outlives the call's order
    for (int k = 0; k < 4; ++k)
      if (P.side[k]) {
        int e = (int)cudaEventRecord(P.ev_join[k], P.side[k]);
        if (!e) e = (int)cudaStreamWaitEvent(s, P.ev_join[k], 0);
        if (!err) err = e;
      }
  for (size_t i = 0; i < P.side_y.size() && !err; ++i)
    if (P.side_y[i]) err = launch_side_add(P.side_rows[i], P.n_side_rows[i], P.side_y[i], y, dtype, s);
  if (P.n_heavy && !err) err = launch_heavy_epilogue(P.d_heavy_rows, P.d_heavy_acc, P.n_heavy, y, s);
  return err;
}

int run_plan_peers(Plan& P, const void* x, void* y, double alpha, double beta, void* stream, void* const* peer_y,
                   const int64_t* peer_lo, const int64_t* peer_hi, int n_peers) {
  if (n_peers > kMaxFusedPeers || (n_peers > 0 && !P.single_writer)) return (int)cudaErrorInvalidValue;
  return run_plan(P, x, y, alpha, beta, (cudaStream_t)stream, [](size_t) {}, [](size_t) {}, peer_y, peer_lo, peer_hi,
                  n_peers);
}

}  // namespace as

using namespace as;

extern "C" {

const char* as_last_error(void) { return g_last_error.c_str(); }

as_status_t as_set_allocator(void* (*alloc)(size_t, void*, void*), void (*release)(void*, void*, void*), void* ctx) {
  return guard([&] {
    if (!alloc != !release) fail(AS_ERR_INVALID_ARG, "alloc and release must both be set or both be NULL");
    g_hooks.alloc = alloc;
    g_hooks.release = release;
    g_hooks.ctx = alloc ? ctx : nullptr;
  });
}
const char* as_version(void) { return "alphasparse-b200 0.1 (sm_100a)"; }

as_status_t as_matrix_create(int64_t m, int64_t n, int64_t nnz, const int64_t* row, const int64_t* col,
                             const void* val, as_dtype_t dt, int index_base, as_matrix_t* out) {
  return guard([&] {
    if (!out) fail(AS_ERR_INVALID_ARG, "out is NULL");
    auto* M = new as_matrix_s();
    try {
      M->A = matrix_from_coo(m, n, nnz, row, col, val, dt, index_base);
    } catch (...) {
      delete M;
      throw;
    }
    *out = M;
  });
}

as_status_t as_matrix_create_csr(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const void* val,
                                 as_dtype_t dt, as_matrix_t* out) {
  return guard([&] {
    if (!out) fail(AS_ERR_INVALID_ARG, "out is NULL");
    auto* M = new as_matrix_s();
    try {
      M->A = matrix_from_csr(m, n, row_ptr, col, val, dt);
    } catch (...) {
      delete M;
      throw;
    }
    *out = M;
  });
}

as_status_t as_matrix_create_mtx(const char* path, as_dtype_t dt, as_matrix_t* out) {
  return guard([&] {
    if (!out || !path) fail(AS_ERR_INVALID_ARG, "NULL argument");
    auto* M = new as_matrix_s();
    try {
      M->A = matrix_from_mtx(path, dt);
    } catch (...) {
      delete M;
      throw;
    }
    *out = M;
  });
}

as_status_t as_matrix_stats(as_matrix_t M, as_stats_t* out) {
  return guard([&] {
    if (!M || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    *out = matrix_stats(M->A);
  });
}

as_status_t as_matrix_row_slice(as_matrix_t M, int64_t r0, int64_t r1, as_matrix_t* out) {
  return guard([&] {
    if (!M || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    auto* S = new as_matrix_s();
    try {
      S->A = matrix_row_slice(M->A, r0, r1);
    } catch (...) {
      delete S;
      throw;
    }
    *out = S;
  });
}

as_status_t as_matrix_export_csr(as_matrix_t M, int64_t* row_ptr, int64_t* col, void* val) {
  return guard([&] {
    if (!M) fail(AS_ERR_INVALID_ARG, "NULL matrix");
    const Matrix& A = M->A;
    if (row_ptr) std::memcpy(row_ptr, A.row_ptr.data(), A.row_ptr.size() * 8);
    if (col)
      for (int64_t i = 0; i < A.nnz(); ++i) col[i] = A.col[i];
    if (val) {
      if (A.dt == AS_R64F) std::memcpy(val, A.val.data(), A.val.size() * 8);
      else
        for (int64_t i = 0; i < A.nnz(); ++i) ((float*)val)[i] = (float)A.val[i];
    }
  });
}

void as_matrix_destroy(as_matrix_t M) { delete M; }

as_status_t as_graph_parse(const char* text, as_graph_t* out) {
  return guard([&] {
    if (!text || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    auto* G = new as_graph_s();
    try {
      G->g = parse_graph(text);
      G->canon = print_graph(G->g);
    } catch (...) {
      delete G;
      throw;
    }
    *out = G;
  });
}

as_status_t as_graph_print(as_graph_t G, char* buf, size_t* len) {
  if (!G) {
    set_last_error("NULL graph");
    return AS_ERR_INVALID_ARG;
  }
  return copy_string(G->canon, buf, len);
}

void as_graph_destroy(as_graph_t G) { delete G; }

as_status_t as_plan_ex(as_matrix_t M, as_graph_t G, int device, void* stream, int flags, as_plan_t* out) {
  return guard([&] {
    NvtxRange nv("as_plan");
    if (!M || !G || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    Plan* P = make_plan(M->A, G->g, G->canon, device, stream, flags);
    auto* h = new as_plan_s();
    h->P.reset(P);
    *out = h;
  });
}

as_status_t as_plan(as_matrix_t M, as_graph_t G, int device, void* stream, as_plan_t* out) {
  return as_plan_ex(M, G, device, stream, 0, out);
}

as_status_t as_plan_info(as_plan_t P, as_plan_info_t* out) {
  return guard([&] {
    if (!P || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    *out = P->P->info;
    out->single_writer = P->P->single_writer ? 1 : 0;
    out->modeled_arrays = P->P->modeled_arrays;
    out->device_built = P->P->dev_built ? 1 : 0;
  });
}

as_status_t as_plan_export(as_plan_t P, const char* key, void* host_dst, size_t* bytes) {
  return guard([&] {
    if (!P || !key || !bytes) fail(AS_ERR_INVALID_ARG, "NULL argument");
    if (std::strncmp(key, "dev.", 4) == 0) {  // device readback (readback.cpp)
      if (P->P->device < 0) fail(AS_ERR_INVALID_ARG, "host-only plan has no device arrays");
      auto arrs = device_arrays(*P->P);
      std::vector<uint8_t> val;
      bool found = false;
      if (std::strcmp(key, "dev.keys") == 0) {
        std::string s;
        for (auto& kv : arrs) s += (s.empty() ? "" : ";") + kv.first;
        val.assign(s.begin(), s.end());
        found = true;
      }
      for (auto& kv : arrs)
        if (kv.first == key) {
          val = std::move(kv.second);
          found = true;
        }
      if (!found) fail(AS_ERR_NOT_FOUND, std::string("no export key ") + key);
      if (host_dst && *bytes < val.size()) fail(AS_ERR_INVALID_ARG, "destination too small");
      if (host_dst && !val.empty()) std::memcpy(host_dst, val.data(), val.size());
      *bytes = val.size();
      return;
    }
    if (!P->P->host_kept) fail(AS_ERR_INVALID_ARG, "plan built without AS_PLAN_KEEP_HOST");
    size_t need = 0;
    if (!export_key(P->P->host, key, nullptr, &need)) fail(AS_ERR_NOT_FOUND, std::string("no export key ") + key);
    if (host_dst && *bytes < need) fail(AS_ERR_INVALID_ARG, "destination too small");
    if (host_dst) export_key(P->P->host, key, host_dst, &need);
    *bytes = need;
  });
}

as_status_t as_plan_keys(as_plan_t P, char* buf, size_t* len) {
  if (!P || !P->P->host_kept) {
    set_last_error("plan built without AS_PLAN_KEEP_HOST");
    return AS_ERR_INVALID_ARG;
  }
  std::string s;
  for (auto& k : export_keys(P->P->host)) {
    if (!s.empty()) s += ";";
    s += k;
  }
  return copy_string(s, buf, len);
}

void as_plan_destroy(as_plan_t P) { delete P; }


as_status_t as_spmv(as_plan_t h, const void* alpha, const void* x, const void* beta, void* y, void* stream) {
  return guard([&] {
    NvtxRange nv("as_spmv");
    if (!h || !alpha || !beta) fail(AS_ERR_INVALID_ARG, "NULL argument");
    Plan& P = *h->P;
    if (P.device < 0) fail(AS_ERR_INVALID_ARG, "host-only plan cannot run as_spmv");
    if ((P.n > 0 && !x) || (P.m > 0 && !y)) fail(AS_ERR_INVALID_ARG, "NULL x or y");
    const size_t sv = P.dt == AS_R64F ? 8 : 4;
    if (((uintptr_t)x | (uintptr_t)y) & (sv - 1)) fail(AS_ERR_INVALID_ARG, "x and y must be aligned to the value size");
    if (x && y && (const char*)x < (const char*)y + P.m * sv && (const char*)y < (const char*)x + P.n * sv)
      fail(AS_ERR_INVALID_ARG, "x and y alias");
    double a = P.dt == AS_R64F ? *(const double*)alpha : (double)*(const float*)alpha;
    double b = P.dt == AS_R64F ? *(const double*)beta : (double)*(const float*)beta;
    cudaError_t prior = cudaGetLastError();
    if (prior != cudaSuccess) fail(AS_ERR_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(prior));
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != P.device) cudaSetDevice(P.device);
    int err = 0;
    if (P.graph_mode) {
      // AS_PLAN_GRAPH: the launch sequence is captured once per (x, y, alpha, beta) into a
      // CUDA graph and replayed (one launch instead of one per part: latency-bound plans)
      if (!P.gexec || P.gx != x || P.gy != y || P.ga != a || P.gb != b) {
        if (P.gexec) cudaGraphExecDestroy(P.gexec);
        P.gexec = nullptr;
        if (!P.cap_stream) check_cuda(cudaStreamCreateWithFlags(&P.cap_stream, cudaStreamNonBlocking), "capture stream");
        check_cuda(cudaStreamBeginCapture(P.cap_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
        err = run_plan(P, x, y, a, b, P.cap_stream, [](size_t) {}, [](size_t) {});
        cudaGraph_t graph = nullptr;
        cudaError_t e2 = cudaStreamEndCapture(P.cap_stream, &graph);
        if (!err && e2 == cudaSuccess) err = (int)cudaGraphInstantiate(&P.gexec, graph, 0);
        else if (!err) err = (int)e2;
        if (graph) cudaGraphDestroy(graph);
        P.gx = x;
        P.gy = y;
        P.ga = a;
        P.gb = b;
      }
      if (!err) err = (int)cudaGraphLaunch(P.gexec, (cudaStream_t)stream);
    } else {
      err = run_plan(P, x, y, a, b, (cudaStream_t)stream, [](size_t) {}, [](size_t) {});
    }
    if (cur != P.device) cudaSetDevice(cur);
    if (err) fail(AS_ERR_CUDA, std::string("launch: ") + cudaGetErrorString((cudaError_t)err));
  });
}

// Host-buffer SpMV.  With several launches whose spans allow it (e.g. a ROW_DIV graph), the
// copies are pipelined against the kernels: x goes up in chunks on a copy stream (chunk
// boundaries = the running maximum of the launches' last column), launch i waits only for
// the chunk holding its last column, and every y row range no later launch writes goes down
// on a second copy stream as soon as the launch that finishes it is done -- PCIe is full
// duplex, so H2D of x, the kernels and D2H of y overlap instead of running back to back.
as_status_t as_spmv_host(as_plan_t h, const void* alpha, const void* x_host, const void* beta, void* y_host,
                         void* stream) {
  return guard([&] {
    NvtxRange nv("as_spmv_host");
    if (!h || !alpha || !beta) fail(AS_ERR_INVALID_ARG, "NULL argument");
    Plan& P = *h->P;
    if (P.device < 0) fail(AS_ERR_INVALID_ARG, "host-only plan");
    if ((P.n > 0 && !x_host) || (P.m > 0 && !y_host)) fail(AS_ERR_INVALID_ARG, "NULL x or y");
    const size_t sv = P.dt == AS_R64F ? 8 : 4;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(P.device);
    if (!P.d_x) P.d_x = dev_alloc(std::max<size_t>(16, P.n * sv), P.stream);
    if (!P.d_y) P.d_y = dev_alloc(std::max<size_t>(16, P.m * sv), P.stream);
    cudaStream_t s = (cudaStream_t)stream;
    double a = P.dt == AS_R64F ? *(const double*)alpha : (double)*(const float*)alpha;
    double b = P.dt == AS_R64F ? *(const double*)beta : (double)*(const float*)beta;
    cudaError_t prior = cudaGetLastError();
    if (prior != cudaSuccess) fail(AS_ERR_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(prior));
    const size_t L = P.launches.size();
    const bool pipe = L >= 2 && !P.n_heavy && !P.concurrent && P.spans.size() == L && !std::getenv("AS_HOST_NOPIPE");
    char* dx = (char*)P.d_x;
    char* dy = (char*)P.d_y;
    int err = 0;
    if (!pipe) {
      check_cuda(cudaMemcpyAsync(dx, x_host, P.n * sv, cudaMemcpyHostToDevice, s), "H2D x");
      if (b != 0.0) check_cuda(cudaMemcpyAsync(dy, y_host, P.m * sv, cudaMemcpyHostToDevice, s), "H2D y");
      err = run_plan(P, dx, dy, a, b, s, [](size_t) {}, [](size_t) {});
      if (!err) err = (int)cudaMemcpyAsync(y_host, dy, P.m * sv, cudaMemcpyDeviceToHost, s);
    } else {
      if (!P.s_h2d) {
        check_cuda(cudaStreamCreateWithFlags(&P.s_h2d, cudaStreamNonBlocking), "copy stream");
        check_cuda(cudaStreamCreateWithFlags(&P.s_d2h, cudaStreamNonBlocking), "copy stream");
      }
      size_t ev = 0;
      auto fork = [&](cudaStream_t from, cudaStream_t to) {  // `to` waits for work so far on `from`
        cudaEvent_t e = P.host_event(ev++);
        check_cuda(cudaEventRecord(e, from), "event");
        check_cuda(cudaStreamWaitEvent(to, e, 0), "wait");
        return e;
      };
      // the copy streams start after everything already queued on s (earlier users of d_x/d_y)
      fork(s, P.s_h2d);
      fork(s, P.s_d2h);
      if (b != 0.0) {
        check_cuda(cudaMemcpyAsync(dy, y_host, P.m * sv, cudaMemcpyHostToDevice, P.s_h2d), "H2D y");
        fork(P.s_h2d, s);
      }
      // x prefix each launch needs (running max of chi + 1) and the chunk events
      std::vector<int64_t> need(L);
      int64_t run = 0;
      for (size_t i = 0; i < L; ++i) {
        run = std::max(run, std::min<int64_t>(P.spans[i].chi + 1, P.n));
        need[i] = run;
      }
      int64_t sent = 0;
      std::vector<std::pair<int64_t, cudaEvent_t>> chunks;  // (end column, event)
      for (size_t i = 0; i < L; ++i) {
        int64_t e = i + 1 == L ? P.n : need[i];
        if (e > sent) {
          check_cuda(cudaMemcpyAsync(dx + sent * sv, (const char*)x_host + sent * sv, (e - sent) * sv,
                                     cudaMemcpyHostToDevice, P.s_h2d), "H2D x chunk");
          cudaEvent_t ce = P.host_event(ev++);
          check_cuda(cudaEventRecord(ce, P.s_h2d), "event");
          chunks.push_back({e, ce});
          sent = e;
        }
      }
      // rows final after launch i: below the lowest row any later launch writes
      std::vector<int64_t> fin(L);
      int64_t lo = P.m;
      for (size_t i = L; i-- > 0;) {
        fin[i] = lo;
        if (P.spans[i].rlo <= P.spans[i].rhi) lo = std::min(lo, P.spans[i].rlo);
      }
      int64_t done = 0;
      size_t ci = 0;
      err = run_plan(
          P, dx, dy, a, b, s,
          [&](size_t i) {
            while (ci < chunks.size() && chunks[ci].first < need[i]) ++ci;
            if (need[i] > 0 && ci < chunks.size()) check_cuda(cudaStreamWaitEvent(s, chunks[ci].second, 0), "wait");
          },
          [&](size_t i) {
            int64_t f = i + 1 == L ? P.m : fin[i];
            if (f > done && (f - done) * (int64_t)sv >= (1 << 20)) {  // >= 1 MB per D2H chunk
              fork(s, P.s_d2h);
              check_cuda(cudaMemcpyAsync((char*)y_host + done * sv, dy + done * sv, (f - done) * sv,
                                         cudaMemcpyDeviceToHost, P.s_d2h), "D2H y chunk");
              done = f;
            }
          });
      if (!err && done < P.m) {
        fork(s, P.s_d2h);
        check_cuda(cudaMemcpyAsync((char*)y_host + done * sv, dy + done * sv, (P.m - done) * sv,
                                   cudaMemcpyDeviceToHost, P.s_d2h), "D2H y tail");
      }
      fork(P.s_d2h, s);
      fork(P.s_h2d, s);
    }
    if (err) {
      cudaSetDevice(cur);
      fail(AS_ERR_CUDA, std::string("launch: ") + cudaGetErrorString((cudaError_t)err));
    }
    check_cuda(cudaStreamSynchronize(s), "sync");
    cudaSetDevice(cur);
  });
}

// k independent host-buffer SpMVs, pipelined across them: x_{i+1} goes up on a copy stream
// while SpMV i runs and y_{i-1} comes down on another (PCIe is full duplex), with two device
// buffer pairs; every x_i is copied up and every y_i copied back.  Steady state per SpMV =
// max(H2D x, kernels, D2H y) instead of their sum.
as_status_t as_spmv_host_batch(as_plan_t h, int64_t k, const void* alpha, const void* const* x_host,
                               const void* beta, void* const* y_host, void* stream) {
  return guard([&] {
    NvtxRange nv("as_spmv_host_batch");
    if (!h || !alpha || !beta || (k > 0 && (!x_host || !y_host))) fail(AS_ERR_INVALID_ARG, "NULL argument");
    if (k < 0) fail(AS_ERR_INVALID_ARG, "k < 0");
    Plan& P = *h->P;
    if (P.device < 0) fail(AS_ERR_INVALID_ARG, "host-only plan");
    for (int64_t i = 0; i < k; ++i)
      if ((P.n > 0 && !x_host[i]) || (P.m > 0 && !y_host[i])) fail(AS_ERR_INVALID_ARG, "NULL x or y");
    const size_t sv = P.dt == AS_R64F ? 8 : 4;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(P.device);
    void** bx[2] = {&P.d_x, &P.d_x1};
    void** by[2] = {&P.d_y, &P.d_y1};
    for (int j = 0; j < 2; ++j) {
      if (!*bx[j]) *bx[j] = dev_alloc(std::max<size_t>(16, P.n * sv), P.stream);
      if (!*by[j]) *by[j] = dev_alloc(std::max<size_t>(16, P.m * sv), P.stream);
    }
    cudaStream_t s = (cudaStream_t)stream;
    const double a = P.dt == AS_R64F ? *(const double*)alpha : (double)*(const float*)alpha;
    const double b = P.dt == AS_R64F ? *(const double*)beta : (double)*(const float*)beta;
    cudaError_t prior = cudaGetLastError();
    if (prior != cudaSuccess) fail(AS_ERR_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(prior));
    if (!P.s_h2d) {
      check_cuda(cudaStreamCreateWithFlags(&P.s_h2d, cudaStreamNonBlocking), "copy stream");
      check_cuda(cudaStreamCreateWithFlags(&P.s_d2h, cudaStreamNonBlocking), "copy stream");
    }
    size_t ev = 0;
    auto mark = [&](cudaStream_t on) {
      cudaEvent_t e = P.host_event(ev++);
      check_cuda(cudaEventRecord(e, on), "event");
      return e;
    };
    // the copy streams start after everything already queued on s
    cudaEvent_t start = mark(s);
    check_cuda(cudaStreamWaitEvent(P.s_h2d, start, 0), "wait");
    check_cuda(cudaStreamWaitEvent(P.s_d2h, start, 0), "wait");
    std::vector<cudaEvent_t> computed((size_t)k), drained((size_t)k);
    int err = 0;
    for (int64_t i = 0; i < k && !err; ++i) {
      const int j = (int)(i & 1);
      char* dx = (char*)*bx[j];
      char* dy = (char*)*by[j];
      // x buffer j is free once SpMV i-2 has read it; y buffer j once y_{i-2} came down.  The
      // two are tracked apart so x_i goes up WHILE y_{i-2} comes down (PCIe is full duplex:
      // 64 MB each way take 1.39 ms together vs 1.21 + 1.18 ms one after the other,
      // tools/pcie_bw.py); waiting for both before x_i serialised the directions
      if (i >= 2) check_cuda(cudaStreamWaitEvent(P.s_h2d, computed[(size_t)i - 2], 0), "wait");
      check_cuda(cudaMemcpyAsync(dx, x_host[i], P.n * sv, cudaMemcpyHostToDevice, P.s_h2d), "H2D x");
      if (b != 0.0) {
        if (i >= 2) check_cuda(cudaStreamWaitEvent(P.s_h2d, drained[(size_t)i - 2], 0), "wait");
        check_cuda(cudaMemcpyAsync(dy, y_host[i], P.m * sv, cudaMemcpyHostToDevice, P.s_h2d), "H2D y");
      }
      check_cuda(cudaStreamWaitEvent(s, mark(P.s_h2d), 0), "wait");
      if (b == 0.0 && i >= 2) check_cuda(cudaStreamWaitEvent(s, drained[(size_t)i - 2], 0), "wait");
      err = run_plan(P, dx, dy, a, b, s, [](size_t) {}, [](size_t) {});
      if (err) break;
      computed[(size_t)i] = mark(s);
      check_cuda(cudaStreamWaitEvent(P.s_d2h, computed[(size_t)i], 0), "wait");
      check_cuda(cudaMemcpyAsync(y_host[i], dy, P.m * sv, cudaMemcpyDeviceToHost, P.s_d2h), "D2H y");
      drained[(size_t)i] = mark(P.s_d2h);
    }
    check_cuda(cudaStreamWaitEvent(s, mark(P.s_d2h), 0), "wait");
    check_cuda(cudaStreamWaitEvent(s, mark(P.s_h2d), 0), "wait");
    if (err) {
      cudaSetDevice(cur);
      fail(AS_ERR_CUDA, std::string("launch: ") + cudaGetErrorString((cudaError_t)err));
    }
    check_cuda(cudaStreamSynchronize(s), "sync");
    cudaSetDevice(cur);
  });
}

as_status_t as_plan_profile(as_plan_t h, const void* x, void* y, int reps, void* stream, double* ms, double* bytes,
                            size_t* n) {
  return guard([&] {
    if (!h || !n) fail(AS_ERR_INVALID_ARG, "NULL argument");
    Plan& P = *h->P;
    if (P.device < 0) fail(AS_ERR_INVALID_ARG, "host-only plan");
    // entries: [pre-pass], parts in launch order, [heavy-row epilogue] (as_plan_info.kernels)
    const size_t L = P.launches.size();
    const size_t cnt = (P.n_prepass ? 1 : 0) + L + (P.n_heavy ? 1 : 0);
    if (!ms || !bytes) {
      *n = cnt;
      return;
    }
    if (*n < cnt) fail(AS_ERR_INVALID_ARG, "output arrays too small");
    if ((P.n > 0 && !x) || (P.m > 0 && !y) || reps < 1) fail(AS_ERR_INVALID_ARG, "NULL x / y or reps < 1");
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != P.device) cudaSetDevice(P.device);
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<cudaEvent_t> ev(L + 2);
    for (auto& e : ev) check_cuda(cudaEventCreate(&e), "event");
    std::vector<double> acc(L + 2, 0.0);
    int err = 0;
    // per-launch times need the launches in one stream order: a concurrent plan (R-conc) is
    // profiled serialised (its parts add atomically, so the result is the same)
    struct Serial {
      Plan& P;
      bool c;
      ~Serial() { P.concurrent = c; }
    } serial{P, P.concurrent};
    P.concurrent = false;
    for (int r = 0; r < reps && !err; ++r) {
      check_cuda(cudaEventRecord(ev[0], s), "event");
      err = run_plan(
          P, x, y, 1.0, 0.0, s, [&](size_t i) { if (i == 0) cudaEventRecord(ev[1], s); },
          [&](size_t i) { cudaEventRecord(ev[i + 2], s); });
      if (!err) err = (int)cudaStreamSynchronize(s);
      if (err) break;
      float t = 0;
      if (L) cudaEventElapsedTime(&t, ev[0], ev[1]);
      acc[0] += t;
      for (size_t i = 0; i < L; ++i) {
        cudaEventElapsedTime(&t, ev[i + 1], ev[i + 2]);
        acc[i + 1] += t;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (!err && L == 0) cudaGetLastError();  // no launch: ev[1] was never recorded
    if (cur != P.device) cudaSetDevice(cur);
    if (err) fail(AS_ERR_CUDA, std::string("profile: ") + cudaGetErrorString((cudaError_t)err));
    const size_t sv = P.dt == AS_R64F ? 8 : 4;
    size_t o = 0;
    if (P.n_prepass) {
      ms[o] = acc[0] / reps;
      bytes[o++] = P.prepass_bytes;
    }
    for (size_t i = 0; i < L; ++i) {
      ms[o] = acc[i + 1] / reps;
      bytes[o++] = i < P.launch_bytes.size() ? P.launch_bytes[i] : 0.0;
    }
    if (P.n_heavy) {  // the epilogue runs after the last part; its time is not separated
      ms[o] = 0.0;
      bytes[o++] = (double)P.n_heavy * (4 + 8 + 2 * sv);
    }
    *n = cnt;
  });
}

as_status_t as_spmm(as_plan_t h, int64_t k, const void* alpha, const void* X, int64_t ldx, const void* beta, void* Y,
                    int64_t ldy, void* stream) {
  return guard([&] {
    NvtxRange nv("as_spmm");
    if (!h || !alpha || !beta) fail(AS_ERR_INVALID_ARG, "NULL argument");
    Plan& P = *h->P;
    if (P.device < 0) fail(AS_ERR_INVALID_ARG, "host-only plan cannot run as_spmm");
    if (!P.spmm) fail(AS_ERR_INVALID_ARG, "plan built without AS_PLAN_SPMM");
    if (k < 1 || ldx < k || ldy < k) fail(AS_ERR_INVALID_ARG, "need k >= 1, ldx >= k, ldy >= k");
    if ((P.n > 0 && !X) || (P.m > 0 && !Y)) fail(AS_ERR_INVALID_ARG, "NULL X or Y");
    const size_t sv = P.dt == AS_R64F ? 8 : 4;
    if (((uintptr_t)X | (uintptr_t)Y) & (sv - 1)) fail(AS_ERR_INVALID_ARG, "X and Y must be aligned to the value size");
    const char *xa = (const char*)X, *xe = xa + (size_t)(P.n ? (P.n - 1) * ldx + k : 0) * sv;
    const char *ya = (const char*)Y, *ye = ya + (size_t)(P.m ? (P.m - 1) * ldy + k : 0) * sv;
    if (X && Y && xa < ye && ya < xe) fail(AS_ERR_INVALID_ARG, "X and Y alias");
    const double a = P.dt == AS_R64F ? *(const double*)alpha : (double)*(const float*)alpha;
    const double b = P.dt == AS_R64F ? *(const double*)beta : (double)*(const float*)beta;
    cudaError_t prior = cudaGetLastError();
    if (prior != cudaSuccess) fail(AS_ERR_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(prior));
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != P.device) cudaSetDevice(P.device);
    const int dtc = P.dt == AS_R64F ? 1 : 0;
    for (const DevPart& d : P.launches)  // validate every part before the first launch
      if (d.fam == FAM_DENSE && d.b > 64)
        fail(AS_ERR_PLAN_INFEASIBLE, "as_spmm: DENSE tiles larger than 64 are not implemented for SpMM");
    int err = 0;
    if (P.n_prepass) {  // same rule as the SpMV: a fill of all rows when it moves fewer bytes (beta == 0)
      if (b == 0.0 && (double)P.m * sv <= (double)P.n_prepass * (4 + 32))
        err = launch_spmm_prepass(nullptr, 0, P.m, 0.0, Y, ldy, k, dtc, stream);
      else
        err = launch_spmm_prepass(P.d_prepass, P.n_prepass, P.m, b, Y, ldy, k, dtc, stream);
    }
    for (size_t i = 0; i < P.launches.size() && !err; ++i)
      err = launch_spmm_part(P.launches[i], P.spmm_parts[i], a, b, X, ldx, Y, ldy, k, stream);
    if (cur != P.device) cudaSetDevice(cur);
    if (err) fail(AS_ERR_CUDA, std::string("spmm launch: ") + cudaGetErrorString((cudaError_t)err));
  });
}

as_status_t as_search(as_matrix_t M, const as_search_cfg_t* cfg, int device, void* stream, as_plan_t* best,
                      char* best_graph, size_t* len) {
  as_status_t st = AS_OK;
  as_status_t g = guard([&] {
    NvtxRange nv("as_search");
    if (!M || !cfg || !best) fail(AS_ERR_INVALID_ARG, "NULL argument");
    st = search_impl(M->A, cfg, device, stream, best, best_graph, len);
  });
  return g != AS_OK ? g : st;
}

as_status_t as_matrix_features(as_matrix_t M, double* out) {
  return guard([&] {
    if (!M || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    std::vector<double> f = matrix_features(M->A);
    std::copy(f.begin(), f.end(), out);
  });
}

as_status_t as_graph_device_buildable(as_matrix_t M, as_graph_t G, int flags, int* out) {
  return guard([&] {
    if (!M || !G || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    DevSpec sp;
    *out = dev_build_spec(G->g, M->A, flags, &sp) ? 1 : 0;
  });
}

as_status_t as_random_graph(as_matrix_t M, uint64_t seed, char* buf, size_t* len) {
  std::string s;
  as_status_t st = guard([&] {
    if (!M) fail(AS_ERR_INVALID_ARG, "NULL matrix");
    s = random_graph(M->A, seed);
  });
  if (st != AS_OK) return st;
  return copy_string(s, buf, len);
}

as_status_t as_matrix_col_span(as_matrix_t M, int64_t* lo, int64_t* hi) {
  return guard([&] {
    if (!M || !lo || !hi) fail(AS_ERR_INVALID_ARG, "NULL argument");
    int64_t a = INT64_MAX, b = -1;
    for (int32_t c : M->A.col) {
      a = std::min<int64_t>(a, c);
      b = std::max<int64_t>(b, c);
    }
    *lo = b < 0 ? 0 : a;
    *hi = b;
  });
}

as_status_t as_dist_row_cuts_ptr(const int64_t* row_ptr, int64_t m, int world, int64_t* cuts) {
  return guard([&] {
    if (!row_ptr || !cuts || m < 0 || world < 1) fail(AS_ERR_INVALID_ARG, "NULL argument, m < 0 or world < 1");
    std::vector<int64_t> rp(row_ptr, row_ptr + m + 1);
    auto c = row_cuts(rp, world);
    std::memcpy(cuts, c.data(), c.size() * 8);
  });
}

as_status_t as_dist_row_cuts(as_matrix_t M, int world, int64_t* cuts) {
  return guard([&] {
    if (!M || !cuts) fail(AS_ERR_INVALID_ARG, "NULL argument");
    auto c = row_cuts(M->A.row_ptr, world);
    std::memcpy(cuts, c.data(), c.size() * 8);
  });
}

}  // extern "C"
