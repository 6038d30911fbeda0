// Internal structures of libalphasparse (not part of the ABI).
#pragma once
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/as.h"
#include "devpart.h"

namespace as {

struct Error : std::exception {
  as_status_t st;
  std::string msg;
  Error(as_status_t s, std::string m) : st(s), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};
[[noreturn]] inline void fail(as_status_t s, const std::string& m) { throw Error(s, m); }
void set_last_error(const std::string& m);
void check_cuda(cudaError_t e, const char* what);

// Runs f, converting exceptions to statuses (every C entry point).
template <class F>
inline as_status_t guard(F f) {
  try {
    f();
    return AS_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.st;
  } catch (const std::bad_alloc&) {
    set_last_error("host out of memory");
    return AS_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return AS_ERR_INVALID_ARG;
  }
}

// Device memory of plans and scratch: cudaMalloc/cudaFree on the current device, or the
// caller's hooks (as_set_allocator, e.g. torch's caching allocator).  dev_alloc throws
// AS_ERR_OOM on failure.
void* dev_alloc(size_t bytes, void* stream);
void dev_free(void* p, void* stream);

// ------------------------------------------------------------------ graph IR
struct Value {
  enum Kind { INT, FLOAT, LIST, IDENT } k = INT;
  int64_t i = 0;
  double f = 0;
  std::vector<int64_t> l;
  std::string s;
};

struct Op {
  std::string name;
  std::vector<std::pair<std::string, Value>> params;  // canonical order, defaults filled
  std::vector<std::vector<Op>> br;
  int id = 0;  // pre-order node id
  int64_t geti(const char* k) const;
  double getf(const char* k) const;
  const std::vector<int64_t>& getl(const char* k) const;
  const std::string& gets(const char* k) const;
};
using Seq = std::vector<Op>;

Seq parse_graph(const std::string& text);  // parse + expand replicated branches + validate
std::string print_graph(const Seq& g);
bool is_branching(const std::string& name);

// Model-Driven Format Compression (model.cpp, NEXT-2)
bool fit_array_model(const std::vector<int64_t>& a, int budget, IdxModel* out);
bool model_may_fit(const std::vector<int64_t>& pre, int64_t n, int64_t am0, int64_t am1, int64_t al0, int64_t al1,
                   int budget);

// search cost model (surrogate.cpp, NEXT-3)
size_t graph_feature_count();
std::vector<double> graph_features(const Seq& g);
void surrogate_fit_predict(const double* X, const double* y, size_t n, size_t d, const double* Xq, size_t nq,
                           double* out, int rounds, int max_depth, double lr);

// ------------------------------------------------------------------ matrix (host, canonical CSR)
struct DevCsr;  // the canonical CSR uploaded for the on-device builder (devbuild.cu), cached
struct Matrix {
  int64_t m = 0, n = 0;
  as_dtype_t dt = AS_R64F;
  std::vector<int64_t> row_ptr;  // m+1
  std::vector<int32_t> col;      // nnz, ascending within a row
  std::vector<double> val;       // nnz (fp32 data widened exactly)
  mutable std::shared_ptr<DevCsr> dcache;  // device copy (devbuild.cu), shared by all plans of the matrix
  int64_t nnz() const { return (int64_t)col.size(); }
};

// ------------------------------------------------------------------ built format (host side)

struct Level {
  bool present = false;
  bool nnz = false;                 // NNZ_BLOCK (else ROW_BLOCK)
  int64_t size = 0;
  std::vector<int64_t> start;       // n_blocks + 1 nz offsets (unpadded)
  std::vector<int64_t> first_row;   // n_blocks
  int64_t count() const { return start.empty() ? 0 : (int64_t)start.size() - 1; }
};

struct HostPart {
  std::string kind;  // "csr" | "dia" | "dense"
  // COMPRESS output
  std::vector<int64_t> origin, row_ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
  // mapping
  Level lv[3];  // 0 BMTB, 1 BMW, 2 BMT
  bool pad = false;
  int pad_scope = -1;  // -1 GLOBAL, else level index
  int vec = 1;
  std::vector<int64_t> pad_width, grp_first_bmt, grp_base;
  std::vector<int32_t> pad_col;
  std::vector<double> pad_val;
  std::vector<uint32_t> bitmap;
  int bm_words = 0;
  bool sort_bmtb = false;
  Red red[3] = {RED_NONE, RED_NONE, RED_NONE};  // per level (BMTB, BMW, BMT)
  int tpb = 0, grid = 0, stages = 2;  // SET_RESOURCE
  int64_t xcache = 0;                 // SET_RESOURCE xcache: hot x entries staged in shared memory per CTA
  int stream = 0;                     // SET_RESOURCE stream: launch stream (R-conc); parts on different
                                      // streams run concurrently
  // DIA
  int64_t r0 = 0, mb = 0;
  std::vector<int64_t> dia_off;
  std::vector<double> dia_val;  // D * mb
  // DENSE
  int64_t b = 0;
  std::vector<int64_t> tile_row_id, tile_row_ptr, tile_col;
  std::vector<double> tile_val;
  // writer rule
  std::vector<int64_t> excl, atom;  // global rows
  int mode = 0;                      // 0 STORE, 1 ADD, 3 side stream: scratch + add epilogue (R-conc)
  Fam fam = FAM_NONE;
  std::string fam_name;
};

struct HostPlan {
  int64_t m = 0, n = 0;
  as_dtype_t dt = AS_R64F;
  std::vector<HostPart> parts;       // DFS leaf order
  std::vector<int64_t> launch_order; // non-empty parts
  std::vector<int64_t> prepass;      // ascending global rows
  int64_t distinct_cols = 0;
};

HostPlan build_plan(const Matrix& A, const Seq& g);  // throws Error(AS_ERR_PLAN_INFEASIBLE)
std::vector<int64_t> row_cuts(const std::vector<int64_t>& row_ptr, int world);

// export of logical arrays: returns false if key absent; sets bytes and fills dst if non-null
bool export_key(const HostPlan& hp, const std::string& key, void* dst, size_t* bytes);
std::vector<std::string> export_keys(const HostPlan& hp);

// ------------------------------------------------------------------ random graphs (search generator)
std::string random_graph(const Matrix& A, uint64_t seed);

// ------------------------------------------------------------------ small utilities
// NVTX range over a scope (SURVEY §5 tracing): header-only NVTX3, a no-op unless a tool
// (nsys / ncu --nvtx) injects itself.  Names: "as_plan", "as_spmv", "as_search", ...
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class F>
void parallel_for(int64_t n, F f, int64_t grain = 1 << 16);

}  // namespace as

struct as_matrix_s {
  as::Matrix A;
};
struct as_graph_s {
  as::Seq g;
  std::string canon;
};

#include <thread>
namespace as {
template <class F>
void parallel_for(int64_t n, F f, int64_t grain) {
  int64_t nt = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), n / grain));
  if (nt <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t) {
    int64_t a = n * t / nt, e = n * (t + 1) / nt;
    th.emplace_back([=] { f(a, e); });
  }
  for (auto& x : th) x.join();
}
}  // namespace as
