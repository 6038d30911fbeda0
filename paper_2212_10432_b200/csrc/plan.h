// Plan object (internal): device-resident format + launch list.
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace as {

struct Plan {
  int device = -1;
  void* stream = nullptr;        // creation stream (allocator hooks free on it)
  as_dtype_t dt = AS_R64F;
  int64_t m = 0, n = 0, nnz_real = 0;
  HostPlan host;                 // logical metadata (kept for host-only plans / AS_PLAN_KEEP_HOST)
  bool host_kept = false;
  std::vector<DevPart> launches; // in launch order
  std::vector<int64_t> launch_part;  // part index (DFS order) of every launch
  const int32_t* d_prepass = nullptr;
  int64_t n_prepass = 0;
  std::vector<void*> allocs;
  size_t dev_bytes = 0;
  double bytes_model = 0;        // bytes of the device arrays the kernels read
  as_plan_info_t info{};
  void* d_x = nullptr;           // scratch for as_spmv_host
  void* d_y = nullptr;
  void* d_x1 = nullptr;          // second buffer pair of as_spmv_host_batch
  void* d_y1 = nullptr;
  // per launch: x columns read [clo, chi] and global y rows written [rlo, rhi] (supersets;
  // empty = clo > chi).  as_spmv_host pipelines chunked copies against launches with them.
  struct Span {
    int64_t clo, chi, rlo, rhi;
  };
  std::vector<Span> spans;
  std::vector<double> launch_bytes;  // per launch: algorithmic bytes (arrays + x + y), beta == 0
  double prepass_bytes = 0;
  // every row's final value is produced by exactly one STORE (no pre-pass, no ADD parts,
  // no atomic rows, no fp32 heavy-row epilogue): as_spmv_dist may fuse peer stores
  bool single_writer = false;
  bool dev_built = false;  // format built by the on-device Designer (devbuild.cu)
  int modeled_arrays = 0;  // index arrays replaced by fitted models (NEXT-2)
  int fused_arrays = 0;    // per-BMT metadata arrays fused into one (short-array fusion, NEXT-2)
  bool spmm = false;              // AS_PLAN_SPMM: SpMM arrays of the CSR-family parts uploaded
  bool graph_mode = false;        // AS_PLAN_GRAPH: as_spmv replays a captured CUDA graph
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_stream = nullptr;
  const void* gx = nullptr;       // (x, y, alpha, beta) the graph was captured with
  void* gy = nullptr;
  double ga = 0, gb = 0;
  std::vector<SpmmPart> spmm_parts;  // per launch (empty for DIA / DENSE parts)
  void upload_spmm(cudaStream_t s);
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // as_spmv_host copy streams (lazy)
  std::vector<cudaEvent_t> evs;                    // as_spmv_host events (lazy)
  cudaEvent_t host_event(size_t i);
  // R-conc: per launch its SET_RESOURCE stream.  Launches naming the first launch's stream
  // run on the caller's stream; the others (side parts, writer mode 3) on side stream k
  // (created by upload), forked after the pre-pass and joined before the epilogues.  A side
  // part writes its own scratch vector side_y (its atomic rows zeroed first), whose rows
  // side_rows are added into y after the join (k_side_add).
  std::vector<int> launch_stream;
  int main_stream = 0;
  bool concurrent = false;
  cudaStream_t side[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<void*> side_y;
  std::vector<const int32_t*> side_rows, side_zero;
  std::vector<int64_t> n_side_rows, n_side_zero;
  std::string canon;

  ~Plan();
  void* up(const void* h, size_t bytes, cudaStream_t s, size_t pad_to = 0);
  const int32_t* up_i32(const std::vector<int64_t>& v, cudaStream_t s, const char* what);
  const void* up_vals(const std::vector<double>& v, cudaStream_t s, size_t pad_elems = 0);
  void upload(cudaStream_t s);
  void upload_pad(const HostPart& h, DevPart& d, cudaStream_t s, const std::vector<int32_t>* pad_col = nullptr);
  bool encode_xcache(const HostPart& h, DevPart& d, cudaStream_t s, std::vector<int32_t>& col_enc,
                     std::vector<int32_t>& pad_enc);
  void try_xwin(const HostPart& h, DevPart& d, cudaStream_t s);
  void mark_heavy_rows(cudaStream_t s);
  const int32_t* d_heavy_rows = nullptr;  // fp32 A25 heavy rows (sorted) + fp64 scratch
  double* d_heavy_acc = nullptr;
  int64_t n_heavy = 0;
  void compute_model();
};

// On-device Designer (devbuild.cu) for NNZ-blocked graphs: dev_build_spec decides whether
// a graph is in the device-built family (and parses its parameters), dev_build builds the
// format into P (launches, pre-pass, heavy rows, spans, bytes model, info).
struct DevSpec {
  int sort = 0;       // 0 none, 1 SORT, 2 SORT_SUB
  int64_t g = 0;      // SORT_SUB group
  int64_t K = 0;      // BMW_NNZ_BLOCK (0: no BMW level)
  int64_t k = 0;      // BMT_NNZ_BLOCK
  bool pad = false;
  int pad_scope = -1; // -1 GLOBAL, 1 BMW
  int64_t vec = 1;
  int wred = RED_NONE;
  int tpb = 0, grid = 0, stages = 2;
  int64_t xcache = 0;
};
bool dev_build_spec(const Seq& g, const Matrix& A, int flags, DevSpec* sp);
void dev_build(Plan& P, const Matrix& A, const DevSpec& sp, cudaStream_t s);

// "dev.<key>" exports: the device arrays read back and decoded to the logical layout
// (readback.cpp); keys "dev.p<part>.<name>"
std::vector<std::pair<std::string, std::vector<uint8_t>>> device_arrays(const Plan& P);

// Enqueue one SpMV of the plan on `stream` (pre-pass, parts, epilogue); with n_peers > 0
// every part's final STORE of a row in [peer_lo[i], peer_hi[i]) also goes to peer_y[i]
// (+ the row offset).  Returns cudaError_t.
int run_plan_peers(Plan& P, const void* x, void* y, double alpha, double beta, void* stream, void* const* peer_y,
                   const int64_t* peer_lo, const int64_t* peer_hi, int n_peers);

}  // namespace as

struct as_plan_s {
  std::unique_ptr<as::Plan> P;
};
