// Device-resident format of one plan part + its launch geometry (POD, passed by value to
// the sm_100a kernels).  Pointers are device pointers; a NULL index array means the array
// is linear by construction and is computed instead of loaded (reading A17, the paper's
// Model-Driven Format Compression example "row_offset = 64*bid").
#pragma once
#include <cstddef>
#include <cstdint>

namespace as {

enum Fam {
  FAM_NONE = 0,
  FAM_THREAD_ROW,    // BMT_ROW_BLOCK (+ROW parents, +BMT_PAD) + THREAD_TOTAL|THREAD_BITMAP_RED_G
  FAM_NNZ_THREAD,    // BMT_NNZ_BLOCK + THREAD_BITMAP_RED_G (row straddlers -> atomics, "_G")
  FAM_NNZ_WARP,      // BMW_* + BMT_NNZ_BLOCK + THREAD_BITMAP_RED_G + WARP_SEG_ADD_RED|WARP_BITMAP_RED
  FAM_WARP_ROW,      // BMW_* (single-row) [+BMT_NNZ+THREAD_TOTAL] + WARP_TOTAL_RED
  FAM_BLOCK_TOTAL,   // BMTB_* (single-row) + SHMEM_TOTAL_RED
  FAM_BLOCK_OFFSET,  // BMTB_* + SHMEM_OFFSET_RED (CSR-stream)
  FAM_DIA,           // DIA part of DIA_DECOM
  FAM_DENSE,         // DENSE part of DENSE_DECOM
  FAM_COMPOSE        // any other legal level/reduction composition (compose.cu, P:313/P:322 adapters)
};

// reduction of one level (BMTB, BMW, BMT) of the implementing stage
enum Red { RED_NONE = 0, RED_TOTAL = 1, RED_BITMAP = 2, RED_SEG = 3, RED_OFFSET = 4 };

constexpr int kMaxDiags = 64;
constexpr int kMaxPatches = 8;

// Model-Driven Format Compression (§V-D, NEXT-2): an index array replaced by
// model(i) = b + k1*(i / w) + k2*(i % w) (linear: w = 1; periodic linear; step: k2 = 0) with
// up to kMaxPatches exceptions (i, value) -- "a small number of errors can be tolerated by
// adding if statements".  kind 0 = no model.
struct IdxModel {
  int64_t b = 0, k1 = 0, k2 = 0, w = 1;
  int kind = 0, np = 0;
  int64_t pi[kMaxPatches] = {0}, pv[kMaxPatches] = {0};
};
constexpr int kMaxFusedPeers = 7;  // as_spmv_dist fused peer stores: up to 8 ranks

struct DevPart {
  int fam = FAM_NONE;
  int dtype = 1;  // AS_R32F = 0, AS_R64F = 1
  int mode = 0;   // 0 STORE (y = a*s + b*y), 1 ADD (y += a*s); atomics always add
  int variant = 0;
  int64_t m_p = 0, nnz_p = 0, n = 0;
  // COMPRESS output
  const int32_t* origin = nullptr;  // NULL -> org_model(row) if fitted, else origin_base + row
  int64_t origin_base = 0;
  IdxModel org_model;
  const int32_t* row_ptr = nullptr;
  const int32_t* col = nullptr;
  const void* val = nullptr;
  // BMT level
  int64_t n_bmt = 0;
  int64_t k = 0;                          // BMT_NNZ size
  int64_t s = 0;                          // BMT_ROW size
  const int32_t* bmt_start = nullptr;     // NNZ BMTs: NULL -> t*k
  const int32_t* bmt_row_ptr = nullptr;   // ROW BMTs: NULL -> brp_model(t) if fitted, else min(t*s, m_p)
  IdxModel brp_model;
  const int32_t* bmt_first_row = nullptr;  // NULL -> fr_model(t) (NNZ BMTs, model-driven compression)
  IdxModel fr_model;
  const uint32_t* bitmap = nullptr;
  int bm_words = 0;
  // short-array fusion ("combining multiple short-data-type arrays"): first_row and
  // the bitmap words of a BMT interleaved in one array of fr_stride = bm_stride int32 words
  // per BMT ({first_row, bm0, bm1, ...}), so one sector serves all of a BMT's metadata
  int bm_stride = 0, fr_stride = 1;
  const uint32_t* bits = nullptr;         // tile form: packed head bits, 1 per nonzero
  int tile = 0;                           // NNZ_WARP tile kernel (k in {1,2,4})
  // BMW level
  int64_t n_bmw = 0;
  const int32_t* bmw_bmt_ptr = nullptr;   // NNZ_WARP: BMT range per BMW; NULL -> bwp_model(w) if fitted, else w*bmts_per_bmw
  IdxModel bwp_model;
  int64_t bmts_per_bmw = 0;
  const int32_t* bmw_start = nullptr;     // WARP_ROW: nz start per BMW
  const int32_t* bmw_first_row = nullptr; // WARP_ROW: NULL -> w
  int bmw_all_excl = 0;
  // BMTB level
  int64_t n_bmtb = 0;
  const int32_t* bmtb_start = nullptr;    // NULL -> b*k1
  int64_t k1 = 0;
  const int32_t* bmtb_first_row = nullptr;
  int64_t max_block_nnz = 0;
  int64_t smem_cap = 0, smem_rcap = 0;    // TMA CSR-stream: staged elements / row offsets per stage
  // x-window staging (k_nnz_thread_xw): ring size (power of 2), exact CTA count, rounds per
  // CTA, and per (CTA, round) the [lo, hi] x range
  int64_t xw_size = 0, xw_grid = 0, xw_rpc = 0;
  const int32_t* xwin = nullptr;
  // FAM_COMPOSE: per-level reductions (Red), which levels exist (a missing BMT level is
  // uploaded as NNZ_BLOCK(1) BMTs), BMTB -> child block range (BMWs, else BMTs), and whether
  // no level reduces below GMEM (every nonzero written on its own)
  int tred = 0, wred = 0, bred = 0;
  int has_w = 0, has_b = 0, per_elem = 0, t_synth = 0;
  const int32_t* bmtb_child = nullptr;
  // hot-x cache (SET_RESOURCE xcache): xh_n columns staged in shared memory per CTA, encoded
  // as ~slot in col / pad_col; persistent grid of xh_ctas CTAs per SM
  const int32_t* xh_cols = nullptr;
  int64_t xh_n = 0;
  int xh_ctas = 0;
  // BMT_PAD (slot-major interleaved)
  int pad = 0, vec = 1;
  int64_t n_grp = 0, grp_regular = 0;     // BMTs per group if regular, else 0
  int pad_grp_bmw = 0;                    // pad groups are exactly the BMWs (scope=BMW)
  const int32_t* grp_first_bmt = nullptr; // n_grp + 1
  const int64_t* grp_base = nullptr;      // n_grp slot offsets; NULL -> pb_model(g)
  const int32_t* grp_width = nullptr;     // n_grp; NULL -> pw_model(g) (Model-Driven Format Compression)
  IdxModel pb_model, pw_model;
  const int32_t* pad_col = nullptr;
  const void* pad_val = nullptr;
  // DIA
  int D = 0;
  int64_t r0 = 0, mb = 0, dia_stride = 0;
  int32_t dia_off[kMaxDiags] = {0};
  const void* dia_val = nullptr;
  // DENSE
  int64_t b = 0, n_tile_rows = 0, row_lo = 0, row_hi = 0;
  const int32_t* tile_row_id = nullptr;
  const int32_t* tile_row_ptr = nullptr;
  const int32_t* tile_col = nullptr;
  const void* tile_val = nullptr;
  // fp32 plans: rows whose chain of fp32 partial additions would exceed the A25 bound add
  // into an fp64 scratch instead (sorted global row ids, scratch slot = index)
  const int32_t* heavy_rows = nullptr;
  const uint32_t* heavy_bits = nullptr;   // 1 bit per global row: is heavy
  int64_t n_heavy = 0;
  double* heavy_acc = nullptr;
  // as_spmv_dist, AS_EXCH_PEER on single-writer plans: every STORE of a final y value is
  // also written to the same offset of each peer's y_full band (P2P stores over NVLink into
  // CUDA IPC mappings), fusing the exchange into the SpMV epilogue
  void* peer_y[kMaxFusedPeers] = {nullptr};
  int64_t peer_lo[kMaxFusedPeers] = {0}, peer_hi[kMaxFusedPeers] = {0};  // plan rows [lo, hi) peer i reads
  int n_peer = 0;
  // launch
  int tpb = 256, grid = 0;
  size_t smem = 0;
  // scalars (filled per call)
  double alpha = 1.0, beta = 0.0;
};

// kernels.cu
int launch_part(const DevPart& p, const void* x, void* y, void* stream);      // returns cudaError_t
int launch_prepass(const int32_t* rows, int64_t n, double beta, void* y, int dtype, void* stream);
int launch_l2_flush(void* buf, size_t bytes, int pattern, void* stream);  // memset + read-back
int launch_side_add(const int32_t* rows, int64_t n, const void* ys, void* y, int dtype, void* stream);  // R-conc
int launch_heavy_epilogue(const int32_t* rows, const double* acc, int64_t n, void* y, void* stream);  // fp32 y
int prepare_part(DevPart& p);  // per-kernel attributes (smem opt-in); returns cudaError_t
// compose.cu
int launch_compose(const DevPart& p, const void* x, void* y, void* stream);
int prepare_compose(DevPart& p);
const char* fam_kernel_name(const DevPart& p);
int device_max_smem_optin(int device);
int device_sm_count(int device);
int xw_ctas_per_sm(int dtype, int pad, int vec, int tpb, size_t smem);

// spmm.cu (NEXT-4): the plain CSR arrays of a CSR-family part, uploaded with AS_PLAN_SPMM
struct SpmmPart {
  const int32_t* rows = nullptr;  // m_p global output rows
  const int32_t* rp = nullptr;    // m_p + 1
  const int32_t* col = nullptr;
  const void* val = nullptr;
  const uint8_t* add = nullptr;   // per row: 1 = add alpha*s (atomic-class or ADD-mode row), 0 = store
  int64_t m_p = 0;
};
int launch_spmm_part(const DevPart& p, const SpmmPart& s, double alpha, double beta, const void* X, int64_t ldx,
                     void* Y, int64_t ldy, int64_t k, void* stream);
// rows != NULL: y[r][:] = beta*y[r][:] for the n listed rows; else for all m rows
int launch_spmm_prepass(const int32_t* rows, int64_t n, int64_t m, double beta, void* Y, int64_t ldy, int64_t k,
                        int dtype, void* stream);

// dist_kernels.cu: peer-memory exchange of as_spmv_dist (AS_EXCH_PEER)
constexpr int kMaxPeers = 64;  // AS_DIST_MAX_WORLD
struct PeerPush {
  void* dst[kMaxPeers];                 // peer y_full + band offset (IPC mappings)
  unsigned long long* flag[kMaxPeers];  // peer flag arrays (IPC mappings)
  int64_t lo[kMaxPeers], hi[kMaxPeers]; // bytes [lo, hi) of the band peer p receives (its halo window)
  int n = 0;
};
// Push bytes [pp.lo[p], pp.hi[p]) of src to every pp.dst[p] (empty ranges: flags only), then
// release the epoch into every peer's flag array.
int launch_push(const void* src, PeerPush pp, unsigned* ctr, unsigned* target, unsigned long long epoch, int rank,
                void* stream);
int launch_wait(const unsigned long long* flags, int world, int rank, unsigned long long epoch,
                unsigned long long timeout_ns, int* status, void* stream);

}  // namespace as
