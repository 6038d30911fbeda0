// Multi-GPU ROW_DIV SpMV: as_dist_* entry points.
//
// One process per GPU.  Rank r runs its band plan into y_full[cuts[r]:cuts[r+1]] and then,
// per call, either nothing, an NCCL AllGatherV (grouped broadcasts), or the peer-memory
// push of dist_kernels.cu.  NCCL is resolved at run time with dlopen so that the library
// loads (and the CPU tests run) where no NCCL is installed; inside a torch process the
// already-loaded libnccl.so.2 is reused.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <map>
#include <string>

#include "internal.h"
#include "plan.h"

using namespace as;

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl t;
    t.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!t.h) t.h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!t.h) return t;
    t.getUniqueId = (decltype(t.getUniqueId))dlsym(t.h, "ncclGetUniqueId");
    t.commInitRank = (decltype(t.commInitRank))dlsym(t.h, "ncclCommInitRank");
    t.commDestroy = (decltype(t.commDestroy))dlsym(t.h, "ncclCommDestroy");
    t.broadcast = (decltype(t.broadcast))dlsym(t.h, "ncclBroadcast");
    t.groupStart = (decltype(t.groupStart))dlsym(t.h, "ncclGroupStart");
    t.groupEnd = (decltype(t.groupEnd))dlsym(t.h, "ncclGroupEnd");
    t.errStr = (decltype(t.errStr))dlsym(t.h, "ncclGetErrorString");
    if (!t.getUniqueId || !t.commInitRank || !t.commDestroy || !t.broadcast || !t.groupStart || !t.groupEnd ||
        !t.errStr)
      t.h = nullptr;
    return t;
  }();
  if (!n.h) fail(AS_ERR_NCCL, "libnccl.so.2 not found (or missing symbols)");
  return n;
}

void ck_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(AS_ERR_NCCL, std::string(what) + ": " + nccl().errStr(r));
}

// cuMemGetAddressRange through the runtime's driver entry point (no libcuda link dependency)
void alloc_range(void* p, char** base, size_t* size) {
  using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (Fn)f;
  }();
  if (!fn) fail(AS_ERR_CUDA, "cuMemGetAddressRange unavailable");
  unsigned long long b = 0;
  if (fn(&b, size, (unsigned long long)(uintptr_t)p) != 0) fail(AS_ERR_INVALID_ARG, "y_full is not device memory");
  *base = (char*)(uintptr_t)b;
}

constexpr uint32_t kMagic = 0x41534450;  // "ASDP"
struct Blob {                            // AS_DIST_HANDLE_BYTES
  cudaIpcMemHandle_t y;                  // allocation holding y_full
  int64_t y_off;                         // y_full - allocation base
  cudaIpcMemHandle_t flags;              // the rank's flag array (offset 0)
  int32_t rank;
  uint32_t magic;
};
static_assert(sizeof(Blob) <= AS_DIST_HANDLE_BYTES, "blob too large");

}  // namespace

struct as_dist_s {
  int rank = 0, world = 1, device = -1;
  ncclComm_t comm = nullptr;
  std::vector<int64_t> cuts;
  // device words: flags[world] (written by peers), then the push CTA counter and the status
  unsigned long long* flags = nullptr;
  unsigned* ctr = nullptr;
  int* status = nullptr;
  void* words = nullptr;
  unsigned target = 0;
  unsigned long long epoch = 0;
  std::map<std::string, char*> opened;             // IPC handle bytes -> mapped base (opened once)
  std::vector<unsigned long long*> peer_flags;     // [world], NULL for self / unopened
  std::map<void*, std::vector<char*>> peer_y;      // local y_full -> peers' y_full mappings
  std::vector<int64_t> win;                        // [2*world]: rows [lo, hi] of y_full rank q reads; empty = all
};

extern "C" {

as_status_t as_dist_unique_id(void* id) {
  return guard([&] {
    if (!id) fail(AS_ERR_INVALID_ARG, "NULL id");
    ncclUniqueId u;
    ck_nccl(nccl().getUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

as_status_t as_dist_init(int rank, int world, const void* id, int device, as_dist_t* out) {
  return guard([&] {
    if (!out) fail(AS_ERR_INVALID_ARG, "NULL out");
    if (world < 1 || world > AS_DIST_MAX_WORLD || rank < 0 || rank >= world)
      fail(AS_ERR_INVALID_ARG, "rank/world out of range (world <= AS_DIST_MAX_WORLD)");
    auto D = std::make_unique<as_dist_s>();
    D->rank = rank;
    D->world = world;
    D->device = device;
    D->peer_flags.assign(world, nullptr);
    if (device >= 0) {
      int cur = 0;
      check_cuda(cudaGetDevice(&cur), "cudaGetDevice");
      check_cuda(cudaSetDevice(device), "cudaSetDevice");
      // flags must be a plain cudaMalloc allocation (exported through CUDA IPC)
      const size_t bytes = 8 * (size_t)world + 16;
      cudaError_t e = cudaMalloc(&D->words, bytes);
      if (e == cudaSuccess) e = cudaMemset(D->words, 0, bytes);
      if (e != cudaSuccess) {
        cudaSetDevice(cur);
        check_cuda(e, "dist flags");
      }
      D->flags = (unsigned long long*)D->words;
      D->ctr = (unsigned*)(D->flags + world);
      D->status = (int*)(D->ctr + 2);
      if (id) {
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        ncclResult_t r = nccl().commInitRank(&D->comm, world, u, rank);
        if (r != ncclSuccess) {
          cudaFree(D->words);
          cudaSetDevice(cur);
          ck_nccl(r, "ncclCommInitRank");
        }
      }
      cudaSetDevice(cur);
    } else if (id) {
      fail(AS_ERR_INVALID_ARG, "an NCCL communicator needs a device");
    }
    *out = D.release();
  });
}

as_status_t as_dist_set_cuts(as_dist_t D, const int64_t* cuts) {
  return guard([&] {
    if (!D || !cuts) fail(AS_ERR_INVALID_ARG, "NULL argument");
    if (cuts[0] != 0) fail(AS_ERR_INVALID_ARG, "cuts[0] must be 0");
    for (int r = 0; r < D->world; ++r)
      if (cuts[r + 1] < cuts[r]) fail(AS_ERR_INVALID_ARG, "cuts must be non-decreasing");
    D->cuts.assign(cuts, cuts + D->world + 1);
  });
}

as_status_t as_dist_set_windows(as_dist_t D, const int64_t* lo_hi) {
  return guard([&] {
    if (!D) fail(AS_ERR_INVALID_ARG, "NULL dist");
    if (!lo_hi) {
      D->win.clear();
      return;
    }
    D->win.assign(lo_hi, lo_hi + 2 * (size_t)D->world);
  });
}

as_status_t as_dist_ipc_handle(as_dist_t D, void* y_full, void* handle) {
  return guard([&] {
    if (!D || !y_full || !handle) fail(AS_ERR_INVALID_ARG, "NULL argument");
    if (D->device < 0) fail(AS_ERR_INVALID_ARG, "host-only dist");
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(D->device);
    Blob b{};
    char* base = nullptr;
    size_t size = 0;
    try {
      alloc_range(y_full, &base, &size);
      check_cuda(cudaIpcGetMemHandle(&b.y, base), "cudaIpcGetMemHandle(y_full)");
      check_cuda(cudaIpcGetMemHandle(&b.flags, D->words), "cudaIpcGetMemHandle(flags)");
    } catch (...) {
      cudaSetDevice(cur);
      throw;
    }
    cudaSetDevice(cur);
    b.y_off = (char*)y_full - base;
    b.rank = D->rank;
    b.magic = kMagic;
    std::memset(handle, 0, AS_DIST_HANDLE_BYTES);
    std::memcpy(handle, &b, sizeof(b));
  });
}

as_status_t as_dist_open_peers(as_dist_t D, void* y_full, const void* handles) {
  return guard([&] {
    if (!D || !y_full || !handles) fail(AS_ERR_INVALID_ARG, "NULL argument");
    if (D->device < 0) fail(AS_ERR_INVALID_ARG, "host-only dist");
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(D->device);
    std::vector<char*> ys(D->world, nullptr);
    auto open = [&](const cudaIpcMemHandle_t& h) -> char* {
      std::string key((const char*)&h, sizeof(h));
      auto it = D->opened.find(key);
      if (it != D->opened.end()) return it->second;
      void* p = nullptr;
      check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      D->opened[key] = (char*)p;
      return (char*)p;
    };
    try {
      for (int r = 0; r < D->world; ++r) {
        Blob b;
        std::memcpy(&b, (const char*)handles + (size_t)r * AS_DIST_HANDLE_BYTES, sizeof(b));
        if (b.magic != kMagic || b.rank != r) fail(AS_ERR_INVALID_ARG, "handles must be as_dist_ipc_handle blobs in rank order");
        if (r == D->rank) continue;
        ys[r] = open(b.y) + b.y_off;
        if (!D->peer_flags[r]) D->peer_flags[r] = (unsigned long long*)open(b.flags);
      }
    } catch (...) {
      cudaSetDevice(cur);
      throw;
    }
    cudaSetDevice(cur);
    D->peer_y[y_full] = ys;
  });
}

as_status_t as_spmv_dist(as_dist_t D, as_plan_t local, const void* alpha, const void* x_full, const void* beta,
                         void* y_full, int exchange, void* stream) {
  return guard([&] {
    NvtxRange nv("as_spmv_dist");
    if (!D || !local || !y_full) fail(AS_ERR_INVALID_ARG, "NULL argument");
    if (D->cuts.empty()) fail(AS_ERR_INVALID_ARG, "as_dist_set_cuts first");
    Plan& P = *local->P;
    if (P.device != D->device) fail(AS_ERR_INVALID_ARG, "plan and dist are on different devices");
    const int r = D->rank;
    const int64_t r0 = D->cuts[r], r1 = D->cuts[r + 1], m = D->cuts[D->world];
    if (P.m != r1 - r0) fail(AS_ERR_INVALID_ARG, "plan rows != this rank's band (cuts[r+1]-cuts[r])");
    const size_t sv = P.dt == AS_R64F ? 8 : 4;
    if (x_full && (const char*)x_full < (const char*)y_full + m * sv && (const char*)y_full < (const char*)x_full + P.n * sv)
      fail(AS_ERR_INVALID_ARG, "x_full and y_full alias");
    std::vector<char*>* peers = nullptr;
    if (exchange == AS_EXCH_PEER) {
      auto it = D->peer_y.find(y_full);
      if (it == D->peer_y.end()) fail(AS_ERR_INVALID_ARG, "y_full not registered (as_dist_open_peers)");
      peers = &it->second;
    } else if (exchange == AS_EXCH_NCCL) {
      if (!D->comm) fail(AS_ERR_INVALID_ARG, "no NCCL communicator (as_dist_init without id)");
    } else if (exchange != AS_EXCH_NONE) {
      fail(AS_ERR_INVALID_ARG, "exchange must be AS_EXCH_NONE, AS_EXCH_NCCL or AS_EXCH_PEER");
    }
    char* band = (char*)y_full + r0 * sv;
    // fused exchange: single-writer band plans store every final y value into the peers'
    // y_full directly from the SpMV epilogue; the push kernel then only signals (0 bytes)
    const bool fused = exchange == AS_EXCH_PEER && P.single_writer && D->world - 1 <= kMaxFusedPeers &&
                       !std::getenv("AS_DIST_NO_FUSE");
    // rows [a, b) of this band peer q receives: all of it, or its halo window
    auto window = [&](int q, int64_t& a, int64_t& b) {
      a = 0;
      b = r1 - r0;
      if (D->win.empty()) return;
      a = std::max<int64_t>(0, D->win[2 * q] - r0);
      b = std::min<int64_t>(r1 - r0, D->win[2 * q + 1] + 1 - r0);
      if (b < a) b = a;
    };
    if (fused && P.m > 0) {
      void* pys[kMaxFusedPeers];
      int64_t plo[kMaxFusedPeers], phi[kMaxFusedPeers];
      int np = 0;
      for (int q = 0; q < D->world; ++q) {
        if (q == r) continue;
        window(q, plo[np], phi[np]);
        if (phi[np] <= plo[np]) continue;  // peer reads none of this band
        pys[np++] = (*peers)[q] + r0 * sv;
      }
      const double a = P.dt == AS_R64F ? *(const double*)alpha : (double)*(const float*)alpha;
      const double b = P.dt == AS_R64F ? *(const double*)beta : (double)*(const float*)beta;
      int cur0 = 0;
      cudaGetDevice(&cur0);
      cudaSetDevice(D->device);
      cudaError_t prior = cudaGetLastError();
      int e = prior != cudaSuccess ? (int)prior : run_plan_peers(P, x_full, band, a, b, stream, pys, plo, phi, np);
      cudaSetDevice(cur0);
      if (e) fail(AS_ERR_CUDA, std::string("fused band SpMV: ") + cudaGetErrorString((cudaError_t)e));
    } else if (P.m > 0) {
      as_status_t st = as_spmv(local, alpha, x_full, beta, band, stream);
      if (st != AS_OK) fail(st, as_last_error());
    }
    if (exchange == AS_EXCH_NONE) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(D->device);
    int err = 0;
    if (exchange == AS_EXCH_NCCL) {
      const Nccl& n = nccl();
      ncclResult_t res = n.groupStart();
      for (int q = 0; q < D->world && res == ncclSuccess; ++q) {
        const int64_t cnt = D->cuts[q + 1] - D->cuts[q];
        if (cnt <= 0) continue;
        char* p = (char*)y_full + D->cuts[q] * sv;
        res = n.broadcast(p, p, (size_t)cnt, sv == 8 ? ncclFloat64 : ncclFloat32, q, D->comm, (cudaStream_t)stream);
      }
      ncclResult_t e2 = n.groupEnd();
      cudaSetDevice(cur);
      ck_nccl(res != ncclSuccess ? res : e2, "AllGatherV (grouped ncclBroadcast)");
      return;
    }
    PeerPush pp;
    for (int q = 0; q < D->world; ++q) {
      if (q == r) continue;
      int64_t a = 0, b = 0;
      if (!fused) window(q, a, b);  // fused: the SpMV already stored the rows, flags only
      pp.dst[pp.n] = (*peers)[q] + r0 * sv;
      pp.flag[pp.n] = D->peer_flags[q];
      pp.lo[pp.n] = a * (int64_t)sv;
      pp.hi[pp.n] = b * (int64_t)sv;
      ++pp.n;
    }
    ++D->epoch;
    err = launch_push(band, pp, D->ctr, &D->target, D->epoch, r, stream);
    if (!err) err = launch_wait(D->flags, D->world, r, D->epoch, AS_DIST_WAIT_TIMEOUT_NS, D->status, stream);
    cudaSetDevice(cur);
    if (err) fail(AS_ERR_CUDA, std::string("peer exchange: ") + cudaGetErrorString((cudaError_t)err));
  });
}

as_status_t as_dist_check(as_dist_t D) {
  return guard([&] {
    if (!D) fail(AS_ERR_INVALID_ARG, "NULL dist");
    if (D->device < 0) return;
    int cur = 0, st = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(D->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(&st, D->status, sizeof(int), cudaMemcpyDeviceToHost);
    cudaSetDevice(cur);
    check_cuda(e, "as_dist_check");
    if (st) fail(AS_ERR_CUDA, "peer exchange timed out waiting for a peer's flag");
  });
}

void as_dist_destroy(as_dist_t D) {
  if (!D) return;
  if (D->device >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(D->device);
    cudaDeviceSynchronize();
    for (auto& kv : D->opened) cudaIpcCloseMemHandle(kv.second);
    if (D->comm) nccl().commDestroy(D->comm);
    if (D->words) cudaFree(D->words);
    cudaSetDevice(cur);
  }
  delete D;
}

}  // extern "C"
