// Peer-memory exchange of the ROW_DIV multi-GPU path (as_spmv_dist, AS_EXCH_PEER).
//
// After the band SpMV, ONE kernel streams this rank's y band (or, with halo windows, only the
// rows each peer reads) into every peer's y_full over
// NVLink (P2P stores into CUDA IPC mappings of the peers' buffers) and, once every CTA's
// stores are fenced at system scope, the last CTA publishes the call's epoch into each
// peer's flag array with a release store.  Each rank's stream then runs a one-CTA wait
// kernel that acquires its peers' flags for that epoch (bounded by a timeout so a missing
// peer cannot hang the GPU).  No NCCL on this path: one pass over the band instead of the
// AllGatherV's rounds.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "devpart.h"

namespace as {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <class E>
__global__ void __launch_bounds__(512) k_push(const E* __restrict__ src, PeerPush pp, unsigned* ctr, unsigned target,
                                              unsigned long long epoch, int rank) {
  // pp.lo / pp.hi in elements of E here (converted by launch_push)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int p = 0; p < pp.n; ++p)
    for (int64_t i = pp.lo[p] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pp.hi[p]; i += stride)
      ((E*)pp.dst[p])[i] = src[i];
  __threadfence_system();  // this thread's peer stores before the CTA's arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(ctr, 1u);
    if (prev + 1 == target) {  // last CTA of this call: every CTA's stores are fenced
      __threadfence_system();
      for (int p = 0; p < pp.n; ++p) st_release_sys(pp.flag[p] + rank, epoch);
    }
  }
}

__global__ void k_wait(const unsigned long long* flags, int world, int rank, unsigned long long epoch,
                       unsigned long long timeout_ns, int* status) {
  const int r = threadIdx.x;
  if (r < world && r != rank) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(flags + r) < epoch) {
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(status, 1);
        break;
      }
      __nanosleep(200);
    }
  }
}

}  // namespace

int launch_push(const void* src, PeerPush pp, unsigned* ctr, unsigned* target, unsigned long long epoch, int rank,
                void* stream) {
  // widest element every address and range bound is aligned to
  uintptr_t a = (uintptr_t)src;
  int64_t most = 0;
  for (int p = 0; p < pp.n; ++p) {
    a |= (uintptr_t)pp.dst[p];
    if (pp.hi[p] > pp.lo[p]) {
      a |= (uintptr_t)pp.lo[p] | (uintptr_t)pp.hi[p];
      most = std::max(most, pp.hi[p] - pp.lo[p]);
    }
  }
  const int esz = (a & 15) == 0 ? 16 : (a & 7) == 0 ? 8 : 4;
  for (int p = 0; p < pp.n; ++p) {
    pp.lo[p] /= esz;
    pp.hi[p] = pp.hi[p] > pp.lo[p] * esz ? pp.hi[p] / esz : pp.lo[p];
  }
  const int64_t cnt = most / esz;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = std::max<int64_t>(1, std::min<int64_t>((cnt + 511) / 512, (int64_t)sms * 2));
  // the CTA arrival counter is monotonic; this call's CTAs bring it to `want`.  The host
  // target advances only once the launch is known to have been accepted, so a failed launch
  // cannot leave it ahead of the device counter (which would stall every later epoch)
  const unsigned want = *target + (unsigned)g;
  cudaStream_t s = (cudaStream_t)stream;
  if (esz == 16) k_push<uint4><<<g, 512, 0, s>>>((const uint4*)src, pp, ctr, want, epoch, rank);
  else if (esz == 8) k_push<uint64_t><<<g, 512, 0, s>>>((const uint64_t*)src, pp, ctr, want, epoch, rank);
  else k_push<uint32_t><<<g, 512, 0, s>>>((const uint32_t*)src, pp, ctr, want, epoch, rank);
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) *target = want;
  return (int)e;
}

int launch_wait(const unsigned long long* flags, int world, int rank, unsigned long long epoch,
                unsigned long long timeout_ns, int* status, void* stream) {
  const int t = (world + 31) / 32 * 32;
  k_wait<<<1, t, 0, (cudaStream_t)stream>>>(flags, world, rank, epoch, timeout_ns, status);
  return (int)cudaGetLastError();
}

}  // namespace as
