// Monotonic dynamic shared-memory opt-in (shared by the kernel translation units).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace as {

// Dynamic shared-memory opt-in of a kernel function.  The attribute is process-wide per
// device and function, and every plan launching the function relies on it: raise it to
// `bytes` only if it is lower (a later plan with a smaller need must not lower it under an
// earlier plan, which would make that plan's launches fail).
template <class K>
inline cudaError_t smem_optin(K kern, size_t bytes) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, kern);
  if (e != cudaSuccess) return e;
  if ((size_t)a.maxDynamicSharedSizeBytes >= bytes) return cudaSuccess;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace as
