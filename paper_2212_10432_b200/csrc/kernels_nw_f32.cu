// NNZ_WARP launch group of the SpMV kernel family, value type float (see klaunch.h).
#include "kernels_impl.cuh"

namespace as {
AS_KERNELS_INSTANTIATE_NNZ_WARP(float)
}  // namespace as
