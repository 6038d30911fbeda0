// Remaining launch groups of the SpMV kernel family (thread-row, warp-row, block, DIA,
// dense), both value types (see klaunch.h).
#include "kernels_impl.cuh"

namespace as {
AS_KERNELS_INSTANTIATE_OTHER(float)
AS_KERNELS_INSTANTIATE_OTHER(double)
}  // namespace as
