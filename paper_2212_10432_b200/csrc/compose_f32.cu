// k_compose group: value type float, BMT_PAD false (see compose.cu).
#include "compose_impl.cuh"

namespace as {
AS_COMPOSE_INSTANTIATE(float, false)
}  // namespace as
