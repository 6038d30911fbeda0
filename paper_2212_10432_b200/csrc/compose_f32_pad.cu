// k_compose group: value type float, BMT_PAD true (see compose.cu).
#include "compose_impl.cuh"

namespace as {
AS_COMPOSE_INSTANTIATE(float, true)
}  // namespace as
