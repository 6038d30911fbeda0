// k_compose group: value type double, BMT_PAD true (see compose.cu).
#include "compose_impl.cuh"

namespace as {
AS_COMPOSE_INSTANTIATE(double, true)
}  // namespace as
