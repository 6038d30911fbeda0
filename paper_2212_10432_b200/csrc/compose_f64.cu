// k_compose group: value type double, BMT_PAD false (see compose.cu).
#include "compose_impl.cuh"

namespace as {
AS_COMPOSE_INSTANTIATE(double, false)
}  // namespace as
