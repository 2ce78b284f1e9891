// 16-bit variants of fluid_interior, codec mode 1 (hlbm_launch.h: qmode).
#include "hlbm_interior.cuh"

namespace hlbm {
HLBM_INTERIOR_Q16_UNIT(1)
}  // namespace hlbm
