// D3Q19 16-bit variants of fluid_interior for the non-default codecs: codec mode 0 (bit presets
// 16/15 ... 12/11) and mode 1 (16-bit slots, custom ranges).  Mode 2 and fp32:
// hlbm_interior_q19.cu.
#include "hlbm_interior.cuh"
#include "hlbm_launch.h"

namespace hlbm {

template <int M>
static cudaError_t launch19_mode(const StepArgs& A, int nblocks, bool force, bool special, bool dither,
                                 cudaStream_t st) {
  const bool stats = A.do_stats != 0;
#define HLBM_Q19M(F, D, S)                                                               \
  return (S && special) ? launch_interior_t<true, F, true, D, S, M, 19>(A, nblocks, st)   \
                        : launch_interior_t<true, F, false, D, S, M, 19>(A, nblocks, st)
  if (force) {
    if (dither) { if (stats) HLBM_Q19M(true, true, true); HLBM_Q19M(true, true, false); }
    if (stats) HLBM_Q19M(true, false, true);
    HLBM_Q19M(true, false, false);
  }
  if (dither) { if (stats) HLBM_Q19M(false, true, true); HLBM_Q19M(false, true, false); }
  if (stats) HLBM_Q19M(false, false, true);
  HLBM_Q19M(false, false, false);
#undef HLBM_Q19M
}

cudaError_t launch_fluid_interior19_m01(const StepArgs& A, int nblocks, bool force, bool special, bool dither,
                                        int qmode, cudaStream_t st) {
  return qmode == 0 ? launch19_mode<0>(A, nblocks, force, special, dither, st)
                    : launch19_mode<1>(A, nblocks, force, special, dither, st);
}

}  // namespace hlbm
