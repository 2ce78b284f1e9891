// D3Q19 variants of fluid_interior (LAT = 19; hlbm_interior.cuh, two-chain streaming): fp32 and
// 16-bit codes with the default QuantSpec (codec mode 2); the other codec modes (0: any bit preset,
// 1: 16-bit slots with custom ranges) are compiled in hlbm_interior_q19m.cu.  Solids run through the
// compacted kernels.
#include "hlbm_interior.cuh"
#include "hlbm_launch.h"

namespace hlbm {

cudaError_t launch_fluid_interior19_m01(const StepArgs& A, int nblocks, bool force, bool special, bool dither,
                                        int qmode, cudaStream_t st);

cudaError_t launch_fluid_interior19(const StepArgs& A, bool q16, bool force, bool special, bool dither,
                                    int qmode, cudaStream_t st) {
  const int nblocks = A.g.nzt * A.g.nyt * A.g.nxs;
  if (nblocks == 0) return cudaSuccess;
  if (q16 && qmode != 2) return launch_fluid_interior19_m01(A, nblocks, force, special, dither, qmode, st);
  const bool stats = A.do_stats != 0;
  // SPECIAL only changes the statistics (boundary / solid cells are finished by pull_cells)
#define HLBM_Q19(Q, F, D, S, M)                                                     \
  return (S && special) ? launch_interior_t<Q, F, true, D, S, M, 19>(A, nblocks, st) \
                        : launch_interior_t<Q, F, false, D, S, M, 19>(A, nblocks, st)
  if (!q16) {
    if (force) { if (stats) HLBM_Q19(false, true, false, true, 0); HLBM_Q19(false, true, false, false, 0); }
    if (stats) HLBM_Q19(false, false, false, true, 0);
    HLBM_Q19(false, false, false, false, 0);
  }
  if (force) {
    if (dither) { if (stats) HLBM_Q19(true, true, true, true, 2); HLBM_Q19(true, true, true, false, 2); }
    if (stats) HLBM_Q19(true, true, false, true, 2);
    HLBM_Q19(true, true, false, false, 2);
  }
  if (dither) { if (stats) HLBM_Q19(true, false, true, true, 2); HLBM_Q19(true, false, true, false, 2); }
  if (stats) HLBM_Q19(true, false, false, true, 2);
  HLBM_Q19(true, false, false, false, 2);
#undef HLBM_Q19
}

}  // namespace hlbm
