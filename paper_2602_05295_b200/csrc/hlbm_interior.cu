// fluid_interior launch dispatch + the fp32 variants (kernel template: hlbm_interior.cuh; the
// 16-bit variants are compiled in hlbm_interior_q{0,1,2}.cu, one translation unit per codec mode).
#include "hlbm_interior.cuh"
#include "hlbm_launch.h"

namespace hlbm {

static cudaError_t launch_interior_fp32(const StepArgs& A, int nblocks, bool force, bool special,
                                        cudaStream_t st) {
  if (!A.do_stats)
    return force ? launch_interior_t<false, true, false, false, false, 0>(A, nblocks, st)
                 : launch_interior_t<false, false, false, false, false, 0>(A, nblocks, st);
  if (special)
    return force ? launch_interior_t<false, true, true, false, true, 0>(A, nblocks, st)
                 : launch_interior_t<false, false, true, false, true, 0>(A, nblocks, st);
  return force ? launch_interior_t<false, true, false, false, true, 0>(A, nblocks, st)
               : launch_interior_t<false, false, false, false, true, 0>(A, nblocks, st);
}

cudaError_t launch_fluid_interior(const StepArgs& A, bool q16, bool force, bool special, bool dither,
                                  int qmode, cudaStream_t st) {
  const int nblocks = A.g.nzt * A.g.nyt * A.g.nxs;
  if (nblocks == 0) return cudaSuccess;
  if (!q16) return launch_interior_fp32(A, nblocks, force, special, st);
  switch (qmode) {
    case 0: return launch_interior_q16_m0(A, nblocks, force, special, dither, st);
    case 1: return launch_interior_q16_m1(A, nblocks, force, special, dither, st);
    case 2: return launch_interior_q16_m2(A, nblocks, force, special, dither, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hlbm
