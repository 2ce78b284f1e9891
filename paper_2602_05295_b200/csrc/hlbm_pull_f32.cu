// fp32 instantiations of the compacted boundary kernels (hlbm_cells.cuh: pull_cells, pull_list3)
#include "hlbm_cells.cuh"

namespace hlbm {
cudaError_t launch_pull_cells_f32(const StepArgs& A, const int64_t* cells, const uint32_t* masks, int64_t n,
                                  int mode, bool force, cudaStream_t st, int q, int64_t base) {
  return launch_pull_cells_t<false>(A, cells, masks, n, mode, force, false, st, q, base);
}
}  // namespace hlbm
