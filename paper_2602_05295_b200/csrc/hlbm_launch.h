// Host-side launchers shared by the C-ABI translation unit.
#pragma once
#include "hlbm_params.cuh"

namespace hlbm {

struct Ranges {
  double mn[10], mx[10];
  double levels[10];
};
struct MaskGeo {
  int nx, ny, nz;
  int bc_ywall_lo, bc_ywall_hi, bc_zwall_lo, bc_zwall_hi;
  int q;   // velocity set (27 or 19): links counted
};

// qmode: 0 generic bit widths, 1 all 16-bit, 2 all 16-bit with the default QuantSpec ranges
struct MeshLinks {               // cut-link table of a static triangle mesh (device arrays)
  int64_t* cells = nullptr;      // sorted local linear cell indices
  uint32_t* masks = nullptr;     // bit i: the pull link x -> x - c_i crosses the mesh
  double* t64 = nullptr;         // (nb, 27) hit parameter, NaN where uncut (exported)
  float* t32 = nullptr;          // (nb, 27) the same in float for the step kernel
  int* tri = nullptr;            // (nb, 27) triangle index, -1 where uncut
  uint32_t* wmasks = nullptr;    // with wall faces: bit i = the link crosses a wall (bounce-back; the
                                 // list is then the union of mesh-cut and wall-adjacent cells)
  int32_t* dense = nullptr;      // per-cell list position or -1 (built for the fused Alg.-1 step)
  int64_t nb = 0;
};
cudaError_t build_mesh_links(const double* dV, const int* dF, int nf, int nx, int ny, int nz, MeshLinks& out,
                             cudaStream_t st, int q = 27);

cudaError_t launch_bits_from_list(const int64_t* cells, int64_t n, int nz, int row_words, uint32_t* bits,
                                  cudaStream_t st);

cudaError_t launch_fluid_interior(const StepArgs& A, bool q16, bool force, bool special, bool dither,
                                  int qmode, cudaStream_t st);
// D3Q19 interior step (two-chain moment-space streaming; fp32, or q16 with any codec mode)
cudaError_t launch_fluid_interior19(const StepArgs& A, bool q16, bool force, bool special, bool dither,
                                    int qmode, cudaStream_t st);
// mode 0: voxel bounce-back on masked links; 1: reset listed solid cells to rest;
// 2: triangle mesh, Eq.-8 boundary populations on masked links (t table in A.cut_t);
// 3: fused single-kernel step over all cells with a dense per-cell mask (Alg. 1 baseline)
cudaError_t launch_pull_cells(const StepArgs& A, const int64_t* cells, const uint32_t* masks,
                              int64_t n, int mode, bool q16, bool force, bool dither, cudaStream_t st,
                              int q = 27, int64_t base = 0);
// original HOME-LBM step (Alg. 1): post-collision storage cut, own-population
// reconstruction into shared memory, streaming within 8^3 tiles, voxel solid links inline
cudaError_t launch_alg1(const StepArgs& A, const uint32_t* fmask, bool q16, bool force, bool dither, int q,
                        cudaStream_t st, bool collide, const int32_t* mesh_idx = nullptr,
                        const uint32_t* mesh_masks = nullptr);
// dense per-cell position in the mesh cut-link list (-1: not listed), for the fused step
cudaError_t launch_mesh_index(const int64_t* cells, int64_t nb, int64_t n, int32_t* out, cudaStream_t st);
cudaError_t launch_import(const Geo& g, const Ranges& R, bool q16, void* dst, const double* rho,
                          const double* mom, const double* stress, int x0, int cnt,
                          unsigned long long* sat, unsigned int* nonpos, cudaStream_t st);
cudaError_t launch_export(const Geo& g, const Ranges& R, bool q16, const void* src, double* rho,
                          double* mom, double* stress, int x0, int cx, int y0, int cy, int z0, int cz,
                          cudaStream_t st);
cudaError_t launch_fused_masks(const uint32_t* links, const uint8_t* cls, int64_t n, uint32_t* out,
                               cudaStream_t st);
cudaError_t launch_classify(const uint8_t* mask_ext, const MaskGeo& m, uint32_t* links, uint8_t* cls,
                            cudaStream_t st);
int64_t compact_tiles(int64_t n);
cudaError_t launch_compact(const uint8_t* cls, const uint32_t* links, int64_t n, uint8_t want,
                           int64_t* counts, int64_t* total, int64_t* out_cells, uint32_t* out_masks,
                           bool count_only, cudaStream_t st);
cudaError_t launch_special_bits(const uint8_t* cls, int nx, int ny, int nz, int row_words,
                                uint32_t* bits, cudaStream_t st);
cudaError_t launch_fill_ghosts(const Geo& g, int NC, void* buf, cudaStream_t st);
// the node of largest |u|^2 (non-finite first) of the state A.in: key = u2 bits << 32 | ~linear index
cudaError_t launch_locate(const StepArgs& A, bool q16, unsigned long long* out, cudaStream_t st);
cudaError_t launch_pack_codes(const Geo& g, int NC, void* buf, uint32_t* dense, int dir, cudaStream_t st);
cudaError_t launch_init_modes(const Geo& g, bool q16, const Ranges& R, void* dst, double rho0,
                              const double* modes, int nmodes, cudaStream_t st);

}  // namespace hlbm
