// Kernel-side parameter blocks and HBM layout of the slab state.
//
// Layout: one allocation per buffer, x-plane major so that an x-plane
// holding every component is contiguous (halo planes ship without packing):
//     state[xs][c][ys][zs],  xs = 0 .. nx+1 (0, nx+1: ghost planes)
//                            ys = y + 1 in 0 .. ny+1, zs = z + 2 in 1 .. nz+2 (row stride zp)
// The y/z ghost rows/columns hold the periodic images of the opposite edge; every kernel that
// writes an edge cell also writes its images, so a tile never wraps and one TMA box per plane
// covers it.  Column 0 is padding: with z = 0 at the even column 2, every even-z cell pair is
// an aligned 8-byte word pair (one st.global.v2 per component in the interior kernel).
//   fp32: c = 0..9  -> d = rho-1, j_x, j_y, j_z, sneq_xx, xy, xz, yy, yz, zz   (float)
//   q16 : c = 0..4  -> u32 words, word k = code(2k) | code(2k+1) << 16
#pragma once
#include <cuda.h>
#include <stdint.h>
#include "hlbm_math.cuh"

namespace hlbm {

#ifndef HLBM_HALO_WARPS
#define HLBM_HALO_WARPS 1
#endif
#ifndef HLBM_PULL_RT
#define HLBM_PULL_RT 1
#endif
#ifndef HLBM_IDLE_ROWS
#define HLBM_IDLE_ROWS 1
#endif
#ifndef HLBM_NW
#define HLBM_NW 16
#endif
constexpr int kNW = HLBM_NW;     // warps per CTA: halo warp(s) + one warp per interior y row
constexpr int kCtaPerSm = kNW > 16 ? 1 : 16 / kNW;   // resident CTAs per SM (<= 128 registers per thread)
constexpr int kHaloWarps = HLBM_HALO_WARPS;   // 1: warp 0 does both halo rows; 2: warps 0 and 15
constexpr int kRows = kNW - kHaloWarps;   // interior rows per tile
constexpr int kBoxRows = kRows + 2;   // rows of a plane tile in shared memory (+1 halo row per side)
constexpr int kZW = 64;          // z cells covered by one warp (32 lanes x 2 cells)
constexpr int kZT = 60;          // interior z cells per tile (lanes 1..30; lanes 0 and 31 are halo)
constexpr int kZOff = 2;         // storage column of z = 0
constexpr int kNSlot = 18;       // exchanged values per cell pair: (cx 3) x (cy +-1) x (kz 3)
constexpr int kMaxXseg = 128;    // longest x segment of one interior CTA (auto_xseg caps here too)

struct Geo {
  int nx, ny, nz;          // local interior dims (x = slab axis)
  int zp;                  // padded row length (>= nz + 3, multiple of 4)
  int64_t cstride;         // (ny+2)*zp        elements between components
  int64_t pstride;         // NC*(ny+2)*zp     elements between x planes
  int x_lo_src, x_hi_src;  // storage plane read for source plane -1 / nx ; -1 => inflow constants
  int nzt, nyt, nxs, xseg; // tiling of the interior kernel
  int xb, xr;              // destination x-range [xb, xr) of this launch (segments start at xb)
  int gx0, gny, gnz;       // slab offset in the global grid (dither key)
  int gnx_total;           // global nx
};

struct Stats {                 // device-side accumulators (reset by the host per step batch)
  double mass_dev;             // sum over fluid cells of (rho - 1)
  double mom[3];
  unsigned int max_u2_bits;    // float bits of max |u|^2 (NaN sorts above +inf)
  unsigned int nonfinite;
  unsigned long long sat[10];
  double force[3];             // momentum exchange on the triangle mesh (mode 2 links)
  double torque[3];
};

struct StepArgs {
  CUtensorMap tmap_in;              // 4-D map over `in`: (zs, ys, c, xs), box (64, 16, NC, 1)
  const void* in;
  void* out;
  Geo g;
  Relax R;
  Codec Q;
  float inflow[10];                 // internal-form state of an inflow ghost plane
  float pre_step[10], pre_off[10];  // q16 decode straight into the coeffs_pre input scales
  float pre_k[10];                  // fp32: input scales of coeffs_pre (hlbm_math.cuh pre_scale)
  float inflow_pre[10];             // inflow ghost state in coeffs_pre scales
  const uint32_t* special_bits;     // per (xs,y) row bitmask of boundary/solid cells, or null
  int bits_row_words;               // u32 words per bitmask row
  uint32_t step_key;                // dither key for this step
  int do_stats;
  Stats* stats;
  const float* cut_t;               // mesh mode: (n_list, 27) hit parameters t (p = x - t c_i)
  const uint32_t* wall_masks;       // mesh mode with wall faces: per list entry, links into a wall
  float solid_v[3], solid_w[3], solid_c[3];   // rigid-body velocity, angular velocity, centre
};

// element offset of cell (y, z) of storage plane sp (component 0)
__host__ __device__ __forceinline__ int64_t cell_off(const Geo& g, int sp, int y, int z) {
  return (int64_t)sp * g.pstride + (int64_t)(y + 1) * g.zp + (z + kZOff);
}

__host__ __device__ __forceinline__ int wrapi(int a, int n) {
  a %= n;
  return a < 0 ? a + n : a;
}

}  // namespace hlbm
