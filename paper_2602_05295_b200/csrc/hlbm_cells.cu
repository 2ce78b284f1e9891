// Compacted per-cell kernels (split scheme, §4.2 / Alg. 3 role):
//
//   pull_cells      one thread per listed cell: full pull update over the 27 links, with every
//                   link whose source x - c_i is solid replaced by half-way bounce-back
//                   f_i(x) <- f+_opp(i)(x) (opposite table lattice.py:198-201).
//                   Run over the boundary-cell list after fluid_interior; with no list and
//                   zero masks it is also the full-grid GPU reference update.
//   reset_solid     solid cells -> rest state (they never feed a fluid cell: every link out of
//                   a solid cell is cut and bounced back).
//   classify / compact   voxel mask -> sorted boundary-cell list + 27-bit link masks and the
//                   solid list, deterministic (block prefix sums, no atomics in the ordering).
//   import / export reference layout (rho, mom, stress float64) <-> internal state.
#include <algorithm>
#include <climits>
#include "hlbm_cells.cuh"

namespace hlbm {

cudaError_t launch_pull_cells_f32(const StepArgs& A, const int64_t* cells, const uint32_t* masks, int64_t n,
                                  int mode, bool force, cudaStream_t st, int q, int64_t base);
cudaError_t launch_pull_cells_q16(const StepArgs& A, const int64_t* cells, const uint32_t* masks, int64_t n,
                                  int mode, bool force, bool dither, cudaStream_t st, int q, int64_t base);

cudaError_t launch_pull_cells(const StepArgs& A, const int64_t* cells, const uint32_t* masks,
                              int64_t n, int mode, bool q16, bool force, bool dither,
                              cudaStream_t st, int q, int64_t base) {
  if (q16) return launch_pull_cells_q16(A, cells, masks, n, mode, force, dither, st, q, base);
  if (dither) return cudaErrorInvalidValue;
  return launch_pull_cells_f32(A, cells, masks, n, mode, force, st, q, base);
}

// ------------------------------------------------------------------ mask -> lists
// solid flag on the padded grid; mask_ext holds local planes -1..nx (x-ghosts already resolved
// by the host per the x BCs / neighbouring slabs); y/z: wall ghost = solid, else periodic wrap.
// Order of the checks mirrors oracle/step.py:padded_solid (x padded first, then y, then z).
__device__ __forceinline__ bool padded_solid(const uint8_t* mask_ext, const MaskGeo& m, int x, int y,
                                             int z) {
  if (z < 0) { if (m.bc_zwall_lo) return true; z += m.nz; }
  else if (z >= m.nz) { if (m.bc_zwall_hi) return true; z -= m.nz; }
  if (y < 0) { if (m.bc_ywall_lo) return true; y += m.ny; }
  else if (y >= m.ny) { if (m.bc_ywall_hi) return true; y -= m.ny; }
  return mask_ext[((int64_t)(x + 1) * m.ny + y) * m.nz + z] != 0;
}

// per cell: link mask (fluid cells) and class flags: bit0 boundary, bit1 solid
__global__ void classify_cells(const uint8_t* __restrict__ mask_ext, MaskGeo m,
                               uint32_t* __restrict__ links, uint8_t* __restrict__ cls) {
  const int64_t n = (int64_t)m.nx * m.ny * m.nz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i / ((int64_t)m.ny * m.nz));
    const int64_t r = i - (int64_t)x * m.ny * m.nz;
    const int y = (int)(r / m.nz), z = (int)(r - (int64_t)y * m.nz);
    const bool solid = mask_ext[i + (int64_t)m.ny * m.nz] != 0;
    uint32_t lm = 0;
    if (!solid) {
#pragma unroll
      for (int k = 1; k < 27; ++k)
        if (k < m.q && padded_solid(mask_ext, m, x - kCX[k], y - kCY[k], z - kCZ[k])) lm |= 1u << k;
    }
    links[i] = lm;
    cls[i] = (uint8_t)((lm != 0 ? 1 : 0) | (solid ? 2 : 0));
  }
}

// dense per-cell mask of the fused step: link bits of fluid cells, bit 0 for solid cells
__global__ void fused_masks_kernel(const uint32_t* __restrict__ links, const uint8_t* __restrict__ cls, int64_t n,
                                   uint32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = links[i] | ((cls[i] & 2u) ? 1u : 0u);
}

cudaError_t launch_fused_masks(const uint32_t* links, const uint8_t* cls, int64_t n, uint32_t* out,
                               cudaStream_t st) {
  fused_masks_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(links, cls, n, out);
  return cudaGetLastError();
}

constexpr int kCompactTPB = 256;
constexpr int kCompactPer = 16;   // cells per thread per tile
constexpr int kCompactTile = kCompactTPB * kCompactPer;

// counts[b] = number of cells in tile b with (cls & want)
__global__ void compact_count(const uint8_t* __restrict__ cls, int64_t n, uint8_t want,
                              int64_t* __restrict__ counts) {
  __shared__ int warp_tot[kCompactTPB / 32];
  const int64_t base = (int64_t)blockIdx.x * kCompactTile;
  int c = 0;
  for (int k = 0; k < kCompactPer; ++k) {
    const int64_t i = base + (int64_t)k * kCompactTPB + threadIdx.x;
    if (i < n && (cls[i] & want)) ++c;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kCompactTPB / 32; ++w) t += warp_tot[w];
    counts[blockIdx.x] = t;
  }
}

// exclusive scan of the per-tile counts (single CTA, sequential chunks)
__global__ void compact_scan(int64_t* __restrict__ counts, int64_t nblocks, int64_t* __restrict__ total) {
  __shared__ int64_t carry;
  __shared__ int64_t buf[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nblocks; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nblocks ? counts[i] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int64_t t = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nblocks) counts[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// ordered scatter: within a tile, cells keep increasing linear index order
__global__ void compact_scatter(const uint8_t* __restrict__ cls, const uint32_t* __restrict__ links,
                                int64_t n, uint8_t want, const int64_t* __restrict__ offsets,
                                int64_t* __restrict__ out_cells, uint32_t* __restrict__ out_masks) {
  __shared__ int warp_tot[kCompactTPB / 32];
  __shared__ int64_t running;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kCompactTile;
  if (threadIdx.x == 0) running = offsets[blockIdx.x];
  __syncthreads();
  for (int k = 0; k < kCompactPer; ++k) {
    const int64_t i = base + (int64_t)k * kCompactTPB + threadIdx.x;
    const bool f = i < n && (cls[i] & want);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[w] = __popc(bal);
    __syncthreads();
    int64_t pre = running;
    for (int j = 0; j < w; ++j) pre += warp_tot[j];
    if (f) {
      const int64_t pos = pre + __popc(bal & ((1u << lane) - 1u));
      out_cells[pos] = i;
      if (out_masks) out_masks[pos] = links[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int j = 0; j < kCompactTPB / 32; ++j) t += warp_tot[j];
      running += t;
    }
    __syncthreads();
  }
}

// bitmask of special (boundary or solid) cells, one u32 word per 32 z-cells of a row
__global__ void special_bits_kernel(const uint8_t* __restrict__ cls, int nx, int ny, int nz, int row_words,
                                    uint32_t* __restrict__ bits) {
  const int64_t nwords = (int64_t)nx * ny * row_words;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / row_words;
    const int wz = (int)(i - row * row_words);
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int z = wz * 32 + b;
      if (z < nz && cls[row * nz + z]) v |= 1u << b;
    }
    bits[i] = v;
  }
}

// ------------------------------------------------------------------ import / export
// Exact float64 ranges for the codec (the SPEC quantizer is evaluated in float64 on import /
// export so that set_moments -> get_moments reproduces oracle/codec.py bit-for-bit).

// planes [x0, x0+cnt) of the interior; inputs are device copies of the reference layout
// (rho[cnt][ny][nz], mom[3][cnt][ny][nz], stress[6][cnt][ny][nz], float64)
template <bool Q16>
__global__ void import_f64(Geo g, Ranges R, void* dst, const double* __restrict__ rho,
                           const double* __restrict__ mom, const double* __restrict__ stress, int x0,
                           int cnt, unsigned long long* __restrict__ sat, unsigned int* __restrict__ nonpos) {
  const int64_t yz = (int64_t)g.ny * g.nz, n = yz * cnt;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int xl = (int)(i / yz);
    const int64_t r = i - (int64_t)xl * yz;
    const double rh = rho[i];
    if (!(rh > 0.0)) atomicAdd(nonpos, 1u);   // moments.py:147 "density must be positive" (host rejects)
    const double j0 = mom[i], j1 = mom[n + i], j2 = mom[2 * n + i];
    // sneq = stress - mom mom / rho  (moments.py:93-96, _outer_voigt :124-133)
    const double v[10] = {rh,
                          j0,
                          j1,
                          j2,
                          stress[i] - j0 * j0 / rh,
                          stress[n + i] - j0 * j1 / rh,
                          stress[2 * n + i] - j0 * j2 / rh,
                          stress[3 * n + i] - j1 * j1 / rh,
                          stress[4 * n + i] - j1 * j2 / rh,
                          stress[5 * n + i] - j2 * j2 / rh};
    const int yy = (int)(r / g.nz), zz = (int)(r - (int64_t)yy * g.nz);
    const int64_t off = cell_off(g, x0 + xl + 1, yy, zz);
    if (!Q16) {
      float* p = reinterpret_cast<float*>(dst) + off;
      p[0] = (float)(rh - 1.0);
      for (int c = 1; c < 10; ++c) p[c * g.cstride] = (float)v[c];
    } else {
      uint32_t code[10];
      for (int c = 0; c < 10; ++c) {
        // m' = (clamp(m) - min)/(max - min); q = floor(m'(2^b-1) + 1/2)
        const double m = v[c];
        if (sat && (m < R.mn[c] || m > R.mx[c])) atomicAdd(&sat[c], 1ull);
        const double mc = fmin(fmax(m, R.mn[c]), R.mx[c]);
        const double t = (mc - R.mn[c]) / (R.mx[c] - R.mn[c]) * R.levels[c] + 0.5;
        code[c] = (uint32_t)fmin(fmax(floor(t), 0.0), R.levels[c]);
      }
      uint32_t* p = reinterpret_cast<uint32_t*>(dst) + off;
      for (int k = 0; k < 5; ++k) p[k * g.cstride] = code[2 * k] | (code[2 * k + 1] << 16);
    }
  }
}

// export a box [x0,x0+cx) x [y0,y0+cy) x [z0,z0+cz) of the interior (y, z wrap periodically)
template <bool Q16>
__global__ void export_f64(Geo g, Ranges R, const void* src, double* __restrict__ rho,
                           double* __restrict__ mom, double* __restrict__ stress, int x0, int cx, int y0,
                           int cy, int z0, int cz) {
  const int64_t n = (int64_t)cx * cy * cz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int xl = (int)(i / ((int64_t)cy * cz));
    const int64_t r = i - (int64_t)xl * cy * cz;
    const int yl = (int)(r / cz), zl = (int)(r - (int64_t)yl * cz);
    const int y = wrapi(y0 + yl, g.ny), z = wrapi(z0 + zl, g.nz);
    const int64_t off = cell_off(g, x0 + xl + 1, y, z);
    double v[10];
    if (!Q16) {
      const float* p = reinterpret_cast<const float*>(src) + off;
      for (int c = 0; c < 10; ++c) v[c] = (double)p[c * g.cstride];
      v[0] += 1.0;
    } else {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(src) + off;
      for (int k = 0; k < 5; ++k) {
        const uint32_t wv = p[k * g.cstride];
        // m = min + q (max - min)/(2^b - 1)
        v[2 * k] = R.mn[2 * k] + (double)(wv & 0xFFFFu) * ((R.mx[2 * k] - R.mn[2 * k]) / R.levels[2 * k]);
        v[2 * k + 1] =
            R.mn[2 * k + 1] + (double)(wv >> 16) * ((R.mx[2 * k + 1] - R.mn[2 * k + 1]) / R.levels[2 * k + 1]);
      }
    }
    const double rh = v[0], j0 = v[1], j1 = v[2], j2 = v[3];
    rho[i] = rh;
    mom[i] = j0;
    mom[n + i] = j1;
    mom[2 * n + i] = j2;
    // stress = sneq + mom mom / rho   (neq_recompose, moments.py:99-102)
    stress[i] = v[4] + j0 * j0 / rh;
    stress[n + i] = v[5] + j0 * j1 / rh;
    stress[2 * n + i] = v[6] + j0 * j2 / rh;
    stress[3 * n + i] = v[7] + j1 * j1 / rh;
    stress[4 * n + i] = v[8] + j1 * j2 / rh;
    stress[5 * n + i] = v[9] + j2 * j2 / rh;
  }
}

// rho = rho0, u = sum_m a_m sin(2 pi k_m . x_global / N + phi_m), sneq = 0; modes are
// 7 doubles (kx, ky, kz, ax, ay, az, phi).  Used for the synthetic turbulence box.
template <bool Q16>
__global__ void init_modes(Geo g, Ranges R, void* dst, double rho0, const double* __restrict__ modes,
                           int nmodes) {
  const int64_t yz = (int64_t)g.ny * g.nz, n = yz * g.nx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i / yz);
    const int64_t r = i - (int64_t)x * yz;
    const int y = (int)(r / g.nz), z = (int)(r - (int64_t)y * g.nz);
    const int gx = g.gx0 + x;
    double u[3] = {0.0, 0.0, 0.0};
    for (int m = 0; m < nmodes; ++m) {
      const double* md = modes + 7 * m;
      // phase in turns, reduced exactly before the float sincos
      double t = md[0] * gx / (double)g.gnx_total + md[1] * y / (double)g.gny + md[2] * z / (double)g.gnz;
      t -= floor(t);
      const float sn = sinpif((float)(2.0 * t + md[6] / 3.141592653589793));
      u[0] += md[3] * sn;
      u[1] += md[4] * sn;
      u[2] += md[5] * sn;
    }
    const double v[10] = {rho0, rho0 * u[0], rho0 * u[1], rho0 * u[2], 0, 0, 0, 0, 0, 0};
    const int64_t off = cell_off(g, x + 1, y, z);
    if (!Q16) {
      float* p = reinterpret_cast<float*>(dst) + off;
      p[0] = (float)(rho0 - 1.0);
      for (int c = 1; c < 10; ++c) p[c * g.cstride] = (float)v[c];
    } else {
      uint32_t code[10];
      for (int c = 0; c < 10; ++c) {
        const double mc = fmin(fmax(v[c], R.mn[c]), R.mx[c]);
        const double t = (mc - R.mn[c]) / (R.mx[c] - R.mn[c]) * R.levels[c] + 0.5;
        code[c] = (uint32_t)fmin(fmax(floor(t), 0.0), R.levels[c]);
      }
      uint32_t* p = reinterpret_cast<uint32_t*>(dst) + off;
      for (int k = 0; k < 5; ++k) p[k * g.cstride] = code[2 * k] | (code[2 * k + 1] << 16);
    }
  }
}

// copy edge columns of every interior row into the z ghost columns (periodic images)
// planes [g.xb, g.xr) only: disjoint x-ranges of one step may run on concurrent streams
__global__ void fill_ghosts(Geo g, int NC, uint32_t* buf) {
  const int64_t n = (int64_t)(g.xr - g.xb) * NC * 2 * g.ny;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pc = i / (2 * g.ny);
    const int k = (int)(i - pc * 2 * g.ny);
    const int xr = (int)(pc / NC), c = (int)(pc - (int64_t)xr * NC), x = g.xb + xr;
    uint32_t* row = buf + (int64_t)(x + 1) * g.pstride + (int64_t)c * g.cstride + (int64_t)((k >> 1) + 1) * g.zp;
    if (k & 1) row[g.nz + kZOff] = row[kZOff];            // z = nz  <- image of z = 0
    else row[kZOff - 1] = row[g.nz - 1 + kZOff];         // z = -1  <- image of z = nz-1
  }
}

// ghost rows (after the columns are filled, so corners are consistent)
__global__ void fill_ghost_rows(Geo g, int NC, uint32_t* buf) {
  const int rowsz = g.zp;   // whole padded rows (the z ghost columns included)
  const int64_t n = (int64_t)(g.xr - g.xb) * NC * 2 * rowsz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pc = i / (2 * rowsz);
    const int k = (int)(i - pc * 2 * rowsz);
    const int xr = (int)(pc / NC), c = (int)(pc - (int64_t)xr * NC), x = g.xb + xr;
    uint32_t* base = buf + (int64_t)(x + 1) * g.pstride + (int64_t)c * g.cstride;
    const int zz = k >> 1;
    if (k & 1) base[(int64_t)(g.ny + 1) * g.zp + zz] = base[(int64_t)1 * g.zp + zz];
    else base[zz] = base[(int64_t)g.ny * g.zp + zz];
  }
}

// interior words of the state (q16 words or fp32 components) <-> dense (NC, nx, ny, nz)
__global__ void pack_codes(Geo g, int NC, const uint32_t* __restrict__ buf, uint32_t* __restrict__ dense, int dir) {
  const int64_t nc = (int64_t)g.nx * g.ny * g.nz, n = NC * nc;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / nc);
    const int64_t cell = i - (int64_t)k * nc;
    const int x = (int)(cell / ((int64_t)g.ny * g.nz));
    const int64_t r = cell - (int64_t)x * g.ny * g.nz;
    const int y = (int)(r / g.nz), z = (int)(r - (int64_t)y * g.nz);
    const int64_t off = cell_off(g, x + 1, y, z) + (int64_t)k * g.cstride;
    if (dir == 0) dense[i] = buf[off];
    else const_cast<uint32_t*>(buf)[off] = dense[i];
  }
}

template __global__ void import_f64<false>(Geo, Ranges, void*, const double*, const double*, const double*, int, int, unsigned long long*, unsigned int*);
template __global__ void import_f64<true>(Geo, Ranges, void*, const double*, const double*, const double*, int, int, unsigned long long*, unsigned int*);

}  // namespace hlbm

// ------------------------------------------------------------------ host-side launchers
namespace hlbm {

static unsigned grid_for(int64_t n, int tpb) {
  int64_t b = (n + tpb - 1) / tpb;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_import(const Geo& g, const Ranges& R, bool q16, void* dst, const double* rho,
                          const double* mom, const double* stress, int x0, int cnt,
                          unsigned long long* sat, unsigned int* nonpos, cudaStream_t st) {
  const int64_t n = (int64_t)g.ny * g.nz * cnt;
  if (q16) import_f64<true><<<grid_for(n, 256), 256, 0, st>>>(g, R, dst, rho, mom, stress, x0, cnt, sat, nonpos);
  else import_f64<false><<<grid_for(n, 256), 256, 0, st>>>(g, R, dst, rho, mom, stress, x0, cnt, sat, nonpos);
  return cudaGetLastError();
}

cudaError_t launch_export(const Geo& g, const Ranges& R, bool q16, const void* src, double* rho,
                          double* mom, double* stress, int x0, int cx, int y0, int cy, int z0, int cz,
                          cudaStream_t st) {
  const int64_t n = (int64_t)cx * cy * cz;
  if (q16) export_f64<true><<<grid_for(n, 256), 256, 0, st>>>(g, R, src, rho, mom, stress, x0, cx, y0, cy, z0, cz);
  else export_f64<false><<<grid_for(n, 256), 256, 0, st>>>(g, R, src, rho, mom, stress, x0, cx, y0, cy, z0, cz);
  return cudaGetLastError();
}

cudaError_t launch_fill_ghosts(const Geo& g, int NC, void* buf, cudaStream_t st) {
  if (g.xr <= g.xb) return cudaSuccess;
  const int64_t n1 = (int64_t)(g.xr - g.xb) * NC * 2 * g.ny;
  fill_ghosts<<<grid_for(n1, 256), 256, 0, st>>>(g, NC, reinterpret_cast<uint32_t*>(buf));
  const int64_t n2 = (int64_t)(g.xr - g.xb) * NC * 2 * g.zp;
  fill_ghost_rows<<<grid_for(n2, 256), 256, 0, st>>>(g, NC, reinterpret_cast<uint32_t*>(buf));
  return cudaGetLastError();
}

cudaError_t launch_pack_codes(const Geo& g, int NC, void* buf, uint32_t* dense, int dir, cudaStream_t st) {
  const int64_t n = (int64_t)NC * g.nx * g.ny * g.nz;
  pack_codes<<<grid_for(n, 256), 256, 0, st>>>(g, NC, reinterpret_cast<uint32_t*>(buf), dense, dir);
  return cudaGetLastError();
}

cudaError_t launch_init_modes(const Geo& g, bool q16, const Ranges& R, void* dst, double rho0,
                              const double* modes, int nmodes, cudaStream_t st) {
  const int64_t n = (int64_t)g.nx * g.ny * g.nz;
  if (q16) init_modes<true><<<grid_for(n, 256), 256, 0, st>>>(g, R, dst, rho0, modes, nmodes);
  else init_modes<false><<<grid_for(n, 256), 256, 0, st>>>(g, R, dst, rho0, modes, nmodes);
  return cudaGetLastError();
}

cudaError_t launch_classify(const uint8_t* mask_ext, const MaskGeo& m, uint32_t* links, uint8_t* cls,
                            cudaStream_t st) {
  const int64_t n = (int64_t)m.nx * m.ny * m.nz;
  classify_cells<<<grid_for(n, 256), 256, 0, st>>>(mask_ext, m, links, cls);
  return cudaGetLastError();
}

int64_t compact_tiles(int64_t n) { return (n + kCompactTile - 1) / kCompactTile; }

// counts must hold compact_tiles(n) entries, total one entry (device)
cudaError_t launch_compact(const uint8_t* cls, const uint32_t* links, int64_t n, uint8_t want,
                           int64_t* counts, int64_t* total, int64_t* out_cells, uint32_t* out_masks,
                           bool count_only, cudaStream_t st) {
  const int64_t nt = compact_tiles(n);
  if (nt == 0) return cudaMemsetAsync(total, 0, sizeof(int64_t), st);
  if (count_only) {
    compact_count<<<(unsigned)nt, kCompactTPB, 0, st>>>(cls, n, want, counts);
    compact_scan<<<1, 1024, 0, st>>>(counts, nt, total);
  } else {
    compact_scatter<<<(unsigned)nt, kCompactTPB, 0, st>>>(cls, links, n, want, counts, out_cells, out_masks);
  }
  return cudaGetLastError();
}

cudaError_t launch_special_bits(const uint8_t* cls, int nx, int ny, int nz, int row_words,
                                uint32_t* bits, cudaStream_t st) {
  const int64_t n = (int64_t)nx * ny * row_words;
  special_bits_kernel<<<grid_for(n, 256), 256, 0, st>>>(cls, nx, ny, nz, row_words, bits);
  return cudaGetLastError();
}


// divergence locator (runs only after a step reported divergence): the node of largest |u|^2 in the
// current state, non-finite moments ranking above every finite value; key = u2 bits << 32 | ~index
// (ties: the smallest linear index)
template <bool Q16>
__global__ void locate_kernel(const __grid_constant__ StepArgs A, unsigned long long* __restrict__ out) {
  const Geo& g = A.g;
  const int64_t n = (int64_t)g.nx * g.ny * g.nz;
  unsigned long long best = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i / ((int64_t)g.ny * g.nz));
    const int64_t r = i - (int64_t)x * g.ny * g.nz;
    const int y = (int)(r / g.nz), z = (int)(r - (int64_t)y * g.nz);
    float s[10];
    load_cell<Q16>(A, x + 1, y, z, s);
    bool fin = true;
#pragma unroll
    for (int c = 0; c < 10; ++c) fin = fin && isfinite(s[c]);
    const float rho = 1.0f + s[0];
    const float u2 = (s[1] * s[1] + s[2] * s[2] + s[3] * s[3]) / (rho * rho);
    const uint32_t bits = (fin && isfinite(u2)) ? __float_as_uint(fmaxf(u2, 0.f)) : 0xFFFFFFFFu;
    const unsigned long long key = ((unsigned long long)bits << 32) | (0xFFFFFFFFull - (unsigned long long)(uint32_t)i);
    best = key > best ? key : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
    best = v > best ? v : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

cudaError_t launch_locate(const StepArgs& A, bool q16, unsigned long long* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, 8, st);
  if (e != cudaSuccess) return e;
  if (q16) locate_kernel<true><<<148 * 8, 256, 0, st>>>(A, out);
  else locate_kernel<false><<<148 * 8, 256, 0, st>>>(A, out);
  return cudaGetLastError();
}
}  // namespace hlbm
