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

#include "hlbm_launch.h"

namespace hlbm {

// D3Q27 order of lattice.py:99-116
__device__ constexpr int kCX[27] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1};
__device__ constexpr int kCY[27] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, -1, 1, -1, 1};
__device__ constexpr int kCZ[27] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, -1, 1};

__device__ __forceinline__ int src_plane(const Geo& g, int x) {   // storage plane of source x
  if (x < 0) return g.x_lo_src;
  if (x >= g.nx) return g.x_hi_src;
  return x + 1;
}

template <bool Q16>
__device__ __forceinline__ void load_cell(const StepArgs& A, int sp, int y, int z, float s[10]) {
  const Geo& g = A.g;
  if (sp < 0) {
#pragma unroll
    for (int c = 0; c < 10; ++c) s[c] = A.inflow[c];
    return;
  }
  const int64_t off = cell_off(g, sp, y, z);   // y, z may be -1 / n: ghost images
  if (!Q16) {
    const float* p = reinterpret_cast<const float*>(A.in) + off;
#pragma unroll
    for (int c = 0; c < 10; ++c) s[c] = __ldg(p + c * g.cstride);
  } else {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(A.in) + off;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t wv = __ldg(p + k * g.cstride);
      s[2 * k] = __fmaf_rn(code_lo_f(wv) - 8388608.0f, A.Q.dec_step[2 * k], A.Q.dec_off[2 * k]);
      s[2 * k + 1] = __fmaf_rn(code_hi_f(wv) - 8388608.0f, A.Q.dec_step[2 * k + 1], A.Q.dec_off[2 * k + 1]);
    }
  }
}

// per-cell context of the mesh mode (Eq. 8): post-collision state of x
struct MeshCtx {
  float rho, d, nxx, nxy, nxz, nyy, nyz, nzz;   // neq part of rho S+ at x: X - j+ j+ / rho
  const float* t;                               // this cell's 27 hit parameters
  float F[3], T[3];                              // momentum exchange accumulators
};

__device__ __forceinline__ void add_moments(float m[10], int cx, int cy, int cz, float ft) {
  m[0] += ft;
  if (cx) m[1] += cx * ft;
  if (cy) m[2] += cy * ft;
  if (cz) m[3] += cz * ft;
  if (cx) m[4] += ft;
  if (cx && cy) m[5] += cx * cy * ft;
  if (cx && cz) m[6] += cx * cz * ft;
  if (cy) m[7] += ft;
  if (cy && cz) m[8] += cy * cz * ft;
  if (cz) m[9] += ft;
}

// one link of the pull update; accumulates the raw moments of ft into m
//   MODE 0: masked links take the half-way bounce-back population f+_opp(i)(x)
//   MODE 2: masked links take the Eq.-8 boundary population at p = x - t c_i
template <int I, bool Q16, bool FORCE, int MODE, int Q>
__device__ __forceinline__ void pull_link(const StepArgs& A, int x, int y, int z, uint32_t mask,
                                          float m[10], MeshCtx& mc) {
  constexpr int cx = kCX[I], cy = kCY[I], cz = kCZ[I];
  const Geo& g = A.g;
  const bool cut = (mask >> I) & 1u;
  const bool bb = MODE == 0 && cut;
  const int sx = bb ? x : x - cx;
  const int sy = bb ? y : y - cy;   // ghost rows/columns hold the periodic images
  const int sz = bb ? z : z - cz;
  float s[10];
  load_cell<Q16>(A, src_plane(g, sx), sy, sz, s);
  const Coef<float> C = coeffs<float, FORCE>(s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], s[8], s[9], A.R);
  float E, O;
  eval_eo<cx, cy, cz, float, Q>(C, E, O);
  float ft = bb ? (E - O) : (E + O);
  if (MODE == 2 && cut) {
    // Eq. 8: rho_p = rho_x, u_p = v + w x (p - c), rho S_p = rho u_p u_p + (rho S_x - rho u_x u_x)
    const float t = mc.t[I];
    const float px = (float)x - t * cx, py = (float)y - t * cy, pz = (float)z - t * cz;
    const float rx = px - A.solid_c[0], ry = py - A.solid_c[1], rz = pz - A.solid_c[2];
    const float ux = A.solid_v[0] + A.solid_w[1] * rz - A.solid_w[2] * ry;
    const float uy = A.solid_v[1] + A.solid_w[2] * rx - A.solid_w[0] * rz;
    const float uz = A.solid_v[2] + A.solid_w[0] * ry - A.solid_w[1] * rx;
    const float r = mc.rho;
    const Coef<float> Cp = hermite<float>(mc.d, r * ux, r * uy, r * uz, ux, uy, uz, r * ux * ux + mc.nxx,
                                          r * ux * uy + mc.nxy, r * ux * uz + mc.nxz, r * uy * uy + mc.nyy,
                                          r * uy * uz + mc.nyz, r * uz * uz + mc.nzz);
    float Ep, Op;
    eval_eo<cx, cy, cz, float, Q>(Cp, Ep, Op);
    const float fp = Ep + Op;
    // momentum exchange: Delta P = -(f_p - f_streamed) c_i on the solid
    const float df = fp - ft;
    const float dPx = -df * cx, dPy = -df * cy, dPz = -df * cz;
    mc.F[0] += dPx; mc.F[1] += dPy; mc.F[2] += dPz;
    mc.T[0] += ry * dPz - rz * dPy;
    mc.T[1] += rz * dPx - rx * dPz;
    mc.T[2] += rx * dPy - ry * dPx;
    ft = fp;
  }
  add_moments(m, cx, cy, cz, ft);
}

template <int I, bool Q16, bool FORCE, int MODE, int Q>
struct PullAll {
  __device__ __forceinline__ static void run(const StepArgs& A, int x, int y, int z, uint32_t mask,
                                             float m[10], MeshCtx& mc) {
    pull_link<I, Q16, FORCE, MODE, Q>(A, x, y, z, mask, m, mc);
    PullAll<I + 1, Q16, FORCE, MODE, Q>::run(A, x, y, z, mask, m, mc);
  }
};
template <bool Q16, bool FORCE, int MODE, int Q>
struct PullAll<Q, Q16, FORCE, MODE, Q> {
  __device__ __forceinline__ static void run(const StepArgs&, int, int, int, uint32_t, float*, MeshCtx&) {}
};

template <typename E>
__device__ __forceinline__ void put_cell(const Geo& g, E* plane, int y, int z, const E* v, int ncomp) {
  // the cell and, at y/z edges, its periodic images in the ghost layers (both y ghost rows
  // when ny == 1, both z ghost columns when nz == 1)
  const int ys[3] = {y, y == 0 ? g.ny : INT_MIN, y == g.ny - 1 ? -1 : INT_MIN};
  const int zs[3] = {z, z == 0 ? g.nz : INT_MIN, z == g.nz - 1 ? -1 : INT_MIN};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      if (ys[a] == INT_MIN || zs[b] == INT_MIN) continue;
      E* p = plane + (int64_t)(ys[a] + 1) * g.zp + (zs[b] + kZOff);
      for (int c = 0; c < ncomp; ++c) p[c * g.cstride] = v[c];
    }
}

template <bool Q16, bool DITHER>
__device__ __forceinline__ void store_cell(const StepArgs& A, int x, int y, int z, const float s[10],
                                           bool stat, float red[5]) {
  const Geo& g = A.g;
  const int64_t plane_off = (int64_t)(x + 1) * g.pstride;
  if (!Q16) {
    put_cell(g, reinterpret_cast<float*>(A.out) + plane_off, y, z, s, 10);
  } else {
    float nz[10];
    if (DITHER) {
      const uint32_t gi = (uint32_t)(((int64_t)(g.gx0 + x) * g.gny + y) * g.gnz + z);
      const uint32_t h0 = mix32(gi + A.step_key);
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const uint32_t h = dither_word(h0, k);
        nz[2 * k] = noise16(h & 0xFFFFu);
        nz[2 * k + 1] = noise16(h >> 16);
      }
    }
    uint32_t code[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) {
      float t = __fmaf_rn(s[c], A.Q.enc_scale[c], A.Q.enc_off[c]);
      if (DITHER) t += nz[c];
      code[c] = min(f2u16_floor(t), A.Q.levels[c]);
      const float r = __fmaf_rn(s[c], A.Q.sat_a[c], A.Q.sat_b[c]);
      if (stat && !(fabsf(r) <= 1.0f)) atomicAdd(&A.stats->sat[c], 1ull);
    }
    uint32_t wd[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) wd[k] = __byte_perm(code[2 * k], code[2 * k + 1], 0x5410);
    put_cell(g, reinterpret_cast<uint32_t*>(A.out) + plane_off, y, z, wd, 5);
  }
  if (stat) {
    red[0] += s[0]; red[1] += s[1]; red[2] += s[2]; red[3] += s[3];
    const float inv = rcp_nr(1.0f + s[0]);
    const float u2 = (s[1] * s[1] + s[2] * s[2] + s[3] * s[3]) * inv * inv;
    red[4] = (u2 > red[4] || u2 != u2) ? u2 : red[4];
  }
}

__device__ __forceinline__ void flush_stats(const StepArgs& A, float red[5]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) red[k] += __shfl_xor_sync(0xffffffffu, red[k], o);
  float m = red[4];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float t = __shfl_xor_sync(0xffffffffu, m, o);
    m = (t > m || t != t) ? t : m;
  }
  if (lane == 0) {
    atomicAdd(&A.stats->mass_dev, (double)red[0]);
    atomicAdd(&A.stats->mom[0], (double)red[1]);
    atomicAdd(&A.stats->mom[1], (double)red[2]);
    atomicAdd(&A.stats->mom[2], (double)red[3]);
    atomicMax(&A.stats->max_u2_bits, __float_as_uint(m));
  }
}

// MODE 0: pull update of listed (or all) cells with voxel bounce-back on masked links;
// MODE 1: reset listed solid cells to rest; MODE 2: mesh links (Eq. 8) + momentum exchange;
// MODE 3: the fused single-kernel step (Alg. 1, original HOME-LBM): every cell of the
//         slab, one thread each, 27-link pull with the solid links resolved inline from a dense
//         per-cell mask (bit 0: the cell is solid -> rest; bits 1..26: cut links -> bounce-back)
// Q: the velocity set, 27 or 19 (D3Q19 runs on this per-cell path only).  Without a cell list
// the thread index is the local linear cell index offset by `base` (an x-range of the slab).
template <bool Q16, bool FORCE, bool DITHER, int MODE, int Q>
__global__ void __launch_bounds__(128) pull_cells(const __grid_constant__ StepArgs A,
                                                  const int64_t* __restrict__ cells,
                                                  const uint32_t* __restrict__ masks, int64_t n, int64_t base) {
  const Geo& g = A.g;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float red[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  MeshCtx mc;
  mc.F[0] = mc.F[1] = mc.F[2] = mc.T[0] = mc.T[1] = mc.T[2] = 0.f;
  if (idx < n) {
    const int64_t cell = cells ? cells[idx] : base + idx;
    const int64_t yz = (int64_t)g.ny * g.nz;
    const int x = (int)(cell / yz);
    const int64_t r = cell - (int64_t)x * yz;
    const int y = (int)(r / g.nz), z = (int)(r - (int64_t)y * g.nz);
    float s[10];
    const uint32_t fmask = (MODE == 3 && masks) ? masks[cell] : 0u;
    if (MODE == 1 || (MODE == 3 && (fmask & 1u))) {
#pragma unroll
      for (int c = 0; c < 10; ++c) s[c] = 0.f;
    } else {
      const uint32_t mask = MODE == 3 ? fmask : (masks ? masks[idx] : 0u);
      if (MODE == 2) {
        float o[10];
        load_cell<Q16>(A, x + 1, y, z, o);
        const Post<float> P = collide<float, FORCE>(o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], o[8], o[9], A.R);
        const float rho = 1.0f + P.d;
        mc.rho = rho;
        mc.d = P.d;
        // rho (S_x - u_x u_x) of the post-collision state
        mc.nxx = P.Xxx - P.jpx * P.ux; mc.nxy = P.Xxy - P.jpx * P.uy; mc.nxz = P.Xxz - P.jpx * P.uz;
        mc.nyy = P.Xyy - P.jpy * P.uy; mc.nyz = P.Xyz - P.jpy * P.uz; mc.nzz = P.Xzz - P.jpz * P.uz;
        mc.t = A.cut_t + idx * 27;
      }
      float m[10];
#pragma unroll
      for (int c = 0; c < 10; ++c) m[c] = 0.f;
      PullAll<0, Q16, FORCE, MODE == 3 ? 0 : MODE, Q>::run(A, x, y, z, mask, m, mc);
      raw_to_state<float>(m, s);
    }
    store_cell<Q16, DITHER>(A, x, y, z, s, A.do_stats && MODE != 1 && !(MODE == 3 && (fmask & 1u)), red);
  }
  if (A.do_stats && MODE != 1) flush_stats(A, red);
  if (MODE == 2 && A.do_stats) {
    float v[6] = {mc.F[0], mc.F[1], mc.F[2], mc.T[0], mc.T[1], mc.T[2]};
#pragma unroll
    for (int k = 0; k < 6; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if ((threadIdx.x & 31) == 0) {
      for (int k = 0; k < 3; ++k) {
        atomicAdd(&A.stats->force[k], (double)v[k]);
        atomicAdd(&A.stats->torque[k], (double)v[3 + k]);
      }
    }
  }
}

// ------------------------------------------------------------------ original HOME-LBM step
// PAPER.md Alg. 1 (lines 312-334, the in-repo baseline of the split scheme's attribution,
// PAPER.md:418-429): the stored state is the POST-collision moments (Alg. 1's storage cut);
// one thread per lattice node of an 8 x 8 x 8 tile (the paper's tile size).
//   1. every node of the tile and its one-cell halo (10^3 nodes, ~2 per thread) loads its moments
//      and reconstructs its own 27 populations f^t (moments.py:64-90) into shared memory
//      (108 KB, direction-major so consecutive threads hit consecutive banks);
//   2. per interior node and direction i: the link test against the dense per-node mask (bit i:
//      x - c_i is solid); no intersection -> stream f_i(x) <- f^t_i(x - c_i) from shared memory;
//      intersection -> the boundary population, for voxel solids the half-way bounce-back
//      f^t_opp(i)(x) of the node itself (lattice.py:198-201);
//   3. extract the temporary moments (moments.py:25-39), collide them (collision.py:137-194)
//      and write the post-collision moments back; solid nodes stay at rest.
// (S o C)^n o S = S o (C o S)^n: n steps of this kernel from m0, then one streaming S, equal
// n split steps (Alg. 2 cut) from S(m0) (tests/test_gpu_alg1.py).
constexpr int kA1 = 8;                      // tile edge (interior nodes)
constexpr int kA1H = kA1 + 2;               // with the halo
constexpr int kA1N = kA1H * kA1H * kA1H;    // nodes reconstructed per tile

template <int I, int Q>
struct ReconAll {   // ft_i of every direction i < Q of one node -> shared memory (stride kA1N)
  __device__ __forceinline__ static void run(const Coef<float>& C, float* f) {
    float E, O;
    eval_eo<kCX[I], kCY[I], kCZ[I], float, Q>(C, E, O);
    f[I * kA1N] = E + O;
    ReconAll<I + 1, Q>::run(C, f);
  }
};
template <int Q>
struct ReconAll<Q, Q> {
  __device__ __forceinline__ static void run(const Coef<float>&, float*) {}
};

template <int I, int Q>
struct GatherAll {  // stream (or bounce back) every direction into the raw moments of node (lx,ly,lz)
  __device__ __forceinline__ static void run(const float* f, int own, uint32_t mask, float m[10]) {
    constexpr int cx = kCX[I], cy = kCY[I], cz = kCZ[I];
    constexpr int opp = I == 0 ? 0 : ((I & 1) ? I + 1 : I - 1);
    const bool cut = (mask >> I) & 1u;
    const float ft = cut ? f[opp * kA1N + own] : f[I * kA1N + own - (cx * kA1H + cy) * kA1H - cz];
    add_moments(m, cx, cy, cz, ft);
    GatherAll<I + 1, Q>::run(f, own, mask, m);
  }
};
template <int Q>
struct GatherAll<Q, Q> {
  __device__ __forceinline__ static void run(const float*, int, uint32_t, float*) {}
};

template <bool Q16, bool FORCE, bool DITHER, int Q, bool COLLIDE>
__global__ void __launch_bounds__(kA1 * kA1 * kA1, 2) alg1_step(const __grid_constant__ StepArgs A,
                                                                const uint32_t* __restrict__ fmask) {
  extern __shared__ float fsm[];   // [Q][kA1N]
  const Geo& g = A.g;
  const int tz = (g.nz + kA1 - 1) / kA1, ty = (g.ny + kA1 - 1) / kA1;
  int b = blockIdx.x;
  const int bz = b % tz;
  b /= tz;
  const int by = b % ty, bx = b / ty;
  const int x0 = bx * kA1, y0 = by * kA1, z0 = bz * kA1;
  // 1. reconstruct f^t of the haloed tile (post-collision moments -> populations, no collision)
  for (int i = threadIdx.x; i < kA1N; i += blockDim.x) {
    const int hz = i % kA1H, hy = (i / kA1H) % kA1H, hx = i / (kA1H * kA1H);
    const int x = x0 - 1 + hx, y = y0 - 1 + hy, z = z0 - 1 + hz;
    if (x > g.nx || y > g.ny || z > g.nz) continue;   // beyond the halo of a ragged tile: unused
    float s[10];
    load_cell<Q16>(A, src_plane(g, x), y, z, s);      // ghost rows / columns: periodic images
    const float inv = rcp_nr(1.0f + s[0]);
    const float ux = s[1] * inv, uy = s[2] * inv, uz = s[3] * inv;
    // rho S = sneq + j j / rho (moments.py:93-102), the full stress of the stored state
    const Coef<float> C = hermite<float>(s[0], s[1], s[2], s[3], ux, uy, uz, __fmaf_rn(s[1], ux, s[4]),
                                         __fmaf_rn(s[1], uy, s[5]), __fmaf_rn(s[1], uz, s[6]),
                                         __fmaf_rn(s[2], uy, s[7]), __fmaf_rn(s[2], uz, s[8]),
                                         __fmaf_rn(s[3], uz, s[9]));
    ReconAll<0, Q>::run(C, fsm + i);
  }
  __syncthreads();
  // 2./3. one interior node per thread
  const int lz = threadIdx.x % kA1, ly = (threadIdx.x / kA1) % kA1, lx = threadIdx.x / (kA1 * kA1);
  const int x = x0 + lx, y = y0 + ly, z = z0 + lz;
  float red[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  if (x < g.nx && y < g.ny && z < g.nz) {
    const int64_t cell = ((int64_t)x * g.ny + y) * g.nz + z;
    const uint32_t mask = fmask ? fmask[cell] : 0u;
    float s[10];
    if (mask & 1u) {
#pragma unroll
      for (int c = 0; c < 10; ++c) s[c] = 0.f;
    } else {
      float m[10];
#pragma unroll
      for (int c = 0; c < 10; ++c) m[c] = 0.f;
      const int own = ((lx + 1) * kA1H + (ly + 1)) * kA1H + (lz + 1);
      GatherAll<0, Q>::run(fsm, own, mask, m);
      float pre[10];
      raw_to_state<float>(m, pre);
      if (!COLLIDE) {   // the streaming operator S alone (hlbm_stream)
#pragma unroll
        for (int c = 0; c < 10; ++c) s[c] = pre[c];
      } else {
      const Post<float> P = collide<float, FORCE>(pre[0], pre[1], pre[2], pre[3], pre[4], pre[5], pre[6], pre[7],
                                                  pre[8], pre[9], A.R);
      s[0] = P.d; s[1] = P.jpx; s[2] = P.jpy; s[3] = P.jpz;
      s[4] = P.Xxx - P.jpx * P.ux; s[5] = P.Xxy - P.jpx * P.uy; s[6] = P.Xxz - P.jpx * P.uz;
      s[7] = P.Xyy - P.jpy * P.uy; s[8] = P.Xyz - P.jpy * P.uz; s[9] = P.Xzz - P.jpz * P.uz;
      }
    }
    store_cell<Q16, DITHER>(A, x, y, z, s, A.do_stats && !(mask & 1u), red);
  }
  if (A.do_stats) flush_stats(A, red);
}

template <bool Q16, bool FORCE, bool DITHER, int Q, bool COLLIDE>
static cudaError_t launch_alg1_t(const StepArgs& A, const uint32_t* fmask, cudaStream_t st) {
  const Geo& g = A.g;
  const int64_t tiles = (int64_t)((g.nx + kA1 - 1) / kA1) * ((g.ny + kA1 - 1) / kA1) * ((g.nz + kA1 - 1) / kA1);
  const int smem = Q * kA1N * (int)sizeof(float);
  static bool attr = false;   // once per instantiation (not on every launch)
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(alg1_step<Q16, FORCE, DITHER, Q, COLLIDE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  alg1_step<Q16, FORCE, DITHER, Q, COLLIDE><<<(unsigned)tiles, kA1 * kA1 * kA1, smem, st>>>(A, fmask);
  return cudaGetLastError();
}

cudaError_t launch_alg1(const StepArgs& A, const uint32_t* fmask, bool q16, bool force, bool dither, int q,
                        cudaStream_t st, bool collide) {
  if (!collide) {   // S alone: no force term
    if (q16) return dither ? (q == 19 ? launch_alg1_t<true, false, true, 19, false>(A, fmask, st)
                                      : launch_alg1_t<true, false, true, 27, false>(A, fmask, st))
                           : (q == 19 ? launch_alg1_t<true, false, false, 19, false>(A, fmask, st)
                                      : launch_alg1_t<true, false, false, 27, false>(A, fmask, st));
    return q == 19 ? launch_alg1_t<false, false, false, 19, false>(A, fmask, st)
                   : launch_alg1_t<false, false, false, 27, false>(A, fmask, st);
  }
#define HLBM_A1(QQ, F, D)                                                          \
  if (q16 == QQ && force == F && dither == D)                                     \
    return q == 19 ? launch_alg1_t<QQ, F, D, 19, true>(A, fmask, st) : launch_alg1_t<QQ, F, D, 27, true>(A, fmask, st);
  HLBM_A1(false, false, false)
  HLBM_A1(false, true, false)
  HLBM_A1(true, false, false)
  HLBM_A1(true, true, false)
  HLBM_A1(true, false, true)
  HLBM_A1(true, true, true)
#undef HLBM_A1
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ compacted lists, three warps per 32 cells
// The voxel boundary-cell list of the split scheme (MODE 0: half-way bounce-back) runs in
// blocks of 3 warps over 32 consecutive list entries: warp w takes the links with c_x = w - 1 (9 of
// the 27), lane l the l-th cell, so each link's loads stay coalesced across the lanes (consecutive
// boundary cells are mostly consecutive in z) while three times as many independent link chains are
// in flight as with one thread walking all 27 links.  The three partial raw-moment sums meet in
// shared memory and are added in a fixed order (deterministic); warp 0 finishes the cell.
template <int I, int CXW, bool Q16, bool FORCE, int MODE, int Q>
struct PullGroup {
  __device__ __forceinline__ static void run(const StepArgs& A, int x, int y, int z, uint32_t mask, float m[10],
                                             MeshCtx& mc) {
    if constexpr (kCX[I] == CXW) pull_link<I, Q16, FORCE, MODE, Q>(A, x, y, z, mask, m, mc);
    PullGroup<I + 1, CXW, Q16, FORCE, MODE, Q>::run(A, x, y, z, mask, m, mc);
  }
};
template <int CXW, bool Q16, bool FORCE, int MODE, int Q>
struct PullGroup<Q, CXW, Q16, FORCE, MODE, Q> {
  __device__ __forceinline__ static void run(const StepArgs&, int, int, int, uint32_t, float*, MeshCtx&) {}
};

template <bool Q16, bool FORCE, bool DITHER, int MODE, int Q>
__global__ void __launch_bounds__(96) pull_list3(const __grid_constant__ StepArgs A,
                                                 const int64_t* __restrict__ cells,
                                                 const uint32_t* __restrict__ masks, int64_t n) {
  __shared__ float part[2][10][32];   // the c_x = 0 and +1 warps' partial sums
  const Geo& g = A.g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float red[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  MeshCtx mc;   // unused by MODE 0
  for (int64_t base = (int64_t)blockIdx.x * 32; base < n; base += (int64_t)gridDim.x * 32) {
    const int64_t idx = base + lane;
    const bool valid = idx < n;
    float m[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) m[c] = 0.f;
    int x = 0, y = 0, z = 0;
    if (valid) {
      const int64_t cell = cells[idx];
      const int64_t yz = (int64_t)g.ny * g.nz;
      x = (int)(cell / yz);
      const int64_t r = cell - (int64_t)x * yz;
      y = (int)(r / g.nz);
      z = (int)(r - (int64_t)y * g.nz);
      const uint32_t mask = masks[idx];
      if (w == 0) PullGroup<0, -1, Q16, FORCE, MODE, Q>::run(A, x, y, z, mask, m, mc);
      else if (w == 1) PullGroup<0, 0, Q16, FORCE, MODE, Q>::run(A, x, y, z, mask, m, mc);
      else PullGroup<0, 1, Q16, FORCE, MODE, Q>::run(A, x, y, z, mask, m, mc);
    }
    if (w > 0) {
#pragma unroll
      for (int c = 0; c < 10; ++c) part[w - 1][c][lane] = m[c];
    }
    __syncthreads();
    if (w == 0 && valid) {
#pragma unroll
      for (int c = 0; c < 10; ++c) m[c] = (m[c] + part[0][c][lane]) + part[1][c][lane];
      float st[10];
      raw_to_state<float>(m, st);
      store_cell<Q16, DITHER>(A, x, y, z, st, A.do_stats != 0, red);
    }
    __syncthreads();
  }
  if (A.do_stats && w == 0) flush_stats(A, red);
}

cudaError_t launch_pull_cells(const StepArgs& A, const int64_t* cells, const uint32_t* masks,
                              int64_t n, int mode, bool q16, bool force, bool dither,
                              cudaStream_t st, int q, int64_t base) {
  if (n <= 0) return cudaSuccess;
  // voxel boundary lists: 3 warps per 32 cells (the mesh lists keep one thread per cell: their
  // Eq.-8 context -- the cell's own collision -- would be recomputed by each of the three warps;
  // measured 2.86 vs 2.77 ms on the 505k-triangle vehicle)
  if (cells && mode == 0 && base == 0) {
    const int64_t nblk = std::min<int64_t>((n + 31) / 32, (int64_t)148 * 16);
#define HLBM_PL3(QQ, F, D)                                                                                  \
    if (q16 == QQ && force == F && dither == D) {                                                           \
      if (q == 19) pull_list3<QQ, F, D, 0, 19><<<(unsigned)nblk, 96, 0, st>>>(A, cells, masks, n);            \
      else pull_list3<QQ, F, D, 0, 27><<<(unsigned)nblk, 96, 0, st>>>(A, cells, masks, n);                     \
      return cudaGetLastError();                                                                            \
    }
    HLBM_PL3(false, false, false)
    HLBM_PL3(false, true, false)
    HLBM_PL3(true, false, false)
    HLBM_PL3(true, true, false)
    HLBM_PL3(true, false, true)
    HLBM_PL3(true, true, true)
#undef HLBM_PL3
    return cudaErrorInvalidValue;
  }
  const int tpb = 128;
  const int64_t nb = (n + tpb - 1) / tpb;
#define HLBM_PULL(QQ, F, D)                                                                                    \
  if (q16 == QQ && force == F && dither == D) {                                                              \
    if (q == 19) {                                                                                           \
      if (mode == 0) pull_cells<QQ, F, D, 0, 19><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base);      \
      else if (mode == 1) pull_cells<QQ, F, D, 1, 19><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base); \
      else if (mode == 2) pull_cells<QQ, F, D, 2, 19><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base); \
      else pull_cells<QQ, F, D, 3, 19><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base);                  \
    } else if (mode == 0) pull_cells<QQ, F, D, 0, 27><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base); \
    else if (mode == 1) pull_cells<QQ, F, D, 1, 27><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base);   \
    else if (mode == 2) pull_cells<QQ, F, D, 2, 27><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base);   \
    else pull_cells<QQ, F, D, 3, 27><<<(unsigned)nb, tpb, 0, st>>>(A, cells, masks, n, base);                  \
    return cudaGetLastError();                                                                               \
  }
  HLBM_PULL(false, false, false)
  HLBM_PULL(false, true, false)
  HLBM_PULL(true, false, false)
  HLBM_PULL(true, true, false)
  HLBM_PULL(true, false, true)
  HLBM_PULL(true, true, true)
#undef HLBM_PULL
  return cudaErrorInvalidValue;
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

}  // namespace hlbm
