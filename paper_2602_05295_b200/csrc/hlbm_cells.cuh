// Per-cell device helpers and the compacted-list kernel templates shared by the translation units
// hlbm_cells.cu (setup / IO kernels), hlbm_pull_{f32,q16}.cu (pull_cells, pull_list3) and
// hlbm_alg1.cu (the original HOME-LBM kernel).  Split from one file so the build parallelises.
#pragma once
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
      s[2 * k] = __fmaf_rn(code_lo_f(wv) - A.Q.dec_c[2 * k], A.Q.dec_step[2 * k], A.Q.dec_off[2 * k]);
      s[2 * k + 1] = __fmaf_rn(code_hi_f(wv) - A.Q.dec_c[2 * k + 1], A.Q.dec_step[2 * k + 1], A.Q.dec_off[2 * k + 1]);
    }
  }
}

// per-cell context of the mesh mode (Eq. 8): post-collision state of x
struct MeshCtx {
  float rho, d, nxx, nxy, nxz, nyy, nyz, nzz;   // neq part of rho S+ at x: X - j+ j+ / rho
  const float* t;                               // this cell's 27 hit parameters
  uint32_t wmask;                                // links into a wall face (bounce-back, wins over the mesh)
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
  const bool wcut = MODE == 2 && ((mc.wmask >> I) & 1u);   // wall face: half-way bounce-back
  const bool cut = ((mask >> I) & 1u) && !wcut;
  const bool bb = (MODE == 0 && cut) || wcut;
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
        nz[2 * k] = noise16u(h & 0xFFFFu) + A.Q.enc_nb[2 * k];
        nz[2 * k + 1] = noise16u(h >> 16) + A.Q.enc_nb[2 * k + 1];
      }
    }
    uint32_t code[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) {
      // floor(t) = the floor of the exact value (hlbm_math.cuh Codec::enc_int, noise16u)
      float t = DITHER ? __fadd_rd(__fmaf_rn(s[c], A.Q.enc_scale[c], A.Q.enc_off[c]), nz[c])
                : A.Q.enc_frac[c] == 0.f ? __fmaf_rd(s[c], A.Q.enc_scale[c], A.Q.enc_int[c])
                                         : __fadd_rd(__fmaf_rn(s[c], A.Q.enc_scale[c], A.Q.enc_frac[c]), A.Q.enc_int[c]);
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
        mc.wmask = A.wall_masks ? A.wall_masks[idx] : 0u;
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

// runtime-direction forms of eval_eo / pull_link (MODE 0): the same operations in the same order as
// the templates (a skipped term is an added zero, a sign a negated operand), so bit-identical; one
// link's code serves all 27, so a warp's 9 links fit the instruction cache (the fully unrolled
// per-warp groups spent most of their stall samples on instruction fetch)
template <int Q>
__device__ __forceinline__ void eval_eo_rt(const Coef<float>& C, int cx, int cy, int cz, float& E, float& O) {
  float e = C.K0;
  if (cx) e = e + C.Qxx;
  if (cy) e = e + C.Qyy;
  if (cz) e = e + C.Qzz;
  if (cx && cy) e = (cx * cy > 0) ? e + C.Qxy : e - C.Qxy;
  if (cx && cz) e = (cx * cz > 0) ? e + C.Qxz : e - C.Qxz;
  if (cy && cz) e = (cy * cz > 0) ? e + C.Qyz : e - C.Qyz;
  float o = 0.f;
  bool first = true;
  auto acc = [&](int sgn, float v) {
    if (first) { o = (sgn > 0) ? v : -v; first = false; }
    else o = (sgn > 0) ? o + v : o - v;
  };
  if (cx) acc(cx, C.Lx);
  if (cy) acc(cy, C.Ly);
  if (cz) acc(cz, C.Lz);
  if (cx && cy) { acc(cy, C.Txxy); acc(cx, C.Txyy); }
  if (cx && cz) { acc(cz, C.Txxz); acc(cx, C.Txzz); }
  if (cy && cz) { acc(cy, C.Tyzz); acc(cz, C.Tyyz); }
  if (cx && cy && cz) acc(cx * cy * cz, C.Txyz);
  const int c2 = cx * cx + cy * cy + cz * cz;
  const float om = Q == 19 ? (c2 == 0 ? 72.f : (c2 == 1 ? 12.f : 6.f))
                           : (cx ? 1.f : 4.f) * (cy ? 1.f : 4.f) * (cz ? 1.f : 4.f);
  if (om != 1.f) { e = e * om; o = first ? o : o * om; }
  E = e;
  O = o;
}

template <bool Q16, bool FORCE, int Q>
__device__ __forceinline__ void pull_link_rt(const StepArgs& A, int I, int x, int y, int z, uint32_t mask,
                                             float m[10]) {
  const int cx = kCX[I], cy = kCY[I], cz = kCZ[I];
  const bool bb = (mask >> I) & 1u;   // MODE 0: half-way bounce-back
  float s[10];
  load_cell<Q16>(A, src_plane(A.g, bb ? x : x - cx), bb ? y : y - cy, bb ? z : z - cz, s);
  const Coef<float> C = coeffs<float, FORCE>(s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], s[8], s[9], A.R);
  float E, O;
  eval_eo_rt<Q>(C, cx, cy, cz, E, O);
  add_moments(m, cx, cy, cz, bb ? (E - O) : (E + O));
}

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
#if HLBM_PULL_RT
      if (MODE == 0) {
        (void)mc;
#pragma unroll 1
        for (int I = 0; I < Q; ++I)
          if (kCX[I] == w - 1) pull_link_rt<Q16, FORCE, Q>(A, I, x, y, z, mask, m);
      } else
#endif
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

// launcher of the compacted kernels for one storage type (instantiated in hlbm_pull_f32.cu /
// hlbm_pull_q16.cu)
template <bool QQ>
cudaError_t launch_pull_cells_t(const StepArgs& A, const int64_t* cells, const uint32_t* masks,
                                int64_t n, int mode, bool force, bool dither, cudaStream_t st, int q,
                                int64_t base) {
  if (n <= 0) return cudaSuccess;
  // voxel boundary lists: 3 warps per 32 cells (the mesh lists keep one thread per cell: their
  // Eq.-8 context -- the cell's own collision -- would be recomputed by each of the three warps;
  // measured 2.86 vs 2.77 ms on the 505k-triangle vehicle)
  if (cells && mode == 0 && base == 0) {
    const int64_t nblk = std::min<int64_t>((n + 31) / 32, (int64_t)148 * 16);
#define HLBM_PL3(F, D)                                                                                      \
    if (force == F && dither == D) {                                                                        \
      if (q == 19) pull_list3<QQ, F, D, 0, 19><<<(unsigned)nblk, 96, 0, st>>>(A, cells, masks, n);            \
      else pull_list3<QQ, F, D, 0, 27><<<(unsigned)nblk, 96, 0, st>>>(A, cells, masks, n);                     \
      return cudaGetLastError();                                                                            \
    }
    HLBM_PL3(false, false)
    HLBM_PL3(true, false)
    if (QQ) {
      HLBM_PL3(false, true)
      HLBM_PL3(true, true)
    }
#undef HLBM_PL3
    return cudaErrorInvalidValue;
  }
  const int tpb = 128;
  const int64_t nb = (n + tpb - 1) / tpb;
#define HLBM_PULL(F, D)                                                                                        \
  if (force == F && dither == D) {                                                                           \
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
  HLBM_PULL(false, false)
  HLBM_PULL(true, false)
  if (QQ) {
    HLBM_PULL(false, true)
    HLBM_PULL(true, true)
  }
#undef HLBM_PULL
  return cudaErrorInvalidValue;
}

}  // namespace hlbm
