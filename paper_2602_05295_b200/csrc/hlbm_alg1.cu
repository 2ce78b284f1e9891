// The original HOME-LBM kernel (Alg. 1); per-cell helpers in hlbm_cells.cuh.
#include "hlbm_cells.cuh"

namespace hlbm {
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

// triangle mesh (Alg. 1's link-intersection test, with the cut links of the
// static mesh precomputed, hlbm_mesh.cu): a cut link takes the Eq.-8 boundary population at
// p = x - t c_i built from the node's own post-collision moments -- the stored Alg.-1 state -- as
// the split scheme's compacted kernel builds it from the post-collision state of x
// (hlbm_cells.cuh pull_link, MODE 2); links into a wall face bounce back.
template <int I, int Q>
struct GatherMesh {
  __device__ __forceinline__ static void run(const StepArgs& A, const float* f, int own, uint32_t mask,
                                             uint32_t wmask, const float* tk, int x, int y, int z,
                                             const MeshCtx& mc, float m[10]) {
    constexpr int cx = kCX[I], cy = kCY[I], cz = kCZ[I];
    constexpr int opp = I == 0 ? 0 : ((I & 1) ? I + 1 : I - 1);
    const bool wc = (wmask >> I) & 1u;
    const bool cut = ((mask >> I) & 1u) && !wc;
    float ft = wc ? f[opp * kA1N + own] : f[I * kA1N + own - (cx * kA1H + cy) * kA1H - cz];
    if (cut) {
      const float t = tk[I];
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
      ft = Ep + Op;
    }
    add_moments(m, cx, cy, cz, ft);
    GatherMesh<I + 1, Q>::run(A, f, own, mask, wmask, tk, x, y, z, mc, m);
  }
};
template <int Q>
struct GatherMesh<Q, Q> {
  __device__ __forceinline__ static void run(const StepArgs&, const float*, int, uint32_t, uint32_t, const float*,
                                             int, int, int, const MeshCtx&, float*) {}
};

template <bool Q16, bool FORCE, bool DITHER, int Q, bool COLLIDE, bool MESH>
__global__ void __launch_bounds__(kA1 * kA1 * kA1, 2) alg1_step(const __grid_constant__ StepArgs A,
                                                                const uint32_t* __restrict__ fmask,
                                                                const int32_t* __restrict__ midx,
                                                                const uint32_t* __restrict__ mmasks) {
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
      const int k = MESH ? midx[cell] : -1;
      if (MESH && k >= 0) {
        float o[10];   // the node's own stored (post-collision) moments
        load_cell<Q16>(A, x + 1, y, z, o);
        MeshCtx mc;
        mc.rho = 1.0f + o[0];
        mc.d = o[0];
        mc.nxx = o[4]; mc.nxy = o[5]; mc.nxz = o[6]; mc.nyy = o[7]; mc.nyz = o[8]; mc.nzz = o[9];
        GatherMesh<0, Q>::run(A, fsm, own, mmasks[k], A.wall_masks ? A.wall_masks[k] : 0u, A.cut_t + (int64_t)k * 27,
                              x, y, z, mc, m);
      } else {
        GatherAll<0, Q>::run(fsm, own, mask, m);
      }
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

template <bool Q16, bool FORCE, bool DITHER, int Q, bool COLLIDE, bool MESH>
static cudaError_t launch_alg1_m(const StepArgs& A, const uint32_t* fmask, const int32_t* midx,
                                 const uint32_t* mmasks, cudaStream_t st) {
  const Geo& g = A.g;
  const int64_t tiles = (int64_t)((g.nx + kA1 - 1) / kA1) * ((g.ny + kA1 - 1) / kA1) * ((g.nz + kA1 - 1) / kA1);
  const int smem = Q * kA1N * (int)sizeof(float);
  static bool attr = false;   // once per instantiation (not on every launch)
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(alg1_step<Q16, FORCE, DITHER, Q, COLLIDE, MESH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  alg1_step<Q16, FORCE, DITHER, Q, COLLIDE, MESH><<<(unsigned)tiles, kA1 * kA1 * kA1, smem, st>>>(A, fmask, midx,
                                                                                                   mmasks);
  return cudaGetLastError();
}

// mesh_idx (dense list positions) selects the triangle-mesh variant (D3Q27 only, like set_mesh)
template <bool Q16, bool FORCE, bool DITHER, int Q, bool COLLIDE>
static cudaError_t launch_alg1_t(const StepArgs& A, const uint32_t* fmask, const int32_t* midx,
                                 const uint32_t* mmasks, cudaStream_t st) {
  if constexpr (Q == 27) {
    if (midx) return launch_alg1_m<Q16, FORCE, DITHER, Q, COLLIDE, true>(A, fmask, midx, mmasks, st);
  }
  return launch_alg1_m<Q16, FORCE, DITHER, Q, COLLIDE, false>(A, fmask, nullptr, nullptr, st);
}

__global__ void mesh_index_kernel(const int64_t* __restrict__ cells, int64_t nb, int32_t* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += (int64_t)gridDim.x * blockDim.x)
    out[cells[k]] = (int32_t)k;
}

cudaError_t launch_mesh_index(const int64_t* cells, int64_t nb, int64_t n, int32_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0xFF, (size_t)n * 4, st);   // -1: not listed
  if (e != cudaSuccess || nb <= 0) return e;
  mesh_index_kernel<<<(unsigned)std::min<int64_t>((nb + 255) / 256, 148 * 8), 256, 0, st>>>(cells, nb, out);
  return cudaGetLastError();
}

cudaError_t launch_alg1(const StepArgs& A, const uint32_t* fmask, bool q16, bool force, bool dither, int q,
                        cudaStream_t st, bool collide, const int32_t* midx, const uint32_t* mm) {
  if (!collide) {   // S alone: no force term
    if (q16) return dither ? (q == 19 ? launch_alg1_t<true, false, true, 19, false>(A, fmask, midx, mm, st)
                                      : launch_alg1_t<true, false, true, 27, false>(A, fmask, midx, mm, st))
                           : (q == 19 ? launch_alg1_t<true, false, false, 19, false>(A, fmask, midx, mm, st)
                                      : launch_alg1_t<true, false, false, 27, false>(A, fmask, midx, mm, st));
    return q == 19 ? launch_alg1_t<false, false, false, 19, false>(A, fmask, midx, mm, st)
                   : launch_alg1_t<false, false, false, 27, false>(A, fmask, midx, mm, st);
  }
#define HLBM_A1(QQ, F, D)                                                          \
  if (q16 == QQ && force == F && dither == D)                                     \
    return q == 19 ? launch_alg1_t<QQ, F, D, 19, true>(A, fmask, midx, mm, st) : launch_alg1_t<QQ, F, D, 27, true>(A, fmask, midx, mm, st);
  HLBM_A1(false, false, false)
  HLBM_A1(false, true, false)
  HLBM_A1(true, false, false)
  HLBM_A1(true, true, false)
  HLBM_A1(true, false, true)
  HLBM_A1(true, true, true)
#undef HLBM_A1
  return cudaErrorInvalidValue;
}

}  // namespace hlbm
