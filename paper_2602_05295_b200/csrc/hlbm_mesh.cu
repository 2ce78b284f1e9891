// Triangle-mesh solid coupling, preprocessing (static geometry; Alg. 3 and the surface
// voxelisation of PAPER.md:396-397).
//
// The paper tests links against triangles every step in a triangle-parallel kernel and adds the
// corrections with atomicAdd into a full-precision buffer that is then re-quantised.  For a
// static mesh the B200 build does the geometry once:
//   1. mark_candidates: every triangle marks the nodes of its bounding box grown by one cell
//   2. ordered compaction of the marked nodes (hlbm_cells.cu)
//   3. intersect: every (triangle, candidate node, direction) tests the pull link x -> x - c_i
//      in float64 (Moller-Trumbore, eps = 1e-9 inclusive, oracle/mesh.py:segment_triangle);
//      the earliest t wins (atomicMin on the float64 bits), ties go to the lowest triangle
//      (second pass)
//   4. the cells with at least one cut link form the boundary list; per cut link the kernel
//      keeps t (p = x - t c_i)
// Every step the compacted kernel (pull_cells, mode 2) replaces each cut link with the Eq.-8
// boundary population: the fused Alg.-1 semantics, deterministic, no atomics and no second
// (full-precision) state buffer.
//
// All float64 arithmetic uses explicit __dmul_rn/__dadd_rn/__dsub_rn so nvcc cannot contract
// it into FMAs: the results match the NumPy oracle bit for bit.
#include "hlbm_launch.h"

namespace hlbm {

__device__ constexpr int mCX[27] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1};
__device__ constexpr int mCY[27] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, -1, 1, -1, 1};
__device__ constexpr int mCZ[27] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, -1, 1};

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 dsub3(D3 a, D3 b) {
  return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)};
}
// cross(a,b) = (a1 b2 - a2 b1, a2 b0 - a0 b2, a0 b1 - a1 b0)    (oracle/mesh.py:cross)
__device__ __forceinline__ D3 dcross(D3 a, D3 b) {
  return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
          __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
          __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
// dot(a,b) = (a0 b0 + a1 b1) + a2 b2                               (oracle/mesh.py:dot)
__device__ __forceinline__ double ddot(D3 a, D3 b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}

constexpr double kEps = 1e-9, kDetEps = 1e-12;

// hit parameter t in (eps, 1+eps] of o + t d with the triangle, or -1
__device__ __forceinline__ double seg_tri(D3 o, D3 d, D3 v0, D3 v1, D3 v2) {
  const D3 e1 = dsub3(v1, v0), e2 = dsub3(v2, v0);
  const D3 pvec = dcross(d, e2);
  const double det = ddot(e1, pvec);
  if (!(fabs(det) >= kDetEps)) return -1.0;
  const double inv = __ddiv_rn(1.0, det);
  const D3 tvec = dsub3(o, v0);
  const double u = __dmul_rn(ddot(tvec, pvec), inv);
  const D3 qvec = dcross(tvec, e1);
  const double v = __dmul_rn(ddot(d, qvec), inv);
  const double t = __dmul_rn(ddot(e2, qvec), inv);
  const bool hit = (u >= -kEps) && (u <= __dadd_rn(1.0, kEps)) && (v >= -kEps) &&
                   (__dadd_rn(u, v) <= __dadd_rn(1.0, kEps)) && (t > kEps) && (t <= __dadd_rn(1.0, kEps));
  return hit ? t : -1.0;
}

struct MeshGeo {
  int nx, ny, nz;
  int q;   // velocity set: links 1 .. q-1 are tested (27 or 19)
};

__device__ __forceinline__ bool tri_box(const double* V, const int* F, int k, MeshGeo g, int lo[3], int hi[3]) {
  const int a = F[3 * k], b = F[3 * k + 1], c = F[3 * k + 2];
  const int n[3] = {g.nx, g.ny, g.nz};
  for (int ax = 0; ax < 3; ++ax) {
    const double p0 = V[3 * a + ax], p1 = V[3 * b + ax], p2 = V[3 * c + ax];
    lo[ax] = max((int)floor(fmin(fmin(p0, p1), p2)) - 1, 0);
    hi[ax] = min((int)ceil(fmax(fmax(p0, p1), p2)) + 1, n[ax] - 1);
    if (hi[ax] < lo[ax]) return false;
  }
  return true;
}

__global__ void mark_candidates(const double* __restrict__ V, const int* __restrict__ F, int nf, MeshGeo g,
                                uint8_t* __restrict__ mark) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nf; k += gridDim.x * blockDim.x) {
    int lo[3], hi[3];
    if (!tri_box(V, F, k, g, lo, hi)) continue;
    for (int x = lo[0]; x <= hi[0]; ++x)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int z = lo[2]; z <= hi[2]; ++z) mark[((int64_t)x * g.ny + y) * g.nz + z] = 1;
  }
}

__global__ void index_candidates(const int64_t* __restrict__ cand, int64_t m, int* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    idx[cand[i]] = (int)i;
}

// pass 0: atomicMin of the t bits per (candidate, direction); pass 1: lowest triangle among ties
__global__ void intersect(const double* __restrict__ V, const int* __restrict__ F, int nf, MeshGeo g,
                          const int* __restrict__ idx, unsigned long long* __restrict__ tkey,
                          int* __restrict__ tri, int pass) {
  // one warp per triangle: lanes stride over (node, direction) pairs of the box
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int k = blockIdx.x * wpb + (threadIdx.x >> 5); k < nf; k += gridDim.x * wpb) {
    int lo[3], hi[3];
    if (!tri_box(V, F, k, g, lo, hi)) continue;
    const D3 v0 = {V[3 * F[3 * k]], V[3 * F[3 * k] + 1], V[3 * F[3 * k] + 2]};
    const D3 v1 = {V[3 * F[3 * k + 1]], V[3 * F[3 * k + 1] + 1], V[3 * F[3 * k + 1] + 2]};
    const D3 v2 = {V[3 * F[3 * k + 2]], V[3 * F[3 * k + 2] + 1], V[3 * F[3 * k + 2] + 2]};
    const int ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
    const int nl = g.q - 1;
    const int64_t work = (int64_t)ex * ey * ez * nl;
    for (int64_t w = lane; w < work; w += 32) {
      const int i = 1 + (int)(w % nl);
      const int64_t node = w / nl;
      const int z = lo[2] + (int)(node % ez), y = lo[1] + (int)((node / ez) % ey), x = lo[0] + (int)(node / ((int64_t)ez * ey));
      const D3 o = {(double)x, (double)y, (double)z};
      const D3 d = {(double)-mCX[i], (double)-mCY[i], (double)-mCZ[i]};
      const double t = seg_tri(o, d, v0, v1, v2);
      if (t < 0.0) continue;
      const int c = idx[((int64_t)x * g.ny + y) * g.nz + z];
      const int64_t slot = (int64_t)c * 27 + i;
      const unsigned long long bits = (unsigned long long)__double_as_longlong(t);
      if (pass == 0) atomicMin(&tkey[slot], bits);
      else if (tkey[slot] == bits) atomicMin(&tri[slot], k);
    }
  }
}

// per candidate: link mask, class flag (bit 0 = has a cut link)
__global__ void finalize_candidates(const unsigned long long* __restrict__ tkey, int64_t m,
                                    uint32_t* __restrict__ masks, uint8_t* __restrict__ flag, int q) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
    uint32_t mk = 0;
    for (int i = 1; i < q; ++i)
      if (tkey[c * 27 + i] != ~0ull) mk |= 1u << i;
    masks[c] = mk;
    flag[c] = mk ? 1 : 0;
  }
}

// gather the cut-link table of the selected candidates (list order)
__global__ void gather_links(const int64_t* __restrict__ sel, int64_t nb, const int64_t* __restrict__ cand,
                             const unsigned long long* __restrict__ tkey, const int* __restrict__ tri,
                             int64_t* __restrict__ cells, double* __restrict__ t64, float* __restrict__ t32,
                             int* __restrict__ tri_out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nb * 27; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / 27;
    const int i = (int)(e - b * 27);
    const int64_t c = sel[b];
    if (i == 0) cells[b] = cand[c];
    const unsigned long long k = tkey[c * 27 + i];
    const double t = (k == ~0ull) ? __longlong_as_double(0x7ff8000000000000ll) : __longlong_as_double((long long)k);
    t64[e] = t;
    t32[e] = (float)t;
    tri_out[e] = (k == ~0ull) ? -1 : tri[c * 27 + i];
  }
}

// special-cell bitmask bits for a list of local cells (one u32 word per 32 z cells of a row)
__global__ void bits_from_list(const int64_t* __restrict__ cells, int64_t n, int nz, int row_words,
                               uint32_t* __restrict__ bits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cells[i];
    const int64_t row = c / nz;
    const int z = (int)(c - row * nz);
    atomicOr(&bits[row * row_words + (z >> 5)], 1u << (z & 31));
  }
}

static unsigned grid_of(int64_t n, int tpb) {
  int64_t b = (n + tpb - 1) / tpb;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t build_mesh_links(const double* dV, const int* dF, int nf, int nx, int ny, int nz, MeshLinks& out,
                             cudaStream_t st, int q) {
  const MeshGeo g{nx, ny, nz, q};
  const int64_t n = (int64_t)nx * ny * nz;
  uint8_t* mark = nullptr;
  int* idx = nullptr;
  int64_t *counts = nullptr, *total = nullptr, *cand = nullptr;
  cudaError_t e;
#define MK(call)                       \
  do {                                 \
    if ((e = (call)) != cudaSuccess) { \
      goto done;                       \
    }                                  \
  } while (0)
  {
    MK(cudaMalloc(&mark, n));
    MK(cudaMemsetAsync(mark, 0, n, st));
    mark_candidates<<<grid_of(nf, 128), 128, 0, st>>>(dV, dF, nf, g, mark);
    const int64_t nt = compact_tiles(n);
    MK(cudaMalloc(&counts, (nt + 1) * 8));
    MK(cudaMalloc(&total, 8));
    MK(launch_compact(mark, nullptr, n, 1, counts, total, nullptr, nullptr, true, st));
    int64_t m = 0;
    MK(cudaMemcpyAsync(&m, total, 8, cudaMemcpyDeviceToHost, st));
    MK(cudaStreamSynchronize(st));
    out.nb = 0;
    if (m == 0) goto done;
    MK(cudaMalloc(&cand, m * 8));
    MK(launch_compact(mark, nullptr, n, 1, counts, total, cand, nullptr, false, st));
    MK(cudaMalloc(&idx, n * 4));
    index_candidates<<<grid_of(m, 256), 256, 0, st>>>(cand, m, idx);
    unsigned long long* tkey = nullptr;
    int* tri = nullptr;
    uint32_t* cmask = nullptr;
    uint8_t* flag = nullptr;
    MK(cudaMalloc(&tkey, m * 27 * 8));
    MK(cudaMalloc(&tri, m * 27 * 4));
    MK(cudaMalloc(&cmask, m * 4));
    MK(cudaMalloc(&flag, m));
    MK(cudaMemsetAsync(tkey, 0xFF, m * 27 * 8, st));
    MK(cudaMemsetAsync(tri, 0x7F, m * 27 * 4, st));
    for (int pass = 0; pass < 2; ++pass)
      intersect<<<grid_of((int64_t)nf * 32, 256), 256, 0, st>>>(dV, dF, nf, g, idx, tkey, tri, pass);
    finalize_candidates<<<grid_of(m, 256), 256, 0, st>>>(tkey, m, cmask, flag, q);
    // compact the candidates that carry a cut link (candidate order = cell order)
    const int64_t nt2 = compact_tiles(m);
    int64_t* counts2 = nullptr;
    int64_t* sel = nullptr;
    uint32_t* smask = nullptr;
    MK(cudaMalloc(&counts2, (nt2 + 1) * 8));
    MK(launch_compact(flag, cmask, m, 1, counts2, total, nullptr, nullptr, true, st));
    int64_t nb = 0;
    MK(cudaMemcpyAsync(&nb, total, 8, cudaMemcpyDeviceToHost, st));
    MK(cudaStreamSynchronize(st));
    if (nb > 0) {
      MK(cudaMalloc(&sel, nb * 8));
      MK(cudaMalloc(&smask, nb * 4));
      MK(launch_compact(flag, cmask, m, 1, counts2, total, sel, smask, false, st));
      MK(cudaMalloc(&out.cells, nb * 8));
      MK(cudaMalloc(&out.t64, nb * 27 * 8));
      MK(cudaMalloc(&out.t32, nb * 27 * 4));
      MK(cudaMalloc(&out.tri, nb * 27 * 4));
      gather_links<<<grid_of(nb * 27, 256), 256, 0, st>>>(sel, nb, cand, tkey, tri, out.cells, out.t64, out.t32,
                                                         out.tri);
      out.masks = smask;
      smask = nullptr;
      out.nb = nb;
    }
    MK(cudaStreamSynchronize(st));
    cudaFree(tkey);
    cudaFree(tri);
    cudaFree(cmask);
    cudaFree(flag);
    cudaFree(counts2);
    cudaFree(sel);
    cudaFree(smask);
  }
done:
#undef MK
  cudaFree(mark);
  cudaFree(idx);
  cudaFree(counts);
  cudaFree(total);
  cudaFree(cand);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

cudaError_t launch_bits_from_list(const int64_t* cells, int64_t n, int nz, int row_words, uint32_t* bits,
                                  cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  bits_from_list<<<grid_of(n, 256), 256, 0, st>>>(cells, n, nz, row_words, bits);
  return cudaGetLastError();
}

}  // namespace hlbm
