// fluid_interior: the split scheme's divergence-free fluid update (Alg. 2, lines
// 340-357) over every cell of a slab, sm_100a.
//
// Per cell:  load stored moments -> moment-space collision (collision.py:137-194) ->
// third-order Hermite reconstruction of the 27 post-collision populations (moments.py:64-90)
// -> pull streaming f_i(x) <- f_i(x - c_i) -> moment extraction
// (moments.py:25-39) -> neq split (moments.py:93-96) -> store (fp32 or 16-bit codes).
//
// Mapping:
//   * CTA = 16 warps; warp w holds y row (y0 - 1 + w); rows 1..14 are written, rows 0/15 are
//     halo rows that only produce the populations their neighbour needs.
//   * lane l holds the z pair at storage columns (zs0 + 2l, zs0 + 2l + 1); every arithmetic op
//     is packed f32x2 (FFMA2/FADD2/FMUL2).  Columns zs0+1 .. zs0+60 are written.
//   * the CTA marches along x over a segment; the x-direction of streaming is a register
//     rotation (two 10-moment accumulators), never a memory exchange.
//   * streaming is sum-factorised by axis: z shifts are warp shuffles, y shifts exchange 18
//     f32x2 per lane through shared memory, x shifts are the marching accumulators.
//   * each input plane tile (64 z x 16 y x NC components) is ONE 4-D tensor TMA copy
//     (cp.async.bulk.tensor + mbarrier) into shared memory, STAGES planes ahead; the y/z ghost
//     layers of the layout make every tile in-bounds (no wrap).
#include "hlbm_params.cuh"

namespace hlbm {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HLBM_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      " @!p bra HLBM_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int slot_of(int cx, int cy, int kz) {
  return ((cx + 1) * 2 + (cy > 0 ? 0 : 1)) * 3 + kz;
}

// value of P at the shifted pair: lane's cells take the neighbour at z-1 / z+1
__device__ __forceinline__ V from_zm(V v) {   // value at (z - 1) for both cells
  float up = __shfl_up_sync(0xffffffffu, v.y, 1);
  return make_float2(up, v.x);
}
__device__ __forceinline__ V from_zp(V v) {   // value at (z + 1)
  float dn = __shfl_down_sync(0xffffffffu, v.x, 1);
  return make_float2(v.y, dn);
}

template <int NC, int STAGES>
struct Smem {
  uint32_t stage[STAGES][NC][kNW][kZW];
  V exch[2][kNSlot][kNW][32];   // double-buffered y exchange
  uint64_t bar[STAGES];         // TMA stage full (1 arrival + tx bytes)
  uint64_t full[2][kNW];        // warp w's exchange slots of buffer b written (1 arrival)
  uint64_t empty[2][kNW];       // ... consumed by every y-stage neighbour of w
  uint32_t stage_cnt[STAGES];   // warps done reading a stage; the last one refills it
  float red[kNW][5];
};

// Producer (one thread): the whole plane tile of source plane p is one tensor copy.
template <int NC>
__device__ __forceinline__ void issue_plane(const StepArgs& A, int p, uint32_t (*stage)[kNW][kZW],
                                            uint64_t* bar, int zs0, int ys0) {
  const Geo& g = A.g;
  const int sp = (p < 0) ? g.x_lo_src : (p >= g.nx ? g.x_hi_src : p + 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (sp < 0) {   // inflow ghost plane: constants, nothing to load
    mbar_arrive_expect_tx(bar, 0u);
    return;
  }
  mbar_arrive_expect_tx(bar, (uint32_t)(NC * kNW * kZW * 4));
  tma_load_4d(&stage[0][0][0], &A.tmap_in, zs0, ys0, 0, sp, bar);
}

// Partial moments of one destination plane.  Index order of the 6 "kx=0" moments:
// (ky,kz) = 00, 01, 02, 10, 11, 20.  A plane that has received the cx=+1 contribution
// of source q-1 and the cx=0 contribution of source q carries 9 values (a: kx=0,
// b: kx=1 for (ky,kz) = 00, 01, 10; the kx=2 partial equals b[0]).
struct Part9 {
  V a[6];
  V b[3];
};
struct Part6 {   // only the cx=+1 contribution of source q-1: kx=1/kx=2 partials are copies
  V a[6];
};

// ---------------------------------------------------------------------------------------
// reconstruction of the 9 populations with a given cx, z-stage, hand-off of the cy = +-1
// results to shared memory; returns the cy = 0 results g[kz] (added to the x accumulators
// before the barrier so nothing but the accumulators is live across it).
//
// Centre weights omega(0) = 4 are not multiplied in: the cx = 0 branch runs at 1/4 scale and
// the cy = 0 results at 1/4 scale; the consumers fold the factor into their FMAs.  Scaling by
// a power of two commutes with rounding, so the results are bit-identical to the unscaled
// evaluation.
template <int CX>
__device__ __forceinline__ void recon_cx(const Coef<V>& C, V (*exch)[kNW][32], int w, int lane,
                                         V g0out[3]) {
  V G00, G10, G20, G01, G11, G21, G02, G12;
  if (CX == 0) {   // (x 1/4)
    G00 = C.K0; G10 = C.Ly; G20 = C.Qyy;
    G01 = C.Lz; G11 = C.Qyz; G21 = C.Tyyz;
    G02 = C.Qzz; G12 = C.Tyzz;
  } else if (CX > 0) {
    G00 = vadd(vadd(C.K0, C.Qxx), C.Lx); G10 = vadd(vadd(C.Ly, C.Txxy), C.Qxy);
    G20 = vadd(C.Qyy, C.Txyy);
    G01 = vadd(vadd(C.Lz, C.Txxz), C.Qxz); G11 = vadd(C.Qyz, C.Txyz); G21 = C.Tyyz;
    G02 = vadd(C.Qzz, C.Txzz); G12 = C.Tyzz;
  } else {
    G00 = vsub(vadd(C.K0, C.Qxx), C.Lx); G10 = vsub(vadd(C.Ly, C.Txxy), C.Qxy);
    G20 = vsub(C.Qyy, C.Txyy);
    G01 = vsub(vadd(C.Lz, C.Txxz), C.Qxz); G11 = vsub(C.Qyz, C.Txyz); G21 = C.Tyyz;
    G02 = vsub(C.Qzz, C.Txzz); G12 = C.Tyzz;
  }
#pragma unroll
  for (int cyi = 0; cyi < 3; ++cyi) {
    const int CY = (cyi == 0) ? 1 : (cyi == 1 ? -1 : 0);   // +1, -1, then 0
    V B0, B1, B2;
    if (CY == 0) {   // (x 1/4)
      B0 = G00; B1 = G01; B2 = G02;
    } else if (CY > 0) {
      B0 = vadd(vadd(G00, G20), G10); B1 = vadd(vadd(G01, G21), G11); B2 = vadd(G02, G12);
    } else {
      B0 = vsub(vadd(G00, G20), G10); B1 = vsub(vadd(G01, G21), G11); B2 = vsub(G02, G12);
    }
    // cz level: ft(cz=0) = 4 B0, ft(+-1) = (B0 + B2) +- B1
    const V t = vadd(B0, B2);
    const V fp = vadd(t, B1), fm = vsub(t, B1);
    // z-stage (pull): cz=+1 comes from z-1, cz=-1 from z+1.  Lane pair (z0, z0+1):
    //   P = (fp(z0-1), fp(z0)) = (up, fp.x),  M = (fm(z0+1), fm(z0+2)) = (fm.y, dn)
    // formed with scalar adds so no shifted register pair has to be assembled.
    const float up = __shfl_up_sync(0xffffffffu, fp.y, 1);
    const float dn = __shfl_down_sync(0xffffffffu, fm.x, 1);
    const V T2 = make_float2(__fadd_rn(up, fm.y), __fadd_rn(fp.x, dn));
    const V g1 = make_float2(__fsub_rn(up, fm.y), __fsub_rn(fp.x, dn));
    const V g0 = vfma(B0, vsplat(4.0f), T2), g2 = T2;
    if (CY == 0) {
      g0out[0] = g0; g0out[1] = g1; g0out[2] = g2;
    } else {
      exch[slot_of(CX, CY, 0)][w][lane] = g0;
      exch[slot_of(CX, CY, 1)][w][lane] = g1;
      exch[slot_of(CX, CY, 2)][w][lane] = g2;
    }
  }
}

// y-stage for one cx: neighbour contributions (row y-1 sent cy=+1, row y+1 sent cy=-1)
// as t = A + B (even in cy) and d = A - B (odd in cy), per kz.
template <int CX>
__device__ __forceinline__ void ystage(V (*exch)[kNW][32], int w, int lane, V t[3], V d[2]) {
  const V A0 = exch[slot_of(CX, 1, 0)][w - 1][lane];
  const V A1 = exch[slot_of(CX, 1, 1)][w - 1][lane];
  const V A2 = exch[slot_of(CX, 1, 2)][w - 1][lane];
  const V B0 = exch[slot_of(CX, -1, 0)][w + 1][lane];
  const V B1 = exch[slot_of(CX, -1, 1)][w + 1][lane];
  const V B2 = exch[slot_of(CX, -1, 2)][w + 1][lane];
  t[0] = vadd(A0, B0); t[1] = vadd(A1, B1); t[2] = vadd(A2, B2);
  d[0] = vsub(A0, B0); d[1] = vsub(A1, B1);
}

// ---------------------------------------------------------------------------------------
// codec constants: QMODE 2 = the default QuantSpec ranges as immediates
struct DefQ {
  __host__ __device__ static constexpr double mn(int c) { return c == 0 ? 0.8 : (c < 4 ? -0.6 : -0.1); }
  __host__ __device__ static constexpr double mx(int c) { return c == 0 ? 1.5 : (c < 4 ? 0.6 : 0.1); }
  __host__ __device__ static constexpr float dec_step(int c) { return (float)((mx(c) - mn(c)) / 65535.0); }
  __host__ __device__ static constexpr float dec_off(int c) { return (float)(mn(c) - (c == 0 ? 1.0 : 0.0)); }
  __host__ __device__ static constexpr float enc_scale(int c) { return (float)(65535.0 / (mx(c) - mn(c))); }
  __host__ __device__ static constexpr float enc_off(int c) {
    return (float)(((c == 0 ? 1.0 : 0.0) - mn(c)) * (65535.0 / (mx(c) - mn(c))) + 0.5);
  }
};
template <int QMODE> __device__ __forceinline__ float q_dec_step(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::dec_step(c) : Q.dec_step[c];
}
template <int QMODE> __device__ __forceinline__ float q_dec_off(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::dec_off(c) : Q.dec_off[c];
}
template <int QMODE> __device__ __forceinline__ float q_enc_scale(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::enc_scale(c) : Q.enc_scale[c];
}
template <int QMODE> __device__ __forceinline__ float q_enc_off(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::enc_off(c) : Q.enc_off[c];
}

template <bool Q16, int QMODE>
__device__ __forceinline__ void load_state(const uint32_t (*st)[kNW][kZW], int w, int lane,
                                           bool inflow, const StepArgs& A, V s[10]) {
  if (inflow) {
#pragma unroll
    for (int c = 0; c < 10; ++c) s[c] = vsplat(A.inflow[c]);
    return;
  }
  if (!Q16) {
#pragma unroll
    for (int c = 0; c < 10; ++c) s[c] = *reinterpret_cast<const V*>(&st[c][w][2 * lane]);
  } else {
    const V two23 = vsplat(8388608.0f);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint2 wv = *reinterpret_cast<const uint2*>(&st[k][w][2 * lane]);
      const V lo = make_float2(code_lo_f(wv.x), code_lo_f(wv.y));
      const V hi = make_float2(code_hi_f(wv.x), code_hi_f(wv.y));
      s[2 * k] = vfma(vsub(lo, two23), vsplat(q_dec_step<QMODE>(A.Q, 2 * k)),
                      vsplat(q_dec_off<QMODE>(A.Q, 2 * k)));
      s[2 * k + 1] = vfma(vsub(hi, two23), vsplat(q_dec_step<QMODE>(A.Q, 2 * k + 1)),
                          vsplat(q_dec_off<QMODE>(A.Q, 2 * k + 1)));
    }
  }
}

// image writes of an edge cell into the y/z ghost layers (periodic images; harmless for walls)
template <typename E>
__device__ __forceinline__ void write_images(const Geo& g, E* base_plane, int y, int z, const E* vals,
                                             int ncomp) {
  const int ys[2] = {y, y == 0 ? g.ny : (y == g.ny - 1 ? -1 : y)};
  const int zs[2] = {z, z == 0 ? g.nz : (z == g.nz - 1 ? -1 : z)};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      if (a == 0 && b == 0) continue;
      if ((a && ys[1] == y) || (b && zs[1] == z)) continue;
      E* p = base_plane + (int64_t)(ys[a] + 1) * g.zp + (zs[b] + 1);
      for (int c = 0; c < ncomp; ++c) p[c * g.cstride] = vals[c];
    }
}

// store of one finished cell pair + fused statistics.  zs = storage column of the .x cell
// (even -> 8-byte aligned pair); logical z of .x is zs - 1.
template <bool Q16, bool DITHER, int QMODE>
__device__ __forceinline__ void store_pair(const StepArgs& A, const V m[10], int q, int y, int zs,
                                           bool wx, bool wy, bool statx, bool staty, float red[5]) {
  const Geo& g = A.g;
  V s[10];
  raw_to_state(m, s);
  const int64_t plane_off = (int64_t)(q + 1) * g.pstride;
  const int64_t off = plane_off + (int64_t)(y + 1) * g.zp + zs;
  const int zx = zs - 1, zy = zs;
  const bool edge = (y == 0) || (y == g.ny - 1) || (wx && (zx == 0 || zx == g.nz - 1)) ||
                    (wy && (zy == 0 || zy == g.nz - 1));
  constexpr bool B16 = QMODE >= 1;
  if (!Q16) {
    float* out = reinterpret_cast<float*>(A.out) + off;
    if (wx && wy) {
#pragma unroll
      for (int c = 0; c < 10; ++c) *reinterpret_cast<V*>(out + c * g.cstride) = s[c];
    } else {
#pragma unroll
      for (int c = 0; c < 10; ++c) {
        if (wx) out[c * g.cstride] = s[c].x;
        if (wy) out[c * g.cstride + 1] = s[c].y;
      }
    }
    if (edge) {
      float vx[10], vy[10];
#pragma unroll
      for (int c = 0; c < 10; ++c) { vx[c] = s[c].x; vy[c] = s[c].y; }
      float* bp = reinterpret_cast<float*>(A.out) + plane_off;
      if (wx && (y == 0 || y == g.ny - 1 || zx == 0 || zx == g.nz - 1)) write_images(g, bp, y, zx, vx, 10);
      if (wy && (y == 0 || y == g.ny - 1 || zy == 0 || zy == g.nz - 1)) write_images(g, bp, y, zy, vy, 10);
    }
  } else {
    float mx0 = 0.f, mx1 = 0.f;
    V nz[10];
    if (DITHER) {
      const uint32_t gi = (uint32_t)(((int64_t)(g.gx0 + q) * g.gny + y) * g.gnz + zx);
      const uint32_t h0a = mix32(gi + A.step_key), h0b = mix32(gi + 1u + A.step_key);
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const uint32_t kk = (uint32_t)(k + 1) * 0x9E3779B9u;
        const uint32_t ha = mix32(h0a ^ kk), hb = mix32(h0b ^ kk);
        nz[2 * k] = make_float2(noise16(ha & 0xFFFFu), noise16(hb & 0xFFFFu));
        nz[2 * k + 1] = make_float2(noise16(ha >> 16), noise16(hb >> 16));
      }
    }
    V t[10];
    float lo0 = 1e30f, hi0 = -1e30f, lo1 = 1e30f, hi1 = -1e30f;
#pragma unroll
    for (int c = 0; c < 10; ++c) {
      t[c] = vfma(s[c], vsplat(q_enc_scale<QMODE>(A.Q, c)), vsplat(q_enc_off<QMODE>(A.Q, c)));
      if (B16) {   // every component maps [min, max] onto [0.5, 65535.5]
        lo0 = fminf(lo0, t[c].x); hi0 = fmaxf(hi0, t[c].x);
        lo1 = fminf(lo1, t[c].y); hi1 = fmaxf(hi1, t[c].y);
      } else {
        const V r = vfma(s[c], vsplat(A.Q.sat_a[c]), vsplat(A.Q.sat_b[c]));
        mx0 = fmaxf(mx0, fabsf(r.x));
        mx1 = fmaxf(mx1, fabsf(r.y));
      }
      if (DITHER) t[c] = vadd(t[c], nz[c]);
    }
    if (B16) {
      mx0 = (lo0 < 0.5f || hi0 > 65535.5f || hi0 != hi0) ? 2.0f : 0.0f;
      mx1 = (lo1 < 0.5f || hi1 > 65535.5f || hi1 != hi1) ? 2.0f : 0.0f;
    }
    uint32_t wd[5][2];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (B16) {   // 16-bit slots: the saturating cvt is the clamp
        wd[k][0] = pack2_u16_floor(t[2 * k].x, t[2 * k + 1].x);
        wd[k][1] = pack2_u16_floor(t[2 * k].y, t[2 * k + 1].y);
      } else {
        const uint32_t a0 = min(f2u16_floor(t[2 * k].x), A.Q.levels[2 * k]);
        const uint32_t b0 = min(f2u16_floor(t[2 * k + 1].x), A.Q.levels[2 * k + 1]);
        const uint32_t a1 = min(f2u16_floor(t[2 * k].y), A.Q.levels[2 * k]);
        const uint32_t b1 = min(f2u16_floor(t[2 * k + 1].y), A.Q.levels[2 * k + 1]);
        wd[k][0] = __byte_perm(a0, b0, 0x5410);
        wd[k][1] = __byte_perm(a1, b1, 0x5410);
      }
    }
    uint32_t* out = reinterpret_cast<uint32_t*>(A.out) + off;
    if (wx && wy) {
#pragma unroll
      for (int k = 0; k < 5; ++k) *reinterpret_cast<uint2*>(out + k * g.cstride) = make_uint2(wd[k][0], wd[k][1]);
    } else {
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        if (wx) out[k * g.cstride] = wd[k][0];
        if (wy) out[k * g.cstride + 1] = wd[k][1];
      }
    }
    if (edge) {
      uint32_t vx[5], vy[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) { vx[k] = wd[k][0]; vy[k] = wd[k][1]; }
      uint32_t* bp = reinterpret_cast<uint32_t*>(A.out) + plane_off;
      if (wx && (y == 0 || y == g.ny - 1 || zx == 0 || zx == g.nz - 1)) write_images(g, bp, y, zx, vx, 5);
      if (wy && (y == 0 || y == g.ny - 1 || zy == 0 || zy == g.nz - 1)) write_images(g, bp, y, zy, vy, 5);
    }
    // saturation: |r| > 1  <=>  m outside [min, max]  (rare slow path)
    const bool satx = statx && !(mx0 <= 1.0f), saty = staty && !(mx1 <= 1.0f);
    if (satx || saty) {
#pragma unroll
      for (int c = 0; c < 10; ++c) {
        const V r = vfma(s[c], vsplat(A.Q.sat_a[c]), vsplat(A.Q.sat_b[c]));
        const unsigned n = (satx && !(fabsf(r.x) <= 1.0f)) + (saty && !(fabsf(r.y) <= 1.0f));
        if (n) atomicAdd(&A.stats->sat[c], (unsigned long long)n);
      }
    }
  }
  if (statx) {
    red[0] += s[0].x; red[1] += s[1].x; red[2] += s[2].x; red[3] += s[3].x;
    const float inv = rcp_nr(1.0f + s[0].x);
    const float u2 = (s[1].x * s[1].x + s[2].x * s[2].x + s[3].x * s[3].x) * inv * inv;
    red[4] = (u2 > red[4] || u2 != u2) ? u2 : red[4];
  }
  if (staty) {
    red[0] += s[0].y; red[1] += s[1].y; red[2] += s[2].y; red[3] += s[3].y;
    const float inv = rcp_nr(1.0f + s[0].y);
    const float u2 = (s[1].y * s[1].y + s[2].y * s[2].y + s[3].y * s[3].y) * inv * inv;
    red[4] = (u2 > red[4] || u2 != u2) ? u2 : red[4];
  }
}

template <bool Q16, bool FORCE, bool SPECIAL, bool DITHER, int QMODE, int STAGES>
__global__ void __launch_bounds__(kNW * 32, 1) fluid_interior(const __grid_constant__ StepArgs A) {
  constexpr int NC = Q16 ? 5 : 10;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem<NC, STAGES>& S = *reinterpret_cast<Smem<NC, STAGES>*>(smem_raw);
  const Geo& g = A.g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

  int item = blockIdx.x;
  const int zt = item % g.nzt;
  item /= g.nzt;
  const int yt = item % g.nyt;
  const int xsi = item / g.nyt;
  const int zs0 = zt * kZT;                 // storage column of the window start
  const int zlo = zs0, zhi = min(zs0 + kZT, g.nz);   // interior logical z range of this tile
  const int ys0 = yt * kRows;               // storage row of warp 0
  const int yrow = ys0 + w - 1;             // logical y of this warp's row
  const bool row_interior = (w >= 1) && (w <= kRows) && (yrow < g.ny);
  const int xs = xsi * g.xseg, xe = min(xs + g.xseg, g.nx);
  const int NP = xe - xs + 2;

  const int zst = zs0 + 2 * lane;           // storage column of this lane's .x cell
  const bool wx = row_interior && (zst - 1 >= zlo) && (zst - 1 < zhi);
  const bool wy = row_interior && (zst >= zlo) && (zst < zhi);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.bar[s], 1);
      S.stage_cnt[s] = 0;
    }
    // y-stage consumers are warps 1..kNW-2; warp v's slots are read by v-1 and v+1
    for (int b = 0; b < 2; ++b)
      for (int v = 0; v < kNW; ++v) {
        mbar_init(&S.full[b][v], 1);
        const int nc = (v - 1 >= 1 && v - 1 <= kNW - 2) + (v + 1 >= 1 && v + 1 <= kNW - 2);
        mbar_init(&S.empty[b][v], nc);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&A.tmap_in)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int it = 0; it < STAGES && it < NP; ++it)
      issue_plane<NC>(A, xs - 1 + it, S.stage[it % STAGES], &S.bar[it % STAGES], zs0, ys0);
  }

  float red[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  Part9 Ac, Ad;   // dest p-1 partials (two register sets: the loop is unrolled x2)
  Part6 Bc, Bd;   // dest p partials
#pragma unroll
  for (int k = 0; k < 6; ++k) Ac.a[k] = Bc.a[k] = vsplat(0.f);
#pragma unroll
  for (int k = 0; k < 3; ++k) Ac.b[k] = vsplat(0.f);

  // one source plane: (A9, B6) carried in, (nb, nn) carried out
  auto body = [&](const int it, const Part9& A9, const Part6& B6, Part9& nb, Part6& nn) {
    const int p = xs - 1 + it;
    const int q = p - 1;   // destination plane finished in this iteration
    const bool store_plane = row_interior && q >= xs && q < xe;
    V (*exch)[kNW][32] = S.exch[it & 1];
    uint32_t sbits = 0;
    if (SPECIAL && store_plane && (wx || wy)) {   // lanes past the last z cell read nothing
      const int zq = max(zst - 1, 0);   // word holding the pair (z of .x may be -1 at tile 0)
      const int64_t bi = ((int64_t)q * g.ny + yrow) * A.bits_row_words + (zq >> 5);
      const uint32_t wv = __ldg(A.special_bits + bi);
      if (zst - 1 < 0) sbits = (wv & 1u) << 1;                  // only .y (z = 0) is a cell
      else {
        const uint32_t lo = wv >> (zq & 31);
        uint32_t hi = lo >> 1;
        if ((zq & 31) == 31 && zq + 1 < g.nz) hi = __ldg(A.special_bits + bi + 1);
        sbits = (lo & 1u) | ((hi & 1u) << 1);
      }
    }
    const int sp = (p < 0) ? g.x_lo_src : (p >= g.nx ? g.x_hi_src : p + 1);
    const bool inflow = sp < 0;
    const int st = it % STAGES;
    const int b = it & 1;
    const bool ycons = (w >= 1) && (w <= kNW - 2);   // runs the y-stage (reads both neighbours)
    mbar_wait(&S.bar[st], (uint32_t)((it / STAGES) & 1));
    V fin[10];   // dest q, raw-moment order m000 m100 m010 m001 m200 m110 m101 m020 m011 m002
    {
      V s[10];
      load_state<Q16, QMODE>(S.stage[it % STAGES], w, lane, inflow, A, s);
      const Coef<V> C =
          coeffs<V, FORCE>(s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], s[8], s[9], A.R);
      // the stage has been consumed by this warp (C depends on every loaded value); the last
      // warp to get here refills it with the plane STAGES iterations ahead
      __syncwarp();
      if (lane == 0) {
        const uint32_t old = atomicAdd(&S.stage_cnt[st], 1u);
        if (old == kNW - 1) {
          S.stage_cnt[st] = 0;
          if (it + STAGES < NP)
            issue_plane<NC>(A, xs - 1 + it + STAGES, S.stage[st], &S.bar[st], zs0, ys0);
        }
      }
      // my slots of buffer b were read by my neighbours two planes ago
      mbar_wait(&S.empty[b][w], (uint32_t)(((it >> 1) & 1) ^ 1));
      V gz[3];
      // cx = -1 -> dest q (final contribution)
      const V c4 = vsplat(4.0f), cm4 = vsplat(-4.0f), c16 = vsplat(16.0f);
      recon_cx<-1>(C, exch, w, lane, gz);          // gz at 1/4 scale (cy = 0)
      fin[0] = vfma(gz[0], c4, A9.a[0]);
      fin[3] = vfma(gz[1], c4, A9.a[1]);
      fin[9] = vfma(gz[2], c4, A9.a[2]);
      fin[2] = A9.a[3];
      fin[8] = A9.a[4];
      fin[7] = A9.a[5];
      fin[1] = vfma(gz[0], cm4, A9.b[0]);
      fin[6] = vfma(gz[1], cm4, A9.b[1]);
      fin[5] = A9.b[2];
      fin[4] = vfma(gz[0], c4, A9.b[0]);
      // cx = 0 -> dest p                          (gz at 1/16 scale: cx = 0 and cy = 0)
      recon_cx<0>(C, exch, w, lane, gz);
      nb.b[0] = B6.a[0]; nb.b[1] = B6.a[1]; nb.b[2] = B6.a[3];
      nb.a[0] = vfma(gz[0], c16, B6.a[0]);
      nb.a[1] = vfma(gz[1], c16, B6.a[1]);
      nb.a[2] = vfma(gz[2], c16, B6.a[2]);
      nb.a[3] = B6.a[3]; nb.a[4] = B6.a[4]; nb.a[5] = B6.a[5];
      // cx = +1 -> dest p+1                       (gz at 1/4 scale, folded after the y-stage)
      recon_cx<1>(C, exch, w, lane, gz);
      nn.a[0] = gz[0]; nn.a[1] = gz[1]; nn.a[2] = gz[2];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.full[b][w]);
    if (ycons) {
      mbar_wait(&S.full[b][w - 1], (uint32_t)((it >> 1) & 1));
      mbar_wait(&S.full[b][w + 1], (uint32_t)((it >> 1) & 1));
      V t[3], d[2];
      ystage<-1>(exch, w, lane, t, d);
      fin[0] = vadd(fin[0], t[0]); fin[3] = vadd(fin[3], t[1]); fin[9] = vadd(fin[9], t[2]);
      fin[2] = vadd(fin[2], d[0]); fin[8] = vadd(fin[8], d[1]); fin[7] = vadd(fin[7], t[0]);
      fin[1] = vsub(fin[1], t[0]); fin[6] = vsub(fin[6], t[1]); fin[5] = vsub(fin[5], d[0]);
      fin[4] = vadd(fin[4], t[0]);
      ystage<0>(exch, w, lane, t, d);              // cx = 0 slots are at 1/4 scale
      const V c4 = vsplat(4.0f);
      nb.a[0] = vfma(t[0], c4, nb.a[0]); nb.a[1] = vfma(t[1], c4, nb.a[1]); nb.a[2] = vfma(t[2], c4, nb.a[2]);
      nb.a[3] = vfma(d[0], c4, nb.a[3]); nb.a[4] = vfma(d[1], c4, nb.a[4]); nb.a[5] = vfma(t[0], c4, nb.a[5]);
      ystage<1>(exch, w, lane, t, d);
      nn.a[0] = vfma(nn.a[0], c4, t[0]); nn.a[1] = vfma(nn.a[1], c4, t[1]); nn.a[2] = vfma(nn.a[2], c4, t[2]);
      nn.a[3] = d[0]; nn.a[4] = d[1]; nn.a[5] = t[0];
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.empty[b][w - 1]);
        mbar_arrive(&S.empty[b][w + 1]);
      }
      if (store_plane) {
        const bool sx = A.do_stats && wx && !(SPECIAL && (sbits & 1u));
        const bool sy = A.do_stats && wy && !(SPECIAL && (sbits & 2u));
        store_pair<Q16, DITHER, QMODE>(A, fin, q, yrow, zst, wx, wy, sx, sy, red);
      }
    }
  };

  for (int it = 0; it < NP; it += 2) {
    body(it, Ac, Bc, Ad, Bd);
    if (it + 1 < NP) body(it + 1, Ad, Bd, Ac, Bc);
  }

  if (A.do_stats) {
    // block reduction of the fused statistics
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float v = red[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      red[k] = v;
    }
    float m = red[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float t = __shfl_xor_sync(0xffffffffu, m, o);
      m = (t > m || t != t) ? t : m;
    }
    red[4] = m;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 5; ++k) S.red[w][k] = red[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a[4] = {0, 0, 0, 0};
      float mm = 0.f;
      for (int i = 0; i < kNW; ++i) {
        for (int k = 0; k < 4; ++k) a[k] += (double)S.red[i][k];
        const float t = S.red[i][4];
        mm = (t > mm || t != t) ? t : mm;
      }
      atomicAdd(&A.stats->mass_dev, a[0]);
      atomicAdd(&A.stats->mom[0], a[1]);
      atomicAdd(&A.stats->mom[1], a[2]);
      atomicAdd(&A.stats->mom[2], a[3]);
      atomicMax(&A.stats->max_u2_bits, __float_as_uint(mm));
    }
  }
}

// ------------------------------------------------------------------------ host launcher
template <bool Q16, bool FORCE, bool SPECIAL, bool DITHER, int QMODE>
static cudaError_t launch_t(const StepArgs& A, int nblocks, cudaStream_t st) {
  constexpr int STAGES = Q16 ? 4 : 2;
  constexpr int NC = Q16 ? 5 : 10;
  const size_t smem = sizeof(Smem<NC, STAGES>);
  auto k = fluid_interior<Q16, FORCE, SPECIAL, DITHER, QMODE, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<nblocks, kNW * 32, smem, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_fluid_interior(const StepArgs& A, bool q16, bool force, bool special, bool dither,
                                  int qmode, cudaStream_t st) {
  const int nblocks = A.g.nzt * A.g.nyt * A.g.nxs;
  if (nblocks == 0) return cudaSuccess;
#define HLBM_F(F, S)                                                               \
  if (!q16 && force == F && special == S) return launch_t<false, F, S, false, 0>(A, nblocks, st);
  HLBM_F(false, false) HLBM_F(false, true) HLBM_F(true, false) HLBM_F(true, true)
#undef HLBM_F
#define HLBM_Q(F, S, D, M)                                                                     \
  if (q16 && force == F && special == S && dither == D && qmode == M)                         \
    return launch_t<true, F, S, D, M>(A, nblocks, st);
#define HLBM_QM(M)                                                                            \
  HLBM_Q(false, false, false, M) HLBM_Q(false, true, false, M)                                 \
  HLBM_Q(true, false, false, M) HLBM_Q(true, true, false, M)                                   \
  HLBM_Q(false, false, true, M) HLBM_Q(false, true, true, M)                                   \
  HLBM_Q(true, false, true, M) HLBM_Q(true, true, true, M)
  HLBM_QM(0) HLBM_QM(1) HLBM_QM(2)
#undef HLBM_QM
#undef HLBM_Q
  return cudaErrorInvalidValue;
}

}  // namespace hlbm
