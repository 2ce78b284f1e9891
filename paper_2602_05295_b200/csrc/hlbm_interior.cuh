// fluid_interior: the split scheme's divergence-free fluid update (Alg. 2, lines
// 340-357) over every cell of a slab, sm_100a.
//
// Per cell:  load stored moments -> moment-space collision (collision.py:137-194) ->
// third-order Hermite reconstruction of the 27 post-collision populations (moments.py:64-90)
// -> pull streaming f_i(x) <- f_i(x - c_i) -> moment extraction
// (moments.py:25-39) -> neq split (moments.py:93-96) -> store (fp32 or 16-bit codes).
//
// Mapping:
//   * tile = 15 y rows x 60 z cells, marched along x over a segment.  CTA = 16 warps: warps
//     1..15 own the interior rows y0 .. y0+14; warp 0 is the halo warp: per plane it evaluates
//     only the 9 populations that enter the tile from each of the rows y0-1 (cy = +1) and
//     y0+15 (cy = -1) -- 0.8 of a row's work, so the SMSP holding it is not the slowest one
//     (two halo tasks on row warps would add 0.4 of a row to two SMSPs and gate every warp).
//   * lane l holds the z pair at storage columns (zs0 + 2l, zs0 + 2l + 1); every arithmetic op
//     is packed f32x2 (FFMA2/FADD2/FMUL2).  Lanes 1..30 are written (aligned 8-byte pairs:
//     z = 0 sits at the even storage column kZOff); lanes 0 and 31 are the z halo.
//   * the x-direction of streaming is a register rotation (two 10-moment accumulators),
//     never a memory exchange.
//   * streaming is sum-factorised by axis: z shifts are warp shuffles, y shifts exchange 18
//     f32x2 per lane through shared memory (neighbour-only mbarrier handshakes, no CTA
//     barrier), x shifts are the marching accumulators.
//   * each input plane tile (64 z x 17 y x NC components) is ONE 4-D tensor TMA copy
//     (cp.async.bulk.tensor + mbarrier) into shared memory, STAGES planes ahead; the y/z ghost
//     layers of the layout make every tile in-bounds (no wrap).
//   * LAT = 19 (D3Q19): a second streaming chain with the 1-D weights (2, -1, -1), merged with
//     the D3Q27 chain in the x stage (see xslotB).
//   * collision + Hermite run on inputs pre-scaled by the decode (coeffs_pre, hlbm_math.cuh).
#pragma once
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
#ifdef HLBM_WAIT_HINT_NS   // optional suspend-time hint (ns) for the blocking try_wait
  asm volatile(
      "{\n .reg .pred p;\n"
      "HLBM_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra HLBM_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(HLBM_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n"
      "HLBM_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HLBM_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}


template <int NC, int STAGES, int NB, int NS = kNSlot>
struct Smem {
  uint32_t stage[STAGES][NC][kBoxRows][kZW];
  V exch[NB][NS][kNW][32];      // y exchange (NB buffers); "row" 0 = halo warp (see ystage)
  uint64_t bar[STAGES];         // TMA stage full (1 arrival + tx bytes)
  uint64_t full[NB][kNW];       // warp w's exchange slots of buffer b written (32 lane arrivals)
  uint64_t empty[NB][kNW];      // ... consumed by every y-stage neighbour of w (32 per reader)
  uint64_t cons[STAGES];        // every lane of every warp has read the stage (refill allowed)
  float red[kNW][5];
  float acc[kNW][5][32];        // per-lane statistics accumulators (STATS variants; no registers)
};

// Producer (one thread): the whole plane tile of source plane p is one tensor copy.
template <int NC>
__device__ __forceinline__ void issue_plane(const StepArgs& A, int p, uint32_t (*stage)[kBoxRows][kZW],
                                            uint64_t* bar, int zs0, int ys0) {
  const Geo& g = A.g;
  const int sp = (p < 0) ? g.x_lo_src : (p >= g.nx ? g.x_hi_src : p + 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (sp < 0) {   // inflow ghost plane: constants, nothing to load
    mbar_arrive_expect_tx(bar, 0u);
    return;
  }
  mbar_arrive_expect_tx(bar, (uint32_t)(NC * kBoxRows * kZW * 4));
  tma_load_4d(&stage[0][0][0], &A.tmap_in, zs0, ys0, 0, sp, bar);
}

// Partial moments of one destination plane, index order of the 6 (ay,az) combinations
// 00, 01, 02, 10, 11, 20.  The x march keeps, per destination plane, N = the cx=+1 contribution
// of source q-1 (identical for every ax) and M = N + the cx=0 contribution of source q (ax = 0);
// the ax = 1 / ax = 2 partials of plane q are N's 00, 01, 10 entries.  N of plane q is read for
// the last time in the iteration that creates N of plane q+2, which overwrites it in place, so
// the x2-unrolled loop rotates two M and two N register sets without copying any partial.
struct Part6 {
  V a[6];
};

// ---------------------------------------------------------------------------------------
// Moment-space streaming: sum factorisation by axis on the 17 monomial coefficient fields.
// Along one axis a field F_k (monomial degree k) enters the destination's moment of order a
// through T^{a+k} f = f(x-1) [c=+1] + (-1)^{a+k} f(x+1) [c=-1] + [a+k==0] 4 f(x)  (weights
// w1 = omega/6 with omega(0) = 4, omega(+-1) = 1; the 1/216 is folded into the coefficients).
// With Ap = sum_k F_k and Am = sum_k (-1)^k F_k:  out_a(x) = Ap(x-1) + (-1)^a Am(x+1)
// + [a==0] 4 F_0(x).  z first (warp shuffles, 8 (kx,ky) groups), then y (shared-memory ring,
// 9 (kx,az) groups), then x (register march, 6 (ay,az) groups); the truncation ax+ay+az <= 2
// prunes the outputs after every axis.  105 packed + 32 scalar FP ops per cell pair, against
// 127 + 36 for evaluating the 27 nodal populations first.

// exchange slot of (kx, s, az): s = 0 sent to row y+1 (Yp), s = 1 sent to row y-1 (Ym)
__device__ __forceinline__ constexpr int xslot(int kx, int s, int az) { return (kx * 2 + s) * 3 + az; }

// D3Q19 (LAT = 19): 216 w = prod_axis(4, 1, 1) + prod_axis(2, -1, -1) over (c = 0, +-1) -- rest
// 64 + 8 = 72, axis 16 - 4 = 12, face 4 + 2 = 6, corner 1 - 1 = 0 (lattice.py:119-124) -- so the
// step is the D3Q27 chain A plus a chain B with the 1-D weights (2, -1, -1).  Along an axis,
// chain B's output is 2 F0 [a == 0] minus chain A's neighbour sums, so after the z stage chain B
// equals -chain A for az >= 1 and differs only in its az = 0 fields, zB = 2 F0 - S = 6 F0 - z0.
// The exchange carries chain B's az = 0 y sums in 6 extra slots; the chains merge in the x stage,
// whose neighbour sums take W = Y_A - Y_B and whose centre term takes 4 Y_A + 2 Y_B.
__device__ __forceinline__ constexpr int xslotB(int kx, int s) { return 18 + kx * 2 + s; }
template <int LAT> struct LatSlots { static constexpr int n = LAT == 19 ? 24 : kNSlot; };

// z pull of one (kx,ky) group from its inputs F0 (kz=0), F1 (kz=1), F2 (kz=2); N inputs present
template <int N>
__device__ __forceinline__ void zgroup(V F0, V F1, V F2, V z[3]) {
  V Ap, Am;
  if (N == 3) {
    const V P = vadd(F0, F2);
    Ap = vadd(P, F1);
    Am = vsub(P, F1);
  } else if (N == 2) {
    Ap = vadd(F0, F1);
    Am = vsub(F0, F1);
  } else {
    Ap = F0;
    Am = F0;
  }
  // lane pair (z0, z0+1): Ap(z-1) = (up, Ap.x), Am(z+1) = (Am.y, dn), combined with scalar adds
  // so no shifted register pair has to be assembled
  const float up = __shfl_up_sync(0xffffffffu, Ap.y, 1);
  const float dn = __shfl_down_sync(0xffffffffu, Am.x, 1);
  const V S = make_float2(__fadd_rn(up, Am.y), __fadd_rn(Ap.x, dn));
  z[1] = make_float2(__fsub_rn(up, Am.y), __fsub_rn(Ap.x, dn));
  z[0] = vfma(F0, vsplat(4.0f), S);
  z[2] = S;
}
// chain B (D3Q19) az = 0 value of a group from its chain-A z0 and kz = 0 input
__device__ __forceinline__ V zchainB(V F0, V z0) { return vfma(F0, vsplat(6.0f), vneg(z0)); }

// z-stage of the groups with a given kx: Z[ky][az]; LAT 19 also ZB[ky] (chain B, az = 0)
template <int KX, int LAT = 27>
__device__ __forceinline__ void zstage(const Coef<V>& C, V Z[3][3], V* ZB = nullptr) {
  const V o = vsplat(0.f);
  if (KX == 0) {
    zgroup<3>(C.K0, C.Lz, C.Qzz, Z[0]);
    zgroup<3>(C.Ly, C.Qyz, C.Tyzz, Z[1]);
    zgroup<2>(C.Qyy, C.Tyyz, o, Z[2]);
    if (LAT == 19) { ZB[0] = zchainB(C.K0, Z[0][0]); ZB[1] = zchainB(C.Ly, Z[1][0]); ZB[2] = zchainB(C.Qyy, Z[2][0]); }
  } else if (KX == 1) {
    zgroup<3>(C.Lx, C.Qxz, C.Txzz, Z[0]);
    zgroup<2>(C.Qxy, C.Txyz, o, Z[1]);
    zgroup<1>(C.Txyy, o, o, Z[2]);
    if (LAT == 19) { ZB[0] = zchainB(C.Lx, Z[0][0]); ZB[1] = zchainB(C.Qxy, Z[1][0]); ZB[2] = zchainB(C.Txyy, Z[2][0]); }
  } else {
    zgroup<2>(C.Qxx, C.Txxz, o, Z[0]);
    zgroup<1>(C.Txxy, o, o, Z[1]);
    if (LAT == 19) { ZB[0] = zchainB(C.Qxx, Z[0][0]); ZB[1] = zchainB(C.Txxy, Z[1][0]); }
  }
}
// chain-B y sums of (kx, az = 0)
template <int KX>
__device__ __forceinline__ void ysumsB(const V ZB[3], V& Yp, V& Ym) {
  if (KX < 2) {
    const V P = vadd(ZB[0], ZB[2]);
    Yp = vadd(P, ZB[1]);
    Ym = vsub(P, ZB[1]);
  } else {
    Yp = vadd(ZB[0], ZB[1]);
    Ym = vsub(ZB[0], ZB[1]);
  }
}

// y sums of (kx, az): Yp = sum_ky Z, Ym = sum_ky (-1)^ky Z
template <int KX>
__device__ __forceinline__ void ysums(const V Z[3][3], int az, V& Yp, V& Ym) {
  if (KX < 2) {
    const V P = vadd(Z[0][az], Z[2][az]);
    Yp = vadd(P, Z[1][az]);
    Ym = vsub(P, Z[1][az]);
  } else {
    Yp = vadd(Z[0][az], Z[1][az]);
    Ym = vsub(Z[0][az], Z[1][az]);
  }
}

// own row, one kx: both y sums to the exchange, the ky = 0 centre values returned (LAT 19: and
// chain B's az = 0 centre value in *zcb)
template <int KX, int LAT = 27>
__device__ __forceinline__ void recon_row(const Coef<V>& C, V (*exch)[kNW][32], int w, int lane, V zc[3],
                                          V* zcb = nullptr) {
  V Z[3][3], ZB[3];
  zstage<KX, LAT>(C, Z, ZB);
  if constexpr (LAT == 19) {
    V p, m;
    ysumsB<KX>(ZB, p, m);
    exch[xslotB(KX, 0)][w][lane] = p;
    exch[xslotB(KX, 1)][w][lane] = m;
    *zcb = ZB[0];
  }
#pragma unroll
  for (int az = 0; az < 3; ++az) {
    V p, m;
    ysums<KX>(Z, az, p, m);
    exch[xslot(KX, 0, az)][w][lane] = p;
    exch[xslot(KX, 1, az)][w][lane] = m;
    zc[az] = Z[0][az];
  }
}

// halo row: only the y sum that enters the tile (S = 0: row y0-1 sends Yp up; S = 1: row
// y0+15 sends Ym down), into the exchange slots of "row" 0
template <int S, int LAT = 27>
__device__ __forceinline__ void recon_halo(const Coef<V>& C, V (*exch)[kNW][32], int xrow, int lane) {
#define HLBM_HALO_KX(KX)                                  \
  {                                                       \
    V Z[3][3], ZB[3];                                     \
    zstage<KX, LAT>(C, Z, ZB);                            \
    _Pragma("unroll") for (int az = 0; az < 3; ++az) {    \
      V p, m;                                             \
      ysums<KX>(Z, az, p, m);                             \
      exch[xslot(KX, S, az)][xrow][lane] = S == 0 ? p : m; \
    }                                                     \
    if constexpr (LAT == 19) {                            \
      V p, m;                                             \
      ysumsB<KX>(ZB, p, m);                               \
      exch[xslotB(KX, S)][xrow][lane] = S == 0 ? p : m;   \
    }                                                     \
  }
  HLBM_HALO_KX(0) HLBM_HALO_KX(1) HLBM_HALO_KX(2)
#undef HLBM_HALO_KX
}

// y pull + x stage of one destination row.  The exchange rows form a ring over the warps: row
// warp w (1..15) reads the Yp slots of wu = w-1 and the Ym slots of wd = (w+1) mod 16, so the
// first row reads the halo warp's row-(y0-1) values and the last its row-(y0+15) values.
//   fin (dest q):   Mq (sources q-1, q), Nq (source q-1) + x-pull of Xm (cx = -1)
//   nb  (dest p):   Np (source p-1) + 4 Xc (cx = 0)
//   nn  (dest p+1): Xp (cx = +1), identical for every ax; written over Nq (combo by combo,
//                   each Nq entry is read before its slot is rewritten)
// Raw-moment order of fin: m000 m100 m010 m001 m200 m110 m101 m020 m011 m002; partial index
// order (ay,az) = 00, 01, 02, 10, 11, 20 (b: 00, 01, 10).
template <int LAT = 27>
__device__ __forceinline__ void yx_stage(V (*exch)[kNW][32], int wu, int wd, int lane, const V zc[3][3],
                                         const Part6& Mq, Part6& NqNn, const Part6& Np, V fin[10], Part6& nb,
                                         const V* zcb = nullptr) {
  const V c4 = vsplat(4.0f);
#pragma unroll
  for (int az = 0; az < 3; ++az) {
    V Y[3][3];   // [kx][ay]: chain A (D3Q27), or W = Y_A - Y_B (D3Q19)
    V cen[3];    // D3Q19 centre terms 4 Y_A[0][ay] + 2 Y_B[0][ay]
    bool zero1 = false;   // D3Q19, az = 1: W[kx][1] = 0 (chain B's ay = 1 output equals chain A's)
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      if constexpr (LAT == 19) {
        if (az == 0) {
          const V A = exch[xslot(kx, 0, 0)][wu][lane], B = exch[xslot(kx, 1, 0)][wd][lane];
          const V AB = exch[xslotB(kx, 0)][wu][lane], BB = exch[xslotB(kx, 1)][wd][lane];
          const V SA = vadd(A, B), SB = vadd(AB, BB);
          const V YA0 = vfma(zc[kx][0], c4, SA), YB0 = vfma(zcb[kx], vsplat(2.0f), vneg(SB));
          Y[kx][0] = vsub(YA0, YB0);
          Y[kx][1] = vsub(vadd(A, AB), vadd(B, BB));
          Y[kx][2] = vadd(SA, SB);
          if (kx == 0) {
            cen[0] = vfma(YA0, c4, vadd(YB0, YB0));
            const V d = vsub(A, B), dB = vsub(BB, AB);
            cen[1] = vfma(d, c4, vadd(dB, dB));
            cen[2] = vfma(SA, c4, vmul(SB, -2.0f));
          }
        } else {
          Y[kx][0] = vmul(zc[kx][az], 6.0f);
          zero1 = (az == 1);
          if (kx == 0) {   // only the centre column needs the exchanged values
            const V A = exch[xslot(0, 0, az)][wu][lane], B = exch[xslot(0, 1, az)][wd][lane];
            cen[0] = vmul(vfma(zc[0][az], vsplat(2.0f), vadd(A, B)), 6.0f);
            if (az == 1) cen[1] = vmul(vsub(A, B), 6.0f);
          }
        }
      } else {
        const V A = exch[xslot(kx, 0, az)][wu][lane];
        const V B = exch[xslot(kx, 1, az)][wd][lane];
        const V S = vadd(A, B);
        Y[kx][0] = vfma(zc[kx][az], c4, S);
        if (az <= 1) Y[kx][1] = vsub(A, B);
        if (az == 0) Y[kx][2] = S;
      }
    }
#pragma unroll
    for (int ay = 0; ay + az <= 2; ++ay) {
      const int c = ay == 0 ? az : (ay == 1 ? 3 + az : 5);          // partial index of (ay, az)
      const int m0 = ay == 0 ? (az == 0 ? 0 : (az == 1 ? 3 : 9)) : (ay == 1 ? (az == 0 ? 2 : 8) : 7);
      if (LAT == 19 && zero1 && ay == 1) {   // W = 0: no neighbour contribution along x
        fin[m0] = Mq.a[c];
        nb.a[c] = vadd(cen[1], Np.a[c]);
        NqNn.a[c] = vsplat(0.f);
        continue;
      }
      const V P = vadd(Y[0][ay], Y[2][ay]);
      const V Xp = vadd(P, Y[1][ay]);
      const V Xm = vsub(P, Y[1][ay]);
      fin[m0] = vadd(Mq.a[c], Xm);
      if (ay + az <= 1) {
        const int m1 = ay == 0 ? (az == 0 ? 1 : 6) : 5;
        fin[m1] = vsub(NqNn.a[c], Xm);
      }
      if (ay + az == 0) fin[4] = vadd(NqNn.a[0], Xm);
      if constexpr (LAT == 19) nb.a[c] = vadd(cen[ay], Np.a[c]);
      else nb.a[c] = vfma(Y[0][ay], c4, Np.a[c]);
      NqNn.a[c] = Xp;
    }
  }
}

// ---------------------------------------------------------------------------------------
// codec constants: QMODE 2 = the default QuantSpec ranges as immediates
struct DefQ {
  __host__ __device__ static constexpr double mn(int c) { return c == 0 ? 0.8 : (c < 4 ? -0.6 : -0.1); }
  __host__ __device__ static constexpr double mx(int c) { return c == 0 ? 1.5 : (c < 4 ? 0.6 : 0.1); }
  __host__ __device__ static constexpr double step_d(int c) { return (mx(c) - mn(c)) / 65535.0; }
  __host__ __device__ static constexpr double q0(int c) {   // code of the centre (rho = 1, else 0)
    return (double)(long long)(((c == 0 ? 1.0 : 0.0) - mn(c)) / step_d(c) + 0.5);
  }
  __host__ __device__ static constexpr float dec_step(int c) { return (float)step_d(c); }
  __host__ __device__ static constexpr float dec_off(int c) {   // re-centred (Codec::dec_c)
    return (float)(mn(c) - (c == 0 ? 1.0 : 0.0) + q0(c) * step_d(c));
  }
  __host__ __device__ static constexpr float dec_c(int c) { return (float)(8388608.0 + q0(c)); }
  __host__ __device__ static constexpr float enc_scale(int c) { return (float)(65535.0 / (mx(c) - mn(c))); }
  __host__ __device__ static constexpr double enc_off_d(int c) {
    return ((c == 0 ? 1.0 : 0.0) - mn(c)) * (65535.0 / (mx(c) - mn(c))) + 0.5;
  }
  __host__ __device__ static constexpr float enc_off(int c) { return (float)enc_off_d(c); }
  __host__ __device__ static constexpr float enc_int(int c) { return (float)(double)(long long)enc_off_d(c); }
  __host__ __device__ static constexpr float enc_frac(int c) {
    return (float)(enc_off_d(c) - (double)(long long)enc_off_d(c));
  }
  __host__ __device__ static constexpr float enc_nb(int c) {   // Codec::enc_nb
    return (float)(-1.5 + 1.0 / 131072.0 - ((double)enc_off(c) - enc_off_d(c)));
  }
};
template <int QMODE> __device__ __forceinline__ float q_dec_step(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::dec_step(c) : Q.dec_step[c];
}
template <int QMODE> __device__ __forceinline__ float q_dec_off(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::dec_off(c) : Q.dec_off[c];
}
template <int QMODE> __device__ __forceinline__ float q_dec_c(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::dec_c(c) : Q.dec_c[c];
}
template <int QMODE> __device__ __forceinline__ float q_enc_nb(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::enc_nb(c) : Q.enc_nb[c];
}
template <int QMODE> __device__ __forceinline__ float q_enc_scale(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::enc_scale(c) : Q.enc_scale[c];
}
template <int QMODE> __device__ __forceinline__ float q_enc_off(const Codec& Q, int c) {
  return QMODE == 2 ? DefQ::enc_off(c) : Q.enc_off[c];
}
// t = m * scale + enc_off ready for floor(): round-to-nearest when a dither add (rounding down)
// follows; else rounded down -- in one FMA when enc_off is an integer, else as (m * scale + frac)
// + int (Codec::enc_int).  The same rule as store_cell (hlbm_cells.cuh).
template <bool DITHER, int QMODE>
__device__ __forceinline__ V q_encode_t(const Codec& Q, int c, V m) {
  const V sc = vsplat(q_enc_scale<QMODE>(Q, c));
  if (DITHER) return vfma(m, sc, vsplat(q_enc_off<QMODE>(Q, c)));
  if (QMODE == 2) {
    if (DefQ::enc_frac(c) == 0.f) return vfma_rd(m, sc, vsplat(DefQ::enc_int(c)));
    return vadd_rd(vfma(m, sc, vsplat(DefQ::enc_frac(c))), vsplat(DefQ::enc_int(c)));
  }
  return Q.enc_frac[c] == 0.f ? vfma_rd(m, sc, vsplat(Q.enc_int[c]))
                              : vadd_rd(vfma(m, sc, vsplat(Q.enc_frac[c])), vsplat(Q.enc_int[c]));
}

// PRE: the values come out in the coeffs_pre input scales (hlbm_math.cuh) -- folded into the
// decode FMA for 16-bit codes, one multiply per component for fp32
template <bool Q16, int QMODE, bool PRE>
__device__ __forceinline__ void load_state(const uint32_t (*st)[kBoxRows][kZW], int row, int lane,
                                           bool inflow, const StepArgs& A, V s[10]) {
  if (inflow) {
#pragma unroll
    for (int c = 0; c < 10; ++c) s[c] = vsplat(PRE ? A.inflow_pre[c] : A.inflow[c]);
    return;
  }
  if (!Q16) {
#pragma unroll
    for (int c = 0; c < 10; ++c) {
      s[c] = *reinterpret_cast<const V*>(&st[c][row][2 * lane]);
      if (PRE) s[c] = vmul(s[c], A.pre_k[c]);
    }
  } else if (PRE) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint2 wv = *reinterpret_cast<const uint2*>(&st[k][row][2 * lane]);
      const V lo = make_float2(code_lo_f(wv.x), code_lo_f(wv.y));
      const V hi = make_float2(code_hi_f(wv.x), code_hi_f(wv.y));
      s[2 * k] = vfma(vsub(lo, vsplat(q_dec_c<QMODE>(A.Q, 2 * k))), vsplat(A.pre_step[2 * k]), vsplat(A.pre_off[2 * k]));
      s[2 * k + 1] = vfma(vsub(hi, vsplat(q_dec_c<QMODE>(A.Q, 2 * k + 1))), vsplat(A.pre_step[2 * k + 1]), vsplat(A.pre_off[2 * k + 1]));
    }
  } else {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint2 wv = *reinterpret_cast<const uint2*>(&st[k][row][2 * lane]);
      const V lo = make_float2(code_lo_f(wv.x), code_lo_f(wv.y));
      const V hi = make_float2(code_hi_f(wv.x), code_hi_f(wv.y));
      s[2 * k] = vfma(vsub(lo, vsplat(q_dec_c<QMODE>(A.Q, 2 * k))), vsplat(q_dec_step<QMODE>(A.Q, 2 * k)),
                      vsplat(q_dec_off<QMODE>(A.Q, 2 * k)));
      s[2 * k + 1] = vfma(vsub(hi, vsplat(q_dec_c<QMODE>(A.Q, 2 * k + 1))), vsplat(q_dec_step<QMODE>(A.Q, 2 * k + 1)),
                          vsplat(q_dec_off<QMODE>(A.Q, 2 * k + 1)));
    }
  }
}

// reconstruction coefficients of a loaded cell pair (load_state<.., PRE = !FORCE> scales)
template <bool FORCE, bool Q16>
__device__ __forceinline__ Coef<V> coeffs_int(const V s[10], const Relax& R) {
  if constexpr (FORCE)
    return coeffs<V, true>(s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], s[8], s[9], R);
  else
    return coeffs_pre<V, Q16>(s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], s[8], s[9]);
}

// a finished cell pair (z even, z+1) of row y: `cell` points at component 0 of the pair in its
// plane (8-byte aligned: z + kZOff is even); the uniform component stride is g.cstride elements.
// Edge pairs also go to their periodic images in the y/z ghost layers (plane_base = component 0
// of the plane).  E: element type of the layout (float / uint32_t), W: the 8-byte pair type.
template <typename E, typename W>
__device__ __forceinline__ void put_pair(const Geo& g, E* cell, E* plane_base, int y, int z, const W* vals,
                                         int ncomp) {
  const uint32_t cs = (uint32_t)g.cstride * (uint32_t)sizeof(E);   // < 2^32 bytes per component plane
  char* p = reinterpret_cast<char*>(cell);
#pragma unroll
  for (int c = 0; c < ncomp; ++c) *reinterpret_cast<W*>(p + (size_t)(c * cs)) = vals[c];
  const bool ye = (y == 0) || (y == g.ny - 1), ze = (z == 0) || (z == g.nz - 2);
  if (ye || ze) {
    const int yi = y == 0 ? g.ny : (y == g.ny - 1 ? -1 : y);
    const int zi = z == 0 ? g.nz : (z == g.nz - 2 ? -2 : z);   // image pair start (pad column included)
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        if ((a == 0 && b == 0) || (a && !ye) || (b && !ze)) continue;
        E* q = plane_base + (int64_t)((a ? yi : y) + 1) * g.zp + ((b ? zi : z) + kZOff);
        for (int c = 0; c < ncomp; ++c) *reinterpret_cast<W*>(q + c * g.cstride) = vals[c];
      }
  }
}

// NaN-propagating min / max (PTX min.NaN / max.NaN): a NaN component makes the whole tree NaN,
// so the saturation test below counts it (fminf / fmaxf would drop it), as pull_cells does
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// three-input forms (sm_100 FMNMX3.NAN): the 10-value trees of the saturation test take 5
// instructions each instead of 9
__device__ __forceinline__ float fmin3_nan(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// store of one finished cell pair + fused statistics; z = logical z of the .x cell (even)
template <bool Q16, bool DITHER, bool STATS, int QMODE>
__device__ __forceinline__ void store_pair(const StepArgs& A, const V m[10], int q, int y, int z, int64_t cell_off0, bool statx,
                                           bool staty, float* acc) {
  const Geo& g = A.g;
  V s[10], inv;
  raw_to_state<V, Q16>(m, s, &inv);
  if (STATS) {
    // mass, momentum, max |u|^2 -- accumulated before the encode (shorter live ranges of s and
    // 1/rho; measured 2.08 -> 2.02 ms for the STATS variant at 512^3) (NaN in any cell already makes the mass sum non-finite)
    const V ju = vmul(vfma(s[3], s[3], vfma(s[2], s[2], vmul(s[1], s[1]))), vmul(inv, inv));
    // branch-free: excluded (boundary / solid) cells contribute zeros through selects, so a warp
    // holding special cells does not diverge (the divergent form cost ~15% of the STATS step of
    // a 512x256x256 scene with a mesh)
    const V a = vadd(make_float2(statx ? s[0].x : 0.f, statx ? s[1].x : 0.f),
                     make_float2(staty ? s[0].y : 0.f, staty ? s[1].y : 0.f));
    const V c = vadd(make_float2(statx ? s[2].x : 0.f, statx ? s[3].x : 0.f),
                     make_float2(staty ? s[2].y : 0.f, staty ? s[3].y : 0.f));
    acc[0] += a.x; acc[32] += a.y; acc[64] += c.x; acc[96] += c.y;
    acc[128] = fmaxf(acc[128], fmaxf(statx ? ju.x : 0.f, staty ? ju.y : 0.f));
  }
  const int64_t plane_off = (int64_t)(q + 1) * g.pstride;
  const int64_t cell_off = plane_off + cell_off0;
  constexpr bool B16 = QMODE >= 1;
  if (!Q16) {
    put_pair(g, reinterpret_cast<float*>(A.out) + cell_off, reinterpret_cast<float*>(A.out) + plane_off, y, z, s, 10);
  } else {
    V nz[10];
    if (DITHER) {
      const uint32_t gi = (uint32_t)(((int64_t)(g.gx0 + q) * g.gny + y) * g.gnz + z);
      const uint32_t h0a = mix32(gi + A.step_key), h0b = mix32(gi + 1u + A.step_key);
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const uint32_t ha = dither_word(h0a, k), hb = dither_word(h0b, k);
        nz[2 * k] = vadd(make_float2(noise16u(ha & 0xFFFFu), noise16u(hb & 0xFFFFu)),
                         vsplat(q_enc_nb<QMODE>(A.Q, 2 * k)));
        nz[2 * k + 1] = vadd(make_float2(noise16u(ha >> 16), noise16u(hb >> 16)),
                             vsplat(q_enc_nb<QMODE>(A.Q, 2 * k + 1)));
      }
    }
    V t[10];
#pragma unroll
    for (int c = 0; c < 10; ++c)
      t[c] = q_encode_t<DITHER, QMODE>(A.Q, c, s[c]);
    if (STATS) {
      // saturation counters: m outside [min, max]  (checked before the dither is added)
      bool satx, saty;
      if (B16) {   // every component maps [min, max] onto [0.5, 65535.5]: two min/max trees
        const float lo0 = fmin3_nan(fmin3_nan(t[0].x, t[1].x, t[2].x), fmin3_nan(t[3].x, t[4].x, t[5].x),
                                    fmin3_nan(t[6].x, t[7].x, fmin_nan(t[8].x, t[9].x)));
        const float hi0 = fmax3_nan(fmax3_nan(t[0].x, t[1].x, t[2].x), fmax3_nan(t[3].x, t[4].x, t[5].x),
                                    fmax3_nan(t[6].x, t[7].x, fmax_nan(t[8].x, t[9].x)));
        const float lo1 = fmin3_nan(fmin3_nan(t[0].y, t[1].y, t[2].y), fmin3_nan(t[3].y, t[4].y, t[5].y),
                                    fmin3_nan(t[6].y, t[7].y, fmin_nan(t[8].y, t[9].y)));
        const float hi1 = fmax3_nan(fmax3_nan(t[0].y, t[1].y, t[2].y), fmax3_nan(t[3].y, t[4].y, t[5].y),
                                    fmax3_nan(t[6].y, t[7].y, fmax_nan(t[8].y, t[9].y)));
        satx = statx && !(lo0 >= 0.5f && hi0 <= 65535.5f);   // NaN counts as saturated
        saty = staty && !(lo1 >= 0.5f && hi1 <= 65535.5f);
        if (satx || saty) {   // rare: per-component counts from the same t
#pragma unroll
          for (int c = 0; c < 10; ++c) {
            const unsigned n = (satx && !(t[c].x >= 0.5f && t[c].x <= 65535.5f)) +
                               (saty && !(t[c].y >= 0.5f && t[c].y <= 65535.5f));
            if (n) atomicAdd(&A.stats->sat[c], (unsigned long long)n);
          }
        }
      } else {     // generic bit widths: |r| > 1 with r = (m - mid) / half
        float mx0 = 0.f, mx1 = 0.f;
#pragma unroll
        for (int c = 0; c < 10; ++c) {
          const V r = vfma(s[c], vsplat(A.Q.sat_a[c]), vsplat(A.Q.sat_b[c]));
          mx0 = fmax_nan(mx0, fabsf(r.x));
          mx1 = fmax_nan(mx1, fabsf(r.y));
        }
        satx = statx && !(mx0 <= 1.0f);
        saty = staty && !(mx1 <= 1.0f);
        if (satx || saty) {
#pragma unroll
          for (int c = 0; c < 10; ++c) {
            const V r = vfma(s[c], vsplat(A.Q.sat_a[c]), vsplat(A.Q.sat_b[c]));
            const unsigned n = (satx && !(fabsf(r.x) <= 1.0f)) + (saty && !(fabsf(r.y) <= 1.0f));
            if (n) atomicAdd(&A.stats->sat[c], (unsigned long long)n);
          }
        }
      }
    }
    if (DITHER) {
#pragma unroll
      for (int c = 0; c < 10; ++c) t[c] = vadd_rd(t[c], nz[c]);
    }
    uint2 wd[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (B16) {   // 16-bit slots: the saturating cvt is the clamp
        wd[k].x = pack2_u16_floor(t[2 * k].x, t[2 * k + 1].x);
        wd[k].y = pack2_u16_floor(t[2 * k].y, t[2 * k + 1].y);
      } else {
        const uint32_t a0 = min(f2u16_floor(t[2 * k].x), A.Q.levels[2 * k]);
        const uint32_t b0 = min(f2u16_floor(t[2 * k + 1].x), A.Q.levels[2 * k + 1]);
        const uint32_t a1 = min(f2u16_floor(t[2 * k].y), A.Q.levels[2 * k]);
        const uint32_t b1 = min(f2u16_floor(t[2 * k + 1].y), A.Q.levels[2 * k + 1]);
        wd[k].x = __byte_perm(a0, b0, 0x5410);
        wd[k].y = __byte_perm(a1, b1, 0x5410);
      }
    }
    put_pair(g, reinterpret_cast<uint32_t*>(A.out) + cell_off, reinterpret_cast<uint32_t*>(A.out) + plane_off, y,
             z, wd, 5);
  }
}

template <bool Q16, bool FORCE, bool SPECIAL, bool DITHER, bool STATS, int QMODE, int STAGES, int NB, int LAT = 27>
__global__ void __launch_bounds__(kNW * 32, kCtaPerSm) fluid_interior(const __grid_constant__ StepArgs A) {
  constexpr int NC = Q16 ? 5 : 10;
  using Sm = Smem<NC, STAGES, NB, LatSlots<LAT>::n>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sm& S = *reinterpret_cast<Sm*>(smem_raw);
  const Geo& g = A.g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

  int item = blockIdx.x;
  const int xsi = item / (g.nzt * g.nyt);
  item -= xsi * (g.nzt * g.nyt);
  const int zt = item % g.nzt;
  const int yt = item / g.nzt;
  const int zs0 = zt * kZT;                 // storage column of the window start
  const int y0 = yt * kRows;                // first interior row; the box starts at storage row y0
  const int yrow = y0 + w - 1;              // logical y of this warp's row (row warps 1..15)
  const int zc = zs0 - kZOff + 2 * lane;    // logical z of this lane's .x cell (even)
  const bool row_warp = (w >= 1) && (w <= kRows);
  const bool wr = row_warp && (yrow < g.ny) && (lane >= 1) && (lane <= 30) && (zc < g.nz);
  const int xs = g.xb + xsi * g.xseg, xe = min(xs + g.xseg, g.xr);
  const int NP = xe - xs + 2;
  const bool lo_inflow = g.x_lo_src < 0, hi_inflow = g.x_hi_src < 0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.bar[s], 1);
      mbar_init(&S.cons[s], kNW * 32);
    }
    // readers of exchange row v: cy=+1 slots by v+1 (row warps), cy=-1 slots by v-1 (row warps)
    // or, for the halo row 0, by the last row warp
    for (int b = 0; b < NB; ++b)
      for (int v = 0; v < kNW; ++v) {
        mbar_init(&S.full[b][v], 32);
        const int readers = (v == 0) ? (kHaloWarps == 1 ? 2 : 1)
                            : (v > kRows ? 1 : (v + 1 <= kRows) + (v - 1 >= 1));
        mbar_init(&S.empty[b][v], 32 * readers);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&A.tmap_in)) : "memory");
  }
  // STATS + SPECIAL: the special-cell bits of the CTA's whole tile (planes xs..xe-1, its kRows rows,
  // the 64-cell window of each row as two words: bit 2l / 2l+1 = lane l's cells) are copied to
  // shared memory once, before the march.  A global load per plane instead left its DRAM latency
  // on a scoreboard the plane's loop waited on (+16% on the STATS step of a scene with solids).
  uint32_t (*sbm)[2] = reinterpret_cast<uint32_t (*)[2]>(smem_raw + sizeof(Sm));
  if (STATS && SPECIAL) {
    const int z0 = zs0 - kZOff;                 // logical z of bit 0 of the window
    const int wa = z0 >= 0 ? (z0 >> 5) : -1;    // first bitmask word touched
    const int sh = z0 - 32 * wa;                // 0..31
    for (int i = threadIdx.x; i < (xe - xs) * kRows; i += blockDim.x) {
      const int pl = xs + i / kRows, r = y0 + i % kRows;
      uint32_t lo = 0, hi = 0;
      if (r < g.ny) {
        const uint32_t* row = A.special_bits + ((int64_t)pl * g.ny + r) * A.bits_row_words;
        uint32_t wv[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int idx = wa + k;   // bits beyond nz are zero in the bitmask
          wv[k] = (idx >= 0 && idx < A.bits_row_words) ? __ldg(row + idx) : 0u;
        }
        lo = __funnelshift_r(wv[0], wv[1], sh);
        hi = __funnelshift_r(wv[1], wv[2], sh);
      }
      sbm[i][0] = lo;
      sbm[i][1] = hi;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int it = 0; it < STAGES && it < NP; ++it)
      issue_plane<NC>(A, xs - 1 + it, S.stage[it], &S.bar[it], zs0, y0);
  }

  int st = 0;
  uint32_t sph = 0;
  // this lane is done reading stage st (the halo warp refills it once every lane has arrived)
  auto consumed = [&]() { mbar_arrive(&S.cons[st]); };
  auto plane_inflow = [&](const int p) { return (p < 0 && lo_inflow) || (p >= g.nx && hi_inflow); };

  float* acc = &S.acc[w][0][lane];
  if (STATS) {
#pragma unroll
    for (int k = 0; k < 5; ++k) acc[32 * k] = 0.f;
  }
  if (!row_warp) {
    // ---- halo warp(s): the populations entering the tile from rows y0-1 (Yp slots of exchange
    // row 0) and y0+kRows (Ym slots of row 0, or of row 15 with a second halo warp)
    const bool do_lo = (w == 0), do_hi = (kHaloWarps == 1) || (w == kNW - 1);
    const int xrow = (kHaloWarps == 1) ? 0 : w;   // exchange row written by this warp
    for (int it = 0; it < NP; ++it) {
      const int b = (NB == 2) ? (it & 1) : 0;
      const uint32_t eph = (uint32_t)((NB == 2) ? (it >> 1) : it) & 1u;
      const bool inflow = plane_inflow(xs - 1 + it);
      mbar_wait(&S.bar[st], sph);
      mbar_wait(&S.empty[b][xrow], eph ^ 1u);
      if (do_lo) {
        V s[10];
        load_state<Q16, QMODE, !FORCE>(S.stage[st], 0, lane, inflow, A, s);
        const Coef<V> C = coeffs_int<FORCE, Q16>(s, A.R);
        if (!do_hi) consumed();
        recon_halo<0, LAT>(C, S.exch[b], 0, lane);
      }
      if (do_hi) {
        V s[10];
        load_state<Q16, QMODE, !FORCE>(S.stage[st], kBoxRows - 1, lane, inflow, A, s);
        const Coef<V> C = coeffs_int<FORCE, Q16>(s, A.R);
        consumed();
        recon_halo<1, LAT>(C, S.exch[b], xrow, lane);
      }
      mbar_arrive(&S.full[b][xrow]);
      // producer (warp 0): once every warp has read plane it, its stage takes plane it + STAGES
      if (w == 0 && lane == 0 && it + STAGES < NP) {
        mbar_wait(&S.cons[st], sph);
        issue_plane<NC>(A, xs - 1 + it + STAGES, S.stage[st], &S.bar[st], zs0, y0);
      }
      if (++st == STAGES) { st = 0; sph ^= 1u; }
    }
  } else {
    // ---- row warps
    Part6 Ma, Mb, Na, Nb;   // rotating plane partials (x2 unroll, see Part6)
#pragma unroll
    for (int k = 0; k < 6; ++k) Ma.a[k] = Na.a[k] = Nb.a[k] = vsplat(0.f);
    const int wu = w - 1, wd = (w + 1) % kNW;   // exchange rows read by this warp
    // rows past the first row beyond ny (the last y tile of a grid whose ny is not a multiple of
    // kRows) feed nothing that is stored: such a warp keeps the barrier protocol -- same waits and
    // arrivals, so the ring's phases stay paced -- and skips the arithmetic, leaving its SM
    // sub-partition's issue slots to the active rows (q16 no-stats: 512^3 1.764 -> 1.743 ms,
    // 400^3 0.854 -> 0.840, 256^3 0.285 -> 0.280; the STATS variants came out ~1% slower with the
    // second loop and the HBM-bound fp32 kernel gained nothing, so they keep the single loop)
    const bool active = !HLBM_IDLE_ROWS || STATS || !Q16 || yrow <= g.ny;
    const int64_t cell0 = (int64_t)(yrow + 1) * g.zp + (zc + kZOff);   // pair offset inside a plane

    // one source plane p: Mq, Nq (dest q = p-1), Np (dest p) carried in; nb = M of dest p and
    // N of dest p+1 (written over Nq) carried out
    auto body = [&](const int it, const Part6& Mq, Part6& NqNn, const Part6& Np, Part6& nb) {
      const int p = xs - 1 + it;
      const int q = p - 1;   // destination plane finished in this iteration
      const bool store_plane = wr && it >= 2;
      // STATS + SPECIAL: boundary / solid cells are finished by the compacted kernels and stay out
      // of the statistics; their two bits come from the CTA's shared-memory copy of the bitmask
      uint32_t sbits = 0;
      if (STATS && SPECIAL && store_plane)
        sbits = (sbm[(q - xs) * kRows + (w - 1)][lane >> 4] >> (2 * (lane & 15))) & 3u;
      const int b = (NB == 2) ? (it & 1) : 0;
      const uint32_t eph = (uint32_t)((NB == 2) ? (it >> 1) : it) & 1u;
      V (*exch)[kNW][32] = S.exch[b];
      mbar_wait(&S.bar[st], sph);
      V fin[10];   // dest q, raw-moment order m000 m100 m010 m001 m200 m110 m101 m020 m011 m002
      V zcen[3][3];  // [kx][az]: ky = 0 z-stage values of this source row (y centre term)
      V zcb[3];      // D3Q19: chain B's az = 0 centre values
      {
        V s[10];
        load_state<Q16, QMODE, !FORCE>(S.stage[st], w, lane, plane_inflow(p), A, s);
        const Coef<V> C = coeffs_int<FORCE, Q16>(s, A.R);
        consumed();   // C depends on every loaded value
        // my slots of buffer b were read by my neighbours NB planes ago
        mbar_wait(&S.empty[b][w], eph ^ 1u);
        recon_row<0, LAT>(C, exch, w, lane, zcen[0], &zcb[0]);
        recon_row<1, LAT>(C, exch, w, lane, zcen[1], &zcb[1]);
        recon_row<2, LAT>(C, exch, w, lane, zcen[2], &zcb[2]);
      }
      if (++st == STAGES) { st = 0; sph ^= 1u; }
      mbar_arrive(&S.full[b][w]);
      mbar_wait(&S.full[b][wu], eph);
      mbar_wait(&S.full[b][wd], eph);
      yx_stage<LAT>(exch, wu, wd, lane, zcen, Mq, NqNn, Np, fin, nb, zcb);
      mbar_arrive(&S.empty[b][wu]);
      mbar_arrive(&S.empty[b][wd]);
      if (store_plane) {
        const bool sx = STATS && !(sbits & 1u), sy = STATS && !(sbits & 2u);
        store_pair<Q16, DITHER, STATS, QMODE>(A, fin, q, yrow, zc, cell0, sx, sy, acc);
      }
    };

    if (active) {
      for (int it = 0; it < NP; it += 2) {
        body(it, Ma, Nb, Na, Mb);
        if (it + 1 < NP) body(it + 1, Mb, Na, Nb, Ma);
      }
    } else {
      // the same waits and arrivals per plane as `body`, no arithmetic
      for (int it = 0; it < NP; ++it) {
        const int b = (NB == 2) ? (it & 1) : 0;
        const uint32_t eph = (uint32_t)((NB == 2) ? (it >> 1) : it) & 1u;
        mbar_wait(&S.bar[st], sph);
        consumed();
        mbar_wait(&S.empty[b][w], eph ^ 1u);
        if (++st == STAGES) { st = 0; sph ^= 1u; }
        mbar_arrive(&S.full[b][w]);
        mbar_wait(&S.full[b][wu], eph);
        mbar_wait(&S.full[b][wd], eph);
        mbar_arrive(&S.empty[b][wu]);
        mbar_arrive(&S.empty[b][wd]);
      }
    }
  }

  if (STATS) {
    // block reduction of the fused statistics
    float red[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) red[k] = acc[32 * k];
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
#ifndef HLBM_Q16_STAGES
#define HLBM_Q16_STAGES 3
#endif
#ifndef HLBM_Q16_NB
#define HLBM_Q16_NB 1   // measured: a second exchange buffer buys nothing (2.23 vs 2.25 ms, 512^3)
#endif
#ifndef HLBM_F32_STAGES
#define HLBM_F32_STAGES 3
#endif
#ifndef HLBM_F32_NB
#define HLBM_F32_NB 1   // fp32 tiles leave room for one exchange buffer next to 3 stages
#endif
template <bool Q16, int LAT = 27> struct InteriorCfg {
  // fp32 D3Q19: the 24-slot exchange leaves room for 2 TMA stages only (227 KB per CTA)
  static constexpr int STAGES = Q16 ? HLBM_Q16_STAGES : (LAT == 19 ? 2 : HLBM_F32_STAGES);
  static constexpr int NB = Q16 ? HLBM_Q16_NB : HLBM_F32_NB;
};

template <bool Q16, bool FORCE, bool SPECIAL, bool DITHER, bool STATS, int QMODE, int LAT = 27>
static cudaError_t launch_interior_t(const StepArgs& A, int nblocks, cudaStream_t st) {
  constexpr int STAGES = InteriorCfg<Q16, LAT>::STAGES, NB = InteriorCfg<Q16, LAT>::NB;
  constexpr int NC = Q16 ? 5 : 10;
  // STATS + SPECIAL: + the tile's special-cell bitmask (kMaxXseg planes x kRows rows x 64 bits)
  const size_t smem = sizeof(Smem<NC, STAGES, NB, LatSlots<LAT>::n>) +
                      ((STATS && SPECIAL) ? (size_t)kMaxXseg * kRows * 8 : 0);
  auto k = fluid_interior<Q16, FORCE, SPECIAL, DITHER, STATS, QMODE, STAGES, NB, LAT>;
  static bool attr = false;   // once per instantiation, not on every launch
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k<<<nblocks, kNW * 32, smem, st>>>(A);
  return cudaGetLastError();
}

// 16-bit dispatch units (one translation unit per codec mode, hlbm_interior_q{0,1,2}.cu)
#define HLBM_INTERIOR_Q16_UNIT(M)                                                                        \
  cudaError_t launch_interior_q16_m##M(const StepArgs& A, int nblocks, bool force, bool special, bool dither, \
                                       cudaStream_t st) {                                                \
    const bool stats = A.do_stats != 0;                                                                  \
    if (!stats) {                                                                                        \
      if (force) return dither ? launch_interior_t<true, true, false, true, false, M>(A, nblocks, st)    \
                               : launch_interior_t<true, true, false, false, false, M>(A, nblocks, st);  \
      return dither ? launch_interior_t<true, false, false, true, false, M>(A, nblocks, st)              \
                    : launch_interior_t<true, false, false, false, false, M>(A, nblocks, st);            \
    }                                                                                                    \
    if (special) {                                                                                       \
      if (force) return dither ? launch_interior_t<true, true, true, true, true, M>(A, nblocks, st)      \
                               : launch_interior_t<true, true, true, false, true, M>(A, nblocks, st);    \
      return dither ? launch_interior_t<true, false, true, true, true, M>(A, nblocks, st)                \
                    : launch_interior_t<true, false, true, false, true, M>(A, nblocks, st);              \
    }                                                                                                    \
    if (force) return dither ? launch_interior_t<true, true, false, true, true, M>(A, nblocks, st)       \
                             : launch_interior_t<true, true, false, false, true, M>(A, nblocks, st);     \
    return dither ? launch_interior_t<true, false, false, true, true, M>(A, nblocks, st)                 \
                  : launch_interior_t<true, false, false, false, true, M>(A, nblocks, st);               \
  }

cudaError_t launch_interior_q16_m0(const StepArgs& A, int nblocks, bool force, bool special, bool dither,
                                   cudaStream_t st);
cudaError_t launch_interior_q16_m1(const StepArgs& A, int nblocks, bool force, bool special, bool dither,
                                   cudaStream_t st);
cudaError_t launch_interior_q16_m2(const StepArgs& A, int nblocks, bool force, bool special, bool dither,
                                   cudaStream_t st);

}  // namespace hlbm
