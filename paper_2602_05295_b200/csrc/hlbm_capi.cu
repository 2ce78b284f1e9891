// C-ABI implementation: context, buffers, stepping (host side of include/hlbm.h).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hlbm.h"
#include "hlbm_launch.h"

using namespace hlbm;

struct hlbm_ctx {
  hlbm_config cfg{};
  int q16 = 0, NC = 10;
  int q = 27;        // velocity set (D3Q19 steps with the per-cell fused kernel)
  bool b16 = true;   // every component uses all 16 bits of its slot
  int qmode = 0;     // interior-kernel codec variant (hlbm_launch.h)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  size_t elem_bytes = 4;
  int64_t plane_elems = 0, total_elems = 0;
  int zp = 0;
  int num_sms = 148;
  CUtensorMap tmap[2];
  void* buf[2] = {nullptr, nullptr};
  int cur = 0;
  Stats* d_stats = nullptr;
  Stats* h_stats = nullptr;      // pinned host copy (one D2H per Solver.step, no extra sync)
  Relax R{};
  Codec Q{};
  Ranges RG{};
  float inflow[10] = {};
  double om_d = 0.0;                          // 1 - s in double (coeffs_pre input scales)
  double dec_step_d[10] = {}, dec_off_d[10] = {};
  int x_lo_src = 0, x_hi_src = 0;
  // solids
  int64_t* d_bcells = nullptr;
  uint32_t* d_bmasks = nullptr;
  int64_t nb = 0;
  int64_t* d_scells = nullptr;
  int64_t ns = 0;
  uint32_t* d_bits = nullptr;
  int bits_row_words = 0;
  uint32_t* d_fused = nullptr;   // dense per-cell mask of the fused Alg.-1 step (voxel solids)
  MeshLinks mesh;                // triangle-mesh cut links (replaces the voxel lists when set)
  float solid_v[3] = {0, 0, 0}, solid_w[3] = {0, 0, 0}, solid_c[3] = {0, 0, 0};
  std::vector<int64_t> off_b, off_s, off_m;   // per-plane offsets (nx+1) into the sorted lists
  int pending_stats = 0;                      // statistics requested for the step in progress
  int pending_solid = 0;                      // hlbm_fluid_update ran, its solid correction not yet
  double* d_stage = nullptr;                  // host<->device staging of the float64 import/export
  size_t stage_bytes = 0;
  int64_t steps = 0;
  int64_t launches = 0;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  // peer-store halo (hlbm_ipc_*): the x-lo (0) and x-hi (1) neighbours' state buffers mapped
  // through CUDA IPC; a neighbour's current buffer is (our cur) ^ rel -- every rank flips its
  // buffer once per step, so the relation holds until a rank re-imports its state
  struct Peer {
    void* buf[2] = {nullptr, nullptr};
    int nx = 0, rel = 0;
    bool open = false, owner = false;
    cudaIpcMemHandle_t h[2];
  } peer[2];
  double last_t_fluid = 0, last_t_solid = 0;
  std::string err;
};

namespace {

int fail(hlbm_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(ctx, HLBM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// x-segment length of the interior kernel: each CTA marches xseg planes (+2 re-read planes).
// Time ~ ceil(blocks / sms) * (xseg + 2); pick the xseg minimising it relative to the work.
// Segments are capped at 128 planes: longer ones measured slower on B200 (all CTAs of a wave
// then stream the same few x-planes; fp32 512^3: 3.63 ms at 512 planes vs 2.63 ms at 128).
int auto_xseg(int nx, int tiles_yz, int sms) {
  int best = std::min(nx, 128);
  double best_cost = 1e30;
  for (int xs = std::min(nx, 128); xs >= 1; --xs) {
    const int64_t blocks = (int64_t)tiles_yz * ((nx + xs - 1) / xs);
    const double waves = std::ceil((double)blocks / sms);
    const double cost = waves * (xs + 2) * sms / ((double)tiles_yz * nx);
    if (cost < best_cost * (1.0 - 1e-3)) {
      best_cost = cost;
      best = xs;
    }
  }
  return best;
}

// device staging buffer of at least `bytes` (kept for later calls)
int staging(hlbm_ctx* ctx, size_t bytes) {
  if (ctx->stage_bytes >= bytes) return HLBM_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(ctx->d_stage);
  ctx->d_stage = nullptr;
  ctx->stage_bytes = 0;
  CK(cudaMalloc(&ctx->d_stage, bytes));
  ctx->stage_bytes = bytes;
  return HLBM_OK;
}

Geo make_geo(const hlbm_ctx* ctx, int xb = 0, int xr = -1) {
  const hlbm_config& c = ctx->cfg;
  if (xr < 0) xr = c.nx;
  Geo g{};
  g.nx = c.nx; g.ny = c.ny; g.nz = c.nz;
  g.zp = ctx->zp;
  g.cstride = (int64_t)(c.ny + 2) * ctx->zp;
  g.pstride = ctx->plane_elems;
  g.x_lo_src = ctx->x_lo_src;
  g.x_hi_src = ctx->x_hi_src;
  g.nzt = (c.nz + kZT - 1) / kZT;
  g.nyt = (c.ny + kRows - 1) / kRows;
  const int nr = std::max(xr - xb, 0);
  g.xb = xb;
  g.xr = xr;
  g.xseg = c.xseg > 0 ? std::min(std::min(c.xseg, kMaxXseg), std::max(nr, 1))
                      : auto_xseg(std::max(nr, 1), g.nzt * g.nyt, ctx->num_sms * kCtaPerSm);
  g.nxs = nr > 0 ? (nr + g.xseg - 1) / g.xseg : 0;
  g.gx0 = c.x0; g.gny = c.gny; g.gnz = c.gnz; g.gnx_total = c.gnx;
  return g;
}

uint32_t step_key(int64_t step, uint32_t seed) {   // oracle/codec.py: step_key
  const uint64_t v = ((uint64_t)step * 0x9E3779B9ull + (uint64_t)seed * 0x85EBCA6Bull + 0x2545F491ull) &
                     0xFFFFFFFFull;
  return mix32((uint32_t)v);
}

StepArgs make_args(hlbm_ctx* ctx, int with_stats, int xb = 0, int xr = -1) {
  StepArgs A{};
  A.tmap_in = ctx->tmap[ctx->cur];
  A.in = ctx->buf[ctx->cur];
  A.out = ctx->buf[1 - ctx->cur];
  A.g = make_geo(ctx, xb, xr);
  A.R = ctx->R;
  A.Q = ctx->Q;
  for (int i = 0; i < 10; ++i) {
    A.inflow[i] = ctx->inflow[i];
    const double k = pre_scale(i, ctx->om_d);
    A.pre_step[i] = (float)(ctx->dec_step_d[i] * k);
    A.pre_off[i] = (float)(ctx->dec_off_d[i] * k);
    A.pre_k[i] = (float)k;
    A.inflow_pre[i] = (float)((double)ctx->inflow[i] * k);
  }
  A.special_bits = ctx->d_bits;
  A.bits_row_words = ctx->bits_row_words;
  A.step_key = step_key(ctx->steps, ctx->cfg.seed);
  A.do_stats = with_stats;
  A.stats = ctx->d_stats;
  A.cut_t = ctx->mesh.t32;
  A.wall_masks = ctx->mesh.wmasks;
  for (int k = 0; k < 3; ++k) {
    A.solid_v[k] = ctx->solid_v[k];
    A.solid_w[k] = ctx->solid_w[k];
    A.solid_c[k] = ctx->solid_c[k];
  }
  return A;
}

unsigned long long* sat_ptr(hlbm_ctx* ctx) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ctx->d_stats) + offsetof(Stats, sat));
}

// 4-D tensor map (zs, ys, c, xs) over one state buffer; box = one CTA plane tile
int make_tensor_map(hlbm_ctx* ctx, int b) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return fail(ctx, HLBM_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const hlbm_config& c = ctx->cfg;
  cuuint64_t dims[4] = {(cuuint64_t)ctx->zp, (cuuint64_t)(c.ny + 2), (cuuint64_t)ctx->NC, (cuuint64_t)(c.nx + 2)};
  cuuint64_t strides[3] = {(cuuint64_t)ctx->zp * 4, (cuuint64_t)(c.ny + 2) * ctx->zp * 4,
                           (cuuint64_t)ctx->plane_elems * 4};
  cuuint32_t box[4] = {(cuuint32_t)kZW, (cuuint32_t)kBoxRows, (cuuint32_t)ctx->NC, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode(&ctx->tmap[b], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, ctx->buf[b], dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, HLBM_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return HLBM_OK;
}

void free_mesh(hlbm_ctx* ctx) {
  cudaFree(ctx->mesh.cells);
  cudaFree(ctx->mesh.masks);
  cudaFree(ctx->mesh.t64);
  cudaFree(ctx->mesh.t32);
  cudaFree(ctx->mesh.tri);
  cudaFree(ctx->mesh.wmasks);
  cudaFree(ctx->mesh.dense);
  ctx->mesh = MeshLinks();
}

// dense per-cell positions in the cut-link list for the fused Alg.-1 kernel (built once per mesh)
int mesh_dense(hlbm_ctx* ctx) {
  if (!ctx->mesh.nb || ctx->mesh.dense) return HLBM_OK;
  const int64_t n = (int64_t)ctx->cfg.nx * ctx->cfg.ny * ctx->cfg.nz;
  CK(cudaMalloc(&ctx->mesh.dense, (size_t)n * 4));
  CK(launch_mesh_index(ctx->mesh.cells, ctx->mesh.nb, n, ctx->mesh.dense, ctx->stream));
  return HLBM_OK;
}

bool has_force(const hlbm_ctx* ctx) {
  return ctx->cfg.force[0] != 0.0 || ctx->cfg.force[1] != 0.0 || ctx->cfg.force[2] != 0.0;
}

// offsets[x] = first position in the sorted local-index list whose cell lies in plane >= x
int plane_offsets(hlbm_ctx* ctx, const int64_t* d_cells, int64_t n, std::vector<int64_t>& off) {
  const hlbm_config& c = ctx->cfg;
  const int64_t pl = (int64_t)c.ny * c.nz;
  off.assign((size_t)c.nx + 1, n);
  if (n == 0) { std::fill(off.begin(), off.end(), 0); return HLBM_OK; }
  std::vector<int64_t> h((size_t)n);
  // the list was built on the context's (non-blocking) stream: a legacy-stream cudaMemcpy would not
  // wait for it (the offsets of the last list built by hlbm_set_mask / hlbm_set_mesh raced the
  // compaction kernel and could misplace cells between the x-ranges of the overlapped step)
  CK(cudaMemcpyAsync(h.data(), d_cells, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int64_t i = 0;
  for (int x = 0; x <= c.nx; ++x) {
    while (i < n && h[(size_t)i] / pl < x) ++i;
    off[(size_t)x] = i;
  }
  return HLBM_OK;
}

// a one-row slab (ny == 1): the interior kernel writes only the y = ny ghost image of an edge row;
// refresh both ghost rows of the planes [xb, xr) of the written buffer (tiny grids only, off the
// hot kernel; only the range's own planes, so ranges on concurrent streams stay independent)
int fix_one_row(hlbm_ctx* ctx, int xb, int xr, cudaStream_t st) {
  if (ctx->cfg.ny != 1) return HLBM_OK;
  CK(launch_fill_ghosts(make_geo(ctx, xb, xr), ctx->NC, ctx->buf[1 - ctx->cur], st));
  ++ctx->launches;
  return HLBM_OK;
}

// interior kernel + compacted boundary kernels for destination planes [xb, xr), on stream st
// (default: the context's stream).  phases: bit 0 the fluid update (interior kernel, every cell,
// no obstacle logic), bit 1 the solid correction (compacted kernels over the boundary / solid /
// cut-link lists, which overwrite their cells of the same output buffer)
constexpr int kPhaseFluid = 1, kPhaseSolid = 2;
int run_range(hlbm_ctx* ctx, int xb, int xr, int with_stats, cudaEvent_t after_interior = nullptr,
              cudaStream_t st = nullptr, int phases = kPhaseFluid | kPhaseSolid) {
  if (xr <= xb) return HLBM_OK;
  if (!st) st = ctx->stream;
  const bool q16 = ctx->q16, force = has_force(ctx), dither = q16 && ctx->cfg.dither;
  const bool special = ctx->nb + ctx->ns + ctx->mesh.nb > 0;
  StepArgs A = make_args(ctx, with_stats, xb, xr);
  const bool fast19 = ctx->q == 19;   // every D3Q19 codec runs the two-chain interior kernel
  if (ctx->q == 19 && !fast19) {
    // D3Q19 with a non-default codec: the per-cell fused kernel over the planes of the range,
    // solid links inline (no separate correction phase)
    if (!(phases & kPhaseFluid)) return HLBM_OK;
    const int64_t pl = (int64_t)ctx->cfg.ny * ctx->cfg.nz;
    CK(launch_pull_cells(A, nullptr, ctx->d_fused, (int64_t)(xr - xb) * pl, 3, q16, force, dither, st, 19,
                         (int64_t)xb * pl));
    ++ctx->launches;
    if (after_interior) CK(cudaEventRecord(after_interior, st));
    return fix_one_row(ctx, xb, xr, st);
  }
  if (phases & kPhaseFluid) {
    if (fast19)   // D3Q19: two-chain streaming; solids through the compacted 19-link kernels below
      CK(launch_fluid_interior19(A, q16, force, special, dither, ctx->qmode, st));
    else
      CK(launch_fluid_interior(A, q16, force, special, dither, ctx->qmode, st));
    ++ctx->launches;
  }
  if (after_interior) CK(cudaEventRecord(after_interior, st));
  if (!(phases & kPhaseSolid)) return fix_one_row(ctx, xb, xr, st);
  auto sub = [&](const std::vector<int64_t>& off, int64_t n, int64_t& a, int64_t& cnt) {
    if (off.empty()) { a = 0; cnt = (xb == 0 && xr == ctx->cfg.nx) ? n : 0; return; }
    a = off[(size_t)xb];
    cnt = off[(size_t)xr] - a;
  };
  int64_t a, cnt;
  sub(ctx->off_b, ctx->nb, a, cnt);
  if (cnt > 0) {
    CK(launch_pull_cells(A, ctx->d_bcells + a, ctx->d_bmasks + a, cnt, 0, q16, force, dither, st, ctx->q));
    ++ctx->launches;
  }
  sub(ctx->off_s, ctx->ns, a, cnt);
  if (cnt > 0) {
    CK(launch_pull_cells(A, ctx->d_scells + a, nullptr, cnt, 1, q16, force, dither, st, ctx->q));
    ++ctx->launches;
  }
  sub(ctx->off_m, ctx->mesh.nb, a, cnt);
  if (cnt > 0) {
    StepArgs Am = A;
    Am.cut_t = ctx->mesh.t32 + a * 27;
    Am.wall_masks = ctx->mesh.wmasks ? ctx->mesh.wmasks + a : nullptr;
    CK(launch_pull_cells(Am, ctx->mesh.cells + a, ctx->mesh.masks + a, cnt, 2, q16, force, dither, st, ctx->q));
    ++ctx->launches;
  }
  return fix_one_row(ctx, xb, xr, st);
}

}  // namespace

// SPEC's two-phase step (fluid_update_step then solid_correction_step): a fluid
// update whose solid correction has not run yet leaves the step uncommitted (the corrected cells
// of the output buffer are still missing); every other state access finishes it first
static int settle(hlbm_ctx* ctx) {
  if (!ctx || !ctx->pending_solid) return HLBM_OK;
  return hlbm_solid_correction(ctx, nullptr);
}
#define SETTLE(ctx)                               \
  do {                                            \
    if (int r_ = settle(ctx)) return r_;          \
  } while (0)

extern "C" {

const char* hlbm_version(void) { return "hlbm-b200 0.1 (sm_100a)"; }

int hlbm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

const char* hlbm_last_error(const hlbm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void hlbm_config_init(hlbm_config* cfg) {
  if (!cfg) return;
  memset(cfg, 0, sizeof(*cfg));
  cfg->struct_size = (int32_t)sizeof(hlbm_config);
  static const double dmn[10] = {0.8, -0.6, -0.6, -0.6, -0.1, -0.1, -0.1, -0.1, -0.1, -0.1};
  static const double dmx[10] = {1.5, 0.6, 0.6, 0.6, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1};
  for (int k = 0; k < 10; ++k) {
    cfg->qmin[k] = dmn[k];
    cfg->qmax[k] = dmx[k];
    cfg->bits[k] = 16;
  }
  cfg->q = 27;
}

int hlbm_create(const hlbm_config* cfg, hlbm_ctx** out) {
  if (!cfg || !out) return HLBM_EINVAL;
  *out = nullptr;
  hlbm_ctx* ctx = new hlbm_ctx();
  auto bad = [&](const std::string& m) {
    int r = fail(ctx, HLBM_EINVAL, m);
    *out = ctx;   // caller reads the message, then destroys
    return r;
  };
  // ABI guard: read only the size field until the caller's layout is known to match
  if (cfg->struct_size != (int32_t)sizeof(hlbm_config))
    return bad("hlbm_config.struct_size is " + std::to_string(cfg->struct_size) + ", this library expects " +
               std::to_string(sizeof(hlbm_config)) + " (binding built against another hlbm.h)");
  ctx->cfg = *cfg;
  hlbm_config& c = ctx->cfg;
  if (c.nx < 1 || c.ny < 1 || c.nz < 4) return bad("grid dims must be >= 1 (nz >= 4)");
  if (c.nz % 4 != 0) return bad("nz must be a multiple of 4");
  if (c.gnx <= 0) c.gnx = c.nx;
  if (c.gny <= 0) c.gny = c.ny;
  if (c.gnz <= 0) c.gnz = c.nz;
  if (c.gny != c.ny || c.gnz != c.nz) return bad("slabs split x only: gny/gnz must equal ny/nz");
  if ((int64_t)c.gnx * c.gny * c.gnz >= (int64_t)1 << 32) return bad("global grid exceeds 2^32 cells");
  if (!(c.tau > 0.5)) return bad("tau must exceed 0.5 (non-negative viscosity)");
  for (int f = 0; f < 6; ++f)
    if (c.bc[f] < 0 || c.bc[f] > 3) return bad("unknown boundary condition");
  for (int f = 2; f < 6; ++f)
    if (c.bc[f] == HLBM_BC_INFLOW || c.bc[f] == HLBM_BC_OUTFLOW)
      return bad("y/z faces support periodic or wall only");
  if ((c.bc[0] == HLBM_BC_PERIODIC) != (c.bc[1] == HLBM_BC_PERIODIC) && !(c.x_lo_remote || c.x_hi_remote))
    return bad("periodic x needs both x faces periodic");
  if ((c.bc[2] == HLBM_BC_PERIODIC) != (c.bc[3] == HLBM_BC_PERIODIC) ||
      (c.bc[4] == HLBM_BC_PERIODIC) != (c.bc[5] == HLBM_BC_PERIODIC))
    return bad("periodic y/z needs both faces periodic");
  if (c.precision != HLBM_FP32 && c.precision != HLBM_Q16) return bad("unknown precision");
  if (c.q == 0) c.q = 27;
  if (c.q != 27 && c.q != 19) return bad("lattice must be D3Q27 or D3Q19");
  ctx->q = c.q;
  ctx->q16 = c.precision == HLBM_Q16;
  ctx->NC = ctx->q16 ? 5 : 10;
  if (ctx->q16) {
    for (int k = 0; k < 10; ++k) {
      if (c.bits[k] == 0) c.bits[k] = 16;
      if (c.bits[k] < 2 || c.bits[k] > 16) return bad("bits per component must lie in [2, 16]");
      if (!(c.qmax[k] > c.qmin[k])) return bad("quantization range needs min < max");
      if (c.bits[k] != 16) ctx->b16 = false;
    }
  }
  if (cudaSetDevice(c.device) != cudaSuccess) return bad("cannot select CUDA device");
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, c.device);

  // relaxation constants (collision.py:158-191)
  const double tau = c.tau, s = 1.0 / tau;
  ctx->R.om = (float)(1.0 - s);
  ctx->om_d = 1.0 - s;
  ctx->R.cxy = (float)((2 * tau - 1) / (2 * tau));
  ctx->R.cd = (float)((tau - 1) / (3 * tau));
  ctx->R.fx = (float)c.force[0];
  ctx->R.fy = (float)c.force[1];
  ctx->R.fz = (float)c.force[2];
  // inflow ghost state: rho = 1, j = u_in, sneq = 0
  for (int k = 0; k < 10; ++k) ctx->inflow[k] = 0.f;
  ctx->inflow[1] = (float)c.u_in[0];
  ctx->inflow[2] = (float)c.u_in[1];
  ctx->inflow[3] = (float)c.u_in[2];
  // codec
  for (int k = 0; k < 10; ++k) {
    const double mn = ctx->q16 ? c.qmin[k] : 0.0, mx = ctx->q16 ? c.qmax[k] : 1.0;
    const double L = ctx->q16 ? (double)((1u << c.bits[k]) - 1u) : 1.0;
    ctx->RG.mn[k] = mn;
    ctx->RG.mx[k] = mx;
    ctx->RG.levels[k] = L;
    const double shift = (k == 0) ? 1.0 : 0.0;   // component 0 is held as d = rho - 1
    // decode re-centred on q0 = the code of the centre value (hlbm_math.cuh Codec::dec_c)
    const double step = (mx - mn) / L;
    const double q0 = ctx->q16 ? std::min(L, std::max(0.0, std::floor((shift - mn) / step + 0.5))) : 0.0;
    ctx->Q.dec_step[k] = (float)step;
    ctx->Q.dec_off[k] = (float)(mn - shift + q0 * step);
    ctx->Q.dec_c[k] = (float)(8388608.0 + q0);
    ctx->dec_step_d[k] = step;
    ctx->dec_off_d[k] = mn - shift + q0 * step;
    const double sc = L / (mx - mn);
    ctx->Q.enc_scale[k] = (float)sc;
    ctx->Q.enc_off[k] = (float)((shift - mn) * sc + 0.5);
    ctx->Q.enc_int[k] = (float)std::floor((shift - mn) * sc + 0.5);
    ctx->Q.enc_frac[k] = (float)((shift - mn) * sc + 0.5 - std::floor((shift - mn) * sc + 0.5));
    ctx->Q.enc_nb[k] = (float)(-1.5 + 1.0 / 131072.0 - ((double)ctx->Q.enc_off[k] - ((shift - mn) * sc + 0.5)));
    const double mid = 0.5 * (mn + mx), half = 0.5 * (mx - mn);
    ctx->Q.sat_a[k] = (float)(1.0 / half);
    ctx->Q.sat_b[k] = (float)((shift - mid) / half);
    ctx->Q.levels[k] = (uint32_t)L;
  }
  if (ctx->q16) {
    static const double dmn[10] = {0.8, -0.6, -0.6, -0.6, -0.1, -0.1, -0.1, -0.1, -0.1, -0.1};
    static const double dmx[10] = {1.5, 0.6, 0.6, 0.6, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1};
    bool def = ctx->b16;
    for (int k = 0; k < 10; ++k) def = def && c.qmin[k] == dmn[k] && c.qmax[k] == dmx[k];
    ctx->qmode = def ? 2 : (ctx->b16 ? 1 : 0);
  }
  // source-plane map for x = -1 / x = nx
  const int nx = c.nx;
  if (c.x_lo_remote) ctx->x_lo_src = 0;
  else if (c.bc[0] == HLBM_BC_PERIODIC) ctx->x_lo_src = nx;
  else if (c.bc[0] == HLBM_BC_INFLOW) ctx->x_lo_src = -1;
  else ctx->x_lo_src = 1;   // outflow: zero-gradient copy; wall: links bounce back
  if (c.x_hi_remote) ctx->x_hi_src = nx + 1;
  else if (c.bc[1] == HLBM_BC_PERIODIC) ctx->x_hi_src = 1;
  else if (c.bc[1] == HLBM_BC_INFLOW) ctx->x_hi_src = -1;
  else ctx->x_hi_src = nx;

  ctx->elem_bytes = 4;
  ctx->zp = (c.nz + kZOff + 1 + 3) / 4 * 4;   // pad column, z ghosts on both sides
  ctx->plane_elems = (int64_t)ctx->NC * (c.ny + 2) * ctx->zp;
  ctx->total_elems = ctx->plane_elems * (nx + 2);
  *out = ctx;
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  ctx->own_stream = true;
  for (int b = 0; b < 2; ++b) {
    CK(cudaMalloc(&ctx->buf[b], ctx->total_elems * 4));
    CK(cudaMemset(ctx->buf[b], 0, ctx->total_elems * 4));
    if (int r = make_tensor_map(ctx, b)) return r;
  }
  CK(cudaMalloc(&ctx->d_stats, sizeof(Stats)));
  CK(cudaMemset(ctx->d_stats, 0, sizeof(Stats)));
  CK(cudaMallocHost(&ctx->h_stats, sizeof(Stats)));
  for (int i = 0; i < 3; ++i) CK(cudaEventCreate(&ctx->ev[i]));
  // default state: rest (rho = 1, j = 0, sneq = 0) in both buffers
  for (int b = 0; b < 2; ++b) {
    CK(launch_init_modes(make_geo(ctx), ctx->q16, ctx->RG, ctx->buf[b], 1.0, nullptr, 0, ctx->stream));
    CK(launch_fill_ghosts(make_geo(ctx), ctx->NC, ctx->buf[b], ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  // wall faces need the boundary lists even without a solid mask (the wall ghost layer is solid,
  // its links bounce back): start from an all-fluid mask (a later hlbm_set_mask replaces it)
  bool wall = false;
  for (int f = 0; f < 6; ++f) wall = wall || c.bc[f] == HLBM_BC_WALL;
  if (wall) {
    const int64_t pl = (int64_t)c.ny * c.nz;
    std::vector<uint8_t> zero((size_t)(pl * c.nx), 0);
    if (int r = hlbm_set_mask(ctx, zero.data(), zero.data(), zero.data())) return r;
  }
  return HLBM_OK;
}

void hlbm_destroy(hlbm_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (int b = 0; b < 2; ++b) cudaFree(ctx->buf[b]);
  cudaFree(ctx->d_stats);
  cudaFreeHost(ctx->h_stats);
  cudaFree(ctx->d_bcells);
  cudaFree(ctx->d_bmasks);
  cudaFree(ctx->d_scells);
  cudaFree(ctx->d_bits);
  cudaFree(ctx->d_fused);
  cudaFree(ctx->d_stage);
  hlbm_ipc_close(ctx);
  free_mesh(ctx);
  for (int i = 0; i < 3; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int hlbm_set_stream(hlbm_ctx* ctx, void* stream) {
  if (!ctx) return HLBM_EINVAL;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  ctx->stream = (cudaStream_t)stream;
  ctx->own_stream = false;
  return HLBM_OK;
}

int64_t hlbm_step_count(const hlbm_ctx* ctx) { return ctx ? ctx->steps : -1; }
int64_t hlbm_launch_count(const hlbm_ctx* ctx) { return ctx ? ctx->launches : -1; }

int hlbm_state_buffer(hlbm_ctx* ctx, void** ptr, int64_t* bytes) {
  if (!ctx) return HLBM_EINVAL;
  SETTLE(ctx);
  if (ptr) *ptr = ctx->buf[ctx->cur];
  if (bytes) *bytes = ctx->total_elems * 4;
  return HLBM_OK;
}

int hlbm_halo_planes(hlbm_ctx* ctx, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                     int64_t* bytes) {
  if (!ctx) return HLBM_EINVAL;
  SETTLE(ctx);
  char* b = (char*)ctx->buf[ctx->cur];
  const int64_t pb = ctx->plane_elems * 4;
  if (send_lo) *send_lo = b + 1 * pb;
  if (send_hi) *send_hi = b + (int64_t)ctx->cfg.nx * pb;
  if (recv_lo) *recv_lo = b;
  if (recv_hi) *recv_hi = b + (int64_t)(ctx->cfg.nx + 1) * pb;
  if (bytes) *bytes = pb;
  return HLBM_OK;
}

int hlbm_next_halo_planes(hlbm_ctx* ctx, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                          int64_t* bytes) {
  if (!ctx) return HLBM_EINVAL;
  char* b = (char*)ctx->buf[1 - ctx->cur];
  const int64_t pb = ctx->plane_elems * 4;
  if (send_lo) *send_lo = b + 1 * pb;
  if (send_hi) *send_hi = b + (int64_t)ctx->cfg.nx * pb;
  if (recv_lo) *recv_lo = b;
  if (recv_hi) *recv_hi = b + (int64_t)(ctx->cfg.nx + 1) * pb;
  if (bytes) *bytes = pb;
  return HLBM_OK;
}

int hlbm_ipc_export(hlbm_ctx* ctx, void* handles, int32_t* cur) {
  if (!ctx || !handles) return fail(ctx, HLBM_EINVAL, "null argument");
  SETTLE(ctx);
  for (int b = 0; b < 2; ++b)
    CK(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handles) + b, ctx->buf[b]));
  if (cur) *cur = ctx->cur;
  return HLBM_OK;
}

int hlbm_ipc_open(hlbm_ctx* ctx, int32_t side, const void* handles, int32_t peer_nx, int32_t peer_cur) {
  if (!ctx || !handles || side < 0 || side > 1 || peer_nx < 1 || (peer_cur & ~1))
    return fail(ctx, HLBM_EINVAL, "bad arguments");
  auto& P = ctx->peer[side];
  if (P.open) return fail(ctx, HLBM_EINVAL, "neighbour already mapped (hlbm_ipc_close first)");
  const auto* h = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
  const auto& O = ctx->peer[1 - side];
  if (O.open && !memcmp(O.h, h, sizeof(O.h))) {   // the same rank on both sides (2 ranks, periodic)
    P.buf[0] = O.buf[0];
    P.buf[1] = O.buf[1];
    P.owner = false;
  } else {
    for (int b = 0; b < 2; ++b) {
      cudaError_t e = cudaIpcOpenMemHandle(&P.buf[b], h[b], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        if (b) cudaIpcCloseMemHandle(P.buf[0]);
        P.buf[0] = P.buf[1] = nullptr;
        return fail(ctx, HLBM_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
    }
    P.owner = true;
  }
  memcpy(P.h, h, sizeof(P.h));
  P.nx = peer_nx;
  P.rel = (peer_cur ^ ctx->cur) & 1;
  P.open = true;
  return HLBM_OK;
}

int hlbm_ipc_sync(hlbm_ctx* ctx, int32_t side, int32_t peer_cur) {
  if (!ctx || side < 0 || side > 1 || (peer_cur & ~1)) return fail(ctx, HLBM_EINVAL, "bad arguments");
  if (!ctx->peer[side].open) return fail(ctx, HLBM_EINVAL, "neighbour not mapped");
  SETTLE(ctx);
  ctx->peer[side].rel = (peer_cur ^ ctx->cur) & 1;
  return HLBM_OK;
}

int hlbm_halo_push(hlbm_ctx* ctx, int32_t next_buffer, void* stream) {
  if (!ctx) return HLBM_EINVAL;
  if (!next_buffer) SETTLE(ctx);
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
  const int64_t pb = ctx->plane_elems * 4;
  const int mine = next_buffer ? 1 - ctx->cur : ctx->cur;
  const char* b = (const char*)ctx->buf[mine];
  for (int side = 0; side < 2; ++side) {
    const auto& P = ctx->peer[side];
    if (!P.open) continue;
    char* dst = (char*)P.buf[mine ^ P.rel];
    if (side == 0)   // our first interior plane -> the x-lo neighbour's hi ghost plane
      CK(cudaMemcpyAsync(dst + (int64_t)(P.nx + 1) * pb, b + pb, pb, cudaMemcpyDeviceToDevice, st));
    else             // our last interior plane -> the x-hi neighbour's lo ghost plane
      CK(cudaMemcpyAsync(dst, b + (int64_t)ctx->cfg.nx * pb, pb, cudaMemcpyDeviceToDevice, st));
  }
  return HLBM_OK;
}

int hlbm_ipc_close(hlbm_ctx* ctx) {
  if (!ctx) return HLBM_EINVAL;
  if (!ctx->peer[0].open && !ctx->peer[1].open) return HLBM_OK;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& P : ctx->peer) {
    if (P.open && P.owner)
      for (int b = 0; b < 2; ++b) cudaIpcCloseMemHandle(P.buf[b]);
    P = hlbm_ctx::Peer{};
  }
  return HLBM_OK;
}

int hlbm_set_moments(hlbm_ctx* ctx, const double* rho, const double* mom, const double* stress) {
  if (!ctx || !rho || !mom || !stress) return fail(ctx, HLBM_EINVAL, "null argument");
  SETTLE(ctx);
  const hlbm_config& c = ctx->cfg;
  const int64_t n = (int64_t)c.nx * c.ny * c.nz;
  const int64_t pl = (int64_t)c.ny * c.nz;
  const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(c.nx, (64ll << 20) / (pl * 80)));
  if (int r = staging(ctx, (size_t)chunk * pl * 10 * 8)) return r;   // reused across calls
  double* dr = ctx->d_stage;
  double* dm = dr + (size_t)chunk * pl;
  double* ds = dm + (size_t)3 * chunk * pl;
  // import into the spare buffer; it becomes current only if every density is positive
  // (moments.py:147), so a rejected call leaves the state untouched.  The check runs on the device.
  void* spare = ctx->buf[1 - ctx->cur];
  CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
  unsigned int* nonpos = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(ctx->d_stats) + offsetof(Stats, nonfinite));
  const Geo g = make_geo(ctx);
  for (int x0 = 0; x0 < c.nx; x0 += chunk) {
    const int cnt = std::min(chunk, c.nx - x0);
    const int64_t m = cnt * pl;
    CK(cudaMemcpyAsync(dr, rho + x0 * pl, m * 8, cudaMemcpyHostToDevice, ctx->stream));
    for (int k = 0; k < 3; ++k)
      CK(cudaMemcpyAsync(dm + k * m, mom + k * n + x0 * pl, m * 8, cudaMemcpyHostToDevice, ctx->stream));
    for (int k = 0; k < 6; ++k)
      CK(cudaMemcpyAsync(ds + k * m, stress + k * n + x0 * pl, m * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(launch_import(g, ctx->RG, ctx->q16, spare, dr, dm, ds, x0, cnt, sat_ptr(ctx), nonpos, ctx->stream));
  }
  unsigned int bad = 0;
  CK(cudaMemcpyAsync(&bad, nonpos, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad) return fail(ctx, HLBM_EINVAL, "density must be positive");
  CK(launch_fill_ghosts(g, ctx->NC, spare, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->cur = 1 - ctx->cur;
  return HLBM_OK;
}

int hlbm_get_moments_box(hlbm_ctx* ctx, int32_t x0, int32_t cx, int32_t y0, int32_t cy, int32_t z0,
                         int32_t cz, double* rho, double* mom, double* stress) {
  if (!ctx || !rho || !mom || !stress) return fail(ctx, HLBM_EINVAL, "null argument");
  SETTLE(ctx);
  const hlbm_config& c = ctx->cfg;
  if (x0 < 0 || cx < 0 || x0 + cx > c.nx || cy < 0 || cz < 0) return fail(ctx, HLBM_EINVAL, "box out of range");
  const int64_t pl = (int64_t)cy * cz;
  if (pl == 0 || cx == 0) return HLBM_OK;
  const int64_t n = pl * cx;
  const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(cx, (64ll << 20) / (pl * 80)));
  if (int r = staging(ctx, (size_t)chunk * pl * 10 * 8)) return r;
  double* dr = ctx->d_stage;
  double* dm = dr + (size_t)chunk * pl;
  double* ds = dm + (size_t)3 * chunk * pl;
  const Geo g = make_geo(ctx);
  for (int xa = 0; xa < cx; xa += chunk) {
    const int cnt = std::min(chunk, cx - xa);
    const int64_t m = cnt * pl;
    CK(launch_export(g, ctx->RG, ctx->q16, ctx->buf[ctx->cur], dr, dm, ds, x0 + xa, cnt, y0, cy, z0, cz,
                     ctx->stream));
    CK(cudaMemcpyAsync(rho + xa * pl, dr, m * 8, cudaMemcpyDeviceToHost, ctx->stream));
    for (int k = 0; k < 3; ++k)
      CK(cudaMemcpyAsync(mom + k * n + xa * pl, dm + k * m, m * 8, cudaMemcpyDeviceToHost, ctx->stream));
    for (int k = 0; k < 6; ++k)
      CK(cudaMemcpyAsync(stress + k * n + xa * pl, ds + k * m, m * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return HLBM_OK;
}

int hlbm_get_moments(hlbm_ctx* ctx, double* rho, double* mom, double* stress) {
  if (!ctx) return HLBM_EINVAL;
  return hlbm_get_moments_box(ctx, 0, ctx->cfg.nx, 0, ctx->cfg.ny, 0, ctx->cfg.nz, rho, mom, stress);
}

int hlbm_init_modes(hlbm_ctx* ctx, double rho0, const double* modes, int32_t nmodes) {
  if (!ctx || (nmodes > 0 && !modes) || nmodes < 0) return fail(ctx, HLBM_EINVAL, "bad modes");
  SETTLE(ctx);
  if (!(rho0 > 0.0)) return fail(ctx, HLBM_EINVAL, "density must be positive");
  double* dmodes = nullptr;
  if (nmodes > 0) {
    CK(cudaMalloc(&dmodes, (size_t)nmodes * 7 * 8));
    CK(cudaMemcpy(dmodes, modes, (size_t)nmodes * 7 * 8, cudaMemcpyHostToDevice));
  }
  CK(launch_init_modes(make_geo(ctx), ctx->q16, ctx->RG, ctx->buf[ctx->cur], rho0, dmodes, nmodes,
                       ctx->stream));
  CK(launch_fill_ghosts(make_geo(ctx), ctx->NC, ctx->buf[ctx->cur], ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(dmodes);
  return HLBM_OK;
}

// dense (NC, nx, ny, nz) host words <-> the padded device layout, one strided 3-D DMA copy per
// component (rows of nz words; device rows at pitch zp, x-planes every NC*(ny+2) rows)
static int copy_dense(hlbm_ctx* ctx, void* host, bool to_host) {
  const hlbm_config& c = ctx->cfg;
  const size_t row = (size_t)c.nz * 4;
  for (int k = 0; k < ctx->NC; ++k) {
    cudaMemcpy3DParms p{};
    cudaPitchedPtr dev = make_cudaPitchedPtr(ctx->buf[ctx->cur], (size_t)ctx->zp * 4, (size_t)ctx->zp,
                                             (size_t)ctx->NC * (c.ny + 2));
    cudaPitchedPtr hst = make_cudaPitchedPtr((char*)host + (size_t)k * c.nx * c.ny * row, row, (size_t)c.nz,
                                             (size_t)c.ny);
    // device element (x+1, k, y+1, z+kZOff) in bytes/rows/slices: x-planes are the slices
    const cudaPos dpos = make_cudaPos((size_t)kZOff * 4, (size_t)k * (c.ny + 2) + 1, 1);
    const cudaPos hpos = make_cudaPos(0, 0, 0);
    p.extent = make_cudaExtent(row, (size_t)c.ny, (size_t)c.nx);
    p.kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
    if (to_host) { p.srcPtr = dev; p.srcPos = dpos; p.dstPtr = hst; p.dstPos = hpos; }
    else { p.srcPtr = hst; p.srcPos = hpos; p.dstPtr = dev; p.dstPos = dpos; }
    CK(cudaMemcpy3DAsync(&p, ctx->stream));
  }
  return HLBM_OK;
}

int hlbm_get_state(hlbm_ctx* ctx, void* words) {
  if (!ctx || !words) return fail(ctx, HLBM_EINVAL, "null argument");
  SETTLE(ctx);
  if (int r = copy_dense(ctx, words, true)) return r;
  CK(cudaStreamSynchronize(ctx->stream));
  return HLBM_OK;
}

int hlbm_set_state(hlbm_ctx* ctx, const void* words) {
  if (!ctx || !words) return fail(ctx, HLBM_EINVAL, "null argument");
  SETTLE(ctx);
  if (int r = copy_dense(ctx, const_cast<void*>(words), false)) return r;
  CK(launch_fill_ghosts(make_geo(ctx), ctx->NC, ctx->buf[ctx->cur], ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return HLBM_OK;
}

int hlbm_set_step_count(hlbm_ctx* ctx, int64_t step) {
  if (!ctx || step < 0) return fail(ctx, HLBM_EINVAL, "bad step");
  ctx->steps = step;   // the dither key of the next step (resume from a checkpoint)
  return HLBM_OK;
}

int hlbm_get_codes(hlbm_ctx* ctx, uint32_t* words) {
  if (!ctx || !words) return fail(ctx, HLBM_EINVAL, "null argument");
  if (!ctx->q16) return fail(ctx, HLBM_EINVAL, "codes exist only for the q16 precision");
  return hlbm_get_state(ctx, words);
}

int hlbm_set_codes(hlbm_ctx* ctx, const uint32_t* words) {
  if (!ctx || !words) return fail(ctx, HLBM_EINVAL, "null argument");
  if (!ctx->q16) return fail(ctx, HLBM_EINVAL, "codes exist only for the q16 precision");
  return hlbm_set_state(ctx, words);
}

int hlbm_set_mask(hlbm_ctx* ctx, const uint8_t* mask, const uint8_t* ghost_lo, const uint8_t* ghost_hi) {
  if (!ctx || !mask) return fail(ctx, HLBM_EINVAL, "null mask");
  SETTLE(ctx);
  const hlbm_config& c = ctx->cfg;
  const int64_t pl = (int64_t)c.ny * c.nz, n = pl * c.nx;
  // planes -1 .. nx of the padded mask along x (oracle/step.py:padded_solid)
  std::vector<uint8_t> ext((size_t)(n + 2 * pl));
  for (int64_t i = 0; i < n; ++i) ext[pl + i] = mask[i] ? 1 : 0;
  auto fill_ghost = [&](uint8_t* dst, const uint8_t* remote, int bc, bool lo) {
    if (remote) {
      for (int64_t i = 0; i < pl; ++i) dst[i] = remote[i] ? 1 : 0;
    } else if (bc == HLBM_BC_PERIODIC) {
      const uint8_t* src = ext.data() + pl + (lo ? (int64_t)(c.nx - 1) * pl : 0);
      memcpy(dst, src, pl);
    } else {
      memset(dst, bc == HLBM_BC_WALL ? 1 : 0, pl);
    }
  };
  fill_ghost(ext.data(), c.x_lo_remote ? ghost_lo : nullptr, c.bc[0], true);
  fill_ghost(ext.data() + pl + n, c.x_hi_remote ? ghost_hi : nullptr, c.bc[1], false);
  if ((c.x_lo_remote && !ghost_lo) || (c.x_hi_remote && !ghost_hi))
    return fail(ctx, HLBM_EINVAL, "remote x faces need the neighbour's ghost mask plane");

  free_mesh(ctx);
  cudaFree(ctx->d_bcells); ctx->d_bcells = nullptr;
  cudaFree(ctx->d_bmasks); ctx->d_bmasks = nullptr;
  cudaFree(ctx->d_scells); ctx->d_scells = nullptr;
  cudaFree(ctx->d_bits); ctx->d_bits = nullptr;
  ctx->nb = ctx->ns = 0;

  uint8_t *d_ext, *d_cls;
  uint32_t* d_links;
  int64_t *d_counts, *d_total;
  const int64_t nt = compact_tiles(n);
  CK(cudaMalloc(&d_ext, ext.size()));
  CK(cudaMalloc(&d_cls, n));
  CK(cudaMalloc(&d_links, n * 4));
  CK(cudaMalloc(&d_counts, (nt + 1) * 8));
  CK(cudaMalloc(&d_total, 8));
  CK(cudaMemcpy(d_ext, ext.data(), ext.size(), cudaMemcpyHostToDevice));
  MaskGeo mg{c.nx, c.ny, c.nz, c.bc[2] == HLBM_BC_WALL, c.bc[3] == HLBM_BC_WALL, c.bc[4] == HLBM_BC_WALL,
             c.bc[5] == HLBM_BC_WALL, ctx->q};
  CK(launch_classify(d_ext, mg, d_links, d_cls, ctx->stream));
  cudaFree(ctx->d_fused);
  ctx->d_fused = nullptr;
  CK(cudaMalloc(&ctx->d_fused, n * 4));
  CK(launch_fused_masks(d_links, d_cls, n, ctx->d_fused, ctx->stream));
  for (int pass = 0; pass < 2; ++pass) {
    const uint8_t want = pass == 0 ? 1 : 2;
    CK(launch_compact(d_cls, d_links, n, want, d_counts, d_total, nullptr, nullptr, true, ctx->stream));
    int64_t tot = 0;
    CK(cudaMemcpyAsync(&tot, d_total, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (tot > 0) {
      int64_t* cells;
      uint32_t* masks = nullptr;
      CK(cudaMalloc(&cells, tot * 8));
      if (pass == 0) CK(cudaMalloc(&masks, tot * 4));
      CK(launch_compact(d_cls, d_links, n, want, d_counts, d_total, cells, masks, false, ctx->stream));
      if (pass == 0) { ctx->d_bcells = cells; ctx->d_bmasks = masks; ctx->nb = tot; }
      else { ctx->d_scells = cells; ctx->ns = tot; }
    }
  }
  if (int r = plane_offsets(ctx, ctx->d_bcells, ctx->nb, ctx->off_b)) return r;
  if (int r = plane_offsets(ctx, ctx->d_scells, ctx->ns, ctx->off_s)) return r;
  ctx->off_m.clear();
  if (ctx->nb + ctx->ns > 0) {
    ctx->bits_row_words = (c.nz + 31) / 32;
    CK(cudaMalloc(&ctx->d_bits, (int64_t)c.nx * c.ny * ctx->bits_row_words * 4));
    CK(launch_special_bits(d_cls, c.nx, c.ny, c.nz, ctx->bits_row_words, ctx->d_bits, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_ext);
  cudaFree(d_cls);
  cudaFree(d_links);
  cudaFree(d_counts);
  cudaFree(d_total);
  return HLBM_OK;
}

int hlbm_set_solid_motion(hlbm_ctx* ctx, const double* motion) {
  if (!ctx) return HLBM_EINVAL;
  for (int k = 0; k < 3; ++k) {
    ctx->solid_v[k] = motion ? (float)motion[k] : 0.f;
    ctx->solid_w[k] = motion ? (float)motion[3 + k] : 0.f;
    ctx->solid_c[k] = motion ? (float)motion[6 + k] : 0.f;
  }
  ctx->solid_c[0] -= (float)ctx->cfg.x0;   // the kernels work in slab-local x
  return HLBM_OK;
}

int hlbm_set_mesh(hlbm_ctx* ctx, const double* vertices, int64_t nv, const int32_t* faces, int64_t nf,
                  const double* motion) {
  if (!ctx || nv < 0 || nf < 0 || (nv && !vertices) || (nf && !faces)) return fail(ctx, HLBM_EINVAL, "bad mesh");
  for (int64_t k = 0; k < 3 * nf; ++k)
    if (faces[k] < 0 || faces[k] >= nv) return fail(ctx, HLBM_EINVAL, "face index out of range");
  for (int64_t k = 0; k < 3 * nv; ++k)
    if (!std::isfinite(vertices[k])) return fail(ctx, HLBM_EINVAL, "non-finite vertex");
  const hlbm_config& c = ctx->cfg;
  // wall faces: their links come from the voxel classifier on an all-fluid mask (round 1 dropped
  // them here silently); the list becomes the union of mesh-cut and wall-adjacent cells
  std::vector<int64_t> wcells;
  std::vector<uint32_t> wmasks;
  bool wall = false;
  for (int f = 0; f < 6; ++f) wall = wall || c.bc[f] == HLBM_BC_WALL;
  if (wall) {
    const int64_t pl = (int64_t)c.ny * c.nz;
    std::vector<uint8_t> zero((size_t)(pl * c.nx), 0);
    if (int r = hlbm_set_mask(ctx, zero.data(), zero.data(), zero.data())) return r;
    wcells.resize((size_t)ctx->nb);
    wmasks.resize((size_t)ctx->nb);
    if (ctx->nb) {
      CK(cudaMemcpy(wcells.data(), ctx->d_bcells, ctx->nb * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(wmasks.data(), ctx->d_bmasks, ctx->nb * 4, cudaMemcpyDeviceToHost));
    }
  }
  // the mesh replaces any voxel lists
  cudaFree(ctx->d_fused); ctx->d_fused = nullptr;
  cudaFree(ctx->d_bcells); ctx->d_bcells = nullptr;
  cudaFree(ctx->d_bmasks); ctx->d_bmasks = nullptr;
  cudaFree(ctx->d_scells); ctx->d_scells = nullptr;
  cudaFree(ctx->d_bits); ctx->d_bits = nullptr;
  ctx->nb = ctx->ns = 0;
  free_mesh(ctx);
  hlbm_set_solid_motion(ctx, motion);
  std::vector<double> V((size_t)3 * nv);
  for (int64_t k = 0; k < nv; ++k) {
    V[3 * k] = vertices[3 * k] - (double)c.x0;   // slab-local x
    V[3 * k + 1] = vertices[3 * k + 1];
    V[3 * k + 2] = vertices[3 * k + 2];
  }
  double* dV = nullptr;
  int* dF = nullptr;
  if (nf > 0) {
    CK(cudaMalloc(&dV, V.size() * 8));
    CK(cudaMalloc(&dF, (size_t)3 * nf * 4));
    CK(cudaMemcpy(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dF, faces, (size_t)3 * nf * 4, cudaMemcpyHostToDevice));
    CK(build_mesh_links(dV, dF, (int)nf, c.nx, c.ny, c.nz, ctx->mesh, ctx->stream, ctx->q));
    cudaFree(dV);
    cudaFree(dF);
  }
  if (!wcells.empty()) {   // merge the wall-adjacent cells into the (sorted) cut-link list
    const int64_t nm = ctx->mesh.nb;
    std::vector<int64_t> mc((size_t)nm);
    std::vector<uint32_t> mm((size_t)nm);
    std::vector<double> mt((size_t)nm * 27);
    std::vector<int> mtri((size_t)nm * 27);
    if (nm) {
      CK(cudaMemcpy(mc.data(), ctx->mesh.cells, nm * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(mm.data(), ctx->mesh.masks, nm * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(mt.data(), ctx->mesh.t64, nm * 27 * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(mtri.data(), ctx->mesh.tri, nm * 27 * 4, cudaMemcpyDeviceToHost));
    }
    std::vector<int64_t> uc;
    std::vector<uint32_t> um, uw;
    std::vector<double> ut;
    std::vector<int> utri;
    size_t i = 0, j = 0;
    while (i < mc.size() || j < wcells.size()) {
      const bool takem = j >= wcells.size() || (i < mc.size() && mc[i] <= wcells[j]);
      const bool takew = i >= mc.size() || (j < wcells.size() && wcells[j] <= mc[i]);
      uc.push_back(takem ? mc[i] : wcells[j]);
      um.push_back(takem ? mm[i] : 0u);
      uw.push_back(takew ? wmasks[j] : 0u);
      for (int k = 0; k < 27; ++k) {
        ut.push_back(takem ? mt[i * 27 + k] : std::nan(""));
        utri.push_back(takem ? mtri[i * 27 + k] : -1);
      }
      if (takem) ++i;
      if (takew) ++j;
    }
    free_mesh(ctx);
    const int64_t nu = (int64_t)uc.size();
    std::vector<float> ut32(ut.size());
    for (size_t k = 0; k < ut.size(); ++k) ut32[k] = (float)ut[k];
    CK(cudaMalloc(&ctx->mesh.cells, nu * 8));
    CK(cudaMalloc(&ctx->mesh.masks, nu * 4));
    CK(cudaMalloc(&ctx->mesh.wmasks, nu * 4));
    CK(cudaMalloc(&ctx->mesh.t64, nu * 27 * 8));
    CK(cudaMalloc(&ctx->mesh.t32, nu * 27 * 4));
    CK(cudaMalloc(&ctx->mesh.tri, nu * 27 * 4));
    CK(cudaMemcpy(ctx->mesh.cells, uc.data(), nu * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->mesh.masks, um.data(), nu * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->mesh.wmasks, uw.data(), nu * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->mesh.t64, ut.data(), nu * 27 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->mesh.t32, ut32.data(), nu * 27 * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->mesh.tri, utri.data(), nu * 27 * 4, cudaMemcpyHostToDevice));
    ctx->mesh.nb = nu;
  }
  ctx->off_b.clear();
  ctx->off_s.clear();
  if (int r = plane_offsets(ctx, ctx->mesh.cells, ctx->mesh.nb, ctx->off_m)) return r;
  if (ctx->mesh.nb > 0) {
    ctx->bits_row_words = (c.nz + 31) / 32;
    const int64_t nw = (int64_t)c.nx * c.ny * ctx->bits_row_words;
    CK(cudaMalloc(&ctx->d_bits, nw * 4));
    CK(cudaMemsetAsync(ctx->d_bits, 0, nw * 4, ctx->stream));
    CK(launch_bits_from_list(ctx->mesh.cells, ctx->mesh.nb, c.nz, ctx->bits_row_words, ctx->d_bits, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return HLBM_OK;
}

int hlbm_get_cut_links(hlbm_ctx* ctx, int64_t* cells, uint32_t* masks, double* t, int32_t* tri, int64_t* n) {
  if (!ctx || !n) return fail(ctx, HLBM_EINVAL, "null argument");
  if (ctx->mesh.wmasks) {   // union list (mesh + wall faces): report the mesh-cut entries only
    const int64_t nu = ctx->mesh.nb;
    std::vector<int64_t> uc((size_t)nu);
    std::vector<uint32_t> um((size_t)nu);
    CK(cudaStreamSynchronize(ctx->stream));
    if (nu) {
      CK(cudaMemcpy(uc.data(), ctx->mesh.cells, nu * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(um.data(), ctx->mesh.masks, nu * 4, cudaMemcpyDeviceToHost));
    }
    int64_t cnt = 0;
    for (int64_t i = 0; i < nu; ++i) cnt += um[(size_t)i] != 0;
    if (!cells) { *n = cnt; return HLBM_OK; }
    if (*n < cnt) return fail(ctx, HLBM_EINVAL, "output buffer too small");
    *n = cnt;
    std::vector<double> ut((size_t)nu * 27);
    std::vector<int> utri((size_t)nu * 27);
    if (nu && t) CK(cudaMemcpy(ut.data(), ctx->mesh.t64, nu * 27 * 8, cudaMemcpyDeviceToHost));
    if (nu && tri) CK(cudaMemcpy(utri.data(), ctx->mesh.tri, nu * 27 * 4, cudaMemcpyDeviceToHost));
    const int64_t off = (int64_t)ctx->cfg.x0 * ctx->cfg.ny * ctx->cfg.nz;
    int64_t o = 0;
    for (int64_t i = 0; i < nu; ++i) {
      if (!um[(size_t)i]) continue;
      cells[o] = uc[(size_t)i] + off;
      if (masks) masks[o] = um[(size_t)i];
      for (int k = 0; k < 27; ++k) {
        if (t) t[o * 27 + k] = ut[(size_t)i * 27 + k];
        if (tri) tri[o * 27 + k] = utri[(size_t)i * 27 + k];
      }
      ++o;
    }
    return HLBM_OK;
  }
  const int64_t nb = ctx->mesh.nb;
  if (!cells) { *n = nb; return HLBM_OK; }
  CK(cudaStreamSynchronize(ctx->stream));
  if (*n < nb) return fail(ctx, HLBM_EINVAL, "output buffer too small");
  *n = nb;
  if (nb == 0) return HLBM_OK;
  CK(cudaMemcpy(cells, ctx->mesh.cells, nb * 8, cudaMemcpyDeviceToHost));
  if (masks) CK(cudaMemcpy(masks, ctx->mesh.masks, nb * 4, cudaMemcpyDeviceToHost));
  if (t) CK(cudaMemcpy(t, ctx->mesh.t64, nb * 27 * 8, cudaMemcpyDeviceToHost));
  if (tri) CK(cudaMemcpy(tri, ctx->mesh.tri, nb * 27 * 4, cudaMemcpyDeviceToHost));
  const int64_t off = (int64_t)ctx->cfg.x0 * ctx->cfg.ny * ctx->cfg.nz;
  for (int64_t i = 0; i < nb; ++i) cells[i] += off;
  return HLBM_OK;
}

int hlbm_get_boundary(hlbm_ctx* ctx, int64_t* cells, uint32_t* masks, int64_t* n) {
  if (!ctx || !n) return fail(ctx, HLBM_EINVAL, "null argument");
  if (!cells) { *n = ctx->nb; return HLBM_OK; }
  if (*n < ctx->nb) return fail(ctx, HLBM_EINVAL, "output buffer too small");
  *n = ctx->nb;
  if (ctx->nb == 0) return HLBM_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(cells, ctx->d_bcells, ctx->nb * 8, cudaMemcpyDeviceToHost));
  if (masks) CK(cudaMemcpy(masks, ctx->d_bmasks, ctx->nb * 4, cudaMemcpyDeviceToHost));
  // local -> global linear index
  const int64_t off = (int64_t)ctx->cfg.x0 * ctx->cfg.ny * ctx->cfg.nz;
  for (int64_t i = 0; i < ctx->nb; ++i) cells[i] += off;
  return HLBM_OK;
}

int hlbm_fluid_update(hlbm_ctx* ctx, int32_t with_stats) {
  if (!ctx) return HLBM_EINVAL;
  SETTLE(ctx);
  if (with_stats) CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (int r = run_range(ctx, 0, ctx->cfg.nx, with_stats, ctx->ev[1], nullptr, kPhaseFluid)) return r;
  ctx->pending_stats = with_stats ? 1 : 0;
  const bool special = ctx->nb + ctx->ns + ctx->mesh.nb > 0;
  if (special) {
    ctx->pending_solid = 1;
    return HLBM_OK;
  }
  CK(cudaEventRecord(ctx->ev[2], ctx->stream));   // no obstacles: the step is complete
  ctx->cur = 1 - ctx->cur;
  ++ctx->steps;
  ctx->pending_stats = 0;
  return HLBM_OK;
}

int hlbm_solid_correction(hlbm_ctx* ctx, hlbm_stats* out) {
  if (!ctx) return HLBM_EINVAL;
  if (ctx->pending_solid) {
    if (int r = run_range(ctx, 0, ctx->cfg.nx, ctx->pending_stats, nullptr, nullptr, kPhaseSolid)) return r;
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    ctx->pending_solid = 0;
    ctx->cur = 1 - ctx->cur;
    ++ctx->steps;
  }
  if (!out) return HLBM_OK;
  const int had_stats = ctx->pending_stats;
  ctx->pending_stats = 0;
  CK(cudaStreamSynchronize(ctx->stream));
  float a = 0.f, b = 0.f;
  cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
  ctx->last_t_fluid = a;
  ctx->last_t_solid = b;
  if (!had_stats) {
    memset(out, 0, sizeof(*out));
    out->step = ctx->steps;
    out->t_fluid_ms = a;
    out->t_solid_ms = b;
    out->finite = 1;
    return HLBM_OK;
  }
  return hlbm_read_stats(ctx, out);
}

int hlbm_stream(hlbm_ctx* ctx) {
  if (!ctx) return HLBM_EINVAL;
  SETTLE(ctx);
  if (ctx->cfg.x_lo_remote || ctx->cfg.x_hi_remote) return fail(ctx, HLBM_EINVAL, "single domain only");
  if (int r = mesh_dense(ctx)) return r;
  StepArgs A = make_args(ctx, 0);
  CK(launch_alg1(A, ctx->d_fused, ctx->q16, false, ctx->q16 && ctx->cfg.dither, ctx->q, ctx->stream, false,
                 ctx->mesh.dense, ctx->mesh.masks));
  ++ctx->launches;
  if (ctx->cfg.ny == 1) CK(launch_fill_ghosts(make_geo(ctx), ctx->NC, ctx->buf[1 - ctx->cur], ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->cur = 1 - ctx->cur;
  return HLBM_OK;
}

int hlbm_step_async(hlbm_ctx* ctx, int32_t nsteps, int32_t with_stats) {
  if (!ctx || nsteps < 0) return fail(ctx, HLBM_EINVAL, "bad arguments");
  SETTLE(ctx);
  for (int s = 0; s < nsteps; ++s) {
    const int st = (with_stats && s == nsteps - 1) ? 1 : 0;
    if (st) CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
    if (int r = run_range(ctx, 0, ctx->cfg.nx, st)) return r;
    ctx->cur = 1 - ctx->cur;
    ++ctx->steps;
  }
  return HLBM_OK;
}

int hlbm_step_begin(hlbm_ctx* ctx, int32_t with_stats) {
  if (!ctx) return HLBM_EINVAL;
  SETTLE(ctx);
  ctx->pending_stats = with_stats ? 1 : 0;
  if (with_stats) CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
  return HLBM_OK;
}

int hlbm_step_range(hlbm_ctx* ctx, int32_t x_begin, int32_t x_end) {
  return hlbm_step_range_on(ctx, x_begin, x_end, nullptr);
}

int hlbm_step_range_on(hlbm_ctx* ctx, int32_t x_begin, int32_t x_end, void* stream) {
  if (!ctx) return HLBM_EINVAL;
  if (x_begin < 0 || x_end > ctx->cfg.nx || x_begin > x_end) return fail(ctx, HLBM_EINVAL, "bad x range");
  return run_range(ctx, x_begin, x_end, ctx->pending_stats, nullptr, (cudaStream_t)stream);
}

int hlbm_step_end(hlbm_ctx* ctx) {
  if (!ctx) return HLBM_EINVAL;
  ctx->cur = 1 - ctx->cur;
  ++ctx->steps;
  ctx->pending_stats = 0;
  return HLBM_OK;
}

int hlbm_step_reference(hlbm_ctx* ctx, int32_t nsteps) {
  if (!ctx || nsteps < 0) return fail(ctx, HLBM_EINVAL, "bad arguments");
  SETTLE(ctx);
  const bool q16 = ctx->q16, force = has_force(ctx), dither = q16 && ctx->cfg.dither;
  const int64_t n = (int64_t)ctx->cfg.nx * ctx->cfg.ny * ctx->cfg.nz;
  for (int s = 0; s < nsteps; ++s) {
    StepArgs A = make_args(ctx, 0);
    CK(launch_pull_cells(A, nullptr, nullptr, n, 0, q16, force, dither, ctx->stream, ctx->q));
    ++ctx->launches;
    if (ctx->nb) {
      CK(launch_pull_cells(A, ctx->d_bcells, ctx->d_bmasks, ctx->nb, 0, q16, force, dither, ctx->stream, ctx->q));
      ++ctx->launches;
    }
    if (ctx->ns) {
      CK(launch_pull_cells(A, ctx->d_scells, nullptr, ctx->ns, 1, q16, force, dither, ctx->stream, ctx->q));
      ++ctx->launches;
    }
    if (ctx->mesh.nb) {
      CK(launch_pull_cells(A, ctx->mesh.cells, ctx->mesh.masks, ctx->mesh.nb, 2, q16, force, dither, ctx->stream, ctx->q));
      ++ctx->launches;
    }
    ctx->cur = 1 - ctx->cur;
    ++ctx->steps;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return HLBM_OK;
}

int hlbm_step_percell(hlbm_ctx* ctx, int32_t nsteps, hlbm_stats* out) {
  if (!ctx || nsteps < 0) return fail(ctx, HLBM_EINVAL, "bad arguments");
  SETTLE(ctx);
  if (ctx->mesh.nb) return fail(ctx, HLBM_EINVAL, "the per-cell step supports voxel solids only");
  const bool q16 = ctx->q16, force = has_force(ctx), dither = q16 && ctx->cfg.dither;
  const int64_t n = (int64_t)ctx->cfg.nx * ctx->cfg.ny * ctx->cfg.nz;
  float tf = 0.f;
  for (int s = 0; s < nsteps; ++s) {
    const int st = (s == nsteps - 1) ? 1 : 0;
    if (st) CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
    StepArgs A = make_args(ctx, st);
    CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    CK(launch_pull_cells(A, nullptr, ctx->d_fused, n, 3, q16, force, dither, ctx->stream, ctx->q));
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    ++ctx->launches;
    CK(cudaEventSynchronize(ctx->ev[1]));
    float a = 0.f;
    cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
    tf += a;
    ctx->cur = 1 - ctx->cur;
    ++ctx->steps;
  }
  if (nsteps == 0) return HLBM_OK;
  ctx->last_t_fluid = tf / nsteps;
  ctx->last_t_solid = 0.0;
  return hlbm_read_stats(ctx, out);
}

// the original HOME-LBM step (Alg. 1): post-collision storage cut, 8^3 tiles with
// shared-memory streaming, voxel solid links inline (hlbm_cells.cu alg1_step)
int hlbm_step_fused(hlbm_ctx* ctx, int32_t nsteps, hlbm_stats* out) {
  if (!ctx || nsteps < 0) return fail(ctx, HLBM_EINVAL, "bad arguments");
  SETTLE(ctx);
  if (ctx->cfg.x_lo_remote || ctx->cfg.x_hi_remote)
    return fail(ctx, HLBM_EINVAL, "the fused Alg.-1 step runs on a single domain");
  if (int r = mesh_dense(ctx)) return r;
  const bool q16 = ctx->q16, force = has_force(ctx), dither = q16 && ctx->cfg.dither;
  float tf = 0.f;
  for (int s = 0; s < nsteps; ++s) {
    const int st = (s == nsteps - 1) ? 1 : 0;
    if (st) CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
    StepArgs A = make_args(ctx, st);
    CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    CK(launch_alg1(A, ctx->d_fused, q16, force, dither, ctx->q, ctx->stream, true, ctx->mesh.dense,
                   ctx->mesh.masks));
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    ++ctx->launches;
    if (ctx->cfg.ny == 1) {   // one-row slab: both ghost rows hold the edge row's image
      CK(launch_fill_ghosts(make_geo(ctx), ctx->NC, ctx->buf[1 - ctx->cur], ctx->stream));
      ++ctx->launches;
    }
    CK(cudaEventSynchronize(ctx->ev[1]));
    float a = 0.f;
    cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
    tf += a;
    ctx->cur = 1 - ctx->cur;
    ++ctx->steps;
  }
  if (nsteps == 0) return HLBM_OK;
  ctx->last_t_fluid = tf / nsteps;
  ctx->last_t_solid = 0.0;
  return hlbm_read_stats(ctx, out);
}

// StepStats from the host copy of the device accumulators (ctx->h_stats, already synchronised)
static int stats_from_host(hlbm_ctx* ctx, hlbm_stats* out) {
  const Stats& h = *ctx->h_stats;
  const hlbm_config& c = ctx->cfg;
  const int64_t nfluid = (int64_t)c.nx * c.ny * c.nz - ctx->ns;
  float mu2;
  memcpy(&mu2, &h.max_u2_bits, 4);
  hlbm_stats s{};
  s.step = ctx->steps;
  s.t_fluid_ms = ctx->last_t_fluid;
  s.t_copy_ms = 0.0;
  s.t_solid_ms = ctx->last_t_solid;
  s.mass = (double)nfluid + h.mass_dev;
  for (int k = 0; k < 3; ++k) s.momentum[k] = h.mom[k];
  s.max_u = std::sqrt((double)mu2);
  for (int k = 0; k < 10; ++k) s.saturation[k] = (int64_t)h.sat[k];
  s.n_fluid = nfluid;
  for (int k = 0; k < 3; ++k) {
    s.force[k] = h.force[k];
    s.torque[k] = h.torque[k];
  }
  s.finite = std::isfinite(s.mass) && std::isfinite(s.momentum[0]) && std::isfinite(s.momentum[1]) &&
             std::isfinite(s.momentum[2]) && std::isfinite(s.max_u);
  if (out) *out = s;
  if (s.finite && s.max_u < 0.9) return HLBM_OK;
  // divergence ("divergence report with step and node"): locate the node in the state
  // the step wrote -- a scan that runs only here, never on the hot path
  std::string where;
  if (staging(ctx, 8) == HLBM_OK) {
    unsigned long long key = 0;
    StepArgs A = make_args(ctx, 0);
    A.in = ctx->buf[ctx->cur];
    if (launch_locate(A, ctx->q16, reinterpret_cast<unsigned long long*>(ctx->d_stage), ctx->stream) == cudaSuccess &&
        cudaMemcpyAsync(&key, ctx->d_stage, 8, cudaMemcpyDeviceToHost, ctx->stream) == cudaSuccess &&
        cudaStreamSynchronize(ctx->stream) == cudaSuccess) {
      const int64_t i = (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull));
      const int64_t yz = (int64_t)c.ny * c.nz;
      const uint32_t bits = (uint32_t)(key >> 32);
      float u2;
      memcpy(&u2, &bits, 4);
      char buf[160];
      snprintf(buf, sizeof buf, " at step %lld, node (%lld, %lld, %lld)%s", (long long)s.step,
               (long long)(c.x0 + i / yz), (long long)((i % yz) / c.nz), (long long)(i % c.nz),
               bits == 0xFFFFFFFFu ? " (non-finite)" : "");
      where = buf;
      if (bits != 0xFFFFFFFFu) {
        snprintf(buf, sizeof buf, ", |u| = %.4g", std::sqrt((double)u2));
        where += buf;
      }
    }
  }
  if (!s.finite) return fail(ctx, HLBM_EDIVERGED, "non-finite moment detected (solver divergence)" + where);
  return fail(ctx, HLBM_EDIVERGED, "max |u| reached 0.9 (solver divergence)" + where);
}

int hlbm_read_stats(hlbm_ctx* ctx, hlbm_stats* out) {
  if (!ctx) return HLBM_EINVAL;
  CK(cudaMemcpyAsync(ctx->h_stats, ctx->d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return stats_from_host(ctx, out);
}

// n steps; the statistics (and the phase times t_fluid / t_solid) are those of the last step.
// One host synchronisation per call: the stats copy is enqueued behind the last kernel.
int hlbm_step(hlbm_ctx* ctx, int32_t nsteps, hlbm_stats* out) {
  if (!ctx || nsteps < 0) return fail(ctx, HLBM_EINVAL, "bad arguments");
  SETTLE(ctx);
  if (nsteps == 0) {
    if (out) { memset(out, 0, sizeof(*out)); out->step = ctx->steps; out->finite = 1; }
    return HLBM_OK;
  }
  for (int s = 0; s < nsteps; ++s) {
    const bool last = s == nsteps - 1;
    if (last) {
      CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
      CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    }
    if (int r = run_range(ctx, 0, ctx->cfg.nx, last ? 1 : 0, last ? ctx->ev[1] : nullptr)) return r;
    if (last) CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    ctx->cur = 1 - ctx->cur;
    ++ctx->steps;
  }
  CK(cudaMemcpyAsync(ctx->h_stats, ctx->d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  float a = 0.f, b = 0.f;
  cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
  ctx->last_t_fluid = a;
  ctx->last_t_solid = b;
  return stats_from_host(ctx, out);
}

}  // extern "C"
