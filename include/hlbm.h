/* hlbm.h -- C-ABI of the B200 HOME-LBM fluid step (libhlbm.so).
 *
 * Drop-in boundary for the reference package's solver path.  The reference
 * (/root/reference/pkg/src/momentlbm) is pure Python and ships the step's arithmetic
 * as NumPy array functions; its solver surface (SimGrid / SolverConfig / StepStats /
 * fluid_update_step / run) is specified in SPEC.md:446-516 but not shipped.  The
 * Python host layer (paper_2602_05295_b200.solver) binds these entry points with
 * ctypes; INTEGRATION.md shows the binding.  Each entry point cites the reference
 * interface it replaces.
 *
 * Conventions: plain pointers and sizes; the library owns all device memory; host
 * arrays are caller-owned and copied.  Every call returns HLBM_OK (0) or an error code;
 * hlbm_last_error() holds the message.  A context is driven by one host thread.
 * Array layout = the reference's (moments.py:11-13): component axis first, then
 * (x, y, z) in C order, float64; stress in Voigt order xx,xy,xz,yy,yz,zz (lattice.py:23).
 */
#ifndef HLBM_H
#define HLBM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HLBM_OK 0
#define HLBM_EINVAL 1      /* -> ValueError (moments.py:33-34; collision.py:102-103,203-204) */
#define HLBM_EDIVERGED 2   /* -> FloatingPointError (collision.py:207-208)      */
#define HLBM_ECUDA 3       /* -> RuntimeError                                               */

#define HLBM_BC_PERIODIC 0
#define HLBM_BC_INFLOW 1
#define HLBM_BC_OUTFLOW 2
#define HLBM_BC_WALL 3

#define HLBM_FP32 0
#define HLBM_Q16 1

typedef struct hlbm_ctx hlbm_ctx;

/* SolverConfig + SimGrid dims + QuantSpec.
 * ABI guard: the caller sets struct_size = sizeof(hlbm_config) (hlbm_config_init does); hlbm_create
 * rejects any other value with HLBM_EINVAL before reading past the first field, so a binding built
 * against a different layout fails loudly instead of reading garbage. */
typedef struct hlbm_config {
  int32_t struct_size;         /* sizeof(hlbm_config) of the caller's layout (352 bytes here)   */
  int32_t nx, ny, nz;          /* local interior dims of this slab (x is the slab axis)       */
  int32_t gnx, gny, gnz;       /* global dims (== local on one GPU)                           */
  int32_t x0;                  /* slab offset along x in the global grid                      */
  int32_t x_lo_remote;         /* 1: x- ghost plane is filled by the caller (neighbour slab)  */
  int32_t x_hi_remote;         /* 1: x+ ghost plane is filled by the caller                   */
  double tau;                  /* relaxation time, tau = 0.5 + 3 nu (collision.py:30-31)      */
  double force[3];             /* uniform body force (collision.py:137-194 `force`)           */
  int32_t bc[6];               /* x-,x+,y-,y+,z-,z+ : HLBM_BC_*               */
  double u_in[3];              /* inflow velocity                                             */
  int32_t precision;           /* HLBM_FP32 or HLBM_Q16                                       */
  double qmin[10], qmax[10];   /* codec ranges (rho, rho u_xyz, sneq xx..zz) */
  int32_t bits[10];            /* bits per component, 2..16                 */
  int32_t dither;              /* 1: counter-hash dither                         */
  uint32_t seed;
  int32_t device;              /* CUDA device ordinal                                         */
  int32_t xseg;                /* interior-kernel x segment length (0 = default)              */
  int32_t q;                   /* velocity set: 27 (D3Q27, default when 0) or 19 (D3Q19:
                                  two-chain interior kernel + 19-link compacted kernels; voxel
                                  solids only; lattice.py:172-211)                               */
} hlbm_config;

/* StepStats. Sums run over fluid cells of this slab. */
typedef struct hlbm_stats {
  int64_t step;
  double t_fluid_ms, t_copy_ms, t_solid_ms;   /* device times of the last step of the call */
  double mass;
  double momentum[3];
  double max_u;
  int64_t saturation[10];
  int64_t n_fluid;
  int32_t finite;
  double force[3];             /* triangle mesh: momentum exchange on the solid */
  double torque[3];
} hlbm_stats;

const char* hlbm_version(void);
/* defaults: struct_size, periodic faces, fp32, the default QuantSpec ranges and
 * 16 bits per component, D3Q27, device 0; the caller then sets dims and tau */
void hlbm_config_init(hlbm_config* cfg);
/* number of visible CUDA devices (0 when no driver / GPU) */
int hlbm_device_count(void);

/* SimGrid + SolverConfig construction.  Validates tau > 1/2
 * (collision.py:102-103, 203-204) and the grid (nz % 4 == 0). */
int hlbm_create(const hlbm_config* cfg, hlbm_ctx** out);
void hlbm_destroy(hlbm_ctx* ctx);
const char* hlbm_last_error(const hlbm_ctx* ctx);

/* Voxel solid mask, uint8 (nx,ny,nz) C order.  ghost_lo / ghost_hi: the (ny,nz) mask planes of
 * the neighbouring slabs for remote faces (NULL: derived from the x BC).  Builds the sorted
 * boundary-cell list and 27-bit link masks on the device (SPEC.md:400-402 SurfaceMask role). */
int hlbm_set_mask(hlbm_ctx* ctx, const uint8_t* mask, const uint8_t* ghost_lo, const uint8_t* ghost_hi);

/* Static triangle mesh (lattice coordinates of this slab's global grid): vertices (nv,3) float64,
 * faces (nf,3) int32; motion = {v[3], omega[3], center[3]} of the rigid body (NULL: at rest).
 * Precomputes the cut-link list (earliest hit per pull link x -> x - c_i)
 * and makes the compacted kernel apply the Eq.-8 boundary populations.
 * Replaces any voxel mask. */
int hlbm_set_mesh(hlbm_ctx* ctx, const double* vertices, int64_t nv, const int32_t* faces, int64_t nf,
                  const double* motion);
int hlbm_set_solid_motion(hlbm_ctx* ctx, const double* motion);
/* cut links: global cells (sorted), 27-bit masks, t (n,27) float64 (NaN uncut), triangle (n,27) */
int hlbm_get_cut_links(hlbm_ctx* ctx, int64_t* cells, uint32_t* masks, double* t, int32_t* tri, int64_t* n);

/* State in the reference layout: rho (nx,ny,nz), mom (3,nx,ny,nz), stress (6,nx,ny,nz) float64
 * (moments.py:25-39 outputs; MomentSet fields moments.py:136-172). */
int hlbm_set_moments(hlbm_ctx* ctx, const double* rho, const double* mom, const double* stress);
int hlbm_get_moments(hlbm_ctx* ctx, double* rho, double* mom, double* stress);
/* box [x0,x0+cx) x [y0,y0+cy) x [z0,z0+cz) of the slab interior (y, z wrap periodically) */
int hlbm_get_moments_box(hlbm_ctx* ctx, int32_t x0, int32_t cx, int32_t y0, int32_t cy, int32_t z0,
                         int32_t cz, double* rho, double* mom, double* stress);
/* rho = rho0, u = sum_m a_m sin(2 pi k_m.x/N + phi_m), sneq = 0; modes: nmodes x 7 doubles */
int hlbm_init_modes(hlbm_ctx* ctx, double rho0, const double* modes, int32_t nmodes);

/* fluid_update_step x nsteps: interior kernel over every cell, then the
 * compacted boundary/solid kernel; blocks until done and fills *out (may be NULL). Returns
 * HLBM_EDIVERGED when max|u| >= 0.9 or a non-finite value appeared; hlbm_last_error
 * then names the step and the node of largest |u| (non-finite first) of the state the step wrote
 * (SPEC.md:467), found by a scan that runs only on divergence. */
int hlbm_step(hlbm_ctx* ctx, int32_t nsteps, hlbm_stats* out);
/* SPEC's split step as two calls (Alg. 2 / Alg. 3 roles):
 * hlbm_fluid_update runs the interior kernel over every cell (no obstacle logic); with obstacles the
 * step stays uncommitted until hlbm_solid_correction runs the compacted boundary / solid / cut-link
 * kernels on the same output buffer (any other state access runs it implicitly).  Without
 * obstacles hlbm_fluid_update commits the step and hlbm_solid_correction is the identity.
 * hlbm_solid_correction fills *out (may be NULL) with the step's StepStats and phase times. */
int hlbm_fluid_update(hlbm_ctx* ctx, int32_t with_stats);
int hlbm_solid_correction(hlbm_ctx* ctx, hlbm_stats* out);
/* the streaming operator S alone (reconstruct the stored moments, pull-stream with the BC and
 * voxel bounce-back / mesh Eq.-8 rules, extract; no collision): converts an Alg.-1 state (post-collision) to
 * the split scheme's storage cut, (S o C)^n o S = S o (C o S)^n.  Not a time step. */
int hlbm_stream(hlbm_ctx* ctx);
/* the same launches, enqueued on the context stream without synchronising */
int hlbm_step_async(hlbm_ctx* ctx, int32_t nsteps, int32_t with_stats);
int hlbm_read_stats(hlbm_ctx* ctx, hlbm_stats* out);
/* full-grid update with the per-cell pull kernel (GPU reference for the fast kernel) */
int hlbm_step_reference(hlbm_ctx* ctx, int32_t nsteps);
/* per-cell gather step: one thread per cell of the slab pulls its 27 (19) sources, each
 * re-evaluating the source's collision and reconstruction, voxel solid links inline; the same
 * Alg.-2 storage cut as hlbm_step (the GPU cross-check of the split kernels, and the D3Q19 path of
 * non-default codecs).  Voxel solids only. */
int hlbm_step_percell(hlbm_ctx* ctx, int32_t nsteps, hlbm_stats* out);
/* the original HOME-LBM step (Alg. 1): the stored state is the
 * POST-collision moments; each node reconstructs its own populations into shared memory (8^3
 * tiles + halo), streams from its neighbours there (solid links: bounce-back inline), extracts,
 * collides and writes back.  The in-repo baseline of the split-scheme attribution
 * (PAPER.md:418-429).  Related to hlbm_step by the half-step alignment (S o C)^n o S = S o (C o S)^n
 * (SPEC.md:495).  Voxel solids, or a triangle mesh (a cut link takes the Eq.-8 population built
 * from the node's own stored post-collision moments); single domain. */
int hlbm_step_fused(hlbm_ctx* ctx, int32_t nsteps, hlbm_stats* out);

/* boundary list: global linear cell indices (sorted) and link masks; cells==NULL -> count only */
int hlbm_get_boundary(hlbm_ctx* ctx, int64_t* cells, uint32_t* masks, int64_t* n);
/* raw packed words of the q16 state, (5,nx,ny,nz) uint32 (SPEC.md:381 packed-buffer dump) */
int hlbm_get_codes(hlbm_ctx* ctx, uint32_t* words);
int hlbm_set_codes(hlbm_ctx* ctx, const uint32_t* words);
/* raw internal state, dense (NC,nx,ny,nz) 32-bit words: fp32 (rho-1, rho u, sneq) or q16 words;
 * with hlbm_set_step_count this is an exact checkpoint/resume */
int hlbm_get_state(hlbm_ctx* ctx, void* words);
int hlbm_set_state(hlbm_ctx* ctx, const void* words);
int hlbm_set_step_count(hlbm_ctx* ctx, int64_t step);

/* multi-GPU plumbing: run on an external stream (e.g. torch's), and expose the device planes
 * that the x-slab halo exchange sends/receives for the CURRENT state buffer. */
int hlbm_set_stream(hlbm_ctx* ctx, void* cuda_stream);
int hlbm_halo_planes(hlbm_ctx* ctx, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                     int64_t* bytes);
/* the same planes of the NEXT state buffer (the one the step in progress writes): the overlapped
 * schedule sends a step's edge planes while the bulk of that step is still being computed */
int hlbm_next_halo_planes(hlbm_ctx* ctx, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                          int64_t* bytes);
/* peer-store halo between processes: instead of a send/receive
 * pair, each rank copies its freshly written edge planes straight into its neighbours' ghost
 * planes through CUDA IPC mappings (NVLink peer memory across GPUs).
 *   hlbm_ipc_export : the cudaIpcMemHandle_t of both state buffers (2 x 64 bytes) and the
 *                     current buffer index, to be passed to the neighbours
 *   hlbm_ipc_open   : map a neighbour's buffers; side 0 = the x-lo neighbour, 1 = x-hi;
 *                     peer_nx = its interior planes, peer_cur = its current buffer index
 *   hlbm_ipc_sync   : re-align after a rank replaced its state (its current index changed)
 *   hlbm_halo_push  : enqueue on `cuda_stream` (NULL: the context's) the copies of our first /
 *                     last interior plane -- of the buffer the step in progress writes when
 *                     next_buffer, else of the current one -- into the lo / hi neighbour's hi / lo
 *                     ghost plane of the matching buffer.  The caller orders it against the
 *                     neighbours' steps (interprocess events; paper_2602_05295_b200/distributed.py)
 *   hlbm_ipc_close  : unmap (also done by hlbm_destroy)
 * The reference has no multi-GPU path; this replaces nothing there. */
int hlbm_ipc_export(hlbm_ctx* ctx, void* handles, int32_t* cur);
int hlbm_ipc_open(hlbm_ctx* ctx, int32_t side, const void* handles, int32_t peer_nx, int32_t peer_cur);
int hlbm_ipc_sync(hlbm_ctx* ctx, int32_t side, int32_t peer_cur);
int hlbm_halo_push(hlbm_ctx* ctx, int32_t next_buffer, void* cuda_stream);
int hlbm_ipc_close(hlbm_ctx* ctx);
/* one step split into x-ranges (edge planes first, bulk later): step_begin resets
 * the statistics when with_stats, step_range enqueues the interior + boundary kernels for the
 * destination planes [x_begin, x_end) of the slab, step_end makes the written buffer current.
 * Ranges of one step must be disjoint; their union must be [0, nx). */
int hlbm_step_begin(hlbm_ctx* ctx, int32_t with_stats);
int hlbm_step_range(hlbm_ctx* ctx, int32_t x_begin, int32_t x_end);
/* step_range on an explicit CUDA stream (NULL: the context's): the edge planes of a slab run on a
 * side stream concurrently with the bulk, whose launch would otherwise wait behind them.  The
 * caller orders the streams (the side stream waits for the step's start; the context's stream
 * waits for the side stream before step_end's successor). */
int hlbm_step_range_on(hlbm_ctx* ctx, int32_t x_begin, int32_t x_end, void* cuda_stream);
int hlbm_step_end(hlbm_ctx* ctx);
/* device pointer of the current state buffer and its size (bytes) */
int hlbm_state_buffer(hlbm_ctx* ctx, void** ptr, int64_t* bytes);
int64_t hlbm_step_count(const hlbm_ctx* ctx);
/* kernel launches issued by this context so far (evidence for the benchmark's launch count) */
int64_t hlbm_launch_count(const hlbm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HLBM_H */
