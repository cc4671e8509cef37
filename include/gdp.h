/*
 * gdp.h — C ABI of the B200-native gradient-domain multigrid hot path
 * (Kazhdan et al., "Gradient-Domain Processing for Large EM Image Stacks",
 *  arXiv 1310.0041; reference text /root/reference/PAPER.md, cited as PAPER.md:L).
 *
 * The library solves, on regular voxel grids with Neumann boundaries, the
 * screened anisotropic Poisson system of the paper's §4:
 *
 *      (alpha - div W grad) x = alpha V - div W G,      W = Diag(bx, by, bz) >= 0
 *
 * by multigrid V-cycles whose every step runs in the
 * library's own sm_100a CUDA kernels.  Two instances are exported as whole solves:
 *   - gdp_diffuse_z               phase 1, Eq. (1): 3D anisotropic
 *                                 diffusion across slices, alpha = 0, G = (dI0/dx, dI0/dy, 0);
 *   - gdp_screened_poisson_slices phase 2, Eq. (2): per-slice 2D
 *                                 screened Poisson (alpha - Delta) I2 = alpha I1 - Delta I0.
 * and two building blocks: gdp_vcycle (one V-cycle on an explicit rhs) and
 * gdp_residual (r = b - A x with fp64 norms, the measure of PAPER.md:355).
 *
 * Discretisation: cell-centred voxels; the gradient is the
 * forward difference on the links between face-adjacent voxels; the divergence is
 * its negative transpose; links leaving the grid do not exist (Neumann).  Hence
 * A x at voxel c is  alpha x_c + sum_d beta_d sum_{n valid nbr of c along d} (x_c - x_n)
 * (interior diagonal 2(bx+by+bz), e.g. 4.2 for W = (1,1,0.1)).
 *
 * LAYOUT: every volume is dense, slice-major, x fastest: element (x,y,z) lives at
 *   [z*ny*nx + y*nx + x], no padding.  u8 intensities decode to
 *   u8/255 rounded to fp32 (IEEE division); fp32 volumes are used as given.
 * OWNERSHIP: all array pointers are owned by the caller; the library never frees
 *   or retains them past the call.  Device-pointer entry points take pointers in
 *   the memory of the ctx's device; host entry points take host pointers (pinned or
 *   pageable) and do their own staging.  `stream` is a cudaStream_t passed as void*
 *   (NULL = the legacy default stream).
 * ERRORS: every entry point returns a gdp_status; nothing throws across the ABI.
 *   On failure gdp_last_error() returns a thread-local message.  A GDP_ENOCONV
 *   return still leaves the best iterate in the output and fills the report.
 * THREADING: one ctx per host thread.  Whole solves block until convergence
 *   (they read back fp64 norms once per V-cycle); gdp_vcycle / gdp_residual
 *   synchronise `stream` only to return their host scalars.
 * DISTRIBUTION: a ctx created with world > 1 owns an NCCL communicator over the
 *   ranks; each rank passes its local z-slab (local dims) and the slab's global
 *   position (z0_global, nz_global); slabs must tile the stack in rank order.
 *   Phase 1 exchanges one ghost plane per slab face per half-sweep and gathers the
 *   coarse levels once per V-cycle; phase 2 is slab-local (independent slices).
 *   A ctx created with gdp_ctx_create_loopback emulates `world` slabs inside one
 *   process on one GPU (same driver, halo exchange by device copies): the caller
 *   passes the whole stack.  Results are bit-identical to the single-rank solve.
 */
#ifndef GDP_H_
#define GDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GDP_MAX_CYCLES 64
#define GDP_MAX_LEVELS 32

typedef enum {
  GDP_OK = 0,
  GDP_EINVAL = 1,   /* null pointer, dims <= 0, alpha/beta < 0 or non-finite,
                       alpha = 0 with all beta = 0 (singular), alpha <= 0 in
                       the slices call, unsupported layout */
  GDP_ECUDA = 2,    /* a CUDA runtime error; gdp_last_error() keeps cudaGetErrorString */
  GDP_ENOCONV = 3,  /* cycle cap or stagnation before rel_tol; output = best iterate */
  GDP_ENOMEM = 4,   /* device allocation failed */
  GDP_ENCCL = 5     /* NCCL error (distributed ctx only) */
} gdp_status;

typedef enum { GDP_U8 = 0, GDP_F32 = 1 } gdp_dtype;

/* Discretisation of the multigrid hierarchy, PAPER.md:305-323 (§4.2), SURVEY.md §8(f) NEXT-3.
 *   CONSTANT: the 6-point (7-point with the centre) finite-difference Laplacian on every level
 *             (this library's main path: finite-volume rediscretised coarse operators, volume-
 *             weighted restriction, cell-centred linear prolongation);
 *   HYBRID:   the same finest operator (same discrete answer), B-spline transfers (1/2, 1, 1/2)
 *             per axis and Galerkin coarse operators P^T A P (27-point);
 *   LINEAR:   the first-order B-spline finite-element operator (27-point, a different discrete
 *             answer: oracle/fem_linear.py), the same transfers, Galerkin coarse operators
 *             (PAPER.md:309-311).
 * HYBRID and LINEAR smooth with multicoloured Gauss-Seidel (8 colours on 27-point levels, 4 per
 * slice in phase 2, red-black on the Hybrid finest level) and solve the coarsest level exactly by
 * generalised fast diagonalisation.  They run single-rank and in core, without the FMG start,
 * graph replay or the dx gate.                                          */
typedef enum { GDP_SCHEME_CONSTANT = 0, GDP_SCHEME_HYBRID = 1, GDP_SCHEME_LINEAR = 2 } gdp_scheme;

typedef struct { int64_t nx, ny, nz; } gdp_dims;

/* W = Diag(bx, by, bz), PAPER.md:150-152 (application value (1, 1, 0.1)). */
typedef struct { float bx, by, bz; } gdp_weights;

typedef struct {
  double rel_tol;     /* stop when ||b - A x|| / ||b|| <= rel_tol (fp64 norms). Default 1e-6
                         (BASELINE.json north_star).  Phase 2: max over slices.           */
  int max_vcycles;    /* cap (<= GDP_MAX_CYCLES).  Default 30.                              */
  int nu_pre;         /* red-black Gauss-Seidel sweeps before restriction.  Default 2.      */
  int nu_post;        /* sweeps after prolongation.  Default 2.                             */
  int coarse_max;     /* coarsest level: <= coarse_max unknowns per independent system and
                         <= 64 cells along each coupled axis.  Default 4096.                */
  int stagnation;     /* stop (GDP_ENOCONV) after this many cycles each reducing the residual
                         by less than 10%.  Default 2.  0 disables.                         */
  int fused;          /* bitmask of fused level passes (bit-identical to the reference
                         schedule of one kernel per half-sweep, fused = 0):
                         1 = 2D register passes (levels without z links, phase 2);
                         2 = 3D z-marching sweeps (levels with z links, phase 1);
                         4 = with 2: a whole 3D level pass (nu sweeps + the restriction or
                             the prolongation + nu sweeps + the norms) in one temporally
                             blocked HBM pass, TMA-staged (nu <= 2, nx % 4 == 0; else per-sweep
                             kernels).  Bit-identical; measured slower than 2 on B200 so far
                             (DESIGN.md section 7), hence off by default;
                         8 = the coarse tail of every V-cycle (single-slab levels under 2M cells)
                             in two cooperative launches (down walk, up walk) around the
                             coarsest solve, instead of ~5 launches per level.  Bit-identical;
                             measured 0.45 ms slower per config-1 step than graph-replayed
                             per-level launches, hence off by default;
                         16 = with 2: each 3D sweep by the TMA-staged single-sweep pass kernel
                             instead of the z-march (bit-identical; measured slower);
                         32 = with 2: each 3D sweep by the vertical-pack z-march (8 x 2 cells per
                             thread as f32x2 packs of one colour, x / b planes in and the final
                             plane out by TMA; nx % 4 == 0, 16-byte aligned arrays; z-coarsened
                             prolongating sweeps keep the 2 kernel).  Bit-identical; 2-9 % faster
                             per launch than 2 on config 1.
                         Default 35.                                                         */
  int use_graphs;     /* 1: every V-cycle of a single-rank in-core solve (with its norm read-back)
                         is captured once as a CUDA graph per (output buffer, cycle variant) and
                         replayed by later solves on the same hierarchy (launch latency; needs a
                         non-NULL stream; bit-identical).  The first solve on a hierarchy and
                         profiled solves launch normally.  Default 1.                        */
  int nu_pre_slices;  /* phase 2 (gdp_screened_poisson_slices) pre-smoothing sweeps; < 0: nu_pre.
                         Default 1.                                                          */
  int nu_post_slices; /* phase 2 post-smoothing sweeps; < 0: nu_post.  Default 2: V(1,2) reaches
                         1e-6 in the same 4 cycles as V(2,2) on config 1 and is the fastest of
                         (2,2) / (2,1) / (1,2) / (1,1) there (tools/omega_sweep.py).          */
  float omega;        /* over-relaxation of the red-black sweeps, 0 < omega < 2 (1 = Gauss-Seidel;
                         the converged answer does not depend on it).  Phases 1 / general.    */
  float omega_slices; /* the same for phase 2.                                              */
  int fmg;            /* full-multigrid start of an in-core solve, single rank or z-slab team (the
                         out-of-core streamer starts from x0): r0 is
                         restricted to level 1, solved there by nested iteration (coarsest
                         solve, then per level a prolongation and one V-cycle), and the
                         correction is prolongated into the first fine V-cycle.  Changes the
                         iterate path, not the stopping rule.  0 = off; 1 = one V-cycle per
                         level; 2 / 3 = V-cycles from level 2, level 1 only smoothed (2) or
                         only interpolated (3); + 4: restrict r0 in a pass of its own instead
                         of inside the init pass (same values; for tests).  Phases 1 / general.
                         The nested cycles use one post-smoothing sweep fewer than the phase.
                         Default 1: config 1 phase 1 converges in 3 cycles instead of 4
                         (tools/fmg_check.py).                        */
  int fmg_slices;     /* the same for phase 2.  Default 3: 3 cycles instead of 4 on config 1. */
  double dx_tol;      /* correction-norm gate of the stopping rule: a
                         single-rank in-core solve stops only when also ||x_k - x_{k-1}||_inf
                         <= dx_tol for its last cycle k (measured exactly: the iterate is kept
                         before a cycle predicted to pass the residual gate from the observed
                         contraction; a cycle that passes unmeasured is followed by a measured
                         one).  Default 1e-4 (reading a9-dx: with the
                         measured contraction <= 0.1 per cycle the error left after such a cycle
                         is <= 1e-5).  0 disables.                                          */
  int scheme;         /* gdp_scheme of the hierarchy (above).  Default GDP_SCHEME_CONSTANT.       */
  int half_staging;   /* NEXT-4, out-of-core phase 1 only: V-cycles whose residual
                         is predicted (observed contraction) to stay above 5e-3 keep the host-resident
                         iterate in fp16 (half the host-link bytes of those passes); the later cycles
                         read it back and store fp32, so the answer is an fp32 iterate.  Default 0. */
  int stream_fuse;    /* NEXT-2, out-of-core phase 1: each finest-level streaming
                         pass applies several sweeps to the host-resident iterate in one host-link
                         round trip (z-lagged stages, bit-identical to the in-core sweeps): the down
                         pass (nu_pre sweeps + restriction) is one pass, and the up pass of a cycle
                         that is not predicted to be the last also runs the next cycle's down sweeps
                         (one round trip per V-cycle).  0: one pass per sweep.  Default 1.       */
} gdp_opts;

typedef struct {
  int status;                          /* gdp_status of the solve                          */
  int vcycles;                         /* V-cycles run                                     */
  int levels;                          /* multigrid levels (incl. finest and coarsest)     */
  double rel_res[GDP_MAX_CYCLES + 1];  /* [0] = initial, [k] = after cycle k (phase 2: max
                                          over slices)                                     */
  double norm_b;                       /* ||b||_2 of the finest rhs (phase 2: of the worst slice) */
  double seconds;                      /* device time of the solve (CUDA events)           */
  double hbm_bytes_est;                /* algorithmic HBM bytes of the solve   */
  int64_t kernel_launches;             /* library kernels launched by the call             */
  double dx_inf;                       /* ||x_k - x_{k-1}||_inf of the last cycle (max over
                                          slices in phase 2); -1 when not measured            */
} gdp_report;

typedef struct gdp_ctx gdp_ctx;

/* Fill *o with the defaults above. */
int gdp_opts_default(gdp_opts* o);

/* Create a context on CUDA `device`.  world == 1: single rank, nccl_unique_id NULL.
 * world > 1: this process is rank `rank`; nccl_unique_id points to the 128-byte
 * ncclUniqueId every rank received (e.g. broadcast by torch.distributed). */
int gdp_ctx_create(gdp_ctx** out, int device, int rank, int world, const void* nccl_unique_id);

/* Create a context emulating `world` ranks in this process on one device: the
 * caller passes the WHOLE volume and the library splits it into `world` z-slabs
 * internally (halo exchange = device copies).  Test vehicle for the partition. */
int gdp_ctx_create_loopback(gdp_ctx** out, int device, int world);

int gdp_ctx_destroy(gdp_ctx* ctx);

/* Write a fresh ncclUniqueId (128 bytes) to `out` (n >= 128) — rank 0 calls it and
 * broadcasts the bytes (e.g. with torch.distributed) before every rank's gdp_ctx_create. */
int gdp_get_unique_id(void* out, size_t n);

/* Phase 1 — Eq. (1).  Solves (alpha - div W grad) I1 = alpha I0 - div W G,
 * G = (dI0/dx, dI0/dy, 0); with alpha = 0 (the paper's AD) the constant null space is
 * removed by pinning mean(I1) = mean(I0) in fp64 (reading c-3).
 *   I0    device, local slab nx*ny*nz of `dtype`
 *   I1    device fp32 output, same shape (may not alias I0)
 *   local local slab dims; z0_global / nz_global its position in the global stack
 *         (world == 1: 0 and local.nz)
 *   W     weights, application value (1, 1, 0.1)                                      */
int gdp_diffuse_z(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* I1, gdp_dims local,
                  int64_t z0_global, int64_t nz_global, gdp_weights W, float alpha,
                  const gdp_opts* opts, gdp_report* report, void* stream);

/* Phase 2 — Eq. (2).  For every slice i independently:
 *   (alpha - Delta) I2_i = alpha I1_i - Delta I0_i,   alpha > 0 (application 0.01).
 *   I0 device (dtype), I1 device fp32, I2 device fp32 output (may alias I1, not I0).
 * Slices are independent systems: no communication even on a distributed ctx.       */
int gdp_screened_poisson_slices(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, const float* I1,
                                float* I2, gdp_dims local, float alpha, const gdp_opts* opts,
                                gdp_report* report, void* stream);

/* Both phases back to back: I1 = diffuse_z(I0), I2 = slices(I0, I1).
 * I1 may be NULL (library scratch).  reports may be NULL.                            */
int gdp_destripe(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* I1, float* I2,
                 gdp_dims local, int64_t z0_global, int64_t nz_global, gdp_weights W,
                 float alpha, const gdp_opts* opts, gdp_report* rep1, gdp_report* rep2,
                 void* stream);

/* Host-buffer entry: I0 and I2 (and I1 if non-NULL) are
 * HOST arrays of the whole local stack (on a distributed ctx: this rank's slab at
 * z0_global of nz_global; single rank: 0 and local.nz).  The library streams z-slabs host->device on
 * side streams, runs both phases, and streams I2 back.  If the stack does not fit in
 * `hbm_budget_bytes` (0 = 90% of free device memory), a single-rank ctx runs OUT OF CORE: the
 * finest level of phase 1 stays in the host buffers (I1 is then required scratch as well as
 * output: NULL is allowed, the library pins a scratch) and is streamed through the device in
 * z-chunks — several sweeps per host-link round trip (opts->stream_fuse, NEXT-2), optionally fp16
 * staging of early iterates (opts->half_staging, NEXT-4) — and phase 2 streams slice batches.
 * Out of core is Constant-scheme and single-rank only: otherwise GDP_ENOMEM.  The report's
 * hbm_bytes_est is then the host-link bytes of phase 1.                                  */
int gdp_destripe_host(gdp_ctx* ctx, const void* I0_host, gdp_dtype dtype, float* I1_host,
                      float* I2_host, gdp_dims local, int64_t z0_global, int64_t nz_global,
                      gdp_weights W, float alpha, size_t hbm_budget_bytes, const gdp_opts* opts,
                      gdp_report* rep1, gdp_report* rep2);

/* NEXT-1 — the §6 NPR filter (after Bhat et al. §6.2): a general 3D
 * screened solve through the same V-cycle,
 *   out = argmin alpha (I - I0)^2 + || grad I - V ||_W^2,
 *   V   = lambda (1 - exp(-|grad I0|^2 / (2 sigma^2))) grad I0  on every link,
 * |grad I0|^2 being the 3D forward-difference gradient at the link's base voxel (DESIGN.md
 * reading n-1).  Intensities are on the u8/255 scale, so the paper's sigma = 5 gray levels is
 * sigma = 5/255 (reading n-2); paper values alpha = 0.001, W = (1, 1, 0.1), lambda = 1.25.
 *   I0   device, nx*ny*nz of dtype;  out  device fp32 (may not alias I0); single rank.
 * Errors: GDP_EINVAL for alpha <= 0, sigma <= 0, lambda < 0 or non-finite parameters.     */
int gdp_npr_filter(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* out, gdp_dims dims, gdp_weights W,
                   float alpha, float lambda, float sigma, const gdp_opts* opts, gdp_report* report,
                   void* stream);

/* One V-cycle on (alpha - div W grad) x = b.  x device fp32 in/out,
 * b device fp32.  With alpha = 0, b is used as given (the caller guarantees sum b = 0
 * up to rounding; the coarsest solve drops the constant mode).
 * *rel_res_after (may be NULL) = ||b - A x|| / ||b|| after the cycle, fp64 (on a distributed
 * or loopback ctx: over the whole stack, per-plane sums added in global plane order).
 * Distributed / loopback ctx: x and b are this rank's slab (loopback: the whole stack); the
 * split levels run the reference schedule with one ghost plane per slab face per half-sweep,
 * the coarse levels are gathered (the iterate is bit-identical to a single-rank fused = 0
 * cycle; tests/test_gpu_parity.py).                                                      */
int gdp_vcycle(gdp_ctx* ctx, float* x, const float* b, gdp_dims local, int64_t z0_global,
               int64_t nz_global, gdp_weights W, float alpha, const gdp_opts* opts,
               double* rel_res_after, void* stream);

/* Residual r = b - A x of the §4 operator, difference form, fp32 per
 * voxel; norm2_r = sum r^2 and norm2_b = sum b^2 accumulated in fp64.  Distributed /
 * loopback ctx: the slab faces read the neighbouring slabs' planes (halo exchange) and the
 * norms are summed over all slabs in global plane order (identical for any partition).
 * r may be NULL (norms only).  Norm pointers are host.                                  */
int gdp_residual(gdp_ctx* ctx, const float* x, const float* b, float* r, gdp_dims local,
                 int64_t z0_global, int64_t nz_global, gdp_weights W, float alpha,
                 double* norm2_r, double* norm2_b, void* stream);

/* NEXT-3 inspection of a Hybrid / Linear hierarchy (single rank).  The hierarchy is the one the
 * solves build for (dims, W, alpha, per_slice, opts->coarse_max): per_slice = 1 is phase 2's
 * set of independent 2D slice systems (W's bz ignored), 0 a 3D system.
 * gdp_scheme_levels: *nlev = number of levels; level_dims[l] (may be NULL) their sizes and
 *   coarsened[3 l + d] (may be NULL) whether axis d (x, y, z) was coarsened from level l - 1,
 *   for l < max_levels.
 * gdp_scheme_apply: y = A_level x on the device (x, y fp32 of level `level`'s size, no aliasing);
 *   level 0 is the finest operator of the scheme, level l >= 1 its Galerkin operator
 *   P_l^T ... P_1^T A P_1 ... P_l (reading L-4).
 * gdp_scheme_residual: r = b - A_0 x (r may be NULL) and fp64 norms ||r||^2, ||b||^2.      */
int gdp_scheme_levels(gdp_ctx* ctx, int scheme, gdp_dims dims, gdp_weights W, float alpha, int per_slice,
                      const gdp_opts* opts, int* nlev, gdp_dims* level_dims, int* coarsened, int max_levels);
int gdp_scheme_apply(gdp_ctx* ctx, int scheme, int level, const float* x, float* y, gdp_dims dims,
                     gdp_weights W, float alpha, int per_slice, const gdp_opts* opts, void* stream);
int gdp_scheme_residual(gdp_ctx* ctx, int scheme, const float* x, const float* b, float* r, gdp_dims dims,
                        gdp_weights W, float alpha, int per_slice, double* norm2_r, double* norm2_b,
                        void* stream);

/* Per-kernel-class device timing (roofline measurement, bench.py).  Between begin and end
 * every library launch is bracketed by CUDA events on its own stream and tagged with the
 * algorithmic bytes it must move.  end() synchronises the
 * recorded events, fills up to `max` entries of `out` (one per kernel class that ran) and
 * sets *n_out.  Process-wide; not thread-safe against concurrent solves.               */
typedef struct {
  char name[32];        /* kernel class, e.g. "rbgs", "down2d"                          */
  int64_t launches;
  double ms;            /* summed device time of those launches                        */
  double alg_bytes;     /* summed bytes of those launches by this library's design model  */
  double alg_bytes_8d;  /* the same counted as SURVEY.md §8(d) does: a finest-level pass reads
                           the rhs inputs (phase 1: I0, 1 B u8 / 4 B f32; phase 2: I1 + I0)
                           in place of the fp32 b this library writes once per solve        */
} gdp_kernel_stat;
int gdp_profile_begin(void);
int gdp_profile_end(gdp_kernel_stat* out, int max, int* n_out);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* gdp_last_error(void);

/* Library version string and the number of kernels launched by this process so far. */
const char* gdp_version(void);
int64_t gdp_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* GDP_H_ */
