// gdp_internal.h — host-side structures of the solver core (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "../../include/gdp.h"
#include "gdp_kernels.h"

namespace gdp {

int set_err(int code, const char* fmt, ...);

struct AxisG {      // host geometry of one axis of one level (finest-grid units)
  int n;            // global cell count
  double H;         // full cell width
  double hl;        // width of the last cell (< H when partial)
  double beta;      // weight of the axis (W diagonal), same on every level
};

struct Level {
  AxisG gx{}, gy{}, gz{};
  int nx = 0, ny = 0, nzl = 0;   // local dims
  long long z0 = 0;              // global z of local plane 0
  LevelK K{};
  XferAxis tx{}, ty{}, tz{};     // transfer from the finer level (valid for level >= 1)
  float* x = nullptr;            // solution / correction (level 0: caller's buffer)
  bool own_x = false;
  float* b = nullptr;            // restricted residual (levels >= 1)
  float* x2 = nullptr;           // second x buffer of the fused passes (down A -> B, up B -> A)
  float* xlo = nullptr;          // ghost planes of x for distributed slabs
  float* xhi = nullptr;
};

struct HierKey {
  long long nx, ny, nzl, z0, nzg;
  float bx, by, bz, alpha;
  int coarse_max;
  float omega = 1.f;  // over-relaxation of the sweeps
  bool operator<(const HierKey& o) const {
    return std::tie(nx, ny, nzl, z0, nzg, bx, by, bz, alpha, coarse_max, omega) <
           std::tie(o.nx, o.ny, o.nzl, o.z0, o.nzg, o.bx, o.by, o.bz, o.alpha, o.coarse_max, o.omega);
  }
};

struct Hier {
  HierKey key{};
  std::vector<Level> lv;
  CoarseK coarse{};
  std::vector<float*> dev_tables;
  double2* partials = nullptr;     // norm partials of level 0
  double2* plane_sums = nullptr;   // per-plane (sum a, sum b), device
  double2* h_plane = nullptr;      // pinned host mirror
  float* scratch_e = nullptr;      // single-level direct solve correction
  float* b0 = nullptr;             // finest-level rhs written out for the fused 2D passes
  unsigned int* dx_dev = nullptr;  // max |x_k - x_{k-1}| of the running cycle (float bits, device)
  unsigned int* dx_host = nullptr; // pinned mirror
  float* xprev = nullptr;          // x_{k-1} of a cycle that can end the solve (a9 correction norm)
  bool warm = false;               // run_vcycle ran once: every lazily allocated buffer exists
  CoopLv* coop_dev = nullptr;      // per level l >= 1 (index l - 1): the cooperative coarse tail's view
  struct CycleGraph {              // one V-cycle (+ its norm read-back) captured as a CUDA graph
    cudaGraphExec_t exec = nullptr;
    int up_norm_per = 0, up_norm_planes = 0;
    long long launches = 0;
  };
  std::map<std::tuple<const void*, const void*, long long>, CycleGraph> graphs;
  size_t partials_cap = 0;         // entries of `partials` per plane
  int up_norm_per = 0;             // >0: the last fused up pass left per-plane partials (this many per plane)
  int up_norm_planes = 0;          // planes of those partials (1: one row for the whole slab)
  bool init_restricted = false;    // launch_init also wrote R r0 into lv[1].b (FMG start)
  int init_norm_per = 0;           // >0: launch_init left the initial-residual partials (this many per plane)
  ~Hier();
};

struct Fine {        // the finest level of one solve
  float* x = nullptr;
  RhsK R{};
  int mode = RHS_B;
  int tI = 1;        // 0 = u8 source, 1 = f32
};

struct Comm;          // NCCL communicator state (gdp_comm.cu)

// A z-slab partition of phase 1 (gdp_dist.cu): the split levels [0, ff) of each local slab
// and the gathered levels [ff, ..) shared by them.
struct DistPlan {
  std::vector<std::unique_ptr<Hier>> parts;  // local slabs (1 per NCCL rank, `loop` in loopback)
  std::unique_ptr<Hier> tail;                // full levels, lv[0] = global level ff
  std::vector<long long> z0;                 // global first plane of each local slab
  std::vector<int> nzl;                      // planes of each local slab
  std::vector<float*> b0;                    // finest rhs of each local slab
  int ff = 0;                                // first full level
  std::vector<size_t> goff, gcnt;            // per slab: elements of the gathered level it restricts into
  int nzg = 0;
  double2* h_planes = nullptr;               // pinned, nzg per-plane sums in global order
  // fused finest level (k_march3d): per local slab two x windows and the rhs with G ghost planes
  // per face ([z0 - G, z0 + nzl + G), interior at offset G); exchanged once per sweep
  static constexpr int G = 3;
  bool slabs_fusable = false;                // every slab of the team (all ranks) holds >= G planes
  bool fused = false;                        // windows allocated
  bool active = false;                       // this call runs the fused finest level (opts.fused & 2)
  std::vector<float*> w0, w1, bw;
  std::vector<float*> cw;                    // split level 1: x with G ghost planes (prolongation source)
  double2* fpart = nullptr;                  // norm partials of the fused up pass (all local slabs)
  size_t fpart_cap = 0;
  // boundary-first halo overlap: the ghost exchange of a sweep's output runs on
  // a communication stream while the sweep's interior planes are computed
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_comm = nullptr;
  ~DistPlan();
};

struct Ctx {
  int device = 0, rank = 0, world = 1;
  int loop = 1;  // loopback slabs emulated in this process (gdp_ctx_create_loopback)
  std::map<HierKey, std::unique_ptr<DistPlan>> dist;
  std::map<HierKey, std::unique_ptr<Hier>> hier;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  Comm* comm = nullptr;
  // host-entry staging (gdp_destripe_host): device copies of I0, I1, I2 and two streams
  void* hbuf[3] = {nullptr, nullptr, nullptr};
  size_t hbuf_cap[3] = {0, 0, 0};
  cudaStream_t hs = nullptr, hcs = nullptr;
  cudaEvent_t hev = nullptr;
  void* scheme_cache = nullptr;  // NEXT-3 hierarchies (gdp_scheme.cu)
  void* h16 = nullptr;           // pinned fp16 host iterate of the out-of-core streamer (NEXT-4), kept
  size_t h16_bytes = 0;          // across solves: pinning tens of GB costs seconds per call
  int get_hier(const HierKey& k, Hier** out);
  int ensure_scratch(size_t bytes);
  int ensure_hbuf(int i, size_t bytes);
  ~Ctx();
};

int build_hier(const HierKey& key, std::unique_ptr<Hier>& out);
int level_chain(const HierKey& key, std::vector<Level>& lv, int& first_full);
int build_hier_levels(const HierKey& key, const std::vector<Level>& chain, int from, int end, bool own0,
                      bool coarsest_here, std::unique_ptr<Hier>& out);
// one V-cycle over levels [l0, end) (l0 = 1: the caller owns level 0, e.g. the out-of-core streamer)
constexpr unsigned RV_PROLONG = 1u;
int run_vcycle(Ctx& ctx, Hier& H, const Fine& f, const gdp_opts& o, cudaStream_t s, int l0 = 0,
               unsigned flags = 0);
int finest_norms(Ctx& ctx, Hier& H, const Fine& f, float* rout, cudaStream_t s);
int solve(Ctx& ctx, Hier& H, const Fine& f, const gdp_opts& o, bool per_slice, gdp_report* rep,
          cudaStream_t s);
double hbm_model(const Hier& H, double s_I, double s_V, int vcycles);

// fused schedule (gdp_fused.cu): return true if the pass was handled
bool fusable2d(const Level& L, const Level& C, const gdp_opts& o);
void fused_down2d(const Level& L, const Level& C, const float* xin, float* xout, const RhsK& R,
                  int mode, int tI, int nu, bool zero_x, cudaStream_t s, bool prolong = false);
void fused_up2d(const Level& L, const Level& C, const float* xin, float* xout, const RhsK& R,
                int mode, int tI, int nu, double2* partials, cudaStream_t s);
int fused_tiles_per_plane(int nu, const Level& L, const Level& C);
// row-marching 2D passes (gdp_rows2d.cu)
int rows2d_items_per_plane(int nu, const LevelK& L);
void rows2d_pass(bool down, int nu, const Level& L, const Level& C, const float* xin, float* xout, const float* b,
                 bool zero_x, double2* partials, cudaStream_t s, bool prolong = false);
bool fusable3d(const Level& L, const Level& C, const gdp_opts& o);
int fused3d_items(const Level& L, const Level& C, int zlo = 0, int zhi = -1);
// temporally blocked whole level passes (gdp_vpass3d.cu)
bool vpass3d_ok(const Level& L, const Level& C, int nu, bool prolong, int tail, const float* xin,
                const float* xout, const float* b);
int vpass3d_items(const Level& L, const Level& C, int nu);
int fused_pass3d(const Level& L, const Level& C, const float* xin, float* xout, const float* b, bool zero_x,
                 bool prolong, int nu, int tail, double2* partials, unsigned int* dxmax, cudaStream_t s,
                 int* items);
int fused_sweep3d(const Level& L, const Level& C, const float* xin, float* xout, const float* b,
                  bool zero_x, bool prolong, int tail, double2* partials, cudaStream_t s, int zlo = 0,
                  int zhi = -1);
// the vertical-pack TMA z-march sweep (gdp_march3dv.cu; fused bit 32)
bool sweep3dv_ok(const Level& L, const Level& C, bool prolong, const float* xin, const float* xout, const float* b);
int sweep3dv_items(const Level& L, const Level& C);
int fused_sweep3dv(const Level& L, const Level& C, const float* xin, float* xout, const float* b, bool zero_x,
                   bool prolong, int tail, double2* partials, cudaStream_t s, int* items);

// out-of-core streaming of the finest level (gdp_stream.cu)
struct HostPin {
  void* p = nullptr;
  ~HostPin();
  int pin(const void* ptr, size_t bytes);
};
// keep_x / keep_R (may be NULL): phase 1 hands its HBM-resident planes [0, R) of the iterate (unpinned
// I1) to the caller instead of copying them back (cudaFree by the caller); phase 2 then reads them
// in place and writes the pinned I1 back (NEXT-2 (ii): phase 2 consumes phase 1's output on the device).
// xh == NULL (the caller does not want I1; needs keep_x / keep_R): the host planes [R, nz) live in a
// pinned scratch returned in *host_scratch (cudaFreeHost by the caller); the returned *host_scratch
// minus R planes is the host iterate's base pointer for phase 2.
int stream_diffuse_z(Ctx& C, const void* I0h, int tI, float* xh, long long nx, long long ny, long long nz,
                     float bx, float by, float bz, const gdp_opts& o, size_t budget, gdp_report* rep,
                     double* shift_out, float** keep_x = nullptr, int* keep_R = nullptr,
                     float** host_scratch = nullptr, void** keep_i0 = nullptr);
int stream_slices(Ctx& C, gdp_ctx* cctx, const void* I0h, gdp_dtype dtype, float* I1h, float* I2h, long long nx,
                  long long ny, long long nz, float alpha, double shift, const gdp_opts& o, size_t budget,
                  gdp_report* rep, const float* I1dev = nullptr, int R = 0, bool write_i1 = true,
                  const void* I0dev = nullptr);

void jacobi_eig(int n, std::vector<double>& A, std::vector<double>& Q, std::vector<double>& lam);

// NEXT-3: the Hybrid / Linear discretisations (gdp_scheme.cu), single rank, in core
void scheme_cache_destroy(void* p);
int scheme_diffuse_z(Ctx& C, const void* I0, int tI, float* I1, long long nx, long long ny, long long nz, float bx,
                     float by, float bz, float alpha, const gdp_opts& o, gdp_report* rep, cudaStream_t s);
int scheme_slices(Ctx& C, const void* I0, int tI, const float* I1, float* I2, long long nx, long long ny,
                  long long nz, float alpha, float vshift, const gdp_opts& o, gdp_report* rep, cudaStream_t s);
int scheme_vcycle(Ctx& C, float* x, const float* b, long long nx, long long ny, long long nz, float bx, float by,
                  float bz, float alpha, const gdp_opts& o, double* rel, cudaStream_t s);
int scheme_levels(Ctx& C, int scheme, long long nx, long long ny, long long nz, float bx, float by, float bz,
                  float alpha, int per_slice, const gdp_opts& o, int* nlev, gdp_dims* dims, int* coarsened, int max);
int scheme_apply(Ctx& C, int scheme, int level, const float* x, float* y, long long nx, long long ny, long long nz,
                 float bx, float by, float bz, float alpha, int per_slice, const gdp_opts& o, cudaStream_t s);
int scheme_residual(Ctx& C, int scheme, const float* x, const float* b, float* r, long long nx, long long ny,
                    long long nz, float bx, float by, float bz, float alpha, int per_slice, const gdp_opts& o,
                    double* rr, double* bb, cudaStream_t s);

// communication (gdp_comm.cu); single-rank contexts make these no-ops
int comm_init(Ctx& c, const void* nccl_unique_id);
void comm_destroy(Ctx& c);
int comm_allreduce_sum2(Ctx& c, double* a, double* b, cudaStream_t s);
int comm_unique_id(void* out, size_t n);
int comm_halo_parts(Ctx& c, DistPlan& D, int l, float* const* xs, cudaStream_t s);
int comm_gather_full(Ctx& c, DistPlan& D, float* full, cudaStream_t s);
int comm_plane_sums(Ctx& c, DistPlan& D, double2* const* local, double2* out, cudaStream_t s);
int comm_ghosts(Ctx& c, DistPlan& D, float* const* wins, cudaStream_t s, int level = 0);
int dist_diffuse_z(Ctx& c, const void* I0, int tI, float* I1, long long nx, long long ny, long long nzl,
                   long long z0g, long long nzg, float bx, float by, float bz, float alpha, const gdp_opts& o,
                   gdp_report* rep, cudaStream_t s);
// gdp_vcycle / gdp_residual on a z-slab partition (x, b, r: the caller's slab, or the whole stack
// in loopback); norms summed over all slabs in global plane order
int dist_vcycle(Ctx& c, float* x, const float* b, long long nx, long long ny, long long nzl, long long z0g,
                long long nzg, float bx, float by, float bz, float alpha, const gdp_opts& o, double* rel,
                cudaStream_t s);
int dist_residual(Ctx& c, const float* x, const float* b, float* r, long long nx, long long ny, long long nzl,
                  long long z0g, long long nzg, float bx, float by, float bz, float alpha, const gdp_opts& o,
                  double* rr, double* bb, cudaStream_t s);

}  // namespace gdp

struct gdp_ctx {
  gdp::Ctx impl;
};
