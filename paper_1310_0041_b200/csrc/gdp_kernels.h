// gdp_kernels.h — internal launch interface between the solver core (gdp_solver.cu)
// and the kernels (gdp_kernels.cu, gdp_fused.cu).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "gdp_device.cuh"

namespace gdp {

extern std::atomic<long long> g_launches;
inline void count_launch(long long n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Per-kernel-class device timing for the bench's roofline (gdp_profile_begin/end).  When
// enabled, each launch is bracketed by two events on its own stream and tagged with the
// algorithmic bytes it must move.  Disabled: no cost.
enum KClass {
  KC_RBGS = 0, KC_RESTRICT, KC_PROLONG, KC_NORMS, KC_COARSE, KC_UTIL,
  KC_DOWN2D, KC_UP2D, KC_DOWN3D, KC_UP3D, KC_COOP, KC_COUNT
};
extern const char* kclass_name[KC_COUNT];
extern bool g_prof_on;
extern double g_prof_finest;  // cells of the finest level of the running solve (0: none)
extern double g_prof_l1;      // cells of its level 1 (0: none)
extern double g_prof_rhs8d;   // SURVEY §8(d) bytes per finest cell of the rhs inputs (phase 1: s_in;
                              // phase 2: I1 4 + s_in) that a pass reading the written b0 stands for
void prof_push(int cls, double bytes, double bytes8d, cudaStream_t s, bool begin);
struct ProfScope {
  int cls;
  cudaStream_t s;
  // launches over the finest level / level 1 are classes of their own (index + KC_COUNT,
  // "name@L0"; index + 2 KC_COUNT, "name@L1").  reads_b0: the launch reads the level's fp32 rhs
  // (4 B per cell); over the finest level §8(d) counts the rhs inputs instead (g_prof_rhs8d).
  ProfScope(int c, double bytes, cudaStream_t st, double cells = 0.0, bool reads_b0 = false) : cls(c), s(st) {
    count_launch();
    const bool fin = cells > 0.0 && cells == g_prof_finest;
    if (fin) cls += KC_COUNT;
    else if (cells > 0.0 && cells == g_prof_l1) cls += 2 * KC_COUNT;
    if (g_prof_on) prof_push(cls, bytes, fin && reads_b0 ? bytes + (g_prof_rhs8d - 4.0) * cells : bytes, s, true);
  }
  ~ProfScope() {
    if (g_prof_on) prof_push(cls, 0.0, 0.0, s, false);
  }
};
// bytes per cell of the finest-level rhs inputs (u8/f32 I, optional fp32 V) or of b
inline double rhs_bytes(int mode, int tI, const RhsK& R) {
  if (mode == RHS_B) return 4.0;
  return (tI == 0 ? 1.0 : 4.0) + (R.vmode == 2 ? 4.0 : 0.0);
}

// fp64 block reduction of two values (warp shuffle, then shared memory); result valid in
// thread (0,0).  Fixed order -> deterministic.
__device__ __forceinline__ void block_sum2(double& a, double& b) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  __shared__ double sa[32], sb[32];
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int lane = tid & 31, warp = tid >> 5;
  if (lane == 0) { sa[warp] = a; sb[warp] = b; }
  __syncthreads();
  if (warp == 0) {
    const int nw = (nthr + 31) >> 5;
    a = lane < nw ? sa[lane] : 0.0;
    b = lane < nw ? sb[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
    }
  }
}

struct CoarseK {
  int nx, ny, nz;     // coarsest level dims (whole level)
  int cx, cy, cz;     // coupled (transformed) axes; an uncoupled z makes nz independent systems
  const float *Fx, *Bx, *lx;
  const float *Fy, *By, *ly;
  const float *Fz, *Bz, *lz;
  float alpha;
  float lam_thr;      // eigenvalues <= lam_thr are dropped (alpha = 0 null space)
};

// reference-schedule kernels (tI: 0 = u8, 1 = f32)
void launch_rbgs(const LevelK& L, float* x, const float* xlo, const float* xhi, const RhsK& R,
                 int mode, int tI, int color, cudaStream_t s);
void launch_restrict(const LevelK& L, const float* x, const float* xlo, const float* xhi,
                     const RhsK& R, int mode, int tI, const XferAxis& tx, const XferAxis& ty,
                     const XferAxis& tz, int ncx, int ncy, int nczl, float* bc, cudaStream_t s);
void launch_restrict_b(const LevelK& L, const float* b, const XferAxis& tx, const XferAxis& ty, const XferAxis& tz,
                       int ncx, int ncy, int nczl, float* bc, cudaStream_t s);
void launch_prolong(const LevelK& L, float* xf, const XferAxis& tx, const XferAxis& ty,
                    const XferAxis& tz, int ncx, int ncy, int nczl, long long cz0, const float* xc,
                    const float* xclo, const float* xchi, cudaStream_t s);
int norms_blocks_per_plane(int nx, int ny);
void launch_norms(const LevelK& L, const float* x, const float* xlo, const float* xhi,
                  const RhsK& R, int mode, int tI, float* rout, double2* partials,
                  double2* plane_out, cudaStream_t s);
void launch_plane_sums(const void* a, int ta, const void* b, int tb, int nx, int ny, int nz,
                       double2* partials, double2* plane_out, cudaStream_t s);
void launch_finalize(const double2* partials, int per, int nplanes, double2* out, cudaStream_t s);
void launch_rhs(const LevelK& L, const RhsK& R, int tI, float* b, cudaStream_t s);
void launch_decode_copy(const void* I, int tI, float* x, long long n, cudaStream_t s);
void launch_npr_rhs(const LevelK& L, const void* I, int tI, float* x0, float* b, float bx, float by, float bz,
                    float lam, float sigma, cudaStream_t s);
// x0 = decode(I), b = finest rhs, and the initial-residual norm partials (init_blocks_per_plane per plane)
int init_blocks_per_plane(int nx, int ny);
// X.bc (optional): also restrict the initial residual r0 into the next level's rhs (plane-local
// x/y coarsening only), the values k_restrict would write (FMG start)
struct InitXfer {
  XferAxis tx, ty;
  int ncx = 0, ncy = 0;
  float* bc = nullptr;
};
void launch_init(const LevelK& L, const RhsK& R, int tI, float* x0, float* b, double2* partials, cudaStream_t s,
                 const InitXfer& X = InitXfer{});
void launch_add_scalar(float* x, long long n, float v, cudaStream_t s);
void launch_axpy(float* x, const float* e, long long n, cudaStream_t s);
void launch_maxdiff(const float* a, const float* b, long long n, unsigned int* out, cudaStream_t s);
// the coarse tail of a V-cycle (levels lc .. nl-2 of a single-slab hierarchy), cooperative grids
struct CoopLv {
  LevelK K;             // the level
  float* x;             // its x
  const float* b;       // its rhs
  XferAxis tx, ty, tz;  // to the next coarser level
  int ncx, ncy, nczl;
  float* bc;            // next level's rhs (down: restricted residual)
  const float* xc;      // next level's x (up: prolongated correction)
};
cudaError_t launch_coop(bool down, const CoopLv* lv, int n, int nu, int zero_first, unsigned int* bar,
                        double cells, double bytes, cudaStream_t s);
size_t coarse_smem_bytes(const CoarseK& C);
cudaError_t launch_coarse(const CoarseK& C, const float* b, float* x, cudaStream_t s);

}  // namespace gdp
