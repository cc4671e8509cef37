// gdp_vpass3d.cu — host side of the temporally blocked 3D level passes (gdp_vpass3d.cuh):
// tensor maps, work plan, variant dispatch.  The kernels are instantiated in gdp_vp_down.cu /
// gdp_vp_up.cu (compiled in parallel).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "gdp_vpass3d.cuh"

namespace gdp {
namespace vp {
GDP_VP_VARIANTS(GDP_VP_EXTERN)
}  // namespace vp

using namespace vp;

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int load_encode() {
  static std::once_flag once;
  static int rc = GDP_OK;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      rc = set_err(GDP_ECUDA, "cuTensorMapEncodeTiled not available from the driver");
      return;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return rc;
}

// L2 promotion 128 B: the boxes start 16 B before a 224-B tile stride, so 256-B promotion over-fetches
// the neighbouring tiles' columns, which are not shared in L2 (the persistent CTAs drift apart by more
// planes than L2 retains): measured DRAM reads of a finest config-1 sweep 1.537 -> 1.474 GB
// (tools/ab_tma.sh; NONE measures the same as 128 B, an evict_last cache hint changes nothing)
#ifndef GDP_TMA_PROMO
#define GDP_TMA_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
// fp32 volume nx x ny x np planes at p, box bw x bh x 1
static int make_map(CUtensorMap* m, const float* p, int nx, int ny, long long np, int bw, int bh) {
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)std::max<long long>(np, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)nx * 4, (cuuint64_t)nx * ny * 4};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              GDP_TMA_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(GDP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return GDP_OK;
}

// the same, for other TMA-staged kernels (gdp_march3dv.cu)
int vp_make_map(CUtensorMap* m, const float* p, int nx, int ny, long long np, int bw, int bh) {
  const int rc = load_encode();
  if (rc != GDP_OK) return rc;
  return make_map(m, p, nx, ny, np, bw, bh);
}

static int g_nsm_vp = 0;
static int nsm() {
  if (!g_nsm_vp) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsm_vp, cudaDevAttrMultiProcessorCount, dev);
    if (g_nsm_vp <= 0) g_nsm_vp = 148;
  }
  return g_nsm_vp;
}

template <int NU, int MCL>
static void plan(const LevelK& L, bool zc, int zlo, int zhi, Pass& P) {
  using GG = Geo<NU>;
  const int TYI = MCL * TY - 2 * GG::HY;
  P.tiles_x = (L.nx + GG::TXI - 1) / GG::TXI;
  P.tiles_y = (L.ny + TYI - 1) / TYI;
  const int tiles = P.tiles_x * P.tiles_y;
  const int nz = zhi - zlo;
  const long long work = (long long)tiles * nz;
  const int grid = (int)std::min<long long>(nsm() / MCL, work);  // clusters
  P.zlo = zlo;
  P.zhi = zhi;
  P.zeven = zc ? 1 : 0;
  P.full = tiles / grid;
  const long long rem = (long long)(tiles - P.full * grid) * nz;
  P.max_segs = P.full + (int)((rem + grid - 1) / grid / std::max(nz, 1)) + 3;
  P.nitems = grid * MCL * P.max_segs;
}

template <int NU>
static cudaError_t dispatch(const Pass& P, bool prolong, bool zc, int tail, cudaStream_t s) {
#define VPL(T, PR, Z) return launch_vp<NU, T, PR, Z>(P, s)
  if (prolong) {  // z not coarsened (vpass3d_ok): up pass (norms / none) or an FMG-start down pass
    if (tail == TAIL_NORMS) VPL(2, true, false);
    if (tail == TAIL_RESTRICT) VPL(1, true, false);
    VPL(0, true, false);
  }
  if (tail == TAIL_RESTRICT) { if (zc) VPL(1, false, true); VPL(1, false, false); }
  if constexpr (NU == 1) {  // single sweeps (fused bit 16)
    if (tail == TAIL_NORMS) VPL(2, false, false);
    VPL(0, false, false);
  }
  return cudaErrorInvalidValue;  // not instantiated (vpass3d_ok refuses it)
#undef VPL
}

// The level-pass kernels serve single-slab levels with x and y coarsened to the next level
// (z too only without a prolongation in the pass), nx % 4 == 0 on both levels (16-byte TMA
// strides) and 16-byte aligned arrays; nu in {1, 2}.
bool vpass3d_ok(const Level& L, const Level& C, int nu, bool prolong, int tail, const float* xin,
                const float* xout, const float* b) {
  if (nu != 1 && nu != 2) return false;
  if (!prolong && tail != TAIL_RESTRICT && nu != 1) return false;  // variants not instantiated
  if (!C.tx.coarsened || !C.ty.coarsened || (prolong && C.tz.coarsened)) return false;
  if ((L.nx & 3) != 0 || (C.nx & 3) != 0) return false;
  if (!al16(xin) || !al16(xout) || !al16(b) || !al16(C.x) || !al16(C.b)) return false;
  if (load_encode() != GDP_OK) return false;
  return (long long)L.nx * L.ny < (1LL << 31) && (long long)C.nx * C.ny < (1LL << 31) && L.nzl == L.gz.n;
}

template <int NU>
static void plan_any(const Level& L, const Level& C, Pass& P) {
  plan<NU, 1>(L.K, C.tz.coarsened != 0, 0, L.nzl, P);
}

int vpass3d_items(const Level& L, const Level& C, int nu) {
  Pass P{};
  if (nu == 1) plan_any<1>(L, C, P);
  else plan_any<2>(L, C, P);
  return P.nitems;
}

// One whole level pass: nu sweeps (down: xin -> xout, then the residual restricted into C.b;
// up: xin + P C.x, nu sweeps -> xout, then the fp64 norms of the residual into `partials`, one
// per item, when tail == 2).  dxmax != NULL: atomically raises *dxmax (float bits) to a bound of
// max |xout - xin| over the level (per cell: its nu updates and its correction, each bounded by
// the largest of the pass).  *items (may be NULL) = partial slots written.
int fused_pass3d(const Level& L, const Level& C, const float* xin, float* xout, const float* b, bool zero_x,
                 bool prolong, int nu, int tail, double2* partials, unsigned int* dxmax, cudaStream_t s,
                 int* items) {
  int rc = load_encode();
  if (rc != GDP_OK) return rc;
  Pass P{};
  P.L = L.K;
  P.xout = xout;
  P.tx = C.tx; P.ty = C.ty; P.tz = C.tz; P.ncx = C.nx; P.ncy = C.ny;
  P.bc = C.b;
  P.partials = partials;
  (void)dxmax;  // not measured by the pass kernels (reserved)
  P.zero_x = zero_x ? 1 : 0;
  const bool zc = C.tz.coarsened != 0;
  if (nu == 1) plan_any<1>(L, C, P);
  else plan_any<2>(L, C, P);
  if ((rc = make_map(&P.tmx, zero_x ? b : xin, L.nx, L.ny, L.nzl, TX, TY)) != GDP_OK) return rc;
  if ((rc = make_map(&P.tmb, b, L.nx, L.ny, L.nzl, TX, TY)) != GDP_OK) return rc;
  if (prolong) {
    if ((rc = make_map(&P.tmc, C.x, C.nx, C.ny, C.nzl, CBX, CBY)) != GDP_OK) return rc;
  } else {
    P.tmc = P.tmb;
  }
  const double N = (double)L.nx * L.ny * L.nzl, Nc = (double)C.nx * C.ny * C.nzl;
  const double bytes = N * ((zero_x ? 4.0 : 8.0) + 4.0) + ((tail == 1 || prolong) ? Nc * 4.0 : 0.0);
  ProfScope ps(tail == 1 ? KC_DOWN3D : KC_UP3D, bytes, s, N, true);
  const cudaError_t e = nu == 1 ? dispatch<1>(P, prolong, zc, tail, s) : dispatch<2>(P, prolong, zc, tail, s);
  if (e != cudaSuccess) return set_err(GDP_ECUDA, "k_vpass3d launch: %s", cudaGetErrorString(e));
  if (items) *items = P.nitems;
  return GDP_OK;
}

}  // namespace gdp
