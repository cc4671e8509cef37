// gdp_solver.cu — solver core behind the C ABI (include/gdp.h).
//
// Owns the multigrid hierarchy, the coarsest-level fast
// diagonalisation, the V-cycle driver with its stopping rule, the mean pin of the
// alpha = 0 diffusion and the C entry points.  Every arithmetic step runs in the
// kernels of gdp_kernels.cu / gdp_fused.cu; the host only orchestrates and reads
// back fp64 norms (a few bytes per V-cycle).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/gdp.h"
#include "gdp_internal.h"

namespace gdp {

std::atomic<long long> g_launches{0};

// ---------------------------------------------------------------------------------
// per-kernel-class profiler
// ---------------------------------------------------------------------------------
const char* kclass_name[KC_COUNT] = {"rbgs", "restrict", "prolong", "norms", "coarse", "util",
                                     "down2d", "up2d", "down3d", "up3d", "coop"};
bool g_prof_on = false;
double g_prof_finest = 0.0;
double g_prof_l1 = 0.0;
double g_prof_rhs8d = 4.0;
struct ProfRec { int cls; double bytes, bytes8d; cudaEvent_t a, b; };
static std::vector<ProfRec> g_prof;
static std::vector<int> g_prof_open;  // stack of open records

void prof_push(int cls, double bytes, double bytes8d, cudaStream_t s, bool begin) {
  if (begin) {
    ProfRec r{cls, bytes, bytes8d, nullptr, nullptr};
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, s);
    g_prof.push_back(r);
    g_prof_open.push_back((int)g_prof.size() - 1);
  } else if (!g_prof_open.empty()) {
    cudaEventRecord(g_prof[g_prof_open.back()].b, s);
    g_prof_open.pop_back();
  }
}

static thread_local std::string t_err;

int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(e_ == cudaErrorMemoryAllocation ? GDP_ENOMEM : GDP_ECUDA,            \
                     "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,   \
                     __LINE__);                                                           \
  } while (0)

#define RET(call)                    \
  do {                               \
    int r_ = (call);                 \
    if (r_ != GDP_OK) return r_;     \
  } while (0)

// ---------------------------------------------------------------------------------
// host geometry
// ---------------------------------------------------------------------------------
static AxisC make_axisc(const AxisG& g) {
  AxisC a{};
  a.n = g.n;
  if (g.beta <= 0.0 || g.n <= 1) { a.k = a.kr = a.kl = 0.f; return a; }
  const double dl = 0.5 * (g.H + g.hl);
  a.k = (float)(g.beta / (g.H * g.H));
  a.kr = (float)(g.beta / (dl * g.H));
  a.kl = (float)(g.beta / (dl * g.hl));
  return a;
}

static AxisG coarsen_axis(const AxisG& f) {
  AxisG c = f;
  c.n = (f.n + 1) / 2;
  c.H = 2.0 * f.H;
  c.hl = (f.n % 2 == 1) ? f.hl : (f.H + f.hl);
  return c;
}

static XferAxis make_xfer(const AxisG& f, const AxisG& c, bool coarsened) {
  XferAxis t{};
  t.coarsened = coarsened ? 1 : 0;
  t.nf = f.n; t.nc = c.n;
  t.Hf = (float)f.H; t.hlf = (float)f.hl;
  t.Hc = (float)c.H; t.hlc = (float)c.hl;
  return t;
}

// cyclic Jacobi eigen-decomposition of a symmetric n x n matrix (row-major), n <= 64
void jacobi_eig(int n, std::vector<double>& A, std::vector<double>& Q, std::vector<double>& lam) {
  Q.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double v = A[(size_t)i * n + j] * A[(size_t)i * n + j];
        tot += v;
        if (i != j) off += v;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[(size_t)p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // columns p, q
          const double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
          A[(size_t)k * n + p] = c * akp - s * akq;
          A[(size_t)k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // rows p, q
          const double apk = A[(size_t)p * n + k], aqk = A[(size_t)q * n + k];
          A[(size_t)p * n + k] = c * apk - s * aqk;
          A[(size_t)q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double qkp = Q[(size_t)k * n + p], qkq = Q[(size_t)k * n + q];
          Q[(size_t)k * n + p] = c * qkp - s * qkq;
          Q[(size_t)k * n + q] = s * qkp + c * qkq;
        }
      }
  }
  lam.resize(n);
  for (int i = 0; i < n; ++i) lam[i] = A[(size_t)i * n + i];
  // sort ascending (column permutation of Q)
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return lam[a] < lam[b]; });
  std::vector<double> Q2((size_t)n * n), l2(n);
  for (int k = 0; k < n; ++k) {
    l2[k] = lam[idx[k]];
    for (int i = 0; i < n; ++i) Q2[(size_t)i * n + k] = Q[(size_t)i * n + idx[k]];
  }
  Q.swap(Q2);
  lam.swap(l2);
}

// Per-axis fast-diagonalisation factors of the 1D finite-volume operator T of an axis.
// T = D^-1 S with S symmetric (D = diag of cell widths) -> M = D^1/2 T D^-1/2 = Q L Q^T,
// forward F = Q^T D^1/2 (row k = mode), backward B = D^-1/2 Q.
static void fd_axis(const AxisG& g, std::vector<float>& F, std::vector<float>& B,
                    std::vector<float>& lamf, double& lmax) {
  const int n = g.n;
  const AxisC a = make_axisc(g);
  std::vector<double> h(n), T((size_t)n * n, 0.0);
  const double dl = 0.5 * (g.H + g.hl);
  for (int i = 0; i < n; ++i) h[i] = (i == n - 1) ? g.hl : g.H;
  auto cld = [&](int i) -> double {
    if (i <= 0) return 0.0;
    return i == n - 1 ? g.beta / (dl * g.hl) : g.beta / (g.H * g.H);
  };
  auto crd = [&](int i) -> double {
    if (i >= n - 1) return 0.0;
    return i == n - 2 ? g.beta / (dl * g.H) : g.beta / (g.H * g.H);
  };
  (void)a;
  for (int i = 0; i < n; ++i) {
    T[(size_t)i * n + i] = cld(i) + crd(i);
    if (i > 0) T[(size_t)i * n + i - 1] = -cld(i);
    if (i < n - 1) T[(size_t)i * n + i + 1] = -crd(i);
  }
  std::vector<double> M((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) M[(size_t)i * n + j] = std::sqrt(h[i]) * T[(size_t)i * n + j] / std::sqrt(h[j]);
  // symmetrise exactly
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double v = 0.5 * (M[(size_t)i * n + j] + M[(size_t)j * n + i]);
      M[(size_t)i * n + j] = M[(size_t)j * n + i] = v;
    }
  std::vector<double> Q, lam;
  jacobi_eig(n, M, Q, lam);
  F.resize((size_t)n * n);
  B.resize((size_t)n * n);
  lamf.resize(n);
  lmax = 0.0;
  for (int k = 0; k < n; ++k) {
    lamf[k] = (float)std::max(lam[k], 0.0);
    lmax = std::max(lmax, lam[k]);
    for (int i = 0; i < n; ++i) {
      F[(size_t)k * n + i] = (float)(Q[(size_t)i * n + k] * std::sqrt(h[i]));
      B[(size_t)i * n + k] = (float)(Q[(size_t)i * n + k] / std::sqrt(h[i]));
    }
  }
}

// ---------------------------------------------------------------------------------
// hierarchy
// ---------------------------------------------------------------------------------
Hier::~Hier() {
  for (auto& L : lv) {
    if (L.own_x && L.x) cudaFree(L.x);
    if (L.b) cudaFree(L.b);
    if (L.x2) cudaFree(L.x2);
    if (L.xlo) cudaFree(L.xlo);
    if (L.xhi) cudaFree(L.xhi);
  }
  for (float* p : dev_tables) cudaFree(p);
  if (partials) cudaFree(partials);
  if (plane_sums) cudaFree(plane_sums);
  if (scratch_e) cudaFree(scratch_e);
  if (b0) cudaFree(b0);
  if (h_plane) cudaFreeHost(h_plane);
  if (dx_dev) cudaFree(dx_dev);
  if (dx_host) cudaFreeHost(dx_host);
  if (xprev) cudaFree(xprev);
  if (coop_dev) cudaFree(coop_dev);
  for (auto& g : graphs)
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
}

static int upload(std::vector<float*>& owned, const std::vector<float>& v, const float** out) {
  float* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(float)));
  owned.push_back(p);
  if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice));
  *out = p;
  return GDP_OK;
}

// One coarsening step of the single-rank rule: axes whose coupling
// beta_d / H_d^2 is >= 1/2 of the strongest coupled axis are halved (ceil).  Returns false
// when F is the coarsest level (<= coarse_max unknowns per system, <= 64 cells per axis).
static bool coarsen_step(const Level& F, int coarse_max, size_t nlev, Level& C, bool co[3]) {
  const AxisG* g[3] = {&F.gx, &F.gy, &F.gz};
  double s[3];
  bool cpl[3];
  long long size = 1;
  int maxn = 1;
  double smax = 0.0;
  for (int d = 0; d < 3; ++d) {
    cpl[d] = g[d]->beta > 0.0 && g[d]->n > 1;
    s[d] = cpl[d] ? g[d]->beta / (g[d]->H * g[d]->H) : 0.0;
    if (cpl[d]) { size *= g[d]->n; maxn = std::max(maxn, g[d]->n); smax = std::max(smax, s[d]); }
  }
  if (!(cpl[0] || cpl[1] || cpl[2])) return false;
  if (size <= coarse_max && maxn <= 64 && nlev > 1) return false;
  if (size <= coarse_max && maxn <= 64 && size <= 64) return false;  // tiny: solve directly
  if ((int)nlev >= GDP_MAX_LEVELS) return false;
  for (int d = 0; d < 3; ++d) co[d] = cpl[d] && s[d] >= 0.5 * smax;
  if (!(co[0] || co[1] || co[2])) return false;
  C = Level();
  C.gx = co[0] ? coarsen_axis(F.gx) : F.gx;
  C.gy = co[1] ? coarsen_axis(F.gy) : F.gy;
  C.gz = co[2] ? coarsen_axis(F.gz) : F.gz;
  C.tx = make_xfer(F.gx, C.gx, co[0]);
  C.ty = make_xfer(F.gy, C.gy, co[1]);
  C.tz = make_xfer(F.gz, C.gz, co[2]);
  C.nx = C.gx.n; C.ny = C.gy.n;
  C.nzl = C.gz.n; C.z0 = 0;  // full in z unless the caller keeps it split
  return true;
}

// level geometry chain of a (possibly z-split) grid.  Levels stay split while z coarsening
// keeps every slab aligned (even z0 and nzl), the slab keeps >= 2 planes and the level is
// not the coarsest; from the first level that cannot, all levels are full in z.  The global
// geometry of every level is the single-rank one, so the V-cycle is partition-independent.
int level_chain(const HierKey& key, std::vector<Level>& lv, int& first_full) {
  lv.clear();
  Level L0;
  L0.gx = AxisG{(int)key.nx, 1.0, 1.0, key.bx};
  L0.gy = AxisG{(int)key.ny, 1.0, 1.0, key.by};
  L0.gz = AxisG{(int)key.nzg, 1.0, 1.0, key.bz};
  L0.nx = (int)key.nx; L0.ny = (int)key.ny; L0.nzl = (int)key.nzl; L0.z0 = key.z0;
  lv.push_back(L0);
  first_full = key.nzl == key.nzg ? 0 : -1;
  for (;;) {
    const Level& F = lv.back();
    Level C;
    bool co[3];
    if (!coarsen_step(F, key.coarse_max, lv.size(), C, co)) break;
    if (first_full < 0) {
      const bool aligned = !co[2] || (F.nzl % 2 == 0 && F.z0 % 2 == 0);
      const int nzl = co[2] ? F.nzl / 2 : F.nzl;
      const long long z0 = co[2] ? F.z0 / 2 : F.z0;
      Level C2;
      bool co2[3];
      const bool coarsest = !coarsen_step(C, key.coarse_max, lv.size() + 1, C2, co2);
      // C may stay split only if the step after it (which may gather) is slab-local too
      const bool next_ok = coarsest || !co2[2] || (nzl % 2 == 0 && z0 % 2 == 0);
      if (aligned && nzl >= 2 && !coarsest && next_ok) {
        C.nzl = nzl;
        C.z0 = z0;
      } else {
        first_full = (int)lv.size();
      }
    }
    lv.push_back(C);
  }
  if (first_full < 0) return set_err(GDP_EINVAL, "z-split hierarchy never becomes full");
  return GDP_OK;
}

// Allocate a hierarchy over levels [from, end) of `chain` (level `from` becomes lv[0]).  If
// own0, level 0 gets its own x and b (a gathered coarse level); else x0 is the caller's.
int build_hier_levels(const HierKey& key, const std::vector<Level>& chain, int from, int end, bool own0,
                      bool coarsest_here, std::unique_ptr<Hier>& out);

int build_hier(const HierKey& key, std::unique_ptr<Hier>& out) {
  std::vector<Level> chain;
  int ff;
  RET(level_chain(key, chain, ff));
  if (ff != 0) return set_err(GDP_EINVAL, "build_hier: z-split grid needs the distributed driver");
  return build_hier_levels(key, chain, 0, (int)chain.size(), false, true, out);
}

int build_hier_levels(const HierKey& key, const std::vector<Level>& chain, int from, int end, bool own0,
                      bool coarsest_here, std::unique_ptr<Hier>& out) {
  auto H = std::make_unique<Hier>();
  H->key = key;
  for (int l = from; l < end; ++l) H->lv.push_back(chain[l]);
  // device buffers and kernel-side coefficients
  long long maxplanes = 0;
  for (size_t l = 0; l < H->lv.size(); ++l) {
    Level& L = H->lv[l];
    L.K.nx = L.nx; L.K.ny = L.ny; L.K.nzl = L.nzl; L.K.z0 = L.z0;
    L.K.ax = make_axisc(L.gx); L.K.ay = make_axisc(L.gy); L.K.az = make_axisc(L.gz);
    L.K.alpha = (float)key.alpha;
    L.K.omega = key.omega;
    const size_t n = (size_t)L.nx * L.ny * L.nzl;
    if (l > 0 || own0) {
      CK(cudaMalloc(&L.x, n * sizeof(float)));
      L.own_x = true;
      CK(cudaMalloc(&L.b, n * sizeof(float)));
    }
    if (L.nzl != L.gz.n) {  // z-split level: ghost planes of x (halo exchange)
      const size_t pl = (size_t)L.nx * L.ny;
      CK(cudaMalloc(&L.xlo, pl * sizeof(float)));
      CK(cudaMalloc(&L.xhi, pl * sizeof(float)));
      CK(cudaMemset(L.xlo, 0, pl * sizeof(float)));
      CK(cudaMemset(L.xhi, 0, pl * sizeof(float)));
    }
    maxplanes = std::max<long long>(maxplanes, L.nzl);
  }
  const int nl = (int)H->lv.size();
  Level& Lc = H->lv[nl - 1];
  if (!coarsest_here) {
    // the coarsest solve lives in another (gathered) hierarchy
    int per = norms_blocks_per_plane(H->lv[0].nx, H->lv[0].ny);
    H->partials_cap = (size_t)per;
    CK(cudaMalloc(&H->partials, (size_t)per * std::max<long long>(maxplanes, 1) * sizeof(double2)));
    CK(cudaMalloc(&H->plane_sums, (size_t)std::max<long long>(maxplanes, 1) * sizeof(double2)));
    CK(cudaMallocHost(&H->h_plane, (size_t)std::max<long long>(maxplanes, 1) * sizeof(double2)));
    out = std::move(H);
    return GDP_OK;
  }
  if (nl == 1) {  // direct solve of level 0: residual / correction scratch
    const size_t n = (size_t)Lc.nx * Lc.ny * Lc.nzl;
    if (!Lc.b) CK(cudaMalloc(&Lc.b, n * sizeof(float)));
    CK(cudaMalloc(&H->scratch_e, n * sizeof(float)));
  }
  // coarsest fast diagonalisation
  CoarseK C{};
  C.nx = Lc.nx; C.ny = Lc.ny; C.nz = Lc.nzl;
  C.cx = Lc.gx.beta > 0 && Lc.gx.n > 1;
  C.cy = Lc.gy.beta > 0 && Lc.gy.n > 1;
  C.cz = Lc.gz.beta > 0 && Lc.gz.n > 1;
  if (C.cz && Lc.nzl != Lc.gz.n)
    return set_err(GDP_EINVAL, "coarsest level split across ranks (agglomeration not built)");
  C.alpha = (float)key.alpha;
  double lsum = 0.0;
  const AxisG* ga[3] = {&Lc.gx, &Lc.gy, &Lc.gz};
  const float** Fp[3] = {&C.Fx, &C.Fy, &C.Fz};
  const float** Bp[3] = {&C.Bx, &C.By, &C.Bz};
  const float** lp[3] = {&C.lx, &C.ly, &C.lz};
  const int cflag[3] = {C.cx, C.cy, C.cz};
  for (int d = 0; d < 3; ++d) {
    if (!cflag[d]) { *Fp[d] = *Bp[d] = *lp[d] = nullptr; continue; }
    std::vector<float> F, B, lam;
    double lmax;
    fd_axis(*ga[d], F, B, lam, lmax);
    lsum += lmax;
    RET(upload(H->dev_tables, F, Fp[d]));
    RET(upload(H->dev_tables, B, Bp[d]));
    RET(upload(H->dev_tables, lam, lp[d]));
  }
  C.lam_thr = key.alpha > 0 ? -1.f : (float)(1e-9 * std::max(lsum, 1e-30));
  const long long nsys = (long long)C.nx * C.ny * (C.cz ? C.nz : 1);
  if ((nsys * 2 + (long long)C.nx * (C.nx + 1)) * sizeof(float) > 200 * 1024)
    return set_err(GDP_EINVAL, "coarsest system of %lld unknowns exceeds shared memory", nsys);
  H->coarse = C;
  // norm partials: level-0 plane rows
  int per = std::max(norms_blocks_per_plane(H->lv[0].nx, H->lv[0].ny), init_blocks_per_plane(H->lv[0].nx, H->lv[0].ny));
  if (nl > 1)
    for (int nu = 1; nu <= 2; ++nu) per = std::max(per, fused_tiles_per_plane(nu, H->lv[0], H->lv[1]));
  H->partials_cap = (size_t)per;
  CK(cudaMalloc(&H->partials, (size_t)per * std::max<long long>(maxplanes, 1) * sizeof(double2)));
  CK(cudaMalloc(&H->plane_sums, (size_t)std::max<long long>(maxplanes, 1) * sizeof(double2)));
  CK(cudaMallocHost(&H->h_plane, (size_t)std::max<long long>(maxplanes, 1) * sizeof(double2)));
  out = std::move(H);
  return GDP_OK;
}

// ---------------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------------
Ctx::~Ctx() {
  hier.clear();
  if (scheme_cache) scheme_cache_destroy(scheme_cache);
  if (h16) cudaFreeHost(h16);
  dist.clear();
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (scratch) cudaFree(scratch);
  for (int i = 0; i < 3; ++i)
    if (hbuf[i]) cudaFree(hbuf[i]);
  if (hs) cudaStreamDestroy(hs);
  if (hcs) cudaStreamDestroy(hcs);
  if (hev) cudaEventDestroy(hev);
}

int Ctx::ensure_hbuf(int i, size_t bytes) {
  if (hbuf_cap[i] >= bytes) return GDP_OK;
  if (hbuf[i]) cudaFree(hbuf[i]);
  hbuf[i] = nullptr;
  hbuf_cap[i] = 0;
  CK(cudaMalloc(&hbuf[i], bytes));
  hbuf_cap[i] = bytes;
  return GDP_OK;
}

int Ctx::get_hier(const HierKey& k, Hier** out) {
  auto it = hier.find(k);
  if (it != hier.end()) { *out = it->second.get(); return GDP_OK; }
  std::unique_ptr<Hier> H;
  RET(build_hier(k, H));
  *out = H.get();
  hier[k] = std::move(H);
  return GDP_OK;
}

int Ctx::ensure_scratch(size_t bytes) {
  if (scratch_bytes >= bytes) return GDP_OK;
  if (scratch) cudaFree(scratch);
  scratch = nullptr;
  scratch_bytes = 0;
  CK(cudaMalloc(&scratch, bytes));
  scratch_bytes = bytes;
  return GDP_OK;
}

// ---------------------------------------------------------------------------------
// V-cycle (reference schedule; the fused schedule replaces the level passes)
// ---------------------------------------------------------------------------------
static int smooth(const Level& L, float* x, const RhsK& R, int mode, int tI, int nu, cudaStream_t s) {
  for (int k = 0; k < nu; ++k)
    for (int color = 0; color < 2; ++color)
      launch_rbgs(L.K, x, L.xlo, L.xhi, R, mode, tI, color, s);
  return GDP_OK;
}

// flags: RV_PROLONG — level l0 starts from the prolongation of level l0+1's x (added to the
// caller's x at level 0, to zero above) instead of zero / the caller's iterate (FMG start)
int run_vcycle(Ctx& ctx, Hier& H, const Fine& f, const gdp_opts& o, cudaStream_t s, int l0, unsigned flags) {
  const int nl = (int)H.lv.size();
  if (nl == 1) {  // level 0 is the coarsest: x += A^-1 (b - A x)
    Level& L = H.lv[0];
    launch_norms(L.K, f.x, L.xlo, L.xhi, f.R, f.mode, f.tI, L.b, H.partials, H.plane_sums, s);
    CK(launch_coarse(H.coarse, L.b, H.scratch_e, s));
    launch_axpy(f.x, H.scratch_e, (long long)L.nx * L.ny * L.nzl, s);
    return GDP_OK;
  }
  H.up_norm_per = 0;
  H.up_norm_planes = 0;
  // per level: 0 reference schedule, 2 fused 2D passes, 3 fused 3D sweeps
  int fz[GDP_MAX_LEVELS] = {0};
  float* cur[GDP_MAX_LEVELS] = {nullptr};  // buffer holding x of a level after its down pass
  const bool nu_ok = o.nu_pre >= 1 && o.nu_post >= 1;
  for (int l = l0; l < nl - 1; ++l) {
    Level& L = H.lv[l];
    Level& C = H.lv[l + 1];
    const bool rhs_ok = l > 0 || f.mode == RHS_B;
    if (rhs_ok && fusable2d(L, C, o)) fz[l] = 2;
    else if (rhs_ok && nu_ok && fusable3d(L, C, o)) fz[l] = 3;
    if (fz[l] && !L.x2) CK(cudaMalloc(&L.x2, sizeof(float) * (size_t)L.nx * L.ny * L.nzl));
  }
  // the coarse tail [lc, nl - 1): single-slab levels under the size threshold run in two cooperative
  // launches (fused bit 8); lc = nl - 1: none
  int lc = nl - 1;
  if (o.fused & 8) {
    static const long long cmax = getenv("GDP_COOP_MAX") ? atoll(getenv("GDP_COOP_MAX")) : 2000000LL;
    for (int l = nl - 2; l >= std::max(l0, 1); --l) {
      const Level& L = H.lv[l];
      if ((long long)L.nx * L.ny * L.nzl >= cmax || L.nzl != L.gz.n || L.xlo) break;
      lc = l;
    }
    if (lc < nl - 1 && !H.coop_dev) {  // the levels' device views, once per hierarchy (before any capture)
      std::vector<CoopLv> v(nl - 1);
      for (int l = 1; l < nl - 1; ++l) {
        const Level& L = H.lv[l];
        const Level& C = H.lv[l + 1];
        v[l - 1] = CoopLv{L.K, L.x, L.b, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.b, C.x};
      }
      CK(cudaMalloc(&H.coop_dev, sizeof(CoopLv) * v.size()));
      CK(cudaMemcpy(H.coop_dev, v.data(), sizeof(CoopLv) * v.size(), cudaMemcpyHostToDevice));
    }
  }
  for (int l = l0; l < nl - 1; ++l) {
    Level& L = H.lv[l];
    Level& C = H.lv[l + 1];
    float* x = l == 0 ? f.x : L.x;
    RhsK R = f.R;
    int mode = f.mode, tI = f.tI;
    if (l > 0) {
      R = RhsK{L.b, nullptr, nullptr, 0.f, 0};
      mode = RHS_B;
      tI = 1;
    }
    if (l >= lc) {  // the cooperative down walk over [lc, nl - 1)
      const bool pro = l == l0 && (flags & RV_PROLONG);
      if (pro) {  // FMG start at l0: x = P x_{l0+1} (zero + correction), then the walk without zeroing
        CK(cudaMemsetAsync(x, 0, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, s));
        launch_prolong(L.K, x, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
      }
      double cells = 0.0;
      for (int q = lc; q < nl - 1; ++q) cells += (double)H.lv[q].nx * H.lv[q].ny * H.lv[q].nzl;
      CK(launch_coop(true, H.coop_dev + (lc - 1), nl - 1 - lc, o.nu_pre, pro ? 0 : 1, nullptr, cells,
                     cells * 4.0 * (2.0 * o.nu_pre + 2.0), s));
      break;
    }
    // FMG start at l0: x (zeroed above level 0) += P x_{l0+1}, in the first fused 3D sweep
    // when there is one to carry it, else by the prolongation kernel
    const bool pro = l == l0 && (flags & RV_PROLONG);
    // the temporally blocked pass (fused & 4): all nu_pre sweeps + restriction in one HBM pass,
    // the FMG prolongation added at load
    const bool vp = fz[l] == 3 && (o.fused & 4) &&
                    vpass3d_ok(L, C, o.nu_pre, pro, 1, x, L.x2, l == 0 ? R.b : L.b);
    const bool pro_fused = pro && ((fz[l] == 3 && o.nu_pre >= 2 && l == 0) || fz[l] == 2 || vp);
    if (pro && !vp) {
      if (l > 0) CK(cudaMemsetAsync(x, 0, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, s));
      if (!pro_fused) launch_prolong(L.K, x, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
    }
    const bool zx = l > 0 && (!pro || vp);  // above level 0 x starts from zero (+ P e at l0 under FMG)
    if (vp) {  // one pass: x (A) -> x2 (B), restricted residual into C.b
      const int nu = o.nu_pre;
      RET(fused_pass3d(L, C, x, L.x2, R.b, zx, pro, nu, 1, nullptr, l == 0 ? H.dx_dev : nullptr, s, nullptr));
      cur[l] = L.x2;
      continue;
    }
    if (fz[l] == 2) {  // one fused pass: x (A) -> x2 (B)
      fused_down2d(L, C, x, L.x2, R, mode, tI, o.nu_pre, zx, s, pro_fused);
      cur[l] = L.x2;
      continue;
    }
    if (fz[l] == 3) {  // nu fused sweeps, the last one restricting; ping-pong A <-> B
      float* c = x;
      for (int k = 0; k < o.nu_pre; ++k) {
        float* d = c == x ? L.x2 : x;
        const int tl = k == o.nu_pre - 1 ? 1 : 0;
        const bool pk = pro_fused && k == 0;
        if ((o.fused & 16) && vpass3d_ok(L, C, 1, pk, tl, c, d, R.b))  // one TMA-staged sweep per launch
          RET(fused_pass3d(L, C, c, d, R.b, zx && k == 0, pk, 1, tl, nullptr, nullptr, s, nullptr));
        else if ((o.fused & 32) && sweep3dv_ok(L, C, pk, c, d, R.b))  // vertical-pack z-march
          RET(fused_sweep3dv(L, C, c, d, R.b, zx && k == 0, pk, tl, nullptr, s, nullptr));
        else
          fused_sweep3d(L, C, c, d, R.b, zx && k == 0, pk, tl, nullptr, s);
        c = d;
      }
      cur[l] = c;
      continue;
    }
    if (zx) CK(cudaMemsetAsync(x, 0, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, s));
    smooth(L, x, R, mode, tI, o.nu_pre, s);
    launch_restrict(L.K, x, L.xlo, L.xhi, R, mode, tI, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.b, s);
    cur[l] = x;
  }
  Level& Lc = H.lv[nl - 1];
  CK(launch_coarse(H.coarse, Lc.b, Lc.x, s));
  if (lc < nl - 1) {  // the cooperative up walk over (nl - 1, lc]
    double cells = 0.0;
    for (int q = lc; q < nl - 1; ++q) cells += (double)H.lv[q].nx * H.lv[q].ny * H.lv[q].nzl;
    CK(launch_coop(false, H.coop_dev + (lc - 1), nl - 1 - lc, o.nu_post, 0, nullptr, cells,
                   cells * 4.0 * (2.0 * o.nu_post + 2.0), s));
  }
  for (int l = std::min(nl - 2, lc - 1); l >= l0; --l) {
    Level& L = H.lv[l];
    Level& C = H.lv[l + 1];
    float* x = l == 0 ? f.x : L.x;
    RhsK R = f.R;
    int mode = f.mode, tI = f.tI;
    if (l > 0) { R = RhsK{L.b, nullptr, nullptr, 0.f, 0}; mode = RHS_B; tI = 1; }
    if (fz[l] == 2) {  // one fused pass: x2 (B) -> x (A), norms of the finest level on the way
      const int per2 = fused_tiles_per_plane(o.nu_post, L, C);
      const bool want = l == 0 && (size_t)per2 <= H.partials_cap;
      fused_up2d(L, C, L.x2, x, R, mode, tI, o.nu_post, want ? H.partials : nullptr, s);
      if (want) { H.up_norm_per = per2; H.up_norm_planes = L.nzl; }
      continue;
    }
    if (fz[l] == 3 && (o.fused & 4) && cur[l] != x &&
        vpass3d_ok(L, C, o.nu_post, true, l == 0 ? 2 : 0, cur[l], x, R.b)) {
      // one pass: x2 (B) + P e -> nu_post sweeps -> x (A), norms of the finest level on the way
      const int items = vpass3d_items(L, C, o.nu_post);
      const bool want = l == 0 && (size_t)items <= H.partials_cap * (size_t)L.nzl;
      int got = 0;
      RET(fused_pass3d(L, C, cur[l], x, R.b, false, true, o.nu_post, want ? 2 : 0, want ? H.partials : nullptr,
                       l == 0 ? H.dx_dev : nullptr, s, &got));
      if (want) { H.up_norm_per = got; H.up_norm_planes = 1; }
      continue;
    }
    if (fz[l] == 3) {  // prolongation fused into the first sweep, norms into the last
      float* c = cur[l];
      // coarse levels: the prolongation by its own kernel (the z-march's coarse-row loads are
      // exposed latency there: e.g. 156 vs 53 + ~25 us on a 256^2 x 128 level); the TMA-staged
      // kernels carry it
      const bool v16 = (o.fused & 16) && vpass3d_ok(L, C, 1, true, 0, c, x, R.b);
      const bool v32 = !v16 && (o.fused & 32) && sweep3dv_ok(L, C, false, c, x, R.b);
      const bool v32p = v32 && sweep3dv_ok(L, C, true, c, x, R.b);  // it also carries the prolongation
      // partial slots of the norms sweep (the kernel that runs it: its own work split)
      const int items = v32 ? sweep3dv_items(L, C) : fused3d_items(L, C);
      const bool want = l == 0 && (size_t)items <= H.partials_cap * (size_t)L.nzl;
      const bool sep = l > 0 && !v16 && !v32p;
      if (sep) launch_prolong(L.K, c, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
      int got = 0;
      for (int k = 0; k < o.nu_post; ++k) {
        float* d = c == x ? L.x2 : x;
        const bool last = k == o.nu_post - 1;
        const int tl = last && want ? 2 : 0;
        if (v16 && vpass3d_ok(L, C, 1, k == 0, tl, c, d, R.b))
          RET(fused_pass3d(L, C, c, d, R.b, false, k == 0, 1, tl, tl ? H.partials : nullptr, nullptr, s,
                           tl ? &got : nullptr));
        else if (v32 && sweep3dv_ok(L, C, k == 0 && !sep, c, d, R.b))
          RET(fused_sweep3dv(L, C, c, d, R.b, false, k == 0 && !sep, tl, tl ? H.partials : nullptr, s,
                             tl ? &got : nullptr));
        else {
          const int n = fused_sweep3d(L, C, c, d, R.b, false, k == 0 && !sep, tl, want ? H.partials : nullptr, s);
          if (tl) got = n;
        }
        c = d;
      }
      if (c != x) CK(cudaMemcpyAsync(x, c, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, cudaMemcpyDeviceToDevice, s));
      if (want) { H.up_norm_per = got > 0 ? got : items; H.up_norm_planes = 1; }
      continue;
    }
    launch_prolong(L.K, x, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
    smooth(L, x, R, mode, tI, o.nu_post, s);
  }
  CK(cudaGetLastError());
  return GDP_OK;
}

// fp64 norms of the finest level -> per-plane (sum r^2, sum b^2) on the host
int finest_norms(Ctx& ctx, Hier& H, const Fine& f, float* rout, cudaStream_t s) {
  Level& L = H.lv[0];
  launch_norms(L.K, f.x, L.xlo, L.xhi, f.R, f.mode, f.tI, rout, H.partials, H.plane_sums, s);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(H.h_plane, H.plane_sums, sizeof(double2) * L.nzl, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return GDP_OK;
}

// rel-res of the current iterate: one system (all planes) or max over slices
static double rel_from_planes(const Hier& H, bool per_slice, double* worst_b) {
  const int nz = H.lv[0].nzl;
  if (!per_slice) {
    double rr = 0.0, bb = 0.0;
    for (int z = 0; z < nz; ++z) { rr += H.h_plane[z].x; bb += H.h_plane[z].y; }
    if (worst_b) *worst_b = std::sqrt(bb);
    return bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
  }
  double worst = 0.0, wb = 0.0;
  for (int z = 0; z < nz; ++z) {
    const double rr = H.h_plane[z].x, bb = H.h_plane[z].y;
    const double v = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
    if (v >= worst) { worst = v; wb = std::sqrt(bb); }
  }
  if (worst_b) *worst_b = wb;
  return worst;
}

// FMG start: the init pass restricts r0 into level 1 on the way when the coarsening is plane-local
static InitXfer init_xfer(Hier& H, const gdp_opts& o) {
  InitXfer X;
  H.init_restricted = false;
  if ((o.fmg & 3) == 0 || (o.fmg & 4) || H.lv.size() < 3 || H.lv[1].tz.coarsened) return X;
  const Level& C = H.lv[1];
  X.tx = C.tx; X.ty = C.ty; X.ncx = C.nx; X.ncy = C.ny; X.bc = C.b;
  H.init_restricted = true;
  return X;
}

// FMG start (nested iteration) for the correction equation A e = r0 of the first cycle:
// r0 = b - A x0 restricted to level 1, the right-hand side restricted on down to the coarsest,
// solved there, then per level l = nl-2 .. 1 a prolongation of e_{l+1} and one V-cycle on
// levels l.. (run_vcycle l0 = l).  Leaves e_1 in lv[1].x; the caller's first fine cycle
// prolongates it into x (RV_PROLONG).
static int fmg_start(Ctx& ctx, Hier& H, const Fine& f, const gdp_opts& o, bool r0_restricted, cudaStream_t s) {
  const int nl = (int)H.lv.size();
  Level& L0 = H.lv[0];
  Level& L1 = H.lv[1];
  if (!r0_restricted)
    launch_restrict(L0.K, f.x, L0.xlo, L0.xhi, f.R, f.mode, f.tI, L1.tx, L1.ty, L1.tz, L1.nx, L1.ny, L1.nzl, L1.b, s);
  for (int l = 1; l < nl - 1; ++l) {  // b_{l+1} = R b_l: the restricted residual of x_l = 0
    Level& L = H.lv[l];
    Level& C = H.lv[l + 1];
    launch_restrict_b(L.K, L.b, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.b, s);
  }
  Level& Lc = H.lv[nl - 1];
  CK(launch_coarse(H.coarse, Lc.b, Lc.x, s));
  // fmg 1: one V-cycle per level 1..nl-2; fmg 2 / 3: V-cycles from level 2 only, level 1 gets
  // the prolongation of e_2 followed by nu_post red-black sweeps (2) or nothing (3)
  const int mode = o.fmg & 3;
  const int lmin = mode == 1 ? 1 : 2;
  // the nested cycles take one post-smoothing sweep fewer (phase 1: V(2,1) instead of V(2,2),
  // 0.33 ms less on config 1, final rel-res 6.2e-7 instead of 5.9e-7 after the same 3 cycles;
  // V(1,1) saves 0.84 ms but ends at 8.1e-7, too close to the gate: tools/fmg_nu.py)
  gdp_opts on = o;
  on.nu_post = std::max(1, o.nu_post - 1);
  for (int l = nl - 2; l >= lmin; --l) RET(run_vcycle(ctx, H, f, on, s, l, RV_PROLONG));
  for (int l = lmin - 1; l >= 1; --l) {
    Level& L = H.lv[l];
    Level& C = H.lv[l + 1];
    CK(cudaMemsetAsync(L.x, 0, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, s));
    launch_prolong(L.K, L.x, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
    if (mode == 2) smooth(L, L.x, RhsK{L.b, nullptr, nullptr, 0.f, 0}, RHS_B, 1, o.nu_post, s);
  }
  return GDP_OK;
}

// full solve: cycles until rel_tol / cap / stagnation (a9)
int solve(Ctx& ctx, Hier& H, const Fine& f, const gdp_opts& o, bool per_slice, gdp_report* rep,
          cudaStream_t s) {
  gdp_report r{};
  r.levels = (int)H.lv.size();
  const bool r0_restricted = H.init_restricted;  // only the init pass just before this solve
  H.init_restricted = false;
  g_prof_finest = (double)H.lv[0].nx * H.lv[0].ny * H.lv[0].nzl;
  g_prof_l1 = H.lv.size() > 1 ? (double)H.lv[1].nx * H.lv[1].ny * H.lv[1].nzl : 0.0;
  if (H.init_norm_per > 0) {  // the initial residual came with launch_init
    launch_finalize(H.partials, H.init_norm_per, H.lv[0].nzl, H.plane_sums, s);
    CK(cudaMemcpyAsync(H.h_plane, H.plane_sums, sizeof(double2) * H.lv[0].nzl, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    H.init_norm_per = 0;
  } else {
    RET(finest_norms(ctx, H, f, nullptr, s));
  }
  double nb = 0.0;
  double rel = rel_from_planes(H, per_slice, &nb);
  r.rel_res[0] = rel;
  r.norm_b = nb;
  if (!std::isfinite(rel)) return set_err(GDP_EINVAL, "non-finite initial residual (non-finite input?)");
  int status = GDP_OK;
  int stall = 0;
  int k = 0;
  const int cap = std::min(o.max_vcycles, GDP_MAX_CYCLES);
  // a9 correction norm: x_{k-1} is kept before a cycle predicted to end the solve and
  // ||x_k - x_{k-1}||_inf measured after it
  const bool dxg = o.dx_tol > 0.0;
  const size_t n0 = (size_t)H.lv[0].nx * H.lv[0].ny * H.lv[0].nzl;
  double dx = 0.0;   // of the last cycle (none yet: no correction); < 0: not measured
  r.dx_inf = 0.0;
  auto done = [&](double rl) { return rl <= o.rel_tol && (!dxg || (dx >= 0.0 && dx <= o.dx_tol)); };
  // one cycle's GPU work, ending with the D2H of its norms (and dx); no host synchronisation inside,
  // so that it can be captured as a CUDA graph (gdp_opts.use_graphs) and replayed by later solves
  auto enqueue = [&](bool fmg, bool keep) -> int {
    if (keep) {
      CK(cudaMemcpyAsync(H.xprev, f.x, n0 * sizeof(float), cudaMemcpyDeviceToDevice, s));
      CK(cudaMemsetAsync(H.dx_dev, 0, sizeof(unsigned int), s));
    }
    if (fmg) RET(fmg_start(ctx, H, f, o, r0_restricted, s));
    RET(run_vcycle(ctx, H, f, o, s, 0, fmg ? RV_PROLONG : 0u));
    H.warm = true;
    if (keep) {
      launch_maxdiff(f.x, H.xprev, (long long)n0, H.dx_dev, s);
      CK(cudaMemcpyAsync(H.dx_host, H.dx_dev, sizeof(unsigned int), cudaMemcpyDeviceToHost, s));
    }
    if (H.up_norm_per > 0) {  // norms of the final iterate came with the fused up pass
      launch_finalize(H.partials, H.up_norm_per, H.up_norm_planes, H.plane_sums, s);
      CK(cudaMemcpyAsync(H.h_plane, H.plane_sums, sizeof(double2) * H.up_norm_planes, cudaMemcpyDeviceToHost, s));
    } else {
      Level& L = H.lv[0];
      launch_norms(L.K, f.x, L.xlo, L.xhi, f.R, f.mode, f.tI, nullptr, H.partials, H.plane_sums, s);
      CK(cudaMemcpyAsync(H.h_plane, H.plane_sums, sizeof(double2) * L.nzl, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaGetLastError());
    return GDP_OK;
  };
  // graphs need a non-legacy stream, buffers that already exist, and no profiler events
  const bool graphs = o.use_graphs && s != nullptr && f.mode == RHS_B && !g_prof_on;
  const long long okey = ((long long)o.nu_pre << 40) ^ ((long long)o.nu_post << 32) ^ ((long long)o.fused << 24) ^
                         ((long long)o.fmg << 16) ^ (long long)H.lv.size();
  while (!done(rel)) {
    if (k >= cap) { status = GDP_ENOCONV; break; }
    const bool fmg = k == 0 && (o.fmg & 3) != 0 && H.lv.size() >= 3;
    // keep x_{k-1} when this cycle is predicted to pass the residual gate: rel-res times the last
    // observed contraction (at least 0.05) within 3x of rel_tol (a cycle that passes unmeasured is
    // followed by a measured one)
    const double rho = k > 0 && r.rel_res[k - 1] > 0.0 ? std::min(1.0, std::max(0.05, rel / r.rel_res[k - 1])) : 1.0;
    const bool keep = dxg && (rel * rho <= 3.0 * o.rel_tol || rel <= o.rel_tol);
    if (keep) {
      if (!H.xprev) CK(cudaMalloc(&H.xprev, n0 * sizeof(float)));
      if (!H.dx_dev) CK(cudaMalloc(&H.dx_dev, sizeof(unsigned int)));
      if (!H.dx_host) CK(cudaMallocHost(&H.dx_host, sizeof(unsigned int)));
    }
    bool ran = false;
    if (graphs && H.warm) {
      const long long vkey = okey ^ ((long long)fmg << 1) ^ ((long long)keep << 2) ^ ((long long)r0_restricted << 3);
      auto key = std::make_tuple((const void*)f.x, (const void*)f.R.b, vkey);
      auto it = H.graphs.find(key);
      if (it == H.graphs.end()) {  // capture once
        Hier::CycleGraph G;
        const long long l0 = g_launches.load();
        cudaGraph_t gr = nullptr;
        if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
          const int rc = enqueue(fmg, keep);
          const cudaError_t ce = cudaStreamEndCapture(s, &gr);
          if (rc == GDP_OK && ce == cudaSuccess && gr && cudaGraphInstantiate(&G.exec, gr, 0) == cudaSuccess) {
            G.up_norm_per = H.up_norm_per;
            G.up_norm_planes = H.up_norm_planes;
            G.launches = g_launches.load() - l0;
            it = H.graphs.emplace(key, G).first;
          }
          if (gr) cudaGraphDestroy(gr);
        }
        const cudaError_t le = cudaGetLastError();  // a failed capture falls back to plain launches
        if (getenv("GDP_GRAPH_DEBUG"))
          fprintf(stderr, "gdp graph capture fmg=%d keep=%d ok=%d err=%s launches=%lld\n", (int)fmg, (int)keep,
                  it != H.graphs.end(), cudaGetErrorString(le), g_launches.load() - l0);
        if (it == H.graphs.end()) it = H.graphs.emplace(key, Hier::CycleGraph{}).first;  // remember the failure
        g_launches.fetch_sub(g_launches.load() - l0);  // the captured launches run below
      }
      if (it->second.exec) {
        CK(cudaGraphLaunch(it->second.exec, s));
        count_launch(it->second.launches);
        H.up_norm_per = it->second.up_norm_per;
        H.up_norm_planes = it->second.up_norm_planes;
        ran = true;
      }
    }
    if (!ran) RET(enqueue(fmg, keep));
    CK(cudaStreamSynchronize(s));
    if (H.up_norm_per > 0)
      for (int z = H.up_norm_planes; z < H.lv[0].nzl; ++z) H.h_plane[z] = make_double2(0.0, 0.0);
    const double nrel = rel_from_planes(H, per_slice, nullptr);
    ++k;
    r.rel_res[k] = nrel;
    if (!std::isfinite(nrel)) return set_err(GDP_EINVAL, "non-finite residual after V-cycle %d", k);
    if (keep) {  // read back with the norms
      float v;
      std::memcpy(&v, H.dx_host, sizeof v);
      dx = v;
    } else {
      dx = -1.0;
    }
    r.dx_inf = dx;
    if (o.stagnation > 0 && nrel > 0.9 * rel) {
      if (++stall >= o.stagnation) { rel = nrel; status = done(nrel) ? GDP_OK : GDP_ENOCONV; break; }
    } else {
      stall = 0;
    }
    rel = nrel;
  }
  r.vcycles = k;
  r.status = status;
  if (rep) {
    const double secs = rep->seconds;
    *rep = r;
    rep->seconds = secs;
  }
  return status;
}

}  // namespace gdp

// =================================================================================
// C ABI
// =================================================================================
using namespace gdp;

static bool finite_nonneg(double v) { return std::isfinite(v) && v >= 0.0; }

static int check_common(gdp_ctx* ctx, gdp_dims d, int64_t z0, int64_t nzg) {
  if (!ctx) return set_err(GDP_EINVAL, "null ctx");
  if (d.nx <= 0 || d.ny <= 0 || d.nz <= 0) return set_err(GDP_EINVAL, "dims must be positive");
  if (d.nx > (1LL << 30) || d.ny > (1LL << 30) || d.nz > 65535)
    return set_err(GDP_EINVAL, "dims too large for this build");
  if (z0 < 0 || nzg < d.nz || z0 + d.nz > nzg)
    return set_err(GDP_EINVAL, "slab [z0, z0+nz) outside [0, nz_global)");
  if (ctx->impl.world == 1 && (z0 != 0 || nzg != d.nz))
    return set_err(GDP_EINVAL, "single-rank ctx needs z0 = 0 and nz_global = nz");
  CK(cudaSetDevice(ctx->impl.device));
  return GDP_OK;
}

static int check_params(gdp_weights W, float alpha) {
  if (!finite_nonneg(W.bx) || !finite_nonneg(W.by) || !finite_nonneg(W.bz) || !finite_nonneg(alpha))
    return set_err(GDP_EINVAL, "alpha and weights must be finite and >= 0");
  if (alpha == 0.f && W.bx == 0.f && W.by == 0.f && W.bz == 0.f)
    return set_err(GDP_EINVAL, "alpha = 0 with all weights 0 is singular");
  return GDP_OK;
}

static gdp_opts resolve_opts(const gdp_opts* o) {
  gdp_opts d;
  gdp_opts_default(&d);
  if (!o) return d;
  gdp_opts r = *o;
  if (!(r.rel_tol > 0)) r.rel_tol = d.rel_tol;
  if (r.max_vcycles <= 0) r.max_vcycles = d.max_vcycles;
  if (r.nu_pre < 0) r.nu_pre = d.nu_pre;
  if (r.nu_post < 0) r.nu_post = d.nu_post;
  if (r.coarse_max <= 0) r.coarse_max = d.coarse_max;
  if (!(r.omega > 0.f && r.omega < 2.f)) r.omega = d.omega;
  if (!(r.omega_slices > 0.f && r.omega_slices < 2.f)) r.omega_slices = d.omega_slices;
  if (!(r.dx_tol >= 0.0) || !std::isfinite(r.dx_tol)) r.dx_tol = d.dx_tol;
  return r;
}

static int check_scheme(const Ctx& C, const gdp_opts& o) {
  if (o.scheme != GDP_SCHEME_HYBRID && o.scheme != GDP_SCHEME_LINEAR)
    return set_err(GDP_EINVAL, "unknown scheme %d", o.scheme);
  if (C.world > 1 || C.loop > 1) return set_err(GDP_EINVAL, "the Hybrid / Linear schemes are single-rank in this build");
  return GDP_OK;
}

static HierKey make_key(gdp_dims d, int64_t z0, int64_t nzg, gdp_weights W, float alpha,
                        const gdp_opts& o) {
  HierKey k{};
  k.nx = d.nx; k.ny = d.ny; k.nzl = d.nz; k.z0 = z0; k.nzg = nzg;
  k.bx = W.bx; k.by = W.by; k.bz = W.bz; k.alpha = alpha;
  k.coarse_max = o.coarse_max;
  k.omega = o.omega;
  return k;
}

extern "C" {

int gdp_opts_default(gdp_opts* o) {
  if (!o) return set_err(GDP_EINVAL, "null opts");
  o->rel_tol = 1e-6;
  o->max_vcycles = 30;
  o->nu_pre = 2;
  o->nu_post = 2;
  o->coarse_max = 4096;
  o->stagnation = 2;
  o->fused = 35;
  o->use_graphs = 1;
  o->nu_pre_slices = 1;
  o->nu_post_slices = 2;
  o->omega = 1.f;
  o->omega_slices = 1.f;
  o->fmg = 1;
  o->fmg_slices = 3;
  o->dx_tol = 1e-4;
  o->scheme = GDP_SCHEME_CONSTANT;
  o->half_staging = 0;
  o->stream_fuse = 1;
  return GDP_OK;
}

int gdp_ctx_create(gdp_ctx** out, int device, int rank, int world, const void* nccl_unique_id) {
  if (!out) return set_err(GDP_EINVAL, "null out");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return set_err(GDP_EINVAL, "bad rank/world");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_err(GDP_EINVAL, "bad device %d (have %d)", device, ndev);
  CK(cudaSetDevice(device));
  auto* c = new gdp_ctx();
  c->impl.device = device;
  c->impl.rank = rank;
  c->impl.world = world;
  if (world > 1) {
    int rc = comm_init(c->impl, nccl_unique_id);
    if (rc != GDP_OK) { delete c; return rc; }
  }
  cudaEventCreate(&c->impl.ev0);
  cudaEventCreate(&c->impl.ev1);
  *out = c;
  return GDP_OK;
}

int gdp_ctx_create_loopback(gdp_ctx** out, int device, int world) {
  if (!out) return set_err(GDP_EINVAL, "null out");
  *out = nullptr;
  if (world < 1) return set_err(GDP_EINVAL, "bad loopback world %d", world);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_err(GDP_EINVAL, "bad device %d (have %d)", device, ndev);
  CK(cudaSetDevice(device));
  auto* c = new gdp_ctx();
  c->impl.device = device;
  c->impl.loop = world;
  cudaEventCreate(&c->impl.ev0);
  cudaEventCreate(&c->impl.ev1);
  *out = c;
  return GDP_OK;
}

int gdp_get_unique_id(void* out, size_t n) { return comm_unique_id(out, n); }

int gdp_ctx_destroy(gdp_ctx* ctx) {
  if (!ctx) return GDP_OK;
  cudaSetDevice(ctx->impl.device);
  comm_destroy(ctx->impl);
  delete ctx;
  return GDP_OK;
}

static void fill_time(gdp_ctx* ctx, gdp_report* rep, cudaStream_t s) {
  if (!rep) return;
  cudaEventSynchronize(ctx->impl.ev1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->impl.ev0, ctx->impl.ev1);
  rep->seconds = ms * 1e-3;
  (void)s;
}

static int diffuse_z_impl(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* I1, gdp_dims local,
                          int64_t z0_global, int64_t nz_global, gdp_weights W, float alpha, const gdp_opts* opts,
                          gdp_report* report, void* stream, float* defer_shift);

int gdp_diffuse_z(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* I1, gdp_dims local,
                  int64_t z0_global, int64_t nz_global, gdp_weights W, float alpha,
                  const gdp_opts* opts, gdp_report* report, void* stream) {
  return diffuse_z_impl(ctx, I0, dtype, I1, local, z0_global, nz_global, W, alpha, opts, report, stream, nullptr);
}

// defer_shift != NULL (single rank, alpha = 0): the mean-pin shift is returned instead of applied;
// the caller applies it in phase 2's init pass (gdp_destripe)
static int diffuse_z_impl(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* I1, gdp_dims local,
                          int64_t z0_global, int64_t nz_global, gdp_weights W, float alpha, const gdp_opts* opts,
                          gdp_report* report, void* stream, float* defer_shift) {
  RET(check_common(ctx, local, z0_global, nz_global));
  RET(check_params(W, alpha));
  if (!I0 || !I1) return set_err(GDP_EINVAL, "null I0/I1");
  if ((const void*)I1 == I0) return set_err(GDP_EINVAL, "I1 may not alias I0");
  if (dtype != GDP_U8 && dtype != GDP_F32) return set_err(GDP_EINVAL, "bad dtype");
  const gdp_opts o = resolve_opts(opts);
  cudaStream_t s = (cudaStream_t)stream;
  Ctx& C = ctx->impl;
  const int tI = dtype == GDP_U8 ? 0 : 1;
  if (o.scheme != GDP_SCHEME_CONSTANT) {  // NEXT-3: Hybrid / Linear (gdp_scheme.cu)
    RET(check_scheme(C, o));
    if (defer_shift) *defer_shift = 0.f;  // the scheme path applies its mean pin itself
    return scheme_diffuse_z(C, I0, tI, I1, local.nx, local.ny, local.nz, W.bx, W.by, W.bz, alpha, o, report, s);
  }
  if (C.world > 1 || C.loop > 1) {  // z-slab partition (gdp_dist.cu)
    const int st = dist_diffuse_z(C, I0, tI, I1, local.nx, local.ny, local.nz, z0_global, nz_global, W.bx, W.by,
                                  W.bz, alpha, o, report, s);
    if (report) report->hbm_bytes_est = 0.0;
    return st;
  }
  const long long before = g_launches.load();
  Hier* H;
  RET(C.get_hier(make_key(local, z0_global, nz_global, W, alpha, o), &H));
  const long long n = local.nx * local.ny * local.nz;
  g_prof_rhs8d = tI == 0 ? 1.0 : 4.0;  // §8(d): phase 1 passes read I0 (s_in) for the rhs
  CK(cudaEventRecord(C.ev0, s));
  Fine f;
  f.x = I1;
  f.mode = RHS_G;
  f.tI = tI;
  f.R = RhsK{nullptr, I0, nullptr, alpha, alpha > 0 ? 1 : 0};
  // Eq. (1): the gradient target uses (bx, by); the rhs is formed on the fly (a2), or written
  // once (same values) together with x0 = I0 and the initial residual norms
  if (H->lv.size() > 1) {  // every schedule reads the written rhs (same values as on the fly)
    if (!H->b0) CK(cudaMalloc(&H->b0, sizeof(float) * (size_t)n));
    launch_init(H->lv[0].K, f.R, tI, I1, H->b0, H->partials, s, init_xfer(*H, o));
    H->init_norm_per = init_blocks_per_plane(H->lv[0].nx, H->lv[0].ny);
    f.mode = RHS_B;
    f.tI = 1;
    f.R = RhsK{H->b0, nullptr, nullptr, 0.f, 0};
  } else {
    launch_decode_copy(I0, tI, I1, n, s);  // x0 = I0
  }
  int st = solve(C, *H, f, o, false, report, s);
  if (st != GDP_OK && st != GDP_ENOCONV) return st;
  if (alpha == 0.f) {  // a10: pin mean(I1) = mean(I0) in fp64 (reading c-3)
    Level& L = H->lv[0];
    launch_plane_sums(I1, 1, I0, tI, L.nx, L.ny, L.nzl, H->partials, H->plane_sums, s);
    CK(cudaMemcpyAsync(H->h_plane, H->plane_sums, sizeof(double2) * L.nzl, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double sx = 0.0, si = 0.0;
    for (int z = 0; z < L.nzl; ++z) { sx += H->h_plane[z].x; si += H->h_plane[z].y; }
    RET(comm_allreduce_sum2(C, &sx, &si, s));
    const double Ntot = (double)local.nx * local.ny * nz_global;
    if (defer_shift) *defer_shift = (float)((si - sx) / Ntot);
    else launch_add_scalar(I1, n, (float)((si - sx) / Ntot), s);
  }
  CK(cudaEventRecord(C.ev1, s));
  CK(cudaGetLastError());
  if (report) {
    fill_time(ctx, report, s);
    report->kernel_launches = g_launches.load() - before;
    report->hbm_bytes_est = hbm_model(*H, tI == 0 ? 1.0 : 4.0, 0.0, report->vcycles);
  }
  if (st == GDP_ENOCONV) set_err(GDP_ENOCONV, "diffuse_z: not converged after %d V-cycles", report ? report->vcycles : -1);
  return st;
}

static int slices_impl(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, const float* I1, float* I2, gdp_dims local,
                       float alpha, const gdp_opts* opts, gdp_report* report, void* stream, const float* vshift);

int gdp_screened_poisson_slices(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, const float* I1,
                                float* I2, gdp_dims local, float alpha, const gdp_opts* opts,
                                gdp_report* report, void* stream) {
  return slices_impl(ctx, I0, dtype, I1, I2, local, alpha, opts, report, stream, nullptr);
}

// vshift != NULL: I1 += *vshift first (phase 1's deferred mean pin), written back into I1
static int slices_impl(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, const float* I1, float* I2, gdp_dims local,
                       float alpha, const gdp_opts* opts, gdp_report* report, void* stream, const float* vshift) {
  if (!ctx) return set_err(GDP_EINVAL, "null ctx");
  if (!I0 || !I1 || !I2) return set_err(GDP_EINVAL, "null I0/I1/I2");
  if (!(alpha > 0.f) || !std::isfinite(alpha)) return set_err(GDP_EINVAL, "slices need finite alpha > 0");
  if ((const void*)I2 == I0 || I2 == I1) return set_err(GDP_EINVAL, "I2 may not alias I0 or I1");
  if (dtype != GDP_U8 && dtype != GDP_F32) return set_err(GDP_EINVAL, "bad dtype");
  if (local.nx <= 0 || local.ny <= 0 || local.nz <= 0) return set_err(GDP_EINVAL, "dims must be positive");
  CK(cudaSetDevice(ctx->impl.device));
  gdp_opts o = resolve_opts(opts);
  if (o.nu_pre_slices >= 0) o.nu_pre = o.nu_pre_slices;  // per-phase smoothing (gdp.h)
  if (o.nu_post_slices >= 0) o.nu_post = o.nu_post_slices;
  o.omega = o.omega_slices;
  o.fmg = o.fmg_slices;
  cudaStream_t s = (cudaStream_t)stream;
  Ctx& C = ctx->impl;
  if (o.scheme != GDP_SCHEME_CONSTANT) {  // NEXT-3: Hybrid / Linear (gdp_scheme.cu)
    RET(check_scheme(C, o));
    return scheme_slices(C, I0, dtype == GDP_U8 ? 0 : 1, I1, I2, local.nx, local.ny, local.nz, alpha,
                         vshift ? *vshift : 0.f, o, report, s);
  }
  const long long before = g_launches.load();
  gdp_weights W{1.f, 1.f, 0.f};  // pi = Diag(1,1,0), Eq. (2)
  Hier* H;
  // slices are independent: the local slab is its own "global" stack (no halo)
  RET(C.get_hier(make_key(local, 0, local.nz, W, alpha, o), &H));
  const int tI = dtype == GDP_U8 ? 0 : 1;
  const long long n = local.nx * local.ny * local.nz;
  g_prof_rhs8d = 4.0 + (tI == 0 ? 1.0 : 4.0);  // §8(d): phase 2 passes read I1 (4) and I0 (s_in)
  CK(cudaEventRecord(C.ev0, s));
  Fine f;
  f.x = I2;
  f.mode = RHS_G;
  f.tI = tI;
  f.R = RhsK{nullptr, I0, I1, alpha, 2};
  if (H->lv.size() > 1) {
    // the passes read the rhs b = alpha I1 + (Lx + Ly) I0 (a11) written once: 4 B/cell
    // per pass instead of I0 + I1 (5 or 8 B/cell); same values as the on-the-fly form.
    // Written together with x0 = I0 and the initial residual norms.
    if (!H->b0) CK(cudaMalloc(&H->b0, sizeof(float) * (size_t)n));
    RhsK Ri = f.R;
    if (vshift) { Ri.vout = const_cast<float*>(I1); Ri.vshift = *vshift; }
    launch_init(H->lv[0].K, Ri, tI, I2, H->b0, H->partials, s, init_xfer(*H, o));
    H->init_norm_per = init_blocks_per_plane(H->lv[0].nx, H->lv[0].ny);
    f.mode = RHS_B;
    f.tI = 1;
    f.R = RhsK{H->b0, nullptr, nullptr, 0.f, 0};
  } else {
    if (vshift) launch_add_scalar(const_cast<float*>(I1), n, *vshift, s);
    launch_decode_copy(I0, tI, I2, n, s);  // x0 = I0
  }
  int st = solve(C, *H, f, o, true, report, s);
  if (st != GDP_OK && st != GDP_ENOCONV) return st;
  CK(cudaEventRecord(C.ev1, s));
  if (report) {
    fill_time(ctx, report, s);
    report->kernel_launches = g_launches.load() - before;
    report->hbm_bytes_est = hbm_model(*H, tI == 0 ? 1.0 : 4.0, 4.0, report->vcycles);
  }
  if (st == GDP_ENOCONV) set_err(GDP_ENOCONV, "screened_poisson_slices: not converged");
  return st;
}

int gdp_npr_filter(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* out, gdp_dims dims, gdp_weights W,
                   float alpha, float lambda, float sigma, const gdp_opts* opts, gdp_report* report, void* stream) {
  RET(check_common(ctx, dims, 0, dims.nz));
  RET(check_params(W, alpha));
  if (!I0 || !out) return set_err(GDP_EINVAL, "null I0/out");
  if ((const void*)out == I0) return set_err(GDP_EINVAL, "out may not alias I0");
  if (dtype != GDP_U8 && dtype != GDP_F32) return set_err(GDP_EINVAL, "bad dtype");
  if (!(alpha > 0.f)) return set_err(GDP_EINVAL, "the NPR filter is a screened solve: alpha > 0");
  if (!(sigma > 0.f) || !std::isfinite(sigma) || !std::isfinite(lambda) || lambda < 0.f)
    return set_err(GDP_EINVAL, "sigma must be finite > 0 and lambda finite >= 0");
  Ctx& C = ctx->impl;
  if (C.world > 1 || C.loop > 1) return set_err(GDP_EINVAL, "gdp_npr_filter is single-rank in this build");
  const gdp_opts o = resolve_opts(opts);
  if (o.scheme != GDP_SCHEME_CONSTANT) return set_err(GDP_EINVAL, "gdp_npr_filter runs the Constant scheme only");
  cudaStream_t s = (cudaStream_t)stream;
  const long long before = g_launches.load();
  Hier* H;
  RET(C.get_hier(make_key(dims, 0, dims.nz, W, alpha, o), &H));
  const long long n = dims.nx * dims.ny * dims.nz;
  CK(cudaEventRecord(C.ev0, s));
  if (!H->b0) CK(cudaMalloc(&H->b0, sizeof(float) * (size_t)n));
  const int tI = dtype == GDP_U8 ? 0 : 1;
  launch_npr_rhs(H->lv[0].K, I0, tI, out, H->b0, W.bx, W.by, W.bz, lambda, sigma, s);  // x0 = I0 and b
  Fine f;
  f.x = out;
  f.mode = RHS_B;
  f.tI = 1;
  f.R = RhsK{H->b0, nullptr, nullptr, 0.f, 0};
  const int st = solve(C, *H, f, o, false, report, s);
  if (st != GDP_OK && st != GDP_ENOCONV) return st;
  CK(cudaEventRecord(C.ev1, s));
  if (report) {
    fill_time(ctx, report, s);
    report->kernel_launches = g_launches.load() - before;
    report->hbm_bytes_est = hbm_model(*H, 4.0, 0.0, report->vcycles);
  }
  if (st == GDP_ENOCONV) set_err(GDP_ENOCONV, "npr_filter: not converged");
  return st;
}

int gdp_destripe(gdp_ctx* ctx, const void* I0, gdp_dtype dtype, float* I1, float* I2,
                 gdp_dims local, int64_t z0_global, int64_t nz_global, gdp_weights W,
                 float alpha, const gdp_opts* opts, gdp_report* rep1, gdp_report* rep2,
                 void* stream) {
  if (!ctx) return set_err(GDP_EINVAL, "null ctx");
  float* I1p = I1;
  if (!I1p) {
    RET(check_common(ctx, local, z0_global, nz_global));
    RET(ctx->impl.ensure_scratch(sizeof(float) * (size_t)(local.nx * local.ny * local.nz)));
    I1p = (float*)ctx->impl.scratch;
  }
  // single rank: phase 1's mean pin is applied in phase 2's init pass (one pass over I1 less)
  const bool defer = ctx->impl.world == 1 && ctx->impl.loop == 1;
  float shift = 0.f;
  int st1 = diffuse_z_impl(ctx, I0, dtype, I1p, local, z0_global, nz_global, W, 0.f, opts, rep1, stream,
                           defer ? &shift : nullptr);
  if (st1 != GDP_OK && st1 != GDP_ENOCONV) return st1;
  int st2 = slices_impl(ctx, I0, dtype, I1p, I2, local, alpha, opts, rep2, stream, defer ? &shift : nullptr);
  if (st2 != GDP_OK) return st2;
  return st1;
}

int gdp_vcycle(gdp_ctx* ctx, float* x, const float* b, gdp_dims local, int64_t z0_global,
               int64_t nz_global, gdp_weights W, float alpha, const gdp_opts* opts,
               double* rel_res_after, void* stream) {
  RET(check_common(ctx, local, z0_global, nz_global));
  RET(check_params(W, alpha));
  if (!x || !b) return set_err(GDP_EINVAL, "null x/b");
  const gdp_opts o = resolve_opts(opts);
  cudaStream_t s = (cudaStream_t)stream;
  Ctx& C = ctx->impl;
  if (o.scheme != GDP_SCHEME_CONSTANT) {  // NEXT-3: Hybrid / Linear (gdp_scheme.cu)
    RET(check_scheme(C, o));
    return scheme_vcycle(C, x, b, local.nx, local.ny, local.nz, W.bx, W.by, W.bz, alpha, o, rel_res_after, s);
  }
  if (C.world > 1 || C.loop > 1)  // z-slab partition: halos per half-sweep, gathered coarse levels
    return dist_vcycle(C, x, b, local.nx, local.ny, local.nz, z0_global, nz_global, W.bx, W.by, W.bz, alpha, o,
                       rel_res_after, s);
  Hier* H;
  RET(C.get_hier(make_key(local, z0_global, nz_global, W, alpha, o), &H));
  Fine f;
  f.x = x;
  f.mode = RHS_B;
  f.tI = 1;
  f.R = RhsK{b, nullptr, nullptr, 0.f, 0};
  RET(run_vcycle(C, *H, f, o, s));
  if (rel_res_after) {
    RET(finest_norms(C, *H, f, nullptr, s));
    double rr = 0.0, bb = 0.0;
    for (int z = 0; z < H->lv[0].nzl; ++z) { rr += H->h_plane[z].x; bb += H->h_plane[z].y; }
    *rel_res_after = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
  }
  return GDP_OK;
}

int gdp_residual(gdp_ctx* ctx, const float* x, const float* b, float* r, gdp_dims local,
                 int64_t z0_global, int64_t nz_global, gdp_weights W, float alpha,
                 double* norm2_r, double* norm2_b, void* stream) {
  RET(check_common(ctx, local, z0_global, nz_global));
  RET(check_params(W, alpha));
  if (!x || !b) return set_err(GDP_EINVAL, "null x/b");
  gdp_opts o;
  gdp_opts_default(&o);
  cudaStream_t s = (cudaStream_t)stream;
  Ctx& C = ctx->impl;
  if (C.world > 1 || C.loop > 1)  // ghost planes from the neighbouring slabs, norms over all slabs
    return dist_residual(C, x, b, r, local.nx, local.ny, local.nz, z0_global, nz_global, W.bx, W.by, W.bz, alpha, o,
                         norm2_r, norm2_b, s);
  Hier* H;
  RET(C.get_hier(make_key(local, z0_global, nz_global, W, alpha, o), &H));
  Fine f;
  f.x = const_cast<float*>(x);
  f.mode = RHS_B;
  f.tI = 1;
  f.R = RhsK{b, nullptr, nullptr, 0.f, 0};
  RET(finest_norms(C, *H, f, r, s));
  double rr = 0.0, bb = 0.0;
  for (int z = 0; z < H->lv[0].nzl; ++z) { rr += H->h_plane[z].x; bb += H->h_plane[z].y; }
  if (norm2_r) *norm2_r = rr;
  if (norm2_b) *norm2_b = bb;
  return GDP_OK;
}

int gdp_scheme_levels(gdp_ctx* ctx, int scheme, gdp_dims dims, gdp_weights W, float alpha, int per_slice,
                      const gdp_opts* opts, int* nlev, gdp_dims* level_dims, int* coarsened, int max_levels) {
  RET(check_common(ctx, dims, 0, dims.nz));
  RET(check_params(W, alpha));
  if (!nlev) return set_err(GDP_EINVAL, "null nlev");
  gdp_opts o = resolve_opts(opts);
  o.scheme = scheme;
  RET(check_scheme(ctx->impl, o));
  return scheme_levels(ctx->impl, scheme, dims.nx, dims.ny, dims.nz, W.bx, W.by, W.bz, alpha, per_slice ? 1 : 0, o,
                       nlev, level_dims, coarsened, max_levels);
}

int gdp_scheme_apply(gdp_ctx* ctx, int scheme, int level, const float* x, float* y, gdp_dims dims, gdp_weights W,
                     float alpha, int per_slice, const gdp_opts* opts, void* stream) {
  RET(check_common(ctx, dims, 0, dims.nz));
  RET(check_params(W, alpha));
  if (!x || !y || (const float*)y == x) return set_err(GDP_EINVAL, "null or aliased x / y");
  gdp_opts o = resolve_opts(opts);
  o.scheme = scheme;
  RET(check_scheme(ctx->impl, o));
  return scheme_apply(ctx->impl, scheme, level, x, y, dims.nx, dims.ny, dims.nz, W.bx, W.by, W.bz, alpha,
                      per_slice ? 1 : 0, o, (cudaStream_t)stream);
}

int gdp_scheme_residual(gdp_ctx* ctx, int scheme, const float* x, const float* b, float* r, gdp_dims dims,
                        gdp_weights W, float alpha, int per_slice, double* norm2_r, double* norm2_b, void* stream) {
  RET(check_common(ctx, dims, 0, dims.nz));
  RET(check_params(W, alpha));
  if (!x || !b) return set_err(GDP_EINVAL, "null x / b");
  gdp_opts o = resolve_opts(nullptr);
  o.scheme = scheme;
  RET(check_scheme(ctx->impl, o));
  return scheme_residual(ctx->impl, scheme, x, b, r, dims.nx, dims.ny, dims.nz, W.bx, W.by, W.bz, alpha,
                         per_slice ? 1 : 0, o, norm2_r, norm2_b, (cudaStream_t)stream);
}

int gdp_profile_begin(void) {
  for (auto& r : g_prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  g_prof.clear();
  g_prof_open.clear();
  g_prof_on = true;
  return GDP_OK;
}

int gdp_profile_end(gdp_kernel_stat* out, int max, int* n_out) {
  g_prof_on = false;
  double ms[3 * KC_COUNT] = {0}, by[3 * KC_COUNT] = {0}, b8[3 * KC_COUNT] = {0};
  long long n[3 * KC_COUNT] = {0};
  for (auto& r : g_prof) {
    float t = 0.f;
    CK(cudaEventSynchronize(r.b));
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.cls] += t;
    by[r.cls] += r.bytes;
    b8[r.cls] += r.bytes8d;
    n[r.cls] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  int k = 0;
  for (int c = 0; c < 3 * KC_COUNT; ++c) {
    if (!n[c]) continue;
    if (out && k < max) {
      static const char* band[3] = {"", "@L0", "@L1"};
      std::snprintf(out[k].name, sizeof out[k].name, "%s%s", kclass_name[c % KC_COUNT], band[c / KC_COUNT]);
      out[k].launches = n[c];
      out[k].ms = ms[c];
      out[k].alg_bytes = by[c];
      out[k].alg_bytes_8d = b8[c];
    }
    ++k;
  }
  if (n_out) *n_out = std::min(k, max);
  return GDP_OK;
}

const char* gdp_last_error(void) { return t_err.c_str(); }

const char* gdp_version(void) { return "gdp-b200 0.1 (sm_100a)"; }

int64_t gdp_kernel_launch_count(void) { return g_launches.load(); }

}  // extern "C"
