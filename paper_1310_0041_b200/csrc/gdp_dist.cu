// gdp_dist.cu — phase 1 (Eq. 1) on a z-slab partition.
//
// Every rank (NCCL) or every loopback slab owns planes [z0, z0 + nzl) of the stack.  The
// level chain is the single-rank one (level_chain): the first levels stay split across the
// slabs, from level `ff` on every level is full and replicated (the "tail", gathered once per
// V-cycle from the restricted residual).  Split levels run the reference schedule with one
// ghost plane per slab face, refreshed before every half-sweep, residual and prolongation.
// Because colours, coefficients and transfers use global z and every kernel evaluates the
// same per-cell arithmetic, the iterates are bit-identical to the single-rank solve for any
// partition (tests/test_gpu_parity.py::test_loopback_partition_bit_identical).
#include <cmath>
#include <cstring>
#include <vector>

#include "gdp_internal.h"

namespace gdp {

DistPlan::~DistPlan() {
  if (h_planes) cudaFreeHost(h_planes);
  for (auto* p : b0) if (p) cudaFree(p);
  for (auto* p : w0) if (p) cudaFree(p);
  for (auto* p : w1) if (p) cudaFree(p);
  for (auto* p : bw) if (p) cudaFree(p);
  for (auto* p : cw) if (p) cudaFree(p);
  if (fpart) cudaFree(fpart);
  if (ev_bnd) cudaEventDestroy(ev_bnd);
  if (ev_comm) cudaEventDestroy(ev_comm);
  if (cs) cudaStreamDestroy(cs);
}

#define CKD(call)                                                                         \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(e_ == cudaErrorMemoryAllocation ? GDP_ENOMEM : GDP_ECUDA, "%s: %s", #call, \
                     cudaGetErrorString(e_));                                             \
  } while (0)
#define RETD(call)                 \
  do {                             \
    int r_ = (call);               \
    if (r_ != GDP_OK) return r_;   \
  } while (0)

// Build the plan for slabs (z0s[i], nzls[i]) of which `local` are processed here.
static int build_plan(const HierKey& gkey, const std::vector<long long>& z0s, const std::vector<int>& nzls,
                      const std::vector<int>& local, std::unique_ptr<DistPlan>& out) {
  auto D = std::make_unique<DistPlan>();
  D->nzg = (int)gkey.nzg;
  // level chains of every slab; the first full level is the earliest any slab needs
  std::vector<std::vector<Level>> chains(z0s.size());
  int ff = 1 << 30;
  for (size_t i = 0; i < z0s.size(); ++i) {
    HierKey k = gkey;
    k.z0 = z0s[i];
    k.nzl = nzls[i];
    int f;
    RETD(level_chain(k, chains[i], f));
    ff = std::min(ff, f);
  }
  if (ff < 1) return set_err(GDP_EINVAL, "distributed stack too small: level 0 must already be gathered");
  D->ff = ff;
  // the restriction into the gathered level maps local planes to coarse planes z0/2 + k: a
  // z-coarsened step needs every slab aligned at that level (no coarse plane straddles two slabs)
  for (size_t i = 0; i < z0s.size(); ++i) {
    const Level& L = chains[i][ff - 1];
    const Level& Cg = chains[i][ff];
    const long long lz0 = ff - 1 == 0 ? z0s[i] : L.z0, lnz = ff - 1 == 0 ? nzls[i] : L.nzl;
    if (Cg.tz.coarsened && (lz0 % 2 != 0 || lnz % 2 != 0))
      return set_err(GDP_EINVAL, "z-slab partition: level %d coarsens z but slab %zu (planes [%lld, %lld)) is not "
                     "aligned to even planes; use an even split or weights with bz < max(bx, by) / 2",
                     ff - 1, i, lz0, lz0 + lnz);
  }
  // the gathered level: the element range each slab restricts into (all-gather-v, gdp_comm.cu)
  {
    const Level& Cg = chains[0][ff];
    const size_t tpl = (size_t)Cg.nx * Cg.ny;
    for (size_t i = 0; i < z0s.size(); ++i) {
      const Level& L = chains[i][ff - 1];
      const bool cz = Cg.tz.coarsened != 0;
      D->goff.push_back((size_t)(cz ? L.z0 / 2 : L.z0) * tpl);
      D->gcnt.push_back((size_t)(cz ? L.nzl / 2 : L.nzl) * tpl);
    }
  }
  // the fused finest level needs every slab (all ranks, not just the local ones: the halo
  // schedule must match) to hold >= G planes on level 0 and on a split level 1
  D->slabs_fusable = true;
  for (size_t i = 0; i < z0s.size(); ++i) {
    if (nzls[i] < DistPlan::G) D->slabs_fusable = false;
    if (ff > 1 && chains[i][1].nzl < DistPlan::G) D->slabs_fusable = false;
  }
  for (int i : local) {
    HierKey k = gkey;
    k.z0 = z0s[i];
    k.nzl = nzls[i];
    std::unique_ptr<Hier> P;
    RETD(build_hier_levels(k, chains[i], 0, ff, false, false, P));
    D->parts.push_back(std::move(P));
    D->z0.push_back(z0s[i]);
    D->nzl.push_back(nzls[i]);
    D->b0.push_back(nullptr);
  }
  // the tail: levels ff.. of the chain, full in z
  std::vector<Level> tail = chains[0];
  for (size_t l = ff; l < tail.size(); ++l) { tail[l].z0 = 0; tail[l].nzl = tail[l].gz.n; }
  HierKey tk = gkey;
  tk.nx = tail[ff].nx; tk.ny = tail[ff].ny; tk.nzl = tail[ff].nzl; tk.nzg = tail[ff].gz.n; tk.z0 = 0;
  RETD(build_hier_levels(tk, tail, ff, (int)tail.size(), true, true, D->tail));
  CKD(cudaMallocHost(&D->h_planes, sizeof(double2) * (size_t)D->nzg));
  out = std::move(D);
  return GDP_OK;
}

// all ranks' slab extents (NCCL) or the loopback split of the whole stack
static int slab_layout(Ctx& c, long long z0, int nzl, long long nzg, std::vector<long long>& z0s,
                       std::vector<int>& nzls, std::vector<int>& local) {
  z0s.clear(); nzls.clear(); local.clear();
  if (c.world > 1) {
    // every rank learns every slab: fp64 sums of one-hot vectors (exact)
    std::vector<double> a(2 * c.world, 0.0);
    for (int r = 0; r < c.world; ++r) {
      double z = r == c.rank ? (double)z0 : 0.0, n = r == c.rank ? (double)nzl : 0.0;
      RETD(comm_allreduce_sum2(c, &z, &n, nullptr));
      a[2 * r] = z;
      a[2 * r + 1] = n;
    }
    for (int r = 0; r < c.world; ++r) { z0s.push_back((long long)a[2 * r]); nzls.push_back((int)a[2 * r + 1]); }
    local.push_back(c.rank);
  } else {
    const int P = c.loop;
    const long long base = nzg / P, rem = nzg % P;
    long long z = 0;
    for (int i = 0; i < P; ++i) {
      const int n = (int)(base + (i < rem ? 1 : 0));
      z0s.push_back(z);
      nzls.push_back(n);
      local.push_back(i);
      z += n;
    }
  }
  long long z = 0;
  for (size_t i = 0; i < z0s.size(); ++i) {
    if (z0s[i] != z || nzls[i] < 1) return set_err(GDP_EINVAL, "slabs must tile [0, nz_global) in rank order");
    z += nzls[i];
  }
  if (z != nzg) return set_err(GDP_EINVAL, "slabs do not cover nz_global");
  return GDP_OK;
}

// ---------------------------------------------------------------------------------
// V-cycle on the partition (reference schedule on split levels)
// ---------------------------------------------------------------------------------
static int team_smooth(Ctx& c, DistPlan& D, int l, float* const* xs, const float* const* bs, int nu, cudaStream_t s) {
  const int np = (int)D.parts.size();
  for (int k = 0; k < nu; ++k)
    for (int color = 0; color < 2; ++color) {
      RETD(comm_halo_parts(c, D, l, xs, s));
      for (int i = 0; i < np; ++i) {
        const Level& L = D.parts[i]->lv[l];
        launch_rbgs(L.K, xs[i], L.xlo, L.xhi, RhsK{bs[i], nullptr, nullptr, 0.f, 0}, RHS_B, 1, color, s);
      }
    }
  return GDP_OK;
}

// the level below level 0 of part i, with its arrays offset so that they are indexed by global
// plane (the split level 1 of the part, or the gathered tail's first level)
static Level coarse_of(DistPlan& D, int i) {
  Level C = D.ff > 1 ? D.parts[i]->lv[1] : D.tail->lv[0];
  if (D.ff > 1) {
    const size_t cpl = (size_t)C.nx * C.ny;
    C.b -= (long long)C.z0 * cpl;
    C.x -= (long long)C.z0 * cpl;
  }
  return C;
}

// nu fused sweeps of the finest level on every local slab (k_march3d over the slab's global
// planes, G ghost planes exchanged before each sweep).  *cur: which window holds x; tail 1 =
// restrict the last sweep, 2 = norms of the last sweep (partials per item, all slabs, summed
// into *rr / *bb over slabs and ranks), prolong = add the coarse correction in the first sweep.
static int team_fused_sweeps(Ctx& c, DistPlan& D, int* cur, int nu, bool prolong, int tail, double* rr,
                             double* bb, cudaStream_t s) {
  const int np = (int)D.parts.size();
  const size_t pl = (size_t)D.parts[0]->lv[0].nx * D.parts[0]->lv[0].ny;
  const int G = DistPlan::G;
  long long items = 0;
  if (prolong && D.ff > 1) {
    // the first sweep also corrects the G ghost planes of the window, whose coarse planes
    // belong to the neighbouring slabs: level 1's x with G ghost planes per face
    for (int i = 0; i < np; ++i) {
      const Level& C = D.parts[i]->lv[1];
      const size_t cpl = (size_t)C.nx * C.ny;
      CKD(cudaMemcpyAsync(D.cw[i] + (size_t)G * cpl, C.x, sizeof(float) * cpl * C.nzl, cudaMemcpyDeviceToDevice, s));
    }
    RETD(comm_ghosts(c, D, D.cw.data(), s, 1));
  }
  // Boundary first (H7): a sweep followed by another one in this pass computes its G bottom and G top
  // planes first, hands their ghost exchange to the communication stream and computes its interior
  // meanwhile; the next sweep waits for the exchange.  Sub-range z-marches are bit-identical to the
  // whole-slab one (the out-of-core streamer relies on the same property); tail sweeps (restriction,
  // norms) and z-coarsened level-1 restrictions stay whole.  The exchange issues the same NCCL calls
  // in the same order on every rank, only on another stream.
  bool ovl = !coarse_of(D, 0).tz.coarsened;
  for (int i = 0; i < np; ++i) ovl = ovl && D.nzl[i] >= 2 * G + 1;
  if (ovl && !D.cs) {
    CKD(cudaStreamCreateWithFlags(&D.cs, cudaStreamNonBlocking));
    CKD(cudaEventCreateWithFlags(&D.ev_bnd, cudaEventDisableTiming));
    CKD(cudaEventCreateWithFlags(&D.ev_comm, cudaEventDisableTiming));
  }
  bool exchanged = false;  // the ghosts of the current source were exchanged on D.cs
  for (int k = 0; k < nu; ++k) {
    std::vector<float*>& src = *cur ? D.w1 : D.w0;
    std::vector<float*>& dst = *cur ? D.w0 : D.w1;
    if (exchanged) CKD(cudaStreamWaitEvent(s, D.ev_comm, 0));
    else RETD(comm_ghosts(c, D, src.data(), s));
    exchanged = false;
    const bool last = k == nu - 1;
    const int t = last ? tail : 0;
    const bool split = ovl && !last;
    auto sweep = [&](int i, int zlo, int zhi) {
      const Level& L = D.parts[i]->lv[0];
      Level C = coarse_of(D, i);
      if (prolong && D.ff > 1)
        C.x = D.cw[i] + ((long long)G - D.parts[i]->lv[1].z0) * (long long)C.nx * C.ny;
      const long long off = (long long)G - D.z0[i];  // window offset of global plane 0 (planes)
      const int n = fused_sweep3d(L, C, src[i] + off * (long long)pl, dst[i] + off * (long long)pl,
                                  D.bw[i] + off * (long long)pl, false, prolong && k == 0, t,
                                  t == 2 ? D.fpart + items : nullptr, s, zlo, zhi);
      if (t == 2) items += n;  // partials of the norms sweep only
    };
    if (!split) {
      for (int i = 0; i < np; ++i) sweep(i, (int)D.z0[i], (int)(D.z0[i] + D.nzl[i]));
    } else {
      for (int i = 0; i < np; ++i) {
        const int z0 = (int)D.z0[i], z1 = (int)(D.z0[i] + D.nzl[i]);
        sweep(i, z0, z0 + G);
        sweep(i, z1 - G, z1);
      }
      CKD(cudaEventRecord(D.ev_bnd, s));
      CKD(cudaStreamWaitEvent(D.cs, D.ev_bnd, 0));
      RETD(comm_ghosts(c, D, dst.data(), D.cs));
      CKD(cudaEventRecord(D.ev_comm, D.cs));
      for (int i = 0; i < np; ++i) sweep(i, (int)D.z0[i] + G, (int)(D.z0[i] + D.nzl[i]) - G);
      exchanged = true;
    }
    *cur ^= 1;
  }
  CKD(cudaGetLastError());
  if (tail == 2) {
    Hier& H = *D.parts[0];
    launch_finalize(D.fpart, (int)items, 1, H.plane_sums, s);
    CKD(cudaMemcpyAsync(H.h_plane, H.plane_sums, sizeof(double2), cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    *rr = H.h_plane[0].x;
    *bb = H.h_plane[0].y;
    RETD(comm_allreduce_sum2(c, rr, bb, s));
  }
  return GDP_OK;
}

// prolongation of level l+1 into level l of every local part (x_l += P x_{l+1}); the coarse level
// is split (ghost planes refreshed first) or the gathered tail's first level
static int team_prolong(Ctx& c, DistPlan& D, int l, float* const* xs, cudaStream_t s) {
  const int np = (int)D.parts.size();
  Level& TF = D.tail->lv[0];
  if (l + 1 < D.ff) {
    std::vector<float*> xc(np);
    for (int i = 0; i < np; ++i) xc[i] = D.parts[i]->lv[l + 1].x;
    RETD(comm_halo_parts(c, D, l + 1, xc.data(), s));
  }
  for (int i = 0; i < np; ++i) {
    Level& L = D.parts[i]->lv[l];
    if (l + 1 < D.ff) {
      Level& C = D.parts[i]->lv[l + 1];
      launch_prolong(L.K, xs[i], C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
    } else {
      launch_prolong(L.K, xs[i], TF.tx, TF.ty, TF.tz, TF.nx, TF.ny, TF.nzl, 0, TF.x, nullptr, nullptr, s);
    }
  }
  return GDP_OK;
}

// One V-cycle of the partition over global levels l0.. (l0 > 0: a nested FMG cycle); flags
// RV_PROLONG: level l0 starts from the prolongation of level l0 + 1 (added to x at level 0, to zero
// above), the single-rank run_vcycle's convention.  *rel: the norms of the fused finest level.
static int team_vcycle(Ctx& c, DistPlan& D, float* const* x0, const gdp_opts& o, cudaStream_t s, int* cur,
                       double* rel, int l0 = 0, unsigned flags = 0) {
  const int np = (int)D.parts.size();
  const int ff = D.ff;
  std::vector<float*> xs(np);
  std::vector<const float*> bs(np);
  Hier& T = *D.tail;
  Level& TF = T.lv[0];
  const size_t tplane = (size_t)TF.nx * TF.ny;
  Fine ft;
  ft.x = TF.x;
  ft.mode = RHS_B;
  ft.tI = 1;
  ft.R = RhsK{TF.b, nullptr, nullptr, 0.f, 0};
  const bool pro = (flags & RV_PROLONG) != 0;
  if (l0 >= ff) {  // the whole cycle lives in the gathered levels (replicated on every rank)
    if (l0 == ff && pro) CKD(cudaMemsetAsync(TF.x, 0, sizeof(float) * tplane * TF.nzl, s));  // run_vcycle adds P e at its level 0
    return run_vcycle(c, T, ft, o, s, l0 - ff, flags);
  }
  const bool fused0 = D.active && l0 == 0;
  if (fused0) RETD(team_fused_sweeps(c, D, cur, o.nu_pre, pro, 1, nullptr, nullptr, s));
  for (int l = fused0 ? 1 : l0; l < ff; ++l) {
    for (int i = 0; i < np; ++i) {
      Level& L = D.parts[i]->lv[l];
      xs[i] = l == 0 ? x0[i] : L.x;
      bs[i] = l == 0 ? D.b0[i] : L.b;
      if (l > 0) CKD(cudaMemsetAsync(xs[i], 0, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, s));
    }
    if (l == l0 && pro) RETD(team_prolong(c, D, l, xs.data(), s));  // FMG start at l0
    RETD(team_smooth(c, D, l, xs.data(), bs.data(), o.nu_pre, s));
    RETD(comm_halo_parts(c, D, l, xs.data(), s));
    for (int i = 0; i < np; ++i) {
      Level& L = D.parts[i]->lv[l];
      RhsK R{bs[i], nullptr, nullptr, 0.f, 0};
      if (l + 1 < ff) {
        Level& C = D.parts[i]->lv[l + 1];
        launch_restrict(L.K, xs[i], L.xlo, L.xhi, R, RHS_B, 1, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.b, s);
      } else {  // into this slab's planes of the gathered level
        const bool cz = TF.tz.coarsened;
        const long long off = cz ? L.z0 / 2 : L.z0;
        const int nczl = cz ? L.nzl / 2 : L.nzl;
        launch_restrict(L.K, xs[i], L.xlo, L.xhi, R, RHS_B, 1, TF.tx, TF.ty, TF.tz, TF.nx, TF.ny, nczl,
                        TF.b + off * tplane, s);
      }
    }
  }
  // gathered levels: one V-cycle of the tail from a zero start (replicated on every rank)
  RETD(comm_gather_full(c, D, TF.b, s));
  CKD(cudaMemsetAsync(TF.x, 0, sizeof(float) * tplane * TF.nzl, s));
  RETD(run_vcycle(c, T, ft, o, s));
  for (int l = ff - 1; l >= (fused0 ? 1 : l0); --l) {
    for (int i = 0; i < np; ++i) {
      Level& L = D.parts[i]->lv[l];
      xs[i] = l == 0 ? x0[i] : L.x;
      bs[i] = l == 0 ? D.b0[i] : L.b;
    }
    RETD(team_prolong(c, D, l, xs.data(), s));
    RETD(team_smooth(c, D, l, xs.data(), bs.data(), o.nu_post, s));
  }
  if (fused0) {
    if (ff > 1) {  // the split level 1 feeds the prolongation: refresh its ghost planes
      std::vector<float*> xc(np);
      for (int i = 0; i < np; ++i) xc[i] = D.parts[i]->lv[1].x;
      RETD(comm_halo_parts(c, D, 1, xc.data(), s));
    }
    double rr = 0.0, bb = 0.0;
    RETD(team_fused_sweeps(c, D, cur, o.nu_post, true, 2, &rr, &bb, s));
    if (rel) *rel = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
  }
  CKD(cudaGetLastError());
  return GDP_OK;
}

// FMG start of the partition (the single-rank fmg_start, level by level): r0 = b - A x0 restricted
// to level 1, the right-hand side restricted on down (split levels per slab, gathered once), the
// coarsest solve, then per level a nested V-cycle started from the prolongation of the level below
// (V(nu_pre, nu_post - 1)); the caller's first fine cycle prolongates e_1 into x (RV_PROLONG).
static int team_fmg_start(Ctx& c, DistPlan& D, float* const* x0, const gdp_opts& o, cudaStream_t s, int* cur) {
  const int np = (int)D.parts.size();
  const int ff = D.ff;
  Hier& T = *D.tail;
  Level& TF = T.lv[0];
  const size_t tplane = (size_t)TF.nx * TF.ny;
  const size_t pl = (size_t)D.parts[0]->lv[0].nx * D.parts[0]->lv[0].ny;
  std::vector<float*> xw(np);  // level-0 x of every part (the fused windows' interior when active)
  for (int i = 0; i < np; ++i) xw[i] = D.active ? (*cur ? D.w1[i] : D.w0[i]) + pl * DistPlan::G : x0[i];
  RETD(comm_halo_parts(c, D, 0, xw.data(), s));
  auto into_gathered = [&](const Level& L, bool b_only, const float* src, const float* b) {
    const bool cz = TF.tz.coarsened;
    const long long off = cz ? L.z0 / 2 : L.z0;
    const int nczl = cz ? L.nzl / 2 : L.nzl;
    if (b_only) launch_restrict_b(L.K, b, TF.tx, TF.ty, TF.tz, TF.nx, TF.ny, nczl, TF.b + off * tplane, s);
    else launch_restrict(L.K, src, L.xlo, L.xhi, RhsK{b, nullptr, nullptr, 0.f, 0}, RHS_B, 1, TF.tx, TF.ty, TF.tz,
                         TF.nx, TF.ny, nczl, TF.b + off * tplane, s);
  };
  for (int i = 0; i < np; ++i) {  // r0 restricted to level 1
    const Level& L = D.parts[i]->lv[0];
    if (ff > 1) {
      const Level& C = D.parts[i]->lv[1];
      launch_restrict(L.K, xw[i], L.xlo, L.xhi, RhsK{D.b0[i], nullptr, nullptr, 0.f, 0}, RHS_B, 1, C.tx, C.ty, C.tz,
                      C.nx, C.ny, C.nzl, C.b, s);
    } else {
      into_gathered(L, false, xw[i], D.b0[i]);
    }
  }
  for (int l = 1; l < ff; ++l)  // the rhs restricted on down the split levels
    for (int i = 0; i < np; ++i) {
      const Level& L = D.parts[i]->lv[l];
      if (l + 1 < ff) {
        const Level& C = D.parts[i]->lv[l + 1];
        launch_restrict_b(L.K, L.b, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.b, s);
      } else {
        into_gathered(L, true, nullptr, L.b);
      }
    }
  RETD(comm_gather_full(c, D, TF.b, s));
  for (size_t j = 0; j + 1 < T.lv.size(); ++j) {  // and through the gathered levels
    const Level& L = T.lv[j];
    const Level& C = T.lv[j + 1];
    launch_restrict_b(L.K, L.b, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.b, s);
  }
  Level& Lc = T.lv.back();
  CKD(launch_coarse(T.coarse, Lc.b, Lc.x, s));
  gdp_opts on = o;
  on.nu_post = std::max(1, o.nu_post - 1);
  const int mode = o.fmg & 3;
  const int lmin = mode == 1 ? 1 : 2;
  const int ntot = ff + (int)T.lv.size();
  for (int l = ntot - 2; l >= lmin; --l) RETD(team_vcycle(c, D, x0, on, s, cur, nullptr, l, RV_PROLONG));
  for (int l = lmin - 1; l >= 1; --l) {  // levels only interpolated (3) or interpolated and smoothed (2)
    if (l >= ff) {
      Level& L = T.lv[l - ff];
      Level& C = T.lv[l - ff + 1];
      CKD(cudaMemsetAsync(L.x, 0, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, s));
      launch_prolong(L.K, L.x, C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
      if (mode == 2)
        for (int k = 0; k < o.nu_post; ++k)
          for (int color = 0; color < 2; ++color)
            launch_rbgs(L.K, L.x, L.xlo, L.xhi, RhsK{L.b, nullptr, nullptr, 0.f, 0}, RHS_B, 1, color, s);
      continue;
    }
    std::vector<float*> xs(np);
    std::vector<const float*> bs(np);
    for (int i = 0; i < np; ++i) {
      Level& L = D.parts[i]->lv[l];
      xs[i] = L.x;
      bs[i] = L.b;
      CKD(cudaMemsetAsync(L.x, 0, sizeof(float) * (size_t)L.nx * L.ny * L.nzl, s));
    }
    RETD(team_prolong(c, D, l, xs.data(), s));
    if (mode == 2) RETD(team_smooth(c, D, l, xs.data(), bs.data(), o.nu_post, s));
  }
  CKD(cudaGetLastError());
  return GDP_OK;
}

// global per-plane (r^2, b^2) of the finest level -> rel-res (one system: all planes)
static int team_norms(Ctx& c, DistPlan& D, float* const* x0, double* rel, double* nb, cudaStream_t s) {
  const int np = (int)D.parts.size();
  RETD(comm_halo_parts(c, D, 0, x0, s));
  std::vector<double2*> loc(np);
  for (int i = 0; i < np; ++i) {
    Hier& H = *D.parts[i];
    Level& L = H.lv[0];
    launch_norms(L.K, x0[i], L.xlo, L.xhi, RhsK{D.b0[i], nullptr, nullptr, 0.f, 0}, RHS_B, 1, nullptr,
                 H.partials, H.plane_sums, s);
    loc[i] = H.plane_sums;
  }
  CKD(cudaGetLastError());
  RETD(comm_plane_sums(c, D, loc.data(), D.h_planes, s));
  double rr = 0.0, bb = 0.0;
  for (int z = 0; z < D.nzg; ++z) { rr += D.h_planes[z].x; bb += D.h_planes[z].y; }
  *rel = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
  if (nb) *nb = std::sqrt(bb);
  return GDP_OK;
}

// the partition plan of this rank's slab (built once per geometry / weights / alpha / options)
static int get_plan(Ctx& c, long long nx, long long ny, long long nzl, long long z0g, long long nzg, float bx,
                    float by, float bz, float alpha, const gdp_opts& o, DistPlan** out) {
  std::vector<long long> z0s;
  std::vector<int> nzls;
  std::vector<int> local;
  RETD(slab_layout(c, z0g, (int)nzl, nzg, z0s, nzls, local));
  HierKey gk{};
  gk.nx = nx; gk.ny = ny; gk.nzl = nzg; gk.z0 = 0; gk.nzg = nzg;
  gk.bx = bx; gk.by = by; gk.bz = bz; gk.alpha = alpha; gk.coarse_max = o.coarse_max;
  gk.omega = o.omega;
  HierKey ck = gk;
  ck.z0 = z0g;  // the plan depends on this rank's slab (NCCL) or on the loopback split
  ck.nzl = nzl;
  auto it = c.dist.find(ck);
  if (it == c.dist.end()) {
    std::unique_ptr<DistPlan> P;
    RETD(build_plan(gk, z0s, nzls, local, P));
    *out = P.get();
    c.dist[ck] = std::move(P);
  } else {
    *out = it->second.get();
  }
  return GDP_OK;
}

// local slabs' pointers into the caller's arrays (loopback: the whole stack is passed)
template <typename T>
static std::vector<T*> slab_ptrs(Ctx& c, DistPlan& D, T* base, long long z0g, size_t plane) {
  const long long base_z = c.world > 1 ? z0g : 0;
  std::vector<T*> v(D.parts.size());
  for (size_t i = 0; i < D.parts.size(); ++i) v[i] = base ? base + (D.z0[i] - base_z) * (long long)plane : nullptr;
  return v;
}

int dist_residual(Ctx& c, const float* x, const float* b, float* r, long long nx, long long ny, long long nzl,
                  long long z0g, long long nzg, float bx, float by, float bz, float alpha, const gdp_opts& o,
                  double* rr, double* bb, cudaStream_t s) {
  DistPlan* D;
  RETD(get_plan(c, nx, ny, nzl, z0g, nzg, bx, by, bz, alpha, o, &D));
  const size_t plane = (size_t)nx * ny;
  auto xs = slab_ptrs(c, *D, const_cast<float*>(x), z0g, plane);
  auto bs = slab_ptrs(c, *D, b, z0g, plane);
  auto rs = slab_ptrs(c, *D, r, z0g, plane);
  RETD(comm_halo_parts(c, *D, 0, xs.data(), s));  // ghost planes of x: the neighbours' faces
  const int np = (int)D->parts.size();
  std::vector<double2*> loc(np);
  for (int i = 0; i < np; ++i) {
    Hier& H = *D->parts[i];
    Level& L = H.lv[0];
    launch_norms(L.K, xs[i], L.xlo, L.xhi, RhsK{bs[i], nullptr, nullptr, 0.f, 0}, RHS_B, 1, rs[i], H.partials,
                 H.plane_sums, s);
    loc[i] = H.plane_sums;
  }
  CKD(cudaGetLastError());
  RETD(comm_plane_sums(c, *D, loc.data(), D->h_planes, s));  // global plane order: partition-independent
  double a = 0.0, q = 0.0;
  for (int z = 0; z < D->nzg; ++z) { a += D->h_planes[z].x; q += D->h_planes[z].y; }
  if (rr) *rr = a;
  if (bb) *bb = q;
  return GDP_OK;
}

int dist_vcycle(Ctx& c, float* x, const float* b, long long nx, long long ny, long long nzl, long long z0g,
                long long nzg, float bx, float by, float bz, float alpha, const gdp_opts& o, double* rel,
                cudaStream_t s) {
  DistPlan* D;
  RETD(get_plan(c, nx, ny, nzl, z0g, nzg, bx, by, bz, alpha, o, &D));
  const size_t plane = (size_t)nx * ny;
  auto xs = slab_ptrs(c, *D, x, z0g, plane);
  auto bs = slab_ptrs(c, *D, const_cast<float*>(b), z0g, plane);
  // the split levels run the reference schedule on the caller's arrays (the fused finest level
  // needs the ghosted windows of a whole solve)
  std::vector<float*> b0own = D->b0;
  struct Restore {
    DistPlan* D;
    std::vector<float*>* own;
    bool active;
    ~Restore() { D->b0 = *own; D->active = active; }
  } restore{D, &b0own, D->active};
  for (size_t i = 0; i < bs.size(); ++i) D->b0[i] = bs[i];
  D->active = false;
  int cur = 0;
  double nrel = 0.0;
  RETD(team_vcycle(c, *D, xs.data(), o, s, &cur, &nrel));
  if (rel) RETD(team_norms(c, *D, xs.data(), rel, nullptr, s));
  CKD(cudaGetLastError());
  return GDP_OK;
}

int dist_diffuse_z(Ctx& c, const void* I0, int tI, float* I1, long long nx, long long ny, long long nzl,
                   long long z0g, long long nzg, float bx, float by, float bz, float alpha, const gdp_opts& o,
                   gdp_report* rep, cudaStream_t s) {
  if (alpha != 0.f) return set_err(GDP_EINVAL, "the z-slab partition implements Eq. (1) (alpha = 0)");
  DistPlan* D;
  RETD(get_plan(c, nx, ny, nzl, z0g, nzg, bx, by, bz, alpha, o, &D));
  const int np = (int)D->parts.size();
  const size_t plane = (size_t)nx * ny;
  const size_t sI = tI == 0 ? 1 : 4;
  // local slabs: pointers into the caller's arrays (loopback: the whole stack here)
  const long long base_z = c.world > 1 ? z0g : 0;
  std::vector<float*> x0(np);
  std::vector<const void*> i0(np);
  const long long before = g_launches.load();
  // fused finest level: every slab holds >= G planes, the next level is x/y-coarsened only
  if (D->w0.empty()) {
    bool ok = (o.fused & 2) != 0 && (long long)nx * ny < (1LL << 31);
    for (int i = 0; i < np && ok; ++i) {
      const Level& L = D->parts[i]->lv[0];
      const Level C = coarse_of(*D, i);
      ok = L.K.az.k != 0.f && C.tx.coarsened && C.ty.coarsened && !C.tz.coarsened;
    }
    ok = ok && D->slabs_fusable;
    if (ok) {
      D->fused = true;
      long long items = 0;
      for (int i = 0; i < np; ++i) {
        float *a = nullptr, *b = nullptr, *w = nullptr;
        const size_t n = plane * (size_t)(D->nzl[i] + 2 * DistPlan::G);
        CKD(cudaMalloc(&a, n * sizeof(float)));
        CKD(cudaMalloc(&b, n * sizeof(float)));
        CKD(cudaMalloc(&w, n * sizeof(float)));
        CKD(cudaMemset(a, 0, n * sizeof(float)));
        CKD(cudaMemset(b, 0, n * sizeof(float)));
        CKD(cudaMemset(w, 0, n * sizeof(float)));
        D->w0.push_back(a);
        D->w1.push_back(b);
        D->bw.push_back(w);
        if (D->ff > 1) {
          const Level& C = D->parts[i]->lv[1];
          float* q = nullptr;
          const size_t cn = (size_t)C.nx * C.ny * (C.nzl + 2 * DistPlan::G);
          CKD(cudaMalloc(&q, cn * sizeof(float)));
          CKD(cudaMemset(q, 0, cn * sizeof(float)));
          D->cw.push_back(q);
        }
        items += fused3d_items(D->parts[i]->lv[0], coarse_of(*D, i), (int)D->z0[i], (int)(D->z0[i] + D->nzl[i]));
      }
      D->fpart_cap = (size_t)items;
      CKD(cudaMalloc(&D->fpart, sizeof(double2) * D->fpart_cap));
    }
  }
  D->active = D->fused && (o.fused & 2) && o.nu_pre >= 1 && o.nu_post >= 1;
  std::vector<float*> b0own = D->b0;  // active: the rhs lives in the ghosted windows for this call
  struct Restore {
    DistPlan* D;
    std::vector<float*>* own;
    ~Restore() { D->b0 = *own; }
  } restore{D, &b0own};
  if (D->active)
    for (int i = 0; i < np; ++i) D->b0[i] = D->bw[i] + plane * DistPlan::G;
  CKD(cudaEventRecord(c.ev0, s));
  for (int i = 0; i < np; ++i) {
    const long long off = D->z0[i] - base_z;
    x0[i] = I1 + off * plane;
    i0[i] = static_cast<const char*>(I0) + off * plane * sI;
    Level& L = D->parts[i]->lv[0];
    if (!D->b0[i]) {
      CKD(cudaMalloc(&D->b0[i], sizeof(float) * plane * D->nzl[i]));
      b0own[i] = D->b0[i];
    }
    float* xi = D->active ? D->w0[i] + plane * DistPlan::G : x0[i];
    launch_decode_copy(i0[i], tI, xi, (long long)plane * D->nzl[i], s);  // x0 = I0
    launch_rhs(L.K, RhsK{nullptr, i0[i], nullptr, 0.f, 0}, tI, D->b0[i], s);
  }
  int cur = 0;  // fused: the window holding x
  std::vector<float*> xw(np);
  for (int i = 0; i < np; ++i) xw[i] = D->active ? D->w0[i] + plane * DistPlan::G : x0[i];
  if (D->active) RETD(comm_ghosts(c, *D, D->bw.data(), s));  // the rhs ghosts, once per solve
  gdp_report r{};
  r.dx_inf = -1.0;  // the a9 correction norm is measured by the single-rank in-core solve only
  r.levels = D->ff + (int)D->tail->lv.size();
  double rel, nb;
  RETD(team_norms(c, *D, xw.data(), &rel, &nb, s));
  r.rel_res[0] = rel;
  r.norm_b = nb;
  if (!std::isfinite(rel)) return set_err(GDP_EINVAL, "non-finite initial residual (non-finite input?)");
  int status = GDP_OK, stall = 0, k = 0;
  const int cap = std::min(o.max_vcycles, GDP_MAX_CYCLES);
  while (rel > o.rel_tol) {
    if (k >= cap) { status = GDP_ENOCONV; break; }
    double nrel = 0.0;
    const bool fmg = k == 0 && (o.fmg & 3) != 0 && D->ff + (int)D->tail->lv.size() >= 3;
    if (fmg) RETD(team_fmg_start(c, *D, x0.data(), o, s, &cur));
    RETD(team_vcycle(c, *D, x0.data(), o, s, &cur, &nrel, 0, fmg ? RV_PROLONG : 0u));
    if (!D->active) RETD(team_norms(c, *D, x0.data(), &nrel, nullptr, s));
    r.rel_res[++k] = nrel;
    if (!std::isfinite(nrel)) return set_err(GDP_EINVAL, "non-finite residual after V-cycle %d", k);
    if (o.stagnation > 0 && nrel > 0.9 * rel) {
      if (++stall >= o.stagnation) { rel = nrel; status = nrel <= o.rel_tol ? GDP_OK : GDP_ENOCONV; break; }
    } else {
      stall = 0;
    }
    rel = nrel;
  }
  if (D->active)  // the iterate back into the caller's slabs
    for (int i = 0; i < np; ++i)
      CKD(cudaMemcpyAsync(x0[i], (cur ? D->w1[i] : D->w0[i]) + plane * DistPlan::G,
                          sizeof(float) * plane * D->nzl[i], cudaMemcpyDeviceToDevice, s));
  // a10: mean(I1) = mean(I0), fp64 sums in global plane order
  std::vector<double2*> loc(np);
  for (int i = 0; i < np; ++i) {
    Hier& H = *D->parts[i];
    launch_plane_sums(x0[i], 1, i0[i], tI, (int)nx, (int)ny, D->nzl[i], H.partials, H.plane_sums, s);
    loc[i] = H.plane_sums;
  }
  RETD(comm_plane_sums(c, *D, loc.data(), D->h_planes, s));
  double sx = 0.0, si = 0.0;
  for (int z = 0; z < D->nzg; ++z) { sx += D->h_planes[z].x; si += D->h_planes[z].y; }
  const double Ntot = (double)nx * ny * nzg;
  for (int i = 0; i < np; ++i) launch_add_scalar(x0[i], (long long)plane * D->nzl[i], (float)((si - sx) / Ntot), s);
  CKD(cudaEventRecord(c.ev1, s));
  CKD(cudaEventSynchronize(c.ev1));
  r.vcycles = k;
  r.status = status;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c.ev0, c.ev1);
  r.seconds = ms * 1e-3;
  r.kernel_launches = g_launches.load() - before;
  if (rep) *rep = r;
  if (status == GDP_ENOCONV) set_err(GDP_ENOCONV, "distributed diffuse_z: not converged after %d V-cycles", k);
  return status;
}

}  // namespace gdp
