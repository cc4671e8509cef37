// gdp_march3d.cu — fused 3D level passes (levels with z links: phase 1, Eq. 1), sm_100a.
//
// One HBM pass = one full red-black Gauss-Seidel sweep of a level, optionally
// preceded by the prolongated coarse correction (a8) and followed by the residual, restricted
// to the coarse level (a5+a6) or reduced to fp64 norms (a5).  This is the paper's streaming
// pass over a sliding window of slices moved on chip: a persistent CTA owns
// an in-plane tile (128 x 32 cells, 4-cell halo recomputed; 16 warps of 2 rows) and marches along z through a chunk
// of planes.  With t the plane being loaded:
//     stage 1 (colour 0) updates plane t-1, stage 2 (colour 1) updates plane t-2,
//     the tail takes the residual of plane t-3 and stores its x,
// which is exactly the reference schedule's two half-sweeps: a point of one colour depends only
// on points of the other colour (colour = (x + y + z_global) & 1).
//
// Data movement per plane step:
//   * x and b planes of the tile are staged into shared memory by cp.async MD planes ahead;
//     every thread stages and later reads only its own cells, so no barrier guards them;
//   * each thread keeps x of its 4 x 2 cells for the six newest planes in registers (ring
//     indexed by z mod 6, the loop is unrolled six-fold so every index is static); z-neighbours
//     are registers, x-neighbours come from the adjacent lane (__shfl), y-neighbours from the
//     thread's own rows or, at warp boundaries, from rows the neighbouring warps published in
//     the previous step (only the pack the next stage reads; double-buffered by step parity);
//   * one __syncthreads per plane step orders those row exchanges.
// Per-cell arithmetic is the reference one (apply_from order, gs_update with the correctly
// rounded 1/D, rw3 / bilerp for the transfers), done on f32x2 packs (FFMA2), so the iterates
// are bit-identical to the reference schedule (tests/test_gpu_parity.py).
#include <cooperative_groups.h>

#include "gdp_internal.h"
#include "gdp_pack.cuh"

namespace cg = cooperative_groups;

namespace gdp {

constexpr int MW = 16;                     // warps per CTA, stacked in y
constexpr int MR = 2;                      // rows per warp
constexpr int MROWS = MW * MR;             // 32
constexpr int MCOLS = 128;                 // 4 columns per lane
constexpr int MHX = 4, MHY = 4;            // halo >= 3 (two half-sweeps + residual); x: lane quads, y: = MR
constexpr int MTXI = MCOLS - 2 * MHX;      // 120
constexpr int MCL = 1;                     // CTAs per cluster, stacked in y: their facing rows are
                                           // exchanged through distributed shared memory, so only
                                           // the cluster's outer rows are halo.  MCL = 2 is
                                           // bit-identical but measured slower on B200 (the
                                           // per-step cluster barrier costs more than the
                                           // 75% -> 87.5% row efficiency gains): 1
constexpr int MTYI = MCL * MROWS - 2 * MHY;  // 56 interior rows per cluster tile
constexpr int MT = MW * 32;                // 512 threads
constexpr int MD = 2;                      // prefetch distance (planes)
constexpr int MXS = 3;                     // x staging slots (>= MD + 1, divides 6)
constexpr int MBS = 6;                     // b staging slots (>= MD + 4: b of plane q is read until step q + 3)
constexpr int MRING = 6;                   // x planes in registers (t-4 .. t, period 6 keeps parity static)
constexpr int MNQ = MR / 2 + 2;            // coarse rows of a thread's prolongation
static_assert(MXS >= MD + 1 && MBS >= MD + 4 && MRING % MXS == 0 && MRING % MBS == 0, "slots");
static_assert(MHY % MR == 0 && MR % 2 == 0 && MHX % 4 == 0 && MTYI % 2 == 0, "tile geometry");

enum { TAIL_NONE = 0, TAIL_RESTRICT = 1, TAIL_NORMS = 2 };

struct March3D {
  LevelK L;              // fine level (single slab: local planes == global planes - z0)
  const float* xin;      // x before the pass (ignored if zero_x)
  float* xout;           // x after the pass (another buffer: tiles read each other's halo)
  const float* b;        // rhs of the level
  int zero_x;            // coarse-level down pass: x starts at 0
  XferAxis tx, ty, tz;   // fine -> coarse (x and y coarsened; z optionally)
  int ncx, ncy;          // coarse plane dims
  float* bc;             // TAIL_RESTRICT: coarse rhs
  const float* xc;       // PROLONG: coarse correction
  double2* partials;     // TAIL_NORMS: one (sum r^2, sum b^2) per item
  int tiles_x, tiles_y;
  int zlo, zhi;          // planes whose final values this launch produces
  // work split over the persistent CTAs: `full` waves of whole tiles (tile k*grid + cta, all
  // planes), then the remaining tiles' (tile, plane) list in tile-major order cut into grid
  // contiguous runs -- so the plane pipeline restarts only at tile boundaries
  int full;
  int zeven;             // runs start on even planes (z-coarsened restriction pairs)
  int max_segs;          // partial slots per CTA (TAIL_NORMS)
  int nitems;            // grid * max_segs
};

struct SmemM {
  float4 xs[MXS][MR][MT];          // staged x rows (memory order c0..c3)
  float4 bs[MBS][MR][MT];          // staged b rows
  float2 ex[2][2][MW][2][32];      // [consumer stage 1|2][step parity][warp][row 0 | row MR-1][lane]: one pack
  float4 et[2][MW][2][32];         // rows 0 | MR-1 after stage 2 (both packs) for the tail
  float2 inv[4][6][2][32];         // 1/D per [plane class][row class][pack][lane]
};
constexpr size_t SMEMM = sizeof(SmemM);

// row / plane classes of the diagonal: the link coefficients of a row depend only on these
__device__ __forceinline__ int row_class(int g, int n) {
  return g < 0 ? 4 : (g >= n ? 5 : (g == 0 ? 1 : (g == n - 1 ? 3 : (g == n - 2 ? 2 : 0))));
}
__device__ __forceinline__ int row_rep(int c, int n) {  // an index of class c (class 0 only exists for n >= 4)
  return c == 0 ? 1 : (c == 1 ? 0 : (c == 2 ? n - 2 : (c == 3 ? n - 1 : (c == 4 ? -1 : n))));
}
__device__ __forceinline__ int plane_class(long long g, int n) {
  return g == 0 ? 1 : (g == n - 1 ? 3 : (g == n - 2 ? 2 : 0));
}

struct Pk { float2 A[MR], B[MR]; };  // x of a thread's 4 x MR cells: A = (c0, c2), B = (c1, c3)

__device__ __forceinline__ float4 row4(const Pk& X, int j) { return make_float4(X.A[j].x, X.A[j].y, X.B[j].x, X.B[j].y); }
__device__ __forceinline__ float4 row4s(const Pk& X, int j) { return make_float4(X.A[j].x, X.B[j].x, X.A[j].y, X.B[j].y); }
__device__ __forceinline__ float2 packA(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 packB(const float4& v) { return make_float2(v.z, v.w); }

template <int TAIL, bool PROLONG, bool ZC, bool VEC>
__global__ void __launch_bounds__(MT, 1) k_march3d(const __grid_constant__ March3D P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemM& S = *reinterpret_cast<SmemM*>(smem_raw);
  const LevelK& L = P.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = L.nx;
  const long long plane = (long long)L.nx * L.ny;  // < 2^31 (checked on the host)
  const int nzg = L.az.n;                          // single slab: local plane == global z
  const float2 al2 = f2(L.alpha);
  const int cplane = P.ncx * P.ncy;
  // exchange partners: the warp below / above, in this CTA or across the cluster boundary
  // (the cluster's outer edges read their own rows: halo)
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = MCL > 1 ? (int)cluster.block_rank() : 0;
  SmemM* Sdn = &S;
  SmemM* Sup = &S;
  int wdn = warp - 1, wup = warp + 1;
  if (warp == 0) {
    if (crank > 0) { Sdn = cluster.map_shared_rank(&S, crank - 1); wdn = MW - 1; }
    else wdn = 0;
  }
  if (warp == MW - 1) {
    if (crank < MCL - 1) { Sup = cluster.map_shared_rank(&S, crank + 1); wup = 0; }
    else wup = MW - 1;
  }
  // cluster: the step barrier is split: arrive once this step's exchange rows are published and
  // read (before the residual tail), wait at the start of the next step
  bool arrived = false;
  auto step_sync = [&]() {
    if constexpr (MCL > 1) {
      if (!arrived) asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      arrived = false;
    } else {
      __syncthreads();
    }
  };
  auto step_arrive = [&]() {
    if constexpr (MCL > 1) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      arrived = true;
    }
  };
  const float* invf = reinterpret_cast<const float*>(&S.inv[0][0][0][0]);

  Pk X[MRING];
#pragma unroll
  for (int k = 0; k < MRING; ++k)
#pragma unroll
    for (int j = 0; j < MR; ++j) X[k].A[j] = X[k].B[j] = f2(0.f);

  double sr = 0.0, sbb = 0.0;

  const int ntiles = P.tiles_x * P.tiles_y, nzr = P.zhi - P.zlo, G = gridDim.x / MCL;
  const int cid = blockIdx.x / MCL;  // the cluster: both CTAs walk the same work list
  const long long wr = (long long)(ntiles - P.full * G) * nzr;  // remaining tile-planes
  auto cut = [&](long long w) {  // start of run w of the remainder (even plane if zeven)
    long long q = wr * w / G;
    if (P.zeven) q -= (q % nzr) & 1;
    return q;
  };
  const long long r0 = cut(cid), r1 = cut(cid + 1);
  int seg = 0;
  long long rs = r0;
  for (;;) {
    int tile, p_lo, p_hi;
    if (seg < P.full) {
      tile = seg * G + cid;
      p_lo = P.zlo;
      p_hi = P.zhi;
    } else {
      if (rs >= r1) break;
      const long long tt = rs / nzr;
      const int z = (int)(rs - tt * nzr);
      tile = P.full * G + (int)tt;
      p_lo = P.zlo + z;
      p_hi = P.zlo + (int)min((long long)nzr, z + (r1 - rs));
      rs += p_hi - p_lo;
    }
    const int item = blockIdx.x * P.max_segs + seg;
    ++seg;
    const int tx_ = tile % P.tiles_x;
    const int ty_ = tile / P.tiles_x;

    // ---- column data of my lane (4 consecutive columns; packs A = (c0, c2), B = (c1, c3))
    const int gx0 = tx_ * MTXI - MHX + 4 * lane;
    bool cin[4];
    float cxl[4], cxr[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      cin[c] = gx0 + c >= 0 && gx0 + c < nx;
      cxl[c] = cl(L.ax, gx0 + c);
      cxr[c] = cr(L.ax, gx0 + c);
    }
    const float2 kxlA = make_float2(cxl[0], cxl[2]), kxrA = make_float2(cxr[0], cxr[2]);
    const float2 kxlB = make_float2(cxl[1], cxl[3]), kxrB = make_float2(cxr[1], cxr[3]);
    const bool lane_full = cin[0] && cin[1] && cin[2] && cin[3];
    const bool lane_any = cin[0] || cin[1] || cin[2] || cin[3];
    const bool pin = lane >= MHX / 4 && lane < 32 - MHX / 4;  // interior columns (whole lanes)

    // ---- row data of my rows
    const int crow = crank * MROWS + warp * MR;   // my first row within the cluster tile
    const int gyw = ty_ * MTYI - MHY + crow;       // even
    float2 ryl[MR], ryr[MR];
    int ivo[MR];   // offset of my (row class, lane) in the 1/D table
    int ro[MR];    // in-plane offset of my row quad (0 if outside)
    bool rin[MR];
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int gy = gyw + j;
      rin[j] = gy >= 0 && gy < L.ny;
      ryl[j] = f2(cl(L.ay, gy));
      ryr[j] = f2(cr(L.ay, gy));
      ivo[j] = (row_class(gy, L.ay.n) * 2 * 32 + lane) * 2;
      ro[j] = rin[j] ? gy * nx + gx0 : 0;
    }
    const bool wint = crow >= MHY && crow < MCL * MROWS - MHY;  // interior rows (whole warps)

    // restriction weights of my children (hoisted; rw3 = (wz * wy) * wx per element)
    float2 rwxA, rwxB, rwy[MR];
    if (TAIL == TAIL_RESTRICT) {
      rwxA = make_float2(rweight(P.tx, gx0), rweight(P.tx, gx0 + 2));
      rwxB = make_float2(rweight(P.tx, gx0 + 1), rweight(P.tx, gx0 + 3));
#pragma unroll
      for (int j = 0; j < MR; ++j) rwy[j] = f2(rweight(P.ty, gyw + j));
    }

    // ---- 1/D table of this tile's columns (the previous item may still read the old one)
    if constexpr (MCL > 1) {  // complete a pending arrive of the previous item's last step
      if (arrived) { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); arrived = false; }
    }
    __syncthreads();
    for (int i = tid; i < 4 * 6 * 2 * 32; i += MT) {
      const int ln = i & 31, pk = (i >> 5) & 1, rc = (i >> 6) % 6, zc = (i >> 6) / 6;
      const int ry = row_rep(rc, L.ay.n);
      const int zr = zc == 0 ? 1 : (zc == 1 ? 0 : (zc == 2 ? nzg - 2 : nzg - 1));
      float v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gx = tx_ * MTXI - MHX + 4 * ln + pk + 2 * h;
        Coef k;
        k.xl = cl(L.ax, gx); k.xr = cr(L.ax, gx);
        k.yl = cl(L.ay, ry); k.yr = cr(L.ay, ry);
        k.zl = cl(L.az, zr); k.zr = cr(L.az, zr);
        const float D = k.diag(L.alpha);
        v[h] = D > 0.f ? relax_inv(L.omega, D) : 0.f;  // == the weight of gs_update
      }
      S.inv[zc][rc][pk][ln] = make_float2(v[0], v[1]);
    }

    // z link coefficients of a plane: branch-free selects on per-kernel constants
    const float kz = L.az.k, kzl = L.az.kl, kzr = L.az.kr;
    auto zcoef = [&](int q, float2& zl2, float2& zr2, int& zoff) {
      const bool first = q == 0, last = q == nzg - 1, penult = q == nzg - 2;
      zl2 = f2(first ? 0.f : (last ? kzl : kz));
      zr2 = f2(last ? 0.f : (penult ? kzr : kz));
      zoff = (first ? 1 : (last ? 3 : (penult ? 2 : 0))) * (6 * 2 * 32 * 2);  // plane_class * table stride
    };

    // ---- prolongation taps (per column / row, fixed for the item)
    float ptx[4];
    bool selfJ[4];
    float pty[MR];
    int pdq[MR];
    const int Ix0 = gx0 >> 1;
    const int Jw = (gyw >> 1) - 1;
    if (PROLONG) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        long long I, J;
        ptaps(P.tx, gx0 + c, I, J, ptx[c]);
        selfJ[c] = J == I;
      }
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        long long I, J;
        ptaps(P.ty, gyw + j, I, J, pty[j]);
        pdq[j] = (int)(J - I);
      }
    }
    auto load_cv = [&](long long cz, float2 (&cv)[MNQ]) {  // coarse rows Jw.., columns (Ix0, Ix0+1)
      const float* xcp = P.xc + cz * cplane;
      const bool cvec = (P.ncx & 1) == 0 && Ix0 >= 0 && Ix0 + 1 < P.ncx;
#pragma unroll
      for (int q = 0; q < MNQ; ++q) {
        const int J = Jw + q;
        const bool rq = J >= 0 && J < P.ncy;
        const float* rp = xcp + J * P.ncx + Ix0;
        if (rq && cvec) cv[q] = __ldg(reinterpret_cast<const float2*>(rp));
        else cv[q] = make_float2((rq && Ix0 >= 0 && Ix0 < P.ncx) ? __ldg(rp) : 0.f,
                                 (rq && Ix0 + 1 >= 0 && Ix0 + 1 < P.ncx) ? __ldg(rp + 1) : 0.f);
      }
    };
    // bilinear correction packs of one coarse plane (bilerp order of k_prolong_rows per element)
    auto bil_plane = [&](const float2 (&cv)[MNQ], float2 (&eA)[MR], float2 (&eB)[MR]) {
      float2 cn[MNQ];
#pragma unroll
      for (int q = 0; q < MNQ; ++q)
        cn[q] = make_float2(__shfl_up_sync(FULL, cv[q].y, 1), __shfl_down_sync(FULL, cv[q].x, 1));
      const float2 txA = make_float2(ptx[0], ptx[2]), txB = make_float2(ptx[1], ptx[3]);
      const float2 uxA = make_float2(1.f - ptx[0], 1.f - ptx[2]), uxB = make_float2(1.f - ptx[1], 1.f - ptx[3]);
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const int q = (j >> 1) + 1;
        const int dq = pdq[j];
        const float2 r0 = cv[q], r1 = cn[q];
        const float2 n0 = dq < 0 ? cv[q - 1] : (dq > 0 ? cv[q + 1] : cv[q]);
        const float2 n1 = dq < 0 ? cn[q - 1] : (dq > 0 ? cn[q + 1] : cn[q]);
        const float2 aJ = make_float2(selfJ[0] ? r0.x : r1.x, selfJ[2] ? r0.y : r0.x);
        const float2 cJ = make_float2(selfJ[0] ? n0.x : n1.x, selfJ[2] ? n0.y : n0.x);
        const float2 bJ = make_float2(selfJ[1] ? r0.x : r0.y, selfJ[3] ? r0.y : r1.y);
        const float2 dJ = make_float2(selfJ[1] ? n0.x : n0.y, selfJ[3] ? n0.y : n1.y);
        const float2 ty2 = f2(pty[j]), uy2 = f2(1.f - pty[j]);
        const float2 sA0 = __ffma2_rn(txA, aJ, __fmul2_rn(uxA, r0));
        const float2 sA1 = __ffma2_rn(txA, cJ, __fmul2_rn(uxA, n0));
        eA[j] = __ffma2_rn(ty2, sA1, __fmul2_rn(uy2, sA0));
        const float2 sB0 = __ffma2_rn(txB, bJ, __fmul2_rn(uxB, r0));
        const float2 sB1 = __ffma2_rn(txB, dJ, __fmul2_rn(uxB, n0));
        eB[j] = __ffma2_rn(ty2, sB1, __fmul2_rn(uy2, sB0));
      }
    };
    // coarse planes (and weight) of fine plane z
    auto ctaps = [&](int z, long long& I, long long& J, float& t) {
      if (ZC) ptaps(P.tz, z, I, J, t);
      else { I = z; J = z; t = 0.f; }
    };

    // ---- plane ranges of this item
    const int a = max(p_lo - 3, 0), e = min(p_hi + 3, nzg);
    const int s1lo = max(p_lo - 2, 0), s1hi = min(p_hi + 2, nzg);
    const int s2lo = max(p_lo - 1, 0), s2hi = min(p_hi + 1, nzg);
    const int tend = p_hi + 3;

    // cp.async staging of plane p into x slot XSL, b slot BSL (own cells only)
    auto issue = [&](int p, int xsl, int bsl) {
      const float* xp = P.xin + (long long)p * plane;
      const float* bp = P.b + (long long)p * plane;
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        if (VEC) {
          const bool ok = rin[j] && lane_full;
          if (!P.zero_x) cp_async16z(&S.xs[xsl][j][tid], xp + ro[j], ok);
          cp_async16z(&S.bs[bsl][j][tid], bp + ro[j], ok);
        } else {
          float* dx = reinterpret_cast<float*>(&S.xs[xsl][j][tid]);
          float* db = reinterpret_cast<float*>(&S.bs[bsl][j][tid]);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const bool ok = rin[j] && cin[c];
            const int o = ok ? ro[j] + c : 0;
            if (!P.zero_x) cp_async4z(dx + c, xp + o, ok);
            cp_async4z(db + c, bp + o, ok);
          }
        }
      }
    };
#pragma unroll
    for (int k = 0; k < MD; ++k) {
      if (a + k < e) issue(a + k, (a + k) % MXS, (a + k) % MBS);
      cp_async_commit();
    }
    float2 cvI[MNQ], cvJ[MNQ];  // coarse rows of the next plane to be loaded
    if (PROLONG && a < e) {
      long long I, J;
      float t;
      ctaps(a, I, J, t);
      load_cv(I, cvI);
      if (ZC) load_cv(J, cvJ);
    }
    float2 racc[MR / 2];  // ZC restriction: coarse rows accumulated over the two child planes
#pragma unroll
    for (int i = 0; i < MR / 2; ++i) racc[i] = f2(0.f);

    // (A x) of pack PK of row j of plane Xo (Xd below, Xu above), apply_from order
    auto stencil = [&](auto PKc, auto Jc, const Pk& Xo, const Pk& Xd, const Pk& Xu, float2 sv, float2 nv,
                       float2 zl2, float2 zr2) -> float2 {
      constexpr int PK = decltype(PKc)::value;
      constexpr int j = decltype(Jc)::value;
      if (PK == 0) {
        const float2 Xc = Xo.A[j];
        const float2 W = make_float2(__shfl_up_sync(FULL, Xo.B[j].y, 1), Xo.B[j].x);
        const float2 Sn = j > 0 ? Xo.A[j - 1] : sv;
        const float2 Nn = j < MR - 1 ? Xo.A[j + 1] : nv;
        float2 s = __fmul2_rn(al2, Xc);
        s = __ffma2_rn(kxlA, sub2(Xc, W), s);
        s = __ffma2_rn(kxrA, sub2(Xc, Xo.B[j]), s);
        s = __ffma2_rn(ryl[j], sub2(Xc, Sn), s);
        s = __ffma2_rn(ryr[j], sub2(Xc, Nn), s);
        s = __ffma2_rn(zl2, sub2(Xc, Xd.A[j]), s);
        return __ffma2_rn(zr2, sub2(Xc, Xu.A[j]), s);
      } else {
        const float2 Xc = Xo.B[j];
        const float2 E = make_float2(Xo.A[j].y, __shfl_down_sync(FULL, Xo.A[j].x, 1));
        const float2 Sn = j > 0 ? Xo.B[j - 1] : sv;
        const float2 Nn = j < MR - 1 ? Xo.B[j + 1] : nv;
        float2 s = __fmul2_rn(al2, Xc);
        s = __ffma2_rn(kxlB, sub2(Xc, Xo.A[j]), s);
        s = __ffma2_rn(kxrB, sub2(Xc, E), s);
        s = __ffma2_rn(ryl[j], sub2(Xc, Sn), s);
        s = __ffma2_rn(ryr[j], sub2(Xc, Nn), s);
        s = __ffma2_rn(zl2, sub2(Xc, Xd.B[j]), s);
        return __ffma2_rn(zr2, sub2(Xc, Xu.B[j]), s);
      }
    };

    // ---- one plane step: K = t mod 6 is static
    auto step = [&](auto KK, int t) {
      constexpr int K = decltype(KK)::value;
      constexpr int PAR = K & 1;  // parity of the step (and of z)
      step_sync();

      // (1) load plane t into X[K], add the coarse correction, publish its boundary rows
      if (t < e) {
        if (t + MD < e) issue(t + MD, (K + MD) % MXS, (K + MD) % MBS);
        cp_async_commit();
        cp_async_wait<MD>();
        Pk& Xt = X[K];
        if (P.zero_x) {
#pragma unroll
          for (int j = 0; j < MR; ++j) Xt.A[j] = Xt.B[j] = f2(0.f);
        } else {
#pragma unroll
          for (int j = 0; j < MR; ++j) {
            const float4 v = S.xs[K % MXS][j][tid];
            Xt.A[j] = make_float2(v.x, v.z);
            Xt.B[j] = make_float2(v.y, v.w);
          }
        }
        if (PROLONG) {
          long long I, J;
          float tz;
          ctaps(t, I, J, tz);
          float2 eA[MR], eB[MR];
          bil_plane(cvI, eA, eB);
          if (ZC && tz != 0.f) {
            float2 fA[MR], fB[MR];
            bil_plane(cvJ, fA, fB);
            const float2 tz2 = f2(tz), uz2 = f2(1.f - tz);
#pragma unroll
            for (int j = 0; j < MR; ++j) {
              eA[j] = __ffma2_rn(tz2, fA[j], __fmul2_rn(uz2, eA[j]));
              eB[j] = __ffma2_rn(tz2, fB[j], __fmul2_rn(uz2, eB[j]));
            }
          }
#pragma unroll
          for (int j = 0; j < MR; ++j) {
            Xt.A[j] = __fadd2_rn(Xt.A[j], eA[j]);
            Xt.B[j] = __fadd2_rn(Xt.B[j], eB[j]);
          }
          if (t + 1 < e) {  // coarse rows of the next plane (latency hidden behind this step)
            ctaps(t + 1, I, J, tz);
            load_cv(I, cvI);
            if (ZC) load_cv(J, cvJ);
          }
        }
        // consumer stage 1 (colour 0): my row 0 serves the warp below's row MR-1 (pack (1+z)&1),
        // my row MR-1 the warp above's row 0 (pack z&1)
        S.ex[0][PAR][warp][0][lane] = (PAR ^ 1) ? Xt.B[0] : Xt.A[0];
        S.ex[0][PAR][warp][1][lane] = PAR ? Xt.B[MR - 1] : Xt.A[MR - 1];
      } else {
#pragma unroll
        for (int j = 0; j < MR; ++j) X[K].A[j] = X[K].B[j] = f2(0.f);
      }

      // (2) a half-sweep of colour C on the plane q held in X[KO]
      auto stage = [&](auto Cc, auto KOc, int q) {
        constexpr int C = decltype(Cc)::value;
        constexpr int KO = decltype(KOc)::value;
        constexpr int KD = (KO + MRING - 1) % MRING, KU = (KO + 1) % MRING;
        constexpr int ZP = KO & 1;  // parity of the plane's z
        float2 zl2, zr2;
        int zoff;
        zcoef(q, zl2, zr2, zoff);
        Pk& Xo = X[KO];
        const float2 sv = Sdn->ex[C][PAR ^ 1][wdn][1][lane];  // pack (C + z)&1 of the row below my row 0
        const float2 nv = Sup->ex[C][PAR ^ 1][wup][0][lane];  // pack (C + 1 + z)&1 of the row above my row MR-1
        static_for<MR>([&](auto Jc) {
          constexpr int j = decltype(Jc)::value;
          constexpr int PK = (C + j + ZP) & 1;  // active pack of row j (gyw even, gx0 even)
          const float4 bv = S.bs[KO % MBS][j][tid];
          const float2 iD = *reinterpret_cast<const float2*>(invf + zoff + ivo[j] + PK * 64);
          const float2 s = stencil(IC<PK>{}, Jc, Xo, X[KD], X[KU], sv, nv, zl2, zr2);
          if (PK == 0) Xo.A[j] = __ffma2_rn(sub2(make_float2(bv.x, bv.z), s), iD, Xo.A[j]);
          else Xo.B[j] = __ffma2_rn(sub2(make_float2(bv.y, bv.w), s), iD, Xo.B[j]);
        });
        if (C == 0) {  // the packs stage 2 needs from my edge rows (the ones just updated)
          S.ex[1][PAR][warp][0][lane] = ZP ? Xo.B[0] : Xo.A[0];
          S.ex[1][PAR][warp][1][lane] = ZP ? Xo.A[MR - 1] : Xo.B[MR - 1];
        } else {       // the tail needs both packs
          S.et[PAR][warp][0][lane] = row4(Xo, 0);
          S.et[PAR][warp][1][lane] = row4(Xo, MR - 1);
        }
      };
      if (t - 1 >= s1lo && t - 1 < s1hi) stage(IC<0>{}, IC<(K + 5) % MRING>{}, t - 1);
      if (t - 2 >= s2lo && t - 2 < s2hi) stage(IC<1>{}, IC<(K + 4) % MRING>{}, t - 2);

      // (3) tail on plane q = t-3: residual -> restriction / norms, store x
      const int q = t - 3;
      const float4 tsv4 = Sdn->et[PAR ^ 1][wdn][1][lane];  // neighbour rows of the tail, read before
      const float4 tnv4 = Sup->et[PAR ^ 1][wup][0][lane];  // the barrier arrive (their buffer is rewritten next step)
      step_arrive();
      if (q >= p_lo && q < p_hi) {
        constexpr int KO = (K + 3) % MRING, KD = (K + 2) % MRING, KU = (K + 4) % MRING;
        constexpr int ZP = KO & 1;
        const Pk& Xo = X[KO];
        if (TAIL != TAIL_NONE && wint) {  // warp-uniform: the stencil shuffles need every lane
          float2 zl2, zr2;
          int zoff;
          zcoef(q, zl2, zr2, zoff);
          const float4 sv4 = tsv4;
          const float4 nv4 = tnv4;
          float2 rA[MR], rB[MR], bA[MR], bB[MR];
          static_for<MR>([&](auto Jc) {
            constexpr int j = decltype(Jc)::value;
            const float4 bv = S.bs[KO % MBS][j][tid];
            bA[j] = make_float2(bv.x, bv.z);
            bB[j] = make_float2(bv.y, bv.w);
            rA[j] = sub2(bA[j], stencil(IC<0>{}, Jc, Xo, X[KD], X[KU], packA(sv4), packA(nv4), zl2, zr2));
            rB[j] = sub2(bB[j], stencil(IC<1>{}, Jc, Xo, X[KD], X[KU], packB(sv4), packB(nv4), zl2, zr2));
          });
          if (TAIL == TAIL_RESTRICT && pin) {
            // volume-weighted child average, fz outer, fy, fx inner (k_restrict order); my
            // columns are the children of coarse columns (Ix0: c0, c1) and (Ix0 + 1: c2, c3)
            const float2 wz2 = f2(ZC ? rweight(P.tz, q) : 1.f);
            constexpr bool first = !ZC || ZP == 0;  // first child plane of the coarse plane
            const bool last = !ZC || ZP == 1 || q == nzg - 1;
            float* bcp = P.bc + (long long)(ZC ? (q >> 1) : q) * cplane;
#pragma unroll
            for (int jp = 0; jp < MR / 2; ++jp) {
              const int j0 = 2 * jp;
              if (!rin[j0]) continue;
              const float2 wzy0 = __fmul2_rn(wz2, rwy[j0]), wzy1 = __fmul2_rn(wz2, rwy[j0 + 1]);
              float2 acc = __ffma2_rn(__fmul2_rn(wzy0, rwxA), rA[j0], first ? f2(0.f) : racc[jp]);
              float2 tt = __ffma2_rn(__fmul2_rn(wzy0, rwxB), rB[j0], acc);
              acc = make_float2(cin[1] ? tt.x : acc.x, cin[3] ? tt.y : acc.y);
              if (rin[j0 + 1]) {
                acc = __ffma2_rn(__fmul2_rn(wzy1, rwxA), rA[j0 + 1], acc);
                tt = __ffma2_rn(__fmul2_rn(wzy1, rwxB), rB[j0 + 1], acc);
                acc = make_float2(cin[1] ? tt.x : acc.x, cin[3] ? tt.y : acc.y);
              }
              if (last) {
                const int J = (gyw + j0) >> 1;
                const bool ok0 = cin[0] && Ix0 < P.ncx && J < P.ncy;
                const bool ok1 = cin[2] && Ix0 + 1 < P.ncx && J < P.ncy;
                float* o = bcp + J * P.ncx + Ix0;
                if (VEC && ok0 && ok1 && (P.ncx & 1) == 0) *reinterpret_cast<float2*>(o) = acc;
                else {
                  if (ok0) o[0] = acc.x;
                  if (ok1) o[1] = acc.y;
                }
              } else {
                racc[jp] = acc;
              }
            }
          } else if (TAIL == TAIL_NORMS && pin) {
#pragma unroll
            for (int j = 0; j < MR; ++j) {
              if (!rin[j]) continue;
              const float rr[4] = {rA[j].x, rB[j].x, rA[j].y, rB[j].y};
              const float bb[4] = {bA[j].x, bB[j].x, bA[j].y, bB[j].y};
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (cin[c]) {
                  sr += (double)rr[c] * (double)rr[c];
                  sbb += (double)bb[c] * (double)bb[c];
                }
            }
          }
        }
        if (wint && pin && lane_any) {  // store the interior rows of plane q
          float* o = P.xout + (long long)q * plane;
#pragma unroll
          for (int j = 0; j < MR; ++j) {
            if (!rin[j]) continue;
            float* orow = o + ro[j];
            if (VEC) *reinterpret_cast<float4*>(orow) = row4s(Xo, j);
            else {
              if (cin[0]) orow[0] = Xo.A[j].x;
              if (cin[1]) orow[1] = Xo.B[j].x;
              if (cin[2]) orow[2] = Xo.A[j].y;
              if (cin[3]) orow[3] = Xo.B[j].y;
            }
          }
        }
      }
    };

    const int t0 = a - a % MRING;
    for (int T = t0; T < tend; T += MRING) {
      static_for<MRING>([&](auto KK) {
        const int t = T + decltype(KK)::value;
        if (t >= a && t < tend) step(KK, t);
      });
    }
    if (TAIL == TAIL_NORMS) {
      block_sum2(sr, sbb);
      if (tid == 0 && P.partials) P.partials[item] = make_double2(sr, sbb);
      sr = sbb = 0.0;
    }
  }
  if (TAIL == TAIL_NORMS && tid == 0 && P.partials)  // unused partial slots of this CTA
    for (; seg < P.max_segs; ++seg) P.partials[blockIdx.x * P.max_segs + seg] = make_double2(0.0, 0.0);
  if constexpr (MCL > 1) {  // the partner may still read my exchange rows
    if (arrived) asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    cluster.sync();
  }
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
static int g_nsm = 0;
static int num_sms() {
  if (!g_nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, dev);
    if (g_nsm <= 0) g_nsm = 148;
  }
  return g_nsm;
}

// co-resident clusters of MCL CTAs (1 CTA / SM each): at most SMs / MCL, fewer when a GPC has
// an odd number of free SMs
static int max_clusters() {
  static int n = 0;
  if (!n) {
    cudaFuncSetAttribute(k_march3d<1, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(MCL * 64);
    cfg.blockDim = dim3(MT);
    cfg.dynamicSmemBytes = SMEMM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = MCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, k_march3d<1, false, false, true>, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = num_sms() / MCL;
    }
    n = c;
  }
  return n;
}

bool fusable3d(const Level& L, const Level& C, const gdp_opts& o) {
  const bool zlinks = L.K.az.k != 0.f || L.K.az.kr != 0.f || L.K.az.kl != 0.f;
  // levels below ~2M cells take the reference kernels (one launch per half-sweep): the persistent
  // z-march's pipeline fill dominates there (config 1: 22.57 vs 22.87 ms per step with graphs)
  static const long long minc = getenv("GDP_F3D_MIN") ? atoll(getenv("GDP_F3D_MIN")) : 2000000LL;
  if ((long long)L.nx * L.ny * L.nzl < minc) return false;
  return (o.fused & 2) && zlinks && C.tx.coarsened && C.ty.coarsened &&
         L.nzl == L.gz.n /* single slab (no ghost planes) */ && L.z0 == 0 &&
         (long long)L.nx * L.ny < (1LL << 31) && (long long)C.nx * C.ny < (1LL << 31);
}

// work decomposition: tiles x z-chunks, the chunk count minimising waves x (chunk + 6)
static void plan3d(const LevelK& L, bool zc, int zlo, int zhi, March3D& P) {
  P.tiles_x = (L.nx + MTXI - 1) / MTXI;
  P.tiles_y = (L.ny + MTYI - 1) / MTYI;
  const int tiles = P.tiles_x * P.tiles_y;
  const int nz = zhi - zlo, nsm = num_sms();
  const long long work = (long long)tiles * nz;
  const int grid = (int)std::min<long long>(max_clusters(), work);  // clusters
  P.zlo = zlo;
  P.zhi = zhi;
  P.zeven = zc ? 1 : 0;
  P.full = tiles / grid;
  const long long rem = (long long)(tiles - P.full * grid) * nz;
  P.max_segs = P.full + (int)((rem + grid - 1) / grid / std::max(nz, 1)) + 3;
  P.nitems = grid * MCL * P.max_segs;
}

int fused3d_items(const Level& L, const Level& C, int zlo, int zhi) {
  March3D P{};
  if (zhi < 0) zhi = L.nzl;
  plan3d(L.K, C.tz.coarsened != 0, zlo, zhi, P);
  return P.nitems;
}

template <int TAIL, bool PROLONG, bool ZC, bool VEC>
static void launch_m3v(const March3D& P, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_march3d<TAIL, PROLONG, ZC, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMM);
    attr = true;
  }
  const int grid = P.nitems / P.max_segs;  // CTAs (clusters x MCL)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(MT);
  cfg.dynamicSmemBytes = SMEMM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MCL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_march3d<TAIL, PROLONG, ZC, VEC>, P);
}
template <int TAIL, bool PROLONG, bool ZC>
static void launch_m3(const March3D& P, cudaStream_t s) {
  if ((P.L.nx & 3) == 0 && al16(P.xin) && al16(P.xout) && al16(P.b)) launch_m3v<TAIL, PROLONG, ZC, true>(P, s);
  else launch_m3v<TAIL, PROLONG, ZC, false>(P, s);
}

// one fused sweep of level L over the planes [zlo, zhi) it finalises (all planes: 0, -1): tail 0
// none, 1 restrict into C.b, 2 norms into partials (one per item).  Plane p of x / b is read at
// xin / b + p * plane and written at xout + p * plane, so a caller streaming z-windows passes
// pointers offset by the window's first plane (the kernel touches planes [zlo-3, zhi+3) only).
int fused_sweep3d(const Level& L, const Level& C, const float* xin, float* xout, const float* b,
                  bool zero_x, bool prolong, int tail, double2* partials, cudaStream_t s, int zlo, int zhi) {
  March3D P{};
  if (zhi < 0) zhi = L.nzl;
  P.L = L.K; P.xin = xin; P.xout = xout; P.b = b; P.zero_x = zero_x ? 1 : 0;
  P.tx = C.tx; P.ty = C.ty; P.tz = C.tz; P.ncx = C.nx; P.ncy = C.ny;
  P.bc = C.b; P.xc = C.x; P.partials = partials;
  const bool zc = C.tz.coarsened != 0;
  plan3d(L.K, zc, zlo, zhi, P);
  const double N = (double)L.nx * L.ny * (zhi - zlo), Nc = (double)C.nx * C.ny * C.nzl * (zhi - zlo) / L.nzl;
  const double bytes = N * ((zero_x ? 4.0 : 8.0) + 4.0) + ((tail == 1 || prolong) ? Nc * 4.0 : 0.0);
  ProfScope ps(tail == 2 || prolong ? KC_UP3D : KC_DOWN3D, bytes, s, zhi - zlo == L.nzl ? N : 0.0, true);
  if (prolong) {
    if (tail == 2) { if (zc) launch_m3<2, true, true>(P, s); else launch_m3<2, true, false>(P, s); }
    else { if (zc) launch_m3<0, true, true>(P, s); else launch_m3<0, true, false>(P, s); }
  } else {
    if (tail == 1) { if (zc) launch_m3<1, false, true>(P, s); else launch_m3<1, false, false>(P, s); }
    else if (tail == 2) launch_m3<2, false, false>(P, s);
    else launch_m3<0, false, false>(P, s);
  }
  return P.nitems;
}

}  // namespace gdp
