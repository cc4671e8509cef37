// gdp_march3dv.cu — the 3D level sweep as a z-march with vertical f32x2 packs and TMA-staged
// planes (levels with z links: phase 1, Eq. 1), sm_100a.
//
// Same schedule as k_march3d (gdp_march3d.cu): one HBM pass = one red-black Gauss-Seidel sweep
// of a level, optionally preceded by the prolongated coarse correction (a8) and
// followed by the residual, restricted to the coarse level (a5 + a6) or reduced to fp64 norms
// (a5); a persistent CTA owns an in-plane tile and marches along z (stage 1, colour 0, on plane
// t-1; stage 2, colour 1, on t-2; the tail on t-3), so the iterate equals the reference
// schedule's half-sweeps bit for bit.  What differs is the data layout, chosen to cut the
// instruction count of a sweep (the per-sweep kernel is issue-bound):
//   * 8 warps x 8 rows, 2 columns per lane: a 64 x 64 tile with a 4-cell halo (77 % of it
//     final, against 70 % for k_march3d's 128 x 32 tile), 16 cells per thread so the per-stage
//     bookkeeping is spread over 8 updates;
//   * a thread's 8 x 2 cells are eight packs V[p][c] = (x[row r(p)][col c], x[row r(p)+2][col c]),
//     r = 0, 1, 4, 5: both cells of a pack have the same colour, so the FFMA2 / FADD2 stencil's
//     x, z and inner y neighbours are register pairs as they stand (k_march3d rebuilds its
//     column packs with register moves: ~24 % of its instructions);
//   * x and b planes arrive by TMA (cp.async.bulk.tensor) two planes ahead, completed on
//     mbarriers (no per-thread cp.async issue); the coarse correction's box likewise;
//   * the final plane leaves by TMA store from a staging tile (no per-row address / bounds code).
#include "gdp_vpass3d.cuh"

namespace gdp {
namespace mv {

using vp::mbar_expect;
using vp::mbar_init;
using vp::mbar_wait;
using vp::row_class;
using vp::row_rep;
using vp::sa;
using vp::tma3;

#ifndef GDP_M3V_MW
#define GDP_M3V_MW 11
#endif
constexpr int MW = GDP_M3V_MW;             // warps, stacked in y
constexpr int MR = 8;              // rows per warp
constexpr int MT = MW * 32;        // 352 threads
constexpr int TX = 64;             // tile columns (2 per lane)
constexpr int TY = MW * MR;        // 88 tile rows
constexpr int HX = 4, HY = 4;      // halo (>= 3: two half-sweeps + the residual)
constexpr int TXI = TX - 2 * HX;   // 56
constexpr int TYI = TY - 2 * HY;   // 80
constexpr int XS = 2;              // x slots (x of plane p issued at step p - 1)
constexpr int BS = 4;              // b slots (b of plane p issued at step p, read until p + 3)
constexpr int SS = 2;              // staged final planes (the tail's lower neighbour; TMA-stored one step later)
constexpr int RING = 4;            // register ring: planes t .. t-3 (even period keeps parity static)
constexpr int NQ = MR / 2 + 2;     // coarse rows a thread's prolongation reads
constexpr int CBX = 40;            // coarse box columns (lx + 2 <= 36; a multiple of 4: TMA rows)
constexpr int CBY = 4 * (MW - 1) + NQ;  // coarse box rows (46)

struct alignas(128) CBox { float v[CBY][CBX]; };

struct Tap { short i, j; float t; };  // parent / neighbour coarse index in the box, weight of the neighbour

template <bool PRO>
struct alignas(128) Smem {
  float xs[XS][TY][TX];
  float bs[BS][TY][TX];
  CBox cs[PRO ? XS : 1];
  float ex[2][2][MW][2][32];       // [consumer colour][parity][warp][row 0 | 7][lane]: one column each
  float2 et[2][MW][2][32];         // rows 0 | 7 after stage 2 (both columns) for the tail
  float inv[4][6][2][32];          // 1/D per [plane class][row class][column][lane]
  Tap tpx[TX], tpy[TY];
  float4 ky[MW][4];                // y links of pack p of warp w: (kyl row r, row r + 2, kyr row r, row r + 2)            // prolongation taps of the tile's columns / rows (box-relative)
  float st[SS][TYI][TXI];          // final interior planes, stored by TMA
  float stpad[4 * TXI + 2 * HX];   // the halo lanes' (discarded) reads past the last slot
  unsigned long long barx[XS];
  unsigned long long barb[BS];
};

struct Sweep {
  CUtensorMap tmx, tmb, tmc, tmo;
  LevelK L;
  float* xout;
  XferAxis tx, ty, tz;
  int ncx, ncy;
  float* bc;
  double2* partials;
  int zero_x;
  int tiles_x, tiles_y;
  int zlo, zhi;
  int full, zeven, max_segs, nitems;
};

enum { TAIL_NONE = 0, TAIL_RESTRICT = 1, TAIL_NORMS = 2 };

// TMA store of a staged box (clipped to the tensor: cells outside the level are not written)
__device__ __forceinline__ void tma_store3(const CUtensorMap* m, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<unsigned long long>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(sa(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// one shared-memory word (asm: keeps the compiler from merging neighbouring words into LDS.64,
// which would leave the vertical packs split across row pairs and cost register moves on use)
__device__ __forceinline__ float lds1(unsigned addr) {
  float v;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// a - b as fma(b, -1, a): the same rounding, no scalar negations for pairs built from two sources
__device__ __forceinline__ float2 subm(float2 a, float2 b) { return __ffma2_rn(b, f2(-1.f), a); }

// pack p holds rows (R0[p], R0[p] + 2) of the thread's 8 rows
__host__ __device__ constexpr int R0(int p) { return p < 2 ? p : p + 2; }

struct Pk { float2 V[4][2]; };  // V[p][c] = (x[row R0(p)][col c], x[row R0(p) + 2][col c])

static __device__ __noinline__ float2 rw_pair8(XferAxis tx, XferAxis ty, int gx, int gy, float wz) {
  const float wx = rweight(tx, gx);
  return make_float2(rw3(wz, rweight(ty, gy), wx), rw3(wz, rweight(ty, gy + 2), wx));
}

// EV (restriction on levels of even nx and ny): every in-level child has its sibling in the level,
// so out-of-level cells only feed coarse cells that are never stored -> no per-cell masks
template <int TAIL, bool PROLONG, bool ZC, bool EV = false>
__global__ void __launch_bounds__(MT, 1) k_m3v(const __grid_constant__ Sweep P) {
  using SM = Smem<PROLONG>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SM& S = *reinterpret_cast<SM*>(smem_raw + ((128u - (sa(smem_raw) & 127u)) & 127u));
  const LevelK& L = P.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = L.nx;
  const int nzg = L.az.n;
  const float2 al2 = f2(L.alpha);
  const int cplane = P.ncx * P.ncy;
  const int wdn = warp > 0 ? warp - 1 : 0, wup = warp < MW - 1 ? warp + 1 : MW - 1;
  const float* invf = &S.inv[0][0][0][0];
  if (tid == 0) {
    for (int i = 0; i < XS; ++i) mbar_init(&S.barx[i], 1);
    for (int i = 0; i < BS; ++i) mbar_init(&S.barb[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = tid; i < SS * TYI * TXI; i += MT) (&S.st[0][0][0])[i] = 0.f;  // finite (0 * x at z faces)
  Pk X[RING];
#pragma unroll
  for (int k = 0; k < RING; ++k)
#pragma unroll
    for (int p = 0; p < 4; ++p) X[k].V[p][0] = X[k].V[p][1] = f2(0.f);
  double sr = 0.0, sbb = 0.0;
  unsigned nxi = 0, nxw = 0, nbi = 0, nst = 0;
  int pend = -1, pbx = 0, pby = 0;  // plane whose staged store is not issued yet (uniform)
  auto flush_store = [&]() {        // after a barrier: the staged plane's writes are visible
    if (pend >= 0) {
      if (tid == 0) {
        tma_store3(&P.tmo, pbx, pby, pend, &S.st[(nst - 1) % SS][0][0]);
      }
      pend = -1;
    }
  };

  const int ntiles = P.tiles_x * P.tiles_y, nzr = P.zhi - P.zlo, G = gridDim.x;
  const int cid = blockIdx.x;
  const long long wr = (long long)(ntiles - P.full * G) * nzr;
  auto cut = [&](long long w) {
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
    const int bx0 = (tile % P.tiles_x) * TXI - HX;  // box origin (x: a multiple of 4, TMA-aligned)
    const int by0 = (tile / P.tiles_x) * TYI - HY;

    // ---- my 2 columns and 8 rows
    const int gx0 = bx0 + 2 * lane;  // even
    const bool cin0 = gx0 >= 0 && gx0 < nx, cin1 = gx0 + 1 >= 0 && gx0 + 1 < nx;
    const bool cin[2] = {cin0, cin1};
    const float kxl[2] = {cl(L.ax, gx0), cl(L.ax, gx0 + 1)}, kxr[2] = {cr(L.ax, gx0), cr(L.ax, gx0 + 1)};
    const bool lane_full = cin0 && cin1;
    const bool pin = lane >= HX / 2 && lane < 32 - HX / 2;  // interior columns (whole lanes)
    const int gyw = by0 + warp * MR;                         // even
    bool rin[MR], rint[MR];
    int ivo[MR];
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      rin[j] = gyw + j >= 0 && gyw + j < L.ny;
      rint[j] = warp * MR + j >= HY && warp * MR + j < TY - HY;
      const int rc = row_class(gyw + j, L.ay.n);
      ivo[j] = rc * 2 * 32 + lane;
    }
    const bool rfull = rin[0] && rin[1] && rin[2] && rin[3] && rin[4] && rin[5] && rin[6] && rin[7];
    if (lane < 4) {  // read after the item's first barrier
      const int g = gyw + R0(lane);
      S.ky[warp][lane] = make_float4(cl(L.ay, g), cl(L.ay, g + 2), cr(L.ay, g), cr(L.ay, g + 2));
    }
    // restriction weights 1/2 x 1/2 for the in-level children (the others are discarded)
    bool rwreg = TAIL == TAIL_RESTRICT;
    if (TAIL == TAIL_RESTRICT) {
#pragma unroll
      for (int c = 0; c < 2; ++c) rwreg = rwreg && (!cin[c] || rweight(P.tx, gx0 + c) == 0.5f);
#pragma unroll
      for (int j = 0; j < MR; ++j) rwreg = rwreg && (!rin[j] || rweight(P.ty, gyw + j) == 0.5f);
    }

    __syncthreads();  // the previous item's readers of the 1/D table are done
    for (int i = tid; i < 4 * 6 * 2 * 32; i += MT) {
      const int ln = i & 31, c = (i >> 5) & 1, rc = (i >> 6) % 6, zc = (i >> 6) / 6;
      const int ry = row_rep(rc, L.ay.n);
      const int zr = zc == 0 ? 1 : (zc == 1 ? 0 : (zc == 2 ? nzg - 2 : nzg - 1));
      const int gx = bx0 + 2 * ln + c;
      Coef k;
      k.xl = cl(L.ax, gx); k.xr = cr(L.ax, gx);
      k.yl = cl(L.ay, ry); k.yr = cr(L.ay, ry);
      k.zl = cl(L.az, zr); k.zr = cr(L.az, zr);
      const float D = k.diag(L.alpha);
      S.inv[zc][rc][c][ln] = D > 0.f ? relax_inv(L.omega, D) : 0.f;  // == the weight of gs_update
    }
    const float kz = L.az.k, kzl = L.az.kl, kzr = L.az.kr;
    auto zcoef = [&](int q, float2& zl2, float2& zr2, int& zoff) {
      const bool first = q == 0, last = q == nzg - 1, penult = q == nzg - 2;
      zl2 = f2(first ? 0.f : (last ? kzl : kz));
      zr2 = f2(last ? 0.f : (penult ? kzr : kz));
      zoff = (first ? 1 : (last ? 3 : (penult ? 2 : 0))) * (6 * 2 * 32);
    };

    // ---- prolongation (coarse box of the plane; regular taps 1/4, 3/4 away from faces)
    // prolongation: cells whose taps (ptaps) are not the regular ones (1/4 from parent +- 1 by
    // parity: faces, partial cells) take their taps from a per-tile table (bit 2 j + c of irr)
    unsigned irr = 0;
    const int cbx0 = ((bx0 >> 1) - 1) & ~3, cby0 = (by0 >> 1) - 1;
    const int Ix0 = gx0 >> 1;
    const int lx = Ix0 - 1 - cbx0, ly = ((gyw >> 1) - 1) - cby0;
    if (PROLONG) {
      auto regular = [](const XferAxis& ax, int i) {
        long long I, J;
        float t;
        ptaps(ax, i, I, J, t);
        return t == 0.25f && I == (i >> 1) && J == ((i & 1) ? I + 1 : I - 1);
      };
      bool xr[2], yr[MR];
#pragma unroll
      for (int c = 0; c < 2; ++c) xr[c] = !cin[c] || regular(P.tx, gx0 + c);
#pragma unroll
      for (int j = 0; j < MR; ++j) yr[j] = !rin[j] || regular(P.ty, gyw + j);
#pragma unroll
      for (int j = 0; j < MR; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if (!(xr[c] && yr[j])) irr |= 1u << (2 * j + c);
      if (tid < TX + TY) {  // the taps of column / row tid (read after the item's first barrier)
        const bool isx = tid < TX;
        const int i = isx ? bx0 + tid : by0 + (tid - TX);
        long long I, J;
        float t;
        ptaps(isx ? P.tx : P.ty, i, I, J, t);
        const int o = isx ? cbx0 : cby0;
        const Tap tp{(short)(I - o), (short)(J - o), t};
        if (isx) S.tpx[tid] = tp;
        else S.tpy[tid - TX] = tp;
      }
    }
    auto prolong_packs = [&](const CBox& box, float2 (&e)[4][2]) {
      // coarse rows q = 0..5 at ly + q, coarse columns k = 0..2 at lx + k; column c0: (I k1,
      // J k0), c1: (I k1, J k2).  Fine row 2m (even): (I q m+1, J q m); 2m+1: (I q m+1, J q m+2).
      float a[NQ][3];
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int k = 0; k < 3; ++k) a[q][k] = box.v[ly + q][lx + k];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int kj = c == 0 ? 0 : 2;
        float2 pq[NQ - 1];  // x-interpolated (coarse row q, q + 1)
#pragma unroll
        for (int q = 0; q < NQ - 1; ++q)
          pq[q] = __ffma2_rn(f2(0.25f), make_float2(a[q][kj], a[q + 1][kj]),
                             __fmul2_rn(f2(0.75f), make_float2(a[q][1], a[q + 1][1])));
        // rows (0, 2): J (q0, q1), I (q1, q2); rows (1, 3): J (q2, q3), I (q1, q2);
        // rows (4, 6): J (q2, q3), I (q3, q4); rows (5, 7): J (q4, q5), I (q3, q4)
        e[0][c] = __ffma2_rn(f2(0.25f), pq[0], __fmul2_rn(f2(0.75f), pq[1]));
        e[1][c] = __ffma2_rn(f2(0.25f), pq[2], __fmul2_rn(f2(0.75f), pq[1]));
        e[2][c] = __ffma2_rn(f2(0.25f), pq[2], __fmul2_rn(f2(0.75f), pq[3]));
        e[3][c] = __ffma2_rn(f2(0.25f), pq[4], __fmul2_rn(f2(0.75f), pq[3]));
      }
      if (irr) {  // faces / partial cells (a few lanes): those cells from the tap tables
        static_for<2 * MR>([&](auto Bc) {
          constexpr int bit = decltype(Bc)::value, j = bit >> 1, c = bit & 1;
          constexpr int p = (j & 1) + ((j >> 2) << 1);
          if (irr & (1u << bit)) {
            const Tap ty = S.tpy[warp * MR + j], tx = S.tpx[2 * lane + c];
            const float v = bilerp(box.v[ty.i][tx.i], box.v[ty.i][tx.j], box.v[ty.j][tx.i], box.v[ty.j][tx.j], tx.t, ty.t);
            if ((j >> 1) & 1) e[p][c].y = v;
            else e[p][c].x = v;
          }
        });
      }
    };

    // ---- plane ranges, TMA issue
    const int a = max(p_lo - 3, 0), e = min(p_hi + 3, nzg);
    const int s1lo = max(p_lo - 2, 0), s1hi = min(p_hi + 2, nzg);
    const int s2lo = max(p_lo - 1, 0), s2hi = min(p_hi + 1, nzg);
    const int tend = p_hi + 3;
    const unsigned nb0 = nbi;  // b of plane p lives in slot (nb0 + p - a) % BS
    auto issue_x = [&](int p) {
      const unsigned s = nxi % XS;
      if (tid == 0) {
        unsigned bytes = P.zero_x ? 0u : (unsigned)(TX * TY * 4);
        if (PROLONG) bytes += (unsigned)(CBX * CBY * 4);
        if (bytes) {
          mbar_expect(&S.barx[s], bytes);
          if (!P.zero_x) tma3(&S.xs[s][0][0], &P.tmx, bx0, by0, p, &S.barx[s]);
          if (PROLONG) tma3(&S.cs[s].v[0][0], &P.tmc, cbx0, cby0, p, &S.barx[s]);
        }
      }
      ++nxi;
    };
    auto issue_b = [&](int p) {
      const unsigned s = nbi % BS;
      if (tid == 0) {
        mbar_expect(&S.barb[s], (unsigned)(TX * TY * 4));
        tma3(&S.bs[s][0][0], &P.tmb, bx0, by0, p, &S.barb[s]);
      }
      ++nbi;
    };
    const bool xbytes = !P.zero_x || PROLONG;
    __syncthreads();  // the 1/D table is written; every slot is free
    for (int k = 0; k < XS - 1; ++k)
      if (a + k < e) issue_x(a + k);
    unsigned nbw = nb0;
    float2 racc[2] = {f2(0.f), f2(0.f)};  // ZC restriction: coarse rows (J, J + 1), (J + 2, J + 3)

    // (A x) of pack (PP, C) of plane Xo, apply_from order; sv / nv: row -1 / row 8 in column C
    auto stencil = [&](auto Pc, auto Cc, const Pk& Xo, const Pk& Xd, const Pk& Xu, float sv, float nv, float2 zl2,
                       float2 zr2) -> float2 {
      constexpr int PP = decltype(Pc)::value, C = decltype(Cc)::value;
      const float2 Xc = Xo.V[PP][C];
      float2 W, E;
      if constexpr (C == 1) W = Xo.V[PP][0];
      else W = make_float2(__shfl_up_sync(FULL, Xo.V[PP][1].x, 1), __shfl_up_sync(FULL, Xo.V[PP][1].y, 1));
      if constexpr (C == 0) E = Xo.V[PP][1];
      else E = make_float2(__shfl_down_sync(FULL, Xo.V[PP][0].x, 1), __shfl_down_sync(FULL, Xo.V[PP][0].y, 1));
      float2 Sn, Nn;
      if constexpr (PP == 0) { Sn = make_float2(sv, Xo.V[1][C].x); Nn = Xo.V[1][C]; }
      if constexpr (PP == 1) { Sn = Xo.V[0][C]; Nn = make_float2(Xo.V[0][C].y, Xo.V[2][C].x); }
      if constexpr (PP == 2) { Sn = make_float2(Xo.V[1][C].y, Xo.V[3][C].x); Nn = Xo.V[3][C]; }
      if constexpr (PP == 3) { Sn = Xo.V[2][C]; Nn = make_float2(Xo.V[2][C].y, nv); }
      float2 s = __fmul2_rn(al2, Xc);
      s = __ffma2_rn(f2(kxl[C]), sub2(Xc, W), s);
      s = __ffma2_rn(f2(kxr[C]), sub2(Xc, E), s);
      const float4 ky = S.ky[warp][PP];
      s = __ffma2_rn(make_float2(ky.x, ky.y), (PP == 0 || PP == 2) ? subm(Xc, Sn) : sub2(Xc, Sn), s);
      s = __ffma2_rn(make_float2(ky.z, ky.w), (PP == 1 || PP == 3) ? subm(Xc, Nn) : sub2(Xc, Nn), s);
      s = __ffma2_rn(zl2, sub2(Xc, Xd.V[PP][C]), s);
      return __ffma2_rn(zr2, sub2(Xc, Xu.V[PP][C]), s);
    };

    auto step = [&](auto KK, int t) {
      constexpr int K = decltype(KK)::value;
      constexpr int PAR = K & 1;
      __syncthreads();
      flush_store();
      if (t + XS - 1 < e) issue_x(t + XS - 1);
      if (t < e) issue_b(t);
      if (t - 1 >= a && t - 1 < e) {  // b of plane t - 1: stage 1 reads it below
        mbar_wait(&S.barb[nbw % BS], (nbw / BS) & 1);
        ++nbw;
      }
      // (1) plane t into X[K] (+ the coarse correction); publish the cells stage 1 of the
      // neighbouring warps reads: colour 1 of row 7 (column t & 1) and of row 0 (column 1 - t & 1)
      if (t < e) {
        const unsigned s = nxw % XS;
        const unsigned ph = (nxw / XS) & 1;
        ++nxw;
        if (xbytes) mbar_wait(&S.barx[s], ph);
        Pk& Xt = X[K];
        if (P.zero_x) {
#pragma unroll
          for (int p = 0; p < 4; ++p) Xt.V[p][0] = Xt.V[p][1] = f2(0.f);
        } else {
          const unsigned r = sa(&S.xs[s][warp * MR][2 * lane]);
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int c = 0; c < 2; ++c)
              Xt.V[p][c] = make_float2(lds1(r + 4 * (R0(p) * TX + c)), lds1(r + 4 * ((R0(p) + 2) * TX + c)));
        }
        if constexpr (PROLONG) {
          float2 ec[4][2];
          prolong_packs(S.cs[s], ec);
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int c = 0; c < 2; ++c) Xt.V[p][c] = __fadd2_rn(Xt.V[p][c], ec[p][c]);
        }
        S.ex[0][PAR][warp][0][lane] = Xt.V[0][1 - PAR].x;  // row 0, column (1 + t) & 1
        S.ex[0][PAR][warp][1][lane] = Xt.V[3][PAR].y;      // row 7, column t & 1
      } else {
#pragma unroll
        for (int p = 0; p < 4; ++p) X[K].V[p][0] = X[K].V[p][1] = f2(0.f);
      }

      // (2) half-sweep of colour C on plane q in X[KO]: packs 0, 2 at column (C + z) & 1,
      // packs 1, 3 at the other column
      auto stage = [&](auto Cc, auto KOc, int q) {
        constexpr int C = decltype(Cc)::value;
        constexpr int KO = decltype(KOc)::value;
        constexpr int KD = (KO + RING - 1) % RING, KU = (KO + 1) % RING;
        constexpr int ZP = KO & 1;  // X[k] holds a plane = k mod RING
        constexpr int C0 = (C + ZP) & 1, C1 = (C + 1 + ZP) & 1;
        float2 zl2, zr2;
        int zoff;
        zcoef(q, zl2, zr2, zoff);
        Pk& Xo = X[KO];
        const float sv = S.ex[C][PAR ^ 1][wdn][1][lane];  // row -1 at column C0
        const float nv = S.ex[C][PAR ^ 1][wup][0][lane];  // row 8 at column C1
        const float* brow = &S.bs[(nb0 + (unsigned)(q - a)) % BS][warp * MR][2 * lane];
        static_for<4>([&](auto Pc) {
          constexpr int PP = decltype(Pc)::value;
          constexpr int CC = (PP & 1) ? C1 : C0;
          const float2 bv = make_float2(brow[R0(PP) * TX + CC], brow[(R0(PP) + 2) * TX + CC]);
          const float2 iD = make_float2(invf[zoff + ivo[R0(PP)] + CC * 32], invf[zoff + ivo[R0(PP) + 2] + CC * 32]);
          const float2 st = stencil(Pc, IC<CC>{}, Xo, X[KD], X[KU], sv, nv, zl2, zr2);
          Xo.V[PP][CC] = __ffma2_rn(iD, sub2(bv, st), Xo.V[PP][CC]);
        });
        if constexpr (C == 0) {  // stage 2 (colour 1) needs my just-updated colour-0 edge cells:
          // its pack-0 column is C1 -> my row 7 there; its pack-3 column is C0 -> my row 0 there
          S.ex[1][PAR][warp][0][lane] = Xo.V[0][C0].x;
          S.ex[1][PAR][warp][1][lane] = Xo.V[3][C1].y;
        } else {  // the tail needs both columns of rows 0 and 7
          S.et[PAR][warp][0][lane] = make_float2(Xo.V[0][0].x, Xo.V[0][1].x);
          S.et[PAR][warp][1][lane] = make_float2(Xo.V[3][0].y, Xo.V[3][1].y);
        }
      };
      if (t - 1 >= s1lo && t - 1 < s1hi) stage(IC<0>{}, IC<(K + RING - 1) % RING>{}, t - 1);
      if (t - 2 >= s2lo && t - 2 < s2hi) stage(IC<1>{}, IC<(K + RING - 2) % RING>{}, t - 2);

      // (3) tail on plane q = t - 3 (final): residual -> restriction / norms, staged for the TMA
      // store; its lower neighbour q - 1 is the plane staged the step before (interior cells only:
      // the halo cells' residuals are discarded), so plane p_lo - 1 is staged too (not stored)
      const int q = t - 3;
      if (q >= max(p_lo - 1, 0) && q < p_hi) {
        constexpr int KO = (K + RING - 3) % RING, KU = (K + RING - 2) % RING;
        constexpr int ZP = KO & 1;
        const Pk& Xo = X[KO];
        if (TAIL != TAIL_NONE && q >= p_lo) {
          Pk Xl;  // plane q - 1 (final), from the staging slot
          {
            const unsigned r = sa(&S.st[(nst + SS - 1) % SS][0][0]) + 4 * ((warp * MR - HY) * TXI + 2 * lane - HX);
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
              for (int c = 0; c < 2; ++c)
                Xl.V[p][c] = make_float2(lds1(r + 4 * (R0(p) * TXI + c)), lds1(r + 4 * ((R0(p) + 2) * TXI + c)));
          }
          float2 zl2, zr2;
          int zoff;
          zcoef(q, zl2, zr2, zoff);
          const float2 tsv = S.et[PAR ^ 1][wdn][1][lane];  // row -1, columns 0 / 1
          const float2 tnv = S.et[PAR ^ 1][wup][0][lane];  // row 8
          const float* brow = &S.bs[(nb0 + (unsigned)(q - a)) % BS][warp * MR][2 * lane];
          const float wz = ZC ? rweight(P.tz, q) : 1.f;
          const bool first = !ZC || ZP == 0;
          float2 acc[2] = {first ? f2(0.f) : racc[0], first ? f2(0.f) : racc[1]};
          float2 nr = f2(0.f), nb = f2(0.f);  // norms: this plane's 16 cells in fp32, then fp64 once
          // order per coarse pair: (rows 2m: c 0, c 1), (rows 2m + 1: c 0, c 1) = fy outer, fx inner
          static_for<8>([&](auto Ic) {
            constexpr int i = decltype(Ic)::value;
            constexpr int PP = i >> 1, CC = i & 1;
            constexpr int RR = R0(PP);
            const float2 bb = make_float2(brow[RR * TX + CC], brow[(RR + 2) * TX + CC]);
            const float2 r = sub2(bb, stencil(IC<PP>{}, IC<CC>{}, Xo, Xl, X[KU], CC ? tsv.y : tsv.x,
                                              CC ? tnv.y : tnv.x, zl2, zr2));
            if (TAIL == TAIL_RESTRICT) {
              const float2 w = (EV || rwreg) ? f2(rw3(wz, 0.5f, 0.5f)) : rw_pair8(P.tx, P.ty, gx0 + CC, gyw + RR, wz);
              float2& ac = acc[PP >> 1];
              const float2 n = __ffma2_rn(w, r, ac);
              if (EV || (lane_full && rfull)) ac = n;
              else ac = make_float2(cin[CC] && rin[RR] ? n.x : ac.x, cin[CC] && rin[RR + 2] ? n.y : ac.y);
            } else if (TAIL == TAIL_NORMS) {
              const bool mx = pin && cin[CC] && rint[RR] && rin[RR];
              const bool my = pin && cin[CC] && rint[RR + 2] && rin[RR + 2];
              const float2 rm = make_float2(mx ? r.x : 0.f, my ? r.y : 0.f);
              const float2 bm = make_float2(mx ? bb.x : 0.f, my ? bb.y : 0.f);
              nr = __ffma2_rn(rm, rm, nr);
              nb = __ffma2_rn(bm, bm, nb);
            }
          });
          if (TAIL == TAIL_NORMS) {
            sr += (double)nr.x + (double)nr.y;
            sbb += (double)nb.x + (double)nb.y;
          }
          if (TAIL == TAIL_RESTRICT && pin) {
            const bool last = !ZC || ZP == 1 || q == nzg - 1;
            if (last) {
              float* bcp = P.bc + (long long)(ZC ? (q >> 1) : q) * cplane;
              if (cin0 && Ix0 < P.ncx) {
#pragma unroll
                for (int m = 0; m < 2; ++m) {  // coarse rows J, J + 1 from rows (4m, 4m+1), (4m+2, 4m+3)
                  const int J = (gyw >> 1) + 2 * m;
                  if (rint[4 * m] && rin[4 * m] && J < P.ncy) bcp[(long long)J * P.ncx + Ix0] = acc[m].x;
                  if (rint[4 * m + 2] && rin[4 * m + 2] && J + 1 < P.ncy)
                    bcp[(long long)(J + 1) * P.ncx + Ix0] = acc[m].y;
                }
              }
            } else {
              racc[0] = acc[0];
              racc[1] = acc[1];
            }
          }
        }
        {  // stage the interior rows of plane q; stored by TMA after the next barrier
          float* stp = &S.st[nst % SS][0][0];
          if (pin) {
#pragma unroll
            for (int j = 0; j < MR; ++j) {
              if (!rint[j]) continue;
              const int p = (j & 1) + ((j >> 2) << 1);
              const bool hi = (j >> 1) & 1;
              float* srow = stp + (warp * MR + j - HY) * TXI + 2 * lane - HX;
              srow[0] = hi ? Xo.V[p][0].y : Xo.V[p][0].x;
              srow[1] = hi ? Xo.V[p][1].y : Xo.V[p][1].x;
            }
          }
          fence_async_smem();
          ++nst;
          if (q >= p_lo) {
            pend = q;
            pbx = bx0 + HX;
            pby = by0 + HY;
          }
        }
      }
      if (tid == 0) tma_store_wait_read0();  // the store issued this step has read its slot
    };

    const int t0 = a - a % RING;
    for (int T = t0; T < tend; T += RING) {
      static_for<RING>([&](auto KK) {
        const int t = T + decltype(KK)::value;
        if (t >= a && t < tend) step(KK, t);
      });
    }
    while (nbw < nbi) {  // b loads not waited by a step
      mbar_wait(&S.barb[nbw % BS], (nbw / BS) & 1);
      ++nbw;
    }
    __syncthreads();
    flush_store();
    if (tid == 0) tma_store_wait_read0();
    if (TAIL == TAIL_NORMS) {
      block_sum2(sr, sbb);
      if (tid == 0 && P.partials) P.partials[item] = make_double2(sr, sbb);
      sr = sbb = 0.0;
    }
  }
  if (TAIL == TAIL_NORMS && tid == 0 && P.partials)
    for (; seg < P.max_segs; ++seg) P.partials[blockIdx.x * P.max_segs + seg] = make_double2(0.0, 0.0);
  if (tid == 0) tma_store_wait_all();
}

template <int TAIL, bool PRO, bool ZC, bool EV = false>
static cudaError_t launch(const Sweep& P, cudaStream_t s) {
  static_assert(sizeof(Smem<PRO>) + 128 + 512 <= 232448, "shared memory");
  auto kern = k_m3v<TAIL, PRO, ZC, EV>;
  static bool attr = false;
  const size_t sm = sizeof(Smem<PRO>) + 128;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  kern<<<P.nitems / P.max_segs, MT, sm, s>>>(P);
  return cudaGetLastError();
}

}  // namespace mv

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
int vp_make_map(CUtensorMap* m, const float* p, int nx, int ny, long long np, int bw, int bh);  // gdp_vpass3d.cu

static int mv_nsm() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static void mv_plan(const LevelK& L, bool zc, int zlo, int zhi, mv::Sweep& P) {
  P.tiles_x = (L.nx + mv::TXI - 1) / mv::TXI;
  P.tiles_y = (L.ny + mv::TYI - 1) / mv::TYI;
  const int tiles = P.tiles_x * P.tiles_y;
  const int nz = zhi - zlo;
  const int grid = (int)std::min<long long>(mv_nsm(), (long long)tiles * nz);
  P.zlo = zlo;
  P.zhi = zhi;
  P.zeven = zc ? 1 : 0;
  P.full = tiles / grid;
  const long long rem = (long long)(tiles - P.full * grid) * nz;
  P.max_segs = P.full + (int)((rem + grid - 1) / grid / std::max(nz, 1)) + 3;
  P.nitems = grid * P.max_segs;
}

// the vertical-pack z-march serves single-slab levels with nx % 4 == 0 (TMA strides), 16-byte
// aligned arrays, x and y coarsened, z not coarsened when the sweep prolongates
bool sweep3dv_ok(const Level& L, const Level& C, bool prolong, const float* xin, const float* xout, const float* b) {
  if (!C.tx.coarsened || !C.ty.coarsened || (prolong && C.tz.coarsened)) return false;
  if ((L.nx & 3) != 0 || (prolong && (C.nx & 3) != 0)) return false;
  if (!al16(xin) || !al16(xout) || !al16(b) || (prolong && !al16(C.x))) return false;
  if (L.nzl != L.gz.n || L.z0 != 0) return false;
  return (long long)L.nx * L.ny < (1LL << 31) && (long long)C.nx * C.ny < (1LL << 31);
}

int sweep3dv_items(const Level& L, const Level& C) {
  mv::Sweep P{};
  mv_plan(L.K, C.tz.coarsened != 0, 0, L.nzl, P);
  return P.nitems;
}

// one sweep of level L (as fused_sweep3d): tail 0 none, 1 restrict into C.b, 2 norms into
// partials (one per item); *items (may be NULL) = partial slots written
int fused_sweep3dv(const Level& L, const Level& C, const float* xin, float* xout, const float* b, bool zero_x,
                   bool prolong, int tail, double2* partials, cudaStream_t s, int* items) {
  mv::Sweep P{};
  P.L = L.K;
  P.xout = xout;
  P.tx = C.tx; P.ty = C.ty; P.tz = C.tz; P.ncx = C.nx; P.ncy = C.ny;
  P.bc = C.b;
  P.partials = partials;
  P.zero_x = zero_x ? 1 : 0;
  const bool zc = C.tz.coarsened != 0;
  mv_plan(L.K, zc, 0, L.nzl, P);
  int rc;
  if ((rc = vp_make_map(&P.tmx, zero_x ? b : xin, L.nx, L.ny, L.nzl, mv::TX, mv::TY)) != GDP_OK) return rc;
  if ((rc = vp_make_map(&P.tmb, b, L.nx, L.ny, L.nzl, mv::TX, mv::TY)) != GDP_OK) return rc;
  if ((rc = vp_make_map(&P.tmo, xout, L.nx, L.ny, L.nzl, mv::TXI, mv::TYI)) != GDP_OK) return rc;
  if (prolong) {
    if ((rc = vp_make_map(&P.tmc, C.x, C.nx, C.ny, C.nzl, mv::CBX, mv::CBY)) != GDP_OK) return rc;
  } else {
    P.tmc = P.tmb;
  }
  const double N = (double)L.nx * L.ny * L.nzl, Nc = (double)C.nx * C.ny * C.nzl;
  const double bytes = N * ((zero_x ? 4.0 : 8.0) + 4.0) + ((tail == 1 || prolong) ? Nc * 4.0 : 0.0);
  ProfScope ps(tail == 2 || prolong ? KC_UP3D : KC_DOWN3D, bytes, s, N, true);  // the norms sweep ends the up pass
  cudaError_t e;
  using namespace mv;
  if (prolong) {
    if (tail == TAIL_NORMS) e = launch<2, true, false>(P, s);
    else if (tail == TAIL_RESTRICT) e = launch<1, true, false>(P, s);
    else e = launch<0, true, false>(P, s);
  } else if (tail == TAIL_RESTRICT) {
    const bool ev = (L.nx & 1) == 0 && (L.ny & 1) == 0;  // C is x/y coarsened (sweep3dv_ok)
    if (ev) e = zc ? launch<1, false, true, true>(P, s) : launch<1, false, false, true>(P, s);
    else e = zc ? launch<1, false, true>(P, s) : launch<1, false, false>(P, s);
  } else if (tail == TAIL_NORMS) {
    e = launch<2, false, false>(P, s);
  } else {
    e = launch<0, false, false>(P, s);
  }
  if (e != cudaSuccess) return set_err(GDP_ECUDA, "k_m3v launch: %s", cudaGetErrorString(e));
  if (items) *items = P.nitems;
  return GDP_OK;
}

}  // namespace gdp
