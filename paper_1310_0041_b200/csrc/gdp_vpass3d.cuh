// gdp_vpass3d.cuh — temporally blocked 3D level passes (levels with z links: phase 1, Eq. 1), sm_100a.
//
// One HBM pass = one whole multigrid pass of a level: the NU red-black
// Gauss-Seidel sweeps before the restriction, or the prolongated correction plus the NU sweeps
// after it, together with the residual that ends the pass (restricted to the coarse level, or
// reduced to fp64 norms).  This is the paper's "multiple Gauss-Seidel relaxations in a single
// streaming pass" over a sliding window of slices moved on chip.
//
// A persistent CTA owns an in-plane tile (128 x 32 cells, 8 warps of 4 rows, 4 columns per lane)
// and marches along z.  With t the plane whose x is loaded at step t:
//     stage k = 1 .. 2 NU (colour (k-1) & 1, sweep (k+1)/2) updates plane t - k,
//     the tail takes the residual of plane t - (2 NU + 1) and stores its x,
// which is exactly the reference schedule's 2 NU half-sweeps: a point of one colour depends only
// on points of the other colour (colour = (x + y + z_global) & 1), and stage k on plane q sees
// planes q +- 1 in the state stage k-1 left them in.  In-plane the valid region shrinks by one
// cell per stage, so the tile carries a halo of >= 2 NU + 1 cells that is recomputed.
//
// Register layout ("vertical packs"): a thread's 4 x 4 cells of a plane are eight f32x2 packs
// V[h][c] = (x[row h][col c], x[row h + 2][col c]), h = 0, 1: both cells of a pack have the same
// colour, and the x / z neighbours of a pack and its inner y neighbour are packs too, so the
// FFMA2 / FADD2 stencil needs (almost) no register moves.
//
// Data movement per plane step:
//   * x and b planes of the tile arrive by TMA (cp.async.bulk.tensor, OOB zero fill) into
//     shared-memory slots completed on mbarriers: x XS - 1 planes ahead, b one plane ahead of
//     its first use and kept until the tail; the coarse correction's box (up pass) comes with x;
//   * each thread keeps its cells of the 2 NU + 2 newest planes in registers (ring indexed by
//     t mod R, the plane loop unrolled R-fold so every index is static); the tail's lower
//     neighbour (the plane the previous step finished) is a thread-private smem copy;
//   * x-neighbours across lanes by __shfl, y-neighbours across warps from the edge rows the
//     neighbouring warp published the step before (double-buffered by step parity);
//   * one __syncthreads per plane step.
// Per-cell arithmetic is the reference one (apply_from order, gs_update with the correctly
// rounded 1/D, rw3 / bilerp for the transfers), so the iterates are bit-identical to the
// reference schedule (tests/test_gpu_parity.py).
#pragma once
#include <cuda.h>

#include "gdp_internal.h"
#include "gdp_pack.cuh"

namespace gdp {
namespace vp {

constexpr int MW = 8;            // warps per CTA, stacked in y
constexpr int MR = 4;            // rows per warp
constexpr int MT = MW * 32;      // 256 threads
constexpr int TX = 128;          // tile columns (4 per lane)
constexpr int TY = MW * MR;      // 32 tile rows
constexpr int CBX = 72;          // coarse box columns (<= 69 used; a multiple of 4)
constexpr int CBY = 18;          // coarse box rows

template <int NU>
struct Geo {
  static constexpr int NST = 2 * NU + 1;        // stages before the tail; the tail is stage NST
  static constexpr int HX = NU == 1 ? 4 : 8;    // x halo (>= NST, whole lanes)
  static constexpr int HY = NST + (NST & 1);    // y halo (>= NST, even: restriction pairs)
  static constexpr int R = 2 * NU + 2;          // register ring: planes t .. t - NST (even)
  static constexpr int BS = 2 * NU + 2;         // b slots (b of plane p issued at step p, read until p + NST)
  static constexpr int TXI = TX - 2 * HX;       // interior columns
  static constexpr int TYI = TY - 2 * HY;       // interior rows
};

struct alignas(128) CBox { float v[CBY][CBX]; };  // TMA destinations are 128-byte aligned

template <int NU, bool PRO>
struct alignas(128) Smem {
  static constexpr int XS = PRO ? 2 : 3;        // x slots: x of plane p issued at step p - XS + 1
  float xs[XS][TY][TX];                         // staged x planes (TMA box layout)
  float bs[Geo<NU>::BS][TY][TX];                // staged b planes
  CBox cs[PRO ? XS : 1];                        // coarse box of the plane (z not coarsened)
  float2 xlow[8][MT];                           // the tail's lower neighbour plane (thread-private packs)
  float2 ex[2 * NU][2][MW][2][32];              // [consumer stage - 1][parity][warp][row 0 | 3][lane]
  float4 et[2][MW][2][32];                      // rows 0 | 3 after the last stage (4 columns)
  float inv[4][6][4][32];                       // 1/D per [plane class][row class][column][lane]
  unsigned long long barx[XS];
  unsigned long long barb[Geo<NU>::BS];
};

struct Pass {
  CUtensorMap tmx, tmb, tmc;                    // x in, b, coarse x (fp32 3D maps)
  LevelK L;
  float* xout;
  XferAxis tx, ty, tz;
  int ncx, ncy;
  float* bc;                                    // TAIL_RESTRICT: coarse rhs
  double2* partials;                            // TAIL_NORMS: (sum r^2, sum b^2) per item
  int zero_x;
  int tiles_x, tiles_y;
  int zlo, zhi;
  int full, zeven, max_segs, nitems;
};

enum { TAIL_NONE = 0, TAIL_RESTRICT = 1, TAIL_NORMS = 2 };

// ---------------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
// box at (c0, c1, c2) of a 3D map; c0 * 4 must be a multiple of 16 bytes (measured on the B200:
// an unaligned innermost coordinate traps with an illegal instruction, tools/tma_probe)
#ifndef GDP_TMA_HINT
#define GDP_TMA_HINT 0
#endif
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, unsigned long long* bar) {
#if GDP_TMA_HINT
  // L2 evict_last: a box's halo columns / rows are the neighbouring tiles' interior a few steps apart
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(
          sa(dst)),
      "l"(reinterpret_cast<unsigned long long>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(sa(bar)), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          sa(dst)),
      "l"(reinterpret_cast<unsigned long long>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(sa(bar))
      : "memory");
#endif
}

// row / plane classes of the diagonal: the link coefficients of a row depend only on these
__device__ __forceinline__ int row_class(int g, int n) {
  return g < 0 ? 4 : (g >= n ? 5 : (g == 0 ? 1 : (g == n - 1 ? 3 : (g == n - 2 ? 2 : 0))));
}
__device__ __forceinline__ int row_rep(int c, int n) {  // an index of class c (class 0 only exists for n >= 4)
  return c == 0 ? 1 : (c == 1 ? 0 : (c == 2 ? n - 2 : (c == 3 ? n - 1 : (c == 4 ? -1 : n))));
}

// Rare paths, out of line (they would otherwise bloat the unrolled plane loop past the
// instruction cache): the prolongation at faces / partial cells, the restriction weights of
// partial cells.
static __device__ __noinline__ void prolong_general(const float* box, XferAxis tx, XferAxis ty, int gx0, int gyw, int lx,
                                             int ly, float* e /* [2][4] packs as 16 floats */) {
  const int Ix0 = gx0 >> 1;
  for (int j = 0; j < 4; ++j) {
    long long Iy, Jy;
    float tyw;
    ptaps(ty, gyw + j, Iy, Jy, tyw);
    const int ri = ly + (int)(Iy - ((gyw >> 1) - 1)), rj = ly + (int)(Jy - ((gyw >> 1) - 1));
    for (int c = 0; c < 4; ++c) {
      long long Ix, Jx;
      float txw;
      ptaps(tx, gx0 + c, Ix, Jx, txw);
      const int ci = lx + (int)(Ix - (Ix0 - 1)), cj = lx + (int)(Jx - (Ix0 - 1));
      const float v = bilerp(box[ri * CBX + ci], box[ri * CBX + cj], box[rj * CBX + ci], box[rj * CBX + cj], txw, tyw);
      e[((j & 1) * 4 + c) * 2 + (j >> 1)] = v;  // pack (h = j & 1, c), component j >> 1
    }
  }
}
static __device__ __noinline__ float2 rw_pair(XferAxis tx, XferAxis ty, int gx, int gy, float wz) {
  const float wx = rweight(tx, gx);
  return make_float2(rw3(wz, rweight(ty, gy), wx), rw3(wz, rweight(ty, gy + 2), wx));
}

struct Pk { float2 V[2][4]; };  // V[h][c] = (x[row h][col c], x[row h + 2][col c])
struct Pk1 { float2 v; };       // one pack

template <int NU, int TAIL, bool PROLONG, bool ZC>
__global__ void __launch_bounds__(MT, 1) k_vpass3d(const __grid_constant__ Pass P) {
  using GG = Geo<NU>;
  constexpr int NST = GG::NST, HX = GG::HX, HY = GG::HY, R = GG::R, BS = GG::BS, TXI = GG::TXI, TYI = GG::TYI;
  using SM = Smem<NU, PROLONG>;
  constexpr int XS = SM::XS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 128-byte aligned view, by pointer arithmetic on the shared array (keeps the address space)
  SM& S = *reinterpret_cast<SM*>(smem_raw + ((128u - (sa(smem_raw) & 127u)) & 127u));
  const LevelK& L = P.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = L.nx;
  const long long plane = (long long)L.nx * L.ny;
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
  for (int i = 0; i < 8; ++i) S.xlow[i][tid] = f2(0.f);  // never NaN (0 * x at faces)

  Pk X[R];
#pragma unroll
  for (int k = 0; k < R; ++k)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < 4; ++c) X[k].V[h][c] = f2(0.f);

  double sr = 0.0, sbb = 0.0;
  // TMA issue / wait counters (uniform): load n of a buffer goes to slot n % slots, phase (n / slots) & 1
  unsigned nxi = 0, nxw = 0, nbi = 0;

  const int ntiles = P.tiles_x * P.tiles_y, nzr = P.zhi - P.zlo, G = gridDim.x;
  const int cid = blockIdx.x;
  const long long wr = (long long)(ntiles - P.full * G) * nzr;  // remaining tile-planes
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
    const int tx_ = tile % P.tiles_x;
    const int ty_ = tile / P.tiles_x;
    const int bx0 = tx_ * TXI - HX;                  // box origin (may be negative: OOB zero fill)
    const int by0 = ty_ * TYI - HY;

    // ---- column data of my lane (4 consecutive columns)
    const int gx0 = bx0 + 4 * lane;
    bool cin[4];
    float2 kxl[4], kxr[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      cin[c] = gx0 + c >= 0 && gx0 + c < nx;
      kxl[c] = f2(cl(L.ax, gx0 + c));
      kxr[c] = f2(cr(L.ax, gx0 + c));
    }
    const bool lane_full = cin[0] && cin[1] && cin[2] && cin[3];
    const bool lane_any = cin[0] || cin[1] || cin[2] || cin[3];
    const bool pin = lane >= HX / 4 && lane < 32 - HX / 4;  // interior columns (whole lanes)

    // ---- row data of my rows (rows h and h + 2 form the packs V[h][.])
    const int gyw = by0 + warp * MR;  // even
    float2 kyl[2], kyr[2];
    int ivo[MR];
    bool rin[MR], rint[MR];
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int gy = gyw + j;
      rin[j] = gy >= 0 && gy < L.ny;
      rint[j] = warp * MR + j >= HY && warp * MR + j < TY - HY;
      ivo[j] = row_class(gy, L.ay.n) * 4 * 32 + lane;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      kyl[h] = make_float2(cl(L.ay, gyw + h), cl(L.ay, gyw + h + 2));
      kyr[h] = make_float2(cr(L.ay, gyw + h), cr(L.ay, gyw + h + 2));
    }
    // restriction weights of my children: 1/2 for two equal children (rweight divides: only the
    // lanes / warps at a partial last cell take it)
    const bool rwreg = TAIL == TAIL_RESTRICT && rweight(P.tx, gx0) == 0.5f && rweight(P.tx, gx0 + 1) == 0.5f &&
                       rweight(P.tx, gx0 + 2) == 0.5f && rweight(P.tx, gx0 + 3) == 0.5f &&
                       rweight(P.ty, gyw) == 0.5f && rweight(P.ty, gyw + 1) == 0.5f &&
                       rweight(P.ty, gyw + 2) == 0.5f && rweight(P.ty, gyw + 3) == 0.5f;
    const bool wany = rint[0] || rint[1] || rint[2] || rint[3];  // warp-uniform
    const bool rfull = rin[0] && rin[1] && rin[2] && rin[3];

    // ---- 1/D table of this tile's columns (the previous item may still read the old one)
    __syncthreads();
    for (int i = tid; i < 4 * 6 * 4 * 32; i += MT) {
      const int ln = i & 31, c = (i >> 5) & 3, rc = (i >> 7) % 6, zc = (i >> 7) / 6;
      const int ry = row_rep(rc, L.ay.n);
      const int zr = zc == 0 ? 1 : (zc == 1 ? 0 : (zc == 2 ? nzg - 2 : nzg - 1));
      const int gx = bx0 + 4 * ln + c;
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
      zoff = (first ? 1 : (last ? 3 : (penult ? 2 : 0))) * (6 * 4 * 32);
    };

    // ---- prolongation taps: regular (1/4, 3/4 from the neighbouring coarse cells) away from the
    // faces and partial cells; elsewhere recomputed by ptaps in the general path
    bool xregl = true, yregw = true;
    const int cbx0 = ((bx0 >> 1) - 1) & ~3, cby0 = (by0 >> 1) - 1;  // coarse box origin (x 16-byte aligned)
    const int Ix0 = gx0 >> 1;
    const int lx = Ix0 - 1 - cbx0;           // local column of coarse column Ix0 - 1
    const int ly = ((gyw >> 1) - 1) - cby0;  // local row of coarse row gyw/2 - 1 (= 2 warp)
    if (PROLONG) {
      auto reg4 = [](const XferAxis& ax, int i0) {  // the taps ptaps gives for the regular pattern
        bool ok = true;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          long long I, J;
          float t;
          ptaps(ax, i0 + c, I, J, t);
          ok = ok && t == 0.25f && I == ((i0 + c) >> 1) && J == ((c & 1) ? I + 1 : I - 1);
        }
        return ok;
      };
      xregl = reg4(P.tx, gx0);
      yregw = reg4(P.ty, gyw);
    }
    // coarse correction packs e[h][c] from a staged coarse box (the bilerp order of k_prolong_rows)
    auto prolong_packs = [&](const CBox& box, float2 (&e)[2][4]) {
      if (xregl && yregw) {
        // coarse rows q = 0..3 (ly + q), columns k = 0..3 (lx + k); regular taps 1/4, 3/4:
        // col c0: (I k1, J k0), c1: (k1, k2), c2: (k2, k1), c3: (k2, k3); rows the same pattern
        float2 v0[4], v1[4], v2[4];  // (row q, row q + 1) values per coarse column k, q = 0, 1, 2
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float a0 = box.v[ly][lx + k], a1 = box.v[ly + 1][lx + k], a2 = box.v[ly + 2][lx + k],
                      a3 = box.v[ly + 3][lx + k];
          v0[k] = make_float2(a0, a1);
          v1[k] = make_float2(a1, a2);
          v2[k] = make_float2(a2, a3);
        }
        constexpr int KI[4] = {1, 1, 2, 2}, KJ[4] = {0, 2, 1, 3};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          // x-interpolated pairs of coarse rows (0,1), (1,2), (2,3) at fine column c
          const float2 p01 = __ffma2_rn(f2(0.25f), v0[KJ[c]], __fmul2_rn(f2(0.75f), v0[KI[c]]));
          const float2 p12 = __ffma2_rn(f2(0.25f), v1[KJ[c]], __fmul2_rn(f2(0.75f), v1[KI[c]]));
          const float2 p23 = __ffma2_rn(f2(0.25f), v2[KJ[c]], __fmul2_rn(f2(0.75f), v2[KI[c]]));
          // rows 0 / 2: (I q1, J q0) / (I q2, J q1) -> pair I = p12, J = p01
          e[0][c] = __ffma2_rn(f2(0.25f), p01, __fmul2_rn(f2(0.75f), p12));
          // rows 1 / 3: (I q1, J q2) / (I q2, J q3) -> pair I = p12, J = p23
          e[1][c] = __ffma2_rn(f2(0.25f), p23, __fmul2_rn(f2(0.75f), p12));
        }
      } else {  // faces and partial cells: general taps (out of line)
        float ev[16];
        prolong_general(&box.v[0][0], P.tx, P.ty, gx0, gyw, lx, ly, ev);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 4; ++c) e[h][c] = make_float2(ev[(h * 4 + c) * 2], ev[(h * 4 + c) * 2 + 1]);
      }
    };

    // ---- plane ranges of this item
    const int a = max(p_lo - NST, 0), e = min(p_hi + NST, nzg);
    const int tend = p_hi + NST;
    const unsigned nb0 = nbi;  // b of plane p lives in slot (nb0 + p - a) % BS
    auto issue_x = [&](int p) {
      const unsigned s = nxi % XS;
      if (tid == 0) {
        unsigned bytes = P.zero_x ? 0u : (unsigned)(TX * TY * 4);
        if (PROLONG) bytes += (unsigned)(CBX * CBY * 4);
        if (bytes) {
          mbar_expect(&S.barx[s], bytes);
          if (!P.zero_x) tma3(&S.xs[s][0][0], &P.tmx, bx0, by0, p, &S.barx[s]);
          if (PROLONG) tma3(&S.cs[s].v[0][0], &P.tmc, cbx0, cby0, p, &S.barx[s]);  // coarse plane p (z kept)
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
    __syncthreads();  // the 1/D table is written; slots are free (all earlier loads were waited)
    for (int k = 0; k < XS - 1; ++k)
      if (a + k < e) issue_x(a + k);
    unsigned nbw = nb0;  // next b load to wait for

    float2 racc[2] = {f2(0.f), f2(0.f)};  // ZC restriction: (coarse row J, J + 1) for columns Ix0, Ix0 + 1

    // (A x) of pack (H, C) of plane Xo (Xd below, Xu above); sv / nv: the cell below row 0 / above
    // row 3 in this column (used by h = 0 / h = 1); apply_from order
    auto stencil = [&](auto Hc, auto Cc, const Pk& Xo, const auto& Xd, const Pk& Xu, float sv, float nv,
                       float2 zl2, float2 zr2, auto D1) -> float2 {
      constexpr int H = decltype(Hc)::value, C = decltype(Cc)::value;
      float2 xd;
      if constexpr (decltype(D1)::value) xd = Xd.v;  // the tail: a single pack of the lower plane
      else xd = Xd.V[H][C];
      const float2 Xc = Xo.V[H][C];
      float2 W, E;
      if constexpr (C > 0) W = Xo.V[H][C - 1];
      else W = make_float2(__shfl_up_sync(FULL, Xo.V[H][3].x, 1), __shfl_up_sync(FULL, Xo.V[H][3].y, 1));
      if constexpr (C < 3) E = Xo.V[H][C + 1];
      else E = make_float2(__shfl_down_sync(FULL, Xo.V[H][0].x, 1), __shfl_down_sync(FULL, Xo.V[H][0].y, 1));
      const float2 Sn = H == 0 ? make_float2(sv, Xo.V[1][C].x) : Xo.V[0][C];
      const float2 Nn = H == 0 ? Xo.V[1][C] : make_float2(Xo.V[0][C].y, nv);
      float2 s = __fmul2_rn(al2, Xc);
      s = __ffma2_rn(kxl[C], sub2(Xc, W), s);
      s = __ffma2_rn(kxr[C], sub2(Xc, E), s);
      s = __ffma2_rn(kyl[H], sub2(Xc, Sn), s);
      s = __ffma2_rn(kyr[H], sub2(Xc, Nn), s);
      s = __ffma2_rn(zl2, sub2(Xc, xd), s);
      return __ffma2_rn(zr2, sub2(Xc, Xu.V[H][C]), s);
    };

    // ---- one plane step: K = t mod R is static
    auto step = [&](auto KK, int t) {
      constexpr int PAR = decltype(KK)::value;  // parity of the step (and of z)
      // the ring is a shift register: X[k] holds plane t - k (the plane loop is unrolled twice
      // only, for the static parity; the shift is register moves)
#pragma unroll
      for (int k = R - 1; k > 0; --k) X[k] = X[k - 1];
      __syncthreads();
      // (0) TMA of later planes (the slots' previous planes are done: barrier above); b of plane
      // t - 1 is waited for before stage 1 reads it
      if (t + XS - 1 < e) issue_x(t + XS - 1);
      if (t < e) issue_b(t);
      if (t - 1 >= a && t - 1 < e) {
        mbar_wait(&S.barb[nbw % BS], (nbw / BS) & 1);
        ++nbw;
      }

      // (1) load plane t into X[K], add the coarse correction, publish its edge rows
      if (t < e) {
        const unsigned s = nxw % XS;
        const unsigned ph = (nxw / XS) & 1;
        ++nxw;
        if (xbytes) mbar_wait(&S.barx[s], ph);
        Pk& Xt = X[0];
        if (P.zero_x) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 4; ++c) Xt.V[h][c] = f2(0.f);
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              Xt.V[h][c] = make_float2(S.xs[s][warp * MR + h][4 * lane + c], S.xs[s][warp * MR + h + 2][4 * lane + c]);
        }
        if constexpr (PROLONG) {
          float2 ec[2][4];
          prolong_packs(S.cs[s], ec);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 4; ++c) Xt.V[h][c] = __fadd2_rn(Xt.V[h][c], ec[h][c]);
        }
        // stage 1 (colour 0) of the warps above / below needs my colour-1 cells of rows 0 / 3:
        // row 0 at columns c with (c + t) odd, row 3 at columns c with (c + 3 + t) odd
        constexpr int P0 = (PAR + 1) & 1;
        constexpr int P3 = PAR & 1;
        S.ex[0][PAR][warp][0][lane] = make_float2(Xt.V[0][P0].x, Xt.V[0][P0 + 2].x);
        S.ex[0][PAR][warp][1][lane] = make_float2(Xt.V[1][P3].y, Xt.V[1][P3 + 2].y);
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 4; ++c) X[0].V[h][c] = f2(0.f);
      }

      // (2) half-sweep k (colour (k-1) & 1) on plane q = t - k, held in X[KO]
      auto stage = [&](auto KSc, int q) {
        constexpr int KS = decltype(KSc)::value;  // 1 .. 2 NU
        constexpr int C = (KS - 1) & 1;
        constexpr int KO = KS, KD = KS + 1, KU = KS - 1;
        constexpr int ZP = (PAR + KS) & 1;        // parity of the plane's z
        constexpr int PA = (C + ZP) & 1;          // active columns: h = 0 at PA, PA + 2; h = 1 at 1 - PA, 3 - PA
        float2 zl2, zr2;
        int zoff;
        zcoef(q, zl2, zr2, zoff);
        Pk& Xo = X[KO];
        // row -1 (the warp below's row 3) at columns PA, PA + 2; row 4 (the warp above's row 0) at
        // columns 1 - PA, 3 - PA
        const float2 sv = S.ex[KS - 1][PAR ^ 1][wdn][1][lane];
        const float2 nv = S.ex[KS - 1][PAR ^ 1][wup][0][lane];
        const unsigned bsl = (nb0 + (unsigned)(q - a)) % BS;
        const float* brow = &S.bs[bsl][warp * MR][4 * lane];
        static_for<4>([&](auto Ic) {
          constexpr int i = decltype(Ic)::value;
          constexpr int H = i >> 1;
          constexpr int CC = (H == 0 ? PA : 1 - PA) + 2 * (i & 1);
          const float2 bv = make_float2(brow[H * TX + CC], brow[(H + 2) * TX + CC]);
          const float2 iD = make_float2(invf[zoff + ivo[H] + CC * 32], invf[zoff + ivo[H + 2] + CC * 32]);
          const float s1 = (i & 1) ? sv.y : sv.x, n1 = (i & 1) ? nv.y : nv.x;
          const float2 s = stencil(IC<H>{}, IC<CC>{}, Xo, X[KD], X[KU], s1, n1, zl2, zr2, IC<0>{});
          Xo.V[H][CC] = __ffma2_rn(sub2(bv, s), iD, Xo.V[H][CC]);
        });
        if constexpr (KS < 2 * NU) {  // the cells the next stage (other colour) needs from my edge rows
          // consumer colour 1 - C: its h = 0 cells at columns PN, PN + 2 need my row 3 there; its
          // h = 1 cells at 1 - PN, 3 - PN need my row 0 there
          constexpr int PN = (1 - C + ZP) & 1;
          S.ex[KS][PAR][warp][0][lane] = make_float2(Xo.V[0][1 - PN].x, Xo.V[0][3 - PN].x);
          S.ex[KS][PAR][warp][1][lane] = make_float2(Xo.V[1][PN].y, Xo.V[1][PN + 2].y);
        } else {  // the tail needs all four columns of rows 0 and 3
          S.et[PAR][warp][0][lane] = make_float4(Xo.V[0][0].x, Xo.V[0][1].x, Xo.V[0][2].x, Xo.V[0][3].x);
          S.et[PAR][warp][1][lane] = make_float4(Xo.V[1][0].y, Xo.V[1][1].y, Xo.V[1][2].y, Xo.V[1][3].y);
        }
      };
      static_for<2 * NU>([&](auto Ic) {
        constexpr int KS = decltype(Ic)::value + 1;
        const int q = t - KS;
        if (q >= max(p_lo - (NST - KS), 0) && q < min(p_hi + (NST - KS), nzg)) stage(IC<KS>{}, q);
      });

      // (3) tail on plane q = t - NST: residual -> restriction / norms, store x
      const int q = t - NST;
      if (q >= p_lo - 1 && q >= 0 && q < p_hi) {
        constexpr int KO = NST, KU = NST - 1;
        constexpr int ZP = (PAR + NST) & 1;
        const Pk& Xo = X[KO];
        if (q >= p_lo && TAIL != TAIL_NONE && wany) {  // warp-uniform: the stencil shuffles need every lane
          float2 zl2, zr2;
          int zoff;
          zcoef(q, zl2, zr2, zoff);
          const float4 tsv = S.et[PAR ^ 1][wdn][1][lane];  // row -1, columns 0..3
          const float4 tnv = S.et[PAR ^ 1][wup][0][lane];  // row 4
          const float sva[4] = {tsv.x, tsv.y, tsv.z, tsv.w}, nva[4] = {tnv.x, tnv.y, tnv.z, tnv.w};
          const unsigned bsl = (nb0 + (unsigned)(q - a)) % BS;
          const float* brow = &S.bs[bsl][warp * MR][4 * lane];
          // restriction (volume-weighted child average, k_restrict order fz outer, fy, fx inner):
          // coarse cells (J, J + 1) x column Ix0 + ip accumulate packs (h = 0: rows 0, 2; then h = 1:
          // rows 1, 3) of columns 2 ip, 2 ip + 1 -- exactly the order the packs are visited here
          const float wz = ZC ? rweight(P.tz, q) : 1.f;
          const bool first = !ZC || ZP == 0;
          float2 acc[2] = {first ? f2(0.f) : racc[0], first ? f2(0.f) : racc[1]};
          const bool rst = TAIL == TAIL_RESTRICT && pin && (rint[0] || rint[2]);  // rows (0, 1) / (2, 3) interior
          static_for<8>([&](auto Ic) {
            constexpr int i = decltype(Ic)::value;
            constexpr int H = i >> 2, CC = i & 3;
            const float2 xl = S.xlow[H * 4 + CC][tid];
            const float2 bb = make_float2(brow[H * TX + CC], brow[(H + 2) * TX + CC]);
            const float2 r = sub2(bb, stencil(IC<H>{}, IC<CC>{}, Xo, Pk1{xl}, X[KU], sva[CC], nva[CC], zl2, zr2, IC<1>{}));
            if (TAIL == TAIL_RESTRICT) {
              if (rst) {
                const float2 w = rwreg ? f2(rw3(wz, 0.5f, 0.5f)) : rw_pair(P.tx, P.ty, gx0 + CC, gyw + H, wz);
                const float2 n = __ffma2_rn(w, r, acc[CC >> 1]);
                if (lane_full && rfull) acc[CC >> 1] = n;
                else acc[CC >> 1] = make_float2(cin[CC] && rin[H] ? n.x : acc[CC >> 1].x,
                                                cin[CC] && rin[H + 2] ? n.y : acc[CC >> 1].y);
              }
            } else if (TAIL == TAIL_NORMS) {
              if (pin && cin[CC]) {
                if (rint[H] && rin[H]) {
                  sr += (double)r.x * (double)r.x;
                  sbb += (double)bb.x * (double)bb.x;
                }
                if (rint[H + 2] && rin[H + 2]) {
                  sr += (double)r.y * (double)r.y;
                  sbb += (double)bb.y * (double)bb.y;
                }
              }
            }
          });
          if (TAIL == TAIL_RESTRICT && rst) {
            const bool last = !ZC || ZP == 1 || q == nzg - 1;
            float* bcp = P.bc + (long long)(ZC ? (q >> 1) : q) * cplane;
            const int J = gyw >> 1;
#pragma unroll
            for (int ip = 0; ip < 2; ++ip) {
              if (last) {
                const int I = Ix0 + ip;
                if (cin[2 * ip] && I < P.ncx) {
                  if (rint[0] && rin[0] && J < P.ncy) bcp[(long long)J * P.ncx + I] = acc[ip].x;
                  if (rint[2] && rin[2] && J + 1 < P.ncy) bcp[(long long)(J + 1) * P.ncx + I] = acc[ip].y;
                }
              } else {
                racc[ip] = acc[ip];
              }
            }
          }
        }
        // keep plane q (final) as the next tail's lower neighbour
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 4; ++c) S.xlow[h * 4 + c][tid] = Xo.V[h][c];
        if (q >= p_lo) {
          if (wany && pin && lane_any) {  // store the interior rows of plane q
            float* o = P.xout + (long long)q * plane;
#pragma unroll
            for (int j = 0; j < MR; ++j) {
              if (!rint[j] || !rin[j]) continue;
              const int h = j & 1;
              float v[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) v[c] = j < 2 ? Xo.V[h][c].x : Xo.V[h][c].y;
              float* orow = o + (long long)(gyw + j) * nx + gx0;
              if (lane_full) *reinterpret_cast<float4*>(orow) = make_float4(v[0], v[1], v[2], v[3]);
              else {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                  if (cin[c]) orow[c] = v[c];
              }
            }
          }
        }  // q >= p_lo
      }
    };

    const int t0 = a & ~1;
    for (int T = t0; T < tend; T += 2) {
      static_for<2>([&](auto KK) {
        const int t = T + decltype(KK)::value;
        if (t >= a && t < tend) step(KK, t);
      });
    }
    // b loads not waited by a step (the last plane when the item ends at e = tend)
    while (nbw < nbi) {
      mbar_wait(&S.barb[nbw % BS], (nbw / BS) & 1);
      ++nbw;
    }
    if (TAIL == TAIL_NORMS) {
      block_sum2(sr, sbb);
      if (tid == 0 && P.partials) P.partials[item] = make_double2(sr, sbb);
      sr = sbb = 0.0;
    }
  }
  if (TAIL == TAIL_NORMS && tid == 0 && P.partials)
    for (; seg < P.max_segs; ++seg) P.partials[blockIdx.x * P.max_segs + seg] = make_double2(0.0, 0.0);
}

template <int NU, bool PRO>
inline size_t smem_bytes() { return sizeof(Smem<NU, PRO>) + 128; }

template <int NU, int TAIL, bool PRO, bool ZC>
cudaError_t launch_vp(const Pass& P, cudaStream_t s) {
  static_assert(sizeof(Smem<NU, PRO>) + 128 + 512 <= 232448, "shared memory of the pass kernel");
  auto kern = k_vpass3d<NU, TAIL, PRO, ZC>;
  static bool attr = false;
  const size_t sm = smem_bytes<NU, PRO>();
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  kern<<<P.nitems / P.max_segs, MT, sm, s>>>(P);
  return cudaGetLastError();
}

#define GDP_VP_EXTERN(NU, T, PR, Z) extern template cudaError_t launch_vp<NU, T, PR, Z>(const Pass&, cudaStream_t);
#define GDP_VP_INST(NU, T, PR, Z) template cudaError_t launch_vp<NU, T, PR, Z>(const Pass&, cudaStream_t);
#define GDP_VP_VARIANTS(X) \
  X(1, 1, false, false) X(1, 1, false, true) X(1, 1, true, false) \
  X(2, 1, false, false) X(2, 1, false, true) X(2, 1, true, false) \
  X(1, 2, true, false) X(1, 0, true, false) X(2, 2, true, false) X(2, 0, true, false) \
  X(1, 0, false, false) X(1, 2, false, false)

}  // namespace vp
}  // namespace gdp
