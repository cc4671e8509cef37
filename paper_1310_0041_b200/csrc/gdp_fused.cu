// gdp_fused.cu — fused level passes of the V-cycle, sm_100a.
//
// One HBM pass per level and direction instead of one per half-sweep:
//   down pass: load x + rhs tile, nu red-black Gauss-Seidel sweeps in registers,
//              residual, volume-weighted restriction -> coarse rhs, store x;
//   up pass:   load x + rhs tile, add the prolongated coarse correction, nu sweeps,
//              residual norms (fp64 partials of the final iterate), store x.
// Temporal blocking (the paper's "multiple relaxation passes" in one streaming pass,
// PAPER.md:243-251) uses overlapped tiles: a tile carries a halo of H >= 2 nu + 1 cells
// recomputed redundantly so that its interior is exact.  Because neighbouring tiles read
// each other's interior as halo, a pass reads x from one buffer and writes another
// (down: A -> B, up: B -> A per level).
//
// 2D passes (levels without z links: every phase-2 level, W = pi):
//   CTA = 8 warps stacked in y; a warp owns 64 columns (2 per lane) x 16 rows in registers.
//   x-neighbours come from the adjacent lane (__shfl), y-neighbours from the thread's own
//   registers; only the warp's first/last rows go through shared memory, once per
//   half-sweep.  Tiles away from the domain faces take a fast path with constant
//   coefficients and vector loads; edge tiles take the general path.  Both paths call the
//   arithmetic of gdp_device.cuh in the same order as the reference schedule, so the
//   iterates are bit-identical to it (tests/test_gpu_parity.py).
#include "gdp_internal.h"
#include "gdp_pack.cuh"

namespace gdp {

constexpr int G_R = 12;                   // rows per warp
constexpr int G_W = 8;                    // warps per CTA (stacked in y)
constexpr int G_COLS = 128;               // columns per warp (4 per lane)
constexpr int G_ROWS = G_R * G_W;         // 96


struct Pass2D {
  LevelK L;
  const float* xin;     // x before the pass (ignored if zero_x)
  float* xout;          // x after the pass
  RhsK R;
  int zero_x;           // coarse-level down pass: x starts at 0
  int fast_ok;          // both in-plane axes coarsened (regular transfers away from faces)
  XferAxis tx, ty;      // fine -> coarse (z is never coarsened by a 2D pass)
  int ncx, ncy;
  float* bc;            // down: coarse rhs
  const float* xc;      // up: coarse correction
  double2* partials;    // up: per (plane, tile) sums of r^2 and b^2 (may be null)
};

__device__ __forceinline__ bool col_interior(const AxisC& a, int i) { return i >= 1 && i <= a.n - 3; }


// (A x) on a pack of two cells with regular coefficients (order of apply_from without z terms)
__device__ __forceinline__ float2 apply2(float2 kx, float2 ky, float2 al, float2 X, float2 W, float2 E,
                                         float2 S, float2 N) {
  float2 s = __fmul2_rn(al, X);
  s = __ffma2_rn(kx, sub2(X, W), s);
  s = __ffma2_rn(kx, sub2(X, E), s);
  s = __ffma2_rn(ky, sub2(X, S), s);
  s = __ffma2_rn(ky, sub2(X, N), s);
  return s;
}

// rhs_from() on a pack with regular coefficients
__device__ __forceinline__ float2 rhs2(float2 kx, float2 ky, float2 I, float2 W, float2 E, float2 S,
                                       float2 N, float2 V, float2 av) {
  float2 g = __fmul2_rn(kx, sub2(I, W));
  g = __ffma2_rn(kx, sub2(I, E), g);
  g = __ffma2_rn(ky, sub2(I, S), g);
  g = __ffma2_rn(ky, sub2(I, N), g);
  return __ffma2_rn(av, V, g);
}

// (A x)_c without z links, scalar (general path): the terms apply_from() adds for zl = zr = 0
// are exact zeros
__device__ __forceinline__ float apply2d(const Coef& k, float alpha, float xc, float xw, float xe,
                                         float xs, float xn) {
  float s = __fmul_rn(alpha, xc);
  s = __fmaf_rn(k.xl, xc - xw, s);
  s = __fmaf_rn(k.xr, xc - xe, s);
  s = __fmaf_rn(k.yl, xc - xs, s);
  s = __fmaf_rn(k.yr, xc - xn, s);
  return s;
}

__device__ __forceinline__ float2 bilerp2(float2 a, float2 b, float2 c, float2 d) {
  // bilerp(a, b, c, d, 0.25, 0.25) on a pack
  const float2 t = f2(0.25f), u = f2(1.f - 0.25f);
  const float2 r0 = __ffma2_rn(t, b, __fmul2_rn(u, a));
  const float2 r1 = __ffma2_rn(t, d, __fmul2_rn(u, c));
  return __ffma2_rn(t, r1, __fmul2_rn(u, r0));
}

// u8 pair -> exact fp32 values, then decode_u8() on both (packed)
__device__ __forceinline__ float2 decode2(unsigned int lo, unsigned int hi) {
  const float2 f = __fadd2_rn(make_float2(__uint_as_float(0x4B000000u | lo), __uint_as_float(0x4B000000u | hi)),
                              f2(-8388608.0f));
  const float2 r = f2(1.0f / 255.0f);
  const float2 q = __fmul2_rn(f, r);
  const float2 e = __ffma2_rn(make_float2(-q.x, -q.y), f2(255.0f), f);
  return __ffma2_rn(e, r, q);
}

// element c (0..3) of a lane's row stored as packs A = (c0, c2), B = (c1, c3)
template <int C>
__device__ __forceinline__ float& el(float2& A, float2& B) {
  if constexpr (C == 0) return A.x;
  else if constexpr (C == 1) return B.x;
  else if constexpr (C == 2) return A.y;
  else return B.y;
}

// load 4 consecutive values (c0..c3) of a row as packs (A, B); 8-byte aligned base
__device__ __forceinline__ void ld4f(const float* p, float2& A, float2& B) {
  const float2 lo = __ldg(reinterpret_cast<const float2*>(p));
  const float2 hi = __ldg(reinterpret_cast<const float2*>(p) + 1);
  A = make_float2(lo.x, hi.x);
  B = make_float2(lo.y, hi.y);
}

template <typename TI> struct Row4;
template <> struct Row4<float> {
  __device__ static __forceinline__ void ld(const void* p, long long i, float2& A, float2& B) {
    ld4f(static_cast<const float*>(p) + i, A, B);
  }
};
template <> struct Row4<uint8_t> {
  __device__ static __forceinline__ void ld(const void* p, long long i, float2& A, float2& B) {
    const unsigned short* u = reinterpret_cast<const unsigned short*>(static_cast<const uint8_t*>(p) + i);
    const unsigned int lo = __ldg(u), hi = __ldg(u + 1);
    A = decode2(lo & 0xffu, hi & 0xffu);
    B = decode2(lo >> 8, hi >> 8);
  }
};

// Row data of one warp row (warp-uniform): link coefficients of the row's y links, whether the
// row is inside the domain, and which 1/D case applies.
struct RowInfo { float yl, yr; int in, dcase; };


// halo of the 2D pass: >= 2 nu + 1; a multiple of 4 in x (16-byte aligned lane quads), even in y
__host__ __device__ constexpr int halo2x(int nu) { return ((2 * nu + 1) + 3) & ~3; }
__host__ __device__ constexpr int halo2y(int nu) { return ((2 * nu + 1) + 1) & ~1; }

template <int NU, bool DOWN>
__device__ __forceinline__ void pass2d_body(const Pass2D& P, float4 (&sh_top)[2][G_W][32],
                                            float4 (&sh_bot)[2][G_W][32], float4 (&sb)[G_W][G_R][32],
                                            RowInfo (&srow)[G_W][G_R + 2], float2 (&sinv)[G_W][4][2][32],
                                            int tile_x, int tile_y, int tiles_x, int tiles_y) {
  constexpr int HX = halo2x(NU), HY = halo2y(NU);
  constexpr int TXI = G_COLS - 2 * HX, TYI = G_ROWS - 2 * HY;
  const LevelK& L = P.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx0 = tile_x * TXI - HX + 4 * lane;    // my first column (multiple of 4)
  const int gyw = tile_y * TYI - HY + warp * G_R;  // my first row (even)
  const int iz = blockIdx.z;
  const long long zg = L.z0 + iz;
  const long long nx = L.nx;
  const long long pbase = (long long)iz * L.nx * L.ny;
  const float alpha = L.alpha;
  const float2 al2 = f2(alpha);

  // ---- per-lane column data, packs A = (c0, c2), B = (c1, c3)
  bool cin[4];
  float cxl[4], cxr[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int gx = gx0 + c;
    cin[c] = gx >= 0 && gx < L.nx;
    cxl[c] = cl(L.ax, gx);
    cxr[c] = cr(L.ax, gx);
  }
  const float2 kxlA = make_float2(cxl[0], cxl[2]), kxrA = make_float2(cxr[0], cxr[2]);
  const float2 kxlB = make_float2(cxl[1], cxl[3]), kxrB = make_float2(cxr[1], cxr[3]);
  const bool lane_full = cin[0] && cin[1] && cin[2] && cin[3];
  const bool vec = (L.nx & 3) == 0 && al16(P.xin) && al16(P.xout) && al16(P.R.b);  // rows start 16-byte aligned

  // ---------------------------------------------------------------- issue all loads
  float4(&bs)[G_R][32] = sb[warp];
  float2 A[G_R], B[G_R];  // x of my 12 rows x 4 columns
#pragma unroll
  for (int j = 0; j < G_R; ++j) {
    const int gy = gyw + j;
    const bool rin = gy >= 0 && gy < L.ny;
    const long long rowp = pbase + (long long)gy * nx + gx0;
    if (rin && lane_full && vec) {
      cp_async16(&bs[j][lane], P.R.b + rowp);
      if (P.zero_x) { A[j] = B[j] = f2(0.f); }
      else {
        const float4 v = __ldg(reinterpret_cast<const float4*>(P.xin + rowp));
        A[j] = make_float2(v.x, v.z);
        B[j] = make_float2(v.y, v.w);
      }
    } else {
      float v[4], w[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const bool in = rin && cin[c];
        v[c] = (in && !P.zero_x) ? __ldg(P.xin + rowp + c) : 0.f;
        w[c] = in ? __ldg(P.R.b + rowp + c) : 0.f;
      }
      A[j] = make_float2(v[0], v[2]);
      B[j] = make_float2(v[1], v[3]);
      bs[j][lane] = make_float4(w[0], w[1], w[2], w[3]);
    }
  }
  // coarse correction values for the up pass (issued before waiting on anything)
  constexpr int NQ = G_R / 2 + 2;
  float2 cv[NQ];  // (v0, v1) at coarse columns (Ix0, Ix0+1), coarse rows Jw .. Jw+NQ-1
  const int Ix0 = gx0 >> 1;
  const int Jw = (gyw >> 1) - 1;
  const long long cplane = (long long)P.ncx * P.ncy;
  if (!DOWN) {
    const float* xcp = P.xc + (long long)iz * cplane;
    const bool cvec = (P.ncx & 1) == 0 && Ix0 >= 0 && Ix0 + 1 < P.ncx;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int J = Jw + q;
      const float* rp = xcp + (long long)J * P.ncx + Ix0;
      if (J >= 0 && J < P.ncy && cvec) cv[q] = __ldg(reinterpret_cast<const float2*>(rp));
      else {
        const bool rin = J >= 0 && J < P.ncy;
        cv[q] = make_float2((rin && Ix0 >= 0 && Ix0 < P.ncx) ? __ldg(rp) : 0.f,
                            (rin && Ix0 + 1 >= 0 && Ix0 + 1 < P.ncx) ? __ldg(rp + 1) : 0.f);
      }
    }
  }

  // ---- per-row data (rows -1 .. G_R of this warp) and the 1/D table, while loads fly
  RowInfo(&ri)[G_R + 2] = srow[warp];
  if (lane < G_R + 2) {
    const int gy = gyw + lane - 1;
    RowInfo r;
    r.yl = cl(L.ay, gy);
    r.yr = cr(L.ay, gy);
    r.in = gy >= 0 && gy < L.ny;
    const int n = L.ay.n;
    r.dcase = !r.in ? 0 : (gy == 0 ? 1 : (gy == n - 1 ? 3 : (gy == n - 2 ? 2 : 0)));
    ri[lane] = r;
  }
  {
    // 1/D of my columns for the four row cases: 0 regular (or outside the domain, whose values
    // never reach it), 1 the first row, 2 the row before the last, 3 the last row
    auto invd = [&](int c, float yl, float yr) {
      Coef k;
      k.xl = cxl[c]; k.xr = cxr[c]; k.yl = yl; k.yr = yr; k.zl = 0.f; k.zr = 0.f;
      return relax_inv(L.omega, k.diag(alpha));  // == the weight of gs_update
    };
    const int ny = L.ay.n;
    const int rows[4] = {1, 0, ny - 2, ny - 1};
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const float yl = k == 0 ? L.ay.k : cl(L.ay, rows[k]);
      const float yr = k == 0 ? L.ay.k : cr(L.ay, rows[k]);
      sinv[warp][k][0][lane] = make_float2(invd(0, yl, yr), invd(2, yl, yr));
      sinv[warp][k][1][lane] = make_float2(invd(1, yl, yr), invd(3, yl, yr));
    }
  }
  cp_async_wait_all();
  __syncwarp();
  // b rows to pack layout in place: (c0, c1, c2, c3) -> (c0, c2 | c1, c3)
#pragma unroll
  for (int j = 0; j < G_R; ++j) {
    const float4 v = bs[j][lane];
    bs[j][lane] = make_float4(v.x, v.z, v.y, v.w);
  }
  auto bpk = [&](int j, int pk) -> float2 {
    const float4* p = &bs[j][lane];
    return reinterpret_cast<const float2*>(p)[pk];
  };

  // ---------------------------------------------------------------- up: add P e_c
  if (!DOWN) {
    float tx[4];
    bool selfJ[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      long long I, J;
      ptaps(P.tx, gx0 + c, I, J, tx[c]);
      selfJ[c] = J == I;
    }
    const float2 txA = make_float2(tx[0], tx[2]), txB = make_float2(tx[1], tx[3]);
    const float2 uxA = make_float2(1.f - tx[0], 1.f - tx[2]), uxB = make_float2(1.f - tx[1], 1.f - tx[3]);
    float2 cn[NQ];  // (vm, vp) at coarse columns Ix0-1, Ix0+2
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      cn[q] = make_float2(__shfl_up_sync(FULL, cv[q].y, 1), __shfl_down_sync(FULL, cv[q].x, 1));
#pragma unroll
    for (int j = 0; j < G_R; ++j) {
      const int gy = gyw + j;
      long long Iy, Jy;
      float ty;
      ptaps(P.ty, gy, Iy, Jy, ty);
      const int q = (j >> 1) + 1;  // == Iy - Jw
      const int dq = (int)(Jy - Iy);
      const float2 r0 = cv[q], r1 = cn[q];
      const float2 n0 = dq < 0 ? cv[q - 1] : (dq > 0 ? cv[q + 1] : cv[q]);
      const float2 n1 = dq < 0 ? cn[q - 1] : (dq > 0 ? cn[q + 1] : cn[q]);
      // pack A = (c0, c2): parents (Ix0, Ix0+1); neighbours c0 -> Ix0-1 | Ix0, c2 -> Ix0 | Ix0+1
      const float2 aJ = make_float2(selfJ[0] ? r0.x : r1.x, selfJ[2] ? r0.y : r0.x);
      const float2 cJ = make_float2(selfJ[0] ? n0.x : n1.x, selfJ[2] ? n0.y : n0.x);
      // pack B = (c1, c3): neighbours c1 -> Ix0+1 | Ix0, c3 -> Ix0+2 | Ix0+1
      const float2 bJ = make_float2(selfJ[1] ? r0.x : r0.y, selfJ[3] ? r0.y : r1.y);
      const float2 dJ = make_float2(selfJ[1] ? n0.x : n0.y, selfJ[3] ? n0.y : n1.y);
      const float2 ty2 = f2(ty), uy2 = f2(1.f - ty);
      // x += bilerp(a, b, c, d, tx, ty) per element
      const float2 sA0 = __ffma2_rn(txA, aJ, __fmul2_rn(uxA, r0));
      const float2 sA1 = __ffma2_rn(txA, cJ, __fmul2_rn(uxA, n0));
      A[j] = __fadd2_rn(A[j], __ffma2_rn(ty2, sA1, __fmul2_rn(uy2, sA0)));
      const float2 sB0 = __ffma2_rn(txB, bJ, __fmul2_rn(uxB, r0));
      const float2 sB1 = __ffma2_rn(txB, dJ, __fmul2_rn(uxB, n0));
      B[j] = __fadd2_rn(B[j], __ffma2_rn(ty2, sB1, __fmul2_rn(uy2, sB0)));
    }
  }

  // ---------------------------------------------------------------- row exchange
  float2 sA, sB, nA, nB;
  auto exchange = [&](int buf) {
    sh_top[buf][warp][lane] = make_float4(A[0].x, A[0].y, B[0].x, B[0].y);
    sh_bot[buf][warp][lane] = make_float4(A[G_R - 1].x, A[G_R - 1].y, B[G_R - 1].x, B[G_R - 1].y);
    __syncthreads();
    const float4 s4 = warp > 0 ? sh_bot[buf][warp - 1][lane]
                               : make_float4(A[0].x, A[0].y, B[0].x, B[0].y);
    const float4 n4 = warp < G_W - 1 ? sh_top[buf][warp + 1][lane]
                                     : make_float4(A[G_R - 1].x, A[G_R - 1].y, B[G_R - 1].x, B[G_R - 1].y);
    sA = make_float2(s4.x, s4.y); sB = make_float2(s4.z, s4.w);
    nA = make_float2(n4.x, n4.y); nB = make_float2(n4.z, n4.w);
  };

  // (A x) of pack PK (0: A, 1: B) in row j: alpha x + sum_links k (x - x_n), apply_from order
  auto stencil = [&](auto PKc, auto Jc, const RowInfo& r) -> float2 {
    constexpr int PK = decltype(PKc)::value;
    constexpr int j = decltype(Jc)::value;
    const float2 yl = f2(r.yl), yr = f2(r.yr);
    if (PK == 0) {
      const float2 X = A[j];
      const float2 W = make_float2(__shfl_up_sync(FULL, B[j].y, 1), B[j].x);
      const float2 S = j > 0 ? A[j - 1] : sA, N = j < G_R - 1 ? A[j + 1] : nA;
      float2 s = __fmul2_rn(al2, X);
      s = __ffma2_rn(kxlA, sub2(X, W), s);
      s = __ffma2_rn(kxrA, sub2(X, B[j]), s);
      s = __ffma2_rn(yl, sub2(X, S), s);
      return __ffma2_rn(yr, sub2(X, N), s);
    } else {
      const float2 X = B[j];
      const float2 E = make_float2(A[j].y, __shfl_down_sync(FULL, A[j].x, 1));
      const float2 S = j > 0 ? B[j - 1] : sB, N = j < G_R - 1 ? B[j + 1] : nB;
      float2 s = __fmul2_rn(al2, X);
      s = __ffma2_rn(kxlB, sub2(X, A[j]), s);
      s = __ffma2_rn(kxrB, sub2(X, E), s);
      s = __ffma2_rn(yl, sub2(X, S), s);
      return __ffma2_rn(yr, sub2(X, N), s);
    }
  };

  // Gauss-Seidel update of the active pack of row j (out-of-domain cells keep finite values
  // that never reach the domain: every link leaving it has coefficient 0)
  auto update = [&](auto PKc, auto Jc) {
    constexpr int PK = decltype(PKc)::value;
    constexpr int j = decltype(Jc)::value;
    const RowInfo r = ri[j + 1];
    const float2 res = sub2(bpk(j, PK), stencil(PKc, Jc, r));
    const float2 iD = sinv[warp][r.dcase][PK][lane];
    if (PK == 0) A[j] = __ffma2_rn(res, iD, A[j]);
    else B[j] = __ffma2_rn(res, iD, B[j]);
  };

  // ---------------------------------------------------------------- nu sweeps
#pragma unroll 1
  for (int hs = 0; hs < 2 * NU; ++hs) {
    const int color = hs & 1;
    exchange(hs & 1);
    const int a0 = (color + gyw + (int)(zg & 1)) & 1;  // active pack of row 0 (gx0 even)
    if (a0 == 0) static_for<G_R>([&](auto J) { update(IC<(decltype(J)::value & 1)>{}, J); });
    else static_for<G_R>([&](auto J) { update(IC<((decltype(J)::value & 1) ^ 1)>{}, J); });
  }

  // ---------------------------------------------------------------- residual, restriction / norms
  exchange((2 * NU) & 1);
  const int lx0 = 4 * lane;     // local column of c = 0
  const int ly0 = warp * G_R;   // local row of j = 0
  const bool pin = lx0 >= HX && lx0 < G_COLS - HX;  // all 4 columns together (HX % 4 == 0)
  double sr = 0.0, sbb = 0.0;
  float* bcp = DOWN ? P.bc + (long long)iz * cplane : nullptr;
  float wx[4];
  if (DOWN) {
#pragma unroll
    for (int c = 0; c < 4; ++c) wx[c] = rweight(P.tx, gx0 + c);
  }
  static_for<G_R / 2>([&](auto JP) {
    constexpr int j0 = 2 * decltype(JP)::value;
    const RowInfo r0 = ri[j0 + 1], r1 = ri[j0 + 2];
    const float2 rA0 = sub2(bpk(j0, 0), stencil(IC<0>{}, IC<j0>{}, r0));
    const float2 rB0 = sub2(bpk(j0, 1), stencil(IC<1>{}, IC<j0>{}, r0));
    const float2 rA1 = sub2(bpk(j0 + 1, 0), stencil(IC<0>{}, IC<j0 + 1>{}, r1));
    const float2 rB1 = sub2(bpk(j0 + 1, 1), stencil(IC<1>{}, IC<j0 + 1>{}, r1));
    const int gy0 = gyw + j0;  // even
    const bool yin0 = ly0 + j0 >= HY && ly0 + j0 < G_ROWS - HY;  // rows j0, j0+1 together (HY even)
    if (DOWN) {
      // volume-weighted child average (fy outer, fx inner as in k_restrict); coarse cells
      // (Ix0, J) from children (c0, c1) and (Ix0+1, J) from (c2, c3)
      const int J = gy0 >> 1;
      const bool ok0 = yin0 && pin && r0.in && gx0 >= 0 && Ix0 < P.ncx && J < P.ncy;
      const bool ok1 = yin0 && pin && r0.in && Ix0 + 1 < P.ncx && J < P.ncy;
      if (ok0 || ok1) {
        const float wy0 = rweight(P.ty, gy0), wy1 = rweight(P.ty, gy0 + 1);
        const float2 wA0 = make_float2(rw3(1.f, wy0, wx[0]), rw3(1.f, wy0, wx[2]));
        const float2 wB0 = make_float2(rw3(1.f, wy0, wx[1]), rw3(1.f, wy0, wx[3]));
        const float2 wA1 = make_float2(rw3(1.f, wy1, wx[0]), rw3(1.f, wy1, wx[2]));
        const float2 wB1 = make_float2(rw3(1.f, wy1, wx[1]), rw3(1.f, wy1, wx[3]));
        float2 acc = __ffma2_rn(wA0, rA0, f2(0.f));
        float2 t = __ffma2_rn(wB0, rB0, acc);
        acc = make_float2(cin[1] ? t.x : acc.x, cin[3] ? t.y : acc.y);
        if (r1.in) {
          acc = __ffma2_rn(wA1, rA1, acc);
          t = __ffma2_rn(wB1, rB1, acc);
          acc = make_float2(cin[1] ? t.x : acc.x, cin[3] ? t.y : acc.y);
        }
        float* o = bcp + (long long)J * P.ncx + Ix0;
        if (ok0 && ok1 && (P.ncx & 1) == 0) *reinterpret_cast<float2*>(o) = acc;
        else {
          if (ok0) o[0] = acc.x;
          if (ok1) o[1] = acc.y;
        }
      }
    } else if (yin0 && pin && P.partials) {
      const float2 bA0 = bpk(j0, 0), bB0 = bpk(j0, 1), bA1 = bpk(j0 + 1, 0), bB1 = bpk(j0 + 1, 1);
      const float rr[2][4] = {{rA0.x, rB0.x, rA0.y, rB0.y}, {rA1.x, rB1.x, rA1.y, rB1.y}};
      const float bv[2][4] = {{bA0.x, bB0.x, bA0.y, bB0.y}, {bA1.x, bB1.x, bA1.y, bB1.y}};
#pragma unroll
      for (int dj = 0; dj < 2; ++dj) {
        if (!(dj ? r1.in : r0.in)) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (cin[c]) {
            sr += (double)rr[dj][c] * (double)rr[dj][c];
            sbb += (double)bv[dj][c] * (double)bv[dj][c];
          }
      }
    }
  });
  if (!DOWN && P.partials) {
    block_sum2(sr, sbb);
    if (threadIdx.x == 0)
      P.partials[((long long)iz * tiles_y + tile_y) * tiles_x + tile_x] = make_double2(sr, sbb);
  }

  // ---------------------------------------------------------------- store x (tile interior)
  if (pin) {
#pragma unroll
    for (int j = 0; j < G_R; ++j) {
      const int gy = gyw + j;
      if (!(ly0 + j >= HY && ly0 + j < G_ROWS - HY) || !ri[j + 1].in) continue;
      float* o = P.xout + pbase + (long long)gy * nx + gx0;
      if (lane_full && vec) {
        *reinterpret_cast<float4*>(o) = make_float4(A[j].x, B[j].x, A[j].y, B[j].y);
      } else {
        if (cin[0]) o[0] = A[j].x;
        if (cin[1]) o[1] = B[j].x;
        if (cin[2]) o[2] = A[j].y;
        if (cin[3]) o[3] = B[j].y;
      }
    }
  }
}

struct Smem2D {
  float4 top[2][G_W][32];        // warp boundary rows, double-buffered by half-sweep parity
  float4 bot[2][G_W][32];
  float4 b[G_W][G_R][32];        // rhs of the tile, per lane (c0, c2 | c1, c3)
  RowInfo row[G_W][G_R + 2];     // per warp row: y coefficients and flags
  float2 inv[G_W][4][2][32];     // per lane 1/D of the four row cases
};
constexpr size_t SMEM2D = sizeof(Smem2D);

struct TileRect {  // tiles [tx0, tx1) x [ty0, ty1) of the tile grid take the register kernel
  int gx, gy;      // tile grid
  int tx0, tx1, ty0, ty1;
};

// register kernel: every tile of a level whose in-plane axes are both coarsened; explicit rhs b
template <int NU, bool DOWN>
__global__ void __launch_bounds__(256, 2) k_pass2d(Pass2D P, TileRect T) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem2D& S = *reinterpret_cast<Smem2D*>(smem_raw);
  pass2d_body<NU, DOWN>(P, S.top, S.bot, S.b, S.row, S.inv, blockIdx.x, blockIdx.y, T.gx, T.gy);
}

// ---------------------------------------------------------------------------------
// edge kernel: tiles touching the domain faces (and every tile of small levels).  The tile
// lives in shared memory and every cell calls the reference per-point functions
// (coefs / rhs_g / apply_from / gs_update / rweight / ptaps / bilerp), so the result is the
// reference schedule's bit for bit.  Runtime loops keep the code small.
// ---------------------------------------------------------------------------------
struct SmemEdge {
  float x[G_ROWS][G_COLS];
  float b[G_ROWS][G_COLS];
};
constexpr size_t SMEMEDGE = sizeof(SmemEdge);

__device__ __forceinline__ void edge_tile(const TileRect& T, int e, int& tx, int& ty) {
  // enumerate the tiles outside the fast rectangle: full rows below / above it, then the
  // left and right columns of the rows it spans
  const int below = T.ty0 * T.gx;
  const int above = (T.gy - T.ty1) * T.gx;
  if (e < below) { ty = e / T.gx; tx = e % T.gx; return; }
  e -= below;
  if (e < above) { ty = T.ty1 + e / T.gx; tx = e % T.gx; return; }
  e -= above;
  const int side = T.tx0 + (T.gx - T.tx1);
  ty = T.ty0 + e / side;
  const int k = e % side;
  tx = k < T.tx0 ? k : T.tx1 + (k - T.tx0);
}

template <int NU, bool DOWN>
__global__ void __launch_bounds__(256, 2) k_pass2d_edge(Pass2D P, TileRect T) {
  constexpr int HX = halo2x(NU), HY = halo2y(NU);
  constexpr int TXI = G_COLS - 2 * HX, TYI = G_ROWS - 2 * HY;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemEdge& S = *reinterpret_cast<SmemEdge*>(smem_raw);
  const LevelK& L = P.L;
  int tx, ty;
  edge_tile(T, blockIdx.x, tx, ty);
  const int iz = blockIdx.y;
  const long long zg = L.z0 + iz;
  const int gxa = tx * TXI - HX, gya = ty * TYI - HY;
  const long long nx = L.nx, plane = (long long)L.nx * L.ny, pbase = (long long)iz * plane;
  const int tid = threadIdx.x;
  auto inside = [&](int gx, int gy) { return gx >= 0 && gx < L.nx && gy >= 0 && gy < L.ny; };

  // load x and b
  for (int i = tid; i < G_ROWS * G_COLS; i += 256) {
    const int ly = i / G_COLS, lx = i % G_COLS, gx = gxa + lx, gy = gya + ly;
    float xv = 0.f, bv = 0.f;
    if (inside(gx, gy)) {
      const long long c = pbase + (long long)gy * nx + gx;
      if (!P.zero_x) xv = P.xin[c];
      bv = __ldg(P.R.b + c);
    }
    S.x[ly][lx] = xv;
    S.b[ly][lx] = bv;
  }
  __syncthreads();
  if (!DOWN) {  // x += P e_c
    const long long cplane = (long long)P.ncx * P.ncy;
    const float* xcp = P.xc + (long long)iz * cplane;
    for (int i = tid; i < G_ROWS * G_COLS; i += 256) {
      const int ly = i / G_COLS, lx = i % G_COLS, gx = gxa + lx, gy = gya + ly;
      if (!inside(gx, gy)) continue;
      long long Ix, Jx, Iy, Jy;
      float txw, tyw;
      ptaps(P.tx, gx, Ix, Jx, txw);
      ptaps(P.ty, gy, Iy, Jy, tyw);
      const float e = bilerp(__ldg(xcp + Iy * P.ncx + Ix), __ldg(xcp + Iy * P.ncx + Jx),
                             __ldg(xcp + Jy * P.ncx + Ix), __ldg(xcp + Jy * P.ncx + Jx), txw, tyw);
      S.x[ly][lx] = __fadd_rn(S.x[ly][lx], e);
    }
    __syncthreads();
  }
  // residual of an in-domain cell whose 4 neighbours are in the tile (or absent)
  auto resid = [&](int lx, int ly, int gx, int gy, float* bval) -> float {
    const Coef k = coefs(L, gx, gy, zg);
    const float xc = S.x[ly][lx];
    Nbr nb;
    nb.w = k.xl != 0.f ? S.x[ly][lx - 1] : xc;
    nb.e = k.xr != 0.f ? S.x[ly][lx + 1] : xc;
    nb.s = k.yl != 0.f ? S.x[ly - 1][lx] : xc;
    nb.n = k.yr != 0.f ? S.x[ly + 1][lx] : xc;
    nb.d = xc;
    nb.u = xc;
    if (bval) *bval = S.b[ly][lx];
    return __fsub_rn(S.b[ly][lx], apply_from(k, L.alpha, xc, nb.w, nb.e, nb.s, nb.n, nb.d, nb.u));
  };
  // nu red-black sweeps (the outermost tile ring is never updated: it is stale anyway)
  for (int hs = 0; hs < 2 * NU; ++hs) {
    const int color = hs & 1;
    for (int i = tid; i < G_ROWS * (G_COLS / 2); i += 256) {
      const int ly = i / (G_COLS / 2), gy = gya + ly;
      const int lx = 2 * (i % (G_COLS / 2)) + ((color + gy + (int)(zg & 1)) & 1);  // gxa even
      const int gx = gxa + lx;
      if (lx == 0 || lx == G_COLS - 1 || ly == 0 || ly == G_ROWS - 1 || !inside(gx, gy)) continue;
      const float xc = S.x[ly][lx];
      const float r = resid(lx, ly, gx, gy, nullptr);
      S.x[ly][lx] = gs_update(xc, r, coefs(L, gx, gy, zg).diag(L.alpha), L.omega);
    }
    __syncthreads();
  }
  // residual -> restriction (down) or norms (up), over the tile interior
  if (DOWN) {
    const long long cplane = (long long)P.ncx * P.ncy;
    float* bcp = P.bc + (long long)iz * cplane;
    const int sx = P.tx.coarsened ? 2 : 1, sy = P.ty.coarsened ? 2 : 1;
    const int ncl = TXI / sx, nrl = TYI / sy;  // coarse cells of the interior
    for (int i = tid; i < ncl * nrl; i += 256) {
      const int cyl = i / ncl, cxl = i % ncl;
      const int gx0 = gxa + HX + sx * cxl, gy0 = gya + HY + sy * cyl;
      if (gx0 >= L.nx || gy0 >= L.ny) continue;
      const int I = P.tx.coarsened ? gx0 >> 1 : gx0, J = P.ty.coarsened ? gy0 >> 1 : gy0;
      float acc = 0.f;
      for (int dy = 0; dy < sy && gy0 + dy < L.ny; ++dy) {
        const float wy = rweight(P.ty, gy0 + dy);
        for (int dx = 0; dx < sx && gx0 + dx < L.nx; ++dx) {
          const int gx = gx0 + dx, gy = gy0 + dy;
          const float r = resid(gx - gxa, gy - gya, gx, gy, nullptr);
          acc = __fmaf_rn(rw3(1.f, wy, rweight(P.tx, gx)), r, acc);
        }
      }
      bcp[(long long)J * P.ncx + I] = acc;
    }
  } else {
    double sr = 0.0, sbb = 0.0;
    if (P.partials) {
      for (int i = tid; i < TYI * TXI; i += 256) {
        const int ly = HY + i / TXI, lx = HX + i % TXI, gx = gxa + lx, gy = gya + ly;
        if (!inside(gx, gy)) continue;
        float bv;
        const float r = resid(lx, ly, gx, gy, &bv);
        sr += (double)r * (double)r;
        sbb += (double)bv * (double)bv;
      }
      block_sum2(sr, sbb);
      if (tid == 0) P.partials[((long long)iz * T.gy + ty) * T.gx + tx] = make_double2(sr, sbb);
    }
  }
  // store the interior
  for (int i = tid; i < TYI * TXI; i += 256) {
    const int ly = HY + i / TXI, lx = HX + i % TXI, gx = gxa + lx, gy = gya + ly;
    if (inside(gx, gy)) P.xout[pbase + (long long)gy * nx + gx] = S.x[ly][lx];
  }
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
bool fusable2d(const Level& L, const Level& C, const gdp_opts& o) {
  const bool nu_ok = o.nu_pre >= 1 && o.nu_pre <= 2 && o.nu_post >= 1 && o.nu_post <= 2;
  return nu_ok && (o.fused & 1) && L.K.az.k == 0.f && L.K.az.kr == 0.f && L.K.az.kl == 0.f && !C.tz.coarsened;
}

static TileRect tiles2d(int nu, const LevelK& L, bool fast_ok) {
  const int TXI = G_COLS - 2 * halo2x(nu), TYI = G_ROWS - 2 * halo2y(nu);
  TileRect T{};
  T.gx = (L.nx + TXI - 1) / TXI;
  T.gy = (L.ny + TYI - 1) / TYI;
  // the register kernel takes every tile of levels whose in-plane axes are both coarsened;
  // other levels (one axis stopped coarsening) go to the shared-memory edge kernel
  T.tx0 = 0; T.ty0 = 0;
  T.tx1 = fast_ok ? T.gx : 0;
  T.ty1 = fast_ok ? T.gy : 0;
  return T;
}

// norm partials per plane left by the fused up pass of level L (coarse level C)
// the up pass on wide planes: prolongation kernel + row-marching sweeps (the prolongation inside
// either fused kernel costs more than its own streaming pass there)
static bool up2d_rows(const Level& L, const Level& C) { return C.tx.coarsened && C.ty.coarsened && L.nx >= 128; }

int fused_tiles_per_plane(int nu, const Level& L, const Level& C) {  // norm partials per plane
  if (up2d_rows(L, C)) return rows2d_items_per_plane(nu, L.K);
  const TileRect T = tiles2d(nu, L.K, false);
  return T.gx * T.gy;
}

template <typename K>
static void set_smem(K k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int NU, bool DOWN>
static void launch2d_nu(const Pass2D& P, const TileRect& T, cudaStream_t s) {
  static bool attr = false;  // opt in to > 48 KB dynamic shared memory once per instantiation
  if (!attr) {
    set_smem(k_pass2d<NU, DOWN>, SMEM2D);
    set_smem(k_pass2d_edge<NU, DOWN>, SMEMEDGE);
    attr = true;
  }
  const int nfast = (T.tx1 - T.tx0) * (T.ty1 - T.ty0);
  const int nedge = T.gx * T.gy - nfast;
  if (nfast > 0) {
    dim3 g(T.tx1 - T.tx0, T.ty1 - T.ty0, P.L.nzl);
    k_pass2d<NU, DOWN><<<g, 256, SMEM2D, s>>>(P, T);
  }
  if (nedge > 0) {
    if (nfast > 0) count_launch();
    dim3 g(nedge, P.L.nzl);
    k_pass2d_edge<NU, DOWN><<<g, 256, SMEMEDGE, s>>>(P, T);
  }
}

static void launch2d(bool down, int nu, const Pass2D& P, cudaStream_t s) {
  const TileRect T = tiles2d(nu, P.L, P.fast_ok != 0);
  const double N = (double)P.L.nx * P.L.ny * P.L.nzl, Nc = (double)P.ncx * P.ncy * P.L.nzl;
  const double bytes = N * ((P.zero_x ? 4.0 : 8.0) + 4.0) + Nc * 4.0;
  ProfScope ps(down ? KC_DOWN2D : KC_UP2D, bytes, s, N, true);
  if (down) {
    if (nu == 1) launch2d_nu<1, true>(P, T, s);
    else launch2d_nu<2, true>(P, T, s);
  } else {
    if (nu == 1) launch2d_nu<1, false>(P, T, s);
    else launch2d_nu<2, false>(P, T, s);
  }
}

void fused_down2d(const Level& L, const Level& C, const float* xin, float* xout, const RhsK& R,
                  int mode, int tI, int nu, bool zero_x, cudaStream_t s, bool prolong) {
  // row-marching kernel (gdp_rows2d.cu) for wide planes: no row halo, no barriers (measured
  // 0.81 vs 1.12 ms on a 1024^2 x 128 down pass); the tile kernel below elsewhere.
  // prolong (FMG start): x += P C.x, added at load by the row kernel (coarse rows staged in
  // shared memory) on planes under 1M cells, else by its own pass
  if (C.tx.coarsened && C.ty.coarsened && L.nx >= 128) {
    // planes of >= 1M cells: the prolongation by its own pass measured faster at 1024^2 x 128
    // (0.31 + 0.48 ms against 0.99 ms with the coarse rows staged inside the row kernel)
    const bool split = prolong && !zero_x && (long long)L.nx * L.ny >= (1LL << 20);
    if (split)
      launch_prolong(L.K, const_cast<float*>(xin), C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
    rows2d_pass(true, nu, L, C, xin, xout, R.b, zero_x, nullptr, s, prolong && !split);
    return;
  }
  if (prolong)
    launch_prolong(L.K, const_cast<float*>(xin), C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
  Pass2D P{};
  P.L = L.K; P.xin = xin; P.xout = xout; P.R = R; P.zero_x = zero_x ? 1 : 0;
  P.fast_ok = C.tx.coarsened && C.ty.coarsened;
  P.tx = C.tx; P.ty = C.ty; P.ncx = C.nx; P.ncy = C.ny;
  P.bc = C.b;
  (void)mode; (void)tI;
  launch2d(true, nu, P, s);
}

void fused_up2d(const Level& L, const Level& C, const float* xin, float* xout, const RhsK& R,
                int mode, int tI, int nu, double2* partials, cudaStream_t s) {
  if (up2d_rows(L, C)) {  // the prolongation inside the row kernel measured slower (1.03 vs 0.31 + 0.65 ms)
    launch_prolong(L.K, const_cast<float*>(xin), C.tx, C.ty, C.tz, C.nx, C.ny, C.nzl, C.z0, C.x, C.xlo, C.xhi, s);
    rows2d_pass(false, nu, L, C, xin, xout, R.b, false, partials, s, false);
    return;
  }
  Pass2D P{};
  P.L = L.K; P.xin = xin; P.xout = xout; P.R = R; P.zero_x = 0;
  P.fast_ok = C.tx.coarsened && C.ty.coarsened;
  P.tx = C.tx; P.ty = C.ty; P.ncx = C.nx; P.ncy = C.ny;
  P.xc = C.x;
  P.partials = partials;
  (void)mode; (void)tI;
  launch2d(false, nu, P, s);
}

}  // namespace gdp
