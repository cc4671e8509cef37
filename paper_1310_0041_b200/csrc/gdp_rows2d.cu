// gdp_rows2d.cu — fused 2D level passes by row marching (levels without z links: every
// phase-2 level, Eq. 2), sm_100a.
//
// One HBM pass per level and direction ("multiple relaxation passes in one
// streaming pass"): down = nu red-black Gauss-Seidel sweeps + residual + volume-weighted
// restriction, up = prolongated correction + nu sweeps + fp64 residual norms.  Each warp owns
// a strip of 128 columns (4 per lane, packs A = (c0, c2), B = (c1, c3): the two cells of one
// colour in a row) of one plane and marches down a chunk of its rows.  With t the row being
// loaded, half-sweep s (colour (s-1) & 1) updates row t-s and the tail takes the residual of
// row t-2nu-1: the row pipeline is exactly the reference schedule's half-sweeps (a point of one
// colour depends only on the other colour), so the iterate is bit-identical to it.
//   * rows of x and b are staged into shared memory by cp.async five rows ahead (each thread
//     stages and reads only its own cells: no barrier anywhere in the kernel);
//   * the last 2nu + 3 rows of x and 2nu + 2 rows of b live in registers as shift registers
//     (index = lag behind the loaded row, shifted once per row; the march is unrolled by two
//     so the colour of every lag is static); y-neighbours are registers, x-neighbours come from
//     the adjacent lane (__shfl);
//   * only the strip's 2nu + 1 (rounded to 4) halo columns per side are recomputed; the row
//     direction has no halo except at chunk boundaries (2nu + 1 rows).
#include <algorithm>

#include "gdp_internal.h"
#include "gdp_pack.cuh"

namespace gdp {

struct Rows2D {
  LevelK L;
  const float* xin;     // x before the pass (ignored if zero_x)
  float* xout;          // x after the pass (another buffer: strips read each other's halo)
  const float* b;       // rhs
  int vec;              // nx % 4 == 0 and 16-byte aligned arrays: float4 / cp.async.16 rows
  int zero_x;
  XferAxis tx, ty;      // fine -> coarse (both in-plane axes coarsened)
  int ncx, ncy;
  float* bc;            // down: coarse rhs
  const float* xc;      // up: coarse correction
  double2* partials;    // up: one (sum r^2, sum b^2) per item (may be null)
  int strips, ych, chunk;
  long long nitems;     // nzl * strips * ych, plane-major
};

template <int NU> struct R2C {
  static constexpr int S = 2 * NU;                    // half-sweeps
  static constexpr int LAG = S + 1;                   // row lag of the tail
  static constexpr int XR = LAG + 2;                  // x rows held in registers: t .. t-LAG-1
  static constexpr int BR = LAG + 1;                  // b rows held in registers: t .. t-LAG
  static constexpr int HX = ((2 * NU + 1) + 3) & ~3;  // halo columns per side (8 / 4)
  static constexpr int TXI = 128 - 2 * HX;            // interior columns of a strip
};
constexpr int R2_WARPS = 4;
constexpr int R2_D = 5;   // prefetch distance (rows)
constexpr int R2_SL = 8;  // staging slots (power of two > R2_D)
constexpr int R2_CS = 8;  // coarse-row slots (rows c-1 .. c+6 live at once)

struct Row4 { float2 A, B; };

// cold paths kept out of line (they would otherwise be inlined into each of the 8 ring steps)
__device__ __noinline__ float2 r2_invd(float xl0, float xr0, float xl1, float xr1, float yl, float yr, float alpha,
                                       float omega) {
  Coef k;
  k.zl = 0.f; k.zr = 0.f; k.yl = yl; k.yr = yr;
  k.xl = xl0; k.xr = xr0;
  const float a = relax_inv(omega, k.diag(alpha));  // == the weight of gs_update
  k.xl = xl1; k.xr = xr1;
  return make_float2(a, relax_inv(omega, k.diag(alpha)));
}
__device__ __noinline__ float r2_rweight(XferAxis a, int i) { return rweight(a, i); }
struct R2Tap { int dq; float t; };
__device__ __noinline__ R2Tap r2_ptaps(XferAxis a, int i) {
  long long I, J;
  float t;
  ptaps(a, i, I, J, t);
  return R2Tap{(int)(J - I), t};
}

template <int NU, bool DOWN, bool VEC, bool PRO>
__device__ __forceinline__ void rows2d_march(const Rows2D& P, float4 (*sx)[R2_WARPS * 32],
                                             float4 (*sb)[R2_WARPS * 32], float2 (*sc)[R2_WARPS * 32],
                                             long long item) {
  using RC = R2C<NU>;
  constexpr int XR = RC::XR, BR = RC::BR, S = RC::S, LAG = RC::LAG;
  const int tid = threadIdx.x, lane = tid & 31;
  const LevelK& L = P.L;
  const int per = P.strips * P.ych;
  const int iz = (int)(item / per);
  const int rem = (int)(item - (long long)iz * per);
  const int strip = rem / P.ych, yc = rem - strip * P.ych;
  const int y_lo = yc * P.chunk, y_hi = min(y_lo + P.chunk, L.ny);
  const int ny = L.ny;
  const long long nx = L.nx;
  const long long pbase = (long long)iz * L.nx * L.ny;
  const int zp = (int)((L.z0 + iz) & 1);  // colour of (x, y, z) = (x + y + zp) & 1
  const float alpha = L.alpha;
  const float2 al2 = f2(alpha);

  // ---- my columns
  const int gx0 = strip * RC::TXI - RC::HX + 4 * lane;
  bool cin[4];
  float cxl[4], cxr[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    cin[c] = gx0 + c >= 0 && gx0 + c < L.nx;
    cxl[c] = cl(L.ax, gx0 + c);
    cxr[c] = cr(L.ax, gx0 + c);
  }
  const float2 kxlA = make_float2(cxl[0], cxl[2]), kxrA = make_float2(cxr[0], cxr[2]);
  const float2 kxlB = make_float2(cxl[1], cxl[3]), kxrB = make_float2(cxr[1], cxr[3]);
  const bool lane_full = cin[0] && cin[1] && cin[2] && cin[3];
  const bool lane_any = cin[0] || cin[1] || cin[2] || cin[3];
  constexpr bool vec = VEC;  // nx % 4 == 0: lane quads are 16-byte aligned
  const bool pin = lane >= RC::HX / 4 && lane < 32 - RC::HX / 4;  // interior columns
  const float2 ivA = r2_invd(cxl[0], cxr[0], cxl[2], cxr[2], L.ay.k, L.ay.k, alpha, L.omega);  // regular rows
  const float2 ivB = r2_invd(cxl[1], cxr[1], cxl[3], cxr[3], L.ay.k, L.ay.k, alpha, L.omega);
  // restriction weights of my columns
  float w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f;
  if (DOWN) {
    w0 = r2_rweight(P.tx, gx0); w1 = r2_rweight(P.tx, gx0 + 1);
    w2 = r2_rweight(P.tx, gx0 + 2); w3 = r2_rweight(P.tx, gx0 + 3);
  }

  // ---- row ranges: loads [a, e), half-sweep s on [lo(s), hi(s)), tail [y_lo, y_hi)
  const int a = max(y_lo - LAG, 0), e = min(y_hi + LAG, ny);
  const int tend = y_hi + LAG;

  // ---- prolongation (PRO)
  const int Ix0 = gx0 >> 1;
  const long long cplane = (long long)P.ncx * P.ncy;
  // PRO: coarse rows (columns Ix0, Ix0 + 1) are cp.async-staged into a private ring of 8 slots
  // indexed by coarse row mod 8: row J goes out with the staging of fine row 2(J-3), so it is
  // complete before the first row that reads it and no register ever waits on it
  const float* xcp = PRO ? P.xc + (long long)iz * cplane : nullptr;
  auto issue_cr = [&](int J) {
    float2* d = &sc[J & (R2_CS - 1)][tid];
    const bool rq = J >= 0 && J < P.ncy;
    const float* rp = xcp + (long long)(rq ? J : 0) * P.ncx;
    const bool v0 = rq && Ix0 >= 0 && Ix0 < P.ncx, v1 = rq && Ix0 + 1 >= 0 && Ix0 + 1 < P.ncx;
    if ((P.ncx & 1) == 0 && v0 && v1) {
      cp_async8z(d, rp + Ix0, true);
    } else {
      cp_async4z(&d->x, v0 ? rp + Ix0 : xcp, v0);
      cp_async4z(&d->y, v1 ? rp + Ix0 + 1 : xcp, v1);
    }
  };
  float ptx[4];
  bool selfJ[4];
  if (PRO) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      long long I, J;
      ptaps(P.tx, gx0 + c, I, J, ptx[c]);
      selfJ[c] = J == I;
    }
    const int c0 = a >> 1;
#pragma unroll
    for (int d = -1; d <= 3; ++d) issue_cr(c0 + d);  // joins the first staging group
  }
  auto issue = [&](int t) {  // stage row t (own quads) into slot t & 7
    const int sl = t & (R2_SL - 1);
    if (PRO && (t & 1) == 0) issue_cr((t >> 1) + 3);
    const long long ro = pbase + (long long)t * nx + gx0;
    if constexpr (VEC) {
      const long long o = lane_full ? ro : 0;
      if (!P.zero_x) cp_async16z(&sx[sl][tid], P.xin + o, lane_full);
      cp_async16z(&sb[sl][tid], P.b + o, lane_full);
    } else {
      float* dx = reinterpret_cast<float*>(&sx[sl][tid]);
      float* db = reinterpret_cast<float*>(&sb[sl][tid]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const long long o = cin[c] ? ro + c : 0;
        if (!P.zero_x) cp_async4z(dx + c, P.xin + o, cin[c]);
        cp_async4z(db + c, P.b + o, cin[c]);
      }
    }
  };
#pragma unroll
  for (int k = 0; k < R2_D; ++k) {
    if (a + k < e) issue(a + k);
    cp_async_commit();
  }

  Row4 X[XR], Bv[BR];  // X[j] / Bv[j]: row t - j
#pragma unroll
  for (int k = 0; k < XR; ++k) X[k].A = X[k].B = f2(0.f);
#pragma unroll
  for (int k = 0; k < BR; ++k) Bv[k].A = Bv[k].B = f2(0.f);

  float2 racc = f2(0.f);  // down: restriction accumulated over the two child rows
  double sr = 0.0, sbb = 0.0;
  float2 nr = make_float2(0.f, 0.f), nb = nr;  // norms: up to 8 rows (32 cells) in fp32, then fp64
  int nrows = 0;

  // (A x) of pack PK of the row in X[KO] (KS south, KN north), apply_from order (z terms exact 0)
  auto stencil = [&](auto PKc, const Row4& Xo, const Row4& Xs, const Row4& Xn, float2 yl, float2 yr) -> float2 {
    constexpr int PK = decltype(PKc)::value;
    if (PK == 0) {
      const float2 Xc = Xo.A;
      const float2 W = make_float2(__shfl_up_sync(FULL, Xo.B.y, 1), Xo.B.x);
      float2 s = __fmul2_rn(al2, Xc);
      s = __ffma2_rn(kxlA, sub2(Xc, W), s);
      s = __ffma2_rn(kxrA, sub2(Xc, Xo.B), s);
      s = __ffma2_rn(yl, sub2(Xc, Xs.A), s);
      return __ffma2_rn(yr, sub2(Xc, Xn.A), s);
    } else {
      const float2 Xc = Xo.B;
      const float2 E = make_float2(Xo.A.y, __shfl_down_sync(FULL, Xo.A.x, 1));
      float2 s = __fmul2_rn(al2, Xc);
      s = __ffma2_rn(kxlB, sub2(Xc, Xo.A), s);
      s = __ffma2_rn(kxrB, sub2(Xc, E), s);
      s = __ffma2_rn(yl, sub2(Xc, Xs.B), s);
      return __ffma2_rn(yr, sub2(Xc, Xn.B), s);
    }
  };

  auto step = [&](auto KK, int t) {
    constexpr int KP = decltype(KK)::value;  // (t + zp) & 1: colour parity of row t
#pragma unroll
    for (int j = XR - 1; j > 0; --j) X[j] = X[j - 1];
#pragma unroll
    for (int j = BR - 1; j > 0; --j) Bv[j] = Bv[j - 1];
    constexpr int K = 0;
    // (1) load row t, add the coarse correction
    if (t < e) {
      if (t + R2_D < e) issue(t + R2_D);
      cp_async_commit();
      cp_async_wait<R2_D>();
      const int sl = t & (R2_SL - 1);
      const float4 bv = sb[sl][tid];
      Bv[K].A = make_float2(bv.x, bv.z);
      Bv[K].B = make_float2(bv.y, bv.w);
      if (P.zero_x) {
        X[K].A = X[K].B = f2(0.f);
      } else {
        const float4 v = sx[sl][tid];
        X[K].A = make_float2(v.x, v.z);
        X[K].B = make_float2(v.y, v.w);
      }
      if (PRO) {
        const int cc = t >> 1;
        int dq;
        float ty;
        if (ptaps_regular(P.ty, t)) { dq = (t & 1) ? 1 : -1; ty = 0.25f; }  // == ptaps_fast
        else { const R2Tap tp = r2_ptaps(P.ty, t); dq = tp.dq; ty = tp.t; }
        const float2 r0 = sc[cc & (R2_CS - 1)][tid];
        const float2 n0 = sc[(cc + dq) & (R2_CS - 1)][tid];
        const float2 r1 = make_float2(__shfl_up_sync(FULL, r0.y, 1), __shfl_down_sync(FULL, r0.x, 1));
        const float2 n1 = make_float2(__shfl_up_sync(FULL, n0.y, 1), __shfl_down_sync(FULL, n0.x, 1));
        const float2 txA = make_float2(ptx[0], ptx[2]), txB = make_float2(ptx[1], ptx[3]);
        const float2 uxA = make_float2(1.f - ptx[0], 1.f - ptx[2]), uxB = make_float2(1.f - ptx[1], 1.f - ptx[3]);
        const float2 aJ = make_float2(selfJ[0] ? r0.x : r1.x, selfJ[2] ? r0.y : r0.x);
        const float2 cJ = make_float2(selfJ[0] ? n0.x : n1.x, selfJ[2] ? n0.y : n0.x);
        const float2 bJ = make_float2(selfJ[1] ? r0.x : r0.y, selfJ[3] ? r0.y : r1.y);
        const float2 dJ = make_float2(selfJ[1] ? n0.x : n0.y, selfJ[3] ? n0.y : n1.y);
        const float2 ty2 = f2(ty), uy2 = f2(1.f - ty);
        const float2 sA0 = __ffma2_rn(txA, aJ, __fmul2_rn(uxA, r0));
        const float2 sA1 = __ffma2_rn(txA, cJ, __fmul2_rn(uxA, n0));
        X[K].A = __fadd2_rn(X[K].A, __ffma2_rn(ty2, sA1, __fmul2_rn(uy2, sA0)));
        const float2 sB0 = __ffma2_rn(txB, bJ, __fmul2_rn(uxB, r0));
        const float2 sB1 = __ffma2_rn(txB, dJ, __fmul2_rn(uxB, n0));
        X[K].B = __fadd2_rn(X[K].B, __ffma2_rn(ty2, sB1, __fmul2_rn(uy2, sB0)));
      }
    } else {
      X[K].A = X[K].B = Bv[K].A = Bv[K].B = f2(0.f);
    }
    // (2) half-sweeps: s updates row t - s with colour (s - 1) & 1
    static_for<S>([&](auto Sc) {
      constexpr int s = decltype(Sc)::value + 1;
      constexpr int KO = s, KS = s + 1, KN = s - 1;  // rows t - s, t - s - 1, t - s + 1
      constexpr int C = (s - 1) & 1;
      constexpr int PK = (C + KP + s) & 1;  // active pack of row t - s: (C + row + z) & 1
      const int q = t - s;
      const int lo = max(y_lo - (LAG - s), 0), hi = min(y_hi + (LAG - s), ny);
      if (q >= lo && q < hi) {
        const float yl = cl(L.ay, q), yr = cr(L.ay, q);
        float2 iD = PK == 0 ? ivA : ivB;
        if (q == 0 || q >= ny - 2)
          iD = PK == 0 ? r2_invd(cxl[0], cxr[0], cxl[2], cxr[2], yl, yr, alpha, L.omega)
                       : r2_invd(cxl[1], cxr[1], cxl[3], cxr[3], yl, yr, alpha, L.omega);
        const float2 sten = stencil(IC<PK>{}, X[KO], X[KS], X[KN], f2(yl), f2(yr));
        if (PK == 0) X[KO].A = __ffma2_rn(sub2(Bv[KO].A, sten), iD, X[KO].A);
        else X[KO].B = __ffma2_rn(sub2(Bv[KO].B, sten), iD, X[KO].B);
      }
    });
    // (3) tail on row q = t - LAG
    const int q = t - LAG;
    if (q >= y_lo && q < y_hi) {
      constexpr int KO = LAG, KS = LAG + 1, KN = LAG - 1;
      const Row4& Xo = X[KO];
      if (DOWN || P.partials) {
        const float2 yl = f2(cl(L.ay, q)), yr = f2(cr(L.ay, q));
        const float2 rA = sub2(Bv[KO].A, stencil(IC<0>{}, Xo, X[KS], X[KN], yl, yr));
        const float2 rB = sub2(Bv[KO].B, stencil(IC<1>{}, Xo, X[KS], X[KN], yl, yr));
        if (DOWN && pin) {
          // volume-weighted child average, fy outer, fx inner (k_restrict order)
          const bool first = (q & 1) == 0;  // even row: first child row of coarse row q >> 1
          const bool last = !first || q == ny - 1;
          const float wy = q + 2 < P.ty.nf ? 0.5f : r2_rweight(P.ty, q);  // == rweight: H / (H + H)
          const float2 wA = make_float2(rw3(1.f, wy, w0), rw3(1.f, wy, w2));
          const float2 wB = make_float2(rw3(1.f, wy, w1), rw3(1.f, wy, w3));
          float2 acc = __ffma2_rn(wA, rA, first ? f2(0.f) : racc);
          const float2 tt = __ffma2_rn(wB, rB, acc);
          acc = make_float2(cin[1] ? tt.x : acc.x, cin[3] ? tt.y : acc.y);
          if (last) {
            const int J = q >> 1;
            const bool ok0 = cin[0] && Ix0 < P.ncx && J < P.ncy;
            const bool ok1 = cin[2] && Ix0 + 1 < P.ncx && J < P.ncy;
            float* o = P.bc + (long long)iz * cplane + (long long)J * P.ncx + Ix0;
            if (ok0 && ok1 && (P.ncx & 1) == 0) *reinterpret_cast<float2*>(o) = acc;
            else {
              if (ok0) o[0] = acc.x;
              if (ok1) o[1] = acc.y;
            }
          } else {
            racc = acc;
          }
        } else if (!DOWN && pin) {
          const float2 bA = Bv[KO].A, bB = Bv[KO].B;
          const float2 ra = make_float2(cin[0] ? rA.x : 0.f, cin[2] ? rA.y : 0.f);
          const float2 rb = make_float2(cin[1] ? rB.x : 0.f, cin[3] ? rB.y : 0.f);
          const float2 ba = make_float2(cin[0] ? bA.x : 0.f, cin[2] ? bA.y : 0.f);
          const float2 bbv = make_float2(cin[1] ? bB.x : 0.f, cin[3] ? bB.y : 0.f);
          nr = __ffma2_rn(rb, rb, __ffma2_rn(ra, ra, nr));
          nb = __ffma2_rn(bbv, bbv, __ffma2_rn(ba, ba, nb));
          if (++nrows == 8) {
            sr += (double)nr.x + (double)nr.y;
            sbb += (double)nb.x + (double)nb.y;
            nr = nb = make_float2(0.f, 0.f);
            nrows = 0;
          }
        }
      }
      if (pin && lane_any) {  // store row q
        float* o = P.xout + pbase + (long long)q * nx + gx0;
        if (vec && lane_full) *reinterpret_cast<float4*>(o) = make_float4(Xo.A.x, Xo.B.x, Xo.A.y, Xo.B.y);
        else {
          if (cin[0]) o[0] = Xo.A.x;
          if (cin[1]) o[1] = Xo.B.x;
          if (cin[2]) o[2] = Xo.A.y;
          if (cin[3]) o[3] = Xo.B.y;
        }
      }
    }
  };

  int t = a;
  if ((a + zp) & 1) step(IC<1>{}, t++);
  for (; t + 1 < tend; t += 2) {
    step(IC<0>{}, t);
    step(IC<1>{}, t + 1);
  }
  if (t < tend) step(IC<0>{}, t);
  if (!DOWN && P.partials) {
    sr += (double)nr.x + (double)nr.y;
    sbb += (double)nb.x + (double)nb.y;
    for (int o = 16; o > 0; o >>= 1) {
      sr += __shfl_down_sync(FULL, sr, o);
      sbb += __shfl_down_sync(FULL, sbb, o);
    }
    if (lane == 0) P.partials[item] = make_double2(sr, sbb);
  }
}

// PRO: the coarse correction is added to x at load (else the caller prolongated beforehand)
template <int NU, bool DOWN, bool PRO>
__global__ void __launch_bounds__(R2_WARPS * 32) k_rows2d(const __grid_constant__ Rows2D P) {
  __shared__ float4 sx[R2_SL][R2_WARPS * 32];
  __shared__ float4 sb[R2_SL][R2_WARPS * 32];
  __shared__ float2 sc[PRO ? R2_CS : 1][R2_WARPS * 32];
  const long long item = (long long)blockIdx.x * R2_WARPS + (threadIdx.x >> 5);
  if (item >= P.nitems) return;  // warp-uniform; the kernel has no block-wide barrier
  if (P.vec) rows2d_march<NU, DOWN, true, PRO>(P, sx, sb, sc, item);
  else rows2d_march<NU, DOWN, false, PRO>(P, sx, sb, sc, item);
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
static int rows2d_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// strips x row chunks: the chunk count minimising waves x (chunk + 2 * lag) over ~16 warps / SM
static void plan_rows2d(int nu, const LevelK& L, Rows2D& P) {
  const int txi = nu == 1 ? R2C<1>::TXI : R2C<2>::TXI;
  const int lag = 2 * nu + 1;
  P.strips = (L.nx + txi - 1) / txi;
  const long long slots = (long long)rows2d_sms() * 16;
  double best = 1e30;
  int bch = 1, bchunk = L.ny + (L.ny & 1);
  for (int ych = 1; ych <= L.ny; ++ych) {
    int chunk = (L.ny + ych - 1) / ych;
    chunk += chunk & 1;  // coarse row pairs never straddle chunks
    const int real = (L.ny + chunk - 1) / chunk;
    const long long items = (long long)L.nzl * P.strips * real;
    const double cost = (double)((items + slots - 1) / slots) * (chunk + 2 * lag);
    if (cost < best - 1e-9) { best = cost; bch = real; bchunk = chunk; }
    if (chunk <= 8) break;
  }
  P.ych = bch;
  P.chunk = bchunk;
  P.nitems = (long long)L.nzl * P.strips * P.ych;
}

int rows2d_items_per_plane(int nu, const LevelK& L) {
  Rows2D P{};
  plan_rows2d(nu, L, P);
  return P.strips * P.ych;
}

void rows2d_pass(bool down, int nu, const Level& L, const Level& C, const float* xin, float* xout, const float* b,
                 bool zero_x, double2* partials, cudaStream_t s, bool prolong) {
  Rows2D P{};
  P.L = L.K; P.xin = xin; P.xout = xout; P.b = b; P.zero_x = zero_x ? 1 : 0;
  P.vec = (L.nx & 3) == 0 && al16(xin) && al16(xout) && al16(b);
  P.tx = C.tx; P.ty = C.ty; P.ncx = C.nx; P.ncy = C.ny;
  P.bc = C.b; P.xc = C.x; P.partials = partials;
  plan_rows2d(nu, L.K, P);
  const double N = (double)L.nx * L.ny * L.nzl, Nc = (double)C.nx * C.ny * C.nzl;
  ProfScope ps(down ? KC_DOWN2D : KC_UP2D, N * ((zero_x ? 4.0 : 8.0) + 4.0) + Nc * ((down ? 4.0 : 0.0) + (prolong ? 4.0 : 0.0)), s, N, true);
  const unsigned grid = (unsigned)((P.nitems + R2_WARPS - 1) / R2_WARPS);
  if (down && prolong) {  // FMG start: the coarse correction added at load
    if (nu == 1) k_rows2d<1, true, true><<<grid, R2_WARPS * 32, 0, s>>>(P);
    else k_rows2d<2, true, true><<<grid, R2_WARPS * 32, 0, s>>>(P);
  } else if (down) {
    if (nu == 1) k_rows2d<1, true, false><<<grid, R2_WARPS * 32, 0, s>>>(P);
    else k_rows2d<2, true, false><<<grid, R2_WARPS * 32, 0, s>>>(P);
  } else if (prolong) {
    if (nu == 1) k_rows2d<1, false, true><<<grid, R2_WARPS * 32, 0, s>>>(P);
    else k_rows2d<2, false, true><<<grid, R2_WARPS * 32, 0, s>>>(P);
  } else {
    if (nu == 1) k_rows2d<1, false, false><<<grid, R2_WARPS * 32, 0, s>>>(P);
    else k_rows2d<2, false, false><<<grid, R2_WARPS * 32, 0, s>>>(P);
  }
}

}  // namespace gdp
