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
#include <type_traits>
#include <utility>

#include "gdp_internal.h"

namespace gdp {

template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}
template <int V> using IC = std::integral_constant<int, V>;

constexpr int F2_R = 16;                  // rows per warp
constexpr int F2_W = 8;                   // warps per CTA (stacked in y)
constexpr int F2_COLS = 64;               // columns per warp (2 per lane)
constexpr int F2_ROWS = F2_R * F2_W;      // 128
constexpr unsigned FULL = 0xffffffffu;

__host__ __device__ constexpr int halo2(int nu) { return ((2 * nu + 1) + 1) & ~1; }

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

// x-neighbours of column C (static) of a lane holding columns (2l, 2l+1)
template <int C>
__device__ __forceinline__ void xnbr(const float (&row)[2], float& w, float& e) {
  if (C == 0) {
    w = __shfl_up_sync(FULL, row[1], 1);
    e = row[1];
  } else {
    w = row[0];
    e = __shfl_down_sync(FULL, row[0], 1);
  }
}

// (A x)_c without z links: the terms apply_from() adds for zl = zr = 0 are exact zeros
__device__ __forceinline__ float apply2d(const Coef& k, float alpha, float xc, float xw, float xe,
                                         float xs, float xn) {
  float s = __fmul_rn(alpha, xc);
  s = __fmaf_rn(k.xl, xc - xw, s);
  s = __fmaf_rn(k.xr, xc - xe, s);
  s = __fmaf_rn(k.yl, xc - xs, s);
  s = __fmaf_rn(k.yr, xc - xn, s);
  return s;
}

template <typename TI> struct Pair;
template <> struct Pair<float> {
  __device__ static __forceinline__ void ld(const void* p, long long i, bool vec, float (&o)[2]) {
    const float* f = static_cast<const float*>(p) + i;
    if (vec) { const float2 v = __ldg(reinterpret_cast<const float2*>(f)); o[0] = v.x; o[1] = v.y; }
    else { o[0] = __ldg(f); o[1] = __ldg(f + 1); }
  }
};
template <> struct Pair<uint8_t> {
  __device__ static __forceinline__ void ld(const void* p, long long i, bool vec, float (&o)[2]) {
    const uint8_t* u = static_cast<const uint8_t*>(p) + i;
    if (vec) {
      const unsigned short v = __ldg(reinterpret_cast<const unsigned short*>(u));
      o[0] = decode_u8(v & 0xffu); o[1] = decode_u8(v >> 8);
    } else { o[0] = decode_u8(__ldg(u)); o[1] = decode_u8(__ldg(u + 1)); }
  }
};

template <int NU, bool DOWN, int MODE, typename TI, bool FAST>
__device__ __forceinline__ void pass2d_body(const Pass2D& P, float2 (&sh_top)[2][F2_W][32],
                                            float2 (&sh_bot)[2][F2_W][32]) {
  constexpr int H = halo2(NU);
  constexpr int TXI = F2_COLS - 2 * H, TYI = F2_ROWS - 2 * H;
  const LevelK& L = P.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx0 = blockIdx.x * TXI - H + 2 * lane;    // my even column
  const int gyw = blockIdx.y * TYI - H + warp * F2_R;  // my first row (even)
  const int iz = blockIdx.z;
  const long long zg = L.z0 + iz;
  const long long nx = L.nx;
  const long long pbase = (long long)iz * L.nx * L.ny;
  const float alpha = L.alpha;
  const bool vec = (L.nx & 1) == 0;  // 8-byte aligned column pairs

  bool cin[2], cint[2];
  float cxl[2], cxr[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int gx = gx0 + c;
    cin[c] = FAST || (gx >= 0 && gx < L.nx);
    cint[c] = FAST || col_interior(L.ax, gx);
    cxl[c] = FAST ? L.ax.k : cl(L.ax, gx);
    cxr[c] = FAST ? L.ax.k : cr(L.ax, gx);
  }
  Coef kint;
  kint.xl = L.ax.k; kint.xr = L.ax.k; kint.yl = L.ay.k; kint.yr = L.ay.k; kint.zl = 0.f; kint.zr = 0.f;
  const float invDint = __frcp_rn(kint.diag(alpha));  // == the 1/D gs_update forms inside

  auto row_in = [&](int gy) { return FAST || (gy >= 0 && gy < L.ny); };
  auto coef_at = [&](int c, int gy) {
    Coef k;
    k.xl = cxl[c]; k.xr = cxr[c];
    k.yl = FAST ? L.ay.k : cl(L.ay, gy);
    k.yr = FAST ? L.ay.k : cr(L.ay, gy);
    k.zl = 0.f; k.zr = 0.f;
    return k;
  };

  float x[F2_R][2], b[F2_R][2];
  // ---------------------------------------------------------------- load x and rhs
#pragma unroll
  for (int j = 0; j < F2_R; ++j) {
    const int gy = gyw + j;
    const long long rowp = pbase + (long long)gy * nx + gx0;
    if (FAST) {
      if (P.zero_x) { x[j][0] = x[j][1] = 0.f; }
      else Pair<float>::ld(P.xin, rowp, vec, x[j]);
      if (MODE == RHS_B) Pair<float>::ld(P.R.b, rowp, vec, b[j]);
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const bool in = row_in(gy) && cin[c];
        x[j][c] = (in && !P.zero_x) ? __ldg(P.xin + rowp + c) : 0.f;
        if (MODE == RHS_B) b[j][c] = in ? __ldg(P.R.b + rowp + c) : 0.f;
      }
    }
  }
  if (MODE == RHS_G) {
    // b = rhs_from(...) on a rolling window of I rows (gy-1, gy, gy+1)
    float Ip[2], Ic[2], In[2];
    auto ldrow = [&](int gy, float (&o)[2]) {
      const long long rowp = pbase + (long long)gy * nx + gx0;
      if (FAST) { Pair<TI>::ld(P.R.I, rowp, vec, o); return; }
#pragma unroll
      for (int c = 0; c < 2; ++c) o[c] = (row_in(gy) && cin[c]) ? ldI<TI>(P.R.I, rowp + c) : 0.f;
    };
    ldrow(gyw - 1, Ip);
    ldrow(gyw, Ic);
#pragma unroll
    for (int j = 0; j < F2_R; ++j) {
      const int gy = gyw + j;
      ldrow(gy + 1, In);
      float Vr[2] = {0.f, 0.f};
      const long long rowp = pbase + (long long)gy * nx + gx0;
      if (P.R.vmode == 1) { Vr[0] = Ic[0]; Vr[1] = Ic[1]; }
      else if (P.R.vmode == 2) {
        if (FAST) Pair<float>::ld(P.R.V, rowp, vec, Vr);
        else {
#pragma unroll
          for (int c = 0; c < 2; ++c) Vr[c] = (row_in(gy) && cin[c]) ? __ldg(P.R.V + rowp + c) : 0.f;
        }
      }
      float Iw[2], Ie[2];
      xnbr<0>(Ic, Iw[0], Ie[0]);
      xnbr<1>(Ic, Iw[1], Ie[1]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const Coef k = coef_at(c, gy);
        const float I0 = Ic[c];
        const float w = k.xl != 0.f ? Iw[c] : I0, e = k.xr != 0.f ? Ie[c] : I0;
        const float s = k.yl != 0.f ? Ip[c] : I0, n = k.yr != 0.f ? In[c] : I0;
        const bool in = row_in(gy) && cin[c];
        b[j][c] = in ? rhs_from(k, I0, w, e, s, n, Vr[c], P.R.av) : 0.f;
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) { Ip[c] = Ic[c]; Ic[c] = In[c]; }
    }
  }

  // ---------------------------------------------------------------- up: add P e_c
  if (!DOWN) {
    const long long cplane = (long long)P.ncx * P.ncy;
    const float* xcp = P.xc + (long long)iz * cplane;
    if (FAST) {
      // parents of my columns: Ix = gx0/2 (col 0 leans on Ix-1, col 1 on Ix+1), weights 3/4, 1/4
      const int Ix = gx0 >> 1;
      const int Jw = (gyw >> 1) - 1;  // first coarse row needed
      float cv[F2_R / 2 + 2][3];
#pragma unroll
      for (int q = 0; q < F2_R / 2 + 2; ++q) {
        const float v = __ldg(xcp + (long long)(Jw + q) * P.ncx + Ix);
        cv[q][1] = v;
        cv[q][0] = __shfl_up_sync(FULL, v, 1);
        cv[q][2] = __shfl_down_sync(FULL, v, 1);
      }
#pragma unroll
      for (int j = 0; j < F2_R; ++j) {
        const int q = (j >> 1) + 1;
        const int qn = (j & 1) ? q + 1 : q - 1;
        // bilerp(a=(Iy,Ix), b=(Iy,Jx), c=(Jy,Ix), d=(Jy,Jx)) as ptaps/bilerp order it
        x[j][0] = __fadd_rn(x[j][0], bilerp(cv[q][1], cv[q][0], cv[qn][1], cv[qn][0], 0.25f, 0.25f));
        x[j][1] = __fadd_rn(x[j][1], bilerp(cv[q][1], cv[q][2], cv[qn][1], cv[qn][2], 0.25f, 0.25f));
      }
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        long long Ix, Jx;
        float tx;
        ptaps(P.tx, gx0 + c, Ix, Jx, tx);
#pragma unroll
        for (int j = 0; j < F2_R; ++j) {
          const int gy = gyw + j;
          if (!(cin[c] && row_in(gy))) continue;
          long long Iy, Jy;
          float ty;
          ptaps(P.ty, gy, Iy, Jy, ty);
          const float e = bilerp(__ldg(xcp + Iy * P.ncx + Ix), __ldg(xcp + Iy * P.ncx + Jx),
                                 __ldg(xcp + Jy * P.ncx + Ix), __ldg(xcp + Jy * P.ncx + Jx), tx, ty);
          x[j][c] = __fadd_rn(x[j][c], e);
        }
      }
    }
  }

  // ---------------------------------------------------------------- row exchange
  float sv[2], nv[2];
  auto exchange = [&](int buf) {
    sh_top[buf][warp][lane] = make_float2(x[0][0], x[0][1]);
    sh_bot[buf][warp][lane] = make_float2(x[F2_R - 1][0], x[F2_R - 1][1]);
    __syncthreads();
    const float2 s2 = warp > 0 ? sh_bot[buf][warp - 1][lane] : make_float2(x[0][0], x[0][1]);
    const float2 n2 = warp < F2_W - 1 ? sh_top[buf][warp + 1][lane] : make_float2(x[F2_R - 1][0], x[F2_R - 1][1]);
    sv[0] = s2.x; sv[1] = s2.y; nv[0] = n2.x; nv[1] = n2.y;
  };

  // one cell update of column C (static) in row j (static)
  auto update = [&](auto Cc, auto Jc) {
    constexpr int C = decltype(Cc)::value;
    constexpr int j = decltype(Jc)::value;
    float w, e;
    xnbr<C>(x[j], w, e);
    const float xc = x[j][C];
    const float s = j > 0 ? x[j - 1][C] : sv[C];
    const float n = j < F2_R - 1 ? x[j + 1][C] : nv[C];
    if (FAST) {
      const float r = __fsub_rn(b[j][C], apply2d(kint, alpha, xc, w, e, s, n));
      x[j][C] = __fmaf_rn(r, invDint, xc);  // == gs_update(xc, r, D_interior)
    } else {
      const int gy = gyw + j;
      if (cint[C] && col_interior(L.ay, gy)) {
        const float r = __fsub_rn(b[j][C], apply2d(kint, alpha, xc, w, e, s, n));
        x[j][C] = __fmaf_rn(r, invDint, xc);
      } else if (cin[C] && row_in(gy)) {
        const Coef k = coef_at(C, gy);
        const float ww = k.xl != 0.f ? w : xc, ee = k.xr != 0.f ? e : xc;
        const float ss = k.yl != 0.f ? s : xc, nn = k.yr != 0.f ? n : xc;
        const float r = __fsub_rn(b[j][C], apply2d(k, alpha, xc, ww, ee, ss, nn));
        x[j][C] = gs_update(xc, r, k.diag(alpha));
      }
    }
  };

  // ---------------------------------------------------------------- nu sweeps
#pragma unroll 1
  for (int hs = 0; hs < 2 * NU; ++hs) {
    const int color = hs & 1;
    exchange(hs & 1);
    const int a0 = (color + gyw + (int)(zg & 1)) & 1;  // active column of row 0
    if (a0 == 0) static_for<F2_R>([&](auto J) { update(IC<(decltype(J)::value & 1)>{}, J); });
    else static_for<F2_R>([&](auto J) { update(IC<((decltype(J)::value & 1) ^ 1)>{}, J); });
  }

  // ---------------------------------------------------------------- residual, row pair by row pair
  exchange((2 * NU) & 1);
  const int lx0 = 2 * lane;     // local column of c = 0 (c = 1 shares interior-ness: H even)
  const int ly0 = warp * F2_R;  // local row of j = 0
  auto resid = [&](auto Jc, auto Cc) -> float {
    constexpr int j = decltype(Jc)::value;
    constexpr int c = decltype(Cc)::value;
    const int gy = gyw + j;
    float w, e;
    xnbr<c>(x[j], w, e);
    const float xc = x[j][c];
    const float s = j > 0 ? x[j - 1][c] : sv[c];
    const float n = j < F2_R - 1 ? x[j + 1][c] : nv[c];
    if (FAST) return __fsub_rn(b[j][c], apply2d(kint, alpha, xc, w, e, s, n));
    const Coef k = coef_at(c, gy);
    const float ww = k.xl != 0.f ? w : xc, ee = k.xr != 0.f ? e : xc;
    const float ss = k.yl != 0.f ? s : xc, nn = k.yr != 0.f ? n : xc;
    return (row_in(gy) && cin[c]) ? __fsub_rn(b[j][c], apply2d(k, alpha, xc, ww, ee, ss, nn)) : 0.f;
  };
  double sr = 0.0, sb = 0.0;
  const long long cplane = (long long)P.ncx * P.ncy;
  float* bcp = DOWN ? P.bc + (long long)iz * cplane : nullptr;
  const bool xin_tile = lx0 >= H && lx0 < F2_COLS - H;
  static_for<F2_R / 2>([&](auto JP) {
    constexpr int j0 = 2 * decltype(JP)::value;
    float r[2][2];
    r[0][0] = resid(IC<j0>{}, IC<0>{});
    r[0][1] = resid(IC<j0>{}, IC<1>{});
    r[1][0] = resid(IC<j0 + 1>{}, IC<0>{});
    r[1][1] = resid(IC<j0 + 1>{}, IC<1>{});
    const int gy0 = gyw + j0;  // even
    const bool yin0 = ly0 + j0 >= H && ly0 + j0 < F2_ROWS - H;  // rows j0, j0+1 share it (H even)
    if (DOWN) {
      if (FAST) {
        // volume-weighted child average of 2 x 2 full cells: weight 0.5 * 0.5 each
        if (xin_tile && yin0) {
          const float w = rw3(1.f, 0.5f, 0.5f);
          float acc = 0.f;
          acc = __fmaf_rn(w, r[0][0], acc);
          acc = __fmaf_rn(w, r[0][1], acc);
          acc = __fmaf_rn(w, r[1][0], acc);
          acc = __fmaf_rn(w, r[1][1], acc);
          bcp[(long long)(gy0 >> 1) * P.ncx + (gx0 >> 1)] = acc;
        }
      } else {
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
          if (P.ty.coarsened && dj == 1) break;  // a coarse row takes both fine rows
          const int gyr = gy0 + dj;
          const int J = P.ty.coarsened ? (gyr >> 1) : gyr;
          const int nyc = P.ty.coarsened ? 2 : 1;
          if (gyr < 0 || J >= P.ncy || !(xin_tile && yin0)) continue;
          if (P.tx.coarsened) {
            const int I = gx0 >> 1;
            if (gx0 < 0 || I >= P.ncx) continue;
            float acc = 0.f;
#pragma unroll
            for (int dy = 0; dy < 2; ++dy) {
              if (dy >= nyc || gyr + dy >= L.ny) break;
              const float wy = rweight(P.ty, gyr + dy);
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                if (gx0 + c >= L.nx) break;
                acc = __fmaf_rn(rw3(1.f, wy, rweight(P.tx, gx0 + c)), r[dj + dy][c], acc);
              }
            }
            bcp[(long long)J * P.ncx + I] = acc;
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int I = gx0 + c;
              if (I < 0 || I >= P.ncx) continue;
              float acc = 0.f;
#pragma unroll
              for (int dy = 0; dy < 2; ++dy) {
                if (dy >= nyc || gyr + dy >= L.ny) break;
                acc = __fmaf_rn(rw3(1.f, rweight(P.ty, gyr + dy), 1.f), r[dj + dy][c], acc);
              }
              bcp[(long long)J * P.ncx + I] = acc;
            }
          }
        }
      }
    } else if (xin_tile && yin0) {
#pragma unroll
      for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if (cin[c] && row_in(gy0 + dj)) {
            sr += (double)r[dj][c] * (double)r[dj][c];
            sb += (double)b[j0 + dj][c] * (double)b[j0 + dj][c];
          }
    }
  });
  if (!DOWN && P.partials) {
    block_sum2(sr, sb);
    if (threadIdx.x == 0)
      P.partials[((long long)iz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = make_double2(sr, sb);
  }

  // ---------------------------------------------------------------- store x (tile interior)
  if (xin_tile) {
#pragma unroll
    for (int j = 0; j < F2_R; ++j) {
      const int gy = gyw + j;
      if (!(ly0 + j >= H && ly0 + j < F2_ROWS - H) || !row_in(gy)) continue;
      float* o = P.xout + pbase + (long long)gy * nx + gx0;
      if (FAST && vec) {
        *reinterpret_cast<float2*>(o) = make_float2(x[j][0], x[j][1]);
      } else {
        if (cin[0]) o[0] = x[j][0];
        if (cin[1]) o[1] = x[j][1];
      }
    }
  }
}

template <int NU, bool DOWN, int MODE, typename TI>
__global__ void __launch_bounds__(256, 2) k_pass2d(Pass2D P) {
  constexpr int H = halo2(NU);
  constexpr int TXI = F2_COLS - 2 * H, TYI = F2_ROWS - 2 * H;
  __shared__ float2 sh_top[2][F2_W][32];
  __shared__ float2 sh_bot[2][F2_W][32];
  // a tile whose cells (halo included) are all >= 2 cells from the low faces and >= 7 from the
  // high faces has regular coefficients and regular transfer taps (no partial cells in reach)
  const int gxa = blockIdx.x * TXI - H, gya = blockIdx.y * TYI - H;
  const bool fast = P.fast_ok && gxa >= 2 && gxa + F2_COLS - 1 <= P.L.nx - 7 && gya >= 2 &&
                    gya + F2_ROWS - 1 <= P.L.ny - 7;
  if (fast) pass2d_body<NU, DOWN, MODE, TI, true>(P, sh_top, sh_bot);
  else pass2d_body<NU, DOWN, MODE, TI, false>(P, sh_top, sh_bot);
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
bool fusable2d(const Level& L, const Level& C, const gdp_opts& o) {
  const bool nu_ok = o.nu_pre >= 1 && o.nu_pre <= 2 && o.nu_post >= 1 && o.nu_post <= 2;
  return nu_ok && o.fused && L.K.az.k == 0.f && L.K.az.kr == 0.f && L.K.az.kl == 0.f && !C.tz.coarsened;
}

template <bool DOWN, int MODE, typename TI>
static void launch2d_t(int nu, const Pass2D& P, dim3 g, cudaStream_t s) {
  switch (nu) {
    case 1: k_pass2d<1, DOWN, MODE, TI><<<g, 256, 0, s>>>(P); break;
    case 2: k_pass2d<2, DOWN, MODE, TI><<<g, 256, 0, s>>>(P); break;
    default: break;
  }
}

static dim3 grid2d(int nu, const LevelK& L) {
  const int H = halo2(nu);
  const int TXI = F2_COLS - 2 * H, TYI = F2_ROWS - 2 * H;
  return dim3((L.nx + TXI - 1) / TXI, (L.ny + TYI - 1) / TYI, L.nzl);
}

int fused_tiles_per_plane(int nu, const LevelK& L) {
  dim3 g = grid2d(nu, L);
  return g.x * g.y;
}

static void launch2d(bool down, int nu, const Pass2D& P, int mode, int tI, cudaStream_t s) {
  dim3 g = grid2d(nu, P.L);
  const double N = (double)P.L.nx * P.L.ny * P.L.nzl, Nc = (double)P.ncx * P.ncy * P.L.nzl;
  const double bytes = N * ((P.zero_x ? 4.0 : 8.0) + rhs_bytes(mode, tI, P.R)) + Nc * 4.0;
  ProfScope ps(down ? KC_DOWN2D : KC_UP2D, bytes, s);
  if (down) {
    if (mode == RHS_B) launch2d_t<true, RHS_B, float>(nu, P, g, s);
    else if (tI == 0) launch2d_t<true, RHS_G, uint8_t>(nu, P, g, s);
    else launch2d_t<true, RHS_G, float>(nu, P, g, s);
  } else {
    if (mode == RHS_B) launch2d_t<false, RHS_B, float>(nu, P, g, s);
    else if (tI == 0) launch2d_t<false, RHS_G, uint8_t>(nu, P, g, s);
    else launch2d_t<false, RHS_G, float>(nu, P, g, s);
  }
}

void fused_down2d(const Level& L, const Level& C, const float* xin, float* xout, const RhsK& R,
                  int mode, int tI, int nu, bool zero_x, cudaStream_t s) {
  Pass2D P{};
  P.L = L.K; P.xin = xin; P.xout = xout; P.R = R; P.zero_x = zero_x ? 1 : 0;
  P.fast_ok = C.tx.coarsened && C.ty.coarsened;
  P.tx = C.tx; P.ty = C.ty; P.ncx = C.nx; P.ncy = C.ny;
  P.bc = C.b;
  launch2d(true, nu, P, mode, tI, s);
}

void fused_up2d(const Level& L, const Level& C, const float* xin, float* xout, const RhsK& R,
                int mode, int tI, int nu, double2* partials, cudaStream_t s) {
  Pass2D P{};
  P.L = L.K; P.xin = xin; P.xout = xout; P.R = R; P.zero_x = 0;
  P.fast_ok = C.tx.coarsened && C.ty.coarsened;
  P.tx = C.tx; P.ty = C.ty; P.ncx = C.nx; P.ncy = C.ny;
  P.xc = C.x;
  P.partials = partials;
  launch2d(false, nu, P, mode, tI, s);
}

}  // namespace gdp
