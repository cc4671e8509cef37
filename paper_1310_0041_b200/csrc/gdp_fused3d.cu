// gdp_fused3d.cu — fused 3D sweeps (levels with z links: phase 1, Eq. 1), sm_100a.
//
// One HBM pass = one full red-black Gauss-Seidel sweep of a level, optionally preceded by the
// prolongated coarse correction and followed by the residual (restricted to the coarse level,
// or fp64 norms of the final iterate).  This is the paper's streaming pass over a sliding
// window of slices done on chip: a CTA owns an in-plane tile (128 x 32
// cells, 4-cell halo) and marches along z through a chunk of planes (3 recomputed planes on
// each side), with a ring of six planes of x and b in shared memory.  Per step, with p the
// plane being prefetched:
//     stage 1 (colour 0) updates plane p-2, stage 2 (colour 1) updates plane p-3,
//     the tail computes the residual of plane p-4 and stores its x,
// which is exactly the reference schedule's two half-sweeps (a point of one colour depends
// only on the other colour).
// Each of the 512 threads owns a 2 (x) x 4 (y) block of every plane: in a stage it updates the
// four cells of the active colour (one per row), reading its own block, the two rows and the
// columns around it, the planes above and below, and b from shared memory.  The tail's block
// is exactly two coarse cells, so restriction needs no extra pass.  Per-cell arithmetic is the
// reference one (apply_from / gs_update order, rw3, bilerp) -> bit-identical iterates.
#include <type_traits>

#include "gdp_internal.h"

namespace gdp {

constexpr int S3_X = 128, S3_Y = 64;      // tile incl. halo
constexpr int S3_HX = 4, S3_HY = 4;       // halo >= 3 (2 half-sweeps + residual), even
constexpr int S3_XI = S3_X - 2 * S3_HX;   // 120
constexpr int S3_YI = S3_Y - 2 * S3_HY;   // 56
constexpr int S3_RING = 6;
constexpr int S3_ZC = 32;                 // planes stored per CTA (z chunk)
constexpr int S3_THREADS = 512;           // 64 column pairs x 8 row octets
constexpr int S3_R = 8;                   // rows per thread

struct Pass3D {
  LevelK L;
  const float* xin;      // x before the pass (ignored if zero_x)
  float* xout;           // x after the pass
  const float* b;        // rhs of the level (explicit)
  int zero_x;
  XferAxis tx, ty;       // fine -> coarse, in-plane only (z not coarsened)
  int ncx, ncy;
  float* bc;             // tail 1: coarse rhs
  const float* xc;       // prolong: coarse correction
  double2* partials;     // tail 2: per CTA (sum r^2, sum b^2)
};

struct Smem3D {
  float x[S3_RING][S3_Y][S3_X];
};
constexpr size_t SMEM3D = sizeof(Smem3D);

template <int TAIL, bool PROLONG>
__global__ void __launch_bounds__(S3_THREADS, 1) k_sweep3d(Pass3D P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem3D& S = *reinterpret_cast<Smem3D*>(smem_raw);
  const LevelK& L = P.L;
  const int tid = threadIdx.x;
  const int gxa = blockIdx.x * S3_XI - S3_HX, gya = blockIdx.y * S3_YI - S3_HY;  // multiples of 4 / even
  const long long nx = L.nx, plane = (long long)L.nx * L.ny;
  const int nzl = L.nzl;
  const float alpha = L.alpha;
  const int p_lo = blockIdx.z * S3_ZC, p_hi = min(p_lo + S3_ZC, nzl);
  const int first = max(p_lo - 3, 0), last = min(p_hi + 3, nzl);

  // my block: columns lx0, lx0+1, rows ly0 .. ly0+7
  const int lx0 = 2 * (tid & 63), ly0 = S3_R * (tid >> 6);
  const int gx0 = gxa + lx0, gy0 = gya + ly0;
  const bool cin0 = gx0 >= 0 && gx0 < L.nx, cin1 = gx0 + 1 >= 0 && gx0 + 1 < L.nx;
  auto cinh = [&](int h) { return h ? cin1 : cin0; };
  auto rinr = [&](int r) { return gy0 + r >= 0 && gy0 + r < L.ny; };
  const bool full = cin0 && cin1 && gy0 >= 0 && gy0 + S3_R - 1 < L.ny;
  const bool vec = (L.nx & 1) == 0;
  Coef kint;
  kint.xl = L.ax.k; kint.xr = L.ax.k; kint.yl = L.ay.k; kint.yr = L.ay.k; kint.zl = L.az.k; kint.zr = L.az.k;
  const float Dint = kint.diag(alpha), invDint = __frcp_rn(Dint);
  // inner block: every cell has the regular in-plane links and is off the tile border
  const bool inner = gx0 >= 1 && gx0 + 1 <= L.ax.n - 3 && gy0 >= 1 && gy0 + S3_R - 1 <= L.ay.n - 3 && lx0 >= 1 &&
                     lx0 + 1 <= S3_X - 2 && ly0 >= 1 && ly0 + S3_R - 1 <= S3_Y - 2;
  // edge neighbours (rows / columns outside my block, inside the tile)
  const int offW = max(lx0 - 1, 0) - lx0, offE = min(lx0 + 2, S3_X - 1) - lx0;
  const int offS = (max(ly0 - 1, 0) - ly0) * S3_X, offN = (min(ly0 + S3_R, S3_Y - 1) - ly0) * S3_X;

  for (int i = tid; i < S3_RING * S3_Y * S3_X; i += S3_THREADS) (&S.x[0][0][0])[i] = 0.f;

  // ---- x of a plane's block: prefetch into registers, publish into the ring
  float2 px[S3_R];
  const long long gbase = (long long)gy0 * nx + gx0;
  auto prefetch = [&](int p) {
    const float* src = P.xin + (long long)p * plane + gbase;
#pragma unroll
    for (int r = 0; r < S3_R; ++r) {
      if (P.zero_x) px[r] = make_float2(0.f, 0.f);
      else if (full && vec) px[r] = __ldg(reinterpret_cast<const float2*>(src + (long long)r * nx));
      else {
        const bool ri = rinr(r);
        px[r] = make_float2((ri && cin0) ? __ldg(src + (long long)r * nx) : 0.f,
                            (ri && cin1) ? __ldg(src + (long long)r * nx + 1) : 0.f);
      }
    }
  };
  auto publish = [&](int s) {
#pragma unroll
    for (int r = 0; r < S3_R; ++r) *reinterpret_cast<float2*>(&S.x[s][ly0 + r][lx0]) = px[r];
  };
  // ---- b of my cells, fetched one step before use
  auto fetch_b1 = [&](int p, int c, float (&dst)[S3_R]) {  // the colour-c cell of each row
    const float* bp = P.b + (long long)p * plane + gbase;
    const int a0 = (c + ly0 + (int)((L.z0 + p) & 1)) & 1;
#pragma unroll
    for (int r = 0; r < S3_R; ++r) {
      const int h = (a0 + r) & 1;
      dst[r] = (full || (rinr(r) && cinh(h))) ? __ldg(bp + (long long)r * nx + h) : 0.f;
    }
  };
  auto fetch_b2 = [&](int p, float2 (&dst)[S3_R]) {  // both cells of each row
    const float* bp = P.b + (long long)p * plane + gbase;
#pragma unroll
    for (int r = 0; r < S3_R; ++r) {
      if (full && vec) dst[r] = __ldg(reinterpret_cast<const float2*>(bp + (long long)r * nx));
      else dst[r] = make_float2((rinr(r) && cin0) ? __ldg(bp + (long long)r * nx) : 0.f,
                                (rinr(r) && cin1) ? __ldg(bp + (long long)r * nx + 1) : 0.f);
    }
  };

  auto coef_at = [&](int r, int h, float czl, float czr) {
    Coef k;
    k.xl = cl(L.ax, gx0 + h); k.xr = cr(L.ax, gx0 + h);
    k.yl = cl(L.ay, gy0 + r); k.yr = cr(L.ay, gy0 + r);
    k.zl = czl; k.zr = czr;
    return k;
  };
  // (A x) of my cell (r, h) of the plane with slot base X (own block origin), Xd / Xu below / above
  auto ax_at = [&](const float* X, const float* Xd, const float* Xu, int r, int h, const Coef& k) -> float {
    const int o = r * S3_X + h;
    const float xc = X[o];
    const float w = X[h ? o - 1 : o + offW];
    const float e = X[h ? o - 1 + offE : o + 1];
    const float sv = X[r ? o - S3_X : h + offS];
    const float nv = X[r < S3_R - 1 ? o + S3_X : h + offN];
    return apply_from(k, alpha, xc, w, e, sv, nv, Xd[o], Xu[o]);
  };

  // one half-sweep of colour c on the plane in slot s (global z zg), b of the active cells in bv
  auto stage = [&](int s, int sd, int su, long long zg, int c, const float (&bv)[S3_R]) {
    const float czl = cl(L.az, zg), czr = cr(L.az, zg);
    const bool fast = inner && czl == L.az.k && czr == L.az.k;
    float* X = &S.x[s][ly0][lx0];
    const float* Xd = &S.x[sd][ly0][lx0];
    const float* Xu = &S.x[su][ly0][lx0];
    const int a0 = (c + ly0 + (int)(zg & 1)) & 1;  // active column of row 0 (gx0 even)
    auto run = [&](auto A0) {
      constexpr int a = decltype(A0)::value;
      if (fast) {
#pragma unroll
        for (int r = 0; r < S3_R; ++r) {
          const int h = (a + r) & 1, o = r * S3_X + h;
          const float xc = X[o];
          X[o] = __fmaf_rn(__fsub_rn(bv[r], ax_at(X, Xd, Xu, r, h, kint)), invDint, xc);  // == gs_update
        }
      } else {
#pragma unroll
        for (int r = 0; r < S3_R; ++r) {
          const int h = (a + r) & 1, o = r * S3_X + h;
          const int ly = ly0 + r, lx = lx0 + h;
          if (!(rinr(r) && cinh(h))) continue;  // out-of-domain cells stay 0
          if (lx == 0 || lx == S3_X - 1 || ly == 0 || ly == S3_Y - 1) continue;  // tile border: stale
          const Coef k = coef_at(r, h, czl, czr);
          const float xc = X[o];
          const float D = k.diag(alpha);
          X[o] = __fmaf_rn(__fsub_rn(bv[r], ax_at(X, Xd, Xu, r, h, k)), D == Dint ? invDint : __frcp_rn(D), xc);
        }
      }
    };
    if (a0 == 0) run(std::integral_constant<int, 0>{});
    else run(std::integral_constant<int, 1>{});
  };

  double sr = 0.0, sbb = 0.0;
  // tile interior: my columns together (HX even), rows one by one (row pairs together, HY even)
  const bool cint = lx0 >= S3_HX && lx0 < S3_X - S3_HX;
  auto rint = [&](int r) { return ly0 + r >= S3_HY && ly0 + r < S3_Y - S3_HY; };
  auto tail = [&](int s, int sd, int su, int p, const float2 (&bt)[S3_R]) {
    const long long zg = L.z0 + p;
    const float czl = cl(L.az, zg), czr = cr(L.az, zg);
    const bool fast = inner && czl == L.az.k && czr == L.az.k;
    const float* X = &S.x[s][ly0][lx0];
    const float* Xd = &S.x[sd][ly0][lx0];
    const float* Xu = &S.x[su][ly0][lx0];
    auto res = [&](int r, int h) {
      const float bv = h ? bt[r].y : bt[r].x;
      return __fsub_rn(bv, ax_at(X, Xd, Xu, r, h, fast ? kint : coef_at(r, h, czl, czr)));
    };
    if (TAIL == 1 && cint) {
      // my block = coarse cells (gx0/2, gy0/2 + j), j < 4 (children rows 2j, 2j+1; fy outer, fx inner)
      float* bcp = P.bc + (long long)p * P.ncx * P.ncy;
      const int I = gx0 >> 1;
      const float wx0 = rweight(P.tx, gx0), wx1 = rweight(P.tx, gx0 + 1);
#pragma unroll
      for (int j = 0; j < S3_R / 2; ++j) {
        const int J = (gy0 >> 1) + j;
        if (!rint(2 * j) || !rinr(2 * j) || !cin0 || I >= P.ncx || J >= P.ncy) continue;
        float acc = 0.f;
#pragma unroll
        for (int dy = 0; dy < 2; ++dy) {
          if (!rinr(2 * j + dy)) break;
          const float wy = rweight(P.ty, gy0 + 2 * j + dy);
          acc = __fmaf_rn(rw3(1.f, wy, wx0), res(2 * j + dy, 0), acc);
          if (cin1) acc = __fmaf_rn(rw3(1.f, wy, wx1), res(2 * j + dy, 1), acc);
        }
        bcp[(long long)J * P.ncx + I] = acc;
      }
    } else if (TAIL == 2 && P.partials && cint) {
#pragma unroll
      for (int r = 0; r < S3_R; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!(rint(r) && rinr(r) && cinh(h))) continue;
          const float rr = res(r, h);
          const float bv = h ? bt[r].y : bt[r].x;
          sr += (double)rr * (double)rr;
          sbb += (double)bv * (double)bv;
        }
    }
    if (cint) {  // store the interior rows of my block of plane p
      float* o = P.xout + (long long)p * plane + gbase;
#pragma unroll
      for (int r = 0; r < S3_R; ++r) {
        if (!rint(r)) continue;
        const float2 v = *reinterpret_cast<const float2*>(X + r * S3_X);
        if (full && vec) *reinterpret_cast<float2*>(o + (long long)r * nx) = v;
        else if (rinr(r)) {
          if (cin0) o[(long long)r * nx] = v.x;
          if (cin1) o[(long long)r * nx + 1] = v.y;
        }
      }
    }
  };

  // x += P e_c on my block of the plane in slot s (coarse plane = p: z is not coarsened)
  long long pI[2] = {0, 0}, pJ[2] = {0, 0};
  float pt[2] = {0.f, 0.f};
  if (PROLONG) {
#pragma unroll
    for (int h = 0; h < 2; ++h) ptaps(P.tx, gx0 + h, pI[h], pJ[h], pt[h]);
  }
  auto prolong = [&](int s, int p) {
    const float* xcp = P.xc + (long long)p * P.ncx * P.ncy;
#pragma unroll
    for (int r = 0; r < S3_R; ++r) {
      if (!rinr(r)) continue;
      long long Iy, Jy;
      float ty;
      ptaps(P.ty, gy0 + r, Iy, Jy, ty);
      const float* rI = xcp + Iy * P.ncx;
      const float* rJ = xcp + Jy * P.ncx;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!cinh(h)) continue;
        const float e = bilerp(__ldg(rI + pI[h]), __ldg(rI + pJ[h]), __ldg(rJ + pI[h]), __ldg(rJ + pJ[h]), pt[h], ty);
        float& v = S.x[s][ly0 + r][lx0 + h];
        v = __fadd_rn(v, e);
      }
    }
  };

  // ---- the march: plane p is prefetched at step p and published at its end;
  // stage 1 covers [p_lo-2, p_hi+2), stage 2 [p_lo-1, p_hi+1), the tail [p_lo, p_hi)
  const int s1lo = max(p_lo - 2, 0), s1hi = min(p_hi + 2, nzl);
  const int s2lo = max(p_lo - 1, 0), s2hi = min(p_hi + 1, nzl);
  float b1[S3_R], b2[S3_R];
  float2 bt[S3_R];
  __syncthreads();
  prefetch(first);
  int sp = first % S3_RING;  // slot of plane p
  publish(sp);
  if (PROLONG) prolong(sp, first);
  auto dec = [](int s, int k) { s -= k; return s < 0 ? s + S3_RING : s; };
  for (int p = first + 1; p <= last + 3; ++p) {
    sp = sp + 1 == S3_RING ? 0 : sp + 1;
    if (p < last) prefetch(p);
    __syncthreads();
    // stage 1 on plane p-2 (its upper neighbour p-1 was published and prolongated last step)
    if (p - 2 >= s1lo && p - 2 < s1hi) stage(dec(sp, 2), dec(sp, 3), dec(sp, 1), L.z0 + p - 2, 0, b1);
    if (p - 1 >= s1lo && p - 1 < s1hi) fetch_b1(p - 1, 0, b1);
    __syncthreads();
    if (p - 3 >= s2lo && p - 3 < s2hi) stage(dec(sp, 3), dec(sp, 4), dec(sp, 2), L.z0 + p - 3, 1, b2);
    if (p - 2 >= s2lo && p - 2 < s2hi) fetch_b1(p - 2, 1, b2);
    __syncthreads();
    if (p - 4 >= p_lo && p - 4 < p_hi) tail(dec(sp, 4), dec(sp, 5), dec(sp, 3), p - 4, bt);
    if (TAIL != 0 && p - 3 >= p_lo && p - 3 < p_hi) fetch_b2(p - 3, bt);
    if (p < last) {
      publish(sp);
      if (PROLONG) prolong(sp, p);
    }
  }
  if (TAIL == 2 && P.partials) {
    block_sum2(sr, sbb);
    if (tid == 0)
      P.partials[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = make_double2(sr, sbb);
  }
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
bool fusable3d(const Level& L, const Level& C, const gdp_opts& o) {
  return (o.fused & 2) && (L.K.az.k != 0.f || L.K.az.kr != 0.f || L.K.az.kl != 0.f) && !C.tz.coarsened &&
         C.tx.coarsened && C.ty.coarsened && L.nzl == L.gz.n /* single slab (no ghost planes) */;
}

int fused3d_tiles(const LevelK& L) {
  return ((L.nx + S3_XI - 1) / S3_XI) * ((L.ny + S3_YI - 1) / S3_YI) * ((L.nzl + S3_ZC - 1) / S3_ZC);
}

template <int TAIL, bool PROLONG>
static void launch3d_t(const Pass3D& P, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sweep3d<TAIL, PROLONG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM3D);
    attr = true;
  }
  dim3 g((P.L.nx + S3_XI - 1) / S3_XI, (P.L.ny + S3_YI - 1) / S3_YI, (P.L.nzl + S3_ZC - 1) / S3_ZC);
  k_sweep3d<TAIL, PROLONG><<<g, S3_THREADS, SMEM3D, s>>>(P);
}

// one fused sweep: tail 0 none, 1 restrict into C.b, 2 norms into partials
void fused_sweep3d(const Level& L, const Level& C, const float* xin, float* xout, const float* b,
                   bool zero_x, bool prolong, int tail, double2* partials, cudaStream_t s) {
  Pass3D P{};
  P.L = L.K; P.xin = xin; P.xout = xout; P.b = b; P.zero_x = zero_x ? 1 : 0;
  P.tx = C.tx; P.ty = C.ty; P.ncx = C.nx; P.ncy = C.ny;
  P.bc = C.b; P.xc = C.x; P.partials = partials;
  const double N = (double)L.nx * L.ny * L.nzl, Nc = (double)C.nx * C.ny * C.nzl;
  const double bytes = N * ((zero_x ? 4.0 : 8.0) + 4.0) + ((tail == 1 || prolong) ? Nc * 4.0 : 0.0);
  ProfScope ps(tail == 1 || !prolong ? KC_DOWN3D : KC_UP3D, bytes, s, N);
  if (prolong) {
    if (tail == 2) launch3d_t<2, true>(P, s);
    else launch3d_t<0, true>(P, s);
  } else {
    if (tail == 1) launch3d_t<1, false>(P, s);
    else if (tail == 2) launch3d_t<2, false>(P, s);
    else launch3d_t<0, false>(P, s);
  }
}

}  // namespace gdp
