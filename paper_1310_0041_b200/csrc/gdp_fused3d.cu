// gdp_fused3d.cu — fused 3D level passes (levels with z links: phase 1, Eq. 1), sm_100a.
//
// One HBM pass = one full red-black Gauss-Seidel sweep of a level, optionally preceded by
// the prolongated coarse correction and followed by the residual (restriction to the coarse
// level, or fp64 norms of the final iterate).  This is the paper's streaming pass over a
// sliding window of slices done on chip: a CTA owns an in-plane tile
// (128 x 32 cells with a 4-cell halo) and marches along z through its slab, keeping a ring of
// six planes in shared memory.  Per step t:
//     plane t+1 is prefetched into registers,
//     stage 1 (colour 0) updates plane t-1, stage 2 (colour 1) updates plane t-2,
//     the tail computes the residual of plane t-3 and stores its x.
// A point of one colour depends only on the other colour, so this wavefront order performs
// exactly the reference schedule's two half-sweeps (colour 0 everywhere, then colour 1).
// Planes are stored checkerboard-split (one array per colour, index x/2) so that the six
// neighbours of an active cell are read without bank conflicts.  Every cell evaluates the
// reference arithmetic of gdp_device.cuh (coefs, apply_from, gs_update, rweight, ptaps,
// bilerp) -> bit-identical to the one-kernel-per-half-sweep schedule.
#include "gdp_internal.h"

namespace gdp {

constexpr int T3_X = 128, T3_Y = 32;      // tile incl. halo
constexpr int T3_HX = 4, T3_HY = 4;       // halo >= 3 (2 half-sweeps + residual), even
constexpr int T3_XI = T3_X - 2 * T3_HX;   // 120
constexpr int T3_YI = T3_Y - 2 * T3_HY;   // 24
constexpr int T3_RING = 6;                // planes t-4 .. t+1
constexpr int T3_HALF = T3_X / 2;         // cells of one colour per row
constexpr int T3_ZC = 32;                 // planes stored per CTA (z chunk); +3 recomputed each side

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
  double2* partials;     // tail 2: per tile (sum r^2, sum b^2)
};

struct Smem3D {
  float c[T3_RING][2][T3_Y][T3_HALF];  // [slot][colour][row][x/2]
};
constexpr size_t SMEM3D = sizeof(Smem3D);

__device__ __forceinline__ int slot_of(int p) { return ((p % T3_RING) + T3_RING) % T3_RING; }

template <int TAIL, bool PROLONG>
__global__ void __launch_bounds__(256, 2) k_pass3d(Pass3D P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& R = reinterpret_cast<Smem3D*>(smem_raw)->c;
  const LevelK& L = P.L;
  const int tid = threadIdx.x;
  const int gxa = blockIdx.x * T3_XI - T3_HX, gya = blockIdx.y * T3_YI - T3_HY;  // both even
  const long long nx = L.nx, plane = (long long)L.nx * L.ny;
  const int nzl = L.nzl;
  const float alpha = L.alpha;
  // z chunk: planes [p_lo, p_hi) are finished and stored; the march covers 3 more on each side
  const int p_lo = blockIdx.z * T3_ZC, p_hi = min(p_lo + T3_ZC, nzl);
  const int first = max(p_lo - 3, 0), last = min(p_hi + 3, nzl);
  // fast path: every updated cell of the tile has the regular in-plane coefficients
  const bool xy_regular = gxa + 1 >= 1 && gxa + T3_X - 2 <= L.nx - 3 && gya + 1 >= 1 && gya + T3_Y - 2 <= L.ny - 3;
  Coef kint;
  kint.xl = L.ax.k; kint.xr = L.ax.k; kint.yl = L.ay.k; kint.yr = L.ay.k; kint.zl = L.az.k; kint.zr = L.az.k;
  const float invDint = __frcp_rn(kint.diag(alpha));
  auto inside = [&](int gx, int gy) { return gx >= 0 && gx < L.nx && gy >= 0 && gy < L.ny; };

  for (int i = tid; i < T3_RING * 2 * T3_Y * T3_HALF; i += 256) (&R[0][0][0][0])[i] = 0.f;

  // ---- plane loader: 4 quads (4 consecutive cells) per thread, register-prefetched
  const bool vec = (L.nx & 3) == 0;
  float4 pre[4];
  auto load_plane = [&](int p) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = tid + 256 * k, row = idx >> 5, q = idx & 31;
      const int gy = gya + row, gx = gxa + 4 * q;
      const float* src = P.xin + (long long)p * plane + (long long)gy * nx + gx;
      if (P.zero_x) pre[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      else if (vec && gy >= 0 && gy < L.ny && gx >= 0 && gx + 3 < L.nx) pre[k] = __ldg(reinterpret_cast<const float4*>(src));
      else {
        float v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = inside(gx + c, gy) ? __ldg(src + c) : 0.f;
        pre[k] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  };
  auto store_plane = [&](int p) {
    const int s = slot_of(p);
    const int zp = (int)((L.z0 + p) & 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = tid + 256 * k, row = idx >> 5, q = idx & 31;
      const int c0 = (row + zp) & 1;  // colour of cells 4q, 4q+2
      *reinterpret_cast<float2*>(&R[s][c0][row][2 * q]) = make_float2(pre[k].x, pre[k].z);
      *reinterpret_cast<float2*>(&R[s][c0 ^ 1][row][2 * q]) = make_float2(pre[k].y, pre[k].w);
    }
  };

  // x at local (lx, ly) of plane p (any colour)
  auto xat = [&](int p, int lx, int ly) -> float {
    const int zp = (int)((L.z0 + p) & 1);
    return R[slot_of(p)][(lx + ly + zp) & 1][ly][lx >> 1];
  };

  // residual of cell (lx, ly) of plane p (reference arithmetic)
  auto resid = [&](int p, int lx, int ly, float* bval) -> float {
    const int gx = gxa + lx, gy = gya + ly;
    const long long zg = L.z0 + p;
    const Coef k = coefs(L, gx, gy, zg);
    const float xc = xat(p, lx, ly);
    Nbr nb;
    nb.w = k.xl != 0.f ? xat(p, lx - 1, ly) : xc;
    nb.e = k.xr != 0.f ? xat(p, lx + 1, ly) : xc;
    nb.s = k.yl != 0.f ? xat(p, lx, ly - 1) : xc;
    nb.n = k.yr != 0.f ? xat(p, lx, ly + 1) : xc;
    nb.d = k.zl != 0.f ? xat(p - 1, lx, ly) : xc;
    nb.u = k.zr != 0.f ? xat(p + 1, lx, ly) : xc;
    const float bc = __ldg(P.b + (long long)p * plane + (long long)gy * nx + gx);
    if (bval) *bval = bc;
    return __fsub_rn(bc, apply_from(k, alpha, xc, nb.w, nb.e, nb.s, nb.n, nb.d, nb.u));
  };

  // per-thread cell map: rows row0 + 4k (k < 8), column pair (2 pi, 2 pi + 1).  All rows of a
  // thread have the parity of row0, so in a stage the thread updates the same column of its pair
  // in every row.
  const int pi = tid & 63, row0 = tid >> 6;
  const float kz = L.az.k;
  float cxl2[2], cxr2[2];  // x coefficients of columns 2pi, 2pi+1
  bool colin[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    cxl2[h] = cl(L.ax, gxa + 2 * pi + h);
    cxr2[h] = cr(L.ax, gxa + 2 * pi + h);
    colin[h] = gxa + 2 * pi + h >= 0 && gxa + 2 * pi + h < L.nx;
  }
  const float Dint = kint.diag(alpha);
  float* const R0 = &R[0][0][0][0];
  auto colarr = [&](int slot, int colour) { return R0 + (slot * 2 + colour) * (T3_Y * T3_HALF); };

  // b of the next stages, prefetched one step ahead: [k] for rows row0 + 4k
  float bpre1[8], bpre2[8];
  auto fetch_b = [&](int p, int c, float (&dst)[8]) {
    const int zp = (int)((L.z0 + p) & 1);
    const int lx = 2 * pi + ((c + row0 + zp) & 1);
    const int gx = gxa + lx;
    const float* bp = P.b + (long long)p * plane + (long long)(gya + row0) * nx + gx;
    const bool cin = gx >= 0 && gx < L.nx;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int gy = gya + row0 + 4 * k;
      dst[k] = (cin && gy >= 0 && gy < L.ny) ? __ldg(bp + (long long)(4 * k) * nx) : 0.f;
    }
  };

  // one half-sweep of colour c on plane p with its b values in bv[]
  auto stage = [&](int p, int c, const float (&bv)[8]) {
    const int zp = (int)((L.z0 + p) & 1);
    const long long zg = L.z0 + p;
    const int par = (c + row0 + zp) & 1;       // which column of my pair has colour c
    const int lx = 2 * pi + par;
    if (lx == 0 || lx == T3_X - 1) return;      // tile border: stale by construction
    const float* Xo = colarr(slot_of(p), c ^ 1) + pi;
    float* Xc = colarr(slot_of(p), c) + pi;
    const float* Xd = colarr(slot_of(p - 1), c ^ 1) + pi;
    const float* Xu = colarr(slot_of(p + 1), c ^ 1) + pi;
    const int dw = par ? 0 : -1, de = par ? 1 : 0;
    const float czl = cl(L.az, zg), czr = cr(L.az, zg);
    if (xy_regular && czl == kz && czr == kz) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int row = row0 + 4 * k;
        if (row == 0 || row == T3_Y - 1) continue;
        const int o = row * T3_HALF;
        const float xc = Xc[o];
        const float r = __fsub_rn(bv[k], apply_from(kint, alpha, xc, Xo[o + dw], Xo[o + de], Xo[o - T3_HALF],
                                                    Xo[o + T3_HALF], Xd[o], Xu[o]));
        Xc[o] = __fmaf_rn(r, invDint, xc);  // == gs_update(xc, r, D)
      }
      return;
    }
    if (!(par ? colin[1] : colin[0])) return;  // out-of-domain column stays 0
    const float pxl = par ? cxl2[1] : cxl2[0], pxr = par ? cxr2[1] : cxr2[0];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int row = row0 + 4 * k;
      const int gy = gya + row;
      if (row == 0 || row == T3_Y - 1 || gy < 0 || gy >= L.ny) continue;
      const int o = row * T3_HALF;
      Coef kk;
      kk.xl = pxl; kk.xr = pxr;
      kk.yl = cl(L.ay, gy); kk.yr = cr(L.ay, gy);
      kk.zl = czl; kk.zr = czr;
      // absent links have coefficient 0 and finite neighbours: their terms vanish exactly
      const float xc = Xc[o];
      const float r = __fsub_rn(bv[k], apply_from(kk, alpha, xc, Xo[o + dw], Xo[o + de], Xo[o - T3_HALF],
                                                  Xo[o + T3_HALF], Xd[o], Xu[o]));
      const float D = kk.diag(alpha);
      Xc[o] = __fmaf_rn(r, D == Dint ? invDint : __frcp_rn(D), xc);
    }
  };

  // residual of both cells of my pair in row `row` of plane p (cells 2pi + h, h = 0, 1)
  auto resid_pair = [&](int p, int row, float (&rr)[2], float (&bb)[2]) {
    const int zp = (int)((L.z0 + p) & 1);
    const long long zg = L.z0 + p;
    const int gy = gya + row;
    const int c0 = (row + zp) & 1;  // colour of column 2pi
    const int s = slot_of(p), sd = slot_of(p - 1), su = slot_of(p + 1);
    const float czl = cl(L.az, zg), czr = cr(L.az, zg);
    const bool fast = xy_regular && czl == kz && czr == kz;
    const float* bp = P.b + (long long)p * plane + (long long)gy * nx + gxa + 2 * pi;
    const bool rin = gy >= 0 && gy < L.ny;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = c0 ^ h;
      const float* Xo = colarr(s, col ^ 1) + row * T3_HALF + pi;
      const float xc = colarr(s, col)[row * T3_HALF + pi];
      const float w = Xo[h ? 0 : -1], e = Xo[h ? 1 : 0];
      const float sv = Xo[-T3_HALF], nv = Xo[T3_HALF];
      const float d = colarr(sd, col ^ 1)[row * T3_HALF + pi], u = colarr(su, col ^ 1)[row * T3_HALF + pi];
      if (!(rin && colin[h])) { rr[h] = 0.f; bb[h] = 0.f; continue; }
      const float bc = __ldg(bp + h);
      bb[h] = bc;
      Coef kk = kint;
      if (!fast) {
        kk.xl = cxl2[h]; kk.xr = cxr2[h];
        kk.yl = cl(L.ay, gy); kk.yr = cr(L.ay, gy);
        kk.zl = czl; kk.zr = czr;
      }
      rr[h] = __fsub_rn(bc, apply_from(kk, alpha, xc, w, e, sv, nv, d, u));
    }
  };

  double sr = 0.0, sbb = 0.0;
  auto tail = [&](int p) {
    if (TAIL == 1) {
      // residuals of plane p into the slot of plane p + 4 (free until the next plane is
      // stored into it), then the volume-weighted child average per coarse cell
      float* RR = colarr(slot_of(p + 4), 0);  // [T3_Y][T3_X]
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int row = row0 + 4 * k;
        if (row < 2 || row >= T3_Y - 2 || pi == 0 || pi == T3_HALF - 1) continue;
        float rr[2], bb[2];
        resid_pair(p, row, rr, bb);
        *reinterpret_cast<float2*>(RR + row * T3_X + 2 * pi) = make_float2(rr[0], rr[1]);
      }
      __syncthreads();
      float* bcp = P.bc + (long long)p * P.ncx * P.ncy;
      const int sx = P.tx.coarsened ? 2 : 1, sy = P.ty.coarsened ? 2 : 1;
      const int ncl = T3_XI / sx, nrl = T3_YI / sy;
      for (int i = tid; i < ncl * nrl; i += 256) {
        const int cyl = i / ncl, cxl = i % ncl;
        const int gx0 = gxa + T3_HX + sx * cxl, gy0 = gya + T3_HY + sy * cyl;
        if (gx0 >= L.nx || gy0 >= L.ny) continue;
        const int I = P.tx.coarsened ? gx0 >> 1 : gx0, J = P.ty.coarsened ? gy0 >> 1 : gy0;
        float acc = 0.f;
        for (int dy = 0; dy < sy && gy0 + dy < L.ny; ++dy) {
          const float wy = rweight(P.ty, gy0 + dy);
          for (int dx = 0; dx < sx && gx0 + dx < L.nx; ++dx) {
            const int gx = gx0 + dx, gy = gy0 + dy;
            acc = __fmaf_rn(rw3(1.f, wy, rweight(P.tx, gx)), RR[(gy - gya) * T3_X + gx - gxa], acc);
          }
        }
        bcp[(long long)J * P.ncx + I] = acc;
      }
    } else if (TAIL == 2 && P.partials) {
      const bool cpin = 2 * pi >= T3_HX && 2 * pi < T3_X - T3_HX;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int row = row0 + 4 * k;
        if (!cpin || row < T3_HY || row >= T3_Y - T3_HY) continue;
        float rr[2], bb[2];
        resid_pair(p, row, rr, bb);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          sr += (double)rr[h] * (double)rr[h];
          sbb += (double)bb[h] * (double)bb[h];
        }
      }
    }
    // store the interior of plane p
    const int zp = (int)((L.z0 + p) & 1);
    for (int i = tid; i < T3_YI * (T3_XI / 4); i += 256) {
      const int ly = T3_HY + i / (T3_XI / 4), lx = T3_HX + 4 * (i % (T3_XI / 4));
      const int gx = gxa + lx, gy = gya + ly;
      if (gy >= L.ny || gx >= L.nx) continue;
      const int c0 = (lx + ly + zp) & 1;
      const float2 a = *reinterpret_cast<const float2*>(&R[slot_of(p)][c0][ly][lx >> 1]);
      const float2 bb = *reinterpret_cast<const float2*>(&R[slot_of(p)][c0 ^ 1][ly][lx >> 1]);
      float* o = P.xout + (long long)p * plane + (long long)gy * nx + gx;
      if (vec && gx + 3 < L.nx) *reinterpret_cast<float4*>(o) = make_float4(a.x, bb.x, a.y, bb.y);
      else {
        const float v[4] = {a.x, bb.x, a.y, bb.y};
        for (int c = 0; c < 4 && gx + c < L.nx; ++c) o[c] = v[c];
      }
    }
  };

  // x += P e_c on every cell of plane p (coarse plane = p: z is not coarsened).  The coarse
  // tile goes to the slot of plane p + 1 (free until that plane is stored) first.
  long long pIx[2] = {0, 0}, pJx[2] = {0, 0};
  float ptx[2] = {0.f, 0.f};
  if (PROLONG) {
#pragma unroll
    for (int h = 0; h < 2; ++h) ptaps(P.tx, gxa + 2 * pi + h, pIx[h], pJx[h], ptx[h]);
  }
  const int cxa = (gxa >> 1) - 1, cya = (gya >> 1) - 1;  // coarse tile origin (>= 1-cell margin)
  constexpr int CTX = T3_X / 2 + 3, CTY = T3_Y / 2 + 3;
  auto prolong = [&](int p) {
    const float* xcp = P.xc + (long long)p * P.ncx * P.ncy;
    float* CT = colarr(slot_of(p + 1), 0);  // [CTY][CTX]
    for (int i = tid; i < CTX * CTY; i += 256) {
      const int cy = cya + i / CTX, cx = cxa + i % CTX;
      CT[i] = (cx >= 0 && cx < P.ncx && cy >= 0 && cy < P.ncy) ? __ldg(xcp + (long long)cy * P.ncx + cx) : 0.f;
    }
    __syncthreads();
    const int zp = (int)((L.z0 + p) & 1);
#pragma unroll 2
    for (int k = 0; k < 8; ++k) {
      const int row = row0 + 4 * k;
      const int gy = gya + row;
      if (gy < 0 || gy >= L.ny) continue;
      long long Iy, Jy;
      float tyw;
      ptaps(P.ty, gy, Iy, Jy, tyw);
      const float* rI = CT + (int)(Iy - cya) * CTX - cxa;
      const float* rJ = CT + (int)(Jy - cya) * CTX - cxa;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!colin[h]) continue;
        const int lx = 2 * pi + h;
        const float e = bilerp(rI[pIx[h]], rI[pJx[h]], rJ[pIx[h]], rJ[pJx[h]], ptx[h], tyw);
        float& v = R[slot_of(p)][(lx + row + zp) & 1][row][pi];
        v = __fadd_rn(v, e);
      }
    }
  };

  // stage 1 covers [p_lo-2, p_hi+2), stage 2 [p_lo-1, p_hi+1), the tail [p_lo, p_hi)
  const int s1lo = max(p_lo - 2, 0), s1hi = min(p_hi + 2, nzl);
  const int s2lo = max(p_lo - 1, 0), s2hi = min(p_hi + 1, nzl);
  __syncthreads();
  load_plane(first);
  store_plane(first);
  for (int p = first; p <= last + 2; ++p) {  // p = plane entering the ring
    __syncthreads();
    if (p + 1 < last) load_plane(p + 1);
    if (PROLONG && p < last) {
      prolong(p);
      __syncthreads();
    }
    // each stage uses the b values fetched one step earlier, then fetches the next step's
    if (p - 1 >= s1lo && p - 1 < s1hi) stage(p - 1, 0, bpre1);
    if (p >= s1lo && p < s1hi) fetch_b(p, 0, bpre1);
    __syncthreads();
    if (p - 2 >= s2lo && p - 2 < s2hi) stage(p - 2, 1, bpre2);
    if (p - 1 >= s2lo && p - 1 < s2hi) fetch_b(p - 1, 1, bpre2);
    __syncthreads();
    if (p - 3 >= p_lo && p - 3 < p_hi) tail(p - 3);
    if (TAIL == 1) __syncthreads();  // the tail's residual plane aliases the incoming slot
    if (p + 1 < last) store_plane(p + 1);
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
         L.nzl == L.gz.n /* single slab: ghost planes not wired into the 3D pass yet */;
}

int fused3d_tiles(const LevelK& L) {
  return ((L.nx + T3_XI - 1) / T3_XI) * ((L.ny + T3_YI - 1) / T3_YI) * ((L.nzl + T3_ZC - 1) / T3_ZC);
}

template <int TAIL, bool PROLONG>
static void launch3d_t(const Pass3D& P, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_pass3d<TAIL, PROLONG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM3D);
    attr = true;
  }
  dim3 g((P.L.nx + T3_XI - 1) / T3_XI, (P.L.ny + T3_YI - 1) / T3_YI, (P.L.nzl + T3_ZC - 1) / T3_ZC);
  k_pass3d<TAIL, PROLONG><<<g, 256, SMEM3D, s>>>(P);
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
