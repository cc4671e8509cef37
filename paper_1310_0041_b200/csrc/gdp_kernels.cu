#include <algorithm>
// gdp_kernels.cu — sm_100a kernels of the multigrid V-cycle.
//
// Reference schedule (opts.fused = 0): one kernel per red-black half-sweep, one per
// residual+restriction, one per prolongation+correction.  The fused schedule lives
// in gdp_fused.cu and calls the same per-point arithmetic (gdp_device.cuh), so both
// schedules produce bit-identical iterates.
#include <cooperative_groups.h>

#include "gdp_kernels.h"

namespace gdp {

// ---------------------------------------------------------------------------------
// neighbour loads with ghost planes (z-slab halos of a distributed ctx)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ Nbr load_nbr(const float* x, const float* xlo, const float* xhi,
                                        const LevelK& L, const Coef& k, int iz, long long c,
                                        float xc) {
  const long long nx = L.nx, plane = (long long)L.nx * L.ny;
  Nbr nb;
  nb.w = k.xl != 0.f ? x[c - 1] : xc;
  nb.e = k.xr != 0.f ? x[c + 1] : xc;
  nb.s = k.yl != 0.f ? x[c - nx] : xc;
  nb.n = k.yr != 0.f ? x[c + nx] : xc;
  nb.d = k.zl != 0.f ? (iz > 0 ? x[c - plane] : xlo[c]) : xc;
  nb.u = k.zr != 0.f ? (iz < L.nzl - 1 ? x[c + plane] : xhi[c - (long long)iz * plane]) : xc;
  return nb;
}

// Interior cells have the regular link coefficients on every axis (and all links present), so
// the general coefficient evaluation and the reciprocal of the diagonal can be skipped: kint and
// 1/D_int are the values coefs() and gs_update() would produce for them.
struct Interior {
  Coef k;
  float invD;
  bool zreg_all;  // level without z links: z never disqualifies a cell
};
__device__ __forceinline__ Interior interior_consts(const LevelK& L) {
  Interior I;
  I.k.xl = L.ax.k; I.k.xr = L.ax.k; I.k.yl = L.ay.k; I.k.yr = L.ay.k; I.k.zl = L.az.k; I.k.zr = L.az.k;
  I.invD = relax_inv(L.omega, I.k.diag(L.alpha));
  I.zreg_all = L.az.k == 0.f && L.az.kr == 0.f && L.az.kl == 0.f;
  return I;
}
__device__ __forceinline__ bool is_interior(const LevelK& L, const Interior& I, int ix, int iy, long long zg) {
  return ix >= 1 && ix <= L.ax.n - 3 && iy >= 1 && iy <= L.ay.n - 3 && (I.zreg_all || (zg >= 1 && zg <= L.az.n - 3));
}

// a4: one red-black Gauss-Seidel half-sweep (colour = (x + y + z_global) & 1); the point
// (ixh, iy, iz) of the half grid (every schedule that runs the reference arithmetic calls this)
template <int MODE, typename TI>
__device__ __forceinline__ void rbgs_point(const LevelK& L, float* __restrict__ x, const float* xlo,
                                           const float* xhi, const RhsK& R, int color, int ixh, int iy, int iz) {
  const long long zg = L.z0 + iz;
  const int ix = 2 * ixh + ((color + iy + (int)(zg & 1)) & 1);
  if (ix >= L.nx) return;
  const long long plane = (long long)L.nx * L.ny;
  const long long c = iz * plane + (long long)iy * L.nx + ix;
  const float xc = x[c];
  const Interior I = interior_consts(L);
  if (MODE == RHS_B && is_interior(L, I, ix, iy, zg)) {
    // all six neighbours exist; slab faces come from the ghost planes
    const float d = I.zreg_all ? xc : (iz > 0 ? x[c - plane] : xlo[c]);
    const float u = I.zreg_all ? xc : (iz < L.nzl - 1 ? x[c + plane] : xhi[c - (long long)iz * plane]);
    const float r = __fsub_rn(R.b[c], apply_from(I.k, L.alpha, xc, x[c - 1], x[c + 1], x[c - L.nx], x[c + L.nx], d, u));
    x[c] = __fmaf_rn(r, I.invD, xc);  // == gs_update(xc, r, D)
    return;
  }
  const Coef k = coefs(L, ix, iy, zg);
  const Nbr nb = load_nbr(x, xlo, xhi, L, k, iz, c, xc);
  const float r = residual_at<MODE, TI>(L, R, k, xc, nb, c, L.nx, plane, nullptr);
  x[c] = gs_update(xc, r, k.diag(L.alpha), L.omega);
}

template <int MODE, typename TI>
__global__ void __launch_bounds__(256) k_rbgs(LevelK L, float* __restrict__ x, const float* xlo,
                                              const float* xhi, RhsK R, int color) {
  const int iy = blockIdx.y * blockDim.y + threadIdx.y;
  if (iy >= L.ny) return;
  rbgs_point<MODE, TI>(L, x, xlo, xhi, R, color, blockIdx.x * blockDim.x + threadIdx.x, iy, blockIdx.z);
}

// a5+a6: residual at the fine level, restricted by volume-weighted child average.
// One thread per coarse cell; every fine cell belongs to exactly one parent.
template <int MODE, typename TI>
__device__ __forceinline__ void restrict_point(const LevelK& L, const float* __restrict__ x, const float* xlo,
                                               const float* xhi, const RhsK& R, const XferAxis& tx,
                                               const XferAxis& ty, const XferAxis& tz, int ncx, int ncy,
                                               float* __restrict__ bc, int cx, int cy, int cz) {
  const long long plane = (long long)L.nx * L.ny;
  const int fx0 = tx.coarsened ? 2 * cx : cx, fx1 = tx.coarsened ? min(2 * cx + 1, L.nx - 1) : cx;
  const int fy0 = ty.coarsened ? 2 * cy : cy, fy1 = ty.coarsened ? min(2 * cy + 1, L.ny - 1) : cy;
  const int fz0 = tz.coarsened ? 2 * cz : cz, fz1 = tz.coarsened ? min(2 * cz + 1, L.nzl - 1) : cz;
  const Interior I = interior_consts(L);
  float acc = 0.f;
  for (int fz = fz0; fz <= fz1; ++fz) {
    const long long zg = L.z0 + fz;
    const float wz = rweight(tz, zg);
    for (int fy = fy0; fy <= fy1; ++fy) {
      const float wy = rweight(ty, fy);
      for (int fx = fx0; fx <= fx1; ++fx) {
        const float wx = rweight(tx, fx);
        const long long c = fz * plane + (long long)fy * L.nx + fx;
        const float xc = x[c];
        float r;
        if (MODE == RHS_B && is_interior(L, I, fx, fy, zg)) {
          const float d = I.zreg_all ? xc : (fz > 0 ? x[c - plane] : xlo[c]);
          const float u = I.zreg_all ? xc : (fz < L.nzl - 1 ? x[c + plane] : xhi[c - (long long)fz * plane]);
          r = __fsub_rn(R.b[c], apply_from(I.k, L.alpha, xc, x[c - 1], x[c + 1], x[c - L.nx], x[c + L.nx], d, u));
        } else {
          const Coef k = coefs(L, fx, fy, zg);
          const Nbr nb = load_nbr(x, xlo, xhi, L, k, fz, c, xc);
          r = residual_at<MODE, TI>(L, R, k, xc, nb, c, L.nx, plane, nullptr);
        }
        acc = __fmaf_rn(rw3(wz, wy, wx), r, acc);
      }
    }
  }
  bc[(long long)cz * ncx * ncy + (long long)cy * ncx + cx] = acc;
}

template <int MODE, typename TI>
__global__ void __launch_bounds__(256) k_restrict(LevelK L, const float* __restrict__ x,
                                                  const float* xlo, const float* xhi, RhsK R,
                                                  XferAxis tx, XferAxis ty, XferAxis tz,
                                                  int ncx, int ncy, int nczl,
                                                  float* __restrict__ bc) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = blockIdx.y * blockDim.y + threadIdx.y;
  if (cx >= ncx || cy >= ncy) return;
  restrict_point<MODE, TI>(L, x, xlo, xhi, R, tx, ty, tz, ncx, ncy, bc, cx, cy, blockIdx.z);
}

// Restriction of a right-hand side alone (FMG start): the sum k_restrict forms for x = 0, where
// r = b - A 0 = b exactly; same children order and weights -> the same values.
__global__ void __launch_bounds__(256) k_restrict_b(LevelK L, const float* __restrict__ b, XferAxis tx, XferAxis ty,
                                                    XferAxis tz, int ncx, int ncy, float* __restrict__ bc) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = blockIdx.y * blockDim.y + threadIdx.y;
  const int cz = blockIdx.z;
  if (cx >= ncx || cy >= ncy) return;
  const long long plane = (long long)L.nx * L.ny;
  const int fx0 = tx.coarsened ? 2 * cx : cx, fx1 = tx.coarsened ? min(2 * cx + 1, L.nx - 1) : cx;
  const int fy0 = ty.coarsened ? 2 * cy : cy, fy1 = ty.coarsened ? min(2 * cy + 1, L.ny - 1) : cy;
  const int fz0 = tz.coarsened ? 2 * cz : cz, fz1 = tz.coarsened ? min(2 * cz + 1, L.nzl - 1) : cz;
  float acc = 0.f;
  for (int fz = fz0; fz <= fz1; ++fz) {
    const float wz = rweight(tz, L.z0 + fz);
    for (int fy = fy0; fy <= fy1; ++fy) {
      const float wy = rweight(ty, fy);
      for (int fx = fx0; fx <= fx1; ++fx)
        acc = __fmaf_rn(rw3(wz, wy, rweight(tx, fx)), __ldg(b + fz * plane + (long long)fy * L.nx + fx), acc);
    }
  }
  bc[(long long)cz * ncx * ncy + (long long)cy * ncx + cx] = acc;
}

// k_restrict_b for x/y coarsening with nx % 4 == 0: coarse cells (2i, 2i+1) of one coarse row
// per thread from one float4 of each child row; per cell the same order (fy outer, fx inner) and
// weights, so the same values.
__global__ void __launch_bounds__(256) k_restrict_b2(LevelK L, const float* __restrict__ b, XferAxis tx, XferAxis ty,
                                                     int ncx, int ncy, float* __restrict__ bc) {
  const int i2 = blockIdx.x * blockDim.x + threadIdx.x;  // coarse columns 2 i2, 2 i2 + 1
  const int cy = blockIdx.y * blockDim.y + threadIdx.y;
  const int cz = blockIdx.z;
  if (2 * i2 >= ncx || cy >= ncy) return;
  const long long plane = (long long)L.nx * L.ny;
  const int fx = 4 * i2;
  const int fy0 = 2 * cy, fy1 = min(2 * cy + 1, L.ny - 1);
  const float w0 = rweight(tx, fx), w1 = rweight(tx, fx + 1), w2 = rweight(tx, fx + 2), w3 = rweight(tx, fx + 3);
  float a0 = 0.f, a1 = 0.f;
  for (int fy = fy0; fy <= fy1; ++fy) {
    const float wy = rweight(ty, fy);
    const float4 v = __ldg(reinterpret_cast<const float4*>(b + cz * plane + (long long)fy * L.nx + fx));
    a0 = __fmaf_rn(rw3(1.f, wy, w0), v.x, a0);
    a0 = __fmaf_rn(rw3(1.f, wy, w1), v.y, a0);
    a1 = __fmaf_rn(rw3(1.f, wy, w2), v.z, a1);
    a1 = __fmaf_rn(rw3(1.f, wy, w3), v.w, a1);
  }
  *reinterpret_cast<float2*>(bc + (long long)cz * ncx * ncy + (long long)cy * ncx + 2 * i2) = make_float2(a0, a1);
}

// a8: x_fine += P x_coarse (cell-centred linear interpolation, constant at the faces; the
// ghost coarse planes of a z-slab come from xclo / xchi).  4 columns x `rows` rows of one fine
// plane per thread: x taps computed
// once per thread, z taps once per plane, float4 read-modify-write of xf; per element the bilerp
// (x then y) and z blend of the reference ordering.
template <bool VEC>
__global__ void __launch_bounds__(256) k_prolong_rows(LevelK L, float* __restrict__ xf, XferAxis tx, XferAxis ty,
                                                      XferAxis tz, int ncx, int ncy, int nczl, long long cz0,
                                                      const float* __restrict__ xc, const float* xclo,
                                                      const float* xchi, int rows) {
  const int gx0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int fz = blockIdx.z;
  if (gx0 >= L.nx) return;
  long long Ix[4], Jx[4];
  float txw[4];
  bool in[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    in[c] = gx0 + c < L.nx;
    const int fx = in[c] ? gx0 + c : gx0;
    if (ptaps_regular(tx, fx)) ptaps_fast(tx, fx, Ix[c], Jx[c], txw[c]); else ptaps(tx, fx, Ix[c], Jx[c], txw[c]);
  }
  const long long I0 = gx0 >> 1;
  const bool xreg = VEC && in[3] && tx.coarsened && (ncx & 1) == 0 && ptaps_regular(tx, gx0) &&
                    ptaps_regular(tx, gx0 + 3);
  long long Iz, Jz;
  float tzw;
  if (ptaps_regular(tz, L.z0 + fz)) ptaps_fast(tz, L.z0 + fz, Iz, Jz, tzw); else ptaps(tz, L.z0 + fz, Iz, Jz, tzw);
  const long long cplane = (long long)ncx * ncy;
  auto zrow = [&](long long zgc) -> const float* {  // global coarse plane -> local / ghost plane
    const long long lz = zgc - cz0;
    if (lz < 0) return xclo;
    if (lz >= nczl) return xchi;
    return xc + lz * cplane;
  };
  const float* pI = zrow(Iz);
  const float* pJ = zrow(Jz);
  float* pf = xf + (long long)fz * L.nx * L.ny;
  const int y0 = blockIdx.y * rows, y1 = min(y0 + rows, L.ny);
  for (int fy = y0; fy < y1; ++fy) {
    long long Iy, Jy;
    float tyw;
    if (ptaps_regular(ty, fy)) ptaps_fast(ty, fy, Iy, Jy, tyw); else ptaps(ty, fy, Iy, Jy, tyw);
    float* row = pf + (long long)fy * L.nx + gx0;
    float v[4];
    if (VEC && in[3]) {
      const float4 q = *reinterpret_cast<const float4*>(row);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = in[c] ? row[c] : 0.f;
    }
    if (xreg) {  // regular x taps: coarse columns I0-1 .. I0+2 once per coarse row
      float e[4], f[4];
      auto quad = [&](const float* p, float (&o)[4]) {
        const float* rI = p + Iy * ncx + I0;
        const float* rJ = p + Jy * ncx + I0;
        const float2 mI = __ldg(reinterpret_cast<const float2*>(rI));
        const float2 mJ = __ldg(reinterpret_cast<const float2*>(rJ));
        const float lI = __ldg(rI - 1), hI = __ldg(rI + 2), lJ = __ldg(rJ - 1), hJ = __ldg(rJ + 2);
        o[0] = bilerp(mI.x, lI, mJ.x, lJ, 0.25f, tyw);    // I = I0,   J = I0-1
        o[1] = bilerp(mI.x, mI.y, mJ.x, mJ.y, 0.25f, tyw);  // I = I0,   J = I0+1
        o[2] = bilerp(mI.y, mI.x, mJ.y, mJ.x, 0.25f, tyw);  // I = I0+1, J = I0
        o[3] = bilerp(mI.y, hI, mJ.y, hJ, 0.25f, tyw);    // I = I0+1, J = I0+2
      };
      quad(pI, e);
      if (tzw != 0.f) {
        quad(pJ, f);
#pragma unroll
        for (int c = 0; c < 4; ++c) e[c] = __fmaf_rn(tzw, f[c], __fmul_rn(1.f - tzw, e[c]));
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = __fadd_rn(v[c], e[c]);
    } else {
      auto bil = [&](const float* p, int c) {
        const float* rI = p + Iy * ncx;
        const float* rJ = p + Jy * ncx;
        return bilerp(__ldg(rI + Ix[c]), __ldg(rI + Jx[c]), __ldg(rJ + Ix[c]), __ldg(rJ + Jx[c]), txw[c], tyw);
      };
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float e = bil(pI, c);
        if (tzw != 0.f) e = __fmaf_rn(tzw, bil(pJ, c), __fmul_rn(1.f - tzw, e));
        v[c] = __fadd_rn(v[c], e);
      }
    }
    if (VEC && in[3]) *reinterpret_cast<float4*>(row) = make_float4(v[0], v[1], v[2], v[3]);
    else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (in[c]) row[c] = v[c];
    }
  }
}

// a5: residual r = b - A x with per-block fp64 partial sums of r^2 and b^2 (one row of
// partials per plane, reduced in a fixed order by k_finalize -> deterministic).
template <int MODE, typename TI>
__global__ void __launch_bounds__(256) k_norms(LevelK L, const float* __restrict__ x,
                                               const float* xlo, const float* xhi, RhsK R,
                                               float* __restrict__ rout, double2* partials) {
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iz = blockIdx.z;
  const long long zg = L.z0 + iz;
  const long long plane = (long long)L.nx * L.ny;
  double sr = 0.0, sb = 0.0;
  const Interior I = interior_consts(L);
  if (ix < L.nx) {
    for (int iy = blockIdx.y * blockDim.y + threadIdx.y; iy < L.ny; iy += gridDim.y * blockDim.y) {
      const long long c = iz * plane + (long long)iy * L.nx + ix;
      const float xc = x[c];
      float bv, r;
      if (MODE == RHS_B && is_interior(L, I, ix, iy, zg)) {
        const float d = I.zreg_all ? xc : (iz > 0 ? x[c - plane] : xlo[c]);
        const float u = I.zreg_all ? xc : (iz < L.nzl - 1 ? x[c + plane] : xhi[c - (long long)iz * plane]);
        bv = R.b[c];
        r = __fsub_rn(bv, apply_from(I.k, L.alpha, xc, x[c - 1], x[c + 1], x[c - L.nx], x[c + L.nx], d, u));
      } else {
        const Coef k = coefs(L, ix, iy, zg);
        const Nbr nb = load_nbr(x, xlo, xhi, L, k, iz, c, xc);
        r = residual_at<MODE, TI>(L, R, k, xc, nb, c, L.nx, plane, &bv);
      }
      if (rout) rout[c] = r;
      sr += (double)r * (double)r;
      sb += (double)bv * (double)bv;
    }
  }
  block_sum2(sr, sb);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const long long bid = ((long long)iz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    partials[bid] = make_double2(sr, sb);
  }
}

// fixed-order reduction of `per` partials per plane -> out[plane]
__global__ void __launch_bounds__(256) k_finalize(const double2* partials, int per,
                                                  double2* out) {
  const int p = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < per; i += blockDim.x) {
    const double2 v = partials[(long long)p * per + i];
    a += v.x;
    b += v.y;
  }
  block_sum2(a, b);
  if (threadIdx.x == 0) out[p] = make_double2(a, b);
}

// a2 / a11: the finest-level rhs written out once per solve (the fused 2D passes read it)
template <typename TI>
__global__ void __launch_bounds__(256) k_rhs(LevelK L, RhsK R, float* __restrict__ b) {
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy = blockIdx.y, iz = blockIdx.z;
  if (ix >= L.nx) return;
  const long long c = (long long)iz * L.nx * L.ny + (long long)iy * L.nx + ix;
  b[c] = rhs_g<TI>(L, R, coefs(L, ix, iy, L.z0 + iz), c, L.nx);
}

// a1 + a2/a11 + a5 in one pass over I: x0 = decode(I) (the initial guess), the finest rhs
// b = av V - div W G (rhs_g), and per-(plane, block) fp64 partials of |b - A x0|^2 and |b|^2
// (the initial residual of the stopping rule, residual_at order).  A thread owns 4 columns and
// slides down a strip of rows keeping the rows above / below in registers.
template <typename TI> struct Quad;
template <> struct Quad<float> {
  __device__ static __forceinline__ void ld(const void* p, long long i, float (&v)[4]) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(p) + i));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};
template <> struct Quad<uint8_t> {
  __device__ static __forceinline__ void ld(const void* p, long long i, float (&v)[4]) {
    const unsigned w = __ldg(reinterpret_cast<const unsigned*>(static_cast<const uint8_t*>(p) + i));
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = decode_u8((w >> (8 * c)) & 0xffu);
  }
};

// per-plane sums for the mean pin (a10), 4 columns per thread (one float4 / 4-byte load per
// field and row), rows strided by gridDim.y; each thread adds its quad left to right in fp64
template <typename TA, typename TB, bool VEC>
__global__ void __launch_bounds__(256) k_plane_sums4(const void* a, const void* b, int nx, int ny,
                                                     double2* partials) {
  const int gx0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int iz = blockIdx.z;
  const long long plane = (long long)nx * ny;
  double sa = 0.0, sb = 0.0;
  if (gx0 < nx) {
    const int n = min(4, nx - gx0);
#pragma unroll 4
    for (int iy = blockIdx.y; iy < ny; iy += gridDim.y) {
      const long long c = iz * plane + (long long)iy * nx + gx0;
      float va[4] = {0.f, 0.f, 0.f, 0.f}, vb[4] = {0.f, 0.f, 0.f, 0.f};
      if (VEC) {
        Quad<TA>::ld(a, c, va);
        if (b) Quad<TB>::ld(b, c, vb);
      } else {
        for (int k = 0; k < n; ++k) {
          va[k] = ldI<TA>(a, c + k);
          if (b) vb[k] = ldI<TB>(b, c + k);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) { sa += (double)va[k]; sb += (double)vb[k]; }
    }
  }
  block_sum2(sa, sb);
  if (threadIdx.x == 0) partials[((long long)iz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = make_double2(sa, sb);
}

template <typename TI, bool VEC>
__global__ void __launch_bounds__(256) k_init(LevelK L, RhsK R, float* __restrict__ x0, float* __restrict__ b,
                                              double2* partials, int S, InitXfer X) {
  const int gx0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int iz = blockIdx.z;
  const long long zg = L.z0 + iz;
  const long long nx = L.nx, plane = (long long)L.nx * L.ny, pbase = (long long)iz * plane;
  const int y0 = blockIdx.y * S, y1 = min(y0 + S, L.ny);
  const float zl = cl(L.az, zg), zr = cr(L.az, zg);
  double sr = 0.0, sb = 0.0;
  if (gx0 < L.nx) {
    bool in[4];
    float kxl[4], kxr[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      in[c] = gx0 + c < L.nx;
      kxl[c] = cl(L.ax, gx0 + c);
      kxr[c] = cr(L.ax, gx0 + c);
    }
    const bool full = in[3];
    auto ldrow = [&](long long base, bool ok, float (&v)[4]) {  // I at [base + gx0 ..], 0 outside
      if (VEC && ok && full) { Quad<TI>::ld(R.I, base + gx0, v); return; }
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = (ok && in[c]) ? ldI<TI>(R.I, base + gx0 + c) : 0.f;
    };
    float rm[4], rc[4], rp[4], dn[4], up[4];
    float acc[4] = {0.f, 0.f, 0.f, 0.f};  // X.bc: restriction of r0 (per coarse column)
    float wxc[4];                          // X.bc: the columns' restriction weights (row invariant)
#pragma unroll
    for (int c = 0; c < 4; ++c) wxc[c] = X.bc ? rweight(X.tx, gx0 + c) : 1.f;
    ldrow(pbase + (long long)(y0 - 1) * nx, y0 - 1 >= 0, rm);
    ldrow(pbase + (long long)y0 * nx, y0 < L.ny, rc);
    for (int gy = y0; gy < y1; ++gy) {
      const long long row = pbase + (long long)gy * nx;
      ldrow(row + nx, gy + 1 < L.ny, rp);
      if (zl != 0.f) ldrow(row - plane, true, dn);
      if (zr != 0.f) ldrow(row + plane, true, up);
      const float left = gx0 > 0 ? ldI<TI>(R.I, row + gx0 - 1) : 0.f;
      const float right = gx0 + 4 < L.nx ? ldI<TI>(R.I, row + gx0 + 4) : 0.f;
      float V[4] = {0.f, 0.f, 0.f, 0.f};
      if (R.vmode == 2) {
        if (VEC && full) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(R.V + row + gx0));
          V[0] = q.x; V[1] = q.y; V[2] = q.z; V[3] = q.w;
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) V[c] = in[c] ? __ldg(R.V + row + gx0 + c) : 0.f;
        }
        if (R.vout) {  // deferred mean pin of phase 1: V += shift (== k_add_scalar), written back
#pragma unroll
          for (int c = 0; c < 4; ++c) V[c] = __fadd_rn(V[c], R.vshift);
          if (VEC && full) *reinterpret_cast<float4*>(R.vout + row + gx0) = make_float4(V[0], V[1], V[2], V[3]);
          else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (in[c]) R.vout[row + gx0 + c] = V[c];
          }
        }
      }
      const float yl = cl(L.ay, gy), yr = cr(L.ay, gy);
      float xo[4], bo[4], ro[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        Coef k;
        k.xl = kxl[c]; k.xr = kxr[c]; k.yl = yl; k.yr = yr; k.zl = zl; k.zr = zr;
        const float Ic = rc[c];
        const float Iw = k.xl != 0.f ? (c > 0 ? rc[c - 1] : left) : Ic;
        const float Ie = k.xr != 0.f ? (c < 3 ? rc[c + 1] : right) : Ic;
        const float Is = k.yl != 0.f ? rm[c] : Ic;
        const float In = k.yr != 0.f ? rp[c] : Ic;
        const float Vc = R.vmode == 0 ? 0.f : (R.vmode == 1 ? Ic : V[c]);
        const float bc = rhs_from(k, Ic, Iw, Ie, Is, In, Vc, R.av);  // == rhs_g
        const float d = k.zl != 0.f ? dn[c] : Ic, u = k.zr != 0.f ? up[c] : Ic;
        const float r = __fsub_rn(bc, apply_from(k, L.alpha, Ic, Iw, Ie, Is, In, d, u));  // == residual_at
        xo[c] = Ic;
        bo[c] = bc;
        ro[c] = r;
        if (in[c]) {
          sr += (double)r * (double)r;
          sb += (double)bc * (double)bc;
        }
      }
      if (VEC && full) {
        *reinterpret_cast<float4*>(x0 + row + gx0) = make_float4(xo[0], xo[1], xo[2], xo[3]);
        *reinterpret_cast<float4*>(b + row + gx0) = make_float4(bo[0], bo[1], bo[2], bo[3]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (in[c]) { x0[row + gx0 + c] = xo[c]; b[row + gx0 + c] = bo[c]; }
      }
      if (X.bc) {  // == k_restrict's sum over the children (fy outer, fx inner), plane-local
        const bool yc = X.ty.coarsened != 0;
        const bool first = !yc || (gy & 1) == 0;
        const float wy = rweight(X.ty, gy);
        const long long cbase = (long long)iz * X.ncx * X.ncy + (long long)(yc ? gy >> 1 : gy) * X.ncx;
        const bool last = !yc || (gy & 1) == 1 || gy + 1 == L.ny;
        if (X.tx.coarsened) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float a = first ? 0.f : acc[h];
#pragma unroll
            for (int c = 2 * h; c < 2 * h + 2; ++c)
              if (in[c]) a = __fmaf_rn(rw3(1.f, wy, wxc[c]), ro[c], a);
            acc[h] = a;
            if (last && in[2 * h]) X.bc[cbase + (gx0 >> 1) + h] = a;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            acc[c] = __fmaf_rn(rw3(1.f, wy, 1.f), ro[c], first ? 0.f : acc[c]);
            if (last && in[c]) X.bc[cbase + gx0 + c] = acc[c];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) { rm[c] = rc[c]; rc[c] = rp[c]; }
    }
  }
  block_sum2(sr, sb);
  if (threadIdx.x == 0) partials[((long long)iz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = make_double2(sr, sb);
}

// NEXT-1: rhs of the §6 NPR filter: b = alpha I0 - div(W V) with the link
// field V = lam (1 - exp(-|grad I0|^2 / 2 sigma^2)) grad I0, |grad I0|^2 the 3D forward-difference
// gradient at the link's base voxel (reading n-1).  One-off pass per solve, evaluated in fp64 and
// rounded once; also writes x0 = I0.  (D^T W V)(c) = sum_d beta_d (V_d(c - e_d) - V_d(c)).
template <typename TI>
__global__ void __launch_bounds__(256) k_npr_rhs(LevelK L, const void* I, float* __restrict__ x0,
                                                 float* __restrict__ b, double bx, double by, double bz,
                                                 double lam, double inv2s2) {
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy = blockIdx.y, iz = blockIdx.z;
  if (ix >= L.nx) return;
  const long long nx = L.nx, plane = (long long)L.nx * L.ny;
  auto at = [&](int x, int y, int z) -> double { return (double)ldI<TI>(I, z * plane + (long long)y * nx + x); };
  // V_d of the link (v, v + e_d); the caller guarantees v + e_d is inside the grid
  auto vlink = [&](int x, int y, int z, int d) -> double {
    const double c = at(x, y, z);
    double m2 = 0.0, gd = 0.0;
    if (x + 1 < L.nx) { const double g = at(x + 1, y, z) - c; m2 += g * g; if (d == 0) gd = g; }
    if (y + 1 < L.ny) { const double g = at(x, y + 1, z) - c; m2 += g * g; if (d == 1) gd = g; }
    if (z + 1 < L.nzl) { const double g = at(x, y, z + 1) - c; m2 += g * g; if (d == 2) gd = g; }
    return lam * (1.0 - exp(-m2 * inv2s2)) * gd;
  };
  const double Ic = at(ix, iy, iz);
  double s = (double)L.alpha * Ic;
  const double beta[3] = {bx, by, bz};
  const int pos[3] = {ix, iy, iz}, n[3] = {L.nx, L.ny, L.nzl};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (beta[d] == 0.0 || n[d] < 2) continue;
    if (pos[d] > 0) s += beta[d] * vlink(ix - (d == 0), iy - (d == 1), iz - (d == 2), d);
    if (pos[d] + 1 < n[d]) s -= beta[d] * vlink(ix, iy, iz, d);
  }
  const long long c = (long long)iz * plane + (long long)iy * nx + ix;
  x0[c] = (float)Ic;
  b[c] = (float)s;
}

void launch_npr_rhs(const LevelK& L, const void* I, int tI, float* x0, float* b, float bx, float by, float bz,
                    float lam, float sigma, cudaStream_t s) {
  ProfScope ps(KC_UTIL, (double)L.nx * L.ny * L.nzl * ((tI ? 4.0 : 1.0) + 8.0), s);
  dim3 g((L.nx + 255) / 256, L.ny, L.nzl);
  const double inv2s2 = 1.0 / (2.0 * (double)sigma * (double)sigma);
  if (tI == 0) k_npr_rhs<uint8_t><<<g, 256, 0, s>>>(L, I, x0, b, bx, by, bz, lam, inv2s2);
  else k_npr_rhs<float><<<g, 256, 0, s>>>(L, I, x0, b, bx, by, bz, lam, inv2s2);
}

template <typename TI>
__global__ void k_decode_copy(const void* I, float* __restrict__ x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = ldI<TI>(I, i);
}

__global__ void k_add_scalar(float* __restrict__ x, long long n, float s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] += s;
}

__global__ void k_axpy(float* __restrict__ x, const float* __restrict__ e, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] += e[i];
}

// a7: coarsest level, exact solve by fast diagonalisation.  The coarsest operator is
// alpha + T_x (+) T_y (+) T_z (Kronecker sum of 1D finite-volume operators), so
// x = V (Lambda^-1 (V^-1 b)) with per-axis eigenvectors computed once on the host.
// With alpha = 0 the constant mode (lambda = 0) is dropped: the coarse problem is
// projected onto the range of A and its mean-zero solution returned (reading c-3).
// One CTA per independent system (the whole level, or one slice when z is uncoupled).
__global__ void __launch_bounds__(512) k_coarse_fd(CoarseK C, const float* __restrict__ b,
                                                   float* __restrict__ x) {
  extern __shared__ float sm[];
  const int nx = C.nx, ny = C.ny, nzs = C.cz ? C.nz : 1;
  const int nsys = nx * ny * nzs;
  const long long off = C.cz ? 0 : (long long)blockIdx.x * nx * ny;
  float* A = sm;
  float* B = sm + nsys;
  for (int i = threadIdx.x; i < nsys; i += blockDim.x) A[i] = b[off + i];
  __syncthreads();
  // along x: consecutive threads take consecutive modes k, so the x matrix is staged in shared
  // memory with a padded row stride (conflict-free column walk); `in` rows are broadcast.  The
  // y / z matrices are staged too (rows broadcast).  Four outputs per thread in flight (ILP);
  // every dot product still runs j = 0, 1, ... in order.
  float* Ms = sm + 2 * nsys;
  constexpr int U = 4;
  const int nt = blockDim.x;
  auto tx = [&](const float* M, float* in, float* out) {
    for (int i = threadIdx.x; i < nx * nx; i += nt) Ms[(i / nx) * (nx + 1) + i % nx] = __ldg(M + i);
    __syncthreads();
    for (int i0 = threadIdx.x; i0 < nsys; i0 += U * nt) {
      const float* mk[U];
      const float* ir[U];
      float acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * nt, nsys - 1);
        mk[u] = Ms + (i % nx) * (nx + 1);
        ir[u] = in + (i / nx) * nx;
        acc[u] = 0.f;
      }
      if (nt % nx == 0) {  // the U outputs share their mode k: one matrix load per j
        for (int j = 0; j < nx; ++j) {
          const float m = mk[0][j];
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = fmaf(m, ir[u][j], acc[u]);
        }
      } else {
        for (int j = 0; j < nx; ++j)
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = fmaf(mk[u][j], ir[u][j], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * nt < nsys) out[i0 + u * nt] = acc[u];
    }
    __syncthreads();
  };
  auto ty = [&](const float* M, float* in, float* out) {  // along y
    for (int i = threadIdx.x; i < ny * ny; i += nt) Ms[i] = __ldg(M + i);
    __syncthreads();
    for (int i0 = threadIdx.x; i0 < nsys; i0 += U * nt) {
      const float* mk[U];
      const float* ic[U];
      float acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * nt, nsys - 1);
        const int xx = i % nx, k = (i / nx) % ny, z = i / (nx * ny);
        mk[u] = Ms + k * ny;
        ic[u] = in + (long long)z * ny * nx + xx;
        acc[u] = 0.f;
      }
      if (nzs == 1 && nt % nx == 0) {  // the U outputs share their column: one input load per j
        for (int j = 0; j < ny; ++j) {
          const float v = ic[0][j * nx];
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = fmaf(mk[u][j], v, acc[u]);
        }
      } else {
        for (int j = 0; j < ny; ++j)
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = fmaf(mk[u][j], ic[u][j * nx], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * nt < nsys) out[i0 + u * nt] = acc[u];
    }
    __syncthreads();
  };
  auto tz = [&](const float* M, float* in, float* out) {  // along z
    const int pl = nx * ny;
    for (int i = threadIdx.x; i < nzs * nzs; i += nt) Ms[i] = __ldg(M + i);
    __syncthreads();
    for (int i0 = threadIdx.x; i0 < nsys; i0 += U * nt) {
      const float* mk[U];
      const float* ic[U];
      float acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = min(i0 + u * nt, nsys - 1);
        mk[u] = Ms + (i / pl) * nzs;
        ic[u] = in + i % pl;
        acc[u] = 0.f;
      }
      for (int j = 0; j < nzs; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = fmaf(mk[u][j], ic[u][(long long)j * pl], acc[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * nt < nsys) out[i0 + u * nt] = acc[u];
    }
    __syncthreads();
  };
  float* cur = A;
  float* nxt = B;
  if (C.cx && nx > 1) { tx(C.Fx, cur, nxt); float* t = cur; cur = nxt; nxt = t; }
  if (C.cy && ny > 1) { ty(C.Fy, cur, nxt); float* t = cur; cur = nxt; nxt = t; }
  if (C.cz && nzs > 1) { tz(C.Fz, cur, nxt); float* t = cur; cur = nxt; nxt = t; }
  for (int i = threadIdx.x; i < nsys; i += blockDim.x) {
    const int xx = i % nx, yy = (i / nx) % ny, zz = i / (nx * ny);
    float lam = C.alpha;
    if (C.cx && nx > 1) lam += __ldg(C.lx + xx);
    if (C.cy && ny > 1) lam += __ldg(C.ly + yy);
    if (C.cz && nzs > 1) lam += __ldg(C.lz + zz);
    cur[i] = lam > C.lam_thr ? cur[i] / lam : 0.f;
  }
  __syncthreads();
  if (C.cx && nx > 1) { tx(C.Bx, cur, nxt); float* t = cur; cur = nxt; nxt = t; }
  if (C.cy && ny > 1) { ty(C.By, cur, nxt); float* t = cur; cur = nxt; nxt = t; }
  if (C.cz && nzs > 1) { tz(C.Bz, cur, nxt); float* t = cur; cur = nxt; nxt = t; }
  for (int i = threadIdx.x; i < nsys; i += blockDim.x) x[off + i] = cur[i];
}

// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
static inline dim3 grid_plane(int nx, int ny, int nz, dim3 blk, int ymax) {
  int gy = (ny + blk.y - 1) / blk.y;
  if (ymax > 0 && gy > ymax) gy = ymax;
  return dim3((nx + blk.x - 1) / blk.x, gy, nz);
}

template <int MODE, typename TI>
static void launch_rbgs_t(const LevelK& L, float* x, const float* xlo, const float* xhi,
                          const RhsK& R, int color, cudaStream_t s) {
  dim3 blk(32, 8);
  dim3 grd(((L.nx + 1) / 2 + blk.x - 1) / blk.x, (L.ny + blk.y - 1) / blk.y, L.nzl);
  k_rbgs<MODE, TI><<<grd, blk, 0, s>>>(L, x, xlo, xhi, R, color);
}

static inline double ncell(const LevelK& L) { return (double)L.nx * L.ny * L.nzl; }

void launch_rbgs(const LevelK& L, float* x, const float* xlo, const float* xhi, const RhsK& R,
                 int mode, int tI, int color, cudaStream_t s) {
  ProfScope ps(KC_RBGS, ncell(L) * (4.0 + rhs_bytes(mode, tI, R) + 2.0), s, ncell(L));
  if (mode == RHS_B) launch_rbgs_t<RHS_B, float>(L, x, xlo, xhi, R, color, s);
  else if (tI == 0) launch_rbgs_t<RHS_G, uint8_t>(L, x, xlo, xhi, R, color, s);
  else launch_rbgs_t<RHS_G, float>(L, x, xlo, xhi, R, color, s);
}

template <int MODE, typename TI>
static void launch_restrict_t(const LevelK& L, const float* x, const float* xlo, const float* xhi,
                              const RhsK& R, const XferAxis& tx, const XferAxis& ty,
                              const XferAxis& tz, int ncx, int ncy, int nczl, float* bc,
                              cudaStream_t s) {
  dim3 blk(32, 8);
  dim3 grd((ncx + 31) / 32, (ncy + 7) / 8, nczl);
  k_restrict<MODE, TI><<<grd, blk, 0, s>>>(L, x, xlo, xhi, R, tx, ty, tz, ncx, ncy, nczl, bc);
}

void launch_restrict(const LevelK& L, const float* x, const float* xlo, const float* xhi,
                     const RhsK& R, int mode, int tI, const XferAxis& tx, const XferAxis& ty,
                     const XferAxis& tz, int ncx, int ncy, int nczl, float* bc, cudaStream_t s) {
  ProfScope ps(KC_RESTRICT, ncell(L) * (4.0 + rhs_bytes(mode, tI, R)) + 4.0 * ncx * ncy * (double)nczl, s, ncell(L));
  if (mode == RHS_B)
    launch_restrict_t<RHS_B, float>(L, x, xlo, xhi, R, tx, ty, tz, ncx, ncy, nczl, bc, s);
  else if (tI == 0)
    launch_restrict_t<RHS_G, uint8_t>(L, x, xlo, xhi, R, tx, ty, tz, ncx, ncy, nczl, bc, s);
  else
    launch_restrict_t<RHS_G, float>(L, x, xlo, xhi, R, tx, ty, tz, ncx, ncy, nczl, bc, s);
}

void launch_restrict_b(const LevelK& L, const float* b, const XferAxis& tx, const XferAxis& ty, const XferAxis& tz,
                       int ncx, int ncy, int nczl, float* bc, cudaStream_t s) {
  ProfScope ps(KC_RESTRICT, ncell(L) * 4.0 + 4.0 * ncx * ncy * (double)nczl, s, ncell(L));
  if (tx.coarsened && ty.coarsened && !tz.coarsened && (L.nx & 3) == 0 && ((uintptr_t)b & 15) == 0 &&
      ((uintptr_t)bc & 7) == 0) {  // two coarse cells per thread from float4 rows
    dim3 blk(64, 4);
    dim3 grd((ncx / 2 + 63) / 64, (ncy + 3) / 4, nczl);
    k_restrict_b2<<<grd, blk, 0, s>>>(L, b, tx, ty, ncx, ncy, bc);
    return;
  }
  dim3 blk(64, 4);
  dim3 grd((ncx + 63) / 64, (ncy + 3) / 4, nczl);
  k_restrict_b<<<grd, blk, 0, s>>>(L, b, tx, ty, tz, ncx, ncy, bc);
}

void launch_prolong(const LevelK& L, float* xf, const XferAxis& tx, const XferAxis& ty,
                    const XferAxis& tz, int ncx, int ncy, int nczl, long long cz0, const float* xc,
                    const float* xclo, const float* xchi, cudaStream_t s) {
  ProfScope ps(KC_PROLONG, ncell(L) * 8.0 + 4.0 * ncx * ncy * (double)nczl, s, ncell(L));
  // 4 columns per thread; rows per thread: 8 on wide planes, 2 on the small coarse ones
  const int nt = std::min(256, std::max(32, ((L.nx + 3) / 4 + 31) / 32 * 32));
  const int rows = L.ny >= 256 ? 8 : 2;
  dim3 g((L.nx + 4 * nt - 1) / (4 * nt), (L.ny + rows - 1) / rows, L.nzl);
  if ((L.nx & 3) == 0 && ((uintptr_t)xf & 15) == 0)
    k_prolong_rows<true><<<g, nt, 0, s>>>(L, xf, tx, ty, tz, ncx, ncy, nczl, cz0, xc, xclo, xchi, rows);
  else
    k_prolong_rows<false><<<g, nt, 0, s>>>(L, xf, tx, ty, tz, ncx, ncy, nczl, cz0, xc, xclo, xchi, rows);
}

int norms_blocks_per_plane(int nx, int ny) {
  dim3 blk(128, 2);
  dim3 g = grid_plane(nx, ny, 1, blk, 32);
  return g.x * g.y;
}

template <int MODE, typename TI>
static void launch_norms_t(const LevelK& L, const float* x, const float* xlo, const float* xhi,
                           const RhsK& R, float* rout, double2* partials, cudaStream_t s) {
  dim3 blk(128, 2);
  dim3 grd = grid_plane(L.nx, L.ny, L.nzl, blk, 32);
  k_norms<MODE, TI><<<grd, blk, 0, s>>>(L, x, xlo, xhi, R, rout, partials);
}

void launch_norms(const LevelK& L, const float* x, const float* xlo, const float* xhi,
                  const RhsK& R, int mode, int tI, float* rout, double2* partials,
                  double2* plane_out, cudaStream_t s) {
  {
  ProfScope ps(KC_NORMS, ncell(L) * (4.0 + rhs_bytes(mode, tI, R) + (rout ? 4.0 : 0.0)), s, ncell(L));
  if (mode == RHS_B) launch_norms_t<RHS_B, float>(L, x, xlo, xhi, R, rout, partials, s);
  else if (tI == 0) launch_norms_t<RHS_G, uint8_t>(L, x, xlo, xhi, R, rout, partials, s);
  else launch_norms_t<RHS_G, float>(L, x, xlo, xhi, R, rout, partials, s);
  }
  ProfScope ps2(KC_UTIL, 0.0, s);
  k_finalize<<<L.nzl, 256, 0, s>>>(partials, norms_blocks_per_plane(L.nx, L.ny), plane_out);
}

static int plane_sums_blocks_per_plane(int nx, int ny) {
  const int gx = (nx + 1023) / 1024;
  return gx * std::max(1, std::min((ny + 1) / 2, 32));
}

void launch_plane_sums(const void* a, int ta, const void* b, int tb, int nx, int ny, int nz,
                       double2* partials, double2* plane_out, cudaStream_t s) {
  int per = 0;
  {
  ProfScope ps(KC_UTIL, (double)nx * ny * nz * ((ta ? 4 : 1) + (b ? (tb ? 4 : 1) : 0)), s);
  // partials per plane <= norms_blocks_per_plane(nx, ny) (the callers' buffers are sized for it)
  per = plane_sums_blocks_per_plane(nx, ny);
  const dim3 grd((nx + 1023) / 1024, per / ((nx + 1023) / 1024), nz);
  auto al = [](const void* p, int t) { return p == nullptr || (t == 0 ? ((uintptr_t)p & 3) == 0 : ((uintptr_t)p & 15) == 0); };
  const bool vec = (nx & 3) == 0 && al(a, ta) && al(b, tb);
#define GDP_PS(TA, TB)                                                                         \
  do {                                                                                         \
    if (vec) k_plane_sums4<TA, TB, true><<<grd, 256, 0, s>>>(a, b, nx, ny, partials);          \
    else k_plane_sums4<TA, TB, false><<<grd, 256, 0, s>>>(a, b, nx, ny, partials);             \
  } while (0)
  if (ta == 1 && tb == 0) GDP_PS(float, uint8_t);
  else if (ta == 1) GDP_PS(float, float);
  else if (tb == 0) GDP_PS(uint8_t, uint8_t);
  else GDP_PS(uint8_t, float);
#undef GDP_PS
  }
  ProfScope ps2(KC_UTIL, 0.0, s);
  k_finalize<<<nz, 256, 0, s>>>(partials, per, plane_out);
}

void launch_finalize(const double2* partials, int per, int nplanes, double2* out, cudaStream_t s) {
  ProfScope ps(KC_UTIL, 0.0, s);
  k_finalize<<<nplanes, 256, 0, s>>>(partials, per, out);
}

static inline int ew_grid(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g > 148 * 32 ? 148 * 32 : (g < 1 ? 1 : g));
}

void launch_rhs(const LevelK& L, const RhsK& R, int tI, float* b, cudaStream_t s) {
  ProfScope ps(KC_UTIL, (double)L.nx * L.ny * L.nzl * ((tI ? 4.0 : 1.0) + (R.vmode == 2 ? 4.0 : 0.0) + 4.0), s);
  dim3 g((L.nx + 255) / 256, L.ny, L.nzl);
  if (tI == 0) k_rhs<uint8_t><<<g, 256, 0, s>>>(L, R, b);
  else k_rhs<float><<<g, 256, 0, s>>>(L, R, b);
}


constexpr int INIT_ROWS = 32;
int init_blocks_per_plane(int nx, int ny) { return ((nx + 1023) / 1024) * ((ny + INIT_ROWS - 1) / INIT_ROWS); }

void launch_init(const LevelK& L, const RhsK& R, int tI, float* x0, float* b, double2* partials, cudaStream_t s,
                 const InitXfer& X) {
  const double n = (double)L.nx * L.ny * L.nzl;
  ProfScope ps(KC_UTIL, n * ((tI ? 4.0 : 1.0) + (R.vmode == 2 ? 4.0 : 0.0) + 8.0) + (X.bc ? 4.0 * X.ncx * X.ncy * L.nzl : 0.0), s);
  dim3 g((L.nx + 1023) / 1024, (L.ny + INIT_ROWS - 1) / INIT_ROWS, L.nzl);
  const bool vec = (L.nx & 3) == 0 && ((uintptr_t)R.I & 15) == 0 && ((uintptr_t)x0 & 15) == 0 &&
                   ((uintptr_t)b & 15) == 0 && (R.vmode != 2 || ((uintptr_t)R.V & 15) == 0);
  if (tI == 0) {
    if (vec) k_init<uint8_t, true><<<g, 256, 0, s>>>(L, R, x0, b, partials, INIT_ROWS, X);
    else k_init<uint8_t, false><<<g, 256, 0, s>>>(L, R, x0, b, partials, INIT_ROWS, X);
  } else {
    if (vec) k_init<float, true><<<g, 256, 0, s>>>(L, R, x0, b, partials, INIT_ROWS, X);
    else k_init<float, false><<<g, 256, 0, s>>>(L, R, x0, b, partials, INIT_ROWS, X);
  }
}

void launch_decode_copy(const void* I, int tI, float* x, long long n, cudaStream_t s) {
  ProfScope ps(KC_UTIL, (double)n * (tI ? 8.0 : 5.0), s);
  if (tI == 0) k_decode_copy<uint8_t><<<ew_grid(n), 256, 0, s>>>(I, x, n);
  else k_decode_copy<float><<<ew_grid(n), 256, 0, s>>>(I, x, n);
}

void launch_add_scalar(float* x, long long n, float v, cudaStream_t s) {
  ProfScope ps(KC_UTIL, (double)n * 8.0, s);
  k_add_scalar<<<ew_grid(n), 256, 0, s>>>(x, n, v);
}

// a9 correction norm: *out = max(*out, max_i |a_i - b_i|) as float bits (values >= 0 order like
// their bit patterns), float4 grid-stride with a warp-shuffle / block max
__global__ void __launch_bounds__(256) k_maxdiff(const float* __restrict__ a, const float* __restrict__ b, long long n,
                                                 int vec, unsigned int* out) {
  float m = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long done = 0;
  if (vec) {
    const long long n4 = n >> 2;
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (long long i = t0; i < n4; i += stride) {
      const float4 u = __ldg(a4 + i), v = __ldg(b4 + i);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(u.x - v.x), fabsf(u.y - v.y)), fmaxf(fabsf(u.z - v.z), fabsf(u.w - v.w))));
    }
    done = n4 << 2;
  }
  for (long long i = done + t0; i < n; i += stride) m = fmaxf(m, fabsf(__ldg(a + i) - __ldg(b + i)));
  if (m != m) m = __int_as_float(0x7f800000);  // a NaN difference reads as +inf (never passes a gate)
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmaxf(m, sm[w]);
    atomicMax(out, __float_as_uint(m));
  }
}

void launch_maxdiff(const float* a, const float* b, long long n, unsigned int* out, cudaStream_t s) {
  ProfScope ps(KC_UTIL, (double)n * 8.0, s);
  const int vec = (((uintptr_t)a | (uintptr_t)b) & 15) == 0;
  k_maxdiff<<<ew_grid(n / 4 + 1), 256, 0, s>>>(a, b, n, vec, out);
}

void launch_axpy(float* x, const float* e, long long n, cudaStream_t s) {
  ProfScope ps(KC_UTIL, (double)n * 12.0, s);
  k_axpy<<<ew_grid(n), 256, 0, s>>>(x, e, n);
}

size_t coarse_smem_bytes(const CoarseK& C) {
  const long long nsys = (long long)C.nx * C.ny * (C.cz ? C.nz : 1);
  const long long nzs = C.cz ? C.nz : 1;
  const long long m = std::max({(long long)C.nx * (C.nx + 1), (long long)C.ny * C.ny, nzs * nzs});
  return (size_t)((2 * nsys + m) * sizeof(float));
}

cudaError_t launch_coarse(const CoarseK& C, const float* b, float* x, cudaStream_t s) {
  const size_t smem = coarse_smem_bytes(C);
  // b read + x write of every coarsest system
  ProfScope ps(KC_COARSE, 8.0 * (double)C.nx * C.ny * C.nz, s);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_coarse_fd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  const int nsys = C.cz ? 1 : C.nz;
  k_coarse_fd<<<nsys, 512, smem, s>>>(C, b, x);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// Coarse tail of a V-cycle in two cooperative launches (the small levels
// are launch- and latency-bound): one persistent grid walks the levels [lc, nl-1) down (zero start,
// nu_pre red-black sweeps, residual restriction) with a grid-wide barrier between the phases, the
// coarsest solve stays its own kernel, and a second grid walks them up (prolongation + correction,
// nu_post sweeps).  Every point runs the reference schedule's arithmetic (rbgs_point,
// restrict_point, prolong_point), so the iterate is bit-identical.  Single-slab levels only.
// ---------------------------------------------------------------------------------
// x_f(cell) += P x_c: the reference prolongation of one fine cell (k_prolong_rows' per-cell order)
__device__ __forceinline__ void prolong_point(const LevelK& L, float* __restrict__ xf, const XferAxis& tx,
                                              const XferAxis& ty, const XferAxis& tz, int ncx, int ncy,
                                              const float* __restrict__ xc, int fx, int fy, int fz) {
  long long Ix, Jx, Iy, Jy, Iz, Jz;
  float txw, tyw, tzw;
  if (ptaps_regular(tx, fx)) ptaps_fast(tx, fx, Ix, Jx, txw); else ptaps(tx, fx, Ix, Jx, txw);
  if (ptaps_regular(ty, fy)) ptaps_fast(ty, fy, Iy, Jy, tyw); else ptaps(ty, fy, Iy, Jy, tyw);
  if (ptaps_regular(tz, L.z0 + fz)) ptaps_fast(tz, L.z0 + fz, Iz, Jz, tzw); else ptaps(tz, L.z0 + fz, Iz, Jz, tzw);
  const long long cplane = (long long)ncx * ncy;
  const float* pI = xc + Iz * cplane;
  const float* pJ = xc + Jz * cplane;
  auto bil = [&](const float* p) {
    const float* rI = p + Iy * ncx;
    const float* rJ = p + Jy * ncx;
    return bilerp(rI[Ix], rI[Jx], rJ[Ix], rJ[Jx], txw, tyw);
  };
  float e = bil(pI);
  if (tzw != 0.f) e = __fmaf_rn(tzw, bil(pJ), __fmul_rn(1.f - tzw, e));
  const long long c = (long long)fz * L.nx * L.ny + (long long)fy * L.nx + fx;
  xf[c] = __fadd_rn(xf[c], e);
}

// grid-wide barrier of the cooperative launch (cooperative_groups: release / acquire at gpu scope)
__device__ __forceinline__ void grid_barrier(unsigned int*, unsigned int&) { cooperative_groups::this_grid().sync(); }

__global__ void __launch_bounds__(256) k_coop_down(const CoopLv* __restrict__ lv, int n, int nu, int zero_first,
                                                   unsigned int* bar) {
  unsigned int gen = 0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (int i = 0; i < n; ++i) {
    const CoopLv V = lv[i];
    const LevelK& L = V.K;
    const long long pl = (long long)L.nx * L.ny, N = pl * L.nzl;
    if (i > 0 || zero_first) {
      for (long long c = tid; c < N; c += nth) V.x[c] = 0.f;
      grid_barrier(bar, gen);
    }
    const RhsK R{V.b, nullptr, nullptr, 0.f, 0};
    const int nxh = (L.nx + 1) / 2;
    const long long NH = (long long)nxh * L.ny * L.nzl;
    for (int k = 0; k < nu; ++k)
      for (int color = 0; color < 2; ++color) {
        for (long long h = tid; h < NH; h += nth) {
          const int ixh = (int)(h % nxh);
          const long long r = h / nxh;
          rbgs_point<RHS_B, float>(L, V.x, nullptr, nullptr, R, color, ixh, (int)(r % L.ny), (int)(r / L.ny));
        }
        grid_barrier(bar, gen);
      }
    const long long NC = (long long)V.ncx * V.ncy * V.nczl;
    for (long long q = tid; q < NC; q += nth) {
      const int cx = (int)(q % V.ncx);
      const long long r = q / V.ncx;
      restrict_point<RHS_B, float>(L, V.x, nullptr, nullptr, R, V.tx, V.ty, V.tz, V.ncx, V.ncy, V.bc, cx,
                                   (int)(r % V.ncy), (int)(r / V.ncy));
    }
    grid_barrier(bar, gen);
  }
}

__global__ void __launch_bounds__(256) k_coop_up(const CoopLv* __restrict__ lv, int n, int nu, unsigned int* bar) {
  unsigned int gen = 0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (int i = n - 1; i >= 0; --i) {
    const CoopLv V = lv[i];
    const LevelK& L = V.K;
    const long long pl = (long long)L.nx * L.ny, N = pl * L.nzl;
    for (long long c = tid; c < N; c += nth) {
      const int fx = (int)(c % L.nx);
      const long long r = c / L.nx;
      prolong_point(L, V.x, V.tx, V.ty, V.tz, V.ncx, V.ncy, V.xc, fx, (int)(r % L.ny), (int)(r / L.ny));
    }
    grid_barrier(bar, gen);
    const RhsK R{V.b, nullptr, nullptr, 0.f, 0};
    const int nxh = (L.nx + 1) / 2;
    const long long NH = (long long)nxh * L.ny * L.nzl;
    for (int k = 0; k < nu; ++k)
      for (int color = 0; color < 2; ++color) {
        for (long long h = tid; h < NH; h += nth) {
          const int ixh = (int)(h % nxh);
          const long long r = h / nxh;
          rbgs_point<RHS_B, float>(L, V.x, nullptr, nullptr, R, color, ixh, (int)(r % L.ny), (int)(r / L.ny));
        }
        if (i > 0 || k < nu - 1 || color == 0) grid_barrier(bar, gen);  // the kernel end orders the last
      }
  }
}

static int coop_grid() {
  static int g = 0;
  if (!g) {
    int dev = 0, nsm = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_coop_down, 256, 0);
    int per2 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_coop_up, 256, 0);
    g = nsm * std::max(1, std::min(std::min(per, per2), 4));
  }
  return g;
}

cudaError_t launch_coop(bool down, const CoopLv* lv, int n, int nu, int zero_first, unsigned int* bar,
                        double cells, double bytes, cudaStream_t s) {
  ProfScope ps(KC_COOP, bytes, s, cells);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(coop_grid());
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency of the whole grid (grid.sync)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (down) return cudaLaunchKernelEx(&cfg, k_coop_down, lv, n, nu, zero_first, bar);
  return cudaLaunchKernelEx(&cfg, k_coop_up, lv, n, nu, bar);
}

}  // namespace gdp
