// gdp_device.cuh — per-voxel arithmetic shared by every kernel of the library.
//
// All schedules (one kernel per half-sweep, fused tile kernels, z-marching kernels)
// call exactly these functions, so a red-black Gauss-Seidel iterate is bit-identical
// whatever the tiling: a point of one colour depends only on points of the other.
//
// Discretisation:
//   A x at cell c = alpha x_c + sum_axes [ cl(i) (x_c - x_{i-1}) + cr(i) (x_c - x_{i+1}) ]
// with link coefficients from a finite-volume rediscretisation on every level:
//   interior link  beta / H^2, links touching a partial last cell (odd sizes under
//   ceil-halving) beta / (d h) with d the centre distance and h the row cell width.
// Level 0 has H = h = 1, i.e. exactly the 7-point Neumann stencil of the paper's
// Constant scheme, diagonal 2(bx+by+bz) in the interior.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gdp {

// 16-byte alignment of an optional pointer (the float4 / cp.async.16 paths need it besides
// nx % 4 == 0; a caller's tensor view may start at any 4-byte offset)
__host__ __device__ __forceinline__ bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

struct AxisC {      // link coefficients of one axis on one level
  int n;            // global cell count along the axis
  float k;          // interior link coefficient
  float kr;         // right link of row n-2 (towards the last cell)
  float kl;         // left link of row n-1 (the last cell)
};

__device__ __forceinline__ float cl(const AxisC& a, long long i) {
  return i <= 0 ? 0.f : (i == a.n - 1 ? a.kl : a.k);
}
__device__ __forceinline__ float cr(const AxisC& a, long long i) {
  return i >= a.n - 1 ? 0.f : (i == a.n - 2 ? a.kr : a.k);
}

struct LevelK {     // one multigrid level as the kernels see it
  int nx, ny, nzl;  // local dims (x, y full; z = this rank's slab)
  long long z0;     // global z of local plane 0
  AxisC ax, ay, az;
  float alpha;      // screening weight (same on every level)
  float omega;      // over-relaxation of the red-black sweeps (1 = Gauss-Seidel)
};

enum RhsMode { RHS_B = 0, RHS_G = 1 };

// Right-hand side of the finest level.
//   RHS_B: explicit b (gdp_vcycle, coarse levels).
//   RHS_G: b = av V - div W G with G = in-plane forward differences of I (Eq. 1 / Eq. 2),
//          evaluated on the fly from I (u8 or f32) and the value target V.
struct RhsK {
  const float* b;
  const void* I;     // gradient source I0
  const float* V;    // value target (vmode 2)
  float av;          // weight of the value term
  int vmode;         // 0: no value term, 1: V = I (decoded), 2: V = float array
  float* vout;       // vmode 2, init pass only: V += vshift is applied and written back here
  float vshift;      //   (phase 1's deferred mean pin, the k_add_scalar arithmetic)
};

// a1: u8 -> u8/255 rounded to fp32 exactly as IEEE division would (the value the oracle
// decodes).  q = u*(1/255) can be off by one ulp; one FMA residual correction restores the
// correctly rounded quotient for every u in [0,255] (verified exhaustively, tests/).
__device__ __forceinline__ float decode_u8(unsigned int u) {
  const float f = (float)u;
  const float r = 1.0f / 255.0f;
  const float q = f * r;
  const float e = __fmaf_rn(-q, 255.0f, f);
  return __fmaf_rn(e, r, q);
}

template <typename T> __device__ __forceinline__ float ldI(const void* p, long long i);
template <> __device__ __forceinline__ float ldI<float>(const void* p, long long i) {
  return __ldg(static_cast<const float*>(p) + i);
}
template <> __device__ __forceinline__ float ldI<uint8_t>(const void* p, long long i) {
  return decode_u8(__ldg(static_cast<const uint8_t*>(p) + i));
}

// Neighbour values of x around cell c.  Where a link does not exist the loader sets
// the neighbour to x_c, so (x_c - x_n) is exactly 0 (never 0 * garbage).
struct Nbr {
  float w, e, s, n, d, u;
};

struct Coef {
  float xl, xr, yl, yr, zl, zr;
  __device__ __forceinline__ float diag(float alpha) const {
    return alpha + ((xl + xr) + (yl + yr)) + (zl + zr);
  }
};

__device__ __forceinline__ Coef coefs(const LevelK& L, int ix, int iy, long long zg) {
  Coef c;
  c.xl = cl(L.ax, ix); c.xr = cr(L.ax, ix);
  c.yl = cl(L.ay, iy); c.yr = cr(L.ay, iy);
  c.zl = cl(L.az, zg); c.zr = cr(L.az, zg);
  return c;
}

// the arithmetic of rhs_g on values already loaded (fused kernels call this directly)
__device__ __forceinline__ float rhs_from(const Coef& k, float Ic, float Iw, float Ie, float Is,
                                          float In, float Vc, float av) {
  float g = __fmul_rn(k.xl, Ic - Iw);
  g = __fmaf_rn(k.xr, Ic - Ie, g);
  g = __fmaf_rn(k.yl, Ic - Is, g);
  g = __fmaf_rn(k.yr, Ic - In, g);
  return __fmaf_rn(av, Vc, g);
}

// Right-hand side at one finest-level cell (a2 / a11): b = av V - div W G with the
// in-plane target gradient G = forward differences of I (Eq. 1, Eq. 2):
//   b_c = sum_{in-plane links} coef * (I_c - I_n)  [+ av V_c]
template <typename TI>
__device__ __forceinline__ float rhs_g(const LevelK& L, const RhsK& R, const Coef& k, long long c,
                                       long long nx) {
  const float Ic = ldI<TI>(R.I, c);
  float Iw = Ic, Ie = Ic, Is = Ic, In = Ic;  // absent link: zero difference
  if (k.xl != 0.f) Iw = ldI<TI>(R.I, c - 1);
  if (k.xr != 0.f) Ie = ldI<TI>(R.I, c + 1);
  if (k.yl != 0.f) Is = ldI<TI>(R.I, c - nx);
  if (k.yr != 0.f) In = ldI<TI>(R.I, c + nx);
  return rhs_from(k, Ic, Iw, Ie, Is, In, R.vmode == 0 ? 0.f : (R.vmode == 1 ? Ic : __ldg(R.V + c)),
                  R.av);
}

// (A x)_c in difference form: alpha x_c + sum_links coef (x_c - x_n).
__device__ __forceinline__ float apply_from(const Coef& k, float alpha, float xc, float xw, float xe,
                                            float xs, float xn, float xd, float xu) {
  float s = __fmul_rn(alpha, xc);
  s = __fmaf_rn(k.xl, xc - xw, s);
  s = __fmaf_rn(k.xr, xc - xe, s);
  s = __fmaf_rn(k.yl, xc - xs, s);
  s = __fmaf_rn(k.yr, xc - xn, s);
  s = __fmaf_rn(k.zl, xc - xd, s);
  s = __fmaf_rn(k.zr, xc - xu, s);
  return s;
}

// Residual r = b - A x at one cell.  Every schedule evaluates exactly this expression.
template <int MODE, typename TI>
__device__ __forceinline__ float residual_at(const LevelK& L, const RhsK& R, const Coef& k,
                                             float xc, const Nbr& nb, long long c, long long nx,
                                             long long plane, float* bval) {
  const float bc = MODE == RHS_B ? R.b[c] : rhs_g<TI>(L, R, k, c, nx);
  if (bval) *bval = bc;
  return __fsub_rn(bc, apply_from(k, L.alpha, xc, nb.w, nb.e, nb.s, nb.n, nb.d, nb.u));
}

// Relaxation weight omega / D of a point: omega times the correctly rounded 1/D (one rounding
// more when omega != 1; exactly 1/D for Gauss-Seidel).  Every schedule uses this value.
__device__ __forceinline__ float relax_inv(float omega, float D) { return __fmul_rn(omega, __frcp_rn(D)); }

// (Over-relaxed) Gauss-Seidel point update in correction form: x_c <- x_c + omega r_c / D_c
// (H1), x_c + r * relax_inv as one FMA.
__device__ __forceinline__ float gs_update(float xc, float r, float D, float omega) {
  return __fmaf_rn(r, relax_inv(omega, D), xc);
}

// Cell-centre coordinate (finest-grid units) of cell i on an axis of n cells of width H,
// the last one of width hl (partial under ceil-halving).
__device__ __forceinline__ float centre(long long i, int n, float H, float hl) {
  return i < n - 1 ? ((float)i + 0.5f) * H : (float)(n - 1) * H + 0.5f * hl;
}

struct XferAxis {   // transfer geometry of one axis between a fine and a coarse level
  int coarsened;    // 0: identity along this axis
  int nf, nc;       // global counts
  float Hf, hlf;    // fine full / last width
  float Hc, hlc;    // coarse full / last width
};

// Restriction weight of fine cell i inside its parent (volume-weighted child average).
__device__ __forceinline__ float rweight(const XferAxis& a, long long i) {
  if (!a.coarsened) return 1.f;
  const long long I = i >> 1;
  const long long c0 = 2 * I, c1 = 2 * I + 1;
  const float h0 = (c0 == a.nf - 1) ? a.hlf : a.Hf;
  const float h1 = (c1 < a.nf) ? ((c1 == a.nf - 1) ? a.hlf : a.Hf) : 0.f;
  const float hi = (i == c0) ? h0 : h1;
  return hi / (h0 + h1);
}

// child weight product of the restriction (explicit rounding, same in every schedule)
__device__ __forceinline__ float rw3(float wz, float wy, float wx) {
  return __fmul_rn(__fmul_rn(wz, wy), wx);
}

// bilinear combination of the prolongation (explicit rounding, same in every schedule)
__device__ __forceinline__ float bilerp(float a, float b, float c, float d, float tx, float ty) {
  const float r0 = __fmaf_rn(tx, b, __fmul_rn(1.f - tx, a));
  const float r1 = __fmaf_rn(tx, d, __fmul_rn(1.f - tx, c));
  return __fmaf_rn(ty, r1, __fmul_rn(1.f - ty, r0));
}

// Cells away from the faces and from the (possibly partial) last coarse cell have the regular
// taps: J = I -/+ 1 by parity and t = 1/4 exactly (what ptaps computes for them).
__device__ __forceinline__ bool ptaps_regular(const XferAxis& a, long long i) {
  return !a.coarsened || (i >= 1 && (i >> 1) + 1 <= a.nc - 2);
}
__device__ __forceinline__ void ptaps_fast(const XferAxis& a, long long i, long long& I, long long& J,
                                           float& t) {
  if (!a.coarsened) { I = i; J = i; t = 0.f; return; }
  I = i >> 1;
  J = (i & 1) ? I + 1 : I - 1;
  t = 0.25f;
}

// Linear prolongation taps of fine cell i: parent I with weight 1-t, neighbour J with t.
__device__ __forceinline__ void ptaps(const XferAxis& a, long long i, long long& I, long long& J,
                                      float& t) {
  if (!a.coarsened) { I = i; J = i; t = 0.f; return; }
  I = i >> 1;
  const float cf = centre(i, a.nf, a.Hf, a.hlf);
  const float cI = centre(I, a.nc, a.Hc, a.hlc);
  if (cf < cI) J = I - 1;
  else if (cf > cI) J = I + 1;
  else { J = I; t = 0.f; return; }
  if (J < 0 || J >= a.nc) { J = I; t = 0.f; return; }
  const float cJ = centre(J, a.nc, a.Hc, a.hlc);
  t = (cf - cI) / (cJ - cI);
}

}  // namespace gdp
