// gdp_scheme.cu — NEXT-3: the paper's Hybrid and Linear discretisations,
// PAPER.md:305-323 (§4.2).
//
//   Hybrid: the 6-point Laplacian at the finest level, the B-spline prolongation (1/2, 1, 1/2)
//           per axis between levels and Galerkin coarse operators P^T A P (27-point);
//   Linear: the first-order B-spline finite-element operator (27-point) at every level, the same
//           transfers, Galerkin coarse operators.
//
// Every level operator of both schemes has the tensor-sum form:
//
//   A = alpha Mx(x)My(x)Mz + bx Kx(x)My(x)Mz + by Mx(x)Ky(x)Mz + bz Mx(x)My(x)Kz
//
// with per-axis tridiagonal "mass" M and "stiffness" K (Hybrid fine: M = I, K = D^T D; Linear
// fine: the hat-function mass / stiffness on [0, n-1]; coarse: P^T M P and P^T K P of the level
// above, because P is a tensor product).  A level is therefore 6 tridiagonal 1D tables, and
// the 27 coefficients of a cell are formed in registers from its three table rows: no 27-point
// coefficient arrays in HBM.  The operator is applied in difference form
//   (A x)_v = rs_v x_v + sum_{n != v} A_vn (x_n - x_v),   rs_v = alpha prod_d rowsum(M_d)_v
// (K rows sum to 0), which keeps the fp32 residual of the singular phase-1 system at rounding
// level as the 7-point path does (reading c-12).
//
// Smoother: multicoloured Gauss-Seidel, one launch per colour — 8 colours (parity of i, j, k) for
// 27-point levels, 4 per slice for the 2D systems of phase 2, red-black where every M is diagonal
// (the Hybrid finest level).  Coarsest level: fast diagonalisation with generalised per-axis
// eigenvectors (K v = lambda M v, V^T M V = I), exact, the constant mode dropped when alpha = 0.
//
// Single rank, in core.  The 7-point (Constant) path of gdp_solver.cu is untouched.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "gdp_internal.h"

namespace gdp {

#define CKS(call)                                                                         \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return set_err(GDP_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define RETS(call)                   \
  do {                               \
    int r_ = (call);                 \
    if (r_ != GDP_OK) return r_;     \
  } while (0)

// ---------------------------------------------------------------------------------------------
// Device view of a level
// ---------------------------------------------------------------------------------------------
// one table row per index of an axis: (m_lo, m_d, m_hi, rowsum M) (k_lo, k_d, k_hi, 0)
struct TsRow { float4 m, k; };

struct TsLv {
  int nx, ny, nz;
  const TsRow* tx;
  const TsRow* ty;
  const TsRow* tz;   // unused (z uncoupled) when per_slice
  float alpha, bx, by, bz;
  // translation-invariant interior: rows ulo[d]..uhi[d] of every axis table are equal, so the 27
  // coefficients there are constants (cst[(c+1)*9 + (b+1)*3 + (a+1)], diagonal cst[13], row sum crs)
  int ulo[3], uhi[3];
  float cst[27];
  float crs;
  int seven;  // every M is the identity: 7-point operator from the K tables
};

__device__ __forceinline__ float tsel(const float4& v, int a) { return a < 0 ? v.x : (a == 0 ? v.y : v.z); }

// S = sum_{n != v} A_vn (x_n - x_v) and the diagonal A_vv of cell (i, j, k); Z: z coupling;
// L.seven: every M of the level is the identity (the Hybrid finest level: 7-point, K tables only).
// Neighbours outside the grid have zero coefficients; their indices are clamped to v (d = 0).
template <bool Z, typename LD>
__device__ __forceinline__ void ts_row(const TsLv& L, int i, int j, int k, size_t v, LD ld, float xv, float& S,
                                       float& diag, float& rs) {
  if (L.seven) {  // boundary coefficients are 0 in the K tables; the clamped neighbour is v itself
    const float4 kx = L.tx[i].k, ky = L.ty[j].k;
    float s = L.bx * (kx.x * ((i > 0 ? ld.off(v, -1, 0, 0) : xv) - xv) + kx.z * ((i + 1 < L.nx ? ld.off(v, 1, 0, 0) : xv) - xv)) +
              L.by * (ky.x * ((j > 0 ? ld.off(v, 0, -1, 0) : xv) - xv) + ky.z * ((j + 1 < L.ny ? ld.off(v, 0, 1, 0) : xv) - xv));
    float d = L.alpha + L.bx * kx.y + L.by * ky.y;
    if (Z) {
      const float4 kz = L.tz[k].k;
      s += L.bz * (kz.x * ((k > 0 ? ld.off(v, 0, 0, -1) : xv) - xv) + kz.z * ((k + 1 < L.nz ? ld.off(v, 0, 0, 1) : xv) - xv));
      d += L.bz * kz.y;
    }
    S = s;
    diag = d;
    rs = L.alpha;
    return;
  }
  if (i >= L.ulo[0] && i <= L.uhi[0] && j >= L.ulo[1] && j <= L.uhi[1] &&
      (!Z || (k >= L.ulo[2] && k <= L.uhi[2]))) {  // interior: constant coefficients, no table loads
    float s = 0.f;
#pragma unroll
    for (int c = -1; c <= 1; ++c) {
      if (!Z && c != 0) continue;
#pragma unroll
      for (int b = -1; b <= 1; ++b)
#pragma unroll
        for (int a = -1; a <= 1; ++a) {
          if (a == 0 && b == 0 && c == 0) continue;
          s += L.cst[(c + 1) * 9 + (b + 1) * 3 + (a + 1)] * (ld.off(v, a, b, c) - xv);
        }
    }
    S = s;
    diag = L.cst[13];
    rs = L.crs;
    return;
  }
  const TsRow X = L.tx[i], Y = L.ty[j];
  TsRow Zr;
  if (Z) Zr = L.tz[k];
  else { Zr.m = make_float4(0.f, 1.f, 0.f, 1.f); Zr.k = make_float4(0.f, 0.f, 0.f, 0.f); }
  const float ax[3] = {L.alpha * X.m.x + L.bx * X.k.x, L.alpha * X.m.y + L.bx * X.k.y, L.alpha * X.m.z + L.bx * X.k.z};
  const float mx[3] = {X.m.x, X.m.y, X.m.z};
  const int im = i > 0 ? i - 1 : i, ip = i + 1 < L.nx ? i + 1 : i;
  float s = 0.f;
  diag = 0.f;
#pragma unroll
  for (int c = -1; c <= 1; ++c) {
    if (!Z && c != 0) continue;
    const float zm = tsel(Zr.m, c), zk = tsel(Zr.k, c);
    const int kk = c < 0 ? (k > 0 ? k - 1 : k) : (c > 0 ? (k + 1 < L.nz ? k + 1 : k) : k);
#pragma unroll
    for (int b = -1; b <= 1; ++b) {
      const float ym = tsel(Y.m, b), yk = tsel(Y.k, b);
      const float p = zm * ym;
      const float q = zm * (L.by * yk) + L.bz * zk * ym;
      if (b == 0 && c == 0) diag = p * ax[1] + q * mx[1];
      if (p == 0.f && q == 0.f) continue;
      const int jj = b < 0 ? (j > 0 ? j - 1 : j) : (b > 0 ? (j + 1 < L.ny ? j + 1 : j) : j);
      const float d0 = ld(im, jj, kk) - xv;
      const float d1 = (b == 0 && c == 0) ? 0.f : ld(i, jj, kk) - xv;
      const float d2 = ld(ip, jj, kk) - xv;
      const float u = ax[0] * d0 + ax[1] * d1 + ax[2] * d2;
      const float w = mx[0] * d0 + mx[1] * d1 + mx[2] * d2;
      s += p * u + q * w;
    }
  }
  S = s;
  rs = L.alpha * X.m.w * Y.m.w * Zr.m.w;
}

struct LdF {
  const float* x;
  int nx, ny;
  __device__ float operator()(int i, int j, int k) const { return __ldg(x + ((size_t)k * ny + j) * nx + i); }
  __device__ float off(size_t v, int a, int b, int c) const {
    return __ldg(x + (long long)v + a + (long long)b * nx + (long long)c * nx * ny);
  }
};
struct LdU8 {
  const uint8_t* x;
  int nx, ny;
  __device__ float operator()(int i, int j, int k) const {
    return decode_u8(__ldg(x + ((size_t)k * ny + j) * nx + i));
  }
  __device__ float off(size_t v, int a, int b, int c) const {
    return decode_u8(__ldg(x + (long long)v + a + (long long)b * nx + (long long)c * nx * ny));
  }
};
// shared-memory tile of three planes (k - 1, k, k + 1) of the staged region (k_ts_gs_tile): global
// (i, j, k) -> slot of plane k, row j - j0, column i - i0; `v` is the cell's index within its plane
// tile.  Cells outside the grid are staged as 0: their coefficients are 0, so they add 0 * (0 - x_v).
struct LdS {
  const float *pm, *p0, *pp;  // planes k - 1, k, k + 1 (pm, pp unused without z coupling)
  int i0, j0, k, sy;
  __device__ const float* pl(int c) const { return c < 0 ? pm : (c > 0 ? pp : p0); }
  __device__ float operator()(int i, int j, int kk) const { return pl(kk - k)[(j - j0) * sy + (i - i0)]; }
  __device__ float off(size_t v, int a, int b, int c) const { return pl(c)[(int)v + a + b * sy]; }
};

// one colour of the multicoloured Gauss-Seidel sweep: ncol 8 (i, j, k parities), 4 (i, j parities,
// every slice) or 2 (red-black, (i + j + k) parity)
// Each thread updates NPT cells of the colour in rows NPT apart (a block covers NPT x blockDim.y
// row slots), computing all of them before storing any: the loads of the NPT cells are in flight
// together (the launches are latency-bound at one cell per thread; neighbours of a colour are
// never written by the same launch, so the order of loads and stores does not matter).
constexpr int NPT = 4;

template <bool Z>
__global__ void __launch_bounds__(256) k_ts_gs(TsLv L, float* __restrict__ x, const float* __restrict__ b,
                                               int ncol, int colour, float omega) {
  const int ih = blockIdx.x * blockDim.x + threadIdx.x;
  const int j0 = blockIdx.y * blockDim.y * NPT + threadIdx.y;
  const int k0 = blockIdx.z;
  float nv[NPT];
  size_t vv[NPT];
  bool ok[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    int j = j0 + q * blockDim.y, k = k0, i;
    if (ncol == 2) {
      i = 2 * ih + ((j + k + colour) & 1);
    } else {
      i = 2 * ih + (colour & 1);
      j = 2 * j + ((colour >> 1) & 1);
      if (ncol == 8) k = 2 * k + ((colour >> 2) & 1);
    }
    ok[q] = i < L.nx && j < L.ny && k < L.nz;
    vv[q] = ((size_t)k * L.ny + j) * L.nx + i;
    nv[q] = 0.f;
    if (ok[q]) {
      const size_t v = vv[q];
      const float xv = __ldg(x + v);
      float S, dg, rs;
      ts_row<Z>(L, i, j, k, v, LdF{x, L.nx, L.ny}, xv, S, dg, rs);
      const float r = __ldg(b + v) - (rs * xv + S);
      nv[q] = xv + omega * r / dg;
    }
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q)
    if (ok[q]) x[vv[q]] = nv[q];
}

// Half of a multicoloured sweep of a 27-point level in shared-memory tiles: the planes of parity
// ck (slices of parity ck without z coupling) get their four in-plane colours (ci, cj) = (0,0),
// (1,0), (0,1), (1,1), which is the colour order ck*4 + ci + 2cj of the one-launch-per-colour path:
// colours of plane k read planes k +- 1 (the other parity, unchanged by this launch) and earlier
// colours of plane k only, so plane-by-plane order gives the same iterate bit for bit.  A CTA owns a
// GT_X x GT_Y tile and marches over the planes of the parity with a three-plane ring; the tile is
// staged with a GT_H = 4 halo and colour phase p recomputes the halo cells within 3 - p of the tile
// (a colour's update reads its 26 neighbours only), so no CTA waits on another.  xin -> xout:
// planes of the other parity are copied through (two launches, ck = 0 then 1, return the iterate
// to the first buffer).  One HBM read and write of x per half-sweep instead of four (per colour).
constexpr int GT_X = 64, GT_Y = 32, GT_H = 4, GT_T = 256;
constexpr int GS_X = GT_X + 2 * GT_H, GS_Y = GT_Y + 2 * GT_H;

template <bool Z>
__global__ void __launch_bounds__(GT_T) k_ts_gs_tile(TsLv L, const float* __restrict__ xin, float* __restrict__ xout,
                                                     const float* __restrict__ b, int ck, float omega, int chunk) {
  __shared__ float sx[3][GS_Y * GS_X];  // planes p at slot p mod 3
  __shared__ float sb[GS_Y * GS_X];
  const int i0 = blockIdx.x * GT_X - GT_H, j0 = blockIdx.y * GT_Y - GT_H;
  const int tid = threadIdx.x;
  const size_t plane = (size_t)L.nx * L.ny;
  auto slot = [](int p) { return ((p % 3) + 3) % 3; };
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = GT_T / 32;
  auto stage = [&](float* dst, const float* src, int p) {  // region of plane p (0 outside the grid)
    const bool pin = p >= 0 && p < L.nz;
    for (int r = warp; r < GS_Y; r += NW) {
      const int j = j0 + r;
      const bool rin = pin && j >= 0 && j < L.ny;
      const float* row = src + (rin ? p * plane + (size_t)j * L.nx : 0);
      for (int c = lane; c < GS_X; c += 32) {
        const int i = i0 + c;
        dst[r * GS_X + c] = (rin && i >= 0 && i < L.nx) ? row[i] : 0.f;
      }
    }
  };
  auto store = [&](const float* src, int p) {  // tile interior of plane p -> xout
    for (int r = warp; r < GT_Y; r += NW) {
      const int j = j0 + GT_H + r;
      if (j >= L.ny) break;
      float* row = xout + p * plane + (size_t)j * L.nx;
      for (int c = lane; c < GT_X; c += 32) {
        const int i = i0 + GT_H + c;
        if (i < L.nx) row[i] = src[(r + GT_H) * GS_X + c + GT_H];
      }
    }
  };
  bool first = true;
  const int kend = min(L.nz, ck + 2 * (int)(blockIdx.z + 1) * chunk);  // this CTA's planes of the parity
  for (int k = ck + 2 * (int)blockIdx.z * chunk; k < kend; k += 2) {
    __syncthreads();  // the previous step's stores have read their slots
    if (first && k >= 1) {
      stage(sx[slot(k - 1)], xin, k - 1);
      __syncthreads();
      store(sx[slot(k - 1)], k - 1);  // the other parity's plane below the first: copied through
    }
    first = false;
    stage(sx[slot(k)], xin, k);
    if (k + 1 < L.nz) stage(sx[slot(k + 1)], xin, k + 1);
    else if (Z) stage(sx[slot(k + 1)], xin, k + 1);  // zeros (out of the grid)
    stage(sb, b, k);
    __syncthreads();
    float* xs = sx[slot(k)];
    LdS ld;
    ld.pm = sx[slot(k - 1)];
    ld.p0 = xs;
    ld.pp = sx[slot(k + 1)];
    ld.i0 = i0; ld.j0 = j0; ld.k = k; ld.sy = GS_X;
#pragma unroll 1
    for (int ph = 0; ph < 4; ++ph) {
      const int ci = ph & 1, cj = ph >> 1, m = GT_H - 1 - ph;  // cells within m of the tile
      const int rlo = GT_H - m, clo = GT_H - m;
      // first row / column of the region with the colour's global parity
      const int r1 = rlo + (((j0 + rlo) & 1) != cj), c1 = clo + (((i0 + clo) & 1) != ci);
      const int nr = (GT_Y + 2 * m - (r1 - rlo) + 1) / 2, nc = (GT_X + 2 * m - (c1 - clo) + 1) / 2;
      for (int t = tid; t < nr * nc; t += GT_T) {
        const int rr = t / nc, cc = t - rr * nc;
        const int r = r1 + 2 * rr, c = c1 + 2 * cc;
        const int i = i0 + c, j = j0 + r;
        if (i < 0 || i >= L.nx || j < 0 || j >= L.ny) continue;
        const int v = r * GS_X + c;
        const float xv = xs[v];
        float S, dg, rs;
        ts_row<Z>(L, i, j, k, (size_t)v, ld, xv, S, dg, rs);
        const float rv = sb[v] - (rs * xv + S);
        xs[v] = xv + omega * rv / dg;
      }
      __syncthreads();
    }
    store(xs, k);
    if (k + 1 < L.nz) store(sx[slot(k + 1)], k + 1);  // the other parity's plane above: copied through
  }
}

// r = b - A x (r may be null) with fp64 partials (sum r^2, sum b^2) per block; a block row covers
// one slice (blockIdx.z = k) so per-slice sums are a fixed-order reduction of its blocks; NPT
// rows per thread (the block reduction is the costly part at one cell per thread)
template <bool Z>
__global__ void __launch_bounds__(256) k_ts_resid(TsLv L, const float* __restrict__ x, const float* __restrict__ b,
                                                  float* __restrict__ r, double2* __restrict__ part) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j0 = blockIdx.y * blockDim.y * NPT + threadIdx.y;
  const int k = blockIdx.z;
  double a2 = 0.0, b2 = 0.0;
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    const int j = j0 + q * blockDim.y;
    if (i < L.nx && j < L.ny) {
      const size_t v = ((size_t)k * L.ny + j) * L.nx + i;
      const float xv = __ldg(x + v);
      float S, dg, rs;
      ts_row<Z>(L, i, j, k, v, LdF{x, L.nx, L.ny}, xv, S, dg, rs);
      const float bv = __ldg(b + v);
      const float rv = bv - (rs * xv + S);
      if (r) r[v] = rv;
      a2 += (double)rv * rv;
      b2 += (double)bv * bv;
    }
  }
  if (part) {
    block_sum2(a2, b2);
    if (threadIdx.x == 0 && threadIdx.y == 0)
      part[((size_t)k * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = make_double2(a2, b2);
  }
}

// out (+)= A u with A in difference form; u f32 or u8 (decoded as the 7-point path decodes it)
template <bool Z, typename LD>
__global__ void __launch_bounds__(256) k_ts_apply(TsLv L, LD ld, float* __restrict__ out, int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= L.nx || j >= L.ny) return;
  const size_t v = ((size_t)k * L.ny + j) * L.nx + i;
  const float uv = ld(i, j, k);
  float S, dg, rs;
  ts_row<Z>(L, i, j, k, v, ld, uv, S, dg, rs);
  const float y = rs * uv + S;
  out[v] = accumulate ? out[v] + y : y;
}

// per-axis transfer (reading L-4): coarsened axes map fine i to coarse i/2 (even) or to
// i/2, i/2 + 1 with 1/2, 1/2 (odd; weight 1 on i/2 when i/2 + 1 does not exist)
struct TsXfer {
  int fx, fy, fz, cx, cy, cz;
  int co_x, co_y, co_z;
};

__device__ __forceinline__ int xf_parents(int i, int co, int nc, int* I, float* w) {
  if (!co) { I[0] = i; w[0] = 1.f; return 1; }
  const int h = i >> 1;
  if (!(i & 1)) { I[0] = h; w[0] = 1.f; return 1; }
  if (h + 1 < nc) { I[0] = h; w[0] = 0.5f; I[1] = h + 1; w[1] = 0.5f; return 2; }
  I[0] = h; w[0] = 1.f; return 1;
}

// coarse b = P^T r: gather the fine children (2I-1, 2I, 2I+1 per coarsened axis)
__device__ __forceinline__ int xf_children(int I, int co, int nf, int nc, int* i, float* w) {
  if (!co) { i[0] = I; w[0] = 1.f; return 1; }
  int n = 0;
  if (2 * I - 1 >= 0) { i[n] = 2 * I - 1; w[n++] = 0.5f; }
  i[n] = 2 * I; w[n++] = 1.f;
  if (2 * I + 1 < nf) { i[n] = 2 * I + 1; w[n++] = (I + 1 < nc) ? 0.5f : 1.f; }
  return n;
}

__global__ void __launch_bounds__(256) k_ts_restrict(TsXfer T, const float* __restrict__ r, float* __restrict__ bc) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int J = blockIdx.y * blockDim.y + threadIdx.y;
  const int K = blockIdx.z;
  if (I >= T.cx || J >= T.cy) return;
  int ix[3], iy[3], iz[3];
  float wx[3], wy[3], wz[3];
  const int nx = xf_children(I, T.co_x, T.fx, T.cx, ix, wx);
  const int ny = xf_children(J, T.co_y, T.fy, T.cy, iy, wy);
  const int nz = xf_children(K, T.co_z, T.fz, T.cz, iz, wz);
  float s = 0.f;
  for (int c = 0; c < nz; ++c)
    for (int bb = 0; bb < ny; ++bb) {
      const float* row = r + ((size_t)iz[c] * T.fy + iy[bb]) * T.fx;
      float t = 0.f;
      for (int a = 0; a < nx; ++a) t += wx[a] * __ldg(row + ix[a]);
      s += wz[c] * wy[bb] * t;
    }
  bc[((size_t)K * T.cy + J) * T.cx + I] = s;
}

__global__ void __launch_bounds__(256) k_ts_prolong(TsXfer T, const float* __restrict__ xc, float* __restrict__ xf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= T.fx || j >= T.fy) return;
  int Ix[2], Iy[2], Iz[2];
  float wx[2], wy[2], wz[2];
  const int nx = xf_parents(i, T.co_x, T.cx, Ix, wx);
  const int ny = xf_parents(j, T.co_y, T.cy, Iy, wy);
  const int nz = xf_parents(k, T.co_z, T.cz, Iz, wz);
  float s = 0.f;
  for (int c = 0; c < nz; ++c)
    for (int bb = 0; bb < ny; ++bb) {
      const float* row = xc + ((size_t)Iz[c] * T.cy + Iy[bb]) * T.cx;
      float t = 0.f;
      for (int a = 0; a < nx; ++a) t += wx[a] * __ldg(row + Ix[a]);
      s += wz[c] * wy[bb] * t;
    }
  const size_t v = ((size_t)k * T.fy + j) * T.fx + i;
  xf[v] += s;
}

// the same with x coarsened: a thread owns the fine pair (2I, 2I + 1), which shares the coarse
// columns I, I + 1 of each parent row (half the coarse loads); per cell the sum is the generic
// kernel's (rows outer, columns inner), so both kernels give the same values
__global__ void __launch_bounds__(256) k_ts_prolong2(TsXfer T, const float* __restrict__ xc, float* __restrict__ xf) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  const int i0 = 2 * I;
  if (i0 >= T.fx || j >= T.fy) return;
  int Iy[2], Iz[2];
  float wy[2], wz[2];
  const int ny = xf_parents(j, T.co_y, T.cy, Iy, wy);
  const int nz = xf_parents(k, T.co_z, T.cz, Iz, wz);
  const bool has1 = i0 + 1 < T.fx, two = I + 1 < T.cx;  // odd cell exists / has a right parent
  float s0 = 0.f, s1 = 0.f;
  for (int c = 0; c < nz; ++c)
    for (int bb = 0; bb < ny; ++bb) {
      const float* row = xc + ((size_t)Iz[c] * T.cy + Iy[bb]) * T.cx;
      const float a = __ldg(row + I);
      const float t0 = 1.f * a;
      float t1 = two ? 0.5f * a : 1.f * a;
      if (two) t1 += 0.5f * __ldg(row + I + 1);
      const float w = wz[c] * wy[bb];
      s0 += w * t0;
      s1 += w * t1;
    }
  float* out = xf + ((size_t)k * T.fy + j) * T.fx + i0;
  out[0] += s0;
  if (has1) out[1] += s1;
}

// coarsest solve by fast diagonalisation, one CTA per independent system (all slices of a
// per-slice level share the x / y factors): y = V^T b along each axis, y /= (alpha + sum beta
// lambda) (0 for the null mode), x = V y.  Vd: n_d x n_d row-major, column p = eigenvector p.
struct TsCoarse {
  int nx, ny, nz, per_slice;
  const float* Vx; const float* Vy; const float* Vz;
  const float* inv;  // nx*ny*(per_slice ? 1 : nz) inverse eigenvalues, x fastest
};

__device__ void ts_axis(const float* __restrict__ src, float* __restrict__ dst, const float* __restrict__ V,
                        int nx, int ny, int nz, int axis, bool transpose) {
  const int N = nx * ny * nz;
  const int n = axis == 0 ? nx : (axis == 1 ? ny : nz);
  const int st = axis == 0 ? 1 : (axis == 1 ? nx : nx * ny);
  for (int t = threadIdx.x; t < N; t += blockDim.x) {
    const int x = t % nx, y = (t / nx) % ny, z = t / (nx * ny);
    const int o = axis == 0 ? x : (axis == 1 ? y : z);
    const int base = t - o * st;
    float s = 0.f;
    for (int q = 0; q < n; ++q) {
      const float vv = transpose ? __ldg(V + q * n + o) : __ldg(V + o * n + q);
      s += vv * src[base + q * st];
    }
    dst[t] = s;
  }
  __syncthreads();
}

// (b and x may alias: every CTA reads its system into shared memory before it writes)
__global__ void __launch_bounds__(1024) k_ts_coarse(TsCoarse C, const float* b, float* x) {
  extern __shared__ float sm[];
  const int nzs = C.per_slice ? 1 : C.nz;
  const int N = C.nx * C.ny * nzs;
  float* s0 = sm;
  float* s1 = sm + N;
  const size_t off = (size_t)blockIdx.x * N;
  for (int t = threadIdx.x; t < N; t += blockDim.x) s0[t] = b[off + t];
  __syncthreads();
  ts_axis(s0, s1, C.Vx, C.nx, C.ny, nzs, 0, true);
  ts_axis(s1, s0, C.Vy, C.nx, C.ny, nzs, 1, true);
  float* a = s0;
  float* c = s1;
  if (!C.per_slice) { ts_axis(s0, s1, C.Vz, C.nx, C.ny, nzs, 2, true); a = s1; c = s0; }
  for (int t = threadIdx.x; t < N; t += blockDim.x) a[t] *= __ldg(C.inv + t);
  __syncthreads();
  if (!C.per_slice) { ts_axis(a, c, C.Vz, C.nx, C.ny, nzs, 2, false); float* tmp = a; a = c; c = tmp; }
  ts_axis(a, c, C.Vy, C.nx, C.ny, nzs, 1, false);
  ts_axis(c, a, C.Vx, C.nx, C.ny, nzs, 0, false);
  for (int t = threadIdx.x; t < N; t += blockDim.x) x[off + t] = a[t];
}

__global__ void k_ts_add(float* __restrict__ x, const float* __restrict__ e, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] += e[i];
}

// fixed-order fp64 sums of per-block partials: out[g] = sum of partials [g*n, (g+1)*n)
__global__ void k_ts_sum(const double2* __restrict__ part, int n, double2* __restrict__ out) {
  double a = 0.0, b = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const double2 p = part[(size_t)blockIdx.x * n + t];
    a += p.x;
    b += p.y;
  }
  block_sum2(a, b);
  if (threadIdx.x == 0) out[blockIdx.x] = make_double2(a, b);
}

// per-slice fp64 sums of (x, decoded I0) for the mean pin
template <typename LD>
__global__ void k_ts_means(const float* __restrict__ x, LD ld, int nx, int ny, double2* __restrict__ out) {
  const int k = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (int t = threadIdx.x; t < nx * ny; t += blockDim.x) {
    a += x[(size_t)k * nx * ny + t];
    b += ld(t % nx, t / nx, k);
  }
  block_sum2(a, b);
  if (threadIdx.x == 0) out[k] = make_double2(a, b);
}

template <typename LD>
__global__ void k_ts_copy(LD ld, int nx, int ny, float* __restrict__ out, float shift) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= nx || j >= ny) return;
  out[((size_t)k * ny + j) * nx + i] = ld(i, j, k) + shift;
}

// ---------------------------------------------------------------------------------------------
// Host: per-axis tables, Galerkin products, level chain
// ---------------------------------------------------------------------------------------------
struct Tri {  // symmetric tridiagonal n x n in fp64: lo[i] = A(i, i-1), d[i] = A(i, i), hi[i] = A(i, i+1)
  std::vector<double> lo, d, hi;
  int n() const { return (int)d.size(); }
  double at(int i, int j) const {
    if (j == i) return d[i];
    if (j == i - 1) return lo[i];
    if (j == i + 1) return hi[i];
    return 0.0;
  }
};

static Tri tri_zero(int n) { Tri t; t.lo.assign(n, 0.0); t.d.assign(n, 0.0); t.hi.assign(n, 0.0); return t; }

// fine tables: Linear = hat mass / stiffness on [0, n-1] (reading L-1); Hybrid = I / D^T D
static void fine_axis(int scheme, int n, Tri& M, Tri& K) {
  M = tri_zero(n);
  K = tri_zero(n);
  if (n == 1) { M.d[0] = 1.0; return; }
  for (int e = 0; e + 1 < n; ++e) {  // element [e, e+1]
    if (scheme == GDP_SCHEME_LINEAR) {
      M.d[e] += 1.0 / 3.0; M.d[e + 1] += 1.0 / 3.0; M.hi[e] += 1.0 / 6.0; M.lo[e + 1] += 1.0 / 6.0;
    }
    K.d[e] += 1.0; K.d[e + 1] += 1.0; K.hi[e] -= 1.0; K.lo[e + 1] -= 1.0;
  }
  if (scheme != GDP_SCHEME_LINEAR)
    for (int i = 0; i < n; ++i) M.d[i] = 1.0;
}

// P of reading L-4 as (index, weight) lists per fine row
static void xfer_rows(int nf, std::vector<std::vector<std::pair<int, double>>>& P) {
  const int nc = (nf + 1) / 2;
  P.assign(nf, {});
  for (int i = 0; i < nf; ++i) {
    const int h = i / 2;
    if (i % 2 == 0) P[i] = {{h, 1.0}};
    else if (h + 1 < nc) P[i] = {{h, 0.5}, {h + 1, 0.5}};
    else P[i] = {{h, 1.0}};
  }
}

// P^T A P (tridiagonal again: coarse supports 2I-1..2I+1 overlap only for |I - J| <= 1)
static Tri galerkin_1d(const Tri& A) {
  const int nf = A.n(), nc = (nf + 1) / 2;
  std::vector<std::vector<std::pair<int, double>>> P;
  xfer_rows(nf, P);
  std::vector<double> C((size_t)nc * nc, 0.0);
  for (int i = 0; i < nf; ++i)
    for (int j = std::max(0, i - 1); j <= std::min(nf - 1, i + 1); ++j) {
      const double a = A.at(i, j);
      if (a == 0.0) continue;
      for (auto& pi : P[i])
        for (auto& pj : P[j]) C[(size_t)pi.first * nc + pj.first] += pi.second * a * pj.second;
    }
  Tri t = tri_zero(nc);
  for (int I = 0; I < nc; ++I) {
    t.d[I] = C[(size_t)I * nc + I];
    if (I > 0) t.lo[I] = C[(size_t)I * nc + I - 1];
    if (I + 1 < nc) t.hi[I] = C[(size_t)I * nc + I + 1];
  }
  return t;
}

static std::vector<TsRow> rows_of(const Tri& M, const Tri& K) {
  std::vector<TsRow> r(M.n());
  for (int i = 0; i < M.n(); ++i) {
    const double rs = M.lo[i] + M.d[i] + M.hi[i];
    r[i].m = make_float4((float)M.lo[i], (float)M.d[i], (float)M.hi[i], (float)rs);
    r[i].k = make_float4((float)K.lo[i], (float)K.d[i], (float)K.hi[i], 0.f);
  }
  return r;
}

static bool is_diag(const Tri& M) {
  for (int i = 0; i < M.n(); ++i)
    if (M.lo[i] != 0.0 || M.hi[i] != 0.0) return false;
  return true;
}

// generalised eigenvectors of (K, M): V^T M V = I, V^T K V = diag(lam); M = L L^T (Cholesky),
// C = L^-1 K L^-T = Q diag(lam) Q^T, V = L^-T Q
static void gen_eig(const Tri& M, const Tri& K, std::vector<double>& V, std::vector<double>& lam) {
  const int n = M.n();
  std::vector<double> Lc((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = M.at(i, j);
      for (int k = 0; k < j; ++k) s -= Lc[(size_t)i * n + k] * Lc[(size_t)j * n + k];
      Lc[(size_t)i * n + j] = (i == j) ? std::sqrt(s) : s / Lc[(size_t)j * n + j];
    }
  // Li = L^-1 (lower triangular)
  std::vector<double> Li((size_t)n * n, 0.0);
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= Lc[(size_t)i * n + k] * Li[(size_t)k * n + c];
      Li[(size_t)i * n + c] = s / Lc[(size_t)i * n + i];
    }
  std::vector<double> T((size_t)n * n, 0.0), C((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)  // T = Li K
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = std::max(0, j - 1); k <= std::min(n - 1, j + 1); ++k) s += Li[(size_t)i * n + k] * K.at(k, j);
      T[(size_t)i * n + j] = s;
    }
  for (int i = 0; i < n; ++i)  // C = T Li^T
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += T[(size_t)i * n + k] * Li[(size_t)j * n + k];
      C[(size_t)i * n + j] = s;
    }
  for (int i = 0; i < n; ++i)  // symmetrise the rounding
    for (int j = 0; j < i; ++j) C[(size_t)i * n + j] = C[(size_t)j * n + i] = 0.5 * (C[(size_t)i * n + j] + C[(size_t)j * n + i]);
  std::vector<double> Q;
  jacobi_eig(n, C, Q, lam);
  V.assign((size_t)n * n, 0.0);  // V = Li^T Q
  for (int i = 0; i < n; ++i)
    for (int p = 0; p < n; ++p) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += Li[(size_t)k * n + i] * Q[(size_t)k * n + p];
      V[(size_t)i * n + p] = s;
    }
}

struct TsLevelH {
  int n[3];            // nx, ny, nz
  int co[3];           // coarsened from the level above (level >= 1)
  Tri M[3], K[3];
  double H[3];         // cell width in finest units (coupling-strength rule)
  TsRow* dev_rows = nullptr;  // tx | ty | tz
  float* x = nullptr;  // level >= 1: correction
  float* b = nullptr;  // level >= 1: restricted residual
  bool rb = false;     // red-black suffices (every M diagonal)
  int ulo[3], uhi[3];  // per axis: rows equal to the middle row (translation-invariant interior)
};

struct TsKey {
  int scheme;
  long long nx, ny, nz;
  float bx, by, bz, alpha;
  int per_slice, coarse_max;
  bool operator<(const TsKey& o) const {
    return std::tie(scheme, nx, ny, nz, bx, by, bz, alpha, per_slice, coarse_max) <
           std::tie(o.scheme, o.nx, o.ny, o.nz, o.bx, o.by, o.bz, o.alpha, o.per_slice, o.coarse_max);
  }
};

struct TsHier {
  TsKey key{};
  std::vector<TsLevelH> lv;
  Hier* main7 = nullptr;     // Hybrid 3D: the main path's hierarchy of the same finest operator, whose
                             // fused z-march sweeps smooth level 0 (non-owning: cached in the Ctx)
  float* r = nullptr;        // residual scratch of level 0 size
  float* b0 = nullptr;       // finest rhs (whole solves)
  double2* part = nullptr;   // block partials
  size_t part_cap = 0;
  double2* sums = nullptr;   // per-slice sums (device)
  double2* h_sums = nullptr; // pinned mirror
  float* cV[3] = {nullptr, nullptr, nullptr};
  float* cinv = nullptr;
  ~TsHier() {
    for (auto& L : lv) {
      if (L.dev_rows) cudaFree(L.dev_rows);
      if (L.x) cudaFree(L.x);
      if (L.b) cudaFree(L.b);
    }
    if (r) cudaFree(r);
    if (b0) cudaFree(b0);
    if (part) cudaFree(part);
    if (sums) cudaFree(sums);
    if (h_sums) cudaFreeHost(h_sums);
    for (auto* p : cV) if (p) cudaFree(p);
    if (cinv) cudaFree(cinv);
  }
};

struct SchemeCache {
  std::map<TsKey, std::unique_ptr<TsHier>> h;
};

void scheme_cache_destroy(void* p) { delete static_cast<SchemeCache*>(p); }

static size_t cells(const TsLevelH& L) { return (size_t)L.n[0] * L.n[1] * L.n[2]; }

// coupling-strength coarsening (DESIGN.md readings): coarsen the coupled axes whose beta / H^2 is
// >= 1/2 of the strongest; stop when a system has <= coarse_max unknowns and <= 64 cells along
// every coupled axis
static bool ts_coarsen(const TsLevelH& F, const float beta[3], int per_slice, int coarse_max, TsLevelH& C) {
  const int nd = per_slice ? 2 : 3;
  long long sys = (long long)F.n[0] * F.n[1] * (per_slice ? 1 : F.n[2]);
  bool small = sys <= coarse_max;
  for (int d = 0; d < nd; ++d)
    if (beta[d] > 0.f && F.n[d] > 64) small = false;
  if (small) return false;
  double smax = 0.0;
  for (int d = 0; d < nd; ++d)
    if (beta[d] > 0.f && F.n[d] > 1) smax = std::max(smax, beta[d] / (F.H[d] * F.H[d]));
  if (smax == 0.0) return false;
  bool any = false;
  for (int d = 0; d < 3; ++d) {
    const bool co = d < nd && beta[d] > 0.f && F.n[d] > 1 && beta[d] / (F.H[d] * F.H[d]) >= 0.5 * smax;
    C.co[d] = co;
    C.n[d] = co ? (F.n[d] + 1) / 2 : F.n[d];
    C.H[d] = co ? 2.0 * F.H[d] : F.H[d];
    if (co) { C.M[d] = galerkin_1d(F.M[d]); C.K[d] = galerkin_1d(F.K[d]); any = true; }
    else { C.M[d] = F.M[d]; C.K[d] = F.K[d]; }
  }
  return any;
}

static int ts_build(const TsKey& key, std::unique_ptr<TsHier>& out) {
  auto H = std::make_unique<TsHier>();
  H->key = key;
  const float beta[3] = {key.bx, key.by, key.per_slice ? 0.f : key.bz};
  TsLevelH L0{};
  L0.n[0] = (int)key.nx; L0.n[1] = (int)key.ny; L0.n[2] = (int)key.nz;
  for (int d = 0; d < 3; ++d) {
    L0.H[d] = 1.0;
    L0.co[d] = 0;
    if (d == 2 && key.per_slice) {  // independent slices: identity mass, no stiffness
      L0.M[d] = tri_zero(L0.n[d]);
      L0.K[d] = tri_zero(L0.n[d]);
      for (int i = 0; i < L0.n[d]; ++i) L0.M[d].d[i] = 1.0;
    } else {
      fine_axis(key.scheme, L0.n[d], L0.M[d], L0.K[d]);
    }
  }
  H->lv.push_back(L0);
  while (H->lv.size() < GDP_MAX_LEVELS) {
    TsLevelH C{};
    if (!ts_coarsen(H->lv.back(), beta, key.per_slice, key.coarse_max, C)) break;
    H->lv.push_back(C);
  }
  for (auto& L : H->lv) {
    L.rb = is_diag(L.M[0]) && is_diag(L.M[1]) && is_diag(L.M[2]);
    for (int d = 0; d < 3; ++d) {  // the interior range whose rows equal the middle row
      const Tri &M = L.M[d], &K = L.K[d];
      const int n = M.n(), mid = n / 2;
      auto same = [&](int i) {
        return i >= 1 && i + 1 < n && M.lo[i] == M.lo[mid] && M.d[i] == M.d[mid] && M.hi[i] == M.hi[mid] &&
               K.lo[i] == K.lo[mid] && K.d[i] == K.d[mid] && K.hi[i] == K.hi[mid];
      };
      if (!same(mid)) { L.ulo[d] = 1; L.uhi[d] = 0; continue; }
      int lo = mid, hi = mid;
      while (same(lo - 1)) --lo;
      while (same(hi + 1)) ++hi;
      L.ulo[d] = lo;
      L.uhi[d] = hi;
    }
    std::vector<TsRow> rows;
    for (int d = 0; d < 3; ++d) {
      auto r = rows_of(L.M[d], L.K[d]);
      rows.insert(rows.end(), r.begin(), r.end());
    }
    CKS(cudaMalloc(&L.dev_rows, sizeof(TsRow) * rows.size()));
    CKS(cudaMemcpy(L.dev_rows, rows.data(), sizeof(TsRow) * rows.size(), cudaMemcpyHostToDevice));
  }
  for (size_t l = 1; l < H->lv.size(); ++l) {
    CKS(cudaMalloc(&H->lv[l].x, sizeof(float) * cells(H->lv[l])));
    CKS(cudaMalloc(&H->lv[l].b, sizeof(float) * cells(H->lv[l])));
  }
  CKS(cudaMalloc(&H->r, sizeof(float) * cells(H->lv[0])));
  // coarsest: generalised eigenvectors per coupled axis
  const TsLevelH& Lc = H->lv.back();
  const int nd = key.per_slice ? 2 : 3;
  std::vector<double> lamd[3];
  for (int d = 0; d < nd; ++d) {
    std::vector<double> V;
    gen_eig(Lc.M[d], Lc.K[d], V, lamd[d]);
    std::vector<float> Vf(V.begin(), V.end());
    CKS(cudaMalloc(&H->cV[d], sizeof(float) * Vf.size()));
    CKS(cudaMemcpy(H->cV[d], Vf.data(), sizeof(float) * Vf.size(), cudaMemcpyHostToDevice));
  }
  const int nzs = key.per_slice ? 1 : Lc.n[2];
  if ((long long)Lc.n[0] * Lc.n[1] * nzs > 6144)
    return set_err(GDP_EINVAL, "scheme: coarsest system %d x %d x %d too large for the direct solve", Lc.n[0], Lc.n[1], nzs);
  std::vector<double> ev((size_t)Lc.n[0] * Lc.n[1] * nzs);
  double emax = 0.0;
  for (int z = 0; z < nzs; ++z)
    for (int y = 0; y < Lc.n[1]; ++y)
      for (int x = 0; x < Lc.n[0]; ++x) {
        double e = key.alpha + key.bx * lamd[0][x] + key.by * lamd[1][y];
        if (!key.per_slice) e += key.bz * lamd[2][z];
        ev[((size_t)z * Lc.n[1] + y) * Lc.n[0] + x] = e;
        emax = std::max(emax, std::fabs(e));
      }
  std::vector<float> inv(ev.size());
  for (size_t t = 0; t < ev.size(); ++t) inv[t] = std::fabs(ev[t]) <= 1e-9 * emax ? 0.f : (float)(1.0 / ev[t]);
  CKS(cudaMalloc(&H->cinv, sizeof(float) * inv.size()));
  CKS(cudaMemcpy(H->cinv, inv.data(), sizeof(float) * inv.size(), cudaMemcpyHostToDevice));
  CKS(cudaMalloc(&H->sums, sizeof(double2) * std::max(1LL, key.nz)));
  CKS(cudaMallocHost(&H->h_sums, sizeof(double2) * std::max(1LL, key.nz)));
  out = std::move(H);
  return GDP_OK;
}

static int ts_get(Ctx& C, const TsKey& k, TsHier** out) {
  if (!C.scheme_cache) C.scheme_cache = new SchemeCache();
  auto& m = static_cast<SchemeCache*>(C.scheme_cache)->h;
  auto it = m.find(k);
  if (it == m.end()) {
    std::unique_ptr<TsHier> h;
    RETS(ts_build(k, h));
    it = m.emplace(k, std::move(h)).first;
  }
  *out = it->second.get();
  return GDP_OK;
}

// the constant coefficients of the interior (from the middle rows, fp64 rounded once)
static void set_interior(TsLv& v, const TsLevelH& L, bool per_slice) {
  for (int d = 0; d < 3; ++d) { v.ulo[d] = L.ulo[d]; v.uhi[d] = L.uhi[d]; }
  const int mx = L.n[0] / 2, my = L.n[1] / 2, mz = L.n[2] / 2;
  auto e = [](const Tri& t, int i, int a) { return a < 0 ? t.lo[i] : (a == 0 ? t.d[i] : t.hi[i]); };
  double rs = v.alpha;
  for (int d = 0; d < (per_slice ? 2 : 3); ++d) {
    const int m = L.n[d] / 2;
    rs *= L.M[d].lo[m] + L.M[d].d[m] + L.M[d].hi[m];
  }
  v.crs = (float)rs;
  for (int c = -1; c <= 1; ++c)
    for (int b = -1; b <= 1; ++b)
      for (int a = -1; a <= 1; ++a) {
        double zm = 1.0, zk = 0.0;
        if (!per_slice) { zm = e(L.M[2], mz, c); zk = e(L.K[2], mz, c); }
        else if (c != 0) zm = 0.0;
        const double xm = e(L.M[0], mx, a), xk = e(L.K[0], mx, a), ym = e(L.M[1], my, b), yk = e(L.K[1], my, b);
        const double C = (double)v.alpha * xm * ym * zm + (double)v.bx * xk * ym * zm + (double)v.by * xm * yk * zm +
                         (double)v.bz * xm * ym * zk;
        v.cst[(c + 1) * 9 + (b + 1) * 3 + (a + 1)] = (float)C;
      }
}

static TsLv dev_level(const TsHier& H, const TsLevelH& L) {
  TsLv v;
  v.nx = L.n[0]; v.ny = L.n[1]; v.nz = L.n[2];
  v.tx = L.dev_rows;
  v.ty = L.dev_rows + L.n[0];
  v.tz = L.dev_rows + L.n[0] + L.n[1];
  v.alpha = H.key.alpha;
  v.bx = H.key.bx; v.by = H.key.by;
  v.bz = H.key.per_slice ? 0.f : H.key.bz;
  v.seven = L.rb ? 1 : 0;
  set_interior(v, L, H.key.per_slice != 0);
  return v;
}

static dim3 grid_xy(int nx, int ny, int nz, dim3 blk) {
  return dim3((nx + blk.x - 1) / blk.x, (ny + blk.y - 1) / blk.y, nz);
}

static const dim3 kBlk(64, 4, 1);

static void ts_sweep(const TsHier& H, const TsLevelH& L, float* x, const float* b, float omega, cudaStream_t s);

// nu sweeps of a level.  The Hybrid finest level of a 3D system is the main path's 7-point operator,
// so its sweeps run on the main path's fused red-black z-march (one HBM pass per sweep instead of one
// per colour; ping-pong through the residual scratch, a final copy when nu is odd).
static void ts_smooth(const TsHier& H, const TsLevelH& L, float* x, const float* b, int nu, float omega,
                      cudaStream_t s) {
  if (&L == &H.lv[0] && L.rb && !H.key.per_slice && H.main7 && H.main7->lv.size() > 1 && nu > 0) {
    const Level& M0 = H.main7->lv[0];
    const Level& M1 = H.main7->lv[1];
    gdp_opts fo;
    gdp_opts_default(&fo);
    fo.fused = 2;
    if (fusable3d(M0, M1, fo)) {
      for (int k = 0; k < nu; ++k) {
        const float* src = (k & 1) ? H.r : x;
        float* dst = (k & 1) ? x : H.r;
        int items = 0;
        if (sweep3dv_ok(M0, M1, false, src, dst, b) &&
            fused_sweep3dv(M0, M1, src, dst, b, false, false, 0, nullptr, s, &items) == GDP_OK)
          continue;
        fused_sweep3d(M0, M1, src, dst, b, false, false, 0, nullptr, s);
      }
      if (nu & 1) cudaMemcpyAsync(x, H.r, sizeof(float) * (size_t)L.n[0] * L.n[1] * L.n[2], cudaMemcpyDeviceToDevice, s);
      return;
    }
  }
  if (&L == &H.lv[0] && L.rb && H.key.per_slice && H.main7 && H.main7->lv.size() > 1 && L.n[0] >= 128 &&
      nu >= 1 && nu <= 2) {  // per-slice 5-point finest level: the main path's row-marching nu-sweep pass
    const Level& M0 = H.main7->lv[0];
    const Level& M1 = H.main7->lv[1];
    rows2d_pass(false, nu, M0, M1, x, H.r, b, false, nullptr, s, false);
    cudaMemcpyAsync(x, H.r, sizeof(float) * (size_t)L.n[0] * L.n[1] * L.n[2], cudaMemcpyDeviceToDevice, s);
    return;
  }
  for (int k = 0; k < nu; ++k) ts_sweep(H, L, x, b, omega, s);
}

static void ts_sweep(const TsHier& H, const TsLevelH& L, float* x, const float* b, float omega, cudaStream_t s) {
  const TsLv v = dev_level(H, L);
  const bool Z = !H.key.per_slice;
  // opt-in (GDP_TS_TILE=1): bit-identical, but measured slower than the per-colour launches on
  // config 1 (Linear 174 vs 133 ms per step: the redundant halo phases and per-cell index math
  // cost more than the HBM passes they save)
  static const bool tile_env = getenv("GDP_TS_TILE") && atoi(getenv("GDP_TS_TILE")) != 0;
  if (!L.rb && tile_env && cells(L) >= (size_t)(1 << 16)) {  // 27-point level: two tiled half-sweeps
    // z-chunks of the parity's planes so that the grid holds ~4 CTAs per SM (planes of one parity are
    // independent in a half-sweep; the other parity's planes at chunk ends are copied twice, same values)
    const int tiles = ((v.nx + GT_X - 1) / GT_X) * ((v.ny + GT_Y - 1) / GT_Y);
    const int npar = (v.nz + 1) / 2;
    const int nch = std::max(1, std::min(npar, (148 * 4 + tiles - 1) / tiles));
    const int chunk = (npar + nch - 1) / nch;
    const dim3 g((v.nx + GT_X - 1) / GT_X, (v.ny + GT_Y - 1) / GT_Y, (npar + chunk - 1) / chunk);
    float* bufs[2] = {x, H.r};  // x -> scratch (ck = 0) -> x (ck = 1)
    for (int ck = 0; ck < 2; ++ck) {
      const float* src = bufs[ck];
      float* dst = bufs[ck ^ 1];
      ProfScope ps(KC_RBGS, 6.0 * (double)cells(L), s, (double)cells(L));
      if (ck >= v.nz) {
        cudaMemcpyAsync(dst, src, sizeof(float) * cells(L), cudaMemcpyDeviceToDevice, s);
        continue;
      }
      if (Z) k_ts_gs_tile<true><<<g, GT_T, 0, s>>>(v, src, dst, b, ck, omega, chunk);
      else k_ts_gs_tile<false><<<g, GT_T, 0, s>>>(v, src, dst, b, ck, omega, chunk);
    }
    return;
  }
  const int ncol = L.rb ? 2 : (Z ? 8 : 4);
  const double per_launch = 12.0 / ncol * (double)cells(L);  // x in + b + x out per sweep, split over colours
  for (int c = 0; c < ncol; ++c) {
    const int hx = (v.nx + 1) / 2;
    const int gy = ncol == 2 ? v.ny : (v.ny + 1) / 2;
    const int gz = ncol == 8 ? (v.nz + 1) / 2 : v.nz;
    dim3 g((hx + kBlk.x - 1) / kBlk.x, (gy + kBlk.y * NPT - 1) / (kBlk.y * NPT), gz);
    ProfScope ps(KC_RBGS, per_launch, s, (double)cells(L));
    if (Z) k_ts_gs<true><<<g, kBlk, 0, s>>>(v, x, b, ncol, c, omega);
    else k_ts_gs<false><<<g, kBlk, 0, s>>>(v, x, b, ncol, c, omega);
  }
}

static int ts_ensure_part(TsHier& H, size_t n) {
  if (H.part_cap >= n) return GDP_OK;
  if (H.part) cudaFree(H.part);
  H.part = nullptr;
  CKS(cudaMalloc(&H.part, sizeof(double2) * n));
  H.part_cap = n;
  return GDP_OK;
}

// residual of level l (into r, may be null) and, if sums != null, per-slice (or whole) fp64 sums
static int ts_resid(TsHier& H, const TsLevelH& L, const float* x, const float* b, float* r, bool norms,
                    cudaStream_t s) {
  if (&L == &H.lv[0] && L.rb && H.main7) {
    // Hybrid finest level: the main path's residual kernel (same 7-/5-point operator), per-plane sums
    Hier& M = *H.main7;
    const Level& M0 = M.lv[0];
    launch_norms(M0.K, x, M0.xlo, M0.xhi, RhsK{b, nullptr, nullptr, 0.f, 0}, RHS_B, 1, r, M.partials, M.plane_sums, s);
    if (norms) CKS(cudaMemcpyAsync(H.sums, M.plane_sums, sizeof(double2) * L.n[2], cudaMemcpyDeviceToDevice, s));
    CKS(cudaGetLastError());
    return GDP_OK;
  }
  const TsLv v = dev_level(H, L);
  const dim3 g((v.nx + kBlk.x - 1) / kBlk.x, (v.ny + kBlk.y * NPT - 1) / (kBlk.y * NPT), v.nz);
  const size_t nb = (size_t)g.x * g.y;
  if (norms) RETS(ts_ensure_part(H, nb * v.nz));
  {
    ProfScope ps(norms && !r ? KC_NORMS : KC_RESTRICT, (8.0 + (r ? 4.0 : 0.0)) * (double)cells(L), s, (double)cells(L));
    if (!H.key.per_slice) k_ts_resid<true><<<g, kBlk, 0, s>>>(v, x, b, r, norms ? H.part : nullptr);
    else k_ts_resid<false><<<g, kBlk, 0, s>>>(v, x, b, r, norms ? H.part : nullptr);
  }
  if (norms) {
    ProfScope ps(KC_UTIL, 16.0 * nb * v.nz, s);
    k_ts_sum<<<v.nz, 256, 0, s>>>(H.part, (int)nb, H.sums);
  }
  CKS(cudaGetLastError());
  return GDP_OK;
}

static TsXfer xfer_of(const TsLevelH& F, const TsLevelH& C) {
  TsXfer T;
  T.fx = F.n[0]; T.fy = F.n[1]; T.fz = F.n[2];
  T.cx = C.n[0]; T.cy = C.n[1]; T.cz = C.n[2];
  T.co_x = C.co[0]; T.co_y = C.co[1]; T.co_z = C.co[2];
  return T;
}

static int ts_cycle(TsHier& H, float* x0, const float* b0, int nu_pre, int nu_post, float omega, cudaStream_t s) {
  const int nl = (int)H.lv.size();
  std::vector<float*> xs(nl), bs(nl);
  xs[0] = x0;
  bs[0] = const_cast<float*>(b0);
  for (int l = 1; l < nl; ++l) { xs[l] = H.lv[l].x; bs[l] = H.lv[l].b; }
  for (int l = 0; l + 1 < nl; ++l) {
    const TsLevelH& L = H.lv[l];
    const TsLevelH& C = H.lv[l + 1];
    if (l > 0) CKS(cudaMemsetAsync(xs[l], 0, sizeof(float) * cells(L), s));
    ts_smooth(H, L, xs[l], bs[l], nu_pre, omega, s);
    RETS(ts_resid(H, L, xs[l], bs[l], H.r, false, s));
    const TsXfer T = xfer_of(L, C);
    ProfScope ps(KC_RESTRICT, 4.0 * (double)cells(L) + 4.0 * (double)cells(C), s);
    k_ts_restrict<<<grid_xy(C.n[0], C.n[1], C.n[2], kBlk), kBlk, 0, s>>>(T, H.r, bs[l + 1]);
  }
  {  // coarsest: direct
    const TsLevelH& L = H.lv[nl - 1];
    TsCoarse cc;
    cc.nx = L.n[0]; cc.ny = L.n[1]; cc.nz = L.n[2];
    cc.per_slice = H.key.per_slice;
    cc.Vx = H.cV[0]; cc.Vy = H.cV[1]; cc.Vz = H.cV[2];
    cc.inv = H.cinv;
    const int nsys = H.key.per_slice ? L.n[2] : 1;
    const int N = L.n[0] * L.n[1] * (H.key.per_slice ? 1 : L.n[2]);
    if (nl == 1) {  // the finest level is the coarsest: correction form (iterative refinement in fp32)
      RETS(ts_resid(H, L, xs[0], bs[0], H.r, false, s));
      {
        ProfScope ps(KC_COARSE, 8.0 * (double)cells(L), s);
        k_ts_coarse<<<nsys, 1024, 2 * N * sizeof(float), s>>>(cc, H.r, H.r);
      }
      ProfScope ps(KC_UTIL, 12.0 * (double)cells(L), s);
      k_ts_add<<<(int)((cells(L) + 255) / 256), 256, 0, s>>>(xs[0], H.r, (long long)cells(L));
    } else {
      ProfScope ps(KC_COARSE, 8.0 * (double)cells(L), s);
      k_ts_coarse<<<nsys, 1024, 2 * N * sizeof(float), s>>>(cc, bs[nl - 1], xs[nl - 1]);
    }
  }
  for (int l = nl - 2; l >= 0; --l) {
    const TsLevelH& L = H.lv[l];
    const TsLevelH& C = H.lv[l + 1];
    const TsXfer T = xfer_of(L, C);
    {
      ProfScope ps(KC_PROLONG, 8.0 * (double)cells(L) + 4.0 * (double)cells(C), s, (double)cells(L));
      if (T.co_x) k_ts_prolong2<<<grid_xy((L.n[0] + 1) / 2, L.n[1], L.n[2], kBlk), kBlk, 0, s>>>(T, xs[l + 1], xs[l]);
      else k_ts_prolong<<<grid_xy(L.n[0], L.n[1], L.n[2], kBlk), kBlk, 0, s>>>(T, xs[l + 1], xs[l]);
    }
    ts_smooth(H, L, xs[l], bs[l], nu_post, omega, s);
  }
  CKS(cudaGetLastError());
  return GDP_OK;
}

// norms of level 0 -> host: rel (3D) or the worst slice (per slice); *worst_b = that system's ||b||
static int ts_rel(TsHier& H, const float* x, const float* b, float* r, cudaStream_t s, double& rel, double& nb) {
  RETS(ts_resid(H, H.lv[0], x, b, r, true, s));
  const int nz = H.lv[0].n[2];
  CKS(cudaMemcpyAsync(H.h_sums, H.sums, sizeof(double2) * nz, cudaMemcpyDeviceToHost, s));
  CKS(cudaStreamSynchronize(s));
  if (H.key.per_slice) {
    rel = 0.0;
    nb = 0.0;
    for (int z = 0; z < nz; ++z) {
      const double bb = H.h_sums[z].y, rr = H.h_sums[z].x;
      const double q = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
      if (!(q <= rel)) { rel = q; nb = std::sqrt(bb); }
    }
  } else {
    double rr = 0.0, bb = 0.0;
    for (int z = 0; z < nz; ++z) { rr += H.h_sums[z].x; bb += H.h_sums[z].y; }
    rel = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
    nb = std::sqrt(bb);
  }
  return GDP_OK;
}

static int ts_solve(TsHier& H, float* x, const float* b, const gdp_opts& o, int nu_pre, int nu_post, float omega,
                    gdp_report* rep, cudaStream_t s) {
  double rel = 0.0, nb = 0.0;
  RETS(ts_rel(H, x, b, nullptr, s, rel, nb));
  if (rep) { rep->rel_res[0] = rel; rep->norm_b = nb; rep->levels = (int)H.lv.size(); rep->dx_inf = -1.0; }
  if (!std::isfinite(rel)) return set_err(GDP_ECUDA, "scheme: non-finite initial residual");
  int k = 0, stall = 0, st = GDP_OK;
  // the gate is taken on this path's fp32 residual with a 10 % margin, so that the fp64 residual of
  // the fp32 iterate (the oracle's measure) also meets rel_tol (reading c-12: the 1e-6 gate is
  // within a few ulps of the fp32 floor on small systems)
  const double gate = 0.9 * o.rel_tol;
  while (rel > gate) {
    if (k >= o.max_vcycles) { st = GDP_ENOCONV; break; }
    RETS(ts_cycle(H, x, b, nu_pre, nu_post, omega, s));
    double r2 = 0.0;
    RETS(ts_rel(H, x, b, nullptr, s, r2, nb));
    ++k;
    if (rep) rep->rel_res[k] = r2;
    if (!std::isfinite(r2)) return set_err(GDP_ECUDA, "scheme: non-finite residual after cycle %d", k);
    stall = (r2 > 0.9 * rel) ? stall + 1 : 0;
    rel = r2;
    if (o.stagnation > 0 && stall >= o.stagnation && rel > gate) { st = rel <= o.rel_tol ? GDP_OK : GDP_ENOCONV; break; }
  }
  if (rep) { rep->vcycles = k; rep->status = st; }
  return st;
}

template <typename LD>
static void ts_launch_apply(const TsLv& v, bool Z, LD ld, float* out, int acc, cudaStream_t s) {
  const dim3 g = grid_xy(v.nx, v.ny, v.nz, kBlk);
  ProfScope ps(KC_UTIL, 8.0 * (double)v.nx * v.ny * v.nz, s);
  if (Z) k_ts_apply<true, LD><<<g, kBlk, 0, s>>>(v, ld, out, acc);
  else k_ts_apply<false, LD><<<g, kBlk, 0, s>>>(v, ld, out, acc);
}

// out (+)= A' u where A' is level 0's operator with (alpha, bx, by, bz) replaced
static void ts_apply_with(const TsHier& H, float alpha, float bx, float by, float bz, const void* u, int tI,
                          float* out, int acc, cudaStream_t s) {
  TsLv v = dev_level(H, H.lv[0]);
  v.alpha = alpha; v.bx = bx; v.by = by; v.bz = bz;
  set_interior(v, H.lv[0], H.key.per_slice != 0);
  const bool Z = !H.key.per_slice;
  if (tI == 0) ts_launch_apply(v, Z, LdU8{(const uint8_t*)u, v.nx, v.ny}, out, acc, s);
  else ts_launch_apply(v, Z, LdF{(const float*)u, v.nx, v.ny}, out, acc, s);
}

static void ts_copy(const void* u, int tI, int nx, int ny, int nz, float* out, float shift, cudaStream_t s) {
  const dim3 g = grid_xy(nx, ny, nz, kBlk);
  ProfScope ps(KC_UTIL, (tI == 0 ? 5.0 : 8.0) * (double)nx * ny * nz, s);
  if (tI == 0) k_ts_copy<<<g, kBlk, 0, s>>>(LdU8{(const uint8_t*)u, nx, ny}, nx, ny, out, shift);
  else k_ts_copy<<<g, kBlk, 0, s>>>(LdF{(const float*)u, nx, ny}, nx, ny, out, shift);
}

// ---------------------------------------------------------------------------------------------
// Entry points (called by the C ABI when opts.scheme != GDP_SCHEME_CONSTANT)
// ---------------------------------------------------------------------------------------------
static TsKey key_of(int scheme, long long nx, long long ny, long long nz, float bx, float by, float bz, float alpha,
                    int per_slice, const gdp_opts& o) {
  TsKey k;
  k.scheme = scheme;
  k.nx = nx; k.ny = ny; k.nz = nz;
  k.bx = bx; k.by = by; k.bz = per_slice ? 0.f : bz;
  k.alpha = alpha;
  k.per_slice = per_slice;
  k.coarse_max = o.coarse_max;
  return k;
}

// Hybrid, 3D: the main path's hierarchy for the same (dims, W, alpha) lends its fused finest-level
// sweeps to ts_smooth (the Hybrid finest operator is the Constant one)
static int attach_main7(Ctx& C, TsHier& H, const gdp_opts& o) {
  if (H.key.scheme != GDP_SCHEME_HYBRID || H.main7) return GDP_OK;
  static const bool off = getenv("GDP_HYBRID_MAIN7") && atoi(getenv("GDP_HYBRID_MAIN7")) == 0;
  if (off) return GDP_OK;
  HierKey k{};
  k.nx = H.key.nx; k.ny = H.key.ny; k.nzl = H.key.nz; k.z0 = 0; k.nzg = H.key.nz;
  k.bx = H.key.bx; k.by = H.key.by; k.bz = H.key.per_slice ? 0.f : H.key.bz; k.alpha = H.key.alpha;
  k.coarse_max = o.coarse_max;
  k.omega = o.omega;
  return C.get_hier(k, &H.main7);
}

int scheme_diffuse_z(Ctx& C, const void* I0, int tI, float* I1, long long nx, long long ny, long long nz, float bx,
                     float by, float bz, float alpha, const gdp_opts& o, gdp_report* rep, cudaStream_t s) {
  TsHier* H;
  RETS(ts_get(C, key_of(o.scheme, nx, ny, nz, bx, by, bz, alpha, 0, o), &H));
  RETS(attach_main7(C, *H, o));
  const long long before = g_launches.load();
  const size_t n = (size_t)nx * ny * nz;
  if (!H->b0) CKS(cudaMalloc(&H->b0, sizeof(float) * n));
  g_prof_finest = (double)n;
  g_prof_l1 = H->lv.size() > 1 ? (double)cells(H->lv[1]) : 0.0;
  g_prof_rhs8d = tI == 0 ? 1.0 : 4.0;
  CKS(cudaEventRecord(C.ev0, s));
  // b = alpha I0 + (bx S_x + by S_y) I0 (reading L-2; the Hybrid fine level gives Eq. (1)'s rhs)
  ts_apply_with(*H, alpha, bx, by, 0.f, I0, tI, H->b0, 0, s);
  ts_copy(I0, tI, (int)nx, (int)ny, (int)nz, I1, 0.f, s);  // x0 = I0
  int st = ts_solve(*H, I1, H->b0, o, o.nu_pre, o.nu_post, o.omega, rep, s);
  if (st != GDP_OK && st != GDP_ENOCONV) return st;
  if (alpha == 0.f) {  // mean pin (reading c-3 / L-3): mean(I1) = mean(I0), fp64
    ProfScope ps(KC_UTIL, (4.0 + (tI == 0 ? 1.0 : 4.0)) * (double)n, s);
    if (tI == 0) k_ts_means<<<(int)nz, 256, 0, s>>>(I1, LdU8{(const uint8_t*)I0, (int)nx, (int)ny}, (int)nx, (int)ny, H->sums);
    else k_ts_means<<<(int)nz, 256, 0, s>>>(I1, LdF{(const float*)I0, (int)nx, (int)ny}, (int)nx, (int)ny, H->sums);
    CKS(cudaMemcpyAsync(H->h_sums, H->sums, sizeof(double2) * nz, cudaMemcpyDeviceToHost, s));
    CKS(cudaStreamSynchronize(s));
    double sx = 0.0, si = 0.0;
    for (long long z = 0; z < nz; ++z) { sx += H->h_sums[z].x; si += H->h_sums[z].y; }
    const float shift = (float)((si - sx) / (double)n);
    ts_copy(I1, 1, (int)nx, (int)ny, (int)nz, I1, shift, s);
  }
  CKS(cudaEventRecord(C.ev1, s));
  CKS(cudaGetLastError());
  if (rep) {
    CKS(cudaEventSynchronize(C.ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, C.ev0, C.ev1);
    rep->seconds = ms * 1e-3;
    rep->kernel_launches = g_launches.load() - before;
    rep->hbm_bytes_est = 0.0;
  }
  g_prof_finest = g_prof_l1 = 0.0;
  if (st == GDP_ENOCONV) set_err(GDP_ENOCONV, "scheme diffuse_z: not converged");
  return st;
}

int scheme_slices(Ctx& C, const void* I0, int tI, const float* I1, float* I2, long long nx, long long ny,
                  long long nz, float alpha, float vshift, const gdp_opts& o, gdp_report* rep, cudaStream_t s) {
  TsHier* H;
  RETS(ts_get(C, key_of(o.scheme, nx, ny, nz, 1.f, 1.f, 0.f, alpha, 1, o), &H));
  RETS(attach_main7(C, *H, o));
  const long long before = g_launches.load();
  const size_t n = (size_t)nx * ny * nz;
  if (!H->b0) CKS(cudaMalloc(&H->b0, sizeof(float) * n));
  g_prof_finest = (double)n;
  g_prof_l1 = H->lv.size() > 1 ? (double)cells(H->lv[1]) : 0.0;
  g_prof_rhs8d = 4.0 + (tI == 0 ? 1.0 : 4.0);
  CKS(cudaEventRecord(C.ev0, s));
  // x0 = I1 (+ the deferred mean-pin shift); b = alpha M2 x0 + S2 I0 (reading L-2)
  ts_copy(I1, 1, (int)nx, (int)ny, (int)nz, I2, vshift, s);
  ts_apply_with(*H, alpha, 0.f, 0.f, 0.f, I2, 1, H->b0, 0, s);
  ts_apply_with(*H, 0.f, 1.f, 1.f, 0.f, I0, tI, H->b0, 1, s);
  const int nu_pre = o.nu_pre_slices >= 0 ? o.nu_pre_slices : o.nu_pre;
  const int nu_post = o.nu_post_slices >= 0 ? o.nu_post_slices : o.nu_post;
  int st = ts_solve(*H, I2, H->b0, o, nu_pre, nu_post, o.omega_slices > 0.f ? o.omega_slices : o.omega, rep, s);
  CKS(cudaEventRecord(C.ev1, s));
  CKS(cudaGetLastError());
  if (rep) {
    CKS(cudaEventSynchronize(C.ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, C.ev0, C.ev1);
    rep->seconds = ms * 1e-3;
    rep->kernel_launches = g_launches.load() - before;
    rep->hbm_bytes_est = 0.0;
  }
  g_prof_finest = g_prof_l1 = 0.0;
  if (st == GDP_ENOCONV) set_err(GDP_ENOCONV, "scheme slices: not converged");
  return st;
}

int scheme_vcycle(Ctx& C, float* x, const float* b, long long nx, long long ny, long long nz, float bx, float by,
                  float bz, float alpha, const gdp_opts& o, double* rel, cudaStream_t s) {
  TsHier* H;
  RETS(ts_get(C, key_of(o.scheme, nx, ny, nz, bx, by, bz, alpha, 0, o), &H));
  RETS(attach_main7(C, *H, o));
  RETS(ts_cycle(*H, x, b, o.nu_pre, o.nu_post, o.omega, s));
  if (rel) {
    double nb;
    RETS(ts_rel(*H, x, b, nullptr, s, *rel, nb));
  }
  return GDP_OK;
}

int scheme_levels(Ctx& C, int scheme, long long nx, long long ny, long long nz, float bx, float by, float bz,
                  float alpha, int per_slice, const gdp_opts& o, int* nlev, gdp_dims* dims, int* coarsened, int max) {
  TsHier* H;
  RETS(ts_get(C, key_of(scheme, nx, ny, nz, bx, by, bz, alpha, per_slice, o), &H));
  *nlev = (int)H->lv.size();
  for (int l = 0; l < (int)H->lv.size() && l < max; ++l) {
    if (dims) dims[l] = gdp_dims{H->lv[l].n[0], H->lv[l].n[1], H->lv[l].n[2]};
    if (coarsened)
      for (int d = 0; d < 3; ++d) coarsened[3 * l + d] = H->lv[l].co[d];
  }
  return GDP_OK;
}

int scheme_apply(Ctx& C, int scheme, int level, const float* x, float* y, long long nx, long long ny, long long nz,
                 float bx, float by, float bz, float alpha, int per_slice, const gdp_opts& o, cudaStream_t s) {
  TsHier* H;
  RETS(ts_get(C, key_of(scheme, nx, ny, nz, bx, by, bz, alpha, per_slice, o), &H));
  if (level < 0 || level >= (int)H->lv.size()) return set_err(GDP_EINVAL, "scheme_apply: level %d of %d", level, (int)H->lv.size());
  const TsLevelH& L = H->lv[level];
  const TsLv v = dev_level(*H, L);
  ts_launch_apply(v, !per_slice, LdF{x, v.nx, v.ny}, y, 0, s);
  CKS(cudaGetLastError());
  return GDP_OK;
}

int scheme_residual(Ctx& C, int scheme, const float* x, const float* b, float* r, long long nx, long long ny,
                    long long nz, float bx, float by, float bz, float alpha, int per_slice, const gdp_opts& o,
                    double* rr, double* bb, cudaStream_t s) {
  TsHier* H;
  RETS(ts_get(C, key_of(scheme, nx, ny, nz, bx, by, bz, alpha, per_slice, o), &H));
  RETS(ts_resid(*H, H->lv[0], x, b, r, true, s));
  CKS(cudaMemcpyAsync(H->h_sums, H->sums, sizeof(double2) * nz, cudaMemcpyDeviceToHost, s));
  CKS(cudaStreamSynchronize(s));
  double a = 0.0, c = 0.0;
  for (long long z = 0; z < nz; ++z) { a += H->h_sums[z].x; c += H->h_sums[z].y; }
  if (rr) *rr = a;
  if (bb) *bb = c;
  return GDP_OK;
}

}  // namespace gdp
