/* cg_omp.c — CPU ORACLE (fp64, C + OpenMP) — TEST INFRASTRUCTURE ONLY.
 *
 * The plain definition of what the hot path computes, written for
 * speed on all host cores so that bench.py can time a strong CPU baseline beside the GPU:
 * the paper's discrete operators assembled link by link with Neumann boundaries (a link joins two
 * voxels of the grid; none leaves it, reading c-1), solved by textbook conjugate gradient in
 * fp64 to ||b - A x|| <= tol ||b||.  It shares no code with the CUDA path (paper_1310_0041_b200/
 * never includes or links it) and mirrors oracle/gdp_oracle.py function for function; the
 * -m "not gpu" tests pin it to that module and to the closed forms.
 *
 * Layout: fp64 arrays (nz, ny, nx), x fastest.  W = (bx, by, bz).
 *   apply_A       (alpha - div W grad) x = alpha x + sum_d beta_d D_d^T D_d x
 *   rhs_diffusion b1 = -div(W G), G = (D_x I0, D_y I0, 0)                          Eq. 1
 *   rhs_blend     b2 = alpha I1 - div(pi grad I0), pi = Diag(1, 1, 0)              Eq. 2
 *   diffuse_z     phase 1: CG from x0 = I0 on the singular alpha = 0 system with b projected to
 *                 mean 0, then mean(I1) = mean(I0) (reading c-3)
 *   slices        phase 2: one CG per slice (independent systems), x0 = I0
 * Returns the CG iteration count (phase 2: the sum over slices); negative on bad arguments.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long long i64;

/* y = A x on one grid of (nz, ny, nx) cells: alpha x + sum over links of beta (x_c - x_n) at
 * both ends, i.e. D^T D x accumulated link by link (the difference form of PAPER.md:229). */
static void apply_A(const double* x, double* y, i64 nx, i64 ny, i64 nz, double bx, double by, double bz,
                    double alpha) {
  const i64 pl = nx * ny;
#pragma omp parallel for schedule(static)
  for (i64 z = 0; z < nz; ++z) {
    for (i64 j = 0; j < ny; ++j) {
      for (i64 i = 0; i < nx; ++i) {
        const i64 c = z * pl + j * nx + i;
        const double xc = x[c];
        double s = alpha * xc;
        if (bx != 0.0) {
          if (i > 0) s += bx * (xc - x[c - 1]);
          if (i < nx - 1) s += bx * (xc - x[c + 1]);
        }
        if (by != 0.0) {
          if (j > 0) s += by * (xc - x[c - nx]);
          if (j < ny - 1) s += by * (xc - x[c + nx]);
        }
        if (bz != 0.0) {
          if (z > 0) s += bz * (xc - x[c - pl]);
          if (z < nz - 1) s += bz * (xc - x[c + pl]);
        }
        y[c] = s;
      }
    }
  }
}

/* b = -div(W G) with G the in-plane forward differences of I (links in x and y only):
 * b_c = sum over in-plane links of beta (I_c - I_n) (G's z component is 0, Eq. 1 / Eq. 2). */
static void rhs_inplane(const double* I, double* b, i64 nx, i64 ny, i64 nz, double bx, double by) {
  apply_A(I, b, nx, ny, nz, bx, by, 0.0, 0.0);
}

static double dot(const double* a, const double* b, i64 n) {
  double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (i64 i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* textbook CG on one system (OpenMP inside every vector operation) */
static int cg(const double* b, double* x, i64 nx, i64 ny, i64 nz, double bx, double by, double bz, double alpha,
              double tol, int maxit) {
  const i64 n = nx * ny * nz;
  double* r = (double*)malloc(sizeof(double) * n);
  double* p = (double*)malloc(sizeof(double) * n);
  double* q = (double*)malloc(sizeof(double) * n);
  if (!r || !p || !q) { free(r); free(p); free(q); return -2; }
  apply_A(x, q, nx, ny, nz, bx, by, bz, alpha);
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) { r[i] = b[i] - q[i]; p[i] = r[i]; }
  const double bb = dot(b, b, n);
  double rr = dot(r, r, n);
  const double thr = tol * tol * (bb > 0.0 ? bb : rr);
  int it = 0;
  while (rr > thr && it < maxit) {
    apply_A(p, q, nx, ny, nz, bx, by, bz, alpha);
    const double pq = dot(p, q, n);
    if (!(pq > 0.0)) break;
    const double a = rr / pq;
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) { x[i] += a * p[i]; r[i] -= a * q[i]; }
    const double rn = dot(r, r, n);
    const double be = rn / rr;
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) p[i] = r[i] + be * p[i];
    rr = rn;
    ++it;
  }
  free(r); free(p); free(q);
  return it;
}

/* the same CG on one small system, single-threaded (phase 2 runs slices in parallel) */
static int cg_serial(const double* b, double* x, i64 nx, i64 ny, double alpha, double tol, int maxit, double* work) {
  const i64 n = nx * ny;
  double *r = work, *p = work + n, *q = work + 2 * n;
  double bb = 0.0, rr = 0.0;
#define APPLY2D(src, dst)                                                            \
  for (i64 j = 0; j < ny; ++j)                                                       \
    for (i64 i = 0; i < nx; ++i) {                                                   \
      const i64 c = j * nx + i;                                                      \
      const double xc = (src)[c];                                                    \
      double s = alpha * xc;                                                         \
      if (i > 0) s += xc - (src)[c - 1];                                             \
      if (i < nx - 1) s += xc - (src)[c + 1];                                        \
      if (j > 0) s += xc - (src)[c - nx];                                            \
      if (j < ny - 1) s += xc - (src)[c + nx];                                       \
      (dst)[c] = s;                                                                  \
    }
  APPLY2D(x, q);
  for (i64 i = 0; i < n; ++i) { r[i] = b[i] - q[i]; p[i] = r[i]; bb += b[i] * b[i]; rr += r[i] * r[i]; }
  const double thr = tol * tol * (bb > 0.0 ? bb : rr);
  int it = 0;
  while (rr > thr && it < maxit) {
    APPLY2D(p, q);
    double pq = 0.0;
    for (i64 i = 0; i < n; ++i) pq += p[i] * q[i];
    if (!(pq > 0.0)) break;
    const double a = rr / pq;
    double rn = 0.0;
    for (i64 i = 0; i < n; ++i) { x[i] += a * p[i]; r[i] -= a * q[i]; rn += r[i] * r[i]; }
    const double be = rn / rr;
    for (i64 i = 0; i < n; ++i) p[i] = r[i] + be * p[i];
    rr = rn;
    ++it;
  }
#undef APPLY2D
  return it;
}

int gdp_oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Phase 1 (Eq. 1): I1 from I0 (fp64, already decoded: u8/255 rounded to fp32, reading c-9). */
int gdp_oracle_diffuse_z(const double* I0, double* I1, i64 nx, i64 ny, i64 nz, double bx, double by, double bz,
                         double tol, int maxit) {
  if (!I0 || !I1 || nx <= 0 || ny <= 0 || nz <= 0) return -1;
  const i64 n = nx * ny * nz;
  double* b = (double*)malloc(sizeof(double) * n);
  if (!b) return -2;
  rhs_inplane(I0, b, nx, ny, nz, bx, by);
  double sb = 0.0, s0 = 0.0;
#pragma omp parallel for reduction(+ : sb, s0) schedule(static)
  for (i64 i = 0; i < n; ++i) { sb += b[i]; s0 += I0[i]; }
  const double mb = sb / (double)n;  /* b is compatible up to rounding: project to mean 0 (c-3) */
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) { b[i] -= mb; I1[i] = I0[i]; }
  const int it = cg(b, I1, nx, ny, nz, bx, by, bz, 0.0, tol, maxit);
  double s1 = 0.0;
#pragma omp parallel for reduction(+ : s1) schedule(static)
  for (i64 i = 0; i < n; ++i) s1 += I1[i];
  const double shift = (s0 - s1) / (double)n;  /* mean(I1) = mean(I0) */
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) I1[i] += shift;
  free(b);
  return it;
}

/* Phase 2 (Eq. 2): per slice (alpha - Lx - Ly) I2 = alpha I1 + (Lx + Ly) I0, CG from I0. */
int gdp_oracle_slices(const double* I0, const double* I1, double* I2, i64 nx, i64 ny, i64 nz, double alpha,
                      double tol, int maxit) {
  if (!I0 || !I1 || !I2 || nx <= 0 || ny <= 0 || nz <= 0 || !(alpha > 0.0)) return -1;
  const i64 pl = nx * ny;
  long long total = 0;
  int bad = 0;
#pragma omp parallel reduction(+ : total, bad)
  {
    double* work = (double*)malloc(sizeof(double) * 4 * pl);
    if (!work) {
      bad += 1;
    } else {
#pragma omp for schedule(dynamic, 1)
      for (i64 z = 0; z < nz; ++z) {
        const double* i0 = I0 + z * pl;
        const double* i1 = I1 + z * pl;
        double* x = I2 + z * pl;
        double* b = work + 3 * pl;
        for (i64 j = 0; j < ny; ++j)  /* b = alpha I1 + (Lx + Ly) I0, link by link */
          for (i64 i = 0; i < nx; ++i) {
            const i64 c = j * nx + i;
            const double ic = i0[c];
            double s = alpha * i1[c];
            if (i > 0) s += ic - i0[c - 1];
            if (i < nx - 1) s += ic - i0[c + 1];
            if (j > 0) s += ic - i0[c - nx];
            if (j < ny - 1) s += ic - i0[c + nx];
            b[c] = s;
          }
        memcpy(x, i0, sizeof(double) * pl);
        total += cg_serial(b, x, nx, ny, alpha, tol, maxit, work);
      }
      free(work);
    }
  }
  if (bad) return -2;
  return (int)(total > 2147483647LL ? 2147483647LL : total);
}
