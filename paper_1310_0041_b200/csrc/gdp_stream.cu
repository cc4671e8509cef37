// gdp_stream.cu — out-of-core z-slab streamer.
//
// For stacks whose finest level does not fit the HBM budget.  The finest level lives in host
// memory: phase 1's iterate x IS the caller's I1 buffer, its rhs b = (bx Lx + by Ly) I0 is
// recomputed on the device for every window from the 1-byte I0 (so a pass moves 4 + s_I bytes
// per voxel host->device and 4 back, instead of 12).  Levels >= 1 stay resident.
//
// Phase 1 (Eq. 1).  Every finest-level pass of the V-cycle (the paper's "streaming pass over
// the slices", two per V-cycle there, nu_pre + nu_post sweeps here) streams z-chunks in order
// through the z-marching kernel (gdp_march3d.cu): chunk [p_lo, p_hi) needs the window
// [p_lo - 3, p_hi + 3) of the pass's input x; the planes it shares with the previous window are
// kept on the device (their host copies are already overwritten by the previous chunk's output,
// which is written back in place).  Three streams overlap the H2D of chunk k+1, the kernels of
// chunk k and the D2H of chunk k-1 (double-buffered windows, events between them).  The
// arithmetic per voxel is the in-core kernels', so the iterate is bit-identical to the in-core
// solve (tests/test_gpu_parity.py::test_out_of_core_*).
//
// fp16 staging ("intermediate solutions ... are stored
// ... using half-precision floating point values"): with gdp_opts.half_staging a V-cycle whose
// residual is predicted (from the observed contraction) to stay above HALF_REL stores the host
// iterate as fp16 in a pinned scratch (2 B instead of 4 per voxel each way); computation stays
// fp32 on the device.  The first cycle predicted below HALF_REL reads the fp16 iterate and writes
// fp32 again, so the answer comes from fp32 cycles (the quantisation error, ~1e-4 on [0, 1], is
// high-frequency and the next cycle's smoothing removes it, as the paper notes).
//
// Phase 2 (Eq. 2).  Slices are independent systems: batches of slices go host->device, are
// solved in core (gdp_screened_poisson_slices) and come back; the mean-pin shift of phase 1 is
// applied to each I1 batch on the way (and written back to the caller's I1).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "gdp_internal.h"

namespace gdp {

#define SK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(e_ == cudaErrorMemoryAllocation ? GDP_ENOMEM : GDP_ECUDA, "%s: %s (%s:%d)", #call, \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)
#define SR(call)                   \
  do {                             \
    int r_ = (call);               \
    if (r_ != GDP_OK) return r_;   \
  } while (0)

// pins a host range for the duration of a call if the caller passed pageable memory
HostPin::~HostPin() { if (p) cudaHostUnregister(p); }
int HostPin::pin(const void* ptr, size_t bytes) {
  if (!ptr || !bytes) return GDP_OK;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) == cudaSuccess && a.type == cudaMemoryTypeHost) return GDP_OK;
  cudaGetLastError();
  SK(cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterDefault));
  p = const_cast<void*>(ptr);
  return GDP_OK;
}

constexpr double HALF_REL = 5e-3;  // fp16 iterate storage while the residual stays above this

__global__ void k_f16_to_f32(const __half* __restrict__ a, float* __restrict__ b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = __half2float(a[i]);
}
__global__ void k_f32_to_f16(const float* __restrict__ a, __half* __restrict__ b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = __float2half_rn(a[i]);
}
static void convert(const void* a, void* b, long long n, bool to_half, cudaStream_t s) {
  if (n <= 0) return;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  ProfScope ps(KC_UTIL, 6.0 * (double)n, s);
  if (to_half) k_f32_to_f16<<<blocks, 256, 0, s>>>(static_cast<const float*>(a), static_cast<__half*>(b), n);
  else k_f16_to_f32<<<blocks, 256, 0, s>>>(static_cast<const __half*>(a), static_cast<float*>(b), n);
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  int alloc(size_t bytes) { SK(cudaMalloc(&p, std::max<size_t>(bytes, 16))); return GDP_OK; }
  float* f() const { return static_cast<float*>(p); }
  unsigned char* u() const { return static_cast<unsigned char*>(p); }
};

struct Streams {
  cudaStream_t s = nullptr, ci = nullptr, co = nullptr;
  cudaEvent_t evI[2] = {nullptr, nullptr}, evK[2] = {nullptr, nullptr}, evO[2] = {nullptr, nullptr};
  ~Streams() {
    for (int i = 0; i < 2; ++i) {
      if (evI[i]) cudaEventDestroy(evI[i]);
      if (evK[i]) cudaEventDestroy(evK[i]);
      if (evO[i]) cudaEventDestroy(evO[i]);
    }
    if (s) cudaStreamDestroy(s);
    if (ci) cudaStreamDestroy(ci);
    if (co) cudaStreamDestroy(co);
  }
  int create() {
    SK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SK(cudaStreamCreateWithFlags(&ci, cudaStreamNonBlocking));
    SK(cudaStreamCreateWithFlags(&co, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      SK(cudaEventCreateWithFlags(&evI[i], cudaEventDisableTiming));
      SK(cudaEventCreateWithFlags(&evK[i], cudaEventDisableTiming));
      SK(cudaEventCreateWithFlags(&evO[i], cudaEventDisableTiming));
      SK(cudaEventRecord(evK[i], s));
      SK(cudaEventRecord(evO[i], co));
    }
    return GDP_OK;
  }
  int sync() {
    SK(cudaStreamSynchronize(ci));
    SK(cudaStreamSynchronize(s));
    SK(cudaStreamSynchronize(co));
    return GDP_OK;
  }
};

// ---------------------------------------------------------------------------------
// phase 1
// ---------------------------------------------------------------------------------
struct Stream1 {
  Hier* H = nullptr;
  const void* I0h = nullptr;  // host, nx*ny*nz of tI
  float* xh = nullptr;        // host, the finest iterate (the caller's I1)
  int tI = 0;
  long long nx = 0, ny = 0, plane = 0;
  int nz = 0, C = 0;          // chunk planes
  size_t sI = 1;
  DevBuf xin[2], xout[2], iw[2], bw[2];
  DevBuf xin16[2], xout16[2];  // fp16 staging of the iterate's window (NEXT-4)
  int R = 0;                      // partial residency: planes [0, R) of the iterate live in xres (HBM)
  DevBuf xres;                    //   (no host-link traffic per pass; copied back once at the end)
  DevBuf i0res;                   // I0 resident on the device (when every plane of x is)
  static constexpr int MAXS = 8;  // sweeps per streaming pass (NEXT-2)
  int ms = 1;                     // sweeps one pass may hold (window memory)
  DevBuf sw[MAXS][2];             // input windows of stages 1.. of a multi-sweep pass
  __half* h16 = nullptr;       // host fp16 iterate (pinned; Ctx::h16, allocated on first use)
  DevBuf part;                // norm partials (init: per plane rows; sweeps: per item)
  DevBuf psum;                // plane sums (mean pin)
  size_t part_cap = 0;
  Streams st;
  long long h2d = 0, d2h = 0;  // bytes moved over the host link
};

enum { SP_INIT = 0, SP_SUMS = 2, SP_WIDEN = 3 };  // the sweeps stream through stream_sweeps

static int chunk_count(const Stream1& S) { return (S.nz + S.C - 1) / S.C; }

// Planes [from, to) of the iterate into the device window dst: the resident planes (< S.R) by a
// device copy, the others over the host link (fp32, or the fp16 scratch converted on the way).
static int x_load(Stream1& S, float* dst, void* stage16, int from, int to, bool in16, cudaStream_t st) {
  const long long pl = S.plane;
  const int r = std::min(to, S.R);
  if (r > from)
    SK(cudaMemcpyAsync(dst, S.xres.f() + (long long)from * pl, sizeof(float) * pl * (r - from), cudaMemcpyDeviceToDevice, st));
  const int h0 = std::max(from, S.R);
  if (to > h0) {
    float* d = dst + (long long)(h0 - from) * pl;
    const long long n = pl * (to - h0);
    if (in16) {
      SK(cudaMemcpyAsync(stage16, S.h16 + h0 * pl, sizeof(__half) * n, cudaMemcpyHostToDevice, st));
      convert(stage16, d, n, false, st);
      S.h2d += (long long)sizeof(__half) * n;
    } else {
      SK(cudaMemcpyAsync(d, S.xh + h0 * pl, sizeof(float) * n, cudaMemcpyHostToDevice, st));
      S.h2d += (long long)sizeof(float) * n;
    }
  }
  return GDP_OK;
}
// the I0 planes [lo, hi) into the device window
static int i0_load(Stream1& S, unsigned char* dst, int lo, int hi, cudaStream_t st) {
  const long long pl = S.plane;
  if (hi <= lo) return GDP_OK;
  if (S.i0res.p) {
    SK(cudaMemcpyAsync(dst, S.i0res.u() + S.sI * lo * pl, S.sI * pl * (hi - lo), cudaMemcpyDeviceToDevice, st));
  } else {
    SK(cudaMemcpyAsync(dst, static_cast<const unsigned char*>(S.I0h) + S.sI * lo * pl, S.sI * pl * (hi - lo),
                       cudaMemcpyHostToDevice, st));
    S.h2d += (long long)S.sI * pl * (hi - lo);
  }
  return GDP_OK;
}
// fp16 conversion of the host part of output planes [lo, hi) held in src (on the kernel stream)
static void x_convert_out(Stream1& S, const float* src, void* stage16, int lo, int hi, cudaStream_t st) {
  const int h0 = std::max(lo, S.R);
  if (hi > h0) convert(src + (long long)(h0 - lo) * S.plane, stage16, S.plane * (hi - h0), true, st);
}
// output planes [lo, hi) of src back to the iterate: resident planes by a device copy, the others over
// the host link (fp32, or the fp16 staged by x_convert_out)
static int x_store(Stream1& S, const float* src, const void* stage16, int lo, int hi, bool out16, cudaStream_t st) {
  const long long pl = S.plane;
  const int r = std::min(hi, S.R);
  if (r > lo)
    SK(cudaMemcpyAsync(S.xres.f() + (long long)lo * pl, src, sizeof(float) * pl * (r - lo), cudaMemcpyDeviceToDevice, st));
  const int h0 = std::max(lo, S.R);
  if (hi > h0) {
    const long long n = pl * (hi - h0);
    if (out16) {
      SK(cudaMemcpyAsync(S.h16 + h0 * pl, stage16, sizeof(__half) * n, cudaMemcpyDeviceToHost, st));
      S.d2h += (long long)sizeof(__half) * n;
    } else {
      SK(cudaMemcpyAsync(S.xh + h0 * pl, src + (long long)(h0 - lo) * pl, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
      S.d2h += (long long)sizeof(float) * n;
    }
  }
  return GDP_OK;
}

// One streaming pass over the finest level.  SP_INIT: x0 = I0 (written to the host iterate),
// initial residual partials (per plane rows).  SP_SUMS: per-plane fp64 sums of x and I0 (the mean pin).  SP_WIDEN:
// the fp16 host iterate back to fp32.  in16 / out16: the host iterate is read from / written to
// the fp16 scratch instead of the caller's fp32 buffer (NEXT-4).
static int stream_pass(Stream1& S, int kind, bool in16 = false, bool out16 = false) {
  Hier& H = *S.H;
  const Level& L0 = H.lv[0];
  Streams& T = S.st;
  const long long pl = S.plane;
  const int K = chunk_count(S);
  for (int k = 0; k < K; ++k) {
    const int b = k & 1;
    const int p_lo = k * S.C, p_hi = std::min(p_lo + S.C, S.nz);
    const int wlo = std::max(p_lo - 3, 0), whi = std::min(p_hi + 3, S.nz);
    // ---- inputs of the window: retained planes (device), new planes (host), I0 (host)
    SK(cudaStreamWaitEvent(T.ci, T.evK[b], 0));  // chunk k-2's kernels are done with buffer set b
    if (kind != SP_INIT) SR(x_load(S, S.xin[b].f(), S.xin16[b].p, p_lo, p_hi, in16, T.ci));  // the chunk's own planes
    if (kind != SP_WIDEN) SR(i0_load(S, S.iw[b].u(), wlo, whi, T.ci));
    SK(cudaEventRecord(T.evI[b], T.ci));
    // ---- kernels
    SK(cudaStreamWaitEvent(T.s, T.evI[b], 0));
    SK(cudaStreamWaitEvent(T.s, T.evO[b], 0));  // chunk k-2's output left the device
    const unsigned char* iwin = S.iw[b].u();
    if (kind == SP_INIT) {
      LevelK Lk = L0.K;
      Lk.nzl = p_hi - p_lo;
      Lk.z0 = p_lo;
      RhsK R{nullptr, iwin + S.sI * (p_lo - wlo) * pl, nullptr, 0.f, 0};
      const int per = init_blocks_per_plane(L0.nx, L0.ny);
      launch_init(Lk, R, S.tI, S.xout[b].f(), S.bw[b].f() + (p_lo - wlo) * pl,
                  static_cast<double2*>(S.part.p) + (long long)p_lo * per, T.s);
    } else if (kind == SP_WIDEN) {
      SK(cudaMemcpyAsync(S.xout[b].f(), S.xin[b].f(), sizeof(float) * pl * (p_hi - p_lo), cudaMemcpyDeviceToDevice,
                         T.s));
    } else {
      const int per = norms_blocks_per_plane(L0.nx, L0.ny);
      launch_plane_sums(S.xin[b].f(), 1, iwin + S.sI * (p_lo - wlo) * pl, S.tI, L0.nx, L0.ny, p_hi - p_lo,
                        static_cast<double2*>(S.part.p), static_cast<double2*>(S.psum.p) + p_lo, T.s);
      (void)per;
    }
    if (kind != SP_SUMS && out16) x_convert_out(S, S.xout[b].f(), S.xout16[b].p, p_lo, p_hi, T.s);
    SK(cudaGetLastError());
    SK(cudaEventRecord(T.evK[b], T.s));
    // ---- output of the window back to the iterate (in place: no later window reads it)
    if (kind != SP_SUMS) {
      SK(cudaStreamWaitEvent(T.co, T.evK[b], 0));
      SR(x_store(S, S.xout[b].f(), S.xout16[b].p, p_lo, p_hi, out16, T.co));
      SK(cudaEventRecord(T.evO[b], T.co));
    }
  }
  SR(T.sync());
  return GDP_OK;
}

// ---------------------------------------------------------------------------------
// NEXT-2 streaming fusion ("temporal blocking is used to
// perform multiple Gauss-Seidel relaxations in a single streaming pass").  One pass streams the
// host iterate through the device once and applies m sweeps to it: stage j (0-based) of chunk k
// updates planes [p_lo - 3j, p_hi - 3j) (the last chunk: up to nz), i.e. it lags stage j-1 by
// the 3 planes a z-march sweep reads beyond its range, so every stage sweeps every plane exactly
// once and the per-voxel arithmetic is the in-core kernels' (bit-identical iterates).  Stage j
// reads its input window [lo_j - 3, hi_j + 3) from a device buffer holding stage j-1's output
// (planes of earlier chunks retained, this chunk's written by stage j-1 directly); the last
// stage's planes go back to the host.  A V-cycle's up pass and the next cycle's down pass become
// one pass (prolongation, nu_post sweeps with the norms, nu_pre sweeps with the restriction).
// ---------------------------------------------------------------------------------
struct Stage { bool prolong; int tail; };
constexpr int LAG = 3;

static void stage_range(const Stream1& S, int k, int j, int& lo, int& hi) {
  const int K = chunk_count(S);
  const int p_lo = k * S.C, p_hi = std::min(p_lo + S.C, S.nz);
  lo = std::max(0, p_lo - LAG * j);
  hi = k == K - 1 ? S.nz : std::max(0, p_hi - LAG * j);
  if (k == 0) lo = 0;
}

static int stream_sweeps(Stream1& S, const std::vector<Stage>& st, long long* items_out, bool in16, bool out16) {
  Hier& H = *S.H;
  const Level& L0 = H.lv[0];
  const Level& L1 = H.lv[1];
  Streams& T = S.st;
  const long long pl = S.plane;
  const int K = chunk_count(S), m = (int)st.size(), nz = S.nz;
  if (m < 1 || m > Stream1::MAXS) return set_err(GDP_EINVAL, "stream_sweeps: %d stages", m);
  long long items = 0;
  int plo[Stream1::MAXS], phi[Stream1::MAXS];  // previous chunk's input window of each stage
  for (int j = 0; j < m; ++j) plo[j] = phi[j] = 0;
  for (int k = 0; k < K; ++k) {
    const int b = k & 1;
    int lo[Stream1::MAXS], hi[Stream1::MAXS], wlo[Stream1::MAXS], whi[Stream1::MAXS];
    for (int j = 0; j < m; ++j) {
      stage_range(S, k, j, lo[j], hi[j]);
      wlo[j] = std::max(lo[j] - LAG, 0);
      whi[j] = std::min(hi[j] + LAG, nz);
    }
    const int blo = wlo[m - 1], bhi = whi[0];  // rhs window: every stage's input range
    // ---- stage 0's input: retained planes of the previous window, new planes from the host
    SK(cudaStreamWaitEvent(T.ci, T.evK[b], 0));  // chunk k-2's kernels are done with buffer set b
    int from = wlo[0];
    if (k > 0 && phi[0] > wlo[0]) {
      SK(cudaMemcpyAsync(S.xin[b].f(), S.xin[b ^ 1].f() + (wlo[0] - plo[0]) * pl, sizeof(float) * pl * (phi[0] - wlo[0]),
                         cudaMemcpyDeviceToDevice, T.ci));
      from = phi[0];
    }
    if (whi[0] > from) SR(x_load(S, S.xin[b].f() + (from - wlo[0]) * pl, S.xin16[b].p, from, whi[0], in16, T.ci));
    SR(i0_load(S, S.iw[b].u(), blo, bhi, T.ci));
    SK(cudaEventRecord(T.evI[b], T.ci));
    // ---- kernels: the rhs of the window, then the stages in order
    SK(cudaStreamWaitEvent(T.s, T.evI[b], 0));
    SK(cudaStreamWaitEvent(T.s, T.evO[b], 0));  // chunk k-2's output left the device
    LevelK Lw = L0.K;
    Lw.nzl = bhi - blo;
    launch_rhs(Lw, RhsK{nullptr, S.iw[b].u(), nullptr, 0.f, 0}, S.tI, S.bw[b].f(), T.s);  // a2 on the window
    const float* bglob = S.bw[b].f() - (long long)blo * pl;
    for (int j = 1; j < m; ++j) {  // retained input planes of stages 1.. (produced by earlier chunks)
      const int rto = std::min(phi[j], lo[j - 1]);
      if (k > 0 && rto > wlo[j])
        SK(cudaMemcpyAsync(S.sw[j][b].f(), S.sw[j][b ^ 1].f() + (wlo[j] - plo[j]) * pl,
                           sizeof(float) * pl * (rto - wlo[j]), cudaMemcpyDeviceToDevice, T.s));
    }
    for (int j = 0; j < m; ++j) {
      if (hi[j] <= lo[j]) continue;
      const float* in = (j == 0 ? S.xin[b].f() : S.sw[j][b].f()) - (long long)wlo[j] * pl;
      float* out = j == m - 1 ? S.xout[b].f() - (long long)lo[j] * pl : S.sw[j + 1][b].f() - (long long)wlo[j + 1] * pl;
      const int tail = st[j].tail;
      const int n = fused_sweep3d(L0, L1, in, out, bglob, false, st[j].prolong, tail,
                                  tail == 2 ? static_cast<double2*>(S.part.p) + items : nullptr, T.s, lo[j], hi[j]);
      if (tail == 2) items += n;  // the norms stage's partials, in plane order over the chunks
    }
    const int olo = lo[m - 1], ohi = hi[m - 1];
    if (ohi > olo && out16) x_convert_out(S, S.xout[b].f(), S.xout16[b].p, olo, ohi, T.s);
    SK(cudaGetLastError());
    SK(cudaEventRecord(T.evK[b], T.s));
    // ---- the last stage's planes back to the iterate (no later window reads them)
    if (ohi > olo) {
      SK(cudaStreamWaitEvent(T.co, T.evK[b], 0));
      SR(x_store(S, S.xout[b].f(), S.xout16[b].p, olo, ohi, out16, T.co));
    }
    SK(cudaEventRecord(T.evO[b], T.co));
    for (int j = 0; j < m; ++j) { plo[j] = wlo[j]; phi[j] = whi[j]; }
  }
  SR(T.sync());
  if (items_out) *items_out = items;
  return GDP_OK;
}

static int read_norms(Stream1& S, double2* plane_rows, int per, int nplanes, double& rr, double& bb) {
  Hier& H = *S.H;
  launch_finalize(plane_rows, per, nplanes, H.plane_sums, S.st.s);
  SK(cudaMemcpyAsync(H.h_plane, H.plane_sums, sizeof(double2) * nplanes, cudaMemcpyDeviceToHost, S.st.s));
  SK(cudaStreamSynchronize(S.st.s));
  rr = bb = 0.0;
  for (int z = 0; z < nplanes; ++z) { rr += H.h_plane[z].x; bb += H.h_plane[z].y; }
  return GDP_OK;
}

// Phase 1 with a host-resident finest level.  xh receives I1 (before the mean pin; *shift_out
// is the pin, applied by the caller).
int stream_diffuse_z(Ctx& C, const void* I0h, int tI, float* xh, long long nx, long long ny, long long nz,
                     float bx, float by, float bz, const gdp_opts& o0, size_t budget, gdp_report* rep,
                     double* shift_out, float** keep_x, int* keep_R, float** host_scratch, void** keep_i0) {
  if (!xh && (!keep_x || !keep_R || !host_scratch))
    return set_err(GDP_EINVAL, "stream_diffuse_z: a NULL host iterate needs the residency hand-off");
  gdp_opts o = o0;
  o.fused |= 2;
  if (o.nu_pre < 1 || o.nu_post < 1)  // every finest-level pass is a fused sweep (restrict / prolong inside)
    return set_err(GDP_EINVAL, "out-of-core phase 1 needs nu_pre >= 1 and nu_post >= 1");
  HierKey key{};
  key.nx = nx; key.ny = ny; key.nzl = nz; key.z0 = 0; key.nzg = nz;
  key.bx = bx; key.by = by; key.bz = bz; key.alpha = 0.f;
  key.coarse_max = o.coarse_max;
  key.omega = o.omega;
  std::vector<Level> chain;
  int ff;
  SR(level_chain(key, chain, ff));
  if (chain.size() < 2) return set_err(GDP_EINVAL, "out-of-core phase 1 needs at least two levels");
  // resident coarse levels: x, x2, b per voxel (plus small tables)
  double coarse = 0.0;
  for (size_t l = 1; l < chain.size(); ++l) coarse += 12.0 * chain[l].nx * chain[l].ny * chain[l].nzl;
  const long long pl = nx * ny;
  const size_t sI = tI == 0 ? 1 : 4;
  // NEXT-2: sweeps per streaming pass.  MS = nu_pre + nu_post fuses a cycle's up pass with the next
  // cycle's down pass, max(nu_pre, nu_post) keeps one pass per half-cycle, 1 is one pass per sweep.
  // Device windows per pass (two sets): x in C + 6 planes, the last stage's output C + 3 (MS - 1),
  // I0 and b C + 3 MS + 3, stage j's input C + 3 j + 6 (j >= 1), fp16 staging 2 B per x plane.
  auto fixed_planes = [&](int ms) {  // bytes per plane x: the C-independent part of the windows
    double f = 4.0 * 6 + 4.0 * 3 * (ms - 1) + (4.0 + sI) * (3 * ms + 3) + 2.0 * (6 + 3 * (ms - 1));
    for (int j = 1; j < ms; ++j) f += 4.0 * (3 * j + 6);
    return 2.0 * f;
  };
  auto per_plane_of = [&](int ms) { return 2.0 * (4.0 + 4.0 + sI + 4.0 + 4.0 * (ms - 1) + 4.0); };
  size_t freeb = 0, totb = 0;
  SK(cudaMemGetInfo(&freeb, &totb));
  const double hard = 0.9 * (double)freeb - coarse;  // what the windows may take at most
  int MS = std::max(o.nu_pre, o.nu_post);
  if (o.stream_fuse && (double)pl * (fixed_planes(o.nu_pre + o.nu_post) + 2 * per_plane_of(o.nu_pre + o.nu_post)) <= hard)
    MS = o.nu_pre + o.nu_post;
  else if (!o.stream_fuse || (double)pl * (fixed_planes(MS) + 2 * per_plane_of(MS)) > hard)
    MS = 1;  // no room (or no wish) for multi-sweep windows: one pass per sweep
  if (MS > Stream1::MAXS) return set_err(GDP_EINVAL, "out-of-core phase 1: at most %d sweeps per pass", Stream1::MAXS);
  const bool fuse = MS == o.nu_pre + o.nu_post && o.stream_fuse;  // cross-cycle fusion in this solve
  // the budget is a target: below two-plane windows the streamer still runs (C = 2) and only
  // a failing allocation is an error; windows beyond a few dozen planes buy nothing (the pipeline
  // keeps two in flight) and would crowd out the coarse levels' lazily allocated buffers
  const double wcap = std::min((double)budget - coarse - 4.0 * 1024 * 1024, hard) - (double)pl * fixed_planes(MS);
  // a13 partial residency first: with 4-plane chunks, what the budget leaves holds planes [0, R) of the
  // iterate in HBM (no host-link traffic for them per pass); the chunks then take what remains, up to
  // 16 planes (two chunks in flight keep the copies and kernels overlapped; more buys nothing)
  const double xb = 4.0 * (double)pl, margin = 64.0 * 1024 * 1024;
  const int Rp = (int)std::max(0.0, std::min((double)nz, std::floor((wcap - margin - 4.0 * pl * per_plane_of(MS)) / xb)));
  const double left = wcap - margin - xb * Rp;
  int Cp = (int)std::min<double>(std::min<double>((double)nz, 16.0), std::max(2.0, std::floor(left / ((double)pl * per_plane_of(MS)))));
  Cp = std::max(2, Cp & ~1);
  Stream1 S;
  S.I0h = I0h; S.xh = xh; S.tI = tI; S.nx = nx; S.ny = ny; S.plane = pl; S.nz = (int)nz; S.C = Cp; S.sI = sI;
  S.ms = MS;
  std::unique_ptr<Hier> Hp;
  SR(build_hier_levels(key, chain, 0, (int)chain.size(), false, true, Hp));
  S.H = Hp.get();
  if (!fusable3d(S.H->lv[0], S.H->lv[1], o))
    return set_err(GDP_EINVAL, "out-of-core phase 1 needs an x/y-coarsened second level (stack too small?)");
  const int cz = (int)nz + 6;  // no window exceeds the stack plus its halo
  size_t free_before = 0;
  SK(cudaMemGetInfo(&free_before, &totb));
  for (int b = 0; b < 2; ++b) {
    SR(S.xin[b].alloc(sizeof(float) * pl * std::min(Cp + 6, cz)));
    SR(S.xout[b].alloc(sizeof(float) * pl * std::min(Cp + 3 * (MS - 1), cz)));
    SR(S.iw[b].alloc(sI * pl * std::min(Cp + 3 * MS + 3, cz)));
    SR(S.bw[b].alloc(sizeof(float) * pl * std::min(Cp + 3 * MS + 3, cz)));
    for (int j = 1; j < MS; ++j) SR(S.sw[j][b].alloc(sizeof(float) * pl * std::min(Cp + 3 * j + 6, cz)));
  }
  const int per_init = init_blocks_per_plane((int)nx, (int)ny);
  long long items_all = 0;
  for (int j = 0; j < MS; ++j) {  // the norms stage can sit at any lag
    long long it = 0;
    for (int k = 0; k < chunk_count(S); ++k) {
      int lo, hi;
      stage_range(S, k, j, lo, hi);
      if (hi > lo) it += fused3d_items(S.H->lv[0], S.H->lv[1], lo, hi);
    }
    items_all = std::max(items_all, it);
  }
  S.part_cap = std::max<size_t>({(size_t)per_init * nz, (size_t)items_all,
                                 (size_t)norms_blocks_per_plane((int)nx, (int)ny) * Cp});
  SR(S.part.alloc(sizeof(double2) * S.part_cap));
  SR(S.psum.alloc(sizeof(double2) * nz));
  // a13 partial residency (sized above): planes [0, R) of the iterate stay in HBM (one copy back at
  // the end), and I0 as well when every plane does and the budget allows
  {
    size_t free_now = 0;
    SK(cudaMemGetInfo(&free_now, &totb));
    const double windows = (double)free_before - (double)free_now;
    const double avail = std::min((double)budget - coarse - windows, 0.85 * (double)free_now - coarse) - margin;
    S.R = (int)std::max(0.0, std::min((double)Rp, std::floor(avail / xb)));
    if (S.R > 0) SR(S.xres.alloc(sizeof(float) * pl * S.R));
    if (!xh) {  // no caller I1: a pinned scratch for the planes that do not stay in HBM only
      float* scr = nullptr;
      if (S.R < nz) SK(cudaMallocHost(&scr, sizeof(float) * pl * (nz - S.R)));
      *host_scratch = scr;
      S.xh = scr ? scr - (long long)S.R * pl : nullptr;  // planes >= R are addressed as in a full array
    }
    if (S.R == nz && avail - xb * nz >= (double)sI * pl * nz) {
      SR(S.i0res.alloc(sI * pl * nz));
      SK(cudaMemcpy(S.i0res.p, I0h, sI * pl * nz, cudaMemcpyHostToDevice));  // once, before any stream work
      S.h2d += (long long)sI * pl * nz;
    }
  }
  SR(S.st.create());
  cudaEvent_t e0, e1;
  SK(cudaEventCreate(&e0));
  SK(cudaEventCreate(&e1));
  SK(cudaEventRecord(e0, S.st.s));

  gdp_report r{};
  r.dx_inf = -1.0;  // the a9 correction norm is measured by the single-rank in-core solve only
  r.levels = (int)S.H->lv.size();
  // initial guess x0 = I0, b, initial residual
  SR(stream_pass(S, SP_INIT));
  double rr, bb;
  SR(read_norms(S, static_cast<double2*>(S.part.p), per_init, (int)nz, rr, bb));
  double rel = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
  r.rel_res[0] = rel;
  r.norm_b = std::sqrt(bb);
  if (!std::isfinite(rel)) return set_err(GDP_EINVAL, "non-finite initial residual (non-finite input?)");
  Fine f;  // levels >= 1 only: run_vcycle(l0 = 1) never touches the finest level
  f.mode = RHS_B;
  int status = GDP_OK, stall = 0, k = 0;
  const int cap = std::min(o.max_vcycles, GDP_MAX_CYCLES);
  bool stored16 = false;  // the host iterate currently lives in the fp16 scratch (NEXT-4)
  double q = 0.1;         // contraction per cycle, observed (first cycle: assumed)
  bool down_done = false; // the last pass already ran the next cycle's down sweeps (NEXT-2)
  std::vector<Stage> down, up;
  for (int i = 0; i < o.nu_pre; ++i) down.push_back(Stage{false, i == o.nu_pre - 1 ? 1 : 0});
  for (int i = 0; i < o.nu_post; ++i) up.push_back(Stage{i == 0, i == o.nu_post - 1 ? 2 : 0});
  while (rel > o.rel_tol || stored16 || down_done) {
    if (k >= cap) { status = GDP_ENOCONV; break; }
    // NEXT-4: this cycle stores fp16 if its residual is predicted to stay above HALF_REL
    const bool h = o.half_staging && rel * q > HALF_REL;
    if (h && !S.h16) {
      const size_t need = sizeof(__half) * (size_t)pl * nz;
      if (C.h16_bytes < need) {
        if (C.h16) cudaFreeHost(C.h16);
        C.h16 = nullptr;
        C.h16_bytes = 0;
        SK(cudaMallocHost(&C.h16, need));
        C.h16_bytes = need;
      }
      S.h16 = static_cast<__half*>(C.h16);
      for (int b = 0; b < 2; ++b) {
        SR(S.xin16[b].alloc(sizeof(__half) * pl * std::min(Cp + 6, cz)));
        SR(S.xout16[b].alloc(sizeof(__half) * pl * std::min(Cp + 3 * (MS - 1), cz)));
      }
    }
    // a list of sweeps: one streaming pass (stream_fuse) or one pass per sweep
    auto run = [&](const std::vector<Stage>& list, long long* items) -> int {  // passes of <= S.ms sweeps
      for (size_t a = 0; a < list.size(); a += S.ms) {
        const std::vector<Stage> part(list.begin() + a, list.begin() + std::min(list.size(), a + S.ms));
        long long it = 0;
        SR(stream_sweeps(S, part, &it, stored16, h));
        stored16 = h;
        bool norms = false;
        for (const Stage& g : part) norms |= g.tail == 2;
        if (norms && items) *items = it;
      }
      return GDP_OK;
    };
    if (!down_done) SR(run(down, nullptr));
    SR(run_vcycle(C, *S.H, f, o, S.st.s, 1));
    SK(cudaStreamSynchronize(S.st.s));
    // NEXT-2: unless this cycle is predicted to be the last, its up pass also runs the next
    // cycle's down sweeps (one host-link round trip per V-cycle instead of two)
    const bool fz = fuse && k + 1 < cap && rel > o.rel_tol && rel * q > 4.0 * o.rel_tol;
    std::vector<Stage> pass = up;
    if (fz) pass.insert(pass.end(), down.begin(), down.end());
    long long items = 0;
    SR(run(pass, &items));
    down_done = fz;
    SR(read_norms(S, static_cast<double2*>(S.part.p), (int)items, 1, rr, bb));
    const double nrel = bb > 0 ? std::sqrt(rr / bb) : std::sqrt(rr);
    ++k;
    r.rel_res[k] = nrel;
    if (!std::isfinite(nrel)) return set_err(GDP_EINVAL, "non-finite residual after V-cycle %d", k);
    q = std::min(1.0, std::max(1e-3, nrel / std::max(rel, 1e-300)));
    if (o.stagnation > 0 && nrel > 0.9 * rel) {
      // (not after a fused pass: the stored iterate is then one the norms did not measure)
      if (++stall >= o.stagnation && !down_done) { rel = nrel; status = nrel <= o.rel_tol ? GDP_OK : GDP_ENOCONV; break; }
    } else {
      stall = 0;
    }
    rel = nrel;
  }
  if (stored16) SR(stream_pass(S, SP_WIDEN, true, false));  // ended on an fp16 cycle (cap)
  r.vcycles = k;
  r.status = status;
  // a10: mean pin, per-plane fp64 sums in plane order (the in-core reduction)
  SR(stream_pass(S, SP_SUMS));
  double2* hp = nullptr;
  SK(cudaMallocHost(&hp, sizeof(double2) * nz));
  cudaMemcpy(hp, S.psum.p, sizeof(double2) * nz, cudaMemcpyDeviceToHost);
  double sx = 0.0, si = 0.0;
  for (long long z = 0; z < nz; ++z) { sx += hp[z].x; si += hp[z].y; }
  cudaFreeHost(hp);
  *shift_out = (si - sx) / ((double)pl * nz);
  if (S.R > 0 && keep_x && keep_R) {  // phase 2 takes the resident planes over (reads them in place)
    SK(cudaStreamSynchronize(S.st.s));
    *keep_x = S.xres.f();
    *keep_R = S.R;
    S.xres.p = nullptr;
    if (keep_i0 && S.i0res.p) {  // I0 resident too: phase 2 reads it in place
      *keep_i0 = S.i0res.p;
      S.i0res.p = nullptr;
    }
  } else if (S.R > 0) {  // the resident planes back to the caller's iterate, once
    SK(cudaMemcpyAsync(S.xh, S.xres.p, sizeof(float) * pl * S.R, cudaMemcpyDeviceToHost, S.st.s));
    SK(cudaStreamSynchronize(S.st.s));
    S.d2h += (long long)sizeof(float) * pl * S.R;
  }
  SK(cudaEventRecord(e1, S.st.s));
  SK(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  r.seconds = ms * 1e-3;
  r.hbm_bytes_est = (double)(S.h2d + S.d2h);  // host-link bytes of the streamed finest level
  if (rep) *rep = r;
  return status;
}

// Phase 2 on slice batches; I1h gets the phase-1 mean pin `shift` added on the way (and written
// back so the caller's I1 is the pinned solution).
int stream_slices(Ctx& C, gdp_ctx* cctx, const void* I0h, gdp_dtype dtype, float* I1h, float* I2h, long long nx,
                  long long ny, long long nz, float alpha, double shift, const gdp_opts& o, size_t budget,
                  gdp_report* rep, const float* I1dev, int R, bool write_i1, const void* I0dev) {
  const long long pl = nx * ny;
  const size_t sI = dtype == GDP_U8 ? 1 : 4;
  // per slice on the device: I0, I1, I2 of two batches + the batch hierarchy (~4 fp32 arrays)
  const double per_slice = (double)pl * (2.0 * (sI + 8.0) + 16.0);
  long long B = (long long)std::floor(((double)budget - 4.0 * 1024 * 1024) / per_slice);
  B = std::max(1LL, std::min(std::min(B, nz), 64LL));
  DevBuf i0[2], i1[2], i2[2];
  for (int b = 0; b < 2; ++b) {
    SR(i0[b].alloc(sI * pl * B));
    SR(i1[b].alloc(sizeof(float) * pl * B));
    SR(i2[b].alloc(sizeof(float) * pl * B));
  }
  Streams T;
  SR(T.create());
  gdp_report agg{};
  agg.dx_inf = -1.0;
  agg.status = GDP_OK;
  const float fs = (float)shift;
  int k = 0;
  for (long long z = 0; z < nz; z += B, ++k) {
    const int b = k & 1;
    const long long nb = std::min(B, nz - z);
    SK(cudaStreamWaitEvent(T.ci, T.evO[b], 0));
    if (I0dev)  // I0 still resident from phase 1
      SK(cudaMemcpyAsync(i0[b].u(), static_cast<const unsigned char*>(I0dev) + sI * z * pl, sI * pl * nb,
                         cudaMemcpyDeviceToDevice, T.ci));
    else
      SK(cudaMemcpyAsync(i0[b].u(), static_cast<const unsigned char*>(I0h) + sI * z * pl, sI * pl * nb,
                         cudaMemcpyHostToDevice, T.ci));
    // I1 of the batch: slices still resident from phase 1 by a device copy, the others from the host
    const long long zr = std::min<long long>(z + nb, R);
    if (zr > z)
      SK(cudaMemcpyAsync(i1[b].f(), I1dev + z * pl, sizeof(float) * pl * (zr - z), cudaMemcpyDeviceToDevice, T.ci));
    const long long zh = std::max<long long>(z, R);
    if (z + nb > zh)
      SK(cudaMemcpyAsync(i1[b].f() + (zh - z) * pl, I1h + zh * pl, sizeof(float) * pl * (z + nb - zh),
                         cudaMemcpyHostToDevice, T.ci));
    SK(cudaEventRecord(T.evI[b], T.ci));
    SK(cudaStreamWaitEvent(T.s, T.evI[b], 0));
    if (fs != 0.f) launch_add_scalar(i1[b].f(), pl * nb, fs, T.s);  // a10 on the way (k_add_scalar arithmetic)
    if (write_i1 && (fs != 0.f || z < R)) {  // the pinned (or still device-resident) I1 back to the caller
      SK(cudaEventRecord(T.evK[b], T.s));
      SK(cudaStreamWaitEvent(T.co, T.evK[b], 0));
      const long long z1 = fs != 0.f ? z + nb : std::min<long long>(z + nb, R);
      SK(cudaMemcpyAsync(I1h + z * pl, i1[b].f(), sizeof(float) * pl * (z1 - z), cudaMemcpyDeviceToHost, T.co));
    }
    gdp_report r{};
    gdp_dims d{nx, ny, nb};
    const int st = gdp_screened_poisson_slices(cctx, i0[b].p, dtype, i1[b].f(), i2[b].f(), d, alpha, &o, &r, T.s);
    if (st != GDP_OK && st != GDP_ENOCONV) return st;
    if (st == GDP_ENOCONV) agg.status = GDP_ENOCONV;
    SK(cudaEventRecord(T.evK[b], T.s));
    SK(cudaStreamWaitEvent(T.co, T.evK[b], 0));
    SK(cudaMemcpyAsync(I2h + z * pl, i2[b].f(), sizeof(float) * pl * nb, cudaMemcpyDeviceToHost, T.co));
    SK(cudaEventRecord(T.evO[b], T.co));
    agg.vcycles = std::max(agg.vcycles, r.vcycles);
    agg.levels = r.levels;
    agg.seconds += r.seconds;
    for (int i = 0; i <= r.vcycles && i <= GDP_MAX_CYCLES; ++i) agg.rel_res[i] = std::max(agg.rel_res[i], r.rel_res[i]);
    agg.norm_b = std::max(agg.norm_b, r.norm_b);
    agg.kernel_launches += r.kernel_launches;
  }
  SR(T.sync());
  (void)C;
  if (rep) *rep = agg;
  return agg.status;
}

}  // namespace gdp
