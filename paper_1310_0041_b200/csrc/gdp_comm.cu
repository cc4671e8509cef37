// gdp_comm.cu — communication of a z-slab partition: one-plane halos of x
// between neighbouring slabs, the gathered coarse right-hand side, and exact per-plane fp64
// sums.  Two backends with one code path above them:
//   * NCCL (world > 1): one slab per process, ncclSend/ncclRecv over NVLink, ncclAllReduce;
//   * loopback (gdp_ctx_create_loopback): `world` slabs inside one process on one GPU, the
//     "exchange" is a device copy between the slabs' buffers.
// Per-plane sums are made exact and partition-independent by giving every element exactly one
// non-zero contributor (each rank fills its own planes of a zeroed array, then a sum-allreduce);
// the gathered coarse level is an all-gather-v of the slabs' plane ranges.
#include <nccl.h>

#include <vector>

#include "gdp_internal.h"

namespace gdp {

struct Comm {
  ncclComm_t nc = nullptr;
  double* d_sum = nullptr;  // scratch for plane sums (2 * nzg doubles)
  size_t d_sum_cap = 0;
};

#define NCK(call)                                                                     \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess)                                                            \
      return set_err(GDP_ENCCL, "%s failed: %s", #call, ncclGetErrorString(r_));      \
  } while (0)

#define CKC(call)                                                                     \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return set_err(GDP_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

int comm_unique_id(void* out, size_t n) {
  if (!out || n < sizeof(ncclUniqueId)) return set_err(GDP_EINVAL, "unique id buffer < %zu bytes", sizeof(ncclUniqueId));
  ncclUniqueId id;
  NCK(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return GDP_OK;
}

int comm_init(Ctx& c, const void* nccl_unique_id) {
  if (!nccl_unique_id) return set_err(GDP_EINVAL, "world > 1 needs an ncclUniqueId");
  c.comm = new Comm();
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof id);
  NCK(ncclCommInitRank(&c.comm->nc, c.world, id, c.rank));
  return GDP_OK;
}

void comm_destroy(Ctx& c) {
  if (!c.comm) return;
  if (c.comm->nc) ncclCommDestroy(c.comm->nc);
  if (c.comm->d_sum) cudaFree(c.comm->d_sum);
  delete c.comm;
  c.comm = nullptr;
}

// scalar fp64 sums over ranks (the rank holding a value is the only non-zero contributor
// per call site, so the result does not depend on the reduction order)
int comm_allreduce_sum2(Ctx& c, double* a, double* b, cudaStream_t s) {
  if (c.world == 1) return GDP_OK;
  if (!c.comm) return set_err(GDP_ENCCL, "allreduce without communicator");
  if (c.comm->d_sum_cap < 2) {
    if (c.comm->d_sum) cudaFree(c.comm->d_sum);
    CKC(cudaMalloc(&c.comm->d_sum, 2 * sizeof(double)));
    c.comm->d_sum_cap = 2;
  }
  double h[2] = {*a, *b};
  CKC(cudaMemcpyAsync(c.comm->d_sum, h, sizeof h, cudaMemcpyHostToDevice, s));
  NCK(ncclAllReduce(c.comm->d_sum, c.comm->d_sum, 2, ncclDouble, ncclSum, c.comm->nc, s));
  CKC(cudaMemcpyAsync(h, c.comm->d_sum, sizeof h, cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  *a = h[0];
  *b = h[1];
  return GDP_OK;
}

// ---------------------------------------------------------------------------------
// slab partition primitives
// ---------------------------------------------------------------------------------
// ghost planes of level `l` for every local part: xlo <- last plane of the slab below,
// xhi <- first plane of the slab above.  xs[i] = x of level l of local part i.
int comm_halo_parts(Ctx& c, DistPlan& D, int l, float* const* xs, cudaStream_t s) {
  const int np = (int)D.parts.size();
  const Level& L0 = D.parts[0]->lv[l];
  const size_t pl = (size_t)L0.nx * L0.ny;
  if (c.world == 1) {  // loopback: all slabs are local
    for (int i = 0; i < np; ++i) {
      const Level& L = D.parts[i]->lv[l];
      if (i > 0) {
        const Level& B = D.parts[i - 1]->lv[l];
        CKC(cudaMemcpyAsync(L.xlo, xs[i - 1] + (size_t)(B.nzl - 1) * pl, pl * sizeof(float), cudaMemcpyDeviceToDevice, s));
      }
      if (i < np - 1)
        CKC(cudaMemcpyAsync(L.xhi, xs[i + 1], pl * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }
    return GDP_OK;
  }
  const Level& L = D.parts[0]->lv[l];
  NCK(ncclGroupStart());
  if (c.rank > 0) {
    NCK(ncclSend(xs[0], pl, ncclFloat, c.rank - 1, c.comm->nc, s));
    NCK(ncclRecv(L.xlo, pl, ncclFloat, c.rank - 1, c.comm->nc, s));
  }
  if (c.rank < c.world - 1) {
    NCK(ncclSend(xs[0] + (size_t)(L.nzl - 1) * pl, pl, ncclFloat, c.rank + 1, c.comm->nc, s));
    NCK(ncclRecv(L.xhi, pl, ncclFloat, c.rank + 1, c.comm->nc, s));
  }
  NCK(ncclGroupEnd());
  return GDP_OK;
}

// G = DistPlan::G ghost planes per face of the finest-level windows (interior at offset G):
// the bottom ghosts of slab i <- the top G interior planes of slab i-1, the top ghosts <- the
// bottom G interior planes of slab i+1 (every slab has >= G planes).
int comm_ghosts(Ctx& c, DistPlan& D, float* const* wins, cudaStream_t s, int level) {
  const int np = (int)D.parts.size();
  const Level& L0 = D.parts[0]->lv[level];
  const size_t pl = (size_t)L0.nx * L0.ny;
  const int G = DistPlan::G;
  std::vector<int> nzl(np);
  for (int i = 0; i < np; ++i) nzl[i] = D.parts[i]->lv[level].nzl;
  const size_t gb = pl * G * sizeof(float);
  if (c.world == 1) {
    for (int i = 0; i < np; ++i) {
      if (i > 0)
        CKC(cudaMemcpyAsync(wins[i], wins[i - 1] + (size_t)nzl[i - 1] * pl, gb, cudaMemcpyDeviceToDevice, s));
      if (i < np - 1)
        CKC(cudaMemcpyAsync(wins[i] + (size_t)(G + nzl[i]) * pl, wins[i + 1] + (size_t)G * pl, gb,
                            cudaMemcpyDeviceToDevice, s));
    }
    return GDP_OK;
  }
  float* w = wins[0];
  const int n = nzl[0];
  NCK(ncclGroupStart());
  if (c.rank > 0) {
    NCK(ncclSend(w + (size_t)G * pl, pl * G, ncclFloat, c.rank - 1, c.comm->nc, s));
    NCK(ncclRecv(w, pl * G, ncclFloat, c.rank - 1, c.comm->nc, s));
  }
  if (c.rank < c.world - 1) {
    NCK(ncclSend(w + (size_t)n * pl, pl * G, ncclFloat, c.rank + 1, c.comm->nc, s));
    NCK(ncclRecv(w + (size_t)(G + n) * pl, pl * G, ncclFloat, c.rank + 1, c.comm->nc, s));
  }
  NCK(ncclGroupEnd());
  return GDP_OK;
}

// complete the gathered coarse rhs: every slab restricted into its own planes [off_r, off_r +
// cnt_r) (elements) of the full buffer; an all-gather-v of those ranges, as one group of
// ncclBroadcast calls rooted at each rank (in place: the bytes moved are the level, once).
// Loopback: the slabs wrote disjoint ranges of one buffer already.
int comm_gather_full(Ctx& c, DistPlan& D, float* full, cudaStream_t s) {
  if (c.world == 1) return GDP_OK;
  NCK(ncclGroupStart());
  for (int r = 0; r < c.world; ++r) {
    float* p = full + D.goff[r];
    NCK(ncclBroadcast(p, p, D.gcnt[r], ncclFloat, r, c.comm->nc, s));
  }
  NCK(ncclGroupEnd());
  return GDP_OK;
}

// global per-plane (sum a, sum b): `local[i]` holds the planes of local part i (device);
// the result is written to host `out` (nzg entries) in global plane order
int comm_plane_sums(Ctx& c, DistPlan& D, double2* const* local, double2* out, cudaStream_t s) {
  const int np = (int)D.parts.size();
  if (c.world == 1) {
    for (int i = 0; i < np; ++i)
      CKC(cudaMemcpyAsync(out + D.z0[i], local[i], sizeof(double2) * D.nzl[i], cudaMemcpyDeviceToHost, s));
    CKC(cudaStreamSynchronize(s));
    return GDP_OK;
  }
  const size_t need = 2 * (size_t)D.nzg;
  if (c.comm->d_sum_cap < need) {
    if (c.comm->d_sum) cudaFree(c.comm->d_sum);
    CKC(cudaMalloc(&c.comm->d_sum, need * sizeof(double)));
    c.comm->d_sum_cap = need;
  }
  CKC(cudaMemsetAsync(c.comm->d_sum, 0, need * sizeof(double), s));
  CKC(cudaMemcpyAsync(c.comm->d_sum + 2 * D.z0[0], local[0], sizeof(double2) * D.nzl[0], cudaMemcpyDeviceToDevice, s));
  NCK(ncclAllReduce(c.comm->d_sum, c.comm->d_sum, need, ncclDouble, ncclSum, c.comm->nc, s));
  CKC(cudaMemcpyAsync(out, c.comm->d_sum, need * sizeof(double), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  return GDP_OK;
}

}  // namespace gdp
