// gdp_comm.cu — communication layer of a distributed ctx (z-slab halos, fp64 sums).
// Single-rank contexts: every call is a no-op.
#include "gdp_internal.h"

namespace gdp {

struct Comm {};

int comm_init(Ctx& c, const void* nccl_unique_id) {
  (void)nccl_unique_id;
  return set_err(GDP_EINVAL, "world > 1: NCCL partition not available in this build (rank %d)", c.rank);
}

void comm_destroy(Ctx& c) {
  delete c.comm;
  c.comm = nullptr;
}

int comm_allreduce_sum2(Ctx& c, double* a, double* b, cudaStream_t s) {
  (void)a; (void)b; (void)s;
  if (c.world == 1) return GDP_OK;
  return set_err(GDP_ENCCL, "allreduce without communicator");
}

int comm_halo_x(Ctx& c, Hier& H, int level, float* x, cudaStream_t s) {
  (void)H; (void)level; (void)x; (void)s;
  if (c.world == 1) return GDP_OK;
  return set_err(GDP_ENCCL, "halo without communicator");
}

}  // namespace gdp
