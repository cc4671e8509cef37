// gdp_fused.cu — fused level passes (filled in by the fused schedule).
#include "gdp_internal.h"

namespace gdp {

bool fused_down(const Level&, const Level&, float*, const RhsK&, int, int, int, cudaStream_t) {
  return false;
}
bool fused_up(const Level&, const Level&, float*, const RhsK&, int, int, int, cudaStream_t) {
  return false;
}

}  // namespace gdp
