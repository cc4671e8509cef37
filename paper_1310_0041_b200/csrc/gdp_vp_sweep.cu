// gdp_vp_sweep.cu — instantiations of the single-sweep level-pass kernels without a transfer
// (a plain sweep, or a sweep ending in the fp64 norms), used one launch per sweep (fused bit 16).
#include "gdp_vpass3d.cuh"

namespace gdp {
namespace vp {
GDP_VP_INST(1, 0, false, false)
GDP_VP_INST(1, 2, false, false)
}  // namespace vp
}  // namespace gdp
