// gdp_vp_up.cu — instantiations of the 3D level-pass kernels that start with the prolongated
// correction (up passes: fp64 norms of the finest level, or nothing).
#include "gdp_vpass3d.cuh"

namespace gdp {
namespace vp {
GDP_VP_INST(1, 2, true, false)
GDP_VP_INST(1, 0, true, false)
GDP_VP_INST(2, 2, true, false)
GDP_VP_INST(2, 0, true, false)
}  // namespace vp
}  // namespace gdp
