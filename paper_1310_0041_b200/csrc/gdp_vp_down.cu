// gdp_vp_down.cu — instantiations of the 3D level-pass kernels that end in a restriction
// (down passes; the FMG start's first pass also adds the prolongated correction).
#include "gdp_vpass3d.cuh"

namespace gdp {
namespace vp {
GDP_VP_INST(1, 1, false, false)
GDP_VP_INST(1, 1, false, true)
GDP_VP_INST(1, 1, true, false)
GDP_VP_INST(2, 1, false, false)
GDP_VP_INST(2, 1, false, true)
GDP_VP_INST(2, 1, true, false)
}  // namespace vp
}  // namespace gdp
