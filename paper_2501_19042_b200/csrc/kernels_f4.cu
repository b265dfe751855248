// Instantiations of the persistent SF kernel for T=float, NB=4 (see sf_launch.cuh).
#include "sf_launch.cuh"

namespace sgsf {
SGSF_DEFINE_LAUNCH(float, 4, 12, 512, 1)
SGSF_DEFINE_LAUNCH(float, 4, 16, 512, 1)
}  // namespace sgsf
