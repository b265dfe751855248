// Instantiations of the persistent SF kernel for T=float, NB=8 (see sf_launch.cuh).
#include "sf_launch.cuh"

namespace sgsf {
SGSF_DEFINE_LAUNCH(float, 8, 12, 384, 1)
SGSF_DEFINE_LAUNCH(float, 8, 16, 384, 1)
}  // namespace sgsf
