// Instantiations of the persistent SF kernel for T=float, NB=16 (see sf_launch.cuh).
#include "sf_launch.cuh"

namespace sgsf {
SGSF_DEFINE_LAUNCH(float, 16, 12, 384, 1)
SGSF_DEFINE_LAUNCH(float, 16, 16, 384, 1)
}  // namespace sgsf
