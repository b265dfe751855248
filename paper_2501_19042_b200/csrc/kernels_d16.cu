// Instantiations of the persistent SF kernel for T=double, NB=16 (see sf_launch.cuh).
#include "sf_launch.cuh"

namespace sgsf {
SGSF_DEFINE_LAUNCH(double, 16, 12, 256, 1)
SGSF_DEFINE_LAUNCH(double, 16, 16, 256, 1)
}  // namespace sgsf
