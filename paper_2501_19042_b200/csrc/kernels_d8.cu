// Instantiations of the persistent SF kernel for T=double, NB=8 (see sf_launch.cuh).
#include "sf_launch.cuh"

namespace sgsf {
SGSF_DEFINE_LAUNCH(double, 8, 12, 256, 1)
SGSF_DEFINE_LAUNCH(double, 8, 16, 256, 1)
}  // namespace sgsf
