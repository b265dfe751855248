// Instantiations of the persistent SF kernel for T=double, NB=32 (see sf_launch.cuh).
#include "sf_launch.cuh"

namespace sgsf {
SGSF_DEFINE_LAUNCH(double, 32, 12, 256, 2)
SGSF_DEFINE_LAUNCH(double, 32, 16, 256, 2)
}  // namespace sgsf
