// Instantiations of the persistent SF kernel for T=double, NB=4 (see sf_launch.cuh).
#include "sf_launch.cuh"

namespace sgsf {
SGSF_DEFINE_LAUNCH(double, 4, 12, 384, 1)
SGSF_DEFINE_LAUNCH(double, 4, 16, 384, 1)
}  // namespace sgsf
