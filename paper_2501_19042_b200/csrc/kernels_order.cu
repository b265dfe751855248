// Longest-first sample order (sf_order.cuh): score + bucket sort launches.
#include "sf_launch.cuh"
#include "sf_order.cuh"

namespace sgsf {

template <int NB, int MP>
static int launch_score(const SolveParams& p, float* score, cudaStream_t stream) {
    start_score_kernel<NB, MP><<<p.batch, kScoreThreads, 0, stream>>>(p, score);
    internal_count_launch(1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SGSF_OK : internal_fail(SGSF_ERR_CUDA, std::string("start_score: ") + cudaGetErrorString(e));
}

int launch_order(const SolveParams& p, float* score, int* order, cudaStream_t stream) {
    const bool wide = p.m1 > 12;
    int rc;
    if (p.n <= 4) rc = wide ? launch_score<4, 16>(p, score, stream) : launch_score<4, 12>(p, score, stream);
    else if (p.n <= 8) rc = wide ? launch_score<8, 16>(p, score, stream) : launch_score<8, 12>(p, score, stream);
    else if (p.n <= 16) rc = wide ? launch_score<16, 16>(p, score, stream) : launch_score<16, 12>(p, score, stream);
    else rc = wide ? launch_score<32, 16>(p, score, stream) : launch_score<32, 12>(p, score, stream);
    if (rc != SGSF_OK) return rc;
    lpt_order_kernel<<<1, kOrderThreads, 0, stream>>>(score, p.batch, order);
    internal_count_launch(1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SGSF_OK : internal_fail(SGSF_ERR_CUDA, std::string("lpt_order: ") + cudaGetErrorString(e));
}

}  // namespace sgsf
