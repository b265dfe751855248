// K1L (sf_large.cuh): launch + instantiations for 32 < n <= 64 robots.
#include "sf_launch.cuh"
#include "sf_large.cuh"

namespace sgsf {

template <typename T, int MP, bool HY = false>
static int launch_large_t(const LaunchInfo& li, SolveParams& p, const sgsf_config_t* cfg, const sgsf_timing_t* timing,
                          cudaStream_t stream) {
    auto kern = sf_large_kernel<T, 64, MP, HY>;
    set_family_constants(p);
    int dev_smem = 0;
    cudaError_t e = cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, li.device);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, cudaGetErrorString(e));
    p.large_coop = 1;
    LargeLayout L = make_large_layout<T, 64>(p.n, p.S, MP, p.want_prev || HY, 1);
    if (L.total > (size_t)dev_smem) {   // phase B's partials do not fit: the one-warp exact pass
        p.large_coop = 0;
        L = make_large_layout<T, 64>(p.n, p.S, MP, p.want_prev || HY, 0);
    }
    if (L.total > (size_t)dev_smem)
        return internal_fail(SGSF_ERR_UNSUPPORTED, "problem too large for one CTA: one sample needs " +
                                                       std::to_string(L.total / 1024) + " KB of shared memory, the device allows " +
                                                       std::to_string(dev_smem / 1024) + " KB");
    p.MP = MP;
    p.spb = 1;
    p.wps = kLargeWarps;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, cudaGetErrorString(e));
    int grid = cfg->grid > 0 ? cfg->grid : li.sm_count;
    if (grid > p.batch) grid = p.batch;
    if (timing && timing->start) cudaEventRecord((cudaEvent_t)timing->start, stream);
    kern<<<grid, 32 * kLargeWarps, L.total, stream>>>(p);
    internal_count_launch(1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, std::string("sf_large launch: ") + cudaGetErrorString(e));
    if (timing && timing->stop) cudaEventRecord((cudaEvent_t)timing->stop, stream);
#ifdef SGSF_COUNTERS
    {
        unsigned long long c[8];
        cudaStreamSynchronize(stream);
        cudaMemcpyFromSymbol(c, g_sgsf_counts, sizeof(c));
        printf("COUNTS(K1L) exact_steps %llu quiet_steps %llu\n", c[5], c[6]);
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_sgsf_counts, z, sizeof(z));
    }
#endif
    return SGSF_OK;
}

int launch_large(const LaunchInfo& li, SolveParams& p, const sgsf_config_t* cfg, const sgsf_timing_t* timing,
                 cudaStream_t stream, bool strict) {
    const bool wide = p.m1 > 12;
    if (cfg->precision == SGSF_PRECISION_HYBRID)
        return wide ? launch_large_t<float, 16, true>(li, p, cfg, timing, stream)
                    : launch_large_t<float, 12, true>(li, p, cfg, timing, stream);
    if (strict)
        return wide ? launch_large_t<double, 16>(li, p, cfg, timing, stream)
                    : launch_large_t<double, 12>(li, p, cfg, timing, stream);
    return wide ? launch_large_t<float, 16>(li, p, cfg, timing, stream)
                : launch_large_t<float, 12>(li, p, cfg, timing, stream);
}

}  // namespace sgsf
