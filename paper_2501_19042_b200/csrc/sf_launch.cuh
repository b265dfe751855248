// sf_launch.cuh -- host-side launch of K1 for one (T, NB, MP) instantiation.
// Each kernels_*.cu translation unit instantiates a few of these so the
// fully-unrolled kernels compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/sgsf.h"
#include "sf_persistent.cuh"

namespace sgsf {

struct LaunchInfo {
    int device, sm_count;
};

int internal_fail(int code, const std::string& msg);
void internal_count_launch(int n);
// longest-first queue order (kernels_order.cu)
int launch_order(const SolveParams& p, float* score, int* order, cudaStream_t stream);
// K1L for 32 < n <= 64 (kernels_large.cu)
int launch_large(const LaunchInfo& li, SolveParams& p, const sgsf_config_t* cfg, const sgsf_timing_t* timing,
                 cudaStream_t stream, bool strict);

template <typename T, int NB, int MP, int MAXT, int TPS>
int launch_persistent(const LaunchInfo& li, SolveParams& p, const sgsf_config_t* cfg, const sgsf_timing_t* timing,
                      cudaStream_t stream) {
    // hybrid precision: the FP32 kernels with guard bands and FP64 values (sf_persistent.cuh, HY)
    const bool hy = sizeof(T) == 4 && cfg->precision == SGSF_PRECISION_HYBRID;
    void (*kern)(const SolveParams) = sf_persistent_kernel<T, NB, MP, MAXT, TPS>;
    if constexpr (sizeof(T) == 4) {
        if (hy) kern = sf_persistent_kernel<T, NB, MP, MAXT, TPS, false, 0, true>;
    }
    int dev_smem = 0;
    cudaError_t e = cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, li.device);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, cudaGetErrorString(e));
    // a slot is a warp group with its own named barrier (ids 1..15): ceil(S/32) warps with one
    // thread per time step, ceil(S/16) warps with two (TPS = 2: 16 steps per warp)
    const int wps = TPS == 2 ? (p.S + 15) / 16 : (p.S + 31) / 32;
    const int slot_threads = 32 * wps;
    // positions on the tensor cores (3xTF32 tcgen05 GEMM, sf_tc.cuh) when a slot is exactly one
    // 128-lane TMEM tile: float, 16 robots, 97..128 steps.  SGSF_NO_TC=1 keeps the FFMA path.
    bool tc = false;
    if constexpr (sizeof(T) == 4 && NB == 16 && TPS == 1 && MP <= 16) {
        const char* off = std::getenv("SGSF_NO_TC");
        if (wps == 4 && !(off && off[0] == '1')) {
            tc = true;
            // (one term-pass variant per instantiation, FULLN = 1 / 2, is 832 instructions smaller but
            // measured 1% slower)
            kern = hy ? sf_persistent_kernel<T, NB, MP, MAXT, TPS, true, 0, true>
                      : sf_persistent_kernel<T, NB, MP, MAXT, TPS, true>;
        }
    }
    {
        const char* nc = std::getenv("SGSF_NO_COOP");
        p.coop = !(nc && nc[0] == '1');
    }
    int spb = cfg->slots_per_block;
    if (spb <= 0) {
        spb = 0;
        for (int s = 1; s * slot_threads <= MAXT && s <= 15; ++s) {
            if (make_layout<T, NB>(p.n, p.S, MP, s, p.want_prev, tc, hy).total > (size_t)dev_smem) break;
            spb = s;
        }
        // small batches: spread samples over the SMs instead of packing few CTAs
        const int spread = (p.batch + li.sm_count - 1) / li.sm_count;
        if (spb > spread) spb = spread > 0 ? spread : 1;
    }
    if (spb <= 0) {
        const size_t need = make_layout<T, NB>(p.n, p.S, MP, 1, p.want_prev, tc, hy).total;
        return internal_fail(SGSF_ERR_UNSUPPORTED,
                             "problem too large for one CTA: one sample slot needs " + std::to_string(need / 1024) +
                                 " KB of shared memory, the device allows " + std::to_string(dev_smem / 1024) +
                                 " KB (use precision='lean' or a shorter horizon)");
    }
    if (spb > 15) return internal_fail(SGSF_ERR_UNSUPPORTED, "at most 15 slots per CTA (named barriers)");
    const int threads = spb * slot_threads;
    if (threads > MAXT) return internal_fail(SGSF_ERR_UNSUPPORTED, "slots_per_block * samples exceeds the CTA size");
    p.spb = spb;
    p.wps = wps;
    p.MP = MP;
    const SmemLayout L = make_layout<T, NB>(p.n, p.S, MP, spb, p.want_prev, tc, hy);
    p.L = L;
    set_family_constants(p);
    if (L.total > (size_t)dev_smem) return internal_fail(SGSF_ERR_UNSUPPORTED, "shared memory budget exceeded");
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, cudaGetErrorString(e));
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, L.total);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, cudaGetErrorString(e));
    if (per_sm < 1) per_sm = 1;
    int grid = cfg->grid > 0 ? cfg->grid : li.sm_count * per_sm;
    const int need = (p.batch + spb - 1) / spb;
    if (grid > need) grid = need;
    if (timing && timing->start) cudaEventRecord((cudaEvent_t)timing->start, stream);
    kern<<<grid, threads, L.total, stream>>>(p);
    internal_count_launch(1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, std::string("sf_persistent launch: ") + cudaGetErrorString(e));
    if (timing && timing->stop) cudaEventRecord((cudaEvent_t)timing->stop, stream);
#ifdef SGSF_COUNTERS
    {
        unsigned long long c[10];
        cudaStreamSynchronize(stream);
        cudaMemcpyFromSymbol(c, g_sgsf_counts, sizeof(c));
        printf("COUNTS finish %llu flagged %llu exact %llu careful %llu flagged_terms %llu near_checks %llu scans %llu exact_f1 %llu hy_recompute %llu\n",
               c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[8]);
        const unsigned long long z[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_sgsf_counts, z, sizeof(z));
    }
#endif
    return SGSF_OK;
}

// instantiated in kernels_*.cu
#define SGSF_DECLARE_LAUNCH(T, NB, MP, MAXT, TPS)                                                   \
    extern template int launch_persistent<T, NB, MP, MAXT, TPS>(const LaunchInfo&, SolveParams&,         \
                                                                const sgsf_config_t*, const sgsf_timing_t*, \
                                                                cudaStream_t);
#define SGSF_DEFINE_LAUNCH(T, NB, MP, MAXT, TPS)                                                             \
    template int launch_persistent<T, NB, MP, MAXT, TPS>(const LaunchInfo&, SolveParams&, const sgsf_config_t*, \
                                                         const sgsf_timing_t*, cudaStream_t);

// (T, NB, MP, MAXT, TPS): MAXT caps the CTA so ptxas can give the
// register-resident term pass the registers it needs; TPS = threads per time
// step.  Up to 16 robots: TPS = 1 (TPS = 2 measured slower there: the term
// pass is latency-bound and the extra warps cap the registers at 80).  32
// robots: TPS = 2, so a lane still owns 16 robots' positions; one slot of
// ceil(S/16) warps per CTA (the state and the position rows fill the CTA).
#define SGSF_FOR_EACH_VARIANT(X)  \
    X(float, 4, 12, 512, 1)       \
    X(float, 4, 16, 512, 1)       \
    X(float, 8, 12, 384, 1)       \
    X(float, 8, 16, 384, 1)       \
    X(float, 16, 12, 384, 1)      \
    X(float, 16, 16, 384, 1)      \
    X(double, 4, 12, 384, 1)      \
    X(double, 4, 16, 384, 1)      \
    X(double, 8, 12, 256, 1)      \
    X(double, 8, 16, 256, 1)      \
    X(double, 16, 12, 256, 1)     \
    X(double, 16, 16, 256, 1)     \
    X(float, 32, 12, 256, 2)      \
    X(float, 32, 16, 256, 2)      \
    X(double, 32, 12, 256, 2)     \
    X(double, 32, 16, 256, 2)

SGSF_FOR_EACH_VARIANT(SGSF_DECLARE_LAUNCH)

}  // namespace sgsf
