// sf_order.cuh -- longest-first sample order for the persistent kernel's queue.
//
// The persistent kernel hands samples to its slots in queue order.  With a
// few samples per slot and iteration counts spread over ~2x, plain index
// order leaves long samples for the end and the last wave idles most SMs.
// Processing the likely-long samples first (LPT list scheduling) shortens
// that tail.  The predictor is the total constraint violation of the start
// iterate, sum over time steps of max(0, 1 - r) over the pair terms and
// max(0, r - 1) over the workspace terms (r = normalised spheroid radius).
// Its rank correlation with the iteration count is ~0.7 on the benchmark
// scenario.  The order only changes which slot runs a sample and when: every
// sample's result is independent of it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sf_persistent.cuh"

namespace sgsf {

constexpr int kScoreThreads = 128;   // (8 steps per round at 16 robots; 256 measured slower)

// one CTA per sample; FP32 is plenty for a heuristic
template <int NB, int MP>
__global__ void __launch_bounds__(kScoreThreads) start_score_kernel(const SolveParams p, float* __restrict__ score) {
    __shared__ float Cs[3 * NB * MP];
    __shared__ float red[kScoreThreads / 32];
    const int b = blockIdx.x;
    const int n = p.n, m1 = p.m1, S = p.S, R3 = 3 * n;
    const int dim = R3 * m1;
    const bool warm = p.init_mode && p.init_mode[b];
    for (int r = threadIdx.x; r < R3; r += blockDim.x) {
        const double* xr = (warm ? p.xi0 : p.xi_bar) + (size_t)b * dim + r * m1;
        double x[MP];
#pragma unroll
        for (int q = 0; q < MP; ++q) x[q] = q < m1 ? xr[q] : 0.0;
        if (!warm) {   // boundary projection of the proposal (load_row)
            double res[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                double e = 0.0;
#pragma unroll
                for (int q = 0; q < MP; ++q)
                    if (q < m1) e = fma(p.B6[c * m1 + q], x[q], e);
                res[c] = e - p.rhs[r * 6 + c];
            }
#pragma unroll
            for (int q = 0; q < MP; ++q) {
                if (q < m1) {
                    double corr = 0.0;
#pragma unroll
                    for (int c = 0; c < 6; ++c) corr = fma(p.PBt[q * 6 + c], res[c], corr);
                    x[q] -= corr;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < MP; ++q) Cs[r * MP + q] = (float)x[q];
    }
    __syncthreads();
    const float ia2 = (float)(1.0 / (p.lat * p.lat)), ib2 = (float)(1.0 / (p.vert * p.vert));
    const float iw2 = (float)(1.0 / (p.ws_lat * p.ws_lat)), iv2 = (float)(1.0 / (p.ws_vert * p.ws_vert));
    // thread = (step slot, robot): its robot's position into shared memory, then its pairs (i, j > i) and its
    // workspace term (few registers: many CTAs per SM; the thread-per-step form held 48 positions in 255
    // registers and took 65 us per 1000 samples)
    constexpr int SPR = kScoreThreads / NB;   // steps per round
    __shared__ float Pt[SPR][3 * NB];
    const int sl = threadIdx.x / NB, i = threadIdx.x % NB;
    float v = 0.f;
    for (int t0 = 0; t0 < S; t0 += SPR) {
        const int t = t0 + sl;
        if (t < S && i < n) {
            float w[MP];
#pragma unroll
            for (int q = 0; q < MP; ++q) w[q] = q < m1 ? (float)p.W[t * m1 + q] : 0.f;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                float acc = 0.f;
#pragma unroll
                for (int q = 0; q < MP; ++q) acc = fmaf(Cs[(ax * n + i) * MP + q], w[q], acc);
                Pt[sl][ax * NB + i] = acc;
            }
        }
        __syncthreads();
        if (t < S && i < n) {
            const float xi = Pt[sl][i], yi = Pt[sl][NB + i], zi = Pt[sl][2 * NB + i];
            for (int j = i + 1; j < n; ++j) {
                const float dx = xi - Pt[sl][j], dy = yi - Pt[sl][NB + j], dz = zi - Pt[sl][2 * NB + j];
                v += fmaxf(0.f, 1.f - sqrtf((dx * dx + dy * dy) * ia2 + dz * dz * ib2));
            }
            const float rx = xi - (float)p.cx, ry = yi - (float)p.cy, rz = zi - (float)p.cz;
            v += fmaxf(0.f, sqrtf((rx * rx + ry * ry) * iw2 + rz * rz * iv2) - 1.f);
        }
        __syncthreads();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
        score[b] = s;
    }
}

// Bucketed counting sort, descending score, one CTA.  Order inside a bucket
// follows atomic arrival (scheduling only; results do not depend on it).
constexpr int kOrderBuckets = 2048;
constexpr int kOrderThreads = 1024;

__global__ void __launch_bounds__(kOrderThreads) lpt_order_kernel(const float* __restrict__ score, int batch,
                                                                  int* __restrict__ order) {
    __shared__ unsigned int cnt[kOrderBuckets];
    __shared__ float smax;
    for (int k = threadIdx.x; k < kOrderBuckets; k += blockDim.x) cnt[k] = 0u;
    float mx = 0.f;
    for (int b = threadIdx.x; b < batch; b += blockDim.x) mx = fmaxf(mx, score[b]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (threadIdx.x == 0) smax = 0.f;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMax((int*)&smax, __float_as_int(mx));   // non-negative floats
    __syncthreads();
    const float scale = smax > 0.f ? (float)(kOrderBuckets - 1) / smax : 0.f;
    auto bucket = [&](float s) {   // bucket 0 = largest scores
        int k = (int)(fmaxf(s, 0.f) * scale);
        k = k > kOrderBuckets - 1 ? kOrderBuckets - 1 : k;
        return kOrderBuckets - 1 - k;
    };
    for (int b = threadIdx.x; b < batch; b += blockDim.x) atomicAdd(&cnt[bucket(score[b])], 1u);
    __syncthreads();
    {   // exclusive scan of the 2048 counts: two per thread, warp scans, then the warp totals
        static_assert(kOrderBuckets == 2 * kOrderThreads, "two buckets per thread");
        __shared__ unsigned int wsum[kOrderThreads / 32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const unsigned int c0 = cnt[2 * threadIdx.x], c1 = cnt[2 * threadIdx.x + 1];
        unsigned int incl = c0 + c1;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {   // scan of the 32 warp totals
            unsigned int w = wsum[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned int y = __shfl_up_sync(0xffffffffu, w, off);
                if (lane >= off) w += y;
            }
            wsum[lane] = w;   // inclusive
        }
        __syncthreads();
        const unsigned int base = (warp ? wsum[warp - 1] : 0u) + incl - (c0 + c1);
        cnt[2 * threadIdx.x] = base;
        cnt[2 * threadIdx.x + 1] = base + c0;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < batch; b += blockDim.x) order[atomicAdd(&cnt[bucket(score[b])], 1u)] = b;
}

}  // namespace sgsf
