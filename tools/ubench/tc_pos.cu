// tc_pos.cu -- check of the 3xTF32 tcgen05 position GEMM used by K1 (descriptor encodings, TMEM
// lane mapping, accuracy against FP64 and plain FP32 FMA).  One CTA of 4 warps:
//   D[128 x 48] = A[128 x 16] (W rows of the permuted steps, tf32 hi / lo in TMEM) x B^T (C hi / lo, smem)
// with the step of TMEM lane 32 w + l = 8 (w + 4 (l >> 3)) + (l & 7), K1's chunk mapping for 4 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench/tc_pos tools/ubench/tc_pos.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2501_19042_b200/csrc/sf_tc.cuh"

using namespace sgsf::tc;

constexpr int S = 101, MP = 12, NB = 16;

// TRUNC: hi = the raw FP32 value (the tensor core reads its top 19 bits), lo = x - (x & ~0x1fff)
template <bool TRUNC>
__device__ __forceinline__ void split(float x, float& hi, float& lo) {
    if (TRUNC) {
        hi = x;
        lo = x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
    } else {
        hi = tf32_rna(x);
        lo = tf32_rna(x - hi);
    }
}

template <int NPROD, int NAX, bool TRUNC = false>
__global__ void tc_pos_kernel(const float* W, const float* C, float* out, long long* cycles) {
    __shared__ __align__(1024) unsigned char bop[3][2][1024];   // [axis][hi, lo] K-major 16 x 16 tf32
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tmem_alloc(&tbase, 128);
    if (tid == 0) mbar_init(&mbar, 1);
    // B operand: C[ax][q][i] (robot-minor) -> row i, column q
    for (int e = tid; e < 3 * 16 * 16; e += blockDim.x) {
        const int ax = e / 256, i = (e / 16) % 16, k = e % 16;
        const float c = k < MP ? C[(ax * MP + k) * NB + i] : 0.f;
        float hi, lo;
        split<TRUNC>(c, hi, lo);
        *reinterpret_cast<float*>(&bop[ax][0][kmajor16_offset(i, k)]) = hi;
        *reinterpret_cast<float*>(&bop[ax][1][kmajor16_offset(i, k)]) = lo;
    }
    fence_proxy_async();
    __syncthreads();
    const uint32_t base = tbase;
    const int ts = 8 * (warp + 4 * (lane >> 3)) + (lane & 7);
    {   // A operand rows: W of this lane's step, hi at columns 0..15, lo at 16..31
        float hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const float w = (ts < S && k < MP) ? W[ts * MP + k] : 0.f;
            split<TRUNC>(w, hi[k], lo[k]);
        }
        const uint32_t lane_addr = base + ((uint32_t)(32 * warp) << 16);
        tmem_st16(lane_addr + 0, hi);
        tmem_st16(lane_addr + 16, lo);
        tmem_wait_st();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    long long t0 = clock64();
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(128, 16);
        for (int ax = 0; ax < NAX; ++ax) {
            const uint32_t d = base + 32 + 16 * ax;
            int first = 1;
            const int pa[4] = {16, 0, 16, 0};   // A column: lo, hi, lo, hi (small products first)
            const int pb[4] = {1, 1, 0, 0};     // B: lo, lo, hi, hi
            for (int prod = 4 - NPROD; prod < 4; ++prod)
                for (int ks = 0; ks < 2; ++ks) {
                    const uint64_t bd = smem_desc(smem_u32(&bop[ax][pb[prod]][0]) + 256 * ks, 128, 512);
                    mma_tf32_ts(d, base + pa[prod] + 8 * ks, bd, idesc, first ? 0u : 1u);
                    first = 0;
                }
        }
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    fence_after_sync();
    float v[48];
    const uint32_t lane_addr = base + ((uint32_t)(32 * warp) << 16);
    tmem_ld16(lane_addr + 32, *reinterpret_cast<float(*)[16]>(&v[0]));
    tmem_ld16(lane_addr + 48, *reinterpret_cast<float(*)[16]>(&v[16]));
    tmem_ld16(lane_addr + 64, *reinterpret_cast<float(*)[16]>(&v[32]));
    tmem_wait_ld();
    long long t1 = clock64();
    if (ts < S)
        for (int c = 0; c < 48; ++c) out[ts * 48 + c] = v[c];
    if (tid == 0) *cycles = t1 - t0;
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(base, 128);
}

int main(int argc, char** argv) {
    std::mt19937 g(1);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    std::vector<float> W(S * MP), C(3 * MP * NB), out(S * 48, 0.f);
    for (auto& x : W) x = u(g);
    for (auto& x : C) x = 5.f * u(g);
    float *dW, *dC, *dO;
    long long* dcy;
    cudaMalloc(&dW, W.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMalloc(&dO, out.size() * 4);
    cudaMalloc(&dcy, 8);
    cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C.data(), C.size() * 4, cudaMemcpyHostToDevice);
    long long cy1;
    tc_pos_kernel<3, 1><<<1, 128>>>(dW, dC, dO, dcy);
    cudaDeviceSynchronize();
    cudaMemcpy(&cy1, dcy, 8, cudaMemcpyDeviceToHost);
    printf("one axis, 3 products: %lld cycles\n", cy1);
    tc_pos_kernel<4, 1><<<1, 128>>>(dW, dC, dO, dcy);
    cudaDeviceSynchronize();
    cudaMemcpy(&cy1, dcy, 8, cudaMemcpyDeviceToHost);
    printf("one axis, 4 products: %lld cycles\n", cy1);
    const int nprod = argc > 1 ? atoi(argv[1]) : 3;
    if (nprod == 5) tc_pos_kernel<3, 3, true><<<1, 128>>>(dW, dC, dO, dcy);   // 3 products, truncation split
    else if (nprod == 4) tc_pos_kernel<4, 3><<<1, 128>>>(dW, dC, dO, dcy);
    else tc_pos_kernel<3, 3><<<1, 128>>>(dW, dC, dO, dcy);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    long long cy;
    cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cy, dcy, 8, cudaMemcpyDeviceToHost);
    double err_tc = 0, err_fma = 0, scale = 0;
    for (int t = 0; t < S; ++t)
        for (int ax = 0; ax < 3; ++ax)
            for (int i = 0; i < NB; ++i) {
                double ref = 0, absum = 0;
                float f = 0.f;
                for (int q = 0; q < MP; ++q) {
                    ref += (double)C[(ax * MP + q) * NB + i] * (double)W[t * MP + q];
                    absum += std::fabs((double)C[(ax * MP + q) * NB + i] * (double)W[t * MP + q]);
                    f = std::fmaf(C[(ax * MP + q) * NB + i], W[t * MP + q], f);
                }
                err_tc = std::fmax(err_tc, std::fabs(out[t * 48 + ax * 16 + i] - ref) / absum);
                err_fma = std::fmax(err_fma, std::fabs(f - ref) / absum);
                scale = std::fmax(scale, std::fabs(ref));
            }
    printf("%dxTF32 tcgen05:", nprod); printf(" max |err| / sum|terms| = %.3g   (FP32 FMA chain: %.3g)   MMA+commit+ld: %lld cycles\n",
           err_tc, err_fma, cy);
    printf("%s\n", err_tc < 4 * err_fma + 1e-6 ? "PASS" : "FAIL");
    return err_tc < 4 * err_fma + 1e-6 ? 0 : 2;
}
