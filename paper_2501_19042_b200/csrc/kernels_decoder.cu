// kernels_decoder.cu -- K4: the generative decoder's forward pass (BASELINE configs 1-3)
// fused into one persistent sm_100a kernel: 4 transposed convolutions (kernel 3, 128 channels, batch norm
// folded into the weights, LeakyReLU / ReLU; dropout is the identity in eval) on the 5th-generation tensor
// cores, then the 1x1 head and the latent->coefficient expansion on the CUDA cores, writing the coefficient
// correction straight into the SF's input layout.
//
// Per CTA, one sample at a time (persistent over the batch, 128 threads = the 128 TMEM lanes):
//   * activations x[c][t] live in shared memory as the MMA's B operand, tf32 hi / lo, K-major with no
//     swizzle: element (row n, channel c) at (c/4) CH + n 16 + (c%4) 4, rows = positions + 1 (row 0 and the
//     rows past L are zero: the convolution's padding).  A kernel-3 convolution is three GEMMs over the SAME
//     operand, one TMEM accumulator per tap, P_k = W_k X; the epilogue adds P_0[t] + P_1[t+1] + P_2[t+2], so
//     no im2col and no shifted view is formed (a descriptor whose start address is not 128-byte aligned
//     corrupts the first 16 rows per 16 bytes of offset: measured with tools/dec_probe.py);
//   * weights stream from global memory (L2-resident, pre-packed on the host in the A operand's layout) in
//     32 KB stages of (tap, 32 input channels, tf32 hi + lo) by cp.async.bulk into two buffers, completion on
//     mbarriers, refilled as soon as the stage's MMAs complete (tcgen05.commit);
//   * P_k[c_out][row] accumulates in TMEM (M = 128, N = L + 2 rounded to 16, three accumulators) over Cin/8
//     K-steps x 3 products (3xTF32: A_hi B_lo + A_lo B_hi + A_hi B_hi, FP32-level accuracy);
//   * the epilogue reads its lane's row with tcgen05.ld, adds the folded bias, applies the activation and
//     writes the next layer's operand (hi / lo split) in place.
// No reference code exists for the networks; the parity target is the PyTorch module in eval mode
// (tests/test_gpu_generative.py: 1e-4).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/sgsf.h"
#include "sf_tc.cuh"

namespace sgsf {
int internal_fail(int code, const std::string& msg);
void internal_count_launch(int n);
}  // namespace sgsf

namespace {

using namespace sgsf;

constexpr int kThreads = 128;
constexpr int kStageBytes = 32768;   // (tap, 32 input channels): 8 K-chunks x 128 rows x 16 B, tf32 hi then lo
constexpr int kHalfStage = kStageBytes / 2;

__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(mbar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tc::smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(tc::smem_u32(mbar))
                 : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T (tf32, both K-major), issued by one thread
__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

struct DecParams {
    int batch, L, c0, c0p, nmma, nrows, nm1, leaky;
    float slope, scale;
    const float* h0;        // B x c0 x L, the first layer's input (latent + state features)
    const uint8_t* wpack;   // all stages of the 4 layers, in order
    const float* bias;      // 4 x 128 (folded)
    const float* head_w;    // 3 x 128
    const float* head_b;    // 3
    const float* exp_w;     // nm1 x L
    const float* exp_b;     // nm1
    double* corr;           // B x 3 nm1
    float* dbg;             // debug (nullable): B x 4 x 128 x L activations after each layer
    int dbg_raw;            // debug: dbg[b][1 + k] = layer 0's raw tap accumulator P_k (columns 0..L-1)
};

__device__ __forceinline__ int layer_cin(const DecParams& p, int l) { return l == 0 ? p.c0p : 128; }
__device__ __forceinline__ int layer_stages(const DecParams& p, int l) { return 3 * (layer_cin(p, l) / 32); }

__global__ void __launch_bounds__(kThreads, 1) decoder_kernel(const DecParams p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int CH = p.nrows * 16;                  // bytes per 4-channel chunk of the activation operand
    unsigned char* act_hi = smem;                 // 32 chunks x nrows x 16 B
    unsigned char* act_lo = smem + 32 * CH;
    unsigned char* wbuf = smem + 64 * CH;         // 2 x 32 KB weight stages
    float* hbuf = (float*)(wbuf + 2 * kStageBytes);   // 3 x L head outputs
    // [0..1] weights landed, [2..3] a stage's MMAs done, [4] a layer's MMAs done.  (The epilogue waits on its own
    // barrier: warps that reach it early would otherwise wait on a stage barrier two phases ahead, which a
    // parity wait cannot tell from the previous phase -- they read TMEM before the MMAs finished.)
    uint64_t* bars = (uint64_t*)(hbuf + 3 * ((p.L + 3) & ~3));
    uint32_t* tslot = (uint32_t*)(bars + 5);

    for (int i = tid; i < 64 * CH / 4; i += kThreads) ((uint32_t*)smem)[i] = 0u;   // padding rows stay zero
    if (tid == 0) {
        for (int i = 0; i < 5; ++i) tc::mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int AS = p.nmma + 32;   // columns per tap accumulator (the epilogue reads 16 past the last row)
    const uint32_t tcols = 3 * AS <= 128 ? 128u : (3 * AS <= 256 ? 256u : 512u);
    if (warp == 0) tc::tmem_alloc(tslot, tcols);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = *tslot;
    const uint32_t idesc = tc::idesc_tf32(128, p.nmma);

    int per_sample = 0;
    for (int l = 0; l < 4; ++l) per_sample += layer_stages(p, l);
    const int my_samples = p.batch > (int)blockIdx.x ? (p.batch - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const long long total = (long long)my_samples * per_sample;
    auto stage_src = [&](long long g) { return p.wpack + (size_t)(g % per_sample) * kStageBytes; };
    if (tid == 32) {   // producer: the first two stages
        for (long long g = 0; g < 2 && g < total; ++g) {
            mbar_expect_tx(&bars[g & 1], kStageBytes);
            bulk_g2s(wbuf + (g & 1) * kStageBytes, stage_src(g), kStageBytes, &bars[g & 1]);
        }
    }

    long long g = 0;   // global stage counter (same sequence in every role)
    uint32_t layers_done = 0;
    for (int s = 0; s < my_samples; ++s) {
        const int b = (int)blockIdx.x + s * (int)gridDim.x;
        // ---- the first layer's input: h0[b] -> rows 1..L, channels 0..c0-1 (c0..c0p-1 zero)
        for (int e = tid; e < p.c0p * p.L; e += kThreads) {
            const int c = e / p.L, t = e - c * p.L;
            const float v = c < p.c0 ? p.h0[((size_t)b * p.c0 + c) * p.L + t] : 0.f;
            const float hi = tc::tf32_rna(v);
            const int off = (c >> 2) * CH + (t + 1) * 16 + (c & 3) * 4;
            *(float*)(act_hi + off) = hi;
            *(float*)(act_lo + off) = tc::tf32_rna(v - hi);
        }
        tc::fence_proxy_async();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();

        for (int l = 0; l < 4; ++l) {
            const int ns = layer_stages(p, l), groups = layer_cin(p, l) / 32;
#ifdef SGSF_DEC_ZERO_ACC
            {   // experiment: zero the three accumulators from the threads, every MMA accumulates
                const uint32_t lrow = tbase + ((uint32_t)(32 * warp) << 16);
                const float z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
                for (int col = 0; col < 3 * AS; col += 16) tc::tmem_st16(lrow + col, z);
                tc::tmem_wait_st();
                tc::fence_before_sync();
                __syncthreads();
                tc::fence_after_sync();
            }
#endif
            for (int st = 0; st < ns; ++st, ++g) {
                const int bi = (int)(g & 1);
                const uint32_t ph = (uint32_t)((g >> 1) & 1);
                if (tid == 0) {   // MMA issuer
                    tc::mbar_wait(&bars[bi], ph);
#ifdef SGSF_DEC_SLEEP
                    __nanosleep(20000);
#endif
                    tc::fence_after_sync();
                    const int tap = st / groups, cg = st - tap * groups;
                    const uint32_t wa = tc::smem_u32(wbuf + bi * kStageBytes);
                    const uint32_t bhi = tc::smem_u32(act_hi) + cg * 8 * CH;
                    const uint32_t blo = tc::smem_u32(act_lo) + cg * 8 * CH;
                    const uint32_t dt = tbase + (uint32_t)(tap * AS);   // this tap's accumulator
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint64_t a_hi = tc::smem_desc(wa + ks * 4096, 2048, 128);
                        const uint64_t a_lo = tc::smem_desc(wa + kHalfStage + ks * 4096, 2048, 128);
                        const uint64_t b_hi = tc::smem_desc(bhi + ks * 2 * CH, CH, 128);
                        const uint64_t b_lo = tc::smem_desc(blo + ks * 2 * CH, CH, 128);
#ifdef SGSF_DEC_ZERO_ACC
                        const uint32_t acc0 = 1u;
#else
                        const uint32_t acc0 = (cg | ks) ? 1u : 0u;   // the tap's first product starts P_tap
#endif
                        mma_tf32_ss(dt, a_hi, b_lo, idesc, acc0);   // small products first
                        mma_tf32_ss(dt, a_lo, b_hi, idesc, 1u);
                        mma_tf32_ss(dt, a_hi, b_hi, idesc, 1u);
                    }
                    tc::mma_commit(&bars[2 + bi]);
                    if (st == ns - 1) tc::mma_commit(&bars[4]);
                }
                if (tid == 32 && g + 2 < total) {   // producer: refill this buffer once its MMAs are done
                    tc::mbar_wait(&bars[2 + bi], ph);
                    mbar_expect_tx(&bars[bi], kStageBytes);
                    bulk_g2s(wbuf + bi * kStageBytes, stage_src(g + 2), kStageBytes, &bars[bi]);
                }
                if (st == ns - 1) {   // ---- epilogue: D -> bias, activation -> the next layer's operand
                    tc::mbar_wait(&bars[4], layers_done & 1u);
                    ++layers_done;
                    tc::fence_after_sync();
                    const int c = tid;   // TMEM lane = output channel
                    const float bias = p.bias[l * 128 + c];
                    const uint32_t lrow = tbase + ((uint32_t)(32 * warp) << 16);
                    for (int t0 = 0; t0 < p.L; t0 += 16) {
                        // out[t] = P_0[t] + P_1[t + 1] + P_2[t + 2] (rows = positions + 1)
                        float v0[16], v1[16], v1n[16], v2[16], v2n[16];
                        tc::tmem_ld16(lrow + t0, v0);
                        tc::tmem_ld16(lrow + AS + t0, v1);
                        tc::tmem_ld16(lrow + AS + t0 + 16, v1n);
                        tc::tmem_ld16(lrow + 2 * AS + t0, v2);
                        tc::tmem_ld16(lrow + 2 * AS + t0 + 16, v2n);
                        tc::tmem_wait_ld();
                        if (p.dbg && p.dbg_raw && l == 0) {
#pragma unroll
                            for (int u = 0; u < 16; ++u)
                                if (t0 + u < p.L) {
                                    p.dbg[(((size_t)b * 4 + 1) * 128 + c) * p.L + t0 + u] = v0[u];
                                    p.dbg[(((size_t)b * 4 + 2) * 128 + c) * p.L + t0 + u] = v1[u];
                                    p.dbg[(((size_t)b * 4 + 3) * 128 + c) * p.L + t0 + u] = v2[u];
                                }
                        }
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int t = t0 + u;
                            if (t < p.L) {
                                const float a1 = u + 1 < 16 ? v1[u + 1] : v1n[u + 1 - 16];
                                const float a2 = u + 2 < 16 ? v2[u + 2] : v2n[u + 2 - 16];
                                float y = ((v0[u] + a1) + a2) + bias;
                                y = y > 0.f ? y : (p.leaky ? p.slope * y : 0.f);
                                const float hi = tc::tf32_rna(y);
                                const int off = (c >> 2) * CH + (t + 1) * 16 + (c & 3) * 4;
                                *(float*)(act_hi + off) = hi;
                                *(float*)(act_lo + off) = tc::tf32_rna(y - hi);
                                if (p.dbg && !(p.dbg_raw && l > 0)) p.dbg[(((size_t)b * 4 + l) * 128 + c) * p.L + t] = y;
                            }
                        }
                    }
                    tc::fence_proxy_async();
                    tc::fence_before_sync();
                    __syncthreads();
                    tc::fence_after_sync();
                }
            }
        }
        // ---- head (1x1, 128 -> 3) over the positions, then the expansion L -> n m1 per axis
        for (int t = tid; t < p.L; t += kThreads) {
            float h[3] = {p.head_b[0], p.head_b[1], p.head_b[2]};
            for (int c = 0; c < 128; ++c) {
                const int off = (c >> 2) * CH + (t + 1) * 16 + (c & 3) * 4;
                const float x = *(const float*)(act_hi + off) + *(const float*)(act_lo + off);
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) h[ax] = fmaf(__ldg(p.head_w + ax * 128 + c), x, h[ax]);
            }
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) hbuf[ax * p.L + t] = h[ax];
        }
        __syncthreads();
        for (int o = tid; o < 3 * p.nm1; o += kThreads) {
            const int ax = o / p.nm1, j = o - ax * p.nm1;
            const float* e = p.exp_w + (size_t)j * p.L;
            float acc = __ldg(p.exp_b + j);
            for (int t = 0; t < p.L; ++t) acc = fmaf(__ldg(e + t), hbuf[ax * p.L + t], acc);
            p.corr[(size_t)b * 3 * p.nm1 + o] = (double)(p.scale * acc);
        }
        __syncthreads();   // hbuf and the activation buffers are rewritten by the next sample
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tbase, tcols);
}

}  // namespace

extern "C" {

size_t sgsf_decoder_pack_bytes(int c0) {
    const int c0p = ((c0 + 31) / 32) * 32;
    return (size_t)3 * (c0p / 32 + 3 * 4) * kStageBytes;
}

int sgsf_decoder_forward_dbg(const sgsf_decoder_t* d, int batch, const float* h0, double* corr, float* dbg,
                             int raw, void* stream);
int sgsf_decoder_forward(const sgsf_decoder_t* d, int batch, const float* h0, double* corr, void* stream) {
    return sgsf_decoder_forward_dbg(d, batch, h0, corr, nullptr, 0, stream);
}
/* (test entry point) as sgsf_decoder_forward, also writing every layer's activations: B x 4 x 128 x L */
int sgsf_decoder_forward_dbg(const sgsf_decoder_t* d, int batch, const float* h0, double* corr, float* dbg,
                             int raw, void* stream) {
    if (!d || (batch > 0 && (!h0 || !corr))) return internal_fail(SGSF_ERR_INVALID, "null argument");
    if (batch == 0) return SGSF_OK;
    if (d->L < 1 || d->L > 150 || d->c0 < 1 || d->c0 > 128 || d->nm1 < 1)
        return internal_fail(SGSF_ERR_UNSUPPORTED, "decoder: latent length 1..150, 1..128 input channels");
    DecParams p;
    std::memset(&p, 0, sizeof(p));
    p.batch = batch;
    p.L = d->L;
    p.c0 = d->c0;
    p.c0p = ((d->c0 + 31) / 32) * 32;
    p.nmma = ((d->L + 2 + 15) / 16) * 16;   // MMA rows: positions -1 .. L (+ padding to 16)
    p.nrows = p.nmma;
    p.nm1 = d->nm1;
    p.leaky = d->leaky;
    p.slope = d->slope;
    p.scale = d->scale;
    p.h0 = h0;
    p.wpack = (const uint8_t*)d->wpack;
    p.bias = d->bias;
    p.head_w = d->head_w;
    p.head_b = d->head_b;
    p.exp_w = d->exp_w;
    p.exp_b = d->exp_b;
    p.corr = corr;
    p.dbg = dbg;
    p.dbg_raw = raw;
    const size_t smem = (size_t)64 * p.nrows * 16 + 2 * kStageBytes + (size_t)3 * ((p.L + 3) & ~3) * 4 + 64 + 16;
    cudaError_t e = cudaFuncSetAttribute(decoder_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, std::string("decoder smem: ") + cudaGetErrorString(e));
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = batch < sms ? batch : sms;
    decoder_kernel<<<grid, kThreads, smem, (cudaStream_t)stream>>>(p);
    internal_count_launch(1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, std::string("decoder launch: ") + cudaGetErrorString(e));
    return SGSF_OK;
}

}  // extern "C"
