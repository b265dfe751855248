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
constexpr int kBuf = 3;              // weight stage buffers (prefetch depth)

// (hi, lo) operand split: hi = x with the low 13 mantissa bits cleared (a tf32 value), lo = x - hi exactly (the
// tensor core reads lo's top 11 significant bits: the pair carries x to ~2^-21 relative)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
    hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    lo = x - hi;
}

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
    int batch, L, c0, c0p, nmma, nrows, nm1, leaky, cz, n, m1;
    float slope, scale;
    const float* h0;        // B x cz x L: the per-sample channels of the first layer's input (the latent)
    const float* feat;      // c0 - cz channels constant along L and over the batch (state features), nullable
    const double* base;     // 3 nm1: straight-line coefficients (nullable: output the correction alone)
    const double* B6;       // 6 x m1 endpoint rows
    const double* PBt;      // m1 x 6 boundary projector
    const double* rhs;      // 3 n x 6 endpoint values
    const uint8_t* wpack;   // all stages of the 4 layers, in order
    const float* bias;      // 4 x 128 (folded)
    const float* head_w;    // 3 x 128
    const float* head_b;    // 3
    const float* exp_w;     // L x nm1 (the Linear's weight, transposed)
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
    unsigned char* wbuf = smem + 64 * CH;         // kBuf x 32 KB weight stages
    float* hbuf = (float*)(wbuf + kBuf * kStageBytes);   // 3 x L head outputs
    float* hw_s = hbuf + 3 * ((p.L + 3) & ~3);              // 3 x 128 head weights
    // [0, kBuf) weights landed, [kBuf, 2 kBuf) a stage's MMAs done, [2 kBuf] a layer's MMAs done.  (The epilogue waits on its own
    // barrier: warps that reach it early would otherwise wait on a stage barrier two phases ahead, which a
    // parity wait cannot tell from the previous phase -- they read TMEM before the MMAs finished.)
    uint64_t* bars = (uint64_t*)(hw_s + 3 * 128);
    uint32_t* tslot = (uint32_t*)(bars + 2 * kBuf + 1);
    uint64_t* const wready = bars;
    uint64_t* const mdone = bars + kBuf;
    uint64_t* const ldone = bars + 2 * kBuf;

    for (int i = tid; i < 64 * CH / 4; i += kThreads) ((uint32_t*)smem)[i] = 0u;   // padding rows stay zero
    for (int i = tid; i < 3 * 128; i += kThreads) hw_s[i] = p.head_w[i];
    if (tid == 0) {
        for (int i = 0; i < 2 * kBuf + 1; ++i) tc::mbar_init(&bars[i], 1);
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
    const int total = my_samples * per_sample;
    auto stage_src = [&](int g) { return p.wpack + (size_t)(g % per_sample) * kStageBytes; };
    if (tid == 32) {   // producer: the first kBuf stages
        for (int g = 0; g < kBuf && g < total; ++g) {
            mbar_expect_tx(&wready[g], kStageBytes);
            bulk_g2s(wbuf + g * kStageBytes, stage_src(g), kStageBytes, &wready[g]);
        }
    }

    int g = 0;   // global stage counter (same sequence in every role)
    uint32_t layers_done = 0;
    for (int s = 0; s < my_samples; ++s) {
        const int b = (int)blockIdx.x + s * (int)gridDim.x;
        // ---- the first layer's input: h0[b] -> rows 1..L, channels 0..c0-1 (c0..c0p-1 zero).  One (4-channel
        // chunk, position) per item: four loads coalesced over the positions, one 16-byte store each of hi / lo
        // (consecutive lanes, consecutive rows: conflict-free)
        {
            const float* src = p.h0 + (size_t)b * p.cz * p.L;
            const int items = (p.c0p >> 2) * p.L;
            for (int it = tid; it < items; it += kThreads) {
                const int g = it / p.L, t = it - g * p.L;
                float v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int c = 4 * g + k;
                    v[k] = c < p.cz ? __ldg(src + c * p.L + t) : (c < p.c0 ? __ldg(p.feat + (c - p.cz)) : 0.f);
                }
                float4 hi, lo;
                split_tf32(v[0], hi.x, lo.x);
                split_tf32(v[1], hi.y, lo.y);
                split_tf32(v[2], hi.z, lo.z);
                split_tf32(v[3], hi.w, lo.w);
                const int off = g * CH + (t + 1) * 16;
                *(float4*)(act_hi + off) = hi;
                *(float4*)(act_lo + off) = lo;
            }
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
                const int bi = (int)(g % kBuf);
                const uint32_t ph = (uint32_t)((g / kBuf) & 1);
                if (tid == 0) {   // MMA issuer
                    tc::mbar_wait(&wready[bi], ph);
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
                    tc::mma_commit(&mdone[bi]);
                    if (st == ns - 1) tc::mma_commit(ldone);
                }
                if (tid == 32 && g + kBuf < total) {   // producer: refill this buffer once its MMAs are done
                    tc::mbar_wait(&mdone[bi], ph);
                    mbar_expect_tx(&wready[bi], kStageBytes);
                    bulk_g2s(wbuf + bi * kStageBytes, stage_src(g + kBuf), kStageBytes, &wready[bi]);
                }
                if (st == ns - 1) {   // ---- epilogue: D -> bias, activation -> the next layer's operand
                    tc::mbar_wait(ldone, layers_done & 1u);
                    ++layers_done;
                    tc::fence_after_sync();
                    const int c = tid, lane = tid & 31;   // TMEM lane = output channel
                    const float bias = p.bias[l * 128 + c];
                    const float slope = p.leaky ? p.slope : 0.f;
                    const uint32_t lrow = tbase + ((uint32_t)(32 * warp) << 16);
                    float v1[16], v2[16];   // P_1, P_2 at columns t0 .. t0 + 15 (carried over from the last chunk)
                    tc::tmem_ld16(lrow + AS, v1);
                    tc::tmem_ld16(lrow + 2 * AS, v2);
                    for (int t0 = 0; t0 < p.L; t0 += 16) {
                        // out[t] = P_0[t] + P_1[t + 1] + P_2[t + 2] (rows = positions + 1)
                        float v0[16], v1n[16], v2n[16];
                        tc::tmem_ld16(lrow + t0, v0);
                        tc::tmem_ld16(lrow + AS + t0 + 16, v1n);
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
                        uint32_t yh[16], yl[16];   // positions past L are zero (the next layer's padding rows)
                        const int valid = p.L - t0;
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const float a1 = u + 1 < 16 ? v1[u + 1] : v1n[u + 1 - 16];
                            const float a2 = u + 2 < 16 ? v2[u + 2] : v2n[u + 2 - 16];
                            float y = ((v0[u] + a1) + a2) + bias;
                            y = y > 0.f ? y : slope * y;
                            y = u < valid ? y : 0.f;
                            float hi, lo;
                            split_tf32(y, hi, lo);
                            yh[u] = __float_as_uint(hi);
                            yl[u] = __float_as_uint(lo);
                        }
                        if (p.dbg && !(p.dbg_raw && l > 0)) {
#pragma unroll
                            for (int u = 0; u < 16; ++u)
                                if (u < valid)
                                    p.dbg[(((size_t)b * 4 + l) * 128 + c) * p.L + t0 + u] =
                                        __uint_as_float(yh[u]) + __uint_as_float(yl[u]);
                        }
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            v1[u] = v1n[u];
                            v2[u] = v2n[u];
                        }
                        // stmatrix.x4: matrix m = position t0 + 4 q + m, its row r = chunk 8 warp + r (16 bytes:
                        // channels of lanes 4 r .. 4 r + 3).  Lane i addresses row i % 8 of matrix i / 8.
                        const int mrow = lane & 7, mmat = lane >> 3;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int t = t0 + 4 * q + mmat;
                            const int row = t < p.L ? t + 1 : p.nrows - 1;   // (a zero padding row)
                            const uint32_t off = (uint32_t)((8 * warp + mrow) * CH + row * 16);
                            tc::stmatrix_x4(tc::smem_u32(act_hi + off), yh[4 * q], yh[4 * q + 1], yh[4 * q + 2],
                                            yh[4 * q + 3]);
                            tc::stmatrix_x4(tc::smem_u32(act_lo + off), yl[4 * q], yl[4 * q + 1], yl[4 * q + 2],
                                            yl[4 * q + 3]);
                        }
                    }
                    tc::fence_proxy_async();
                    tc::fence_before_sync();
                    __syncthreads();
                    tc::fence_after_sync();
                }
            }
        }
        // ---- head (1x1, 128 -> 3) over the positions -> h (3 x L floats), parked in the sample's output row
        // (3 n m1 doubles, read back by decoder_tail_kernel before it writes the row)
        float* hout = (float*)(p.corr + (size_t)b * 3 * p.nm1);
        for (int t = tid; t < p.L; t += kThreads) {   // 16-byte reads: consecutive lanes, consecutive rows
            float h[3] = {p.head_b[0], p.head_b[1], p.head_b[2]};
            for (int g4 = 0; g4 < 32; ++g4) {
                const float4 xh = *(const float4*)(act_hi + g4 * CH + (t + 1) * 16);
                const float4 xl = *(const float4*)(act_lo + g4 * CH + (t + 1) * 16);
                const float x[4] = {xh.x + xl.x, xh.y + xl.y, xh.z + xl.z, xh.w + xl.w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int ax = 0; ax < 3; ++ax) h[ax] = fmaf(hw_s[ax * 128 + 4 * g4 + k], x[k], h[ax]);
            }
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) hout[ax * p.L + t] = h[ax];
        }
        __syncthreads();   // the activation buffers are rewritten by the next sample
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tbase, tcols);
}


// ---- the expansion L -> n m1 per axis (+ the boundary QP layer) for S samples per CTA, so that each exp_w element
// is read once per S samples: reads h (3 x L floats) from the front of each sample's output row, writes the row.
template <int S>
__global__ void __launch_bounds__(256) decoder_tail_kernel(const DecParams p) {
    extern __shared__ __align__(16) unsigned char tsm[];
    const int L = p.L, nm1 = p.nm1, tid = threadIdx.x;
    float* hs = (float*)tsm;                                                   // S x 3 x L
    double* xs = (double*)(tsm + (((size_t)S * 3 * L * 4 + 15) & ~(size_t)15));   // S x 3 nm1
    double* res = xs + (size_t)S * 3 * nm1;                                    // S x 3 n x 6
    const int b0 = blockIdx.x * S, ns = min(S, p.batch - b0);
    for (int i = tid; i < S * 3 * L; i += blockDim.x) {
        const int s = i / (3 * L), k = i - s * 3 * L;
        hs[i] = s < ns ? ((const float*)(p.corr + (size_t)(b0 + s) * 3 * nm1))[k] : 0.f;
    }
    __syncthreads();
    for (int j = tid; j < nm1; j += blockDim.x) {   // exp_w is L x nm1 (transposed): coalesced rows
        const float eb = __ldg(p.exp_b + j);
        float a[S][3];
#pragma unroll
        for (int s = 0; s < S; ++s) a[s][0] = a[s][1] = a[s][2] = eb;
#pragma unroll 10
        for (int t = 0; t < L; ++t) {
            const float e = __ldg(p.exp_w + (size_t)t * nm1 + j);
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) a[s][ax] = fmaf(e, hs[(s * 3 + ax) * L + t], a[s][ax]);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s >= ns) break;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                const double v = (double)(p.scale * a[s][ax]);
                if (p.base)   // xi' = straight line + correction, for the QP layer below
                    xs[((size_t)s * 3 + ax) * nm1 + j] = p.base[(size_t)ax * nm1 + j] + v;
                else
                    p.corr[(size_t)(b0 + s) * 3 * nm1 + (size_t)ax * nm1 + j] = v;
            }
        }
    }
    if (!p.base) return;
    // the boundary QP layer (projection.py:11-25): C - PBt (B6 C - rhs), per robot and axis
    __syncthreads();
    const int R6 = 3 * p.n * 6;
    for (int i = tid; i < ns * R6; i += blockDim.x) {
        const int s = i / R6, e = i - s * R6, r = e / 6, k = e - 6 * r;
        const double* cr = xs + (size_t)s * 3 * nm1 + r * p.m1;
        double acc = 0.0;
        for (int q = 0; q < p.m1; ++q) acc = fma(__ldg(p.B6 + k * p.m1 + q), cr[q], acc);
        res[i] = acc - __ldg(p.rhs + e);
    }
    __syncthreads();
    for (int i = tid; i < ns * 3 * nm1; i += blockDim.x) {   // (sample, r, q): coalesced output rows
        const int s = i / (3 * nm1), e = i - s * 3 * nm1, r = e / p.m1, q = e - r * p.m1;
        double corr = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k) corr = fma(__ldg(p.PBt + q * 6 + k), res[s * R6 + r * 6 + k], corr);
        p.corr[(size_t)(b0 + s) * 3 * nm1 + e] = xs[i] - corr;
    }
}

template <int S>
size_t tail_smem(const DecParams& p) {
    return (((size_t)S * 3 * p.L * 4 + 15) & ~(size_t)15) + (size_t)S * 3 * p.nm1 * 8 +
           (p.base ? (size_t)S * 3 * p.n * 6 * 8 : 0);
}

template <int S>
cudaError_t launch_tail(const DecParams& p, cudaStream_t stream) {
    const size_t smem = tail_smem<S>(p);
    cudaError_t e = cudaFuncSetAttribute(decoder_tail_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    decoder_tail_kernel<S><<<(p.batch + S - 1) / S, 256, smem, stream>>>(p);
    return cudaGetLastError();
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
    p.cz = d->feat ? d->cz : d->c0;
    p.feat = d->feat;
    p.base = d->base;
    p.B6 = d->B6;
    p.PBt = d->PBt;
    p.rhs = d->rhs;
    p.n = d->n;
    p.m1 = d->m1;
    if (d->L > 2 * d->nm1)
        return internal_fail(SGSF_ERR_UNSUPPORTED, "decoder: 3 L floats must fit in a sample's 3 n m1 doubles");
    if (p.base && (!p.B6 || !p.PBt || !p.rhs || p.n * p.m1 != p.nm1))
        return internal_fail(SGSF_ERR_INVALID, "decoder QP layer: B6, PBt, rhs and n m1 = nm1 required");
    p.wpack = (const uint8_t*)d->wpack;
    p.bias = d->bias;
    p.head_w = d->head_w;
    p.head_b = d->head_b;
    p.exp_w = d->exp_w;
    p.exp_b = d->exp_b;
    p.corr = corr;
    p.dbg = dbg;
    p.dbg_raw = raw;
    const size_t smem = (size_t)64 * p.nrows * 16 + kBuf * kStageBytes + (size_t)3 * ((p.L + 3) & ~3) * 4 +
                        3 * 128 * 4 + 128;
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
    // the expansion (+ QP) kernel: up to 8 samples per CTA (each exp_w element read once per CTA), at least
    // about one CTA per SM, within 200 KB of shared memory
    if (tail_smem<8>(p) <= 200 * 1024 && batch >= 8 * sms)
        e = launch_tail<8>(p, (cudaStream_t)stream);
    else if (tail_smem<4>(p) <= 200 * 1024 && batch >= 4 * sms / 2)
        e = launch_tail<4>(p, (cudaStream_t)stream);
    else if (tail_smem<2>(p) <= 200 * 1024)
        e = launch_tail<2>(p, (cudaStream_t)stream);
    else
        e = launch_tail<1>(p, (cudaStream_t)stream);
    internal_count_launch(1);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, std::string("decoder tail launch: ") + cudaGetErrorString(e));
    return SGSF_OK;
}

}  // extern "C"
