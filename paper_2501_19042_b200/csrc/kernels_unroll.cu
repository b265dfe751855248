// kernels_unroll.cu -- unrolled FP64 fixed-point iterations and their reverse sweep (sf_unroll.cuh).
#include <string>

#include "../../include/sgsf.h"
#include "sf_unroll.cuh"

namespace sgsf {
int internal_fail(int code, const std::string& msg);
void internal_count_launch(int n);

namespace {

constexpr int UT = 256;                    // threads per CTA (one CTA per sample)
constexpr double kCosHalfPiD = 6.123233995736766e-17;   // cos(pi/2) in FP64: the zero-vector target's z

struct ULayout {
    double *W, *Km, *Kd, *Mm, *Md, *G;     // constants
    double *C, *A, *Bv, *E, *U, *FT;       // per-sample state, 3 x n x m1 each
    double *mean1, *mean2;                 // 3 x m1 each
    double *posw, *puw, *Rw;               // window rows, 3 x TW x n (<= 3 x 256) each
};

__host__ __device__ inline size_t ulayout(double* base, int n, int S, int m1, ULayout* L) {
    const size_t D = (size_t)3 * n * m1, mm = (size_t)m1 * m1, win = 3 * UT;
    size_t o = 0;
    auto take = [&](double** dst, size_t count) {
        if (L) *dst = base + o;
        o += (count + 1) & ~size_t(1);   // 16-byte alignment
    };
    ULayout dummy;
    ULayout* l = L ? L : &dummy;
    take(&l->W, (size_t)S * m1);
    take(&l->Km, mm);
    take(&l->Kd, mm);
    take(&l->Mm, mm);
    take(&l->Md, mm);
    take(&l->G, mm);
    take(&l->C, D);
    take(&l->A, D);
    take(&l->Bv, D);
    take(&l->E, D);
    take(&l->U, D);
    take(&l->FT, D);
    take(&l->mean1, 3 * (size_t)m1);
    take(&l->mean2, 3 * (size_t)m1);
    take(&l->posw, win);
    take(&l->puw, win);
    take(&l->Rw, win);
    return o;
}

__device__ __forceinline__ void load_constants(const UnrollParams& p, const ULayout& L) {
    const int mm = p.m1 * p.m1;
    for (int e = threadIdx.x; e < p.S * p.m1; e += UT) L.W[e] = p.W[e];
    for (int e = threadIdx.x; e < mm; e += UT) {
        L.Km[e] = p.Km11[e];
        L.Kd[e] = p.Kd11[e];
        L.Mm[e] = p.Mm[e];
        L.Md[e] = p.Md[e];
        L.G[e] = p.G[e];
    }
}

// One pass over all terms of the iterate in L.C, window by window.  Forward (BWD = false): FT =
// F^T (F xi - E), the scatter of the exit residuals (nonzero only for active terms).  Backward:
// FT = F^T (J - I)^T F u for u = L.U.  Thread (i, tl) owns robot i at step t0 + tl and visits every
// partner, so each pair is evaluated by both of its robots with opposite orientation.
template <bool BWD>
__device__ __forceinline__ void term_pass(const UnrollParams& p, const ULayout& L, int TW) {
    const int n = p.n, S = p.S, m1 = p.m1, D = 3 * n * m1;
    const int tid = threadIdx.x, i = tid % n, tl = tid / n;
    const double lat2 = p.lat * p.lat, beta = lat2 / (p.vert * p.vert);
    const double wlat2 = p.ws_lat * p.ws_lat, wbeta = wlat2 / (p.ws_vert * p.ws_vert);
    for (int e = tid; e < D; e += UT) L.FT[e] = 0.0;
    for (int t0 = 0; t0 < S; t0 += TW) {
        const int t = t0 + tl;
        const bool own = tl < TW && t < S;
        if (own) {
            const double* Wr = L.W + t * m1;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                const double* c = L.C + (ax * n + i) * m1;
                double s = 0.0;
                for (int q = 0; q < m1; ++q) s = fma(c[q], Wr[q], s);
                L.posw[(ax * TW + tl) * n + i] = s;
                if (BWD) {
                    const double* u = L.U + (ax * n + i) * m1;
                    double su = 0.0;
                    for (int q = 0; q < m1; ++q) su = fma(u[q], Wr[q], su);
                    L.puw[(ax * TW + tl) * n + i] = su;
                }
            }
        }
        __syncthreads();
        if (own) {
            const double* px = L.posw + (0 * TW + tl) * n;
            const double* py = L.posw + (1 * TW + tl) * n;
            const double* pz = L.posw + (2 * TW + tl) * n;
            const double pix = px[i], piy = py[i], piz = pz[i];
            double fix = 0.0, fiy = 0.0, fiz = 0.0;
            if (BWD) {
                fix = L.puw[(0 * TW + tl) * n + i];
                fiy = L.puw[(1 * TW + tl) * n + i];
                fiz = L.puw[(2 * TW + tl) * n + i];
            }
            double r0 = 0.0, r1 = 0.0, r2 = 0.0;
            for (int j = 0; j < n; ++j) {
                if (j == i) continue;
                const double dx = pix - px[j], dy = piy - py[j], dz = piz - pz[j];
                const double q = fma(dz * beta, dz, fma(dy, dy, dx * dx));
                if (!(q < lat2)) continue;   // interior pair: target = d, no residual, J = I
                if (!BWD) {
                    if (q == 0.0) {   // zero vector: target (lat, 0, vert cos(pi/2)) of the (min, max) orientation
                        const double sg = i < j ? 1.0 : -1.0;
                        r0 -= sg * p.lat;
                        r2 -= sg * p.vert * kCosHalfPiD;
                    } else {
                        const double s = p.lat / sqrt(q);
                        r0 += fma(-s, dx, dx);
                        r1 += fma(-s, dy, dy);
                        r2 += fma(-s, dz, dz);
                    }
                } else {
                    const double fx = fix - L.puw[(0 * TW + tl) * n + j];
                    const double fy = fiy - L.puw[(1 * TW + tl) * n + j];
                    const double fz = fiz - L.puw[(2 * TW + tl) * n + j];
                    if (q == 0.0) {   // locally constant target: J = 0
                        r0 -= fx;
                        r1 -= fy;
                        r2 -= fz;
                    } else {
                        const double s = p.lat / sqrt(q);
                        const double c = fma(dz, fz, fma(dy, fy, dx * fx)) / q;
                        r0 += fma(s, fma(-dx, c, fx), -fx);
                        r1 += fma(s, fma(-dy, c, fy), -fy);
                        r2 += fma(s, fma(-dz * beta, c, fz), -fz);
                    }
                }
            }
            {   // workspace term of robot i (target relative to the centre; interior when r <= 1)
                const double rx = pix - p.cx, ry = piy - p.cy, rz = piz - p.cz;
                const double q = fma(rz * wbeta, rz, fma(ry, ry, rx * rx));
                if (q > wlat2) {
                    const double s = p.ws_lat / sqrt(q);
                    if (!BWD) {
                        r0 += fma(-s, rx, rx);
                        r1 += fma(-s, ry, ry);
                        r2 += fma(-s, rz, rz);
                    } else {
                        const double c = fma(rz, fiz, fma(ry, fiy, rx * fix)) / q;
                        r0 += fma(s, fma(-rx, c, fix), -fix);
                        r1 += fma(s, fma(-ry, c, fiy), -fiy);
                        r2 += fma(s, fma(-rz * wbeta, c, fiz), -fiz);
                    }
                }
            }
            L.Rw[(0 * TW + tl) * n + i] = r0;
            L.Rw[(1 * TW + tl) * n + i] = r1;
            L.Rw[(2 * TW + tl) * n + i] = r2;
        }
        __syncthreads();
        const int tw = min(TW, S - t0);
        for (int e = tid; e < D; e += UT) {   // W^T projection of the window, owner thread per coefficient
            const int k = e % m1, row = e / m1, ax = row / n, ri = row % n;
            double acc = L.FT[e];
            for (int u = 0; u < tw; ++u) acc = fma(L.Rw[(ax * TW + u) * n + ri], L.W[(t0 + u) * m1 + k], acc);
            L.FT[e] = acc;
        }
    }
    __syncthreads();
}

// per-axis robot means (scale 1/n) or sums (scale 1) of X into out[3][m1], fixed order
__device__ __forceinline__ void robot_reduce(const double* X, double* out, int n, int m1, double scale) {
    for (int c = threadIdx.x; c < 3 * m1; c += UT) {
        const int ax = c / m1, q = c % m1;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += X[(ax * n + i) * m1 + q];
        out[c] = s * scale;
    }
}

__global__ void __launch_bounds__(UT) unroll_forward_kernel(const UnrollParams p) {
    extern __shared__ __align__(16) double sm[];
    ULayout L;
    ulayout(sm, p.n, p.S, p.m1, &L);
    const int n = p.n, m1 = p.m1, D = 3 * n * m1, TW = max(1, UT / n);
    const size_t b = blockIdx.x;
    load_constants(p, L);
    const double* xb = p.xi_bar + b * D;
    double* xs = p.xs + b * (size_t)(p.iters + 1) * D;
    double* ls = p.ls + b * (size_t)(p.iters + 1) * D;
    for (int e = threadIdx.x; e < D; e += UT) {
        L.C[e] = p.xi0[b * D + e];
        L.A[e] = p.lam0[b * D + e];
        L.Bv[e] = xb[e];
        xs[e] = L.C[e];
        ls[e] = L.A[e];
    }
    __syncthreads();
    const double inv_n = 1.0 / n;
    for (int it = 0; it < p.iters; ++it) {
        term_pass<false>(p, L, TW);
        for (int e = threadIdx.x; e < D; e += UT) {   // lambda' = lambda - rho F^T r; u = 2 lambda' - lambda + xi_bar
            const double lam = L.A[e], lamn = fma(-p.rho, L.FT[e], lam);
            L.U[e] = 2.0 * lamn - lam + L.Bv[e];
            L.A[e] = lamn;
        }
        __syncthreads();
        robot_reduce(L.C, L.mean1, n, m1, inv_n);
        robot_reduce(L.U, L.mean2, n, m1, inv_n);
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {   // xi' = Mm Cbar + Km11 ubar + Md (C - Cbar) + Kd11 (u - ubar) + cconst
            const int k = e % m1, row = e / m1, ax = row / n;
            const double* c = L.C + row * m1;
            const double* u = L.U + row * m1;
            const double* cb = L.mean1 + ax * m1;
            const double* ub = L.mean2 + ax * m1;
            double s = p.cconst[e];
            for (int q = 0; q < m1; ++q) {
                s = fma(L.Mm[k * m1 + q], cb[q], s);
                s = fma(L.Km[k * m1 + q], ub[q], s);
                s = fma(L.Md[k * m1 + q], c[q] - cb[q], s);
                s = fma(L.Kd[k * m1 + q], u[q] - ub[q], s);
            }
            L.E[e] = s;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {
            L.C[e] = L.E[e];
            xs[(size_t)(it + 1) * D + e] = L.E[e];
            ls[(size_t)(it + 1) * D + e] = L.A[e];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(UT) unroll_backward_kernel(const UnrollParams p) {
    extern __shared__ __align__(16) double sm[];
    ULayout L;
    ulayout(sm, p.n, p.S, p.m1, &L);
    const int n = p.n, m1 = p.m1, D = 3 * n * m1, TW = max(1, UT / n);
    const size_t b = blockIdx.x;
    load_constants(p, L);
    const double* xs = p.xs + b * (size_t)(p.iters + 1) * D;
    const double* gxs = p.gxs ? p.gxs + b * (size_t)(p.iters + 1) * D : nullptr;
    const double* gls = p.gls ? p.gls + b * (size_t)(p.iters + 1) * D : nullptr;
    double* gxb = p.g_xi_bar + b * D;
    for (int e = threadIdx.x; e < D; e += UT) {
        L.A[e] = 0.0;    // adjoint of xi_{k+1}
        L.Bv[e] = 0.0;   // adjoint of lambda_{k+1}
        gxb[e] = 0.0;
    }
    const double inv_n = 1.0 / n;
    for (int it = p.iters - 1; it >= 0; --it) {
        for (int e = threadIdx.x; e < D; e += UT) {
            if (gxs) L.A[e] += gxs[(size_t)(it + 1) * D + e];
            if (gls) L.Bv[e] += gls[(size_t)(it + 1) * D + e];
            L.C[e] = xs[(size_t)it * D + e];
        }
        __syncthreads();
        robot_reduce(L.A, L.mean1, n, m1, inv_n);
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {   // eh = Km11^T xbar_h + Kd11^T (xh - xbar_h)
            const int k = e % m1, row = e / m1, ax = row / n;
            const double* x = L.A + row * m1;
            const double* xbm = L.mean1 + ax * m1;
            double s = 0.0;
            for (int q = 0; q < m1; ++q) {
                s = fma(L.Km[q * m1 + k], xbm[q], s);
                s = fma(L.Kd[q * m1 + k], x[q] - xbm[q], s);
            }
            L.E[e] = s;
            gxb[e] += s;
            const double lt = L.Bv[e] + s;
            L.Bv[e] = lt;
            L.U[e] = lt + s;
        }
        __syncthreads();
        term_pass<true>(p, L, TW);
        robot_reduce(L.E, L.mean2, n, m1, 1.0);
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {   // xh = rho ((n+1) eh_i - sum_j eh_j) G + rho F^T (J - I)^T F u
            const int k = e % m1, row = e / m1, ax = row / n;
            const double* eh = L.E + row * m1;
            const double* es = L.mean2 + ax * m1;
            double s = 0.0;
            for (int q = 0; q < m1; ++q) s = fma(fma((double)(n + 1), eh[q], -es[q]), L.G[q * m1 + k], s);
            L.A[e] = p.rho * (s + L.FT[e]);
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < D; e += UT) {
        p.g_xi0[b * D + e] = L.A[e] + (gxs ? gxs[e] : 0.0);
        p.g_lam0[b * D + e] = L.Bv[e] + (gls ? gls[e] : 0.0);
    }
}

int launch(const void* fn, const UnrollParams& p, cudaStream_t stream, const char* what) {
    if (p.batch == 0) return SGSF_OK;
    const size_t smem = unroll_smem_bytes(p.n, p.S, p.m1);
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem > (size_t)optin)
        return internal_fail(SGSF_ERR_UNSUPPORTED, std::string(what) + ": needs " + std::to_string(smem) +
                                                       " bytes of shared memory per CTA, the device has " +
                                                       std::to_string(optin));
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    void* args[] = {(void*)&p};
    e = cudaLaunchKernel(fn, dim3(p.batch), dim3(UT), args, smem, stream);
    if (e != cudaSuccess) return internal_fail(SGSF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    internal_count_launch(1);
    return SGSF_OK;
}

}  // namespace

size_t unroll_smem_bytes(int n, int S, int m1) { return ulayout(nullptr, n, S, m1, nullptr) * sizeof(double); }

int launch_unroll_forward(const UnrollParams& p, cudaStream_t stream) {
    return launch((const void*)unroll_forward_kernel, p, stream, "sgsf_unroll");
}

int launch_unroll_backward(const UnrollParams& p, cudaStream_t stream) {
    return launch((const void*)unroll_backward_kernel, p, stream, "sgsf_unroll_backward");
}

}  // namespace sgsf
