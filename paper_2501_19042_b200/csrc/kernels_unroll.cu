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
    double *C, *A, *Bv, *E, *U, *FT;       // per-sample state, 3 x n x MP each
    double *mean1, *mean2;                 // 3 x MP each
    double *posw, *puw, *Rw;               // window rows, 3 x TW x n (<= 3 x 256) each
};

// shared arrays use MP (m1 rounded up to 12 or 16) columns, zero-padded: the coefficient loops have
// compile-time trip counts and 16-byte loads, and the padding stays zero through every step
__host__ __device__ inline size_t ulayout(double* base, int n, int S, int MP, ULayout* L) {
    const size_t D = (size_t)3 * n * MP, mm = (size_t)MP * MP, win = 3 * UT;
    size_t o = 0;
    auto take = [&](double** dst, size_t count) {
        if (L) *dst = base + o;
        o += (count + 1) & ~size_t(1);   // 16-byte alignment
    };
    ULayout dummy;
    ULayout* l = L ? L : &dummy;
    take(&l->W, (size_t)S * MP);
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
    take(&l->mean1, 3 * (size_t)MP);
    take(&l->mean2, 3 * (size_t)MP);
    take(&l->posw, win);
    take(&l->puw, win);
    take(&l->Rw, win);
    return o;
}

template <int MP>
__device__ __forceinline__ void load_constants(const UnrollParams& p, const ULayout& L) {
    const int m1 = p.m1;
    for (int e = threadIdx.x; e < p.S * MP; e += UT) {
        const int t = e / MP, q = e % MP;
        L.W[e] = q < m1 ? p.W[t * m1 + q] : 0.0;
    }
    for (int e = threadIdx.x; e < MP * MP; e += UT) {
        const int a = e / MP, b = e % MP;
        const bool in = a < m1 && b < m1;
        const int g = a * m1 + b;
        L.Km[e] = in ? p.Km11[g] : 0.0;
        L.Kd[e] = in ? p.Kd11[g] : 0.0;
        L.Mm[e] = in ? p.Mm[g] : 0.0;
        L.Md[e] = in ? p.Md[g] : 0.0;
        L.G[e] = in ? p.G[g] : 0.0;
    }
}

// padded element e of a 3 x n x MP array -> (row = ax n + i, q); ax by comparison (no division by n)
template <int MP>
__device__ __forceinline__ void unpack(int e, int n, int& row, int& q, int& ax, int& ri) {
    row = e / MP;
    q = e - row * MP;
    ax = (row >= n) + (row >= 2 * n);
    ri = row - ax * n;
}

// dot product of two MP-long rows in shared memory (16-byte loads)
template <int MP>
__device__ __forceinline__ double dot_row(const double* __restrict__ a, const double* __restrict__ b) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < MP; q += 2) {
        const double2 x = *reinterpret_cast<const double2*>(a + q), y = *reinterpret_cast<const double2*>(b + q);
        s0 = fma(x.x, y.x, s0);
        s1 = fma(x.y, y.y, s1);
    }
    return s0 + s1;
}

// One pass over all terms of the iterate in L.C, window by window.  Forward (BWD = false): FT =
// F^T (F xi - E), the scatter of the exit residuals (nonzero only for active terms).  Backward:
// FT = F^T (J - I)^T F u for u = L.U.  Thread (i, tl) owns robot i at step t0 + tl and visits every
// partner, so each pair is evaluated by both of its robots with opposite orientation.
template <int MP, bool BWD>
__device__ __forceinline__ void term_pass(const UnrollParams& p, const ULayout& L, int TW) {
    const int n = p.n, S = p.S, D = 3 * n * MP;
    const int tid = threadIdx.x, i = tid % n, tl = tid / n;
    const double lat2 = p.lat * p.lat, beta = lat2 / (p.vert * p.vert);
    const double wlat2 = p.ws_lat * p.ws_lat, wbeta = wlat2 / (p.ws_vert * p.ws_vert);
    for (int e = tid; e < D; e += UT) L.FT[e] = 0.0;
    for (int t0 = 0; t0 < S; t0 += TW) {
        const int t = t0 + tl;
        const bool own = tl < TW && t < S;
        if (own) {
            const double* Wr = L.W + t * MP;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                L.posw[(ax * TW + tl) * n + i] = dot_row<MP>(L.C + (ax * n + i) * MP, Wr);
                if (BWD) L.puw[(ax * TW + tl) * n + i] = dot_row<MP>(L.U + (ax * n + i) * MP, Wr);
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
#pragma unroll 4
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
            int row, k, ax, ri;
            unpack<MP>(e, n, row, k, ax, ri);
            const double* rw = L.Rw + ax * TW * n + ri;
            const double* wk = L.W + t0 * MP + k;
            double a0 = 0.0, a1 = 0.0;
            int u = 0;
            for (; u + 1 < tw; u += 2) {
                a0 = fma(rw[u * n], wk[u * MP], a0);
                a1 = fma(rw[(u + 1) * n], wk[(u + 1) * MP], a1);
            }
            if (u < tw) a0 = fma(rw[u * n], wk[u * MP], a0);
            L.FT[e] += a0 + a1;
        }
    }
    __syncthreads();
}

// per-axis robot means (scale 1/n) or sums (scale 1) of X into out[3][m1], fixed order
template <int MP>
__device__ __forceinline__ void robot_reduce(const double* X, double* out, int n, double scale) {
    for (int c = threadIdx.x; c < 3 * MP; c += UT) {
        const int ax = c / MP, q = c % MP;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += X[(ax * n + i) * MP + q];
        out[c] = s * scale;
    }
}

template <int MP>
__global__ void __launch_bounds__(UT, 3) unroll_forward_kernel(const UnrollParams p) {
    extern __shared__ __align__(16) double sm[];
    ULayout L;
    ulayout(sm, p.n, p.S, MP, &L);
    const int n = p.n, m1 = p.m1, D = 3 * n * MP, Dg = 3 * n * m1, TW = max(1, UT / n);
    const size_t b = blockIdx.x;
    load_constants<MP>(p, L);
    double* xs = p.xs + b * (size_t)(p.iters + 1) * Dg;
    double* ls = p.ls + b * (size_t)(p.iters + 1) * Dg;
    for (int e = threadIdx.x; e < D; e += UT) {   // padded rows; global rows are m1 long
        int row, q, ax, ri;
        unpack<MP>(e, n, row, q, ax, ri);
        const bool in = q < m1;
        const size_t g = (size_t)row * m1 + q;
        L.C[e] = in ? p.xi0[b * Dg + g] : 0.0;
        L.A[e] = in ? p.lam0[b * Dg + g] : 0.0;
        L.Bv[e] = in ? p.xi_bar[b * Dg + g] : 0.0;
        if (in) {
            xs[g] = L.C[e];
            ls[g] = L.A[e];
        }
    }
    __syncthreads();
    const double inv_n = 1.0 / n;
    for (int it = 0; it < p.iters; ++it) {
        term_pass<MP, false>(p, L, TW);
        for (int e = threadIdx.x; e < D; e += UT) {   // lambda' = lambda - rho F^T r; u = 2 lambda' - lambda + xi_bar
            const double lam = L.A[e], lamn = fma(-p.rho, L.FT[e], lam);
            L.U[e] = 2.0 * lamn - lam + L.Bv[e];
            L.A[e] = lamn;
        }
        __syncthreads();
        robot_reduce<MP>(L.C, L.mean1, n, inv_n);
        robot_reduce<MP>(L.U, L.mean2, n, inv_n);
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {   // xi' = Mm Cbar + Km11 ubar + Md (C - Cbar) + Kd11 (u - ubar) + cconst
            int row, k, ax, ri;
            unpack<MP>(e, n, row, k, ax, ri);
            const double* c = L.C + row * MP;
            const double* u = L.U + row * MP;
            const double* cb = L.mean1 + ax * MP;
            const double* ub = L.mean2 + ax * MP;
            double s = k < m1 ? p.cconst[row * m1 + k] : 0.0;
#pragma unroll
            for (int q = 0; q < MP; ++q) {
                s = fma(L.Mm[k * MP + q], cb[q], s);
                s = fma(L.Km[k * MP + q], ub[q], s);
                s = fma(L.Md[k * MP + q], c[q] - cb[q], s);
                s = fma(L.Kd[k * MP + q], u[q] - ub[q], s);
            }
            L.E[e] = s;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {
            L.C[e] = L.E[e];
            int row, q, ax, ri;
            unpack<MP>(e, n, row, q, ax, ri);
            if (q < m1) {
                const size_t g = (size_t)(it + 1) * Dg + (size_t)row * m1 + q;
                xs[g] = L.E[e];
                ls[g] = L.A[e];
            }
        }
        __syncthreads();
    }
}

template <int MP>
__global__ void __launch_bounds__(UT, 3) unroll_backward_kernel(const UnrollParams p) {
    extern __shared__ __align__(16) double sm[];
    ULayout L;
    ulayout(sm, p.n, p.S, MP, &L);
    const int n = p.n, m1 = p.m1, D = 3 * n * MP, Dg = 3 * n * m1, TW = max(1, UT / n);
    const size_t b = blockIdx.x;
    load_constants<MP>(p, L);
    const double* xs = p.xs + b * (size_t)(p.iters + 1) * Dg;
    const double* gxs = p.gxs ? p.gxs + b * (size_t)(p.iters + 1) * Dg : nullptr;
    const double* gls = p.gls ? p.gls + b * (size_t)(p.iters + 1) * Dg : nullptr;
    double* gxb = p.g_xi_bar + b * Dg;
    for (int e = threadIdx.x; e < D; e += UT) {
        L.A[e] = 0.0;    // adjoint of xi_{k+1}
        L.Bv[e] = 0.0;   // adjoint of lambda_{k+1}
    }
    for (int g = threadIdx.x; g < Dg; g += UT) gxb[g] = 0.0;   // dL/dxi_bar, accumulated per element below
    __syncthreads();
    const double inv_n = 1.0 / n;
    for (int it = p.iters - 1; it >= 0; --it) {
        for (int e = threadIdx.x; e < D; e += UT) {
            int row, q, ax, ri;
            unpack<MP>(e, n, row, q, ax, ri);
            if (q < m1) {
                const size_t g = (size_t)row * m1 + q;
                if (gxs) L.A[e] += gxs[(size_t)(it + 1) * Dg + g];
                if (gls) L.Bv[e] += gls[(size_t)(it + 1) * Dg + g];
                L.C[e] = xs[(size_t)it * Dg + g];
            } else {
                L.C[e] = 0.0;
            }
        }
        __syncthreads();
        robot_reduce<MP>(L.A, L.mean1, n, inv_n);
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {   // eh = Km11^T xbar_h + Kd11^T (xh - xbar_h)
            {
                int row, k, ax, ri;
                unpack<MP>(e, n, row, k, ax, ri);
                const double* x = L.A + row * MP;
                const double* xbm = L.mean1 + ax * MP;
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < MP; ++q) {
                    s = fma(L.Km[q * MP + k], xbm[q], s);
                    s = fma(L.Kd[q * MP + k], x[q] - xbm[q], s);
                }
                L.E[e] = s;
                if (k < m1) gxb[(size_t)row * m1 + k] += s;   // the same thread owns the element every step
                const double lt = L.Bv[e] + s;
                L.Bv[e] = lt;
                L.U[e] = lt + s;
            }
        }
        __syncthreads();
        term_pass<MP, true>(p, L, TW);
        robot_reduce<MP>(L.E, L.mean2, n, 1.0);
        __syncthreads();
        for (int e = threadIdx.x; e < D; e += UT) {   // xh = rho ((n+1) eh_i - sum_j eh_j) G + rho F^T (J - I)^T F u
            int row, k, ax, ri;
            unpack<MP>(e, n, row, k, ax, ri);
            const double* eh = L.E + row * MP;
            const double* es = L.mean2 + ax * MP;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < MP; ++q) s = fma(fma((double)(n + 1), eh[q], -es[q]), L.G[q * MP + k], s);
            L.A[e] = p.rho * (s + L.FT[e]);
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < D; e += UT) {
        int row, q, ax, ri;
        unpack<MP>(e, n, row, q, ax, ri);
        if (q < m1) {
            const size_t g = (size_t)row * m1 + q;
            p.g_xi0[b * Dg + g] = L.A[e] + (gxs ? gxs[g] : 0.0);
            p.g_lam0[b * Dg + g] = L.Bv[e] + (gls ? gls[g] : 0.0);
        }
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

// m1 <= 12 -> 12 padded columns, else 16
size_t unroll_smem_bytes(int n, int S, int m1) {
    return ulayout(nullptr, n, S, m1 <= 12 ? 12 : 16, nullptr) * sizeof(double);
}

int launch_unroll_forward(const UnrollParams& p, cudaStream_t stream) {
    return launch(p.m1 <= 12 ? (const void*)unroll_forward_kernel<12> : (const void*)unroll_forward_kernel<16>, p,
                  stream, "sgsf_unroll");
}

int launch_unroll_backward(const UnrollParams& p, cudaStream_t stream) {
    return launch(p.m1 <= 12 ? (const void*)unroll_backward_kernel<12> : (const void*)unroll_backward_kernel<16>, p,
                  stream, "sgsf_unroll_backward");
}

}  // namespace sgsf
