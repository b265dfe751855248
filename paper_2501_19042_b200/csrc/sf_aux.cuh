// sf_aux.cuh -- the kernels around K1: feasibility verdict (K2), spherical
// variables of the last iteration (K2b), trajectory evaluation, the unit
// entry point of the spherical update, FP64 operator applications for the
// step API, and the FP32 FFMA peak microbenchmark (roofline denominator).
#pragma once

#include "sf_device.cuh"

namespace sgsf {

// window of time steps whose positions the per-sample aux kernels keep in shared memory
constexpr int AUX_TCH = 32;


constexpr int KMAX_AUX = 32;   // max degree + 1 for the (test-only) FP64 step kernels

struct AuxParams {
    int n, S, m1, P;
    double lat, vert, ws_lat, ws_vert, cx, cy, cz;
    const double* W;
    const double* Wd;
    const double* Wdd;
    const double* Km11;
    const double* Kd11;
    const double* cconst;
    const double* B6;
    const double* rhs;
};

// pair index (i < j) -> lexicographic position (assembly.py:235-241)
__device__ __forceinline__ void pair_of(int p, int n, int& i, int& j) {
    int row = 0, base = 0;
    while (p >= base + (n - 1 - row)) {
        base += n - 1 - row;
        ++row;
    }
    i = row;
    j = row + 1 + (p - base);
}

__device__ __forceinline__ double eval_pos(const double* __restrict__ C, const double* __restrict__ Wrow, int m1) {
    double s = 0.0;
    for (int q = 0; q < m1; ++q) s = fma(C[q], Wrow[q], s);
    return s;
}

// ---------------------------------------------------------------- K2: verdict
// check_original_constraints (assembly.py:437-487): margins of problem.py:113-137
// in FP64 on C W^T; block per sample, fixed-order reductions.
// MP (compile-time padded degree + 1, 0 = runtime m1): the position dot products unroll
template <int MP = 0>
__global__ void __launch_bounds__(256) verdict_kernel(AuxParams a, int batch, const double* __restrict__ coeffs,
                               const uint8_t* __restrict__ converged, double tol, uint8_t* ok,
                               uint8_t* feasible, double* pmin_out, double* wmax_out, int* pcount,
                               int* wcount) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int n = a.n, S = a.S, m1 = a.m1, P = a.P, dim = 3 * n * m1;
    double* C = (double*)sm;
    double* pos = C + dim;                       // 3 x n x AUX_TCH (a window of time steps)
    double* Ww = pos + 3 * n * AUX_TCH;          // the window's W rows, AUX_TCH x m1
    double* red_min = Ww + AUX_TCH * m1;         // per warp
    double* red_max = red_min + blockDim.x;
    int* red_pc = (int*)(red_max + blockDim.x);
    int* red_wc = red_pc + blockDim.x;
    int* ptab = red_wc + blockDim.x;             // pair -> i | j << 8 (lexicographic)
    const int b = blockIdx.x;
    if (b >= batch) return;
    for (int e = threadIdx.x; e < dim; e += blockDim.x) C[e] = coeffs[(size_t)b * dim + e];
    for (int q = threadIdx.x; q < P; q += blockDim.x) {
        int i, j;
        pair_of(q, n, i, j);
        ptab[q] = i | (j << 8);
    }
    const double ia2 = a.lat * a.lat, ib2 = a.vert * a.vert;
    const double wa2 = a.ws_lat * a.ws_lat, wb2 = a.ws_vert * a.ws_vert;
    const double inv_ia2 = 1.0 / ia2, inv_ib2 = 1.0 / ib2, inv_wa2 = 1.0 / wa2, inv_wb2 = 1.0 / wb2;
    double pmin = CUDART_INF, wmax = -CUDART_INF;
    int pc = 0, wc = 0;
    for (int t0 = 0; t0 < S; t0 += AUX_TCH) {
        const int tc = min(AUX_TCH, S - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < tc * m1; e += blockDim.x) Ww[e] = a.W[t0 * m1 + e];
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * n * tc; e += blockDim.x) {
            const int row = e / tc, t = e - row * tc;
            if constexpr (MP > 0) {   // the same fma order as eval_pos (q ascending from 0)
                const double* c = C + row * m1;
                const double* w = Ww + t * m1;
                double sacc = 0.0;
#pragma unroll
                for (int q = 0; q < MP; ++q)
                    if (q < m1) sacc = fma(c[q], w[q], sacc);
                pos[row * AUX_TCH + t] = sacc;
            } else {
                pos[row * AUX_TCH + t] = eval_pos(C + row * m1, Ww + t * m1, m1);
            }
        }
        __syncthreads();
        // a warp pass takes tpw terms x tc steps (lane -> (term offset, step)): the last, partial window of
        // the horizon packs several terms per warp instead of idling the lanes past tc
        const int tpw = AUX_TCH / tc, lane = threadIdx.x & 31, sub = lane / tc, t = lane - sub * tc;
        const int nwarps = (int)(blockDim.x >> 5), wid = (int)(threadIdx.x >> 5);
        for (int term0 = wid * tpw; term0 < P + n; term0 += nwarps * tpw) {
            const int term = term0 + sub;
            if (sub >= tpw || term >= P + n) continue;
            double dx, dy, dz, a2, b2;
            if (term < P) {
                const int ij = ptab[term], i = ij & 0xff, j = ij >> 8;
                dx = pos[(0 * n + i) * AUX_TCH + t] - pos[(0 * n + j) * AUX_TCH + t];
                dy = pos[(1 * n + i) * AUX_TCH + t] - pos[(1 * n + j) * AUX_TCH + t];
                dz = pos[(2 * n + i) * AUX_TCH + t] - pos[(2 * n + j) * AUX_TCH + t];
                a2 = ia2;
                b2 = ib2;
            } else {
                const int i = term - P;
                dx = pos[(0 * n + i) * AUX_TCH + t] - a.cx;
                dy = pos[(1 * n + i) * AUX_TCH + t] - a.cy;
                dz = pos[(2 * n + i) * AUX_TCH + t] - a.cz;
                a2 = wa2;
                b2 = wb2;
            }
            verdict_term(term < P, dx, dy, dz, a2, b2, term < P ? inv_ia2 : inv_wa2, term < P ? inv_ib2 : inv_wb2, tol,
                         pmin, wmax, pc, wc);
        }
    }
    // warp reductions, then one combine over the warps (min / max exact, integer counts: any order)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        pmin = fmin(pmin, __shfl_xor_sync(0xffffffffu, pmin, off));
        wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
    }
    pc = __reduce_add_sync(0xffffffffu, pc);
    wc = __reduce_add_sync(0xffffffffu, wc);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red_min[warp] = pmin;
        red_max[warp] = wmax;
        red_pc[warp] = pc;
        red_wc[warp] = wc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
            pmin = fmin(pmin, red_min[q]);
            wmax = fmax(wmax, red_max[q]);
            pc += red_pc[q];
            wc += red_wc[q];
        }
        const bool good = (pc == 0) && (wc == 0);
        if (ok) ok[b] = good;
        if (feasible) feasible[b] = good && (converged ? converged[b] != 0 : true);
        if (pmin_out) pmin_out[b] = pmin;
        if (wmax_out) wmax_out[b] = wmax;
        if (pcount) pcount[b] = pc;
        if (wcount) wcount[b] = wc;
    }
}

// ---------------------------------------------------------------- K2b: spherical variables
__global__ void svars_kernel(AuxParams a, int batch, const double* __restrict__ coeffs, double* paz,
                             double* ppol, double* prad, double* waz, double* wpol, double* wrad) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int n = a.n, S = a.S, m1 = a.m1, P = a.P, dim = 3 * n * m1;
    double* C = (double*)sm;
    double* pos = C + dim;   // 3 x n x AUX_TCH
    const int b = blockIdx.x;
    if (b >= batch) return;
    for (int e = threadIdx.x; e < dim; e += blockDim.x) C[e] = coeffs[(size_t)b * dim + e];
    for (int t0 = 0; t0 < S; t0 += AUX_TCH) {
        const int tc = min(AUX_TCH, S - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * n * tc; e += blockDim.x) {
            const int row = e / tc, t = e - row * tc;
            pos[row * AUX_TCH + t] = eval_pos(C + row * m1, a.W + (t0 + t) * m1, m1);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < (P + n) * tc; e += blockDim.x) {
            const int term = e / tc, tl = e - term * tc, t = t0 + tl;
            double az, pol, rad;
            if (term < P) {
                int i, j;
                pair_of(term, n, i, j);
                ref_spherical(pos[(0 * n + i) * AUX_TCH + tl] - pos[(0 * n + j) * AUX_TCH + tl],
                              pos[(1 * n + i) * AUX_TCH + tl] - pos[(1 * n + j) * AUX_TCH + tl],
                              pos[(2 * n + i) * AUX_TCH + tl] - pos[(2 * n + j) * AUX_TCH + tl], a.lat, a.vert, 1.0,
                              CUDART_INF, &az, &pol, &rad, nullptr, nullptr, nullptr);
                const size_t o = (size_t)b * P * S + (size_t)term * S + t;
                paz[o] = az;
                ppol[o] = pol;
                prad[o] = rad;
            } else {
                const int i = term - P;
                ref_spherical(pos[(0 * n + i) * AUX_TCH + tl] - a.cx, pos[(1 * n + i) * AUX_TCH + tl] - a.cy,
                              pos[(2 * n + i) * AUX_TCH + tl] - a.cz, a.ws_lat, a.ws_vert, 0.0, 1.0, &az, &pol,
                              &rad, nullptr, nullptr, nullptr);
                const size_t o = (size_t)b * n * S + (size_t)i * S + t;
                waz[o] = az;
                wpol[o] = pol;
                wrad[o] = rad;
            }
        }
    }
}

// ---------------------------------------------------------------- trajectory (basis.py:149-160)
__global__ void trajectory_kernel(AuxParams a, int batch, const double* __restrict__ coeffs, double* pos,
                                  double* vel, double* acc) {
    const int n = a.n, S = a.S, m1 = a.m1, dim = 3 * n * m1;
    const size_t total = (size_t)batch * n * S;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / ((size_t)n * S));
        const int rem = (int)(e - (size_t)b * n * S), i = rem / S, t = rem - i * S;
        const double* C = coeffs + (size_t)b * dim;
        for (int ax = 0; ax < 3; ++ax) {
            const double* c = C + (ax * n + i) * m1;
            if (pos) pos[e * 3 + ax] = eval_pos(c, a.W + t * m1, m1);
            if (vel) vel[e * 3 + ax] = eval_pos(c, a.Wd + t * m1, m1);
            if (acc) acc[e * 3 + ax] = eval_pos(c, a.Wdd + t * m1, m1);
        }
    }
}

// ---------------------------------------------------------------- unit entry point of the spherical update
__global__ void spherical_kernel(int count, const double* __restrict__ dx, const double* __restrict__ dy,
                                 const double* __restrict__ dz, double lat, double vert, double lo, double hi,
                                 int mode, double* az, double* pol, double* rad, double* tx, double* ty,
                                 double* tz) {
    const bool pair_family = (lo == 1.0 && hi == CUDART_INF);
    const bool ws_family = (lo == 0.0 && hi == 1.0);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
        double a_, p_, r_, x_, y_, z_;
        ref_spherical(dx[e], dy[e], dz[e], lat, vert, lo, hi, &a_, &p_, &r_, &x_, &y_, &z_);
        if (mode == 0) {
            const Family<float> f = make_family<float>(lat, vert);
            float fx, fy, fz;
            const float ax = (float)dx[e], ay = (float)dy[e], az_ = (float)dz[e];
            if (pair_family) target<float, true>(ax, ay, az_, f, fx, fy, fz);
            else if (ws_family) target<float, false>(ax, ay, az_, f, fx, fy, fz);
            else target_generic<float>(ax, ay, az_, f, lo, hi, fx, fy, fz);
            x_ = fx;
            y_ = fy;
            z_ = fz;
        } else if (mode == 1) {
            const Family<double> f = make_family<double>(lat, vert);
            if (pair_family) target<double, true>(dx[e], dy[e], dz[e], f, x_, y_, z_);
            else if (ws_family) target<double, false>(dx[e], dy[e], dz[e], f, x_, y_, z_);
            else target_generic<double>(dx[e], dy[e], dz[e], f, lo, hi, x_, y_, z_);
        }
        if (az) az[e] = a_;
        if (pol) pol[e] = p_;
        if (rad) rad[e] = r_;
        if (tx) tx[e] = x_;
        if (ty) ty[e] = y_;
        if (tz) tz[e] = z_;
    }
}

// ---------------------------------------------------------------- FP64 operators for the step API
// F xi in the flat layout [D_x; P_x; D_y; P_y; D_z; P_z] (assembly.py:1-20, 285-294)
__global__ void apply_F_kernel(AuxParams a, int batch, const double* __restrict__ xi, double* out) {
    const int n = a.n, S = a.S, m1 = a.m1, P = a.P, dim = 3 * n * m1;
    const int axis_rows = (P + n) * S;
    const size_t total = (size_t)batch * 3 * axis_rows;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / (3 * (size_t)axis_rows));
        const int rem = (int)(e - (size_t)b * 3 * axis_rows), ax = rem / axis_rows, row = rem - ax * axis_rows;
        const double* C = xi + (size_t)b * dim + ax * n * m1;
        const int term = row / S, t = row - term * S;
        double v;
        if (term < P) {
            int i, j;
            pair_of(term, n, i, j);
            v = eval_pos(C + i * m1, a.W + t * m1, m1) - eval_pos(C + j * m1, a.W + t * m1, m1);
        } else {
            v = eval_pos(C + (term - P) * m1, a.W + t * m1, m1);
        }
        out[e] = v;
    }
}

// F^T v: incidence scatter into (3, n, S), then W projection (assembly.py:296-310)
__global__ void apply_FT_kernel(AuxParams a, int batch, const double* __restrict__ v, double* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int n = a.n, S = a.S, m1 = a.m1, P = a.P, dim = 3 * n * m1;
    const int axis_rows = (P + n) * S;
    double* comb = (double*)sm;            // 3 x n x AUX_TCH (a window of time steps)
    double* acc = comb + 3 * n * AUX_TCH;  // dim: the sums over the windows so far (ascending t)
    const int b = blockIdx.x;
    if (b >= batch) return;
    const double* vb = v + (size_t)b * 3 * axis_rows;
    for (int e = threadIdx.x; e < dim; e += blockDim.x) acc[e] = 0.0;
    for (int t0 = 0; t0 < S; t0 += AUX_TCH) {
        const int tc = min(AUX_TCH, S - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * n * tc; e += blockDim.x) {
            const int row = e / tc, t = t0 + (e - row * tc), ax = row / n, i = row - ax * n;
            const double* va = vb + (size_t)ax * axis_rows;
            double s = 0.0;
            int p = 0;
            for (int r = 0; r < n; ++r)
                for (int c = r + 1; c < n; ++c, ++p) {
                    if (r == i) s += va[p * S + t];
                    else if (c == i) s -= va[p * S + t];
                }
            comb[row * AUX_TCH + (t - t0)] = s + va[P * S + i * S + t];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < dim; e += blockDim.x) {
            const int row = e / m1, q = e - row * m1;
            double s = acc[e];
            for (int t = 0; t < tc; ++t) s = fma(comb[row * AUX_TCH + t], a.W[(t0 + t) * m1 + q], s);
            acc[e] = s;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < dim; e += blockDim.x) out[(size_t)b * dim + e] = acc[e];
}

// literal coefficient step from eta: C_i = Km11 eta_bar + Kd11 (eta_i - eta_bar) + cconst_i
__global__ void kkt_step_kernel(AuxParams a, int batch, const double* __restrict__ eta, double* out,
                                double* eq_err) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int n = a.n, m1 = a.m1, dim = 3 * n * m1;
    double* ebar = (double*)sm;          // 3 x m1
    double* emax = ebar + 3 * m1;        // 3n
    const int b = blockIdx.x;
    if (b >= batch) return;
    const double* E = eta + (size_t)b * dim;
    for (int e = threadIdx.x; e < 3 * m1; e += blockDim.x) {
        const int ax = e / m1, q = e - ax * m1;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += E[(ax * n + i) * m1 + q];
        ebar[e] = s / n;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < 3 * n; r += blockDim.x) {
        const int ax = r / n;
        double cn[KMAX_AUX];
        for (int q = 0; q < m1; ++q) {
            double s = a.cconst[r * m1 + q];
            for (int q2 = 0; q2 < m1; ++q2) {
                s = fma(a.Km11[q * m1 + q2], ebar[ax * m1 + q2], s);
                s = fma(a.Kd11[q * m1 + q2], E[r * m1 + q2] - ebar[ax * m1 + q2], s);
            }
            cn[q] = s;
            out[(size_t)b * dim + r * m1 + q] = s;
        }
        double mx = 0.0;
        for (int c = 0; c < 6; ++c) {
            double e = -a.rhs[r * 6 + c];
            for (int q = 0; q < m1; ++q) e = fma(a.B6[c * m1 + q], cn[q], e);
            mx = fmax(mx, fabs(e));
        }
        emax[r] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0 && eq_err) {
        double mx = 0.0;
        for (int r = 0; r < 3 * n; ++r) mx = fmax(mx, emax[r]);
        eq_err[b] = mx;
    }
}

// ---------------------------------------------------------------- FP32 FFMA peak
__global__ void ffma_peak_kernel(float* out, int iters, float seed) {
    float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
    float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
    const float m = 0.9999f, c = 1e-4f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
            a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
        }
    }
    const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678f) out[0] = s;   // keeps the chain alive
}

}  // namespace sgsf

namespace sgsf {

// ---------------------------------------------------------------- pairwise cosine / diversity (metrics.py:83-115)
// mean over i < j of cos(v_i, v_j) with v optionally centred by the column mean.  With u_i = v_i / |v_i|:
//   sum_{i<j} u_i . u_j = (|sum_i u_i|^2 - sum_i |u_i|^2) / 2,
// so the mean is an O(count * dim) reduction instead of a count x count Gram matrix.  All sums run in a
// fixed order (deterministic).
constexpr int COS_THREADS = 256;

__device__ __forceinline__ double block_sum_fixed(double v, double* red) {
    red[threadIdx.x] = v;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

__global__ void cos_colmean_kernel(int count, int dim, const double* __restrict__ V, double* mean) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= dim) return;
    double s = 0.0;
    for (int b = 0; b < count; ++b) s += V[(size_t)b * dim + d];
    mean[d] = s / count;
}

__global__ void cos_rownorm_kernel(int count, int dim, const double* __restrict__ V, const double* __restrict__ mean,
                                   double* inv, double* u2, int* zero) {
    __shared__ double red[COS_THREADS];
    const int b = blockIdx.x;
    double s = 0.0;
    for (int d = threadIdx.x; d < dim; d += blockDim.x) {
        const double x = V[(size_t)b * dim + d] - (mean ? mean[d] : 0.0);
        s = fma(x, x, s);
    }
    const double n2 = block_sum_fixed(s, red);
    if (threadIdx.x == 0) {
        if (n2 == 0.0) {
            atomicOr(zero, 1);
            inv[b] = 0.0;
            u2[b] = 0.0;
        } else {
            const double iv = 1.0 / sqrt(n2);
            inv[b] = iv;
            u2[b] = n2 * iv * iv;
        }
    }
}

__global__ void cos_colsum_kernel(int count, int dim, const double* __restrict__ V, const double* __restrict__ mean,
                                  const double* __restrict__ inv, double* ssum) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= dim) return;
    const double m = mean ? mean[d] : 0.0;
    double s = 0.0;
    for (int b = 0; b < count; ++b) s = fma(V[(size_t)b * dim + d] - m, inv[b], s);
    ssum[d] = s;
}

__global__ void cos_final_kernel(int count, int dim, const double* __restrict__ ssum, const double* __restrict__ u2,
                                 const int* __restrict__ zero, double* out) {
    __shared__ double red[COS_THREADS];
    double a = 0.0, c = 0.0;
    for (int d = threadIdx.x; d < dim; d += blockDim.x) a = fma(ssum[d], ssum[d], a);
    for (int b = threadIdx.x; b < count; b += blockDim.x) c += u2[b];
    const double s2 = block_sum_fixed(a, red);
    const double uu = block_sum_fixed(c, red);
    if (threadIdx.x == 0) out[0] = *zero ? CUDART_NAN : (s2 - uu) / ((double)count * (count - 1));
}

}  // namespace sgsf
