// sf_large.cuh -- K1L: the safety filter for 32 < n <= 64 robots (BASELINE config 4).
//
// Same alternating minimisation and the same per-term arithmetic as K1
// (sf_persistent.cuh), organised for swarms whose state does not fit K1's
// one-thread-per-time-step layout: a 64-robot step has 2016 pair terms, so
// K1's per-step term bitmasks (66 words) and its two [S][3n] position
// buffers (237 KB at H=150) do not fit registers / shared memory.
//
// One CTA of 8 warps per sample (persistent over the ordered sample queue).
// Term pass: warp w takes time steps w, w+8, ...; per step the positions of
// the new and of the previous iterate are evaluated into a per-warp scratch,
// and lane l owns robots l and l+32: it visits every partner, so its
// scattered residual R_i accumulates in registers in a fixed order
// (deterministic; each pair is evaluated by both of its robots, its exit
// residual counted once).  Terms are evaluated exactly (interior test,
// trig-free target for non-interior terms, FP64 reference trig for terms with
// an exactly-zero component) on a step's "exact pass", which also records the
// step's near pairs (distance < 1.5, up to kNearCap, in a fixed ballot order)
// and the min distance rmin of the others.  While rmin - cum > 1 + margin
// (cum: accumulated pair motion, as K1) the far pairs are provably interior,
// so the step is "quiet": only its near pairs are evaluated exactly, by the
// lanes owning their robots, and the far pairs' exit residuals come from the
// O(n) statistics of the position change minus the near pairs' share (the
// far max is recomputed exactly if a near pair attains the statistic's max).
// g = R W accumulates per lane for the active robot rows and is combined
// across warps in warp order (ticket), so the FP sum order is fixed.
// The FP64 xi-step, equality check and commit are K1's DMMA formulation,
// one warp per axis with 8 robot tiles.
#pragma once

#include "sf_persistent.cuh"

namespace sgsf {

constexpr int kLargeWarps = 8;
constexpr int kNearCap = 48;         // near pairs remembered per time step (more: the step stays exact)
constexpr float kLargeSkin = 1.5f;   // near: normalised distance < kLargeSkin at the last exact pass

struct LargeShared {
    int sample;
    int active[2];   // by iteration parity (cleared for the other parity at the top of an iteration)
    int g_ticket;    // fixed-order g accumulation: warp w adds when g_ticket == k * kLargeWarps + w
};

struct LargeLayout {
    size_t W, KMm, KMd, cconst, B6, rhs, PBt;
    size_t C, Cp, lam, U, xb, g, Cf, Cfo, scr, winf, wsq, winf64, eqerr, srmin, scum, sflag, snear, sncnt, sh;
    size_t sdefer, xr, xnl, xcnt, xfm, xzf;
    size_t ner;   // per warp: the R of each near pair of the quiet step at hand (evaluated once per pair)
    size_t gwords;   // doubles of the g region (g itself, or the larger term-pass scratch aliased on it)   // the cooperative exact steps (phase B), double-buffered partials
    size_t total;
};

template <typename T, int NB>
__host__ __device__ inline LargeLayout make_large_layout(int n, int S, int MP, int want_prev, int coop = 1) {
    LargeLayout L;
    size_t o = 0;
    const size_t d = sizeof(double), ts = sizeof(T);
    const size_t dimp = (size_t)3 * n * MP;
    L.W = o;      o = align16(o + (size_t)S * MP * ts);
    L.KMm = o;    o = align16(o + (size_t)MP * 2 * MP * d);
    L.KMd = o;    o = align16(o + (size_t)MP * 2 * MP * d);
    L.cconst = o; o = align16(o + dimp * d);
    L.B6 = o;     o = align16(o + (size_t)6 * MP * d);
    L.rhs = o;    o = align16(o + (size_t)3 * n * 6 * d);
    L.PBt = o;    o = align16(o + (size_t)MP * 6 * d);
    L.C = o;      o = align16(o + dimp * d);
    L.Cp = o;     o = align16(o + (want_prev ? dimp * d : 0));
    L.lam = o;    o = align16(o + dimp * d);
    L.U = o;      o = align16(o + dimp * d);
    L.xb = o;     o = align16(o + dimp * d);
    // g is all-zero during the term pass (it is accumulated after it, and cleared by the xi-step), so the term
    // pass's scratch -- the near-pair R rows of phase A and the partials of phase B -- lives in it; the kernel
    // clears it again before the g accumulation.  (As separate buffers they pushed 64 robots at degree >= 12
    // past the 227 KB of shared memory.)
    // phase B (its partials live in the g region) unless that does not fit: the launcher then retries with coop = 0
    // and the kernel keeps the one-warp exact pass (FP64 "strict" at long horizons)
    const size_t pb = coop ? 1 : 0;
    const size_t xr_b = align16(pb * 2 * kLargeWarps * 2 * 32 * 3 * ts);   // [buf][warp][rr][lane][axis] R parts
    const size_t xnl_b = align16(pb * 2 * kLargeWarps * 2 * kNearCap * 2);  // [buf][warp][rr] near sublists
    const size_t xcnt_b = align16(pb * 2 * kLargeWarps * 2 * 4);             // ... their lengths
    const size_t xfm_b = align16(pb * 2 * kLargeWarps * ts);                 // [buf][warp] min far q
    const size_t xzf_b = align16(pb * 2 * kLargeWarps * 4);                  // ... a far zero component
    const size_t ner_b = align16((size_t)kLargeWarps * kNearCap * 3 * ts);   // phase A: per warp, the near pairs' R
    const size_t scratch = xr_b + xnl_b + xcnt_b + xfm_b + xzf_b > ner_b ? xr_b + xnl_b + xcnt_b + xfm_b + xzf_b : ner_b;
    L.g = o;      o = align16(o + (dimp * d > scratch ? dimp * d : scratch));
    L.gwords = (o - L.g) / d;
    L.ner = L.g;
    L.xr = L.g;
    L.xnl = L.xr + xr_b;
    L.xcnt = L.xnl + xnl_b;
    L.xfm = L.xcnt + xcnt_b;
    L.xzf = L.xfm + xfm_b;
    L.Cf = o;     o = align16(o + (size_t)3 * MP * NB * ts);   // C of the current iterate, robot-minor
    L.Cfo = o;    o = align16(o + (size_t)3 * MP * NB * ts);   // ... of the previous iterate
    L.scr = o;    o = align16(o + (size_t)kLargeWarps * 2 * 3 * NB * ts);
    L.winf = o;   o = align16(o + (size_t)kLargeWarps * ts);
    L.wsq = o;    o = align16(o + (size_t)kLargeWarps * d);
    L.winf64 = o; o = align16(o + (size_t)kLargeWarps * d);   // hybrid: FP64 per-warp exit-residual maxima
    L.eqerr = o;  o = align16(o + (size_t)4 * d);
    L.srmin = o;  o = align16(o + (size_t)S * ts);   // per step: min normalised pair distance at the last exact pass
    L.scum = o;   o = align16(o + (size_t)S * ts);   // ... pair motion bound accumulated since
    L.sflag = o;  o = align16(o + (size_t)S * 4);    // ... 1: no far pair had a zero component
    L.snear = o;  o = align16(o + (size_t)S * kNearCap * 2);   // ... the near pairs (i | j << 8), i < j
    L.sncnt = o;  o = align16(o + (size_t)S * 4);    // ... how many (-1: none recorded / overflow)
    L.sh = o;     o = align16(o + sizeof(LargeShared));
    L.sdefer = o; o = align16(o + pb * S * 4);    // per step: 1 = exact this iteration, taken by phase B
    L.total = o;
    return L;
}

// One term, evaluated exactly: r = d_new - e(d_new) (the lam' residual; 0 for interior terms) and
// x = d_new - e(d_old) (the exit residual against the previous targets).  Terms with an exactly-zero
// component use the FP64 reference formula (sf_device.cuh).
template <typename T, bool PAIR>
__device__ __forceinline__ void exact_term(const T (&dn)[3], const T (&dd)[3], const Family<T>& f, T (&r)[3],
                                           T (&x)[3]) {
    if (dn[0] == T(0) || dn[1] == T(0) || dn[2] == T(0)) {
        T t[3];
        target<T, PAIR>(dn[0], dn[1], dn[2], f, t[0], t[1], t[2]);
#pragma unroll
        for (int a = 0; a < 3; ++a) r[a] = dn[a] - t[a];
    } else {
        const T q = fma_t<T>(dn[2] * f.beta, dn[2], fma_t<T>(dn[1], dn[1], dn[0] * dn[0]));
        const bool in = PAIR ? (q >= f.lim) : (q <= f.lim);
        const T s = in ? T(1) : f.lat * rsq<T>(q);
#pragma unroll
        for (int a = 0; a < 3; ++a) r[a] = in ? T(0) : fma_t<T>(-s, dn[a], dn[a]);
    }
    if (dd[0] == T(0) || dd[1] == T(0) || dd[2] == T(0)) {
        T e[3];
        target<T, PAIR>(dd[0], dd[1], dd[2], f, e[0], e[1], e[2]);
#pragma unroll
        for (int a = 0; a < 3; ++a) x[a] = dn[a] - e[a];
    } else {
        const T q = fma_t<T>(dd[2] * f.beta, dd[2], fma_t<T>(dd[1], dd[1], dd[0] * dd[0]));
        const bool in = PAIR ? (q >= f.lim) : (q <= f.lim);
        const T s = in ? T(1) : f.lat * rsq<T>(q);
#pragma unroll
        for (int a = 0; a < 3; ++a) x[a] = in ? dn[a] - dd[a] : fma_t<T>(-s, dd[a], dn[a]);
    }
}

// Hybrid precision (HY, as K1's): the FP32 term pass screens with narrowed interior limits; the scattered
// residual of every term it does not call interior is recomputed from FP64 positions of the FP64 C (and
// rounded once into the lane's FP32 accumulators); the stop decision re-evaluates the whole exit residual in
// FP64 when the FP32-measured one lies within hy_delta of tol_res.
// FP64 scattered residual d - e(d) of one term (j < 0: the workspace term of robot i), positions from the
// FP64 coefficients; out of line with explicit scalars (the cold path of the hybrid term pass)
template <int MP>
__device__ __noinline__ D3 large_term_r64(const double* __restrict__ C, const double* __restrict__ Wrow, int m1,
                                         int n, int i, int j, double cx, double cy, double cz,
                                         const Family<double> f) {
    D3 d;
    if (j >= 0) {
        d.x = pos64s<MP>(C, Wrow, m1, i) - pos64s<MP>(C, Wrow, m1, j);
        d.y = pos64s<MP>(C, Wrow, m1, n + i) - pos64s<MP>(C, Wrow, m1, n + j);
        d.z = pos64s<MP>(C, Wrow, m1, 2 * n + i) - pos64s<MP>(C, Wrow, m1, 2 * n + j);
    } else {
        d.x = pos64s<MP>(C, Wrow, m1, i) - cx;
        d.y = pos64s<MP>(C, Wrow, m1, n + i) - cy;
        d.z = pos64s<MP>(C, Wrow, m1, 2 * n + i) - cz;
    }
    return resid64(j >= 0, d, d, f);
}

struct LargeExitArgs {   // by value: a non-inlined callee must not take the kernel's parameter block by reference
    const double* W;
    int n, S, m1;
    double cx, cy, cz;
    Family<double> fp, fw;
};
template <int MP>
__device__ __noinline__ double2 large_exit64(const LargeExitArgs p, const double* __restrict__ C,
                                             const double* __restrict__ Cp, int warp, int lane) {
    // every term of this warp's steps, both iterates' FP64 positions: the lane holds robots lane and lane + 32,
    // partners come by warp broadcast (warp-uniform j loop); each pair counted once (i < j)
    const int n = p.n, S = p.S, m1 = p.m1;
    const Family<double>& fp = p.fp;
    const Family<double>& fw = p.fw;
    double mx = 0.0, s2 = 0.0;
    for (int t = warp; t < S; t += kLargeWarps) {
        const double* Wrow = p.W + (size_t)t * m1;
        double pn[2][3], po[2][3];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int i = lane + 32 * rr;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                pn[rr][a] = i < n ? pos64s<MP>(C, Wrow, m1, a * n + i) : 0.0;
                po[rr][a] = i < n ? pos64s<MP>(Cp, Wrow, m1, a * n + i) : 0.0;
            }
        }
        for (int j = 0; j < n; ++j) {
            const int src = j & 31, sj = j >> 5;
            double qn[3], qo[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                qn[a] = __shfl_sync(0xffffffffu, sj ? pn[1][a] : pn[0][a], src);
                qo[a] = __shfl_sync(0xffffffffu, sj ? po[1][a] : po[0][a], src);
            }
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int i = lane + 32 * rr;
                if (i < n && i < j) {
                    const D3 dn{pn[rr][0] - qn[0], pn[rr][1] - qn[1], pn[rr][2] - qn[2]};
                    const D3 dol{po[rr][0] - qo[0], po[rr][1] - qo[1], po[rr][2] - qo[2]};
                    const D3 x = resid64(true, dol, dn, fp);
                    mx = fmax(mx, fmax(fabs(x.x), fmax(fabs(x.y), fabs(x.z))));
                    s2 = fma(x.x, x.x, fma(x.y, x.y, fma(x.z, x.z, s2)));
                }
            }
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int i = lane + 32 * rr;
            if (i < n) {
                const D3 dn{pn[rr][0] - p.cx, pn[rr][1] - p.cy, pn[rr][2] - p.cz};
                const D3 dol{po[rr][0] - p.cx, po[rr][1] - p.cy, po[rr][2] - p.cz};
                const D3 x = resid64(false, dol, dn, fw);
                mx = fmax(mx, fmax(fabs(x.x), fmax(fabs(x.y), fabs(x.z))));
                s2 = fma(x.x, x.x, fma(x.y, x.y, fma(x.z, x.z, s2)));
            }
        }
    }
    mx = warp_max_nonneg(mx);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    return make_double2(mx, s2);
}

template <typename T, int NB, int MP, bool HY = false>
__global__ void __launch_bounds__(32 * kLargeWarps, 1) sf_large_kernel(const SolveParams p) {
    static_assert(NB == 64, "K1L is laid out for 64 robots (lane l owns robots l and l + 32)");
    static_assert(!HY || sizeof(T) == 4, "hybrid precision screens in FP32");
    extern __shared__ __align__(16) unsigned char smem[];
    const LargeLayout L = make_large_layout<T, NB>(p.n, p.S, MP, p.want_prev || HY, p.large_coop);
    constexpr int M2P = 2 * MP;
    constexpr int MT = NB / 8;   // 8-robot DMMA tiles
    constexpr int KT = MP / 2;   // 4-column k-steps over [C | u]
    constexpr int KC = MP / 4;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int n = p.n, S = p.S, m1 = p.m1;
    const int R3 = 3 * n, dim = R3 * m1, dimp = R3 * MP;

    T* Wt = (T*)(smem + L.W);
    double* KMm = (double*)(smem + L.KMm);
    double* KMd = (double*)(smem + L.KMd);
    double* cconst = (double*)(smem + L.cconst);
    double* B6 = (double*)(smem + L.B6);
    double* rhs = (double*)(smem + L.rhs);
    double* PBt = (double*)(smem + L.PBt);
    double* C = (double*)(smem + L.C);
    double* Cp = (double*)(smem + L.Cp);
    double* lam = (double*)(smem + L.lam);
    double* U = (double*)(smem + L.U);
    double* xb = (double*)(smem + L.xb);
    double* g = (double*)(smem + L.g);
    T* Cf = (T*)(smem + L.Cf);
    T* Cfo = (T*)(smem + L.Cfo);
    T* winf = (T*)(smem + L.winf);
    double* wsq = (double*)(smem + L.wsq);
    double* winf64 = (double*)(smem + L.winf64);
    double* eqerr = (double*)(smem + L.eqerr);
    T* srmin = (T*)(smem + L.srmin);
    T* scum = (T*)(smem + L.scum);
    int* sflag = (int*)(smem + L.sflag);
    uint16_t* snear = (uint16_t*)(smem + L.snear);
    int* sncnt = (int*)(smem + L.sncnt);
    LargeShared* sh = (LargeShared*)(smem + L.sh);
    const bool kCoopExact = p.large_coop != 0;   // phase B: exact steps taken by all warps together
    int* sdefer = (int*)(smem + L.sdefer);
    T* xr = (T*)(smem + L.xr);
    uint16_t* xnl = (uint16_t*)(smem + L.xnl);
    int* xcnt = (int*)(smem + L.xcnt);
    T* xfm = (T*)(smem + L.xfm);
    int* xzf = (int*)(smem + L.xzf);

    // shared constants (as K1), zero-padded to MP columns
    for (int i = tid; i < S * MP; i += nt) {
        const int t = i / MP, q = i % MP;
        Wt[i] = (q < m1) ? (T)p.W[t * m1 + q] : T(0);
    }
    for (int i = tid; i < MP * M2P; i += nt) {
        const int q = i / M2P, c = i % M2P, half = c / MP, q2 = c % MP;
        const bool in = q < m1 && q2 < m1;
        KMm[i] = in ? p.KMm[q * 2 * m1 + half * m1 + q2] - p.KMd[q * 2 * m1 + half * m1 + q2] : 0.0;
        KMd[i] = in ? p.KMd[q * 2 * m1 + half * m1 + q2] : 0.0;
    }
    for (int i = tid; i < dimp; i += nt) {
        const int r = i / MP, q = i % MP;
        cconst[i] = (q < m1) ? p.cconst[r * m1 + q] : 0.0;
    }
    for (int i = tid; i < 6 * MP; i += nt) {
        const int c = i / MP, q = i % MP;
        B6[i] = (q < m1) ? p.B6[c * m1 + q] : 0.0;
    }
    for (int i = tid; i < R3 * 6; i += nt) rhs[i] = p.rhs[i];
    for (int i = tid; i < MP * 6; i += nt) PBt[i] = (i / 6 < m1) ? p.PBt[i] : 0.0;
    if (tid == 0) {
        sh->sample = next_sample(p);
        sh->active[0] = sh->active[1] = 0;
    }
    __syncthreads();

    Family<T> fp = make_family<T>(p.lat, p.vert);
    Family<T> fw = make_family<T>(p.ws_lat, p.ws_vert);
    if constexpr (HY) {   // guard bands: a term the FP32 test calls interior is interior in FP64
        fp.lim = (T)p.hy_fp_lim_f;
        fw.lim = (T)p.hy_fw_lim_f;
    }
    const T cen[3] = {(T)p.cx, (T)p.cy, (T)p.cz};
    const double inv_n = 1.0 / n;
    const T inv_lat = T(1) / fp.lat;
    const T skin_lim = T(kLargeSkin * kLargeSkin) * fp.lim;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    T* sn = (T*)(smem + L.scr) + warp * 2 * 3 * NB;   // this warp's positions at the step: new [3][NB] ...
    T* so = sn + 3 * NB;                              // ... and old [3][NB]
    T* ner = (T*)(smem + L.ner) + warp * kNearCap * 3;   // this warp's near-pair R rows of the quiet step
    int sample = sh->sample;
    bool prev_active = false;

    while (sample < p.batch) {
        // ---------------- load the sample (default start = boundary projection), g = 0
        for (int r = tid; r < R3; r += nt) {
            const double* xr = p.xi_bar + (size_t)sample * dim + r * m1;
            double x[MP], c[MP], l[MP];
#pragma unroll
            for (int q = 0; q < MP; ++q) x[q] = (q < m1) ? xr[q] : 0.0;
            const int mode = p.init_mode ? p.init_mode[sample] : 0;
            if (mode) {
                const double* cr = p.xi0 + (size_t)sample * dim + r * m1;
                const double* lr = p.lam0 + (size_t)sample * dim + r * m1;
#pragma unroll
                for (int q = 0; q < MP; ++q) {
                    c[q] = (q < m1) ? cr[q] : 0.0;
                    l[q] = (q < m1) ? lr[q] : 0.0;
                }
            } else {
                double res[6];
#pragma unroll
                for (int cnd = 0; cnd < 6; ++cnd) {
                    double e = 0.0;
#pragma unroll
                    for (int q = 0; q < MP; ++q) e = fma(B6[cnd * MP + q], x[q], e);
                    res[cnd] = e - rhs[r * 6 + cnd];
                }
#pragma unroll
                for (int q = 0; q < MP; ++q) {
                    double corr = 0.0;
#pragma unroll
                    for (int cnd = 0; cnd < 6; ++cnd) corr = fma(PBt[q * 6 + cnd], res[cnd], corr);
                    c[q] = x[q] - corr;
                    l[q] = 0.0;
                }
            }
            const int ax = r / n, i = r - ax * n;
#pragma unroll
            for (int q = 0; q < MP; ++q) {
                const int idx = r * MP + q;
                xb[idx] = x[q];
                C[idx] = c[q];
                lam[idx] = l[q];
                g[idx] = 0.0;
                if (p.want_prev || HY) Cp[idx] = c[q];
                Cf[(ax * MP + q) * NB + i] = (T)c[q];
                Cfo[(ax * MP + q) * NB + i] = (T)c[q];   // no previous iterate: "old" := "new"
            }
        }
        for (int t = tid; t < S; t += nt) {   // the first iterate takes the exact pass everywhere
            sflag[t] = 0;
            sncnt[t] = -1;
            if (kCoopExact) sdefer[t] = 0;
        }
        if (tid == 0) sh->g_ticket = 0;
        __syncthreads();

#ifdef SGSF_LARGE_PT
        __shared__ long long lpt_dur[kLargeWarps];
        __shared__ int lpt_ex[kLargeWarps];
        __shared__ long long lpt_exq[kLargeWarps];
        long long lqa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        long long lmx = 0;   // thread 0: cycles from the U step through the xi-step barrier   // CTA 0 warp 0 quiet steps: positions, statistics, near pairs + ws, far
        double lpt_max = 0, lpt_mean = 0, lpt_exmax = 0, lpt_exmean = 0, lpt_qmax = 0, lpt_excyc = 0;
#endif
        for (int k = 0;; ++k) {
            const int par = k & 1;
#ifdef SGSF_LARGE_PT
            const long long lpt0 = clock64();
            int lpt_nex = 0;
            long long lpt_exc = 0;   // cycles in exact steps (phase B: all of it)
#endif
            if (tid == 0) sh->active[par ^ 1] = 0;   // last read before the previous closing barrier
            // ---------------- term pass
            T gacc[2][3][MP];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int q = 0; q < MP; ++q) gacc[rr][a][q] = T(0);
            T linf = T(0);
            double lsq = 0.0;
            bool lact = false;
            for (int t = warp; t < S; t += kLargeWarps) {
#ifdef SGSF_LARGE_PT
                const long long lq0 = clock64();
#endif
                T w[MP];
                load_row16<T, MP>(Wt + t * MP, w);
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int i = lane + 32 * rr;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        T pn = T(0), po = T(0);
#pragma unroll
                        for (int q = 0; q < MP; ++q) {
                            pn = fma_t<T>(Cf[(a * MP + q) * NB + i], w[q], pn);
                            po = fma_t<T>(Cfo[(a * MP + q) * NB + i], w[q], po);
                        }
                        sn[a * NB + i] = pn;
                        so[a * NB + i] = po;
                    }
                }
                __syncwarp();
#ifdef SGSF_LARGE_PT
                const long long lq1 = clock64();
#endif
                // O(n) statistics of the position change (lane: robots lane, lane + 32) and the pair
                // motion bound: while rmin - cum > 1 + margin, every pair of this step is provably
                // interior now, and if it was interior (and free of zero components) at the last exact
                // pass, the pair exit residuals are the changes Dp_i - Dp_j: inf = per-axis range,
                // sum of squares = n sum Dp^2 - (sum Dp)^2 per axis.  No R contribution.
                T lo[3], hi[3], s1[3], s2[3], dmv = T(0);
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    lo[a] = T(1e30);
                    hi[a] = T(-1e30);
                    s1[a] = T(0);
                    s2[a] = T(0);
                }
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int i = lane + 32 * rr;
                    if (i < n) {
                        T dq = T(0);
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const T dp = sn[a * NB + i] - so[a * NB + i];
                            lo[a] = fmin(lo[a], dp);
                            hi[a] = fmax(hi[a], dp);
                            s1[a] += dp;
                            s2[a] = fma_t<T>(dp, dp, s2[a]);
                            dq = fma_t<T>(a == 2 ? dp * fp.beta : dp, dp, dq);
                        }
                        dmv = fmax(dmv, dq);
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    dmv = fmax(dmv, __shfl_xor_sync(0xffffffffu, dmv, off));
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], off));
                        hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], off));
                        s1[a] += __shfl_xor_sync(0xffffffffu, s1[a], off);
                        s2[a] += __shfl_xor_sync(0xffffffffu, s2[a], off);
                    }
                }
#ifdef SGSF_LARGE_PT
                const long long lq2 = clock64();
#endif
                const T cum_t = scum[t] + T(2) * sqrt(dmv) * inv_lat;
                const int ncnt = sncnt[t];
                // quiet: the far pairs (distance >= rmin >= skin at the last exact pass, no zero component
                // there) are provably interior now and were before; the near pairs are evaluated exactly
                const bool quiet = k > 0 && ncnt >= 0 && sflag[t] != 0 && srmin[t] - cum_t > T(1) + T(1e-3);
                if (lane == 0) SGSF_COUNT(quiet ? 6 : 5, 1);   // diagnostics: quiet / exact steps
#ifdef SGSF_LARGE_PT
                lpt_nex += quiet ? 0 : 1;
                const long long lpt_s0 = clock64();
#endif
                if (kCoopExact && !quiet) {   // an exact step: all eight warps take it together below (phase B)
                    if (lane == 0) sdefer[t] = 1;
                    __syncwarp();   // the scratch is rewritten for the next step
                    continue;
                }
                const uint16_t* nl = snear + (size_t)t * kNearCap;
                T farmin = T(1e30);    // exact pass: min q over the far pairs of this lane's robots
                bool zfar = false;     // ... a zero component in a far pair
                int nbase = 0;         // ... near pairs recorded so far (warp-uniform)
                T nq_sq = T(0), nq_max = T(0);   // quiet: near pairs' share of the O(n) statistics
                uint64_t nmask[2] = {0ull, 0ull};  // quiet: near partners of this lane's robots
                if (quiet) {   // every near pair once, lane e -> entry e: its R (kept for both robots), its exit
                    // residual and its share of the O(n) statistics; the robots then add their pairs' R in list
                    // order below (bitwise what the per-robot evaluation gave: the same d = p_min - p_max)
                    for (int e = lane; e < ncnt; e += 32) {
                        const int code = nl[e], pa = code & 0xff, pb = code >> 8;   // pa < pb
                        T dn[3], dd[3], r[3], x[3];
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            dn[a] = sn[a * NB + pa] - sn[a * NB + pb];
                            dd[a] = so[a * NB + pa] - so[a * NB + pb];
                        }
                        exact_term<T, true>(dn, dd, fp, r, x);
                        if constexpr (HY) {   // not interior under the guarded FP32 test: R from FP64
                            if (r[0] != T(0) || r[1] != T(0) || r[2] != T(0)) {
                                const D3 r64 = large_term_r64<MP>(C, p.W + (size_t)t * m1, m1, n, pa, pb, p.cx, p.cy, p.cz,
                                                                  family64(p, true));
                                r[0] = (T)r64.x;
                                r[1] = (T)r64.y;
                                r[2] = (T)r64.z;
                            }
                        }
                        T m = T(0), q2 = T(0);
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            ner[e * 3 + a] = r[a];
                            linf = fmax(linf, fabs(x[a]));
                            lsq = fma((double)x[a], (double)x[a], lsq);
                            const T xq = (sn[a * NB + pa] - so[a * NB + pa]) - (sn[a * NB + pb] - so[a * NB + pb]);
                            m = fmax(m, fabs(xq));
                            q2 = fma_t<T>(xq, xq, q2);
                        }
                        nq_max = fmax(nq_max, m);
                        nq_sq += q2;
                    }
                    __syncwarp();
                }
#ifdef SGSF_LARGE_PT
                const long long lq2b = clock64();
#endif
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int i = lane + 32 * rr;
                    const bool iv = i < n;
                    T Ri[3] = {T(0), T(0), T(0)};
                    T ni[3], oi[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        ni[a] = sn[a * NB + i];
                        oi[a] = so[a * NB + i];
                    }
                    auto pair_exact = [&](int j, bool count_exit) {   // the pair (i, j), exactly
                        const bool fwd = i < j;   // the pair is (min, max): d = p_min - p_max
                        T dn[3], dd[3], r[3], x[3];
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const T nj = sn[a * NB + j], oj = so[a * NB + j];
                            dn[a] = fwd ? ni[a] - nj : nj - ni[a];
                            dd[a] = fwd ? oi[a] - oj : oj - oi[a];
                        }
                        exact_term<T, true>(dn, dd, fp, r, x);
                        if constexpr (HY) {   // a term not interior under the guarded FP32 test: R from FP64
                            if (r[0] != T(0) || r[1] != T(0) || r[2] != T(0)) {
                                const D3 r64 = large_term_r64<MP>(C, p.W + (size_t)t * m1, m1, n, fwd ? i : j, fwd ? j : i,
                                                                  p.cx, p.cy, p.cz, family64(p, true));
                                r[0] = (T)r64.x;
                                r[1] = (T)r64.y;
                                r[2] = (T)r64.z;
                            }
                        }
#pragma unroll
                        for (int a = 0; a < 3; ++a) Ri[a] += fwd ? r[a] : -r[a];
                        if (fwd && count_exit) {
#pragma unroll
                            for (int a = 0; a < 3; ++a) {
                                linf = fmax(linf, fabs(x[a]));
                                lsq = fma((double)x[a], (double)x[a], lsq);
                            }
                        }
                        return fma_t<T>(dn[2] * fp.beta, dn[2], fma_t<T>(dn[1], dn[1], dn[0] * dn[0]));
                    };
                    if (quiet) {
                        // the near pairs of robot i, in list order: a byte compare (__vcmpeq4 against i in every
                        // byte) of 8 entries per 16-byte load marks the entries that name i, then one pass over
                        // the marks (the per-entry test was ~3K cycles of a ~7K-cycle quiet step)
                        uint64_t hits = 0ull;
                        const uint32_t key = (uint32_t)i * 0x01010101u;
                        for (int c8 = 0; iv && c8 < ncnt; c8 += 8) {
                            const uint4 v = *reinterpret_cast<const uint4*>(nl + c8);
                            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                const uint32_t mt = __vcmpeq4(w4[h], key);
                                const uint64_t two = ((mt & 0xffffu) ? 1ull : 0ull) | ((mt >> 16) ? 2ull : 0ull);
                                hits |= two << (c8 + 2 * h);
                            }
                        }
                        if (ncnt < 64) hits &= (1ull << ncnt) - 1ull;
                        while (hits) {
                            const int e = __ffsll((long long)hits) - 1;
                            hits &= hits - 1ull;
                            const int code = nl[e], pa = code & 0xff, pb = code >> 8;
                            const bool fwd = pa == i;
                            nmask[rr] |= 1ull << (fwd ? pb : pa);
#pragma unroll
                            for (int a = 0; a < 3; ++a) Ri[a] += fwd ? ner[e * 3 + a] : -ner[e * 3 + a];
                        }
                    } else {
                        for (int j = 0; j < n; ++j) {   // warp-uniform: the near list is built with ballots
                            bool is_near = false;
                            if (iv && j != i) {
                                const T qn = pair_exact(j, true);
                                const bool zero = (sn[j] == ni[0]) || (sn[NB + j] == ni[1]) || (sn[2 * NB + j] == ni[2]);
                                if (qn < skin_lim) {
                                    is_near = i < j;
                                } else {
                                    farmin = fmin(farmin, qn);
                                    zfar = zfar || (!HY && zero);   // (HY: an interior pair's zero component does not block quiet steps)
                                }
                            }
                            const uint32_t bm = __ballot_sync(0xffffffffu, is_near);
                            if (bm) {
                                const int pos = nbase + __popc(bm & lanemask_lt);
                                if (is_near && pos < kNearCap) snear[(size_t)t * kNearCap + pos] = (uint16_t)(i | (j << 8));
                                nbase += __popc(bm);
                            }
                        }
                    }
                    if (iv) {   // workspace term of robot i
                        T dn[3], dd[3], r[3], x[3];
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            dn[a] = ni[a] - cen[a];
                            dd[a] = oi[a] - cen[a];
                        }
                        exact_term<T, false>(dn, dd, fw, r, x);
                        if constexpr (HY) {
                            if (r[0] != T(0) || r[1] != T(0) || r[2] != T(0)) {
                                const D3 r64 = large_term_r64<MP>(C, p.W + (size_t)t * m1, m1, n, i, -1, p.cx, p.cy, p.cz,
                                                                  family64(p, false));
                                r[0] = (T)r64.x;
                                r[1] = (T)r64.y;
                                r[2] = (T)r64.z;
                            }
                        }
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            Ri[a] += r[a];
                            linf = fmax(linf, fabs(x[a]));
                            lsq = fma((double)x[a], (double)x[a], lsq);
                        }
                    }
                    if (Ri[0] != T(0) || Ri[1] != T(0) || Ri[2] != T(0)) {
                        lact = true;
#pragma unroll
                        for (int a = 0; a < 3; ++a)
#pragma unroll
                            for (int q = 0; q < MP; ++q) gacc[rr][a][q] = fma_t<T>(Ri[a], w[q], gacc[rr][a][q]);
                    }
                }
#ifdef SGSF_LARGE_PT
                const long long lq3 = clock64();
#endif
                if (quiet) {   // far pairs: the O(n) statistics without the near pairs' share
                    T qinf_p = T(0), qsq_p = T(0);
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        qinf_p = fmax(qinf_p, hi[a] - lo[a]);
                        qsq_p += fmax(fma_t<T>((T)n, s2[a], -s1[a] * s1[a]), T(0));
                    }
                    const T nmax = warp_max_nonneg(nq_max);
                    T nsq = nq_sq;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, off);
                    T far_max = qinf_p;
#ifdef SGSF_LARGE_PT
                    const long long lqf0 = clock64();
#endif
                    if (nmax >= qinf_p) {   // a near pair attains the quiet max: the far max, exactly
                        // D p of every robot over the old-position scratch (dead for this step once the near
                        // pairs are done), the same rounding as the quiet statistics
                        T dpi[2][3];
#pragma unroll
                        for (int rr = 0; rr < 2; ++rr) {
                            const int i = lane + 32 * rr;
#pragma unroll
                            for (int a = 0; a < 3; ++a) dpi[rr][a] = sn[a * NB + i] - so[a * NB + i];
                        }
                        __syncwarp();
#pragma unroll
                        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                            for (int a = 0; a < 3; ++a) so[a * NB + lane + 32 * rr] = dpi[rr][a];
                        __syncwarp();
                        // every unordered pair once, 63 per lane: robot lane takes partners lane+1 .. lane+32,
                        // robot lane+32 takes lane+33 .. 63 and 0 .. lane-1
                        // fixed trip counts and selects instead of early returns, so the loads pipeline (the
                        // branchy form took ~8.4K cycles, 12% of quiet steps); max is exact in any order
                        T fa = T(0), fb = T(0);
                        const bool v0 = lane < n, v1 = lane + 32 < n;
#pragma unroll 8
                        for (int jj = 1; jj <= 32; ++jj) {   // robot lane: partners lane + 1 .. lane + 32
                            const int j = lane + jj;
                            const bool ok = v0 && j < n && !((nmask[0] >> j) & 1ull);
                            T m = T(0);
#pragma unroll
                            for (int a = 0; a < 3; ++a) m = fmax(m, fabs(dpi[0][a] - so[a * NB + j]));
                            if (jj & 1) fa = fmax(fa, ok ? m : T(0));
                            else fb = fmax(fb, ok ? m : T(0));
                        }
#pragma unroll 8
                        for (int jj = 1; jj <= 31; ++jj) {   // robot lane + 32: partners lane + 33 .. 63, 0 .. lane - 1
                            const int j = (lane + 32 + jj) & 63;
                            const bool ok = v1 && j < n && !((nmask[1] >> j) & 1ull);
                            T m = T(0);
#pragma unroll
                            for (int a = 0; a < 3; ++a) m = fmax(m, fabs(dpi[1][a] - so[a * NB + j]));
                            if (jj & 1) fa = fmax(fa, ok ? m : T(0));
                            else fb = fmax(fb, ok ? m : T(0));
                        }
                        const T fm = fmax(fa, fb);
                        far_max = warp_max_nonneg(fm);
#ifdef SGSF_LARGE_PT
                        if (blockIdx.x == 0 && warp == 0 && lane == 0) {
                            lqa[5] += 1;
                            lqa[6] += clock64() - lqf0;
                        }
#endif
                    }
                    if (lane == 0) {
                        scum[t] = cum_t;
                        linf = fmax(linf, far_max);
                        lsq += (double)fmax(qsq_p - nsq, T(0));
                    }
                } else {   // refresh the step's state from the exact pass
                    const T qm = warp_min_nonneg(farmin);
                    const bool zf = __any_sync(0xffffffffu, zfar);
                    if (lane == 0) {
                        srmin[t] = sqrt(qm) * inv_lat;
                        scum[t] = T(0);
                        sflag[t] = zf ? 0 : 1;
                        sncnt[t] = nbase <= kNearCap ? nbase : -1;
                    }
                }
                __syncwarp();   // the scratch is rewritten for the next step
#ifdef SGSF_LARGE_PT
                if (!quiet) lpt_exc += clock64() - lpt_s0;
                if (quiet && blockIdx.x == 0 && warp == 0 && lane == 0) {
                    lqa[0] += lq1 - lq0;
                    lqa[1] += lq2 - lq1;
                    lqa[2] += lq3 - lq2;
                    lqa[7] += lq2b - lq2;
                    lqa[3] += clock64() - lq3;
                    lqa[4] += 1;
                }
#endif
            }
            // ---------------- phase B: the exact steps of this iteration, in ascending order, each taken by all
            // eight warps at once (warp u: partners 8u .. 8u + 7 of every robot; warp 0 also the workspace
            // terms).  A step's partial R rows, near sublists and far minima go to double-buffered shared
            // memory; after a barrier warp e % 8 combines them in warp order (R into its g accumulators, the
            // near list in the serial pass's (robot half, partner, lane) order) while the others start the
            // next step.  An exact pass costs ~93K cycles on one warp, and an iteration has fewer of them than
            // warps, so the serial pass left seven warps waiting.
            if (kCoopExact) {
                __syncthreads();   // every warp's deferred steps are marked
#ifdef SGSF_LARGE_PT
                const long long lpt_b0 = clock64();
#endif
                int e = 0;
                for (int base = 0; base < S; base += 32) {
                    uint32_t bal = __ballot_sync(0xffffffffu, base + lane < S && sdefer[base + lane] != 0);
                    while (bal) {
                        const int t = base + __ffs(bal) - 1;
                        bal &= bal - 1;
                        const int buf = e & 1;
                        {   // this warp's partners of step t
                            T w[MP];
                            load_row16<T, MP>(Wt + t * MP, w);
#pragma unroll
                            for (int rr = 0; rr < 2; ++rr) {
                                const int i = lane + 32 * rr;
#pragma unroll
                                for (int a = 0; a < 3; ++a) {
                                    T pn = T(0), po = T(0);
#pragma unroll
                                    for (int q = 0; q < MP; ++q) {
                                        pn = fma_t<T>(Cf[(a * MP + q) * NB + i], w[q], pn);
                                        po = fma_t<T>(Cfo[(a * MP + q) * NB + i], w[q], po);
                                    }
                                    sn[a * NB + i] = pn;
                                    so[a * NB + i] = po;
                                }
                            }
                            __syncwarp();
                            const int j0 = 8 * warp, j1 = min(j0 + 8, n);
                            T farmin = T(1e30);
                            bool zfar = false;
#pragma unroll
                            for (int rr = 0; rr < 2; ++rr) {
                                const int i = lane + 32 * rr;
                                const bool iv = i < n;
                                T Ri[3] = {T(0), T(0), T(0)};
                                T ni[3], oi[3];
#pragma unroll
                                for (int a = 0; a < 3; ++a) {
                                    ni[a] = sn[a * NB + i];
                                    oi[a] = so[a * NB + i];
                                }
                                int nb = 0;
                                for (int j = j0; j < j1; ++j) {   // warp-uniform: the near sublist is built with ballots
                                    bool is_near = false;
                                    if (iv && j != i) {
                                        const bool fwd = i < j;
                                        T dn[3], dd[3], r[3], x[3];
#pragma unroll
                                        for (int a = 0; a < 3; ++a) {
                                            const T nj = sn[a * NB + j], oj = so[a * NB + j];
                                            dn[a] = fwd ? ni[a] - nj : nj - ni[a];
                                            dd[a] = fwd ? oi[a] - oj : oj - oi[a];
                                        }
                                        exact_term<T, true>(dn, dd, fp, r, x);
                                        if constexpr (HY) {   // not interior under the guarded FP32 test: R from FP64
                                            if (r[0] != T(0) || r[1] != T(0) || r[2] != T(0)) {
                                                const D3 r64 = large_term_r64<MP>(C, p.W + (size_t)t * m1, m1, n, fwd ? i : j,
                                                                                  fwd ? j : i, p.cx, p.cy, p.cz, family64(p, true));
                                                r[0] = (T)r64.x;
                                                r[1] = (T)r64.y;
                                                r[2] = (T)r64.z;
                                            }
                                        }
#pragma unroll
                                        for (int a = 0; a < 3; ++a) Ri[a] += fwd ? r[a] : -r[a];
                                        if (fwd) {
#pragma unroll
                                            for (int a = 0; a < 3; ++a) {
                                                linf = fmax(linf, fabs(x[a]));
                                                lsq = fma((double)x[a], (double)x[a], lsq);
                                            }
                                        }
                                        const T qn = fma_t<T>(dn[2] * fp.beta, dn[2], fma_t<T>(dn[1], dn[1], dn[0] * dn[0]));
                                        const bool zero = (sn[j] == ni[0]) || (sn[NB + j] == ni[1]) || (sn[2 * NB + j] == ni[2]);
                                        if (qn < skin_lim) {
                                            is_near = i < j;
                                        } else {
                                            farmin = fmin(farmin, qn);
                                            zfar = zfar || (!HY && zero);   // (HY: an interior pair's zero component does not block quiet steps)
                                        }
                                    }
                                    const uint32_t bm = __ballot_sync(0xffffffffu, is_near);
                                    if (bm) {
                                        const int pos = nb + __popc(bm & lanemask_lt);
                                        if (is_near && pos < kNearCap)
                                            xnl[((buf * kLargeWarps + warp) * 2 + rr) * kNearCap + pos] = (uint16_t)(i | (j << 8));
                                        nb += __popc(bm);
                                    }
                                }
                                if (warp == 0 && iv) {   // workspace term of robot i
                                    T dn[3], dd[3], r[3], x[3];
#pragma unroll
                                    for (int a = 0; a < 3; ++a) {
                                        dn[a] = ni[a] - cen[a];
                                        dd[a] = oi[a] - cen[a];
                                    }
                                    exact_term<T, false>(dn, dd, fw, r, x);
                                    if constexpr (HY) {
                                        if (r[0] != T(0) || r[1] != T(0) || r[2] != T(0)) {
                                            const D3 r64 = large_term_r64<MP>(C, p.W + (size_t)t * m1, m1, n, i, -1, p.cx, p.cy,
                                                                              p.cz, family64(p, false));
                                            r[0] = (T)r64.x;
                                            r[1] = (T)r64.y;
                                            r[2] = (T)r64.z;
                                        }
                                    }
#pragma unroll
                                    for (int a = 0; a < 3; ++a) {
                                        Ri[a] += r[a];
                                        linf = fmax(linf, fabs(x[a]));
                                        lsq = fma((double)x[a], (double)x[a], lsq);
                                    }
                                }
#pragma unroll
                                for (int a = 0; a < 3; ++a)
                                    xr[(((buf * kLargeWarps + warp) * 2 + rr) * 32 + lane) * 3 + a] = Ri[a];
                                if (lane == 0) xcnt[(buf * kLargeWarps + warp) * 2 + rr] = nb;
                            }
                            const T qm = warp_min_nonneg(farmin);
                            const bool zf = __any_sync(0xffffffffu, zfar);
                            if (lane == 0) {
                                xfm[buf * kLargeWarps + warp] = qm;
                                xzf[buf * kLargeWarps + warp] = zf ? 1 : 0;
                            }
                            __syncwarp();   // the scratch is rewritten for the next step
                        }
                        __syncthreads();   // step t's partials are complete
                        if (warp == (e & (kLargeWarps - 1))) {   // combine them, in warp order
                            T w[MP];
                            load_row16<T, MP>(Wt + t * MP, w);
#pragma unroll
                            for (int rr = 0; rr < 2; ++rr) {
                                T Ri[3] = {T(0), T(0), T(0)};
#pragma unroll
                                for (int u = 0; u < kLargeWarps; ++u)
#pragma unroll
                                    for (int a = 0; a < 3; ++a) Ri[a] += xr[(((buf * kLargeWarps + u) * 2 + rr) * 32 + lane) * 3 + a];
                                if (Ri[0] != T(0) || Ri[1] != T(0) || Ri[2] != T(0)) {
                                    lact = true;
#pragma unroll
                                    for (int a = 0; a < 3; ++a)
#pragma unroll
                                        for (int q = 0; q < MP; ++q) gacc[rr][a][q] = fma_t<T>(Ri[a], w[q], gacc[rr][a][q]);
                                }
                            }
                            int total = 0;   // the near list: (robot half, warp) sublists in order, up to kNearCap
#pragma unroll
                            for (int rr = 0; rr < 2; ++rr) {
                                for (int u = 0; u < kLargeWarps; ++u) {
                                    const int c = xcnt[(buf * kLargeWarps + u) * 2 + rr];
                                    for (int q = lane; q < c && q < kNearCap; q += 32)
                                        if (total + q < kNearCap)
                                            snear[(size_t)t * kNearCap + total + q] =
                                                xnl[((buf * kLargeWarps + u) * 2 + rr) * kNearCap + q];
                                    total += c;
                                }
                            }
                            T qm = T(1e30);
                            int zf = 0;
                            for (int u = 0; u < kLargeWarps; ++u) {
                                qm = fmin(qm, xfm[buf * kLargeWarps + u]);
                                zf |= xzf[buf * kLargeWarps + u];
                            }
                            if (lane == 0) {   // refresh the step's state from the exact pass
                                srmin[t] = sqrt(qm) * inv_lat;
                                scum[t] = T(0);
                                sflag[t] = zf ? 0 : 1;
                                sncnt[t] = total <= kNearCap ? total : -1;
                                sdefer[t] = 0;
                            }
                        }
                        ++e;
                    }
                }
#ifdef SGSF_LARGE_PT
                lpt_exc += clock64() - lpt_b0;
#endif
            }
            // per-warp partials of the exit norm, fixed order
            {
                const T wi = warp_max_nonneg(linf);
                double wq = lsq;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) wq += __shfl_xor_sync(0xffffffffu, wq, off);
                if (lane == 0) {
                    winf[warp] = wi;
                    wsq[warp] = wq;
                }
            }
            // the term-pass scratch aliased on g is cleared before g accumulates (after every warp is done with it)
            __syncthreads();
            for (int e = tid; e < (int)L.gwords; e += nt) g[e] = 0.0;
            __syncthreads();
            // g = sum over the warps of their partial R W, in warp order
            {
                const bool wact = __any_sync(0xffffffffu, lact);
                const int ticket = k * kLargeWarps + warp;
#ifdef SGSF_LARGE_PT
                if (lane == 0) {
                    lpt_dur[warp] = clock64() - lpt0;
                    lpt_ex[warp] = lpt_nex;
                    lpt_exq[warp] = lpt_exc;
                }
#endif
                if (lane == 0)
                    while (*(volatile int*)&sh->g_ticket != ticket) __nanosleep(32);
                __syncwarp();
                __threadfence_block();
                if (wact) {
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        const int i = lane + 32 * rr;
                        if (i < n) {
#pragma unroll
                            for (int a = 0; a < 3; ++a)
#pragma unroll
                                for (int q = 0; q < MP; ++q) g[((a * n) + i) * MP + q] += (double)gacc[rr][a][q];
                        }
                    }
                    if (lane == 0) sh->active[par] = 1;
                }
                __threadfence_block();
                __syncwarp();
                if (lane == 0) *(volatile int*)&sh->g_ticket = ticket + 1;
            }
            __syncthreads();
#ifdef SGSF_LARGE_PT
            if (tid == 0) {
                long long mx = 0, sm = 0, qm = 0, exc = 0;
                int exm = 0, exs = 0;
                for (int w = 0; w < kLargeWarps; ++w) {
                    mx = max(mx, lpt_dur[w]);
                    sm += lpt_dur[w];
                    exm = max(exm, lpt_ex[w]);
                    exs += lpt_ex[w];
                    qm = max(qm, lpt_dur[w] - lpt_exq[w]);
                    exc += lpt_exq[w];
                }
                lpt_qmax += (double)qm;
                lpt_excyc += (double)exc;
                lpt_max += (double)mx;
                lpt_mean += (double)sm / kLargeWarps;
                lpt_exmax += exm;
                lpt_exmean += (double)exs / kLargeWarps;
            }
#endif

            // ---------------- decision (every thread): exit residual of iteration k-1, early stop, SingularKKT
            double emax = 0.0, sqs = 0.0;
            T inf = T(0);
            if (k >= 1) {
                emax = fmax(fmax(eqerr[0], eqerr[1]), eqerr[2]);
                for (int w = 0; w < kLargeWarps; ++w) {
                    inf = fmax(inf, winf[w]);
                    sqs += wsq[w];
                }
            }
            double infd = (double)inf;
            if constexpr (HY) {   // near tol: the exit residual in FP64 (block-uniform: every thread read the same)
                if (k >= 1 && p.early_stop && fabs(infd - p.tol_res) <= p.hy_delta) {
                    LargeExitArgs xa;
                    xa.W = p.W;
                    xa.n = n;
                    xa.S = S;
                    xa.m1 = m1;
                    xa.cx = p.cx;
                    xa.cy = p.cy;
                    xa.cz = p.cz;
                    xa.fp = family64(p, true);
                    xa.fw = family64(p, false);
                    const double2 e = large_exit64<MP>(xa, C, Cp, warp, lane);
                    __syncthreads();   // every thread has read winf / wsq
                    if (lane == 0) {
                        winf64[warp] = e.x;
                        wsq[warp] = e.y;
                    }
                    __syncthreads();
                    infd = 0.0;
                    sqs = 0.0;
                    for (int w = 0; w < kLargeWarps; ++w) {
                        infd = fmax(infd, winf64[w]);
                        sqs += wsq[w];
                    }
                }
            }
            const bool failed = (k >= 1) && (emax > p.tol_eq);
            bool done = failed;
            if (k >= 1) {
                done = done || (p.early_stop && infd <= p.tol_res) || (k >= p.max_iters);
                if (tid == 0) {
                    const size_t hix = (size_t)sample * p.max_iters + (k - 1);
                    p.res_inf[hix] = infd;
                    p.res_l2[hix] = sqrt(sqs);
                }
            }
            if (done) {
                // ---------------- finalize: outputs of the returned iterate, claim the next sample
                if (!failed) {
                    for (int e = tid; e < dim; e += nt) {
                        const int r = e / m1, q = e - r * m1;
                        const size_t o = (size_t)sample * dim + e;
                        p.coeffs[o] = C[r * MP + q];
                        p.mult[o] = lam[r * MP + q];
                        if (p.want_prev && p.coeffs_prev) p.coeffs_prev[o] = Cp[r * MP + q];
                    }
                }
                if (warp == 0) {
                    double acc = 0.0;
                    for (int e = lane; e < dimp; e += 32) {
                        const double dd = C[e] - xb[e];
                        acc = fma(dd, dd, acc);
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    if (lane == 0) {
                        p.iterations[sample] = failed ? 0 : k;
                        p.converged[sample] = (!failed && infd <= p.tol_res) ? 1 : 0;
                        p.displacement[sample] = failed ? CUDART_NAN : sqrt(acc);
                        p.status[sample] = failed ? SAMPLE_SINGULAR_KKT : SAMPLE_OK;
                        p.eq_err[sample] = emax;
#ifdef SGSF_LARGE_PT
                        if (blockIdx.x == 0 && lqa[4])
                            printf("LQ quiet steps %lld: positions %lld statistics %lld near+ws %lld far %lld cycles each; far-max fallback %lld times, %lld cycles each; near stage 1 %lld\n", lqa[4],
                                   lqa[0] / lqa[4], lqa[1] / lqa[4], lqa[2] / lqa[4], lqa[3] / lqa[4], lqa[5], lqa[5] ? lqa[6] / lqa[5] : 0, lqa[7] / lqa[4]);
                        if (blockIdx.x < 4)
                            printf("LPT cta %d sample %d iters %d term-pass cycles: slowest warp %.0f mean %.0f slowest-without-exact %.0f | exact steps per warp: max %.2f mean %.2f, exact-step cycles per iteration (all warps) %.0f\n",
                                   blockIdx.x, sample, k, lpt_max / (k + 1), lpt_mean / (k + 1), lpt_qmax / (k + 1), lpt_exmax / (k + 1),
                                   lpt_exmean / (k + 1), lpt_excyc / (k + 1));
                        if (blockIdx.x < 4) printf("LMX cta %d: xi-step phase %lld cycles per iteration\n", blockIdx.x, lmx / (k + 1));
                        lmx = 0;
                        lpt_max = lpt_mean = lpt_exmax = lpt_exmean = lpt_qmax = lpt_excyc = 0;
#endif
                        sh->sample = next_sample(p);
                        sh->active[0] = sh->active[1] = 0;
                    }
                }
                __syncthreads();
                sample = sh->sample;
                break;
            }
            const bool any_active = sh->active[par] != 0;

            // ---------------- U = 2 lam' - lam + xi_bar (lam' = lam - rho g), element-wise
            if (any_active || prev_active || k == 0) {
                for (int e = tid; e < dimp; e += nt) {
                    const double l = lam[e];
                    const double lp = any_active ? l - p.rho * g[e] : l;
                    U[e] = 2.0 * lp - l + xb[e];
                }
            }
            __syncthreads();

#ifdef SGSF_LARGE_PT
            const long long lmx0 = clock64();
#endif
            // ---------------- xi-step per axis (K1's DMMA formulation), equality check, commit
            const int fr = lane >> 2, fc = lane & 3;
            for (int ax = warp; ax < 3; ax += kLargeWarps) {
                const int rb = ax * n;
                double dacc[MT][2][2];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int rob = 8 * mt + fr;
#pragma unroll
                    for (int nt2 = 0; nt2 < 2; ++nt2)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int q = 8 * nt2 + 2 * fc + e;
                            dacc[mt][nt2][e] = (rob < n && q < MP) ? cconst[(rb + rob) * MP + q] : 0.0;
                        }
                }
                double csum[KT];
#pragma unroll
                for (int kk = 0; kk < KT; ++kk) {
                    const int c = 4 * kk + fc;
                    double bf[2];
#pragma unroll
                    for (int nt2 = 0; nt2 < 2; ++nt2) {
                        const int qb = 8 * nt2 + fr;
                        bf[nt2] = qb < MP ? KMd[qb * M2P + c] : 0.0;
                    }
                    csum[kk] = 0.0;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const int rob = 8 * mt + fr;
                        const double a = rob < n ? (kk < KC ? C[(rb + rob) * MP + c] : U[(rb + rob) * MP + c - MP]) : 0.0;
                        csum[kk] += a;
#pragma unroll
                        for (int nt2 = 0; nt2 < 2; ++nt2) dmma884(dacc[mt][nt2][0], dacc[mt][nt2][1], a, bf[nt2]);
                    }
                }
                {   // mean part: every row gets (column sums / n) . [Mm - Md | Km11 - Kd11]^T
                    double dm[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                    for (int kk = 0; kk < KT; ++kk) {
                        double cs = csum[kk];
                        cs += __shfl_xor_sync(0xffffffffu, cs, 4);
                        cs += __shfl_xor_sync(0xffffffffu, cs, 8);
                        cs += __shfl_xor_sync(0xffffffffu, cs, 16);
                        const int c = 4 * kk + fc;
                        const double a = cs * inv_n;
#pragma unroll
                        for (int nt2 = 0; nt2 < 2; ++nt2) {
                            const int qb = 8 * nt2 + fr;
                            dmma884(dm[nt2][0], dm[nt2][1], a, qb < MP ? KMm[qb * M2P + c] : 0.0);
                        }
                    }
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int nt2 = 0; nt2 < 2; ++nt2) {
                            dacc[mt][nt2][0] += dm[nt2][0];
                            dacc[mt][nt2][1] += dm[nt2][1];
                        }
                }
                if (p.want_prev || HY) {
                    for (int e = lane; e < n * MP; e += 32) Cp[rb * MP + e] = C[rb * MP + e];
                }
                for (int e = lane; e < MP * NB; e += 32) Cfo[ax * MP * NB + e] = Cf[ax * MP * NB + e];
                __syncwarp();   // every lane has read the rows before any lane writes them
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int rob = 8 * mt + fr;
#pragma unroll
                    for (int nt2 = 0; nt2 < 2; ++nt2) {
                        const int q = 8 * nt2 + 2 * fc;
                        if (rob < n && q < MP) {
                            const int idx = (rb + rob) * MP + q;
                            *reinterpret_cast<double2*>(C + idx) = make_double2(dacc[mt][nt2][0], dacc[mt][nt2][1]);
                            Cf[(ax * MP + q) * NB + rob] = (T)dacc[mt][nt2][0];
                            Cf[(ax * MP + q + 1) * NB + rob] = (T)dacc[mt][nt2][1];
                        }
                    }
                }
                if (any_active) {   // commit lam', clear g
                    for (int e = lane; e < n * MP; e += 32) {
                        const int idx = rb * MP + e;
                        lam[idx] = lam[idx] - p.rho * g[idx];
                        g[idx] = 0.0;
                    }
                }
                __syncwarp();
                {   // ||A xi - b||_inf over this axis' new rows
                    double eacc[MT][2];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const int rob = 8 * mt + fr;
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int c6 = 2 * fc + e;
                            eacc[mt][e] = (rob < n && c6 < 6) ? -rhs[(rb + rob) * 6 + c6] : 0.0;
                        }
                    }
#pragma unroll
                    for (int kk = 0; kk < MP / 4; ++kk) {
                        const int q = 4 * kk + fc;
                        const double bv = fr < 6 ? B6[fr * MP + q] : 0.0;
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const int rob = 8 * mt + fr;
                            const double a = rob < n ? C[(rb + rob) * MP + q] : 0.0;
                            dmma884(eacc[mt][0], eacc[mt][1], a, bv);
                        }
                    }
                    double em = 0.0;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) em = fmax(em, fmax(fabs(eacc[mt][0]), fabs(eacc[mt][1])));
                    em = warp_max_nonneg(em);
                    if (lane == 0) eqerr[ax] = em;
                }
            }
            prev_active = any_active;
#ifdef SGSF_LARGE_PT
            if (tid == 0) lmx += clock64() - lmx0;
#endif
            __syncthreads();
        }
    }
}

}  // namespace sgsf
