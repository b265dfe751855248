// sf_persistent.cuh -- K1: the whole safety-filter iteration loop on-chip.
//
// Replaces SafetyFilter.batch_solve -> solve (solver.py:286-407) including
// the spherical kernel (_speedups.pyx:18-73), F^T (assembly.py:296-303), the
// LU xi-step (assembly.py:186-219) and the boundary projection prologue
// (projection.py:11-25).
//
// Persistent CTAs, one resident CTA per SM.  A CTA owns `spb` sample SLOTS;
// a slot pulls the next sample index from a global atomic queue whenever its
// sample finishes, so per-sample iteration-count skew never idles a slot.
//
// Thread layout in the term phase: thread (slot, t) owns time step t of its
// slot's sample for ALL robots; the sampled positions of every robot at t live
// in its registers, so the O(n^2) pair work needs no shared-memory traffic and
// the scatter F^T is a register accumulation in a fixed order (deterministic,
// no atomics).  Each round of the CTA runs five phases separated by barriers:
//
//   T  positions  p_k(t) = C_k W[t]^T                       (term precision)
//      for every pair / workspace term:  targets e_k = proj(d_k),
//        residual r_k = d_k - e_k scattered into R(t);
//        exit residual of iteration k-1:  d_k - proj(d_{k-1})  -> max / sum sq
//   G  lam'  = lam - rho R W            (W^T projection, 2 t-halves per row)
//      one warp per slot: history, early-stop / SingularKKT decision
//   M  finished slots: write outputs, claim next sample;  others: C_bar, u_bar
//   M2 mean part  Mm C_bar + Km11 u_bar;  freshly claimed slots: load + project
//   X  xi-step  C_i = mean part + Md (C_i - C_bar) + Kd11 (u_i - u_bar) + cconst_i,
//      ||A xi - b||_inf check, lam <- lam'
//
// u = 2 lam' - lam + xi_bar (residual identity, precompute.py).  State (C,
// lam, xi_bar) and the xi-step are FP64; T is float ("lean") or double
// ("strict") for positions, term math and the W^T projection.
#pragma once

#include "sf_device.cuh"

namespace sgsf {

enum { SLOT_EMPTY = 0, SLOT_ACTIVE = 1 };
enum { SAMPLE_OK = 0, SAMPLE_SINGULAR_KKT = 1 };

struct SlotState {
    int sample;
    int k;       // xi-steps taken so far
    int state;
    int pad;
};

struct SlotScratch {   // phase-to-phase messages within one round
    int done;
    int failed;
    int pending;
    int pad;
    double last_inf;
    double eqmax;
};

struct SolveParams {
    int n, S, m1, MP, batch, max_iters, early_stop, want_prev, spb;
    double rho, tol_res, tol_eq;
    double lat, vert, ws_lat, ws_vert, cx, cy, cz;
    const double* W;       // S x m1
    const double* KMm;     // m1 x 2m1  [Mm | Km11]
    const double* KMd;     // m1 x 2m1  [Md | Kd11]
    const double* cconst;  // 3n x m1
    const double* B6;      // 6 x m1
    const double* rhs;     // 3n x 6
    const double* PBt;     // m1 x 6
    const double* xi_bar;
    const double* xi0;
    const double* lam0;
    const uint8_t* init_mode;
    double* coeffs;
    double* mult;
    double* res_inf;
    double* res_l2;
    int* iterations;
    uint8_t* converged;
    double* displacement;
    int* status;
    double* eq_err;
    double* coeffs_prev;
    int* queue;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct SmemLayout {
    size_t W, KMm, KMd, cconst, B6, rhs, PBt, st0, st1, sc;
    size_t slot0, slot_stride;
    size_t C, Cp, lam, lamN, xb, means, mpart, eqerr, psq, R, posold, Cf, pinf;
    size_t total;
};

template <typename T, int NB>
__host__ __device__ inline SmemLayout make_layout(int n, int S, int m1, int MP, int spb, int want_prev) {
    const int RS = 3 * NB + 1;
    SmemLayout L;
    size_t o = 0;
    const size_t d = sizeof(double), ts = sizeof(T);
    const int R3 = 3 * n, dim = R3 * m1;
    L.W = o;      o = align16(o + (size_t)S * MP * ts);
    L.KMm = o;    o = align16(o + (size_t)m1 * 2 * m1 * d);
    L.KMd = o;    o = align16(o + (size_t)m1 * 2 * m1 * d);
    L.cconst = o; o = align16(o + (size_t)dim * d);
    L.B6 = o;     o = align16(o + (size_t)6 * m1 * d);
    L.rhs = o;    o = align16(o + (size_t)R3 * 6 * d);
    L.PBt = o;    o = align16(o + (size_t)m1 * 6 * d);
    L.st0 = o;    o = align16(o + (size_t)spb * sizeof(SlotState));
    L.st1 = o;    o = align16(o + (size_t)spb * sizeof(SlotState));
    L.sc = o;     o = align16(o + (size_t)spb * sizeof(SlotScratch));
    L.slot0 = o;
    size_t q = 0;
    L.C = q;      q = align16(q + (size_t)dim * d);
    L.Cp = q;     q = align16(q + (want_prev ? (size_t)dim * d : 0));
    L.lam = q;    q = align16(q + (size_t)dim * d);
    L.lamN = q;   q = align16(q + (size_t)dim * d);
    L.xb = q;     q = align16(q + (size_t)dim * d);
    L.means = q;  q = align16(q + (size_t)6 * m1 * d);
    L.mpart = q;  q = align16(q + (size_t)3 * m1 * d);
    L.eqerr = q;  q = align16(q + (size_t)R3 * d);
    L.psq = q;    q = align16(q + (size_t)S * d);
    L.R = q;      q = align16(q + (size_t)RS * S * ts);
    L.posold = q; q = align16(q + (size_t)RS * S * ts);
    L.Cf = q;     q = align16(q + (size_t)R3 * MP * ts);
    L.pinf = q;   q = align16(q + (size_t)S * ts);
    L.slot_stride = q;
    L.total = o + (size_t)spb * q;
    return L;
}

constexpr int KMAX = 16;   // max degree + 1 handled by the register-unrolled loops

struct SlotPtrs {
    double *C, *Cp, *lam, *lamN, *xb, *means, *mpart, *eqerr, *psq;
    void *R, *posold, *Cf, *pinf;
};

__device__ __forceinline__ SlotPtrs slot_ptrs(unsigned char* smem, const SmemLayout& L, int s) {
    unsigned char* b = smem + L.slot0 + (size_t)s * L.slot_stride;
    SlotPtrs P;
    P.C = (double*)(b + L.C);
    P.Cp = (double*)(b + L.Cp);
    P.lam = (double*)(b + L.lam);
    P.lamN = (double*)(b + L.lamN);
    P.xb = (double*)(b + L.xb);
    P.means = (double*)(b + L.means);
    P.mpart = (double*)(b + L.mpart);
    P.eqerr = (double*)(b + L.eqerr);
    P.psq = (double*)(b + L.psq);
    P.R = (void*)(b + L.R);
    P.posold = (void*)(b + L.posold);
    P.Cf = (void*)(b + L.Cf);
    P.pinf = (void*)(b + L.pinf);
    return P;
}

// ---------------------------------------------------------------- T phase
// Per-thread buffers R (scattered residual) and posold (positions of the
// previous iterate) are [t][RS] with RS = 3 NB + 1: thread t touches only
// its own row, at compile-time offsets, and the odd row stride keeps the
// warp's accesses on distinct banks.
template <int NB> struct RowStride { static constexpr int value = 3 * NB + 1; };

// Returns false (and writes nothing) when the fast pass met an exactly-zero
// component; the caller then reruns the time step with CAREFUL = true.
template <typename T, int NB, bool CAREFUL>
__device__ __forceinline__ bool term_pass(const SolveParams& p, const T* __restrict__ Wt, const SlotPtrs& sp,
                                          int k, int t, const Family<T>& fp, const Family<T>& fw,
                                          T cx, T cy, T cz) {
    constexpr int RS = RowStride<NB>::value;
    const int n = p.n, MP = p.MP;
    const T* Cf = (const T*)sp.Cf;
    T* Rrow = (T*)sp.R + t * RS;
    T* Orow = (T*)sp.posold + t * RS;

    T pos[3 * NB];
    {
        T w[KMAX];
#pragma unroll
        for (int q = 0; q < KMAX; ++q) w[q] = (q < MP) ? Wt[t * MP + q] : T(0);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                T s = T(0);
                if (i < n) {
                    const T* c = Cf + (ax * n + i) * MP;
#pragma unroll
                    for (int q = 0; q < KMAX; ++q)
                        if (q < MP) s = fma_t<T>(c[q], w[q], s);
                }
                pos[ax * NB + i] = s;
            }
        }
    }
    // k == 0: no previous iterate; "old" := "new" (that exit residual is discarded).
    // Idempotent, so it is safe even if this fast pass is redone carefully.
    if (k == 0) {
#pragma unroll
        for (int q = 0; q < 3 * NB; ++q)
            if ((q % NB) < n) Orow[q] = pos[q];
    }

    T acc[3 * NB];
#pragma unroll
    for (int q = 0; q < 3 * NB; ++q) acc[q] = T(0);
    T inf = T(0), sq = T(0), zmin = T(1);

#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if (i < n) {
            const T pix = pos[i], piy = pos[NB + i], piz = pos[2 * NB + i];
            const T oix = Orow[i], oiy = Orow[NB + i], oiz = Orow[2 * NB + i];
#pragma unroll
            for (int j = i + 1; j < NB; ++j) {
                if (j < n) {
                    const T dx = pix - pos[j], dy = piy - pos[NB + j], dz = piz - pos[2 * NB + j];
                    T rx, ry, rz;
                    resid<T, true, CAREFUL>(dx, dy, dz, dx, dy, dz, fp, zmin, rx, ry, rz);
                    acc[i] += rx;
                    acc[NB + i] += ry;
                    acc[2 * NB + i] += rz;
                    acc[j] -= rx;
                    acc[NB + j] -= ry;
                    acc[2 * NB + j] -= rz;
                    const T ox = oix - Orow[j], oy = oiy - Orow[NB + j], oz = oiz - Orow[2 * NB + j];
                    T xx, xy, xz;
                    resid<T, true, CAREFUL>(ox, oy, oz, dx, dy, dz, fp, zmin, xx, xy, xz);
                    inf = fmax(inf, fmax(fabs(xx), fmax(fabs(xy), fabs(xz))));
                    sq = fma_t<T>(xx, xx, fma_t<T>(xy, xy, fma_t<T>(xz, xz, sq)));
                }
            }
            // workspace containment term of robot i
            const T rx = pix - cx, ry = piy - cy, rz = piz - cz;
            T ux, uy, uz;
            resid<T, false, CAREFUL>(rx, ry, rz, rx, ry, rz, fw, zmin, ux, uy, uz);
            acc[i] += ux;
            acc[NB + i] += uy;
            acc[2 * NB + i] += uz;
            T xx, xy, xz;
            resid<T, false, CAREFUL>(oix - cx, oiy - cy, oiz - cz, rx, ry, rz, fw, zmin, xx, xy, xz);
            inf = fmax(inf, fmax(fabs(xx), fmax(fabs(xy), fabs(xz))));
            sq = fma_t<T>(xx, xx, fma_t<T>(xy, xy, fma_t<T>(xz, xz, sq)));
        }
    }
    if (!CAREFUL && zmin == T(0)) return false;

#pragma unroll
    for (int q = 0; q < 3 * NB; ++q) {
        if ((q % NB) < n) {
            Rrow[q] = acc[q];
            Orow[q] = pos[q];
        }
    }
    ((T*)sp.pinf)[t] = inf;
    sp.psq[t] = (double)sq;
    return true;
}

// ---------------------------------------------------------------- load a claimed sample (one row)
__device__ __forceinline__ void load_row(const SolveParams& p, const SlotPtrs& sp, int sample, int r,
                                         const double* __restrict__ B6, const double* __restrict__ rhs,
                                         const double* __restrict__ PBt, bool is_float) {
    const int m1 = p.m1, dim = 3 * p.n * m1;
    const double* xr = p.xi_bar + (size_t)sample * dim + r * m1;
    double x[KMAX], c[KMAX], l[KMAX];
#pragma unroll
    for (int q = 0; q < KMAX; ++q) x[q] = (q < m1) ? xr[q] : 0.0;
    const int mode = p.init_mode ? p.init_mode[sample] : 0;
    if (mode) {
        const double* cr = p.xi0 + (size_t)sample * dim + r * m1;
        const double* lr = p.lam0 + (size_t)sample * dim + r * m1;
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
            c[q] = (q < m1) ? cr[q] : 0.0;
            l[q] = (q < m1) ? lr[q] : 0.0;
        }
    } else {
        double res[6];
#pragma unroll
        for (int cnd = 0; cnd < 6; ++cnd) {
            double e = 0.0;
#pragma unroll
            for (int q = 0; q < KMAX; ++q)
                if (q < m1) e = fma(B6[cnd * m1 + q], x[q], e);
            res[cnd] = e - rhs[r * 6 + cnd];
        }
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
            double corr = 0.0;
#pragma unroll
            for (int cnd = 0; cnd < 6; ++cnd)
                if (q < m1) corr = fma(PBt[q * 6 + cnd], res[cnd], corr);
            c[q] = x[q] - corr;
            l[q] = 0.0;
        }
    }
#pragma unroll
    for (int q = 0; q < KMAX; ++q) {
        if (q < m1) {
            const int idx = r * m1 + q;
            sp.xb[idx] = x[q];
            sp.C[idx] = c[q];
            sp.lam[idx] = l[q];
            if (p.want_prev) sp.Cp[idx] = c[q];
        }
        if (q < p.MP) {
            if (is_float) ((float*)sp.Cf)[r * p.MP + q] = (q < m1) ? (float)c[q] : 0.f;
            else ((double*)sp.Cf)[r * p.MP + q] = (q < m1) ? c[q] : 0.0;
        }
    }
}

// ---------------------------------------------------------------- the kernel
template <typename T, int NB, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) sf_persistent_kernel(const SolveParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLayout L = make_layout<T, NB>(p.n, p.S, p.m1, p.MP, p.spb, p.want_prev);
    constexpr int RS = RowStride<NB>::value;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const int n = p.n, S = p.S, m1 = p.m1, MP = p.MP, spb = p.spb;
    const int R3 = 3 * n, dim = R3 * m1, m2 = 2 * m1;
    const bool is_float = sizeof(T) == 4;

    T* Wt = (T*)(smem + L.W);
    double* KMm = (double*)(smem + L.KMm);
    double* KMd = (double*)(smem + L.KMd);
    double* cconst = (double*)(smem + L.cconst);
    double* B6 = (double*)(smem + L.B6);
    double* rhs = (double*)(smem + L.rhs);
    double* PBt = (double*)(smem + L.PBt);
    SlotState* st[2] = {(SlotState*)(smem + L.st0), (SlotState*)(smem + L.st1)};
    SlotScratch* sc = (SlotScratch*)(smem + L.sc);

    for (int i = tid; i < S * MP; i += nt) {
        const int t = i / MP, q = i % MP;
        Wt[i] = (q < m1) ? (T)p.W[t * m1 + q] : T(0);
    }
    for (int i = tid; i < m1 * m2; i += nt) {
        KMm[i] = p.KMm[i];
        KMd[i] = p.KMd[i];
    }
    for (int i = tid; i < dim; i += nt) cconst[i] = p.cconst[i];
    for (int i = tid; i < 6 * m1; i += nt) B6[i] = p.B6[i];
    for (int i = tid; i < R3 * 6; i += nt) rhs[i] = p.rhs[i];
    for (int i = tid; i < m1 * 6; i += nt) PBt[i] = p.PBt[i];
    if (tid < spb) {
        sc[tid].pending = atomicAdd(p.queue, 1);
        sc[tid].done = 1;
    }
    __syncthreads();
    for (int it = tid; it < spb * R3; it += nt) {
        const int s = it / R3, r = it % R3;
        if (sc[s].pending < p.batch) load_row(p, slot_ptrs(smem, L, s), sc[s].pending, r, B6, rhs, PBt, is_float);
    }
    if (tid < spb) {
        SlotState z;
        z.sample = sc[tid].pending;
        z.k = 0;
        z.state = (z.sample < p.batch) ? SLOT_ACTIVE : SLOT_EMPTY;
        z.pad = 0;
        st[0][tid] = z;
    }
    __syncthreads();

    const int my_slot = tid / S, my_t = tid - (tid / S) * S;
    const bool term_thread = tid < spb * S;
    const Family<T> fp = make_family<T>(p.lat, p.vert);
    const Family<T> fw = make_family<T>(p.ws_lat, p.ws_vert);
    const T cx = (T)p.cx, cy = (T)p.cy, cz = (T)p.cz;
    const int half = (S + 1) / 2;

    for (int round = 0;; ++round) {
        const SlotState* cur = st[round & 1];
        SlotState* nxt = st[(round + 1) & 1];
        bool any = false;
        for (int s = 0; s < spb; ++s) any |= (cur[s].state == SLOT_ACTIVE);
        if (!any) break;

        // ---------------- T: term pass
        if (term_thread && cur[my_slot].state == SLOT_ACTIVE) {
            const SlotPtrs sp = slot_ptrs(smem, L, my_slot);
            const int k = cur[my_slot].k;
            if (!term_pass<T, NB, false>(p, Wt, sp, k, my_t, fp, fw, cx, cy, cz))
                term_pass<T, NB, true>(p, Wt, sp, k, my_t, fp, fw, cx, cy, cz);
        }
        __syncthreads();

        // ---------------- G: lam' = lam - rho R W   and the per-slot decision
        {
            const int nitems = spb * R3 * 2;
            for (int it0 = 0; it0 < nitems; it0 += nt) {
                const int item = it0 + tid;
                const int s = item / (2 * R3), rem = item - s * (2 * R3), r = rem >> 1, h = rem & 1;
                const int rreg = (r / n) * NB + (r % n);
                const bool valid = item < nitems && cur[s].state == SLOT_ACTIVE;
                T g[KMAX];
#pragma unroll
                for (int q = 0; q < KMAX; ++q) g[q] = T(0);
                SlotPtrs sp;
                if (valid) {
                    sp = slot_ptrs(smem, L, s);
                    const T* Rr = (const T*)sp.R + rreg;
                    const int t0 = h ? half : 0, t1 = h ? S : half;
                    for (int t = t0; t < t1; ++t) {
                        const T rv = Rr[t * RS];
                        const T* wr = Wt + t * MP;
#pragma unroll
                        for (int q = 0; q < KMAX; ++q)
                            if (q < MP) g[q] = fma_t<T>(rv, wr[q], g[q]);
                    }
                }
#pragma unroll
                for (int q = 0; q < KMAX; ++q) g[q] += __shfl_xor_sync(0xffffffffu, g[q], 1);
                if (valid) {
                    const int kh = (m1 + 1) >> 1;
                    const int q0 = h ? kh : 0, q1 = h ? m1 : kh;
#pragma unroll
                    for (int q = 0; q < KMAX; ++q)
                        if (q >= q0 && q < q1)
                            sp.lamN[r * m1 + q] = sp.lam[r * m1 + q] - p.rho * (double)g[q];
                }
            }
            for (int s = warp; s < spb; s += nwarps) {
                if (cur[s].state != SLOT_ACTIVE) continue;
                const SlotPtrs sp = slot_ptrs(smem, L, s);
                const int k = cur[s].k;
                double emax = 0.0;
                if (k >= 1)
                    for (int r = lane; r < R3; r += 32) emax = fmax(emax, sp.eqerr[r]);
                T inf = T(0);
                double sqs = 0.0;
                if (k >= 1)
                    for (int t = lane; t < S; t += 32) {
                        inf = fmax(inf, ((const T*)sp.pinf)[t]);
                        sqs += sp.psq[t];
                    }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, off));
                    inf = fmax(inf, __shfl_xor_sync(0xffffffffu, inf, off));
                    sqs += __shfl_xor_sync(0xffffffffu, sqs, off);
                }
                if (lane == 0) {
                    const bool failed = (k >= 1) && (emax > p.tol_eq);
                    bool done = failed;
                    if (k >= 1) {
                        const size_t h = (size_t)cur[s].sample * p.max_iters + (k - 1);
                        p.res_inf[h] = (double)inf;
                        p.res_l2[h] = sqrt(sqs);
                        sc[s].last_inf = (double)inf;
                        done = done || (p.early_stop && (double)inf <= p.tol_res) || (k >= p.max_iters);
                    }
                    sc[s].done = done;
                    sc[s].failed = failed;
                    sc[s].eqmax = emax;
                }
            }
        }
        __syncthreads();

        // ---------------- M: finalize finished slots / swarm means for the others
        for (int it = tid; it < spb * dim; it += nt) {
            const int s = it / dim, e = it - s * dim;
            if (cur[s].state == SLOT_ACTIVE && sc[s].done && !sc[s].failed) {
                const SlotPtrs sp = slot_ptrs(smem, L, s);
                const size_t o = (size_t)cur[s].sample * dim + e;
                p.coeffs[o] = sp.C[e];
                p.mult[o] = sp.lam[e];
                if (p.want_prev && p.coeffs_prev) p.coeffs_prev[o] = sp.Cp[e];
            }
        }
        for (int s = warp; s < spb; s += nwarps) {
            if (cur[s].state != SLOT_ACTIVE || !sc[s].done) continue;
            const SlotPtrs sp = slot_ptrs(smem, L, s);
            double acc = 0.0;
            for (int e = lane; e < dim; e += 32) {
                const double dd = sp.C[e] - sp.xb[e];
                acc = fma(dd, dd, acc);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) {
                const int b = cur[s].sample;
                const bool failed = sc[s].failed;
                p.iterations[b] = failed ? 0 : cur[s].k;
                p.converged[b] = (!failed && sc[s].last_inf <= p.tol_res) ? 1 : 0;
                p.displacement[b] = failed ? CUDART_NAN : sqrt(acc);
                p.status[b] = failed ? SAMPLE_SINGULAR_KKT : SAMPLE_OK;
                p.eq_err[b] = sc[s].eqmax;
                sc[s].pending = atomicAdd(p.queue, 1);
            }
        }
        for (int it = tid; it < spb * 3 * m1; it += nt) {
            const int s = it / (3 * m1), rem = it - s * 3 * m1, ax = rem / m1, q = rem - ax * m1;
            if (cur[s].state != SLOT_ACTIVE || sc[s].done) continue;
            const SlotPtrs sp = slot_ptrs(smem, L, s);
            double cs = 0.0, us = 0.0;
            for (int i = 0; i < n; ++i) {
                const int idx = (ax * n + i) * m1 + q;
                cs += sp.C[idx];
                us += 2.0 * sp.lamN[idx] - sp.lam[idx] + sp.xb[idx];
            }
            sp.means[ax * m1 + q] = cs / n;
            sp.means[3 * m1 + ax * m1 + q] = us / n;
        }
        __syncthreads();

        // ---------------- M2: mean part of the xi-step / load newly claimed samples
        for (int it = tid; it < spb * 3 * m1; it += nt) {
            const int s = it / (3 * m1), rem = it - s * 3 * m1, ax = rem / m1, q = rem - ax * m1;
            if (cur[s].state != SLOT_ACTIVE || sc[s].done) continue;
            const SlotPtrs sp = slot_ptrs(smem, L, s);
            const double* cb = sp.means + ax * m1;
            const double* ub = sp.means + 3 * m1 + ax * m1;
            const double* row = KMm + q * m2;
            double acc = 0.0;
            for (int q2 = 0; q2 < m1; ++q2) acc = fma(row[q2], cb[q2], acc);
            for (int q2 = 0; q2 < m1; ++q2) acc = fma(row[m1 + q2], ub[q2], acc);
            sp.mpart[ax * m1 + q] = acc;
        }
        for (int it = tid; it < spb * R3; it += nt) {
            const int s = it / R3, r = it - s * R3;
            if (cur[s].state == SLOT_ACTIVE && sc[s].done && sc[s].pending < p.batch)
                load_row(p, slot_ptrs(smem, L, s), sc[s].pending, r, B6, rhs, PBt, is_float);
        }
        __syncthreads();

        // ---------------- X: decoupled xi-step, equality check, commit lam'
        for (int it = tid; it < spb * R3; it += nt) {
            const int s = it / R3, r = it - s * R3;
            if (cur[s].state != SLOT_ACTIVE || sc[s].done) continue;
            const SlotPtrs sp = slot_ptrs(smem, L, s);
            const int ax = r / n;
            const double* cb = sp.means + ax * m1;
            const double* ub = sp.means + 3 * m1 + ax * m1;
            double dC[KMAX], dU[KMAX], cn[KMAX];
#pragma unroll
            for (int q = 0; q < KMAX; ++q) {
                if (q < m1) {
                    const int idx = r * m1 + q;
                    dC[q] = sp.C[idx] - cb[q];
                    dU[q] = (2.0 * sp.lamN[idx] - sp.lam[idx] + sp.xb[idx]) - ub[q];
                } else {
                    dC[q] = 0.0;
                    dU[q] = 0.0;
                }
            }
#pragma unroll
            for (int q = 0; q < KMAX; ++q) {
                double acc = 0.0;
                if (q < m1) {
                    const double* row = KMd + q * m2;
                    acc = sp.mpart[ax * m1 + q] + cconst[r * m1 + q];
#pragma unroll
                    for (int q2 = 0; q2 < KMAX; ++q2)
                        if (q2 < m1) acc = fma(row[q2], dC[q2], acc);
#pragma unroll
                    for (int q2 = 0; q2 < KMAX; ++q2)
                        if (q2 < m1) acc = fma(row[m1 + q2], dU[q2], acc);
                }
                cn[q] = acc;
            }
            double emax = 0.0;
#pragma unroll
            for (int cnd = 0; cnd < 6; ++cnd) {
                double e = -rhs[r * 6 + cnd];
#pragma unroll
                for (int q = 0; q < KMAX; ++q)
                    if (q < m1) e = fma(B6[cnd * m1 + q], cn[q], e);
                emax = fmax(emax, fabs(e));
            }
            sp.eqerr[r] = emax;
#pragma unroll
            for (int q = 0; q < KMAX; ++q) {
                if (q < m1) {
                    const int idx = r * m1 + q;
                    if (p.want_prev) sp.Cp[idx] = sp.C[idx];
                    sp.C[idx] = cn[q];
                    sp.lam[idx] = sp.lamN[idx];
                    ((T*)sp.Cf)[r * MP + q] = (T)cn[q];
                }
            }
        }
        if (tid < spb) {
            SlotState z = cur[tid];
            if (z.state == SLOT_ACTIVE) {
                if (sc[tid].done) {
                    z.sample = sc[tid].pending;
                    z.k = 0;
                    z.state = (z.sample < p.batch) ? SLOT_ACTIVE : SLOT_EMPTY;
                } else {
                    z.k += 1;
                }
            }
            nxt[tid] = z;
        }
        __syncthreads();
    }
}

}  // namespace sgsf
