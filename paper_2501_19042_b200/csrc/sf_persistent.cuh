// sf_persistent.cuh -- K1: the whole safety-filter iteration loop on-chip.
//
// Replaces SafetyFilter.batch_solve -> solve (solver.py:286-407) including
// the spherical kernel (_speedups.pyx:18-73), F^T (assembly.py:296-303), the
// LU xi-step (assembly.py:186-219) and the boundary projection prologue
// (projection.py:11-25).
//
// Persistent CTAs.  A CTA hosts `spb` independent sample SLOTS; a slot is a
// group of ceil(S/32) warps with its own named barrier, pulling the next
// sample index from a global atomic queue whenever its sample finishes.
// Slots never wait for each other, so one slot's serial phases (projection,
// means, FP64 xi-step) overlap the other slots' term passes.
//
// Term pass: thread t of a slot owns time step t of its sample for ALL
// robots; the positions of every robot at t live in its registers.  Per
// iteration k it
//   T1 evaluates p_k(t) = C_k W[t]^T (TC variant: read from TMEM, where the
//      3xTF32 tcgen05 GEMM issued at the previous MX commit left it), the O(n) statistics of the position
//      change and the workspace terms, and decides whether the O(n^2) pair
//      scan is needed: a motion bound (every pair had normalised distance >=
//      rmin at the last scan and moved by at most cum since) proves all pairs
//      interior while rmin - cum > 1 + margin,
//   T2 scans the pairs of the time steps that need it, one step at a time
//      with all 32 lanes of the owning warp (ballots give the non-interior
//      pair bits) -- warp-local, so no slot barrier,
//   T3 finishes every step: if every term is interior now and at the
//      previous iterate ("quiet"), the targets equal the differences, the
//      scattered residual is 0 and the exit residual of each term is its
//      change Dp_i - Dp_j -- its inf-norm is the per-axis range of Dp and its
//      l2-norm a per-axis sum (O(n)); otherwise the flagged terms take the
//      exact path (target recompute, scatter of d - e into the R row), and
//      terms with an exactly-zero component rerun on the careful path, which
//      uses the FP64 reference trig formula.
// Then every warp takes the stop decision from the per-step partials (no
// barrier), and MX -- one warp per axis, FP64 tensor-core (DMMA) tiles -- forms
// G: lam' = lam - rho R W over the active steps only, then
// forms the swarm means and the decoupled FP64 xi-step
//   C_i = Mm Cb + Km11 ub + Md (C_i - Cb) + Kd11 (u_i - ub) + cconst_i,
//   u = 2 lam' - lam + xi_bar,
// with the ||A xi - b||_inf check (assembly.py:198-217), and (TC) issues the
// position MMAs of the next iterate.  Two slot barriers per iteration.
// T is float ("lean") or double ("strict") for positions and term math;
// state and xi-step are FP64.
#pragma once

#include <cmath>

#include "sf_device.cuh"
#include "sf_tc.cuh"

namespace sgsf {

enum { SAMPLE_OK = 0, SAMPLE_SINGULAR_KKT = 1 };

// shared-memory offsets of one launch (make_layout below)
struct SmemLayout {
    size_t W, KMm, KMd, cconst, B6, rhs, ptab, tmem;
    size_t slot0, slot_stride;
    size_t C, Cp, lam, U, xb, eqerr, psq, pex, P0, P1, Cf, pinf, sh, sc, cp, ct, cw;
    size_t total;
};

struct SolveParams {
    int n, S, m1, MP, batch, max_iters, early_stop, want_prev, spb, wps;
    int coop;   // HY, NB <= 4: warp-cooperative careful path (hy_careful_item); 0 = serial (SGSF_NO_COOP=1, tests)
    int large_coop;   // K1L: phase B (exact steps by all warps) laid out and taken (0: it did not fit)
    double rho, tol_res, tol_eq;
    // hybrid precision (HY kernels): FP32 screening with guard bands, FP64 values.  hy_delta = half-width of
    // the band around tol_res in which the FP32-measured exit residual is re-evaluated in FP64
    double hy_delta;
    double lat, vert, ws_lat, ws_vert, cx, cy, cz;
    const double* W;       // S x m1
    const double* KMm;     // m1 x 2m1  [Mm | Km11]
    const double* KMd;     // m1 x 2m1  [Md | Kd11]
    const double* cconst;  // 3n x m1
    const double* B6;      // 6 x m1
    const double* rhs;     // 3n x 6
    const double* PBt;     // m1 x 6 (read from global memory: the per-sample prologue only)
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
    const int* order;   // queue position -> sample (longest-first), or null for index order
    // K1: the launch's shared-memory map and the spheroid constants, computed on the host so the
    // kernel reads them from the parameter bank instead of recomputing them
    SmemLayout L;
    float fp_lat_f, fp_lim_f, fp_beta_f, fw_lat_f, fw_lim_f, fw_beta_f;
    float hy_fp_lim_f, hy_fw_lim_f;   // HY: interior limits narrowed by the FP32 guard band
    double fp_lim_d, fp_beta_d, fw_lim_d, fw_beta_d;
};

// the host-side precomputation of SolveParams' constants (make_family's expressions)
inline void set_family_constants(SolveParams& p) {
    // hybrid guard bands.  e_pos bounds the FP32 position error (3xTF32 keeps ~21 bits per product) over the
    // workspace; the interior tests are narrowed by 4 e_pos (x4: positions outside the workspace early on)
    // relative to the smallest semiaxis, and the stop decision re-evaluates in FP64 within
    // max(1% of tol_res, 2 e_pos) of tol_res
    {
        const double c = fmax(fabs(p.cx), fmax(fabs(p.cy), fabs(p.cz)));
        const double e_pos = std::ldexp(1.0, -20) * (fmax(p.ws_lat, p.ws_vert) + c);
        const double ep = 4.0 * 4.0 * e_pos / fmin(p.lat, p.vert), ew = 4.0 * 4.0 * e_pos / fmin(p.ws_lat, p.ws_vert);
        p.hy_fp_lim_f = (float)(p.lat * p.lat * (1.0 + ep));
        p.hy_fw_lim_f = (float)(p.ws_lat * p.ws_lat * (1.0 - ew));
        p.hy_delta = fmax(0.01 * p.tol_res, 2.0 * e_pos);
    }
    p.fp_lat_f = (float)p.lat;
    p.fp_lim_f = (float)(p.lat * p.lat);
    p.fp_beta_f = (float)((p.lat * p.lat) / (p.vert * p.vert));
    p.fw_lat_f = (float)p.ws_lat;
    p.fw_lim_f = (float)(p.ws_lat * p.ws_lat);
    p.fw_beta_f = (float)((p.ws_lat * p.ws_lat) / (p.ws_vert * p.ws_vert));
    p.fp_lim_d = p.lat * p.lat;
    p.fp_beta_d = (p.lat * p.lat) / (p.vert * p.vert);
    p.fw_lim_d = p.ws_lat * p.ws_lat;
    p.fw_beta_d = (p.ws_lat * p.ws_lat) / (p.ws_vert * p.ws_vert);
}

// next sample for a slot: queue position -> sample index
__device__ __forceinline__ int next_sample(const SolveParams& p) {
    const int q = atomicAdd(p.queue, 1);
    return (p.order && q < p.batch) ? p.order[q] : q;
}

// per-slot scalars.  The per-iteration flags are double-buffered by the
// iteration parity: iteration k writes buffer k&1 before the term-pass
// barrier and reads it after; the other buffer was last read before the
// previous iteration's closing barrier, so one thread clears it during the
// term pass with no extra barrier.
constexpr int MAX_SLOT_WORDS = 16;   // time-step bit words (slot size <= 512 threads)
struct SlotShared {
    uint64_t mbar;   // TC: completion of the position MMAs of the next iterate (3 arrivals, one per axis)
    int sample;
    int active[2];   // some term had an active constraint in the term pass
    uint32_t amask[2][MAX_SLOT_WORDS];   // time steps with an active term (their R row is valid)
};

__device__ __forceinline__ void clear_flags(SlotShared* sh, int b, int words) {
    sh->active[b] = 0;
    for (int w = 0; w < words; ++w) sh->amask[b][w] = 0u;
}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Position-row stride (elements of T): a whole number of 16-byte units, and an
// odd number of them, so the per-thread rows are read and written as 16-byte
// vectors with no bank conflicts (8 consecutive rows hit 8 distinct 16-byte
// bank groups).
template <typename T, int NB> struct RowStride {
    static constexpr int per16 = 16 / (int)sizeof(T);
    static constexpr int base = (3 * NB + per16 - 1) / per16;   // 16-byte units
    static constexpr int value = ((base & 1) ? base : base + 1) * per16;
};

// Shared-memory map.  Coefficient-space arrays are padded to MP (m1 rounded
// up to a multiple of 4) columns with zeros, so every loop over the degree
// runs to the compile-time MP with no guards and vector loads.  P0/P1 hold
// the positions of iterates k (old) and k+1 (new) as [t][3 NB + 1] rows
// (thread t owns row t; odd stride -> distinct banks); after the term pass
// the dead old row is reused for the thread's scattered residual R, valid
// where bit t of the slot's active-step mask is set.

// TC: the FP32 copy of C becomes the 3xTF32 B operand of the position GEMM, [axis][hi, lo] blocks of
// 16 robots x 16 k in the UMMA K-major layout (tc::kmajor16_offset)
constexpr int kTcBopBytes = 3 * 2 * 1024;
// round-based cooperative careful path (hy_careful_rounds): per warp 32 items of 8 doubles + 16 owners x 12
// (outputs for the 16 owner lanes of a two-lane-per-step warp; + both iterates' FP64 positions)
constexpr int kCoopOwners = 16;
constexpr int kCoopMaxS = 128;   // n <= 4: the cooperative careful path's scratch and target cache up to this horizon
constexpr int kCoopWarpDoubles = 32 * 8 + kCoopOwners * 12 + 2 * 3 * 32;

// hy: hybrid precision keeps the previous iterate's FP64 coefficients (Cp) and FP64 exit-residual partials
// (pex).  The per-warp partial arrays are sized for the slot's warps: 4 on the tensor-core path.
template <typename T, int NB>
__host__ __device__ inline SmemLayout make_layout(int n, int S, int MP, int spb, int want_prev, bool tc = false,
                                                  bool hy = false) {
    const int RS = RowStride<T, NB>::value;
    SmemLayout L;
    size_t o = 0;
    const size_t d = sizeof(double), ts = sizeof(T);
    const int R3 = 3 * n, dimp = R3 * MP;
    L.W = o;      o = align16(o + (size_t)S * MP * ts);
    L.KMm = o;    o = align16(o + (size_t)MP * 2 * MP * d);
    L.KMd = o;    o = align16(o + (size_t)MP * 2 * MP * d);
    L.cconst = o; o = align16(o + (size_t)dimp * d);
    L.B6 = o;     o = align16(o + (size_t)6 * MP * d);
    L.rhs = o;    o = align16(o + (size_t)R3 * 6 * d);
    L.ptab = o;   o = align16(o + (size_t)NB * (NB - 1) / 2 * sizeof(int));
    L.tmem = o;   o = align16(o + 2 * sizeof(uint32_t));               // TC: TMEM base, finished-slot count
    L.slot0 = o;
    size_t q = 0;
    L.C = q;      q = align16(q + (size_t)dimp * d);
    L.Cp = q;     q = align16(q + ((want_prev || hy) ? (size_t)dimp * d : 0));
    L.lam = q;    q = align16(q + (size_t)dimp * d);
    L.U = q;      q = align16(q + (size_t)dimp * d);                // u = 2 lam' - lam + xi_bar
    L.xb = q;     q = align16(q + (size_t)dimp * d);
    L.eqerr = q;  q = align16(q + (size_t)4 * d);                     // per axis max ||A xi - b|| over its rows
    const size_t pw = tc ? 4 : MAX_SLOT_WORDS;                        // partial-array entries (warps)
    L.psq = q;    q = align16(q + pw * d);                             // per warp sum of the l2 partials
    L.pex = q;    q = align16(q + (hy ? 2 * pw * d : 0));              // hy: FP64 exit-residual partials (inf, l2)
    L.P0 = q;     q = align16(q + (size_t)RS * S * ts);
    L.P1 = q;     q = align16(q + (size_t)RS * S * ts);
    L.Cf = q;     q = align16(q + (tc ? (size_t)kTcBopBytes : (size_t)3 * MP * NB * ts));
    L.pinf = q;   q = align16(q + pw * ts);                            // per warp max of the inf partials
    L.sh = q;     q = align16(q + sizeof(SlotShared));
    // hy, NB <= 4: per warp 32 items of the warp-cooperative careful path (hy_careful_item)
    // (horizons up to kCoopMaxS steps: past that the careful steps stay serial, so long horizons keep fitting)
    const bool coop4 = hy && NB <= 4 && !tc && S <= kCoopMaxS;
    L.cp = q;     q = align16(q + (coop4 ? (size_t)((S + 31) / 32) * 32 * 8 * d : 0));
    // ... and the FP64 trig targets e(d_k) of its zero-component terms per (step, term), tagged (sample, k): the
    // next iteration's e(d_{k-1}) (hy_careful_item)
    L.ct = q;     q = align16(q + (coop4 ? (size_t)S * (NB * (NB - 1) / 2 + NB) * (3 * d + 8) : 0));
    // hy, NB = 32: per warp 32 items + 32 owners' outputs of the round-based cooperative careful path
    L.cw = q;     q = align16(q + ((hy && NB >= 32 && !tc) ? (size_t)((S + 15) / 16) * kCoopWarpDoubles * d : 0));
#ifdef SGSF_SYNC_CHECK
    L.sc = q;     q = align16(q + pw * sizeof(int));                   // debug: per-warp decisions
#else
    L.sc = q;
#endif
    L.slot_stride = q;
    L.total = o + (size_t)spb * q;
    return L;
}

struct SlotPtrs {
    double *C, *Cp, *lam, *U, *xb, *eqerr, *psq, *pex;
    void *P0, *P1, *Cf, *pinf;
    SlotShared* sh;
    double* cp;
    double* ct;
    double* cw;
};

__device__ __forceinline__ SlotPtrs slot_ptrs(unsigned char* smem, const SmemLayout& L, int s) {
    unsigned char* b = smem + L.slot0 + (size_t)s * L.slot_stride;
    SlotPtrs P;
    P.C = (double*)(b + L.C);
    P.Cp = (double*)(b + L.Cp);
    P.lam = (double*)(b + L.lam);
    P.U = (double*)(b + L.U);
    P.xb = (double*)(b + L.xb);
    P.eqerr = (double*)(b + L.eqerr);
    P.psq = (double*)(b + L.psq);
    P.pex = (double*)(b + L.pex);
    P.P0 = (void*)(b + L.P0);
    P.P1 = (void*)(b + L.P1);
    P.Cf = (void*)(b + L.Cf);
    P.pinf = (void*)(b + L.pinf);
    P.sh = (SlotShared*)(b + L.sh);
    P.cp = (double*)(b + L.cp);
    P.ct = (double*)(b + L.ct);
    P.cw = (double*)(b + L.cw);
    return P;
}

// Named barrier of one slot.  The non-.aligned form: lanes of a warp may
// arrive diverged (threads t >= S skip the term pass), which bar.sync
// (= barrier.sync.aligned) does not allow.
__device__ __forceinline__ void slot_barrier(int id, int nthreads) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

#ifdef SGSF_COUNTERS
// event counters of the instrumented build: [0] finish calls, [1] flagged path, [2] exact recompute,
// [3] careful path, [4] flagged terms, [5] near checks, [6] pair scans, [7] fast exact far max, [8] HY FP64
// exit-residual re-evaluations
__device__ unsigned long long g_sgsf_counts[10];
#define SGSF_COUNT(I, V) atomicAdd(&g_sgsf_counts[I], (unsigned long long)(V))
#else
#define SGSF_COUNT(I, V) ((void)0)
#endif

// warp-wide min of non-negative values: one REDUX on the float bits (which
// order like the values), shuffles for double
__device__ __forceinline__ float warp_min_nonneg(float v) {
    return __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(v)));
}
// non-negative doubles order like their (hi, lo) words: REDUX the high words,
// then the low words of the lanes that hold the winning high word
__device__ __forceinline__ double warp_min_nonneg(double v) {
    const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    return __hiloint2double((int)mh, (int)ml);
}
__device__ __forceinline__ float warp_max_nonneg(float v) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}
__device__ __forceinline__ double warp_max_nonneg(double v) {
    const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return __hiloint2double((int)mh, (int)ml);
}

// D += A B for one 8x8x4 FP64 tile (DMMA): A (8x4, row) element [lane/4][lane%4],
// B (4x8, col) element [lane%4][lane/4], D (8x8) elements [lane/4][2 (lane%4) + {0, 1}]
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// 16-byte vector of T (float4 / double2) for the row-times-vector loops
template <typename T> struct Vec16;
template <> struct Vec16<float> {
    using type = float4;
    static constexpr int lanes = 4;
    __device__ __forceinline__ static void unpack(const float4& v, float* o) {
        o[0] = v.x;
        o[1] = v.y;
        o[2] = v.z;
        o[3] = v.w;
    }
};
template <> struct Vec16<double> {
    using type = double2;
    static constexpr int lanes = 2;
    __device__ __forceinline__ static void unpack(const double2& v, double* o) {
        o[0] = v.x;
        o[1] = v.y;
    }
};

template <typename T, int MP>
__device__ __forceinline__ void load_row16(const T* __restrict__ src, T (&dst)[MP]) {
    using V = typename Vec16<T>::type;
    constexpr int L = Vec16<T>::lanes;
    const V* v = reinterpret_cast<const V*>(src);
#pragma unroll
    for (int c = 0; c < MP / L; ++c) Vec16<T>::unpack(v[c], dst + c * L);
}

// ---------------------------------------------------------------- term pass pieces
// One bit per term, pairs i<j in loop order then workspace terms.
template <int NB> struct TermBits {
    static constexpr int count = NB * (NB - 1) / 2 + NB;
    static constexpr int words = (count + 31) / 32;
};

__device__ __forceinline__ bool bit_of(const uint32_t* m, int b) { return (m[b >> 5] >> (b & 31)) & 1u; }

// bit of pair (i < j) and of workspace term i, as closed forms of the loop indices
// (a loop-carried counter keeps nvcc from fully unrolling the register-indexed loops)
template <int NB> __host__ __device__ constexpr int pair_bit(int i, int j) { return i * (2 * NB - i - 1) / 2 + (j - i - 1); }
template <int NB> __host__ __device__ constexpr int ws_bit(int i) { return NB * (NB - 1) / 2 + i; }

// Robots past n become "phantoms" at distinct, far-away positions: every
// pair term with a phantom is interior and has no zero component.  Cf is
// stored robot-minor ([ax][q][NB]) so two robots' coefficients form one
// f32x2 operand.
template <typename T> __device__ __forceinline__ T phantom_pos(int i) { return T(1e30) * T(i + 1); }


// ---- part-wise term pass: a thread owns RH = NB / TPS robots [r0, r0 + RH) of its time step;
// with TPS = 2 the two halves of a step sit in lanes l and l ^ 16 and combine with shuffles.

// positions of robots [r0, r0 + RH) at time step t (phantoms past n)
template <typename T, int NB, int RH, int MP>
__device__ __forceinline__ void positions_part(const T* __restrict__ Wt, const T* __restrict__ Cf, int t, int r0, int n,
                                               T (&pos)[3 * RH]) {
    T w[MP];
    load_row16<T, MP>(Wt + t * MP, w);
    if constexpr (sizeof(T) == 4 && RH % 4 == 0) {
        float2 w2[MP];
#pragma unroll
        for (int q = 0; q < MP; ++q) w2[q] = make_float2(w[q], w[q]);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
            for (int i4 = 0; i4 < RH; i4 += 4) {
                float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < MP; ++q) {
                    const float4 c = *reinterpret_cast<const float4*>(Cf + (ax * MP + q) * NB + r0 + i4);
                    a01 = __ffma2_rn(make_float2(c.x, c.y), w2[q], a01);
                    a23 = __ffma2_rn(make_float2(c.z, c.w), w2[q], a23);
                }
                pos[ax * RH + i4] = a01.x;
                pos[ax * RH + i4 + 1] = a01.y;
                pos[ax * RH + i4 + 2] = a23.x;
                pos[ax * RH + i4 + 3] = a23.y;
            }
        }
    } else {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
            for (int i = 0; i < RH; ++i) {
                T s = T(0);
#pragma unroll
                for (int q = 0; q < MP; ++q) s = fma_t<T>(Cf[(ax * MP + q) * NB + r0 + i], w[q], s);
                pos[ax * RH + i] = s;
            }
        }
    }
    if (n < NB) {   // uniform: phantom robots only in the smaller swarms
#pragma unroll
        for (int q = 0; q < 3 * RH; ++q)
            if (r0 + (q % RH) >= n) pos[q] = phantom_pos<T>(r0 + (q % RH));
    }
}

// 16-byte vector copies of this thread's part of a position row
template <typename T, int NB, int RH>
__device__ __forceinline__ void store_part(T* __restrict__ row, int r0, const T (&pos)[3 * RH]) {
    using V = typename Vec16<T>::type;
    constexpr int L = Vec16<T>::lanes;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
        for (int c = 0; c < RH / L; ++c) {
            V v;
            T* e = reinterpret_cast<T*>(&v);
#pragma unroll
            for (int u = 0; u < L; ++u) e[u] = pos[ax * RH + c * L + u];
            *reinterpret_cast<V*>(row + ax * NB + r0 + c * L) = v;
        }
    }
}
template <typename T, int NB, int RH>
__device__ __forceinline__ void load_part(const T* __restrict__ row, int r0, T (&out)[3 * RH]) {
    using V = typename Vec16<T>::type;
    constexpr int L = Vec16<T>::lanes;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
        for (int c = 0; c < RH / L; ++c) {
            const V v = *reinterpret_cast<const V*>(row + ax * NB + r0 + c * L);
            const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
            for (int u = 0; u < L; ++u) out[ax * RH + c * L + u] = e[u];
        }
    }
}

// combine the two halves of a time step (lanes l, l ^ 16); identity for TPS = 1
template <int TPS, typename V> __device__ __forceinline__ V part_min(V v, unsigned m) {
    if constexpr (TPS == 2) return fmin(v, __shfl_xor_sync(m, v, 16));
    return v;
}
template <int TPS, typename V> __device__ __forceinline__ V part_max(V v, unsigned m) {
    if constexpr (TPS == 2) return fmax(v, __shfl_xor_sync(m, v, 16));
    return v;
}
template <int TPS, typename V> __device__ __forceinline__ V part_sum(V v, unsigned m) {
    if constexpr (TPS == 2) return v + __shfl_xor_sync(m, v, 16);
    return v;
}
template <int TPS> __device__ __forceinline__ uint32_t part_and(uint32_t v, unsigned m) {
    if constexpr (TPS == 2) return v & __shfl_xor_sync(m, v, 16);
    return v;
}

template <typename T> struct PartStats {
    T inf, sq, dmax2;
};

// pairwise (tree) reduction of a register array, log2(N) dependent levels
template <typename T, int N, typename Op> __device__ __forceinline__ T tree_reduce(T (&v)[N], Op op) {
#pragma unroll
    for (int w = N / 2; w >= 1; w /= 2) {
#pragma unroll
        for (int i = 0; i < w; ++i) v[i] = op(v[i], v[i + w]);
    }
    return v[0];
}
struct OpMin { template <typename T> __device__ T operator()(T a, T b) const { return fmin(a, b); } };
struct OpMax { template <typename T> __device__ T operator()(T a, T b) const { return fmax(a, b); } };
struct OpAdd { template <typename T> __device__ T operator()(T a, T b) const { return a + b; } };

// O(n) statistics of the position change Dp of the whole step, from this
// thread's robots (Pold: the old row): per axis min, max, sum and sum of
// squares, combined over the step's lanes.  inf = max over the terms of
// |Dp_i - Dp_j| (pairs: per-axis range) and |Dp_i| (workspace: max(max, -min));
// sq = (n+1) sum Dp^2 - (sum Dp)^2 (= n sum (Dp - mean)^2 + sum Dp^2).  FULL:
// every robot of this part is real (no phantom guards; tree reductions).  All
// lanes in `m` must call it together.
template <typename T, int NB, int RH, int TPS, bool FULL>
__device__ __forceinline__ PartStats<T> quiet_part(const T (&pos)[3 * RH], const T* __restrict__ Pold, int r0, int n,
                                                   T fp_beta, unsigned m) {
    T old[3 * RH];
    load_part<T, NB, RH>(Pold, r0, old);
    T dp[3 * RH];
#pragma unroll
    for (int q = 0; q < 3 * RH; ++q) dp[q] = pos[q] - old[q];   // phantoms: 0 (same far value in both rows)
    T mx = T(0), s2 = T(0), dm = T(0);
    if constexpr (FULL) {
        T dq[RH];
#pragma unroll
        for (int i = 0; i < RH; ++i)
            dq[i] = fma_t<T>(dp[2 * RH + i] * fp_beta, dp[2 * RH + i], fma_t<T>(dp[RH + i], dp[RH + i], dp[i] * dp[i]));
        dm = tree_reduce(dq, OpMax());
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            T lo[RH], hi[RH], s1[RH], sq[RH];
#pragma unroll
            for (int i = 0; i < RH; ++i) {
                lo[i] = hi[i] = s1[i] = dp[ax * RH + i];
                sq[i] = dp[ax * RH + i] * dp[ax * RH + i];
            }
            T l = part_min<TPS>(tree_reduce(lo, OpMin()), m), hh = part_max<TPS>(tree_reduce(hi, OpMax()), m);
            T a1 = part_sum<TPS>(tree_reduce(s1, OpAdd()), m), a2 = part_sum<TPS>(tree_reduce(sq, OpAdd()), m);
            mx = fmax(mx, fmax(hh - l, fmax(hh, -l)));
            s2 += fmax(fma_t<T>((T)(n + 1), a2, -a1 * a1), a2);
        }
    } else {
        T dq[RH];
#pragma unroll
        for (int i = 0; i < RH; ++i) dq[i] = T(0);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            T lo = T(1e38), hi = T(-1e38), s1 = T(0), sq = T(0);
#pragma unroll
            for (int i = 0; i < RH; ++i) {
                if (r0 + i < n) {
                    const T dpi = dp[ax * RH + i];
                    lo = fmin(lo, dpi);
                    hi = fmax(hi, dpi);
                    s1 += dpi;
                    sq = fma_t<T>(dpi, dpi, sq);
                    dq[i] = fma_t<T>(ax == 2 ? dpi * fp_beta : dpi, dpi, dq[i]);
                }
            }
            lo = part_min<TPS>(lo, m);
            hi = part_max<TPS>(hi, m);
            s1 = part_sum<TPS>(s1, m);
            sq = part_sum<TPS>(sq, m);
            mx = fmax(mx, fmax(hi - lo, fmax(hi, -lo)));
            s2 += fmax(fma_t<T>((T)(n + 1), sq, -s1 * s1), sq);
        }
#pragma unroll
        for (int i = 0; i < RH; ++i) dm = fmax(dm, dq[i]);
    }
    PartStats<T> st;
    st.dmax2 = part_max<TPS>(dm, m);
    st.inf = mx;
    st.sq = s2;
    return st;
}

// workspace terms of this thread's robots: a value that is 0 iff some
// component is exactly zero (FULL: the product of the three components,
// which can only underflow to a false "zero" -- that just takes the exact
// careful path), and the non-interior workspace bits cleared in nm (combined
// over the step's lanes; h = this lane's half).  COINC (hybrid): the zeros count only when one of the lane's
// workspace terms is non-interior -- an interior term's reference-trig target is d up to an ulp-level leak,
// which the hybrid kernels take as d (conservative: a non-interior term keeps the lane's zeros)
template <typename T, int NB, int RH, int TPS, bool FULL, bool COINC = false>
__device__ __forceinline__ T ws_part(const T (&pos)[3 * RH], int r0, int h, int n, const Family<T>& fw, T cx, T cy,
                                     T cz, uint32_t (&nm)[TermBits<NB>::words], unsigned m) {
    T zm = T(1), qw = T(0);
    if constexpr (FULL) {
        T zv[RH], qv[RH];
#pragma unroll
        for (int i = 0; i < RH; ++i) {
            const T rx = pos[i] - cx, ry = pos[RH + i] - cy, rz = pos[2 * RH + i] - cz;
            zv[i] = fabs(rx * ry * rz);
            qv[i] = fma_t<T>(rz * fw.beta, rz, fma_t<T>(ry, ry, rx * rx));
        }
        zm = tree_reduce(zv, OpMin());
        qw = tree_reduce(qv, OpMax());
    } else {
#pragma unroll
        for (int i = 0; i < RH; ++i) {
            if (r0 + i < n) {
                const T rx = pos[i] - cx, ry = pos[RH + i] - cy, rz = pos[2 * RH + i] - cz;
                zm = fmin(zm, fmin(fabs(rx), fmin(fabs(ry), fabs(rz))));
                qw = fmax(qw, fma_t<T>(rz * fw.beta, rz, fma_t<T>(ry, ry, rx * rx)));
            }
        }
    }
    if (COINC && qw <= fw.lim) zm = T(1);   // (this lane's workspace terms are all interior)
#pragma unroll
    for (int w = 0; w < TermBits<NB>::words; ++w) nm[w] = 0xffffffffu;
    if (__builtin_expect(__any_sync(m, !(qw <= fw.lim)), 0)) {
        uint32_t out = 0u;   // bit i: workspace term of robot r0 + i non-interior
#pragma unroll
        for (int i = 0; i < RH; ++i) {
            if (r0 + i < n) {
                const T rx = pos[i] - cx, ry = pos[RH + i] - cy, rz = pos[2 * RH + i] - cz;
                const T q = fma_t<T>(rz * fw.beta, rz, fma_t<T>(ry, ry, rx * rx));
                if (!(q <= fw.lim)) out |= 1u << i;
            }
        }
        if constexpr (TPS == 2) {
            const uint32_t other = __shfl_xor_sync(m, out, 16);
            out = h == 0 ? (out | (other << RH)) : (other | (out << RH));
        }
        constexpr int NP = NB * (NB - 1) / 2;
        const unsigned long long sh = (unsigned long long)out << (NP & 31);
        nm[NP >> 5] &= ~(uint32_t)sh;
        if constexpr ((NP & 31) + NB > 32) nm[(NP >> 5) + 1] &= ~(uint32_t)(sh >> 32);
    }
    return part_min<TPS>(zm, m);
}


// by-value packs of register arrays for out-of-line calls
template <typename T, int NB> struct PosPack {
    T v[3 * NB];
};
template <int NB> struct MaskPack {
    uint32_t w[TermBits<NB>::words];
};

// robots of term bit b: pair (i, j) from the lexicographic pair table, or workspace term i (j = -1)
template <int NB> __device__ __forceinline__ void term_robots(const int* __restrict__ ptab, int b, int& i, int& j) {
    constexpr int NP = NB * (NB - 1) / 2;
    if (b < NP) {
        const int ij = ptab[b];
        i = ij & 0xff;
        j = ij >> 8;
    } else {
        i = b - NP;
        j = -1;
    }
}


// ---------------------------------------------------------------- hybrid precision (HY): FP64 values
// The HY kernels screen in FP32 exactly like the lean ones, with the interior tests narrowed by a guard band
// (fp.lim, fw.lim scaled on the host side of the kernel): a term the FP32 test calls interior is interior in
// FP64.  Every value that reaches the state or a stop decision is FP64: the targets and residuals of the
// flagged (non-interior now or before) terms come from FP64 positions of the FP64 coefficients of both
// iterates (C = C_k, Cp = C_{k-1}), in strict's exact operation order; the quiet (all-interior) terms have
// zero scattered residual, so they never touch the state.  The FP32-measured exit residual decides the stop
// unless it lies within hy_delta of tol_res; then the whole exit residual is re-evaluated in FP64
// (hy_step_full over every time step).
struct D3 {
    double x, y, z;
};

// The FP64 stop re-evaluation and scatter out of line: the fields they read, by value -- a
// non-inlined callee must not take the kernel's parameter block by reference (its local copy turns every p.*
// read into a local-memory load); inlined, its code and registers weighed on the whole kernel
struct HyExitArgs {
    const double* W;
    int n, m1;
    double cx, cy, cz, lat, vert, ws_lat, ws_vert, fp_lim_d, fp_beta_d, fw_lim_d, fw_beta_d;
};
__device__ __forceinline__ HyExitArgs hy_exit_args(const SolveParams& p) {
    HyExitArgs a;
    a.W = p.W;
    a.n = p.n;
    a.m1 = p.m1;
    a.cx = p.cx, a.cy = p.cy, a.cz = p.cz;
    a.lat = p.lat, a.vert = p.vert, a.ws_lat = p.ws_lat, a.ws_vert = p.ws_vert;
    a.fp_lim_d = p.fp_lim_d, a.fp_beta_d = p.fp_beta_d, a.fw_lim_d = p.fw_lim_d, a.fw_beta_d = p.fw_beta_d;
    return a;
}

template <int MP>
__device__ __forceinline__ void w64_row(const double* __restrict__ W, int t, int m1, double (&w)[MP]) {
#pragma unroll
    for (int q = 0; q < MP; ++q) w[q] = q < m1 ? __ldg(W + t * m1 + q) : 0.0;
}
// FP64 position of coefficient row `row` (strict's order: fma over q ascending from 0)
template <int MP>
__device__ __forceinline__ double pos64(const double* __restrict__ C, const double (&w)[MP], int row) {
    const double* c = C + row * MP;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < MP; ++q) s = fma(c[q], w[q], s);
    return s;
}

template <typename P>
__device__ __forceinline__ Family<double> family64(const P& p, bool pair) {
    Family<double> f;
    f.lat = pair ? p.lat : p.ws_lat;
    f.lim = pair ? p.fp_lim_d : p.fw_lim_d;
    f.beta = pair ? p.fp_beta_d : p.fw_beta_d;
    f.lat64 = pair ? p.lat : p.ws_lat;
    f.vert64 = pair ? p.vert : p.ws_vert;
    return f;
}

// difference vector of term (i, j) (j < 0: workspace term of robot i, relative to the centre) at step t of C
template <int MP, typename P>
__device__ __forceinline__ D3 term_diff64(const P& p, const double* __restrict__ C, const double (&w)[MP],
                                          int i, int j) {
    const int n = p.n;
    D3 d;
    if (j >= 0) {
        d.x = pos64<MP>(C, w, i) - pos64<MP>(C, w, j);
        d.y = pos64<MP>(C, w, n + i) - pos64<MP>(C, w, n + j);
        d.z = pos64<MP>(C, w, 2 * n + i) - pos64<MP>(C, w, 2 * n + j);
    } else {
        d.x = pos64<MP>(C, w, i) - p.cx;
        d.y = pos64<MP>(C, w, n + i) - p.cy;
        d.z = pos64<MP>(C, w, 2 * n + i) - p.cz;
    }
    return d;
}

// FP64 b - target(d) of one term (zero components: the reference trig formula)
__device__ __forceinline__ D3 resid64(bool pair, const D3& d, const D3& b, const Family<double>& f) {
    double zu = 1.0;
    D3 r;
    if (pair) resid<double, true, true>(d.x, d.y, d.z, b.x, b.y, b.z, f, zu, r.x, r.y, r.z);
    else resid<double, false, true>(d.x, d.y, d.z, b.x, b.y, b.z, f, zu, r.x, r.y, r.z);
    return r;
}

// Warp-cooperative careful path (HY, NB <= 4).  A careful time step (a term with an exactly-zero component
// now or at the previous iterate: FP64 reference trig targets, ~1.6K cycles each) is owned by one lane; a
// symmetric scenario has few such steps -- the fixed endpoints -- and their owners would run every term's
// FP64 positions and trig serially (with the position arrays spilled: ~13K cycles per step at n = 4, measured
// with SGSF_CAREFUL_CLOCK) while the warp waits.  Instead the warp spreads the (careful lane, term) items over
// its lanes: item (k, b) computes, for the k-th careful lane's step, term b's FP64 exit residual x = d_k -
// e(d_{k-1}), its scattered residual r = d_k - e(d_k) and its flags exactly as hy_step_full does (same
// positions, same resid64) into out[0..6]; the owner then reduces its items in term order (hy_step_coop).
// Bit-identical to hy_step_full by construction.
__device__ __forceinline__ bool has_zero(const D3& d) { return d.x == 0.0 || d.y == 0.0 || d.z == 0.0; }
// b - (a target computed earlier): resid's operation for a zero-component term
__device__ __forceinline__ D3 minus(const D3& b, const double* __restrict__ t) { return D3{b.x - t[0], b.y - t[1], b.z - t[2]}; }
constexpr int kCoopItem = 8;   // doubles per item: x (3), r (3), flags (1: not interior or zero, 2: zero)
template <int NB, int MP>
__device__ __forceinline__ void hy_careful_item(const SolveParams& p, const double* Cn, const double* Co, int t, int b,
                                                double* __restrict__ out, double* __restrict__ ct, long long tag) {
    constexpr int NP = NB * (NB - 1) / 2;
    int i = 0, j = -1;
    if (b < NP) {
        int r = b;
        for (i = 0; i < NB; ++i) {
            if (r < NB - 1 - i) break;
            r -= NB - 1 - i;
        }
        j = i + 1 + r;
        if (j >= p.n) return;
    } else {
        i = b - NP;
        if (i >= p.n) return;
    }
    double w[MP];
    w64_row<MP>(p.W, t, p.m1, w);
    const D3 d = term_diff64<MP>(p, Cn, w, i, j), o = term_diff64<MP>(p, Co, w, i, j);
    const bool pair = j >= 0;
    const Family<double> f = family64(p, pair);
    // e(d_{k-1}) of a zero-component term is the e(d_k) this item stored one iteration earlier (the same FP64
    // positions of the same C_{k-1}: the same bits); a trig target is computed once per iterate
    constexpr int NT = NB * (NB - 1) / 2 + NB;
    double* ce = ct + ((size_t)t * NT + b) * 3;
    long long* cs = (long long*)(ct + (size_t)p.S * NT * 3) + (size_t)t * NT + b;
    D3 x, r;
    if (has_zero(o) && *cs == tag - 1) x = minus(d, ce);
    else x = resid64(pair, o, d, f);
    if (has_zero(d)) {
        double e[3];
        if (pair) target<double, true>(d.x, d.y, d.z, f, e[0], e[1], e[2]);
        else target<double, false>(d.x, d.y, d.z, f, e[0], e[1], e[2]);
        r = minus(d, e);
        ce[0] = e[0], ce[1] = e[1], ce[2] = e[2];
        *cs = tag;
    } else {
        r = resid64(pair, d, d, f);
    }
    const double q = fma(d.z * f.beta, d.z, fma(d.y, d.y, d.x * d.x));
    const bool off = pair ? !(q >= f.lim) : !(q <= f.lim);
    const bool zero = (d.x == 0.0 || d.y == 0.0 || d.z == 0.0) && off;   // (hybrid: non-interior)
    out[0] = x.x, out[1] = x.y, out[2] = x.z;
    out[3] = r.x, out[4] = r.y, out[5] = r.z;
    out[6] = (double)(((off || zero) ? 1 : 0) | (zero ? 2 : 0));
}

// streamed variants (the W row through the read-only cache; pos64's order of operations)
template <int MP>
__device__ __forceinline__ double pos64s(const double* __restrict__ C, const double* __restrict__ Wrow, int m1,
                                         int row) {
    const double* c = C + row * MP;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < MP; ++q) s = fma(c[q], q < m1 ? __ldg(Wrow + q) : 0.0, s);
    return s;
}
template <int MP, typename P>
__device__ __forceinline__ D3 term_diff64s(const P& p, const double* __restrict__ C,
                                           const double* __restrict__ Wrow, int i, int j) {
    const int n = p.n, m1 = p.m1;
    D3 d;
    if (j >= 0) {
        d.x = pos64s<MP>(C, Wrow, m1, i) - pos64s<MP>(C, Wrow, m1, j);
        d.y = pos64s<MP>(C, Wrow, m1, n + i) - pos64s<MP>(C, Wrow, m1, n + j);
        d.z = pos64s<MP>(C, Wrow, m1, 2 * n + i) - pos64s<MP>(C, Wrow, m1, 2 * n + j);
    } else {
        d.x = pos64s<MP>(C, Wrow, m1, i) - p.cx;
        d.y = pos64s<MP>(C, Wrow, m1, n + i) - p.cy;
        d.z = pos64s<MP>(C, Wrow, m1, 2 * n + i) - p.cz;
    }
    return d;
}

// Scattered residual R of every term non-interior (guarded FP32 test) in the new iterate at step t, in
// FP64 from C_k: W row loaded once, R accumulated into the thread's (dead) old row.  Returns whether some term
// has a non-zero residual (is active in FP64).
// (every HY helper that takes the kernel's SolveParams by reference must be inlined: a reference to a kernel
// parameter passed to a real call makes the compiler copy the parameter block to local memory and read every
// p.* field from there, on every iteration -- that cost hybrid ~15% of its samples until round 2 found it)
template <typename T, int NB, int MP, typename P>
__device__ __forceinline__ bool hy_scatter_step(const P& p, const double* Cn, int t, const MaskPack<NB> nm,
                                             const int* __restrict__ ptab, T* Pold) {
    double w[MP];
    w64_row<MP>(p.W, t, p.m1, w);
    bool act = false;
    for (int wd = 0; wd < TermBits<NB>::words; ++wd) {
        uint32_t ac = ~nm.w[wd];
        while (ac) {
            const int bit = __ffs(ac) - 1;
            ac &= ac - 1;
            const int b = wd * 32 + bit;
            if (b >= TermBits<NB>::count) break;
            int i, j;
            term_robots<NB>(ptab, b, i, j);
            const D3 dn = term_diff64<MP>(p, Cn, w, i, j);
            const D3 r = resid64(j >= 0, dn, dn, family64(p, j >= 0));
            act = act || r.x != 0.0 || r.y != 0.0 || r.z != 0.0;
            Pold[i] += (T)r.x;
            Pold[NB + i] += (T)r.y;
            Pold[2 * NB + i] += (T)r.z;
            if (j >= 0) {
                Pold[j] -= (T)r.x;
                Pold[NB + j] -= (T)r.y;
                Pold[2 * NB + j] -= (T)r.z;
            }
        }
    }
    return act;
}

// Every term of time step t in FP64: exit residual statistics (max |x|, sum x^2) and, when Rrow != null, the
// careful path -- R row (written over the dead old row), interior bits (zero-component terms count as active)
template <typename T, int NB, int MP> struct HyStepOut {
    double inf, sq;
    bool zero, active;
};
template <typename T, int NB, int MP>
__device__ __forceinline__ HyStepOut<T, NB, MP> hy_step_full(const SolveParams& p, const double* Cn, const double* Co,
                                                         int t, T* Rrow, MaskPack<NB>* nmo) {
    const int n = p.n;
    double w[MP];
    w64_row<MP>(p.W, t, p.m1, w);
    double pn[3 * NB], po[3 * NB], R[3 * NB];
    for (int q = 0; q < 3 * NB; ++q) {
        const int ax = q / NB, i = q % NB;
        pn[q] = i < n ? pos64<MP>(Cn, w, ax * n + i) : 0.0;
        po[q] = i < n ? pos64<MP>(Co, w, ax * n + i) : 0.0;
        R[q] = 0.0;
    }
    const Family<double> fp = family64(p, true), fw = family64(p, false);
    MaskPack<NB> nmw;
    for (int u = 0; u < TermBits<NB>::words; ++u) nmw.w[u] = 0xffffffffu;
    double mx = 0.0, s2 = 0.0;
    bool znow = false, act = false;
    int b = 0;
    for (int i = 0; i < NB; ++i) {
        for (int j = i + 1; j < NB; ++j, ++b) {
            if (j >= n) continue;
            const D3 d{pn[i] - pn[j], pn[NB + i] - pn[NB + j], pn[2 * NB + i] - pn[2 * NB + j]};
            const D3 o{po[i] - po[j], po[NB + i] - po[NB + j], po[2 * NB + i] - po[2 * NB + j]};
            const D3 x = resid64(true, o, d, fp);
            mx = fmax(mx, fmax(fabs(x.x), fmax(fabs(x.y), fabs(x.z))));
            s2 = fma(x.x, x.x, fma(x.y, x.y, fma(x.z, x.z, s2)));
            if (Rrow) {
                const D3 r = resid64(true, d, d, fp);
                R[i] += r.x, R[NB + i] += r.y, R[2 * NB + i] += r.z;
                R[j] -= r.x, R[NB + j] -= r.y, R[2 * NB + j] -= r.z;
                const double q = fma(d.z * fp.beta, d.z, fma(d.y, d.y, d.x * d.x));
                const bool zero = (d.x == 0.0 || d.y == 0.0 || d.z == 0.0) && !(q >= fp.lim);   // (hybrid: non-interior)
                znow = znow || zero;
                if (!(q >= fp.lim) || zero) {
                    nmw.w[b >> 5] &= ~(1u << (b & 31));
                    act = true;
                }
            }
        }
    }
    b = NB * (NB - 1) / 2;
    for (int i = 0; i < NB; ++i, ++b) {
        if (i >= n) continue;
        const D3 d{pn[i] - p.cx, pn[NB + i] - p.cy, pn[2 * NB + i] - p.cz};
        const D3 o{po[i] - p.cx, po[NB + i] - p.cy, po[2 * NB + i] - p.cz};
        const D3 x = resid64(false, o, d, fw);
        mx = fmax(mx, fmax(fabs(x.x), fmax(fabs(x.y), fabs(x.z))));
        s2 = fma(x.x, x.x, fma(x.y, x.y, fma(x.z, x.z, s2)));
        if (Rrow) {
            const D3 r = resid64(false, d, d, fw);
            R[i] += r.x, R[NB + i] += r.y, R[2 * NB + i] += r.z;
            const double q = fma(d.z * fw.beta, d.z, fma(d.y, d.y, d.x * d.x));
            const bool zero = (d.x == 0.0 || d.y == 0.0 || d.z == 0.0) && !(q <= fw.lim);   // (hybrid: non-interior)
            znow = znow || zero;
            if (!(q <= fw.lim) || zero) {
                nmw.w[b >> 5] &= ~(1u << (b & 31));
                act = true;
            }
        }
    }
    if (Rrow) {
        for (int q = 0; q < 3 * NB; ++q)
            if ((q % NB) < n) Rrow[q] = (T)R[q];
        *nmo = nmw;
    }
    HyStepOut<T, NB, MP> r;
    r.inf = mx;
    r.sq = s2;
    r.zero = znow;
    r.active = act;
    return r;
}


// The owner's half of the cooperative careful path: hy_step_full's reductions over its step's items, in
// hy_step_full's term order (same max, same FMA chain, same R sums).
template <typename T, int NB, int MP>
__device__ __forceinline__ HyStepOut<T, NB, MP> hy_step_coop(const double* __restrict__ it, int n, T* Rrow,
                                                         MaskPack<NB>* nmo) {
    double R[3 * NB];
#pragma unroll
    for (int q = 0; q < 3 * NB; ++q) R[q] = 0.0;
    MaskPack<NB> nmw;
#pragma unroll
    for (int u = 0; u < TermBits<NB>::words; ++u) nmw.w[u] = 0xffffffffu;
    double mx = 0.0, s2 = 0.0;
    bool znow = false, act = false;
    int b = 0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
#pragma unroll
        for (int j = i + 1; j < NB; ++j, ++b) {
            if (j >= n) continue;
            const double* e = it + kCoopItem * b;
            mx = fmax(mx, fmax(fabs(e[0]), fmax(fabs(e[1]), fabs(e[2]))));
            s2 = fma(e[0], e[0], fma(e[1], e[1], fma(e[2], e[2], s2)));
            R[i] += e[3], R[NB + i] += e[4], R[2 * NB + i] += e[5];
            R[j] -= e[3], R[NB + j] -= e[4], R[2 * NB + j] -= e[5];
            const int fl = (int)e[6];
            znow = znow || (fl & 2);
            if (fl & 1) {
                nmw.w[b >> 5] &= ~(1u << (b & 31));
                act = true;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i, ++b) {
        if (i >= n) continue;
        const double* e = it + kCoopItem * b;
        mx = fmax(mx, fmax(fabs(e[0]), fmax(fabs(e[1]), fabs(e[2]))));
        s2 = fma(e[0], e[0], fma(e[1], e[1], fma(e[2], e[2], s2)));
        R[i] += e[3], R[NB + i] += e[4], R[2 * NB + i] += e[5];
        const int fl = (int)e[6];
        znow = znow || (fl & 2);
        if (fl & 1) {
            nmw.w[b >> 5] &= ~(1u << (b & 31));
            act = true;
        }
    }
#pragma unroll
    for (int q = 0; q < 3 * NB; ++q)
        if ((q % NB) < n) Rrow[q] = (T)R[q];
    *nmo = nmw;
    HyStepOut<T, NB, MP> r;
    r.inf = mx;
    r.sq = s2;
    r.zero = znow;
    r.active = act;
    return r;
}

// Round-based cooperative careful path (HY, NB = 32: 528 terms per step; the serial hy_step_full of one
// careful step costs ~300K cycles there, with its position arrays in local memory, and stalls its slot).
// The warp takes the careful owner's step 32 terms per round: lane b evaluates term 32 r + b exactly as
// hy_step_full (FP64 positions of both iterates, resid64, the interior flags); then every lane adds, for its
// (robot, axis) entries of the R row, the round's terms in term order (bitwise hy_step_full's sums), and a
// ballot gives the round's word of interior bits.  Only the step's l2 exit partial is summed in another
// (fixed) order.
template <int NB, int MP>
__device__ __forceinline__ bool hy_careful_item2(const SolveParams& p, const double* __restrict__ pos, int b,
                                                 double* __restrict__ out, bool& off, bool& zero) {
    constexpr int NP = NB * (NB - 1) / 2;
    int i = 0, j = -1;
    if (b < NP) {
        int r = b;
        for (i = 0; i < NB; ++i) {
            if (r < NB - 1 - i) break;
            r -= NB - 1 - i;
        }
        j = i + 1 + r;
        if (j >= p.n) return false;
    } else {
        i = b - NP;
        if (i >= p.n) return false;
    }
    // term_diff64's differences, from the step's FP64 positions (pos: [iterate][axis][robot], pos64's bits)
    const double* pn = pos;
    const double* po = pos + 3 * NB;
    D3 d, o;
    if (j >= 0) {
        d = D3{pn[i] - pn[j], pn[NB + i] - pn[NB + j], pn[2 * NB + i] - pn[2 * NB + j]};
        o = D3{po[i] - po[j], po[NB + i] - po[NB + j], po[2 * NB + i] - po[2 * NB + j]};
    } else {
        d = D3{pn[i] - p.cx, pn[NB + i] - p.cy, pn[2 * NB + i] - p.cz};
        o = D3{po[i] - p.cx, po[NB + i] - p.cy, po[2 * NB + i] - p.cz};
    }
    const bool pair = j >= 0;
    const Family<double> f = family64(p, pair);
    const D3 x = resid64(pair, o, d, f), r = resid64(pair, d, d, f);
    const double q = fma(d.z * f.beta, d.z, fma(d.y, d.y, d.x * d.x));
    off = pair ? !(q >= f.lim) : !(q <= f.lim);
    zero = (d.x == 0.0 || d.y == 0.0 || d.z == 0.0) && off;   // (hybrid: non-interior)
    out[0] = x.x, out[1] = x.y, out[2] = x.z;
    out[3] = r.x, out[4] = r.y, out[5] = r.z;
    out[6] = (double)(i | ((pair ? j : 255) << 8));
    return true;
}

// outs: [0] inf, [1] sq, [2] flags (1 zero, 2 active), [3..] the interior-bit words
template <typename T, int NB, int MP>
__device__ __forceinline__ void hy_careful_rounds(const SolveParams& p, const double* Cn, const double* Co, int t,
                                                  double* __restrict__ items, double* __restrict__ outs,
                                                  T* __restrict__ Rrow, int lane) {
    constexpr int NP = NB * (NB - 1) / 2, NT = NP + NB, R3 = 3 * NB, RPL = (R3 + 31) / 32;
    double R[RPL];
#pragma unroll
    for (int u = 0; u < RPL; ++u) R[u] = 0.0;
    double mx = 0.0, s2 = 0.0;
    bool zn = false, ac = false;
    uint32_t* nmo = (uint32_t*)(outs + 3);
    double* pos = items + 32 * 8 + kCoopOwners * 12;   // [iterate][axis][robot]: each robot's FP64 positions, once
    {
        double w[MP];
        w64_row<MP>(p.W, t, p.m1, w);
        for (int q = lane; q < 3 * NB; q += 32) {
            const int ax = q / NB, i = q % NB;
            pos[q] = i < p.n ? pos64<MP>(Cn, w, ax * p.n + i) : 0.0;
            pos[3 * NB + q] = i < p.n ? pos64<MP>(Co, w, ax * p.n + i) : 0.0;
        }
    }
    __syncwarp();
    for (int r0 = 0; r0 < NT; r0 += 32) {
        const int b = r0 + lane;
        double* it = items + 8 * lane;
        bool off = false, zero = false, valid = false;
        if (b < NT) valid = hy_careful_item2<NB, MP>(p, pos, b, it, off, zero);
        if (!valid) it[6] = -1.0;
        if (valid) {
            mx = fmax(mx, fmax(fabs(it[0]), fmax(fabs(it[1]), fabs(it[2]))));
            s2 = fma(it[0], it[0], fma(it[1], it[1], fma(it[2], it[2], s2)));
        }
        const uint32_t offw = __ballot_sync(0xffffffffu, valid && (off || zero));
        zn = zn || __any_sync(0xffffffffu, valid && zero);
        ac = ac || offw != 0u;
        if (lane == 0) nmo[r0 >> 5] = ~offw;
        __syncwarp();
        const int cnt = min(32, NT - r0);
        for (int e = 0; e < cnt; ++e) {   // term order: R[i] += r (first robot / workspace), R[j] -= r
            const double* ie = items + 8 * e;
            const int code = (int)ie[6];
            if (code < 0) continue;
            const int ci = code & 0xff, cj = code >> 8;
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
                const int q = lane + 32 * u;
                if (q < R3) {
                    const int rob = q % NB, ax = q / NB;
                    if (rob == ci) R[u] += ie[3 + ax];
                    else if (rob == cj) R[u] -= ie[3 + ax];
                }
            }
        }
        __syncwarp();   // the items are rewritten next round
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
        const int q = lane + 32 * u;
        if (q < R3 && (q % NB) < p.n) Rrow[q] = (T)R[u];
    }
    if (lane == 0) {
        outs[0] = mx;
        outs[1] = s2;
        outs[2] = (double)((zn ? 1 : 0) | (ac ? 2 : 0));
    }
    __syncwarp();
}

// Flagged terms (active now or at the previous iterate) of one time step,
// O(#flagged): true exit residual, scatter of d - e for terms active now,
// and the corrections of the quiet statistics (qinf, qsq).  The quiet
// inf-norm qinf is the max of |Dp_i - Dp_j| (pairs) and |Dp_i| (workspace)
// over all terms; it stays exact for the unflagged terms unless a flagged
// term attains it, and only then is the max over the unflagged terms
// recomputed.  Runtime-indexed data comes from the position rows in shared
// memory; out of line and not unrolled, so this cold path costs little code
// next to the hot one.  Writes the R row over the (then dead) old row when a
// term is active.
template <typename T> struct StepOut {
    T inf, sq;
    bool active;
};

// insertion of (v, i) into a descending three-deep selection (registers: compile-time indices only)
template <typename T> __device__ __forceinline__ void top3_insert(T (&t)[3], int (&ti)[3], T v, int i) {
    if (v > t[2]) {
        if (v > t[1]) {
            t[2] = t[1];
            ti[2] = ti[1];
            if (v > t[0]) {
                t[1] = t[0];
                ti[1] = ti[0];
                t[0] = v;
                ti[0] = i;
            } else {
                t[1] = v;
                ti[1] = i;
            }
        } else {
            t[2] = v;
            ti[2] = i;
        }
    }
}

template <typename T, int NB, int MP, bool HY>
__device__ __forceinline__ StepOut<T> flagged_path(const T* __restrict__ Pnew, T* __restrict__ Pold, int n,
                                                   const int* __restrict__ ptab, const Family<T>& fp,
                                                   const Family<T>& fw, T cx, T cy, T cz, const MaskPack<NB>& nm,
                                                   const MaskPack<NB>& om, T qinf, T qsq, const SolveParams& p,
                                                   const double* Cn, const double* Co, int t) {
    constexpr int NP = NB * (NB - 1) / 2;
    constexpr int NWD = TermBits<NB>::words;
    const T c3[3] = {cx, cy, cz};
    T flmax = T(0), dsq = T(0);
    bool need_exact = false, act_new = false, act64 = false;
    // pass 1: exit residual of the flagged terms (needs the old row)
#pragma unroll 1
    for (int w = 0; w < NWD; ++w) {
        uint32_t fl = ~(nm.w[w] & om.w[w]);
        while (fl) {
            const int bit = __ffs(fl) - 1;
            fl &= fl - 1;
            const int b = w * 32 + bit;
            if (b >= TermBits<NB>::count) break;
            const bool in_old = (om.w[w] >> bit) & 1u;
            SGSF_COUNT(4, 1);
            act_new = act_new || !((nm.w[w] >> bit) & 1u);
            int i, j;
            term_robots<NB>(ptab, b, i, j);
            const bool pair = j >= 0;
            const Family<T>& fm = pair ? fp : fw;
            T d[3], o[3], x[3];
            T xq = T(0);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                const T ni = Pnew[ax * NB + i], oi = Pold[ax * NB + i];
                if (pair) {
                    const T nj = Pnew[ax * NB + j], oj = Pold[ax * NB + j];
                    d[ax] = ni - nj;
                    o[ax] = oi - oj;
                    x[ax] = (ni - oi) - (nj - oj);   // Dp_i - Dp_j exactly as in quiet_part
                } else {
                    d[ax] = ni - c3[ax];
                    o[ax] = oi - c3[ax];
                    x[ax] = ni - oi;
                }
                xq = fmax(xq, fabs(x[ax]));
                dsq -= x[ax] * x[ax];
            }
            need_exact = need_exact || (xq >= qinf);
            if (!in_old) {   // (HY: an FP32 measurement like the rest; the stop decision re-evaluates in FP64)
                const T qo = fma_t<T>(o[2] * fm.beta, o[2], fma_t<T>(o[1], o[1], o[0] * o[0]));
                const T so = qo > T(0) ? fm.lat * rsq<T>(qo) : T(0);
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) x[ax] = fma_t<T>(-so, o[ax], d[ax]);
            }
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                flmax = fmax(flmax, fabs(x[ax]));
                dsq = fma_t<T>(x[ax], x[ax], dsq);
            }
        }
    }
    T base = qinf;
    // the unflagged max is <= qinf; it matters only when the flagged terms' true max stays below qinf
    if (need_exact && flmax < qinf) {   // exact max of |x| over the unflagged terms (needs the old row)
        SGSF_COUNT(2, 1);
        // F <= 2 flagged terms: on each axis the max over the unflagged pairs of dp_a - dp_b is attained with
        // a among the F+1 largest and b among the F+1 smallest dp (were a outside them, the F+1 pairs
        // (top_k, b) hold an unflagged one at least as large; then the same for b), and the workspace max
        // among the F+1 largest |dp|: three-deep selections and a 3 x 3 candidate set.
        int fb0 = -1, fb1 = -1, fcnt = 0;
#pragma unroll
        for (int w = 0; w < NWD; ++w) {
            const uint32_t fl = ~(nm.w[w] & om.w[w]);
            fcnt += __popc(fl);
            if (fl) {
                fb1 = fb0;
                fb0 = w * 32 + __ffs(fl) - 1;
                const uint32_t r = fl & (fl - 1);
                if (r) fb1 = w * 32 + __ffs(r) - 1;
            }
        }
        base = T(0);
        if (fcnt <= 2) {
            SGSF_COUNT(7, 1);
#pragma unroll 1
            for (int ax = 0; ax < 3; ++ax) {
                T tv[3], bv[3], av[3];
                int ti[3], bi[3], ai[3];
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    tv[u] = T(-1e38);
                    bv[u] = T(-1e38);   // negated values: the smallest dp as the largest -dp
                    av[u] = T(-1);
                    ti[u] = bi[u] = ai[u] = -1;
                }
#pragma unroll 1
                for (int i = 0; i < n; ++i) {
                    const T v = Pnew[ax * NB + i] - Pold[ax * NB + i];
                    top3_insert(tv, ti, v, i);
                    top3_insert(bv, bi, -v, i);
                    top3_insert(av, ai, fabs(v), i);
                }
#pragma unroll
                for (int u = 0; u < 3; ++u) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const int ia = ti[u], ib = bi[k];
                        if (ia >= 0 && ib >= 0 && ia != ib) {
                            const int pb = pair_bit<NB>(min(ia, ib), max(ia, ib));
                            if (pb != fb0 && pb != fb1) base = fmax(base, tv[u] + bv[k]);
                        }
                    }
                    if (ai[u] >= 0 && ws_bit<NB>(ai[u]) != fb0 && ws_bit<NB>(ai[u]) != fb1) base = fmax(base, av[u]);
                }
            }
        }
        auto full_max = [&]() {   // every unflagged term
            T mx = T(0);
            int b = 0;
#pragma unroll 1
            for (int i = 0; i < NB; ++i) {
#pragma unroll 1
                for (int j = i + 1; j < NB; ++j, ++b) {
                    if (j < n && bit_of(nm.w, b) && bit_of(om.w, b)) {
                        T m = T(0);
#pragma unroll
                        for (int ax = 0; ax < 3; ++ax)
                            m = fmax(m, fabs((Pnew[ax * NB + i] - Pold[ax * NB + i]) - (Pnew[ax * NB + j] - Pold[ax * NB + j])));
                        mx = fmax(mx, m);
                    }
                }
            }
#pragma unroll 1
            for (int i = 0; i < n; ++i) {
                if (bit_of(nm.w, NP + i) && bit_of(om.w, NP + i)) {
                    T m = T(0);
#pragma unroll
                    for (int ax = 0; ax < 3; ++ax) m = fmax(m, fabs(Pnew[ax * NB + i] - Pold[ax * NB + i]));
                    mx = fmax(mx, m);
                }
            }
            return mx;
        };
        if (fcnt > 2) base = full_max();
#ifdef SGSF_CHECK_EXACT
        else if (full_max() != base) printf("SGSF_CHECK_EXACT mismatch: F=%d fast %g full %g\n", fcnt, (double)base, (double)full_max());
#endif
    }
    if (act_new) {
        // pass 2: the old row is dead now -- it becomes this thread's R row (d - e of the active terms)
        using V = typename Vec16<T>::type;
        constexpr int L = Vec16<T>::lanes;
        V z;
#pragma unroll
        for (int u = 0; u < L; ++u) reinterpret_cast<T*>(&z)[u] = T(0);
#pragma unroll
        for (int c = 0; c < 3 * NB / L; ++c) reinterpret_cast<V*>(Pold)[c] = z;
#ifndef SGSF_HY_NO_SCATTER   // (attribution experiments only: FP32 scattered residuals)
        if constexpr (HY) {   // FP64 scattered residuals (0 for terms interior in FP64), rounded once
#else
        if constexpr (false) {
#endif
            act64 = hy_scatter_step<T, NB, MP>(p, Cn, t, nm, ptab, Pold);   // (inline: out of line measured 0.5% slower)
        } else {
#pragma unroll 1
        for (int w = 0; w < NWD; ++w) {
            uint32_t ac = ~nm.w[w];
            while (ac) {
                const int bit = __ffs(ac) - 1;
                ac &= ac - 1;
                const int b = w * 32 + bit;
                if (b >= TermBits<NB>::count) break;
                int i, j;
                term_robots<NB>(ptab, b, i, j);
                const bool pair = j >= 0;
                const Family<T>& fm = pair ? fp : fw;
                T d[3];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) d[ax] = Pnew[ax * NB + i] - (pair ? Pnew[ax * NB + j] : c3[ax]);
                const T q = fma_t<T>(d[2] * fm.beta, d[2], fma_t<T>(d[1], d[1], d[0] * d[0]));
                const T s = fm.lat * rsq<T>(q);
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    const T r = fma_t<T>(-s, d[ax], d[ax]);
                    Pold[ax * NB + i] += r;
                    if (pair) Pold[ax * NB + j] -= r;
                }
            }
        }
        }
    }
    StepOut<T> r;
    r.inf = fmax(base, flmax);
    r.sq = fmax(qsq + dsq, T(0));
#ifndef SGSF_HY_NO_SCATTER
    r.active = HY ? act64 : act_new;   // HY: a step whose flagged terms are all interior in FP64 has R = 0
#else
    r.active = act_new;
#endif
    return r;
}

// Careful path: every term in the reference orientation, targets of terms
// with an exactly-zero component from the FP64 trig formula.  Sets the new
// interior bits (zero-component terms count as active) and whether any zero
// occurred.  Returns whether some term is active now.  Out of line: it runs
// only for (time steps of) symmetric scenarios.
template <typename T> struct CarefulOut {
    T inf, sq;
    bool zero, active;
};

// (by-value arguments: taking the address of the caller's register arrays
// would push them to local memory on the hot path)
template <typename T, int NB>
__device__ __noinline__ CarefulOut<T> careful_pass(const PosPack<T, NB> pk, T* __restrict__ Orow, int n,
                                                   const Family<T> fp, const Family<T> fw, T cx, T cy, T cz,
                                                   MaskPack<NB>* nmo) {
    const T* pos = pk.v;
    MaskPack<NB> nmw;
    uint32_t* nm = nmw.w;
    T Rrow[3 * NB];   // accumulated here; written over the (then dead) old row at the end
#pragma unroll
    for (int q = 0; q < 3 * NB; ++q) Rrow[q] = T(0);
#pragma unroll
    for (int w = 0; w < TermBits<NB>::words; ++w) nm[w] = 0xffffffffu;
    T mx = T(0), s2 = T(0);
    bool znow = false, act = false;
    int b = 0;
    for (int i = 0; i < NB; ++i) {
        for (int j = i + 1; j < NB; ++j, ++b) {
            if (i < n && j < n) {
                const T dx = pos[i] - pos[j], dy = pos[NB + i] - pos[NB + j], dz = pos[2 * NB + i] - pos[2 * NB + j];
                T rx, ry, rz, xx, xy, xz;
                T zu = T(1);
                resid<T, true, true>(dx, dy, dz, dx, dy, dz, fp, zu, rx, ry, rz);
                Rrow[i] += rx;
                Rrow[NB + i] += ry;
                Rrow[2 * NB + i] += rz;
                Rrow[j] -= rx;
                Rrow[NB + j] -= ry;
                Rrow[2 * NB + j] -= rz;
                const T ox = Orow[i] - Orow[j], oy = Orow[NB + i] - Orow[NB + j], oz = Orow[2 * NB + i] - Orow[2 * NB + j];
                resid<T, true, true>(ox, oy, oz, dx, dy, dz, fp, zu, xx, xy, xz);
                const T q = fma_t<T>(dz * fp.beta, dz, fma_t<T>(dy, dy, dx * dx));
                const bool zero = (dx == T(0)) || (dy == T(0)) || (dz == T(0));
                znow = znow || zero;
                if (!(q >= fp.lim) || zero) {
                    nm[b >> 5] &= ~(1u << (b & 31));
                    act = true;
                }
                mx = fmax(mx, fmax(fabs(xx), fmax(fabs(xy), fabs(xz))));
                s2 = fma_t<T>(xx, xx, fma_t<T>(xy, xy, fma_t<T>(xz, xz, s2)));
            }
        }
    }
    for (int i = 0; i < NB; ++i, ++b) {
        if (i < n) {
            const T rx = pos[i] - cx, ry = pos[NB + i] - cy, rz = pos[2 * NB + i] - cz;
            T ux, uy, uz, xx, xy, xz;
            T zu = T(1);
            resid<T, false, true>(rx, ry, rz, rx, ry, rz, fw, zu, ux, uy, uz);
            Rrow[i] += ux;
            Rrow[NB + i] += uy;
            Rrow[2 * NB + i] += uz;
            resid<T, false, true>(Orow[i] - cx, Orow[NB + i] - cy, Orow[2 * NB + i] - cz, rx, ry, rz, fw, zu, xx, xy,
                                  xz);
            const T q = fma_t<T>(rz * fw.beta, rz, fma_t<T>(ry, ry, rx * rx));
            const bool zero = (rx == T(0)) || (ry == T(0)) || (rz == T(0));
            znow = znow || zero;
            if (!(q <= fw.lim) || zero) {
                nm[b >> 5] &= ~(1u << (b & 31));
                act = true;
            }
            mx = fmax(mx, fmax(fabs(xx), fmax(fabs(xy), fabs(xz))));
            s2 = fma_t<T>(xx, xx, fma_t<T>(xy, xy, fma_t<T>(xz, xz, s2)));
        }
    }
    for (int q = 0; q < 3 * NB; ++q)
        if ((q % NB) < n) Orow[q] = Rrow[q];
    *nmo = nmw;
    CarefulOut<T> r;
    r.inf = mx;
    r.sq = s2;
    r.zero = znow;
    r.active = act;
    return r;
}

// FP64 exit residual (max |x|, sum x^2) of time step t for the stop decision near tol_res.  A term interior
// at the old iterate (bit set in om -- the guarded FP32 test, so interior in FP64 too) has exit residual
// Dd = D(p_i) - D(p_j) (workspace: D(p_i)), with D p = (C_k - C_{k-1}) W[t]^T: the per-axis range / max |D p|
// of the robots, O(n).  The terms non-interior at the old iterate take the FP64 target formula, and the max
// over the others comes from three-deep top / bottom selections of D p per axis (exact while at most two
// pair terms of the step are non-interior at the old iterate; beyond that the pairs are scanned).
// Register-light (inlined into the decision): the W row is streamed through the read-only cache and D p is
// recomputed rather than stored.
template <int MP>
__device__ __forceinline__ double hy_dp_s(const double* __restrict__ Cn, const double* __restrict__ Co,
                                          const double* __restrict__ Wrow, int m1, int row) {
    const double* cn = Cn + row * MP;
    const double* co = Co + row * MP;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < MP; ++q) v = fma(cn[q] - co[q], q < m1 ? __ldg(Wrow + q) : 0.0, v);
    return v;
}
// hy_dp_s with the W row in registers (the same operations)
template <int MP>
__device__ __forceinline__ double hy_dp_w(const double* __restrict__ Cn, const double* __restrict__ Co,
                                          const double (&w)[MP], int row) {
    const double* cn = Cn + row * MP;
    const double* co = Co + row * MP;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < MP; ++q) v = fma(cn[q] - co[q], w[q], v);
    return v;
}
template <int NB, int MP, typename P>
__device__ __forceinline__ double2 hy_exit64_inline(const P& p, const double* Cn, const double* Co, int t,
                                                    const uint32_t (&omr)[TermBits<NB>::words]) {
    constexpr int NP = NB * (NB - 1) / 2;
    uint32_t om[TermBits<NB>::words];   // (a copy: runtime-indexed lookups below must not pin the caller's registers)
#pragma unroll
    for (int u = 0; u < TermBits<NB>::words; ++u) om[u] = omr[u];
    const int n = p.n, m1 = p.m1;
    const double* Wrow = p.W + (size_t)t * m1;
    double wr[MP];   // the W row, once
    w64_row<MP>(p.W, t, m1, wr);
    // non-interior-at-old terms: count pairs and workspace terms, remember up to two pair bits
    int npf = 0, fb0 = -1, fb1 = -1;
    bool anyf = false;
#pragma unroll
    for (int u = 0; u < TermBits<NB>::words; ++u) {
        const int rem = TermBits<NB>::count - 32 * u;
        uint32_t f = ~om[u] & (rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u));
        anyf = anyf || f != 0u;
        while (f) {
            const int b = 32 * u + __ffs(f) - 1;
            f &= f - 1;
            if (b < NP) {
                ++npf;
                fb1 = fb0;
                fb0 = b;
            }
        }
    }
    double mx = 0.0, s2 = 0.0, base = 0.0;
#pragma unroll 1
    for (int ax = 0; ax < 3; ++ax) {
        double lo = 0.0, hi = 0.0, s1 = 0.0, sq = 0.0;
        double tv[3] = {-1e300, -1e300, -1e300}, bv[3] = {-1e300, -1e300, -1e300}, av[3] = {-1.0, -1.0, -1.0};
        int ti[3] = {-1, -1, -1}, bi[3] = {-1, -1, -1}, ai[3] = {-1, -1, -1};
        // four rows' D p at a time (independent FMA chains), consumed in row order
#pragma unroll 1
        for (int i0 = 0; i0 < n; i0 += 4) {
            double v4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v4[u] = i0 + u < n ? hy_dp_w<MP>(Cn, Co, wr, ax * n + i0 + u) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u;
                if (i >= n) break;
                const double v = v4[u];
                lo = i ? fmin(lo, v) : v;
                hi = i ? fmax(hi, v) : v;
                s1 += v;
                sq = fma(v, v, sq);
                if (anyf) {
                    top3_insert(tv, ti, v, i);
                    top3_insert(bv, bi, -v, i);
                    const int wb = NP + i;
                    if ((om[wb >> 5] >> (wb & 31)) & 1u) top3_insert(av, ai, fabs(v), i);
                }
            }
        }
        mx = fmax(mx, fmax(hi - lo, fmax(hi, -lo)));
        s2 += fmax(fma((double)(n + 1), sq, -s1 * s1), sq);
        if (anyf) {
            if (npf <= 2) {   // the max over pairs (a, b) not flagged lies among the top / bottom three
#pragma unroll
                for (int u = 0; u < 3; ++u)
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const int ia = ti[u], ib = bi[k];
                        if (ia >= 0 && ib >= 0 && ia != ib) {
                            const int pb = pair_bit<NB>(min(ia, ib), max(ia, ib));
                            if (pb != fb0 && pb != fb1) base = fmax(base, tv[u] + bv[k]);
                        }
                    }
            } else if constexpr (NB <= 16) {   // many flagged pairs: every pair interior at the old iterate, with
                // each robot's D p evaluated once (registers: this runs out of line, hy_exit64_call)
                double dv[NB];
#pragma unroll
                for (int i = 0; i < NB; ++i) dv[i] = i < n ? hy_dp_w<MP>(Cn, Co, wr, ax * n + i) : 0.0;
#pragma unroll
                for (int i = 0; i < NB; ++i)
#pragma unroll
                    for (int j = i + 1; j < NB; ++j) {
                        const int pb = pair_bit<NB>(i, j);
                        if (j < n && ((om[pb >> 5] >> (pb & 31)) & 1u)) base = fmax(base, fabs(dv[i] - dv[j]));
                    }
            } else {   // many flagged pairs: scan every pair interior at the old iterate
#pragma unroll 1
                for (int i = 0; i < n; ++i) {
                    const double vi = hy_dp_w<MP>(Cn, Co, wr, ax * n + i);
#pragma unroll 1
                    for (int j = i + 1; j < n; ++j) {
                        const int pb = pair_bit<NB>(i, j);
                        if ((om[pb >> 5] >> (pb & 31)) & 1u)
                            base = fmax(base, fabs(vi - hy_dp_w<MP>(Cn, Co, wr, ax * n + j)));
                    }
                }
            }
            if (ai[0] >= 0) base = fmax(base, av[0]);   // workspace terms interior at the old iterate
        }
    }
    if (anyf) {   // exact residuals of the terms non-interior at the old iterate; their quiet shares leave the l2 sum
        double flmax = 0.0, adj = 0.0;
#pragma unroll 1
        for (int u = 0; u < TermBits<NB>::words; ++u) {
            const int rem = TermBits<NB>::count - 32 * u;
            uint32_t f = ~om[u] & (rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u));
            while (f) {
                const int b = 32 * u + __ffs(f) - 1;
                f &= f - 1;
                int i, j;
                if (b < NP) {
                    i = 0;
                    int rest = b;
                    while (rest >= NB - 1 - i) rest -= NB - 1 - i, ++i;
                    j = i + 1 + rest;
                } else {
                    i = b - NP;
                    j = -1;
                }
                double e2 = 0.0;
#pragma unroll 1
                for (int ax = 0; ax < 3; ++ax) {
                    const double e = hy_dp_w<MP>(Cn, Co, wr, ax * n + i) -
                                     (j >= 0 ? hy_dp_w<MP>(Cn, Co, wr, ax * n + j) : 0.0);
                    e2 = fma(e, e, e2);
                }
                const D3 dn = term_diff64<MP>(p, Cn, wr, i, j), dol = term_diff64<MP>(p, Co, wr, i, j);   // (the W row in registers: pos64s's values)
                const D3 x = resid64(j >= 0, dol, dn, family64(p, j >= 0));
                flmax = fmax(flmax, fmax(fabs(x.x), fmax(fabs(x.y), fabs(x.z))));
                adj += (x.x * x.x + x.y * x.y + x.z * x.z) - e2;
            }
        }
        mx = fmax(base, flmax);
        s2 = fmax(s2 + adj, 0.0);
    }
    return make_double2(mx, s2);
}

template <int NB, int MP>
__device__ __noinline__ double2 hy_exit64_call(const HyExitArgs a, const double* Cn, const double* Co, int t,
                                               const MaskPack<NB> om) {
    return hy_exit64_inline<NB, MP>(a, Cn, Co, t, om.w);
}

// ---------------------------------------------------------------- finishing a time step
// Given the interior bits of every term (nm) and min |component| (zmin), run
// the careful / quiet / flagged path of time step `lt` and write its outputs:
// exit-residual partials, R row (over the dead old row) and its bit in the
// active-step mask of parity buffer `par`; returns its exit-residual partials.
template <typename T> struct Partials {
    T inf, sq;
};

template <typename T, int NB, int MP, bool HY>
__device__ __forceinline__ Partials<T> finish_step(const SolveParams& p, const SlotPtrs& sp, const double* Ck,
                                                   const double* Ckm1, const int* __restrict__ ptab, int lt, int n,
                                                   int par, T* __restrict__ Prow_old,
                                            const T* __restrict__ Prow_new, T qinf, T qsq,
                                            uint32_t (&nm)[TermBits<NB>::words],
                                            T zmin, uint32_t (&imask)[TermBits<NB>::words], bool& zprev,
                                            const Family<T>& fp, const Family<T>& fw, T cx, T cy, T cz,
                                            const double* pre = nullptr) {
    constexpr int NW = TermBits<NB>::words;
    T inf = qinf, sq = qsq;
    bool active = false;
    SGSF_COUNT(0, 1);
    if (__builtin_expect(zmin == T(0) || zprev, 0)) {
        SGSF_COUNT(3, 1);
        if constexpr (HY) {   // careful path from FP64 positions of both iterates
            MaskPack<NB> mo;
#ifdef SGSF_CAREFUL_CLOCK
            const long long hc0 = clock64();
#endif
            HyStepOut<T, NB, MP> co;
            if constexpr (NB <= 4) {   // (the cooperative paths: item lists for NB <= 4, rounds for NB = 32)
                co = pre ? hy_step_coop<T, NB, MP>(pre, n, Prow_old, &mo)
                         : hy_step_full<T, NB, MP>(p, Ck, Ckm1, lt, Prow_old, &mo);
            } else if constexpr (NB >= 32) {
                if (pre) {   // the warp has run hy_careful_rounds for this step: R row written, outputs here
                    const uint32_t* w = (const uint32_t*)(pre + 3);
#pragma unroll
                    for (int u = 0; u < NW; ++u) mo.w[u] = w[u];
                    const int fl = (int)pre[2];
                    co.inf = pre[0];
                    co.sq = pre[1];
                    co.zero = (fl & 1) != 0;
                    co.active = (fl & 2) != 0;
                } else {
                    co = hy_step_full<T, NB, MP>(p, Ck, Ckm1, lt, Prow_old, &mo);
                }
            } else {
                co = hy_step_full<T, NB, MP>(p, Ck, Ckm1, lt, Prow_old, &mo);
            }
#ifdef SGSF_CAREFUL_CLOCK
            if (blockIdx.x == 0 && lt < 64) printf("HC step %d hy_step_full %lld\n", lt, clock64() - hc0);
#endif
#pragma unroll
            for (int w = 0; w < NW; ++w) nm[w] = mo.w[w];
            inf = (T)co.inf;
            sq = (T)co.sq;
            active = co.active;
            zprev = co.zero;
        } else {
            PosPack<T, NB> pk;
#pragma unroll
            for (int q = 0; q < 3 * NB; ++q) pk.v[q] = ((q % NB) < n) ? Prow_new[q] : phantom_pos<T>(q % NB);
            MaskPack<NB> mo;
            const CarefulOut<T> co = careful_pass<T, NB>(pk, Prow_old, n, fp, fw, cx, cy, cz, &mo);
#pragma unroll
            for (int w = 0; w < NW; ++w) nm[w] = mo.w[w];
            inf = co.inf;
            sq = co.sq;
            active = co.active;
            zprev = co.zero;
        }
    } else {
        uint32_t any = 0u;
#pragma unroll
        for (int w = 0; w < NW; ++w) any |= ~(nm[w] & imask[w]);
        if (__builtin_expect(any != 0u, 0)) {
            MaskPack<NB> nmp, omp;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                nmp.w[w] = nm[w];
                omp.w[w] = imask[w];
            }
            SGSF_COUNT(1, 1);
            const StepOut<T> o = flagged_path<T, NB, MP, HY>(Prow_new, Prow_old, n, ptab, fp, fw, cx, cy, cz, nmp, omp,
                                                            inf, sq, p, Ck, Ckm1, lt);
            inf = o.inf;
            sq = o.sq;
            active = o.active;
        }
    }
    // (imask, the interior bits of the previous iterate, becomes nm after the stop decision: HY reads it there)
    if (active) {
        atomicOr(&sp.sh->amask[par][lt >> 5], 1u << (lt & 31));
        sp.sh->active[par] = 1;
    }
    Partials<T> r;
    r.inf = inf;
    r.sq = sq;
    return r;
}

// ---------------------------------------------------------------- load a sample (one coefficient row)
template <typename T, int NB, int MP, bool TC, bool HY>
__device__ __forceinline__ void load_row(const SolveParams& p, const SlotPtrs& sp, int sample, int r,
                                         const double* __restrict__ B6, const double* __restrict__ rhs) {
    const double* __restrict__ PBt = p.PBt;   // m1 x 6, global
    const int m1 = p.m1, dim = 3 * p.n * m1;
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
            for (int cnd = 0; cnd < 6; ++cnd) corr = q < m1 ? fma(PBt[q * 6 + cnd], res[cnd], corr) : corr;
            c[q] = x[q] - corr;
            l[q] = 0.0;
        }
    }
#pragma unroll
    for (int q = 0; q < MP; ++q) {
        const int idx = r * MP + q;
        sp.xb[idx] = x[q];
        sp.C[idx] = c[q];
        sp.lam[idx] = l[q];
        if (p.want_prev || HY) sp.Cp[idx] = c[q];
    }
    const int ax = r / p.n, i = r - ax * p.n;
    if constexpr (TC) {
        unsigned char* b = (unsigned char*)sp.Cf + ax * 2048;
#pragma unroll
        for (int q = 0; q < MP; ++q) {
            const float v = (float)c[q], hi = tc::tf32_rna(v);
            *reinterpret_cast<float*>(b + tc::kmajor16_offset(i, q)) = hi;
            *reinterpret_cast<float*>(b + 1024 + tc::kmajor16_offset(i, q)) = tc::tf32_rna(v - hi);
        }
        tc::fence_proxy_async();   // visible to the tensor core after the next slot barrier
    } else {
#pragma unroll
        for (int q = 0; q < MP; ++q) ((T*)sp.Cf)[(ax * MP + q) * NB + i] = (T)c[q];
    }
}

// TC: the 3xTF32 position GEMM of one axis, D[step][robot] = W[step] . C[robot], issued by one thread.
// A (W rows of the slot's steps, tf32 hi at TMEM columns 0..15, lo at 16..31) is shared by the slots;
// B = this axis' C hi / lo blocks; the small products go first (FP32-level accuracy).
__device__ __forceinline__ void tc_issue_axis(uint32_t tbase, int slot, int ax, const void* cf) {
    constexpr uint32_t idesc = tc::idesc_tf32(128, 16);
    const uint32_t d = tbase + 64 + 64 * slot + 16 * ax;
    // descriptor of the axis' B block; the start-address field (16-byte units) takes the offsets directly
    const uint64_t bd = tc::smem_desc(tc::smem_u32(cf) + ax * 2048, 128, 512);
    constexpr uint32_t acol[3] = {0, 16, 0}, bofs[3] = {1024, 0, 0};   // W_hi C_lo, W_lo C_hi, W_hi C_hi
#pragma unroll
    for (int pr = 0; pr < 3; ++pr)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
            tc::mma_tf32_ts(d, tbase + acol[pr] + 8 * ks, bd + ((bofs[pr] + 256 * ks) >> 4), idesc, (pr | ks) ? 1u : 0u);
}

// Time step of lane `lane` of warp `lwarp` in a slot of `wps` warps, one thread per step.  Steps go to the
// warps in 8-step chunks (warp w takes chunks w, w + wps, ...): every warp covers the whole horizon (the
// exact-path work clusters in time) and 8 consecutive rows keep the 16-byte row accesses conflict-free.
// (Dealing the horizon's last group step by step, for equal step counts, measured 0.7% slower: the
// barrier spread comes from where the flagged steps fall, not from the counts.)
__host__ __device__ __forceinline__ int step_of(int lwarp, int lane, int wps, int /*S*/) {
    return 8 * (lwarp + wps * (lane >> 3)) + (lane & 7);
}

// ||A xi - b||_inf over one axis' rows of the iterate C (assembly.py:198-199): E[robot][c6] = B6[c6] . C_robot -
// rhs as FP64 tensor-core tiles, max-reduced over the warp.  Called by the axis warps at the top of the next
// iteration, where it overlaps the wait for the position MMAs instead of lengthening the xi-step's chain.
template <int MT, int MP>
__device__ __forceinline__ double eq_check_axis(const double* __restrict__ C, const double* __restrict__ B6,
                                                const double* __restrict__ rhs, int rb, int n, int lane) {
    const int fr = lane >> 2, fc = lane & 3;
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
    return warp_max_nonneg(em);
}

// ---------------------------------------------------------------- the kernel
// TC = positions by the 3xTF32 tcgen05 GEMM (float, 16 robots, one thread per step, 4 warps per slot)
// FULLN: 0 = both term-pass variants, chosen at run time by n == NB; 1 = only the phantom-free one
// (n == NB); 2 = only the one with phantoms (n < NB).  A single variant keeps the hot loop's code small.
template <typename T, int NB, int MP, int MAXT, int TPS, bool TC = false, int FULLN = 0, bool HY = false>
__global__ void __launch_bounds__(MAXT, 1) sf_persistent_kernel(const SolveParams p) {
    static_assert(!TC || (sizeof(T) == 4 && NB == 16 && TPS == 1 && MP <= 16), "TC positions: float, 16 robots");
    static_assert(!HY || sizeof(T) == 4, "hybrid precision screens in FP32");
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLayout& L = p.L;   // = make_layout<T, NB>(p.n, p.S, MP, p.spb, p.want_prev, TC), host-computed
    constexpr int RS = RowStride<T, NB>::value;
    constexpr int M2P = 2 * MP;
    constexpr int NW = TermBits<NB>::words;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int n = p.n, S = p.S, m1 = p.m1;
    const int R3 = 3 * n, dim = R3 * m1, dimp = R3 * MP;

    T* Wt = (T*)(smem + L.W);
    double* KMm = (double*)(smem + L.KMm);
    double* KMd = (double*)(smem + L.KMd);
    double* cconst = (double*)(smem + L.cconst);
    double* B6 = (double*)(smem + L.B6);
    double* rhs = (double*)(smem + L.rhs);

    // shared constants, zero-padded to MP columns
    for (int i = tid; i < S * MP; i += nt) {
        const int t = i / MP, q = i % MP;
        Wt[i] = (q < m1) ? (T)p.W[t * m1 + q] : T(0);
    }
    for (int i = tid; i < MP * M2P; i += nt) {
        const int q = i / M2P, c = i % M2P, half = c / MP, q2 = c % MP;
        const bool in = q < m1 && q2 < m1;
        // [Mm - Md | Km11 - Kd11]: the xi-step takes the raw rows (see MX)
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
    int* ptab = (int*)(smem + L.ptab);   // pair index -> (i | j << 8), lexicographic i < j
    if (tid == 0) {
        int b = 0;
        for (int i = 0; i < NB; ++i)
            for (int j = i + 1; j < NB; ++j) ptab[b++] = i | (j << 8);
    }
    uint32_t* tmem_info = (uint32_t*)(smem + L.tmem);   // [0] TMEM base, [1] finished slots
    if constexpr (TC) {
        // TMEM: columns 0..31 = A operand (W rows, tf32 hi / lo), 64 + 64 s = slot s's 16 x 3 positions
        if (tid < 32) tc::tmem_alloc(tmem_info, 256);
        if (tid == 0) {
            tmem_info[1] = 0u;
            for (int s = 0; s < p.spb; ++s) tc::mbar_init(&slot_ptrs(smem, L, s).sh->mbar, 3);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        for (int s = 0; s < p.spb; ++s) {   // B operands start at zero (k >= m1 and robots >= n stay zero)
            uint32_t* b = (uint32_t*)slot_ptrs(smem, L, s).Cf;
            for (int e = tid; e < kTcBopBytes / 4; e += nt) b[e] = 0u;
        }
    }
    __syncthreads();
    if constexpr (TC) {
        const uint32_t tb = tmem_info[0];
        if (tid < 128) {   // A rows: TMEM lane 32 w + l holds the step of lane l of warp w (4 warps per slot)
            const int w = tid >> 5, l = tid & 31, t = step_of(w, l, 4, S);
            float hi[16], lo[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const float v = (t < S && q < m1) ? (float)p.W[t * m1 + q] : 0.f;
                hi[q] = tc::tf32_rna(v);
                lo[q] = tc::tf32_rna(v - hi[q]);
            }
            const uint32_t la = tb + ((uint32_t)(32 * w) << 16);
            tc::tmem_st16(la, hi);
            tc::tmem_st16(la + 16, lo);
            tc::tmem_wait_st();
        }
        tc::fence_proxy_async();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
    }

    // ---- this thread's slot (an independent warp group)
    const int gsize = 32 * p.wps;
    const int slot = tid / gsize, lt = tid - slot * gsize, lane = lt & 31, lwarp = lt >> 5;
    if (slot >= p.spb) return;
    const int bar_id = 1 + slot;
    const SlotPtrs sp = slot_ptrs(smem, L, slot);
    Family<T> fp, fw;   // = make_family<T>(lat, vert), from the parameter bank
    if constexpr (sizeof(T) == 4) {
        fp.lat = p.fp_lat_f, fp.lim = HY ? p.hy_fp_lim_f : p.fp_lim_f, fp.beta = p.fp_beta_f;
        fw.lat = p.fw_lat_f, fw.lim = HY ? p.hy_fw_lim_f : p.fw_lim_f, fw.beta = p.fw_beta_f;
    } else {
        fp.lat = p.lat, fp.lim = p.fp_lim_d, fp.beta = p.fp_beta_d;
        fw.lat = p.ws_lat, fw.lim = p.fw_lim_d, fw.beta = p.fw_beta_d;
    }
    fp.lat64 = p.lat, fp.vert64 = p.vert, fw.lat64 = p.ws_lat, fw.vert64 = p.ws_vert;
    const T cx = (T)p.cx, cy = (T)p.cy, cz = (T)p.cz;
    const int SWT = (S + 31) >> 5;   // words of the active-step mask
    const double inv_n = 1.0 / n;
    const T inv_lat = T(1) / fp.lat;
    // the residual history is written by a warp that has no axis in MX when there is one
    const int hist_lt = p.wps > 3 ? 32 * (p.wps - 1) : 0;
    // time step of this thread and the part of the robots it owns: TPS = 2 puts the two halves
    // of a step in lanes l and l ^ 16 (16 steps per warp); the h = 0 lane owns the step's state
    constexpr int RH = NB / TPS;
    // TPS = 1: steps are dealt to the warps by step_of (8-step chunks over the whole horizon, equal counts)
    const int wpsx = TC ? 4 : p.wps;   // TC: four warps per slot
    const int ts = TPS == 2 ? lwarp * 16 + (lane & 15) : step_of(lwarp, lane, wpsx, S);
    const int h = TPS == 2 ? lane >> 4 : 0;
    const int r0 = h * RH;
    const bool owner = h == 0;
    const unsigned smask = __ballot_sync(0xffffffffu, ts < S);   // lanes of this warp with a step
    if constexpr (HY && NB <= 4 && TPS == 1 && !TC) {   // careful-path target cache: no entry valid yet
        constexpr int NT = NB * (NB - 1) / 2 + NB;
        if (S <= kCoopMaxS) {
            long long* tags = (long long*)(sp.ct + (size_t)S * NT * 3);
            for (int e = lt; e < S * NT; e += gsize) tags[e] = -1;
        }
    }

    constexpr int NP = NB * (NB - 1) / 2;
    constexpr int NPW = (NP + 31) / 32;   // words holding pair bits
#ifdef SGSF_PHASE_TIMING
    // clock64 stamps of slot 0 / thread 0 of CTA 0: [0] loop top (after MX barrier), [5] T1 end,
    // [6] T2 end, [1] after the term-pass barrier, [2] after decision, [3] after G, [4] after MX barrier
    long long pt_last = 0, pt_acc[16] = {0};
    __shared__ long long pt_arrive[4];
    long long pt_spread = 0;
    int pt_lastw[4] = {0, 0, 0, 0};
    int pt_prev = -1, pt_iters = 0;
#define SGSF_PT(ID)                                                                          \
    do {                                                                                      \
        if (tid == 0) {                                                                        \
            const long long now = clock64();                                                  \
            if (pt_prev >= 0) pt_acc[ID] += now - pt_last;                                    \
            pt_last = now;                                                                    \
            pt_prev = ID;                                                                     \
            if (ID == 0) ++pt_iters;                                                          \
        }                                                                                     \
    } while (0)
#else
#define SGSF_PT(ID) ((void)0)
#endif
    uint32_t imask[NW];
    bool zprev = false;
#ifdef SGSF_NEAR_CLOCK
    long long near_cyc = 0;   // this warp's cycles in the T1 near-pair checks (diagnostics)
    int near_its = 0;
#endif
    // Verlet-style pair list: the last scan of this time step split the pairs
    // into "near" (normalised distance < kSkin; their bits in `near`, checked
    // exactly every iteration) and "far" (distance >= rmin >= kSkin).  Since
    // the scan every pair moved by at most cum (sum over iterations of
    // 2 max_i |Dp_i|, normalised), so while rmin - cum > 1 + margin every far
    // pair is provably interior and needs no test.
    constexpr float kSkin = 1.5f;
    const T skin_lim = T(kSkin * kSkin) * fp.lim;
    uint32_t near[NPW];
    T rmin = T(0), cum = T(0);
    bool prev_active = false;   // lam changed in the previous iteration (the U rows are stale)

    if (lt == 0) {
        sp.sh->sample = next_sample(p);
        clear_flags(sp.sh, 0, SWT);
        clear_flags(sp.sh, 1, SWT);
    }
    slot_barrier(bar_id, gsize);
    int sample = sp.sh->sample;

    uint32_t mph = 0;   // TC: parity of the slot's next position-MMA completion
    const uint32_t tbase = TC ? tmem_info[0] : 0u;
    while (sample < p.batch) {
        // ---------------- load the sample, default start = boundary projection
        for (int r = lt; r < R3; r += gsize) load_row<T, NB, MP, TC, HY>(p, sp, sample, r, B6, rhs);
        slot_barrier(bar_id, gsize);
        if constexpr (TC) {
            if (lwarp == 0) {   // positions of the first iterate (warp-uniform operands, one elected lane)
                const uint32_t tb_u = __shfl_sync(0xffffffffu, tbase, 0);
                const int slot_u = __shfl_sync(0xffffffffu, slot, 0);
                if (tc::elect_one()) {
                    tc::fence_after_sync();
#pragma unroll 1
                    for (int ax = 0; ax < 3; ++ax) {
                        tc_issue_axis(tb_u, slot_u, ax, sp.Cf);
                        tc::mma_commit(&sp.sh->mbar);
                    }
                }
            }
        }

        for (int k = 0;; ++k) {
#ifdef SGSF_NEAR_CLOCK
            ++near_its;
#endif
            SGSF_PT(0);
            const int par = k & 1;
            // HY: C_k and C_{k-1} alternate between the C and Cp buffers (the xi-step writes C_{k+1} over C_{k-1});
            // otherwise C is updated in place and Cp is a copy (want_prev)
            double* const Ccur = (HY && par) ? sp.Cp : sp.C;
            double* const Cprv = (HY && par) ? sp.C : sp.Cp;
            double* const Cnext = HY ? Cprv : Ccur;   // where the xi-step writes C_{k+1}
            if (lt == 0) clear_flags(sp.sh, par ^ 1, SWT);   // last read before the previous closing barrier
            // position rows: old = iterate k, new = iterate k+1's input positions; R -> old row
            T* const Pbase_new = (T*)((k & 1) ? sp.P0 : sp.P1);
            T* Prow_old = (T*)((k & 1) ? sp.P1 : sp.P0) + ts * RS;
            T* Prow_new = Pbase_new + ts * RS;
            if (k >= 1) {   // ||A xi - b|| of the iterate the previous xi-step wrote (read after the term-pass barrier)
                constexpr int MTE = (NB + 7) / 8;
                for (int ax = lwarp; ax < 3; ax += p.wps) {
                    const double em = eq_check_axis<MTE, MP>(Ccur, B6, rhs, ax * n, n, lane);
                    if (lane == 0) sp.eqerr[ax] = em;
                }
            }
            // ---------------- T1: positions, O(n) statistics, workspace terms, motion bound, near pairs
            bool need_scan = false;
            uint32_t nm[NW];
            T zmin_ws = T(1), qinf = T(0), qsq = T(0);   // quiet statistics, kept for T3
            T pos[3 * RH];
            if constexpr (TC) {   // warp-collective TMEM loads, before the per-step branch
                tc::mbar_wait(&sp.sh->mbar, mph);
                mph ^= 1u;
                tc::fence_after_sync();
                const uint32_t ta = tbase + ((uint32_t)(32 * lwarp) << 16) + 64 + 64 * slot;
                tc::tmem_ld16(ta, *reinterpret_cast<float(*)[16]>(&pos[0]));
                tc::tmem_ld16(ta + 16, *reinterpret_cast<float(*)[16]>(&pos[16]));
                tc::tmem_ld16(ta + 32, *reinterpret_cast<float(*)[16]>(&pos[32]));
                tc::tmem_wait_ld();
                tc::fence_before_sync();
                SGSF_PT(15);   // phase timing: the wait for the position MMAs + TMEM loads
                if (n < NB) {   // uniform: phantom robots only in the smaller swarms
#pragma unroll
                    for (int q = 0; q < 3 * RH; ++q)
                        if ((q % RH) >= n) pos[q] = phantom_pos<T>(q % RH);
                }
            }
            if (ts < S) {
#ifndef SGSF_NO_POS   // (timing experiments only: positions from the first iterate, results wrong)
                if constexpr (!TC) positions_part<T, NB, RH, MP>(Wt, (const T*)sp.Cf, ts, r0, n, pos);
#else
                if constexpr (!TC) if (k == 0) positions_part<T, NB, RH, MP>(Wt, (const T*)sp.Cf, ts, r0, n, pos);
#endif
                store_part<T, NB, RH>(Prow_new, r0, pos);
                if (k == 0) {
                    store_part<T, NB, RH>(Prow_old, r0, pos);   // no previous iterate: "old" := "new"
#pragma unroll
                    for (int w = 0; w < NW; ++w) imask[w] = 0xffffffffu;
                    zprev = false;
                }
                const bool full = FULLN == 1 || (FULLN == 0 && n == NB);   // no phantom robots: guard-free trees
                PartStats<T> st;
                if (FULLN == 1 || (FULLN == 0 && full))
                    st = quiet_part<T, NB, RH, TPS, FULLN != 2>(pos, Prow_old, r0, n, fp.beta, smask);
                else
                    st = quiet_part<T, NB, RH, TPS, false>(pos, Prow_old, r0, n, fp.beta, smask);
                qinf = st.inf;
                qsq = st.sq;
                cum += T(2) * sqrt(st.dmax2) * inv_lat;
                need_scan = (k == 0) || zprev || !(rmin - cum > T(1) + T(1e-3));
                if (FULLN == 1 || (FULLN == 0 && full))
                    zmin_ws = ws_part<T, NB, RH, TPS, FULLN != 2, HY>(pos, r0, h, n, fw, cx, cy, cz, nm, smask);
                else
                    zmin_ws = ws_part<T, NB, RH, TPS, false, HY>(pos, r0, h, n, fw, cx, cy, cz, nm, smask);
            }
            __syncwarp();   // both halves of every row written before the owners and the scans read them
#ifdef SGSF_NEAR_CLOCK
            const long long nc0 = clock64();
#endif
            if (ts < S && owner && !need_scan) {   // near pairs of the last scan, exactly (a pair active before is near)
#pragma unroll
                for (int w = 0; w < NPW; ++w) {
                    uint32_t bits = near[w];
                    while (bits) {
                        const int bit = __ffs(bits) - 1;
                        bits &= bits - 1;
                        SGSF_COUNT(5, 1);
                        const int ij = ptab[w * 32 + bit], i = ij & 0xff, j = ij >> 8;
                        const T dx = Prow_new[i] - Prow_new[j], dy = Prow_new[NB + i] - Prow_new[NB + j];
                        const T dz = Prow_new[2 * NB + i] - Prow_new[2 * NB + j];
                        const T q = fma_t<T>(dz * fp.beta, dz, fma_t<T>(dy, dy, dx * dx));
                        // (HY: zero components of interior terms do not send the step to the careful path)
                        if (!HY) zmin_ws = fmin(zmin_ws, fmin(fabs(dx), fmin(fabs(dy), fabs(dz))));
                        if (!(q >= fp.lim)) {
                            nm[w] &= ~(1u << bit);
                            if (HY) zmin_ws = fmin(zmin_ws, fmin(fabs(dx), fmin(fabs(dy), fabs(dz))));
                        }
                    }
                }
            }

#ifdef SGSF_NEAR_CLOCK
            __syncwarp();
            if (lane == 0) near_cyc += clock64() - nc0;
#endif
            SGSF_PT(5);
            // ---------------- T2: warp-local O(n^2) pair scans of this warp's queued time steps: all 32 lanes
            // take 1/32 of the pairs of one step; ballots give the non-interior pair bits, REDUX the minima
            T zmin_pairs = T(1);
            uint32_t qmask = __ballot_sync(0xffffffffu, ts < S && owner && need_scan);
            while (qmask) {
                const int src = __ffs(qmask) - 1;
                qmask &= qmask - 1;
                if (lane == 0) SGSF_COUNT(6, 1);
                const int tsrc = TPS == 2 ? lwarp * 16 + src : step_of(lwarp, src, wpsx, S);
                const T* row = Pbase_new + tsrc * RS;
                T qm = T(1e30), zm = T(1);   // min q over the far pairs, min |component| over all pairs
                uint32_t words[NPW], nwords[NPW];
#pragma unroll
                for (int u = 0; u < NPW; ++u) {
                    const int bb = u * 32 + lane;
                    bool outside = false, is_near = false;
                    if (bb < NP) {
                        const int ij = ptab[bb], i = ij & 0xff, j = ij >> 8;
                        if (j < n) {
                            const T dx = row[i] - row[j], dy = row[NB + i] - row[NB + j];
                            const T dz = row[2 * NB + i] - row[2 * NB + j];
                            const T q = fma_t<T>(dz * fp.beta, dz, fma_t<T>(dy, dy, dx * dx));
                            zm = fmin(zm, (HY && q >= fp.lim) ? T(1) : fmin(fabs(dx), fmin(fabs(dy), fabs(dz))));
                            is_near = !(q >= skin_lim);
                            if (!is_near) qm = fmin(qm, q);
                            outside = !(q >= fp.lim);
                        }
                    }
                    words[u] = __ballot_sync(0xffffffffu, outside);
                    nwords[u] = __ballot_sync(0xffffffffu, is_near);
                }
                qm = warp_min_nonneg(qm);
                zm = warp_min_nonneg(zm);
                if (lane == src) {
                    rmin = sqrt(qm) * inv_lat;
                    cum = T(0);
                    zmin_pairs = zm;
#pragma unroll
                    for (int u = 0; u < NPW; ++u) {
                        nm[u] &= ~words[u];
                        near[u] = nwords[u];
                    }
                }
            }

            SGSF_PT(6);
            // ---------------- T3: every time step finishes (quiet / flagged / careful path), by its owner lane
            Partials<T> pr{T(0), T(0)};
            const double* pre = nullptr;
#ifdef SGSF_CAREFUL_CLOCK
            const long long cc0 = clock64();
#endif
            if constexpr (HY && NB <= 4 && TPS == 1 && !TC) {   // careful steps: spread their trig over the warp
                constexpr int NT = NB * (NB - 1) / 2 + NB;
                const bool car = ts < S && (fmin(zmin_ws, zmin_pairs) == T(0) || zprev);
                const uint32_t bal = __ballot_sync(0xffffffffu, car);
                const int nc = __popc(bal);
                if (nc != 0 && nc * NT <= 32 && p.coop && S <= kCoopMaxS) {
                    double* scr = sp.cp + (size_t)lwarp * 32 * kCoopItem;
                    const int kk = lane / NT, bb = lane - kk * NT;
                    const int src = kk < nc ? (int)__fns(bal, 0, kk + 1) : 0;
                    const int tsrc = __shfl_sync(0xffffffffu, ts, src);
                    if (kk < nc)
                        hy_careful_item<NB, MP>(p, Ccur, Cprv, tsrc, bb, scr + kCoopItem * lane, sp.ct,
                                                ((long long)sample << 32) | (unsigned)k);
                    __syncwarp();
                    if (car) pre = scr + kCoopItem * NT * __popc(bal & ((1u << lane) - 1u));
                }
            }
            if constexpr (HY && NB >= 32 && !TC) {   // careful steps: the warp takes each in rounds of 32 terms
                const bool car = ts < S && owner && (fmin(zmin_ws, zmin_pairs) == T(0) || zprev);
                uint32_t bal = __ballot_sync(0xffffffffu, car);
                if (bal && p.coop && (bal >> kCoopOwners) == 0u) {   // (owners are lanes 0..15: two lanes per step)
                    double* wbase = sp.cw + (size_t)lwarp * kCoopWarpDoubles;
                    while (bal) {
                        const int src = __ffs(bal) - 1;
                        bal &= bal - 1;
                        const int tso = __shfl_sync(0xffffffffu, ts, src);
                        T* rowo = (T*)((k & 1) ? sp.P1 : sp.P0) + tso * RS;
                        hy_careful_rounds<T, NB, MP>(p, Ccur, Cprv, tso, wbase, wbase + 256 + 12 * src, rowo, lane);
                    }
                    if (car) pre = wbase + 256 + 12 * lane;
                }
            }
#ifdef SGSF_CAREFUL_CLOCK
            const long long cc1 = clock64();
            const bool was_careful = ts < S && (fmin(zmin_ws, zmin_pairs) == T(0) || zprev);
#endif
            if (ts < S && owner)
                pr = finish_step<T, NB, MP, HY>(p, sp, Ccur, Cprv, ptab, ts, n, par, Prow_old, Prow_new, qinf, qsq, nm, fmin(zmin_ws, zmin_pairs),
                                        imask, zprev, fp, fw, cx, cy, cz, pre);
#ifdef SGSF_CAREFUL_CLOCK
            if (blockIdx.x == 0 && slot == 0 && k < 6 && was_careful)
                printf("CC k %d step %d coop %lld finish %lld pre %d\n", k, ts, cc1 - cc0, clock64() - cc1, pre != nullptr);
#endif
            {   // per-warp exit-residual partials for the decision (fixed order: deterministic); the l2
                // partial is summed over the warp in T (FP32 lean: the history is an l2 norm, checked to
                // 1e-3) and across the warps in FP64
                const T wi = warp_max_nonneg(pr.inf);
                T wqt = pr.sq;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) wqt += __shfl_xor_sync(0xffffffffu, wqt, off);
                const double wq = (double)wqt;
                if (lane == 0) {
                    ((T*)sp.pinf)[lwarp] = wi;
                    sp.psq[lwarp] = wq;
                }
            }
#ifdef SGSF_PHASE_TIMING
            if (slot == 0 && lane == 0 && lwarp < 4) pt_arrive[lwarp] = clock64();   // term-pass barrier arrivals
#endif
            slot_barrier(bar_id, gsize);
            SGSF_PT(1);
#ifdef SGSF_PHASE_TIMING
            if (tid == 0) {   // spread of the four warps' arrivals and which one came last
                long long lo = pt_arrive[0], hi = pt_arrive[0];
                int last = 0;
                for (int w = 1; w < 4; ++w) {
                    lo = min(lo, pt_arrive[w]);
                    if (pt_arrive[w] > hi) hi = pt_arrive[w], last = w;
                }
                pt_spread += hi - lo;
                ++pt_lastw[last];
            }
#endif

            // ---------------- decision (every warp, redundantly): exit residual of iteration k-1, early stop, SingularKKT
            // ||A xi - b|| of the iterate C_k: written by the axis warps at the top of this iteration, before the
            // term-pass barrier; rewritten at the top of the next one, after the closing barrier (race-free)
            const double emax = k >= 1 ? fmax(fmax(sp.eqerr[0], sp.eqerr[1]), sp.eqerr[2]) : 0.0;
            double sqs = 0.0;
            T inf = T(0);
            if (k >= 1) {   // partials: per axis (MX of iteration k-1, read above), per warp (T3 above)
                if (TC) {   // 4 warps per slot: independent loads, fixed summation order
                    T pi[4];
                    double ps[4];
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        pi[w] = ((const T*)sp.pinf)[w];
                        ps[w] = sp.psq[w];
                    }
                    inf = fmax(fmax(pi[0], pi[1]), fmax(pi[2], pi[3]));
                    sqs = ((ps[0] + ps[1]) + ps[2]) + ps[3];
                } else {
                    for (int w = 0; w < p.wps; ++w) {
                        inf = fmax(inf, ((const T*)sp.pinf)[w]);
                        sqs += sp.psq[w];
                    }
                }
            }
            double infd = (double)inf;
#ifndef SGSF_HY_NO_RECOMPUTE   // (attribution experiments only: drops the FP64 stop re-evaluation)
            if constexpr (HY) {
#else
            if constexpr (false) {
#endif
                // the FP32-measured exit residual sits within hy_delta of tol_res (slot-uniform: every warp
                // read the same partials): re-evaluate it in FP64 over every time step, so the stop decision
                // is the one the FP64 iterates give
                if (k >= 1 && p.early_stop && fabs(infd - p.tol_res) <= p.hy_delta) {
                    if (lt == 0) SGSF_COUNT(8, 1);
#ifdef SGSF_HY_CLOCK
                    const long long hyc0 = clock64();
#endif
                    double xi = 0.0, xs = 0.0;
                    if (ts < S && owner) {
                        MaskPack<NB> om;
#pragma unroll
                        for (int w = 0; w < NW; ++w) om.w[w] = imask[w];
                        const double2 e = hy_exit64_call<NB, MP>(hy_exit_args(p), Ccur, Cprv, ts, om);
                        xi = e.x;
                        xs = e.y;
                    }
                    xi = warp_max_nonneg(xi);
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, off);
                    const int pw = TC ? 4 : MAX_SLOT_WORDS;
                    if (lane == 0) {
                        sp.pex[lwarp] = xi;
                        sp.pex[pw + lwarp] = xs;
                    }
                    slot_barrier(bar_id, gsize);
                    infd = 0.0;
                    sqs = 0.0;
                    for (int w = 0; w < p.wps; ++w) {
                        infd = fmax(infd, sp.pex[w]);
                        sqs += sp.pex[pw + w];
                    }
#ifdef SGSF_HY_CLOCK
                    if (lt == 0 && blockIdx.x < 2) printf("HYC cta %d slot %d k %d cycles %lld\n", blockIdx.x, slot, k, clock64() - hyc0);
#endif
                }
            }
            if (ts < S && owner) {   // interior bits of this iterate: the "old" ones of the next
#pragma unroll
                for (int w = 0; w < NW; ++w) imask[w] = nm[w];
            }
            // (a sample can only finish at k >= 1, so `infd` is always the last exit residual there)
            const bool failed = (k >= 1) && (emax > p.tol_eq);
            bool done = failed;
            if (k >= 1) {
                done = done || (p.early_stop && infd <= p.tol_res) || (k >= p.max_iters);
                if (lt == hist_lt) {
                    const size_t hix = (size_t)sample * p.max_iters + (k - 1);
                    p.res_inf[hix] = infd;
                    p.res_l2[hix] = sqrt(sqs);
                }
            }

#ifdef SGSF_SYNC_CHECK
            {   // debug build: every warp of the slot must take the same decision (the slot's barriers depend on it)
                int* sc_dec = (int*)(smem + L.slot0 + (size_t)slot * L.slot_stride + L.sc);
                if (lane == 0) sc_dec[lwarp] = (int)done | ((int)failed << 1) | ((k & 0xffff) << 2);
                slot_barrier(bar_id, gsize);
                if (lt == 0)
                    for (int w = 1; w < p.wps; ++w)
                        if (sc_dec[w] != sc_dec[0]) {
                            printf("SGSF_SYNC_CHECK: slot %d warp %d decision %x != warp 0 %x (sample %d, k %d)\n", slot,
                                   w, sc_dec[w], sc_dec[0], sample, k);
                            __trap();
                        }
                slot_barrier(bar_id, gsize);
            }
#endif
            if (done) {
                // ---------------- finalize: outputs of the returned iterate, claim the next sample
                if (!failed) {
                    for (int e = lt; e < dim; e += gsize) {
                        const int r = e / m1, q = e - r * m1;
                        const size_t o = (size_t)sample * dim + e;
                        p.coeffs[o] = Ccur[r * MP + q];
                        p.mult[o] = sp.lam[r * MP + q];
                        if (p.want_prev && p.coeffs_prev) p.coeffs_prev[o] = Cprv[r * MP + q];
                    }
                }
                if (lwarp == 0) {
                    double acc = 0.0;
                    for (int e = lane; e < dimp; e += 32) {
                        const double dd = Ccur[e] - sp.xb[e];
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
                        sp.sh->sample = next_sample(p);
                        // nothing reads the flags in a final iteration
                        clear_flags(sp.sh, 0, SWT);
                        clear_flags(sp.sh, 1, SWT);
                    }
                }
                slot_barrier(bar_id, gsize);
                sample = sp.sh->sample;
                break;
            }

            SGSF_PT(2);
            const bool any_active = sp.sh->active[par] != 0;

            // ---------------- MX: one warp per axis; rows of an axis never leave their warp, so its
            // sub-steps are ordered by __syncwarp alone.  All products are FP64 tensor-core tiles
            // (DMMA m8n8k4, rows = robots), with the accumulators D[robot][q] held in registers:
            //   G   g = R W over the active time steps (k = active step, compacted in ascending t);
            //       lam' = lam - rho g                                    (only when something was active)
            //   U   u_i = 2 lam'_i - lam_i + xi_bar_i   (only when lam changed now or in the last iteration)
            //   X   C_i = Md C_i + Kd11 u_i + cconst_i + (Mm - Md) Cb + (Km11 - Kd11) ub
            //       (= the decoupled xi-step Mm Cb + Km11 ub + Md (C_i - Cb) + Kd11 (u_i - ub) + cconst_i):
            //       [robots x (C | u)] . [Md | Kd11]^T, plus the column sums of the same fragments (n Cb,
            //       n ub) times [Mm - Md | Km11 - Kd11]^T / n for every row
            //   E   ||A xi - b||_inf over the new rows (B6 C_i - rhs_i), commit
            {
                constexpr int MT = (NB + 7) / 8;   // 8-robot tiles
                constexpr int KT = MP / 2;         // 4-column k-steps over [C | u]
                constexpr int KC = MP / 4;         // ... of which over C
                const bool u_stale = any_active || prev_active || k == 0;
                const int fr = lane >> 2, fc = lane & 3;   // fragment row / column
                for (int ax = lwarp; ax < 3; ax += p.wps) {
                    const int rb = ax * n;   // first row of this axis
                    double gq[MT][2][2];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt) gq[mt][nt][0] = gq[mt][nt][1] = 0.0;
                    if (any_active) {   // G
                        const uint32_t* am = sp.sh->amask[par];
                        int na = 0, c0 = 0, c1 = 0, c2 = 0;   // TC (4 mask words): prefix counts of the words
                        if constexpr (TC) {
                            c0 = __popc(am[0]);
                            c1 = c0 + __popc(am[1]);
                            c2 = c1 + __popc(am[2]);
                            na = c2 + __popc(am[3]);
                        } else {
                            for (int w = 0; w < SWT; ++w) na += __popc(am[w]);
                        }
                        const T* Rb = (const T*)(par ? sp.P1 : sp.P0) + ax * NB;   // the old rows hold R
                        if constexpr (TC) {
                            // TC: k-steps over 4-step chunks with an active step (steps 4c .. 4c + 3, inactive
                            // ones as zero rows) -- a warp-uniform walk over a chunk mask instead of a __fns per
                            // lane and k-step
                            uint32_t cm = 0u;   // bit c: chunk c (steps 4c .. 4c + 3) holds an active step
#pragma unroll
                            for (int w = 0; w < 4; ++w) {   // nonzero nibbles of the word, compacted to a byte
                                uint32_t x = am[w];
                                x = (x | (x >> 1) | (x >> 2) | (x >> 3)) & 0x11111111u;
                                x = (x | (x >> 3)) & 0x03030303u;
                                x = (x | (x >> 6)) & 0x000F000Fu;
                                x = (x | (x >> 12)) & 0xFFu;
                                cm |= x << (8 * w);
                            }
                            while (cm) {
                                const int c = __ffs(cm) - 1;
                                cm &= cm - 1;
                                const int t = 4 * c + fc;
                                const bool act = t < S && ((am[t >> 5] >> (t & 31)) & 1u);
                                double bw[2];
#pragma unroll
                                for (int nt = 0; nt < 2; ++nt) {
                                    const int qb = 8 * nt + fr;
                                    bw[nt] = (act && qb < MP) ? (double)Wt[t * MP + qb] : 0.0;
                                }
#pragma unroll
                                for (int mt = 0; mt < MT; ++mt) {
                                    const int rob = 8 * mt + fr;
                                    const double a = (act && rob < n) ? (double)Rb[t * RS + rob] : 0.0;
#pragma unroll
                                    for (int nt = 0; nt < 2; ++nt) dmma884(gq[mt][nt][0], gq[mt][nt][1], a, bw[nt]);
                                }
                            }
                        } else
                        for (int kk = 0; 4 * kk < na; ++kk) {
                            int rem = 4 * kk + fc, t = -1;   // this lane's k = active step number
                            if (rem < na) {
                                if constexpr (TC) {   // one load: the word from the prefix counts
                                    const int w = (rem >= c0) + (rem >= c1) + (rem >= c2);
                                    const int before = w == 0 ? 0 : (w == 1 ? c0 : (w == 2 ? c1 : c2));
                                    t = w * 32 + (int)__fns(am[w], 0, rem - before + 1);
                                } else {
                                    for (int w = 0;; ++w) {
                                        const uint32_t bits = am[w];
                                        const int c = __popc(bits);
                                        if (rem < c) {
                                            t = w * 32 + (int)__fns(bits, 0, rem + 1);
                                            break;
                                        }
                                        rem -= c;
                                    }
                                }
                            }
                            double bw[2];
#pragma unroll
                            for (int nt = 0; nt < 2; ++nt) {
                                const int qb = 8 * nt + fr;
                                bw[nt] = (t >= 0 && qb < MP) ? (double)Wt[t * MP + qb] : 0.0;
                            }
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt) {
                                const int rob = 8 * mt + fr;
                                const double a = (t >= 0 && rob < n) ? (double)Rb[t * RS + rob] : 0.0;
#pragma unroll
                                for (int nt = 0; nt < 2; ++nt) dmma884(gq[mt][nt][0], gq[mt][nt][1], a, bw[nt]);
                            }
                        }
                    }
                    if (u_stale) {   // U rows of this axis, element-wise in the accumulator layout
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const int rob = 8 * mt + fr;
#pragma unroll
                            for (int nt = 0; nt < 2; ++nt) {
                                const int q = 8 * nt + 2 * fc;
                                if (rob < n && q < MP) {
                                    const int idx = (rb + rob) * MP + q;
                                    const double2 l = *reinterpret_cast<const double2*>(sp.lam + idx);
                                    const double2 x = *reinterpret_cast<const double2*>(sp.xb + idx);
                                    const double lp0 = l.x - p.rho * gq[mt][nt][0], lp1 = l.y - p.rho * gq[mt][nt][1];
                                    *reinterpret_cast<double2*>(sp.U + idx) =
                                        make_double2(2.0 * lp0 - l.x + x.x, 2.0 * lp1 - l.y + x.y);
                                }
                            }
                        }
                        __syncwarp();
                    }
                    SGSF_PT(8);
                    // X: D = cconst + [C | u] . KMd^T, column sums of the A fragments for the mean part
                    double dacc[MT][2][2];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const int rob = 8 * mt + fr;
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int q = 8 * nt + 2 * fc + e;
                                dacc[mt][nt][e] = (rob < n && q < MP) ? cconst[(rb + rob) * MP + q] : 0.0;
                            }
                        }
                    }
                    double csum[KT];
#pragma unroll
                    for (int kk = 0; kk < KT; ++kk) {
                        const int c = 4 * kk + fc;
                        double bf[2];
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt) {
                            const int qb = 8 * nt + fr;
                            bf[nt] = qb < MP ? KMd[qb * M2P + c] : 0.0;
                        }
                        csum[kk] = 0.0;
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const int rob = 8 * mt + fr;
                            const double a = rob < n ? (kk < KC ? Ccur[(rb + rob) * MP + c] : sp.U[(rb + rob) * MP + c - MP])
                                                     : 0.0;
                            csum[kk] += a;
#pragma unroll
                            for (int nt = 0; nt < 2; ++nt) dmma884(dacc[mt][nt][0], dacc[mt][nt][1], a, bf[nt]);
                        }
                    }
                    SGSF_PT(10);
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
                            for (int nt = 0; nt < 2; ++nt) {
                                const int qb = 8 * nt + fr;
                                dmma884(dm[nt][0], dm[nt][1], a, qb < MP ? KMm[qb * M2P + c] : 0.0);
                            }
                        }
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                            for (int nt = 0; nt < 2; ++nt) {
                                dacc[mt][nt][0] += dm[nt][0];
                                dacc[mt][nt][1] += dm[nt][1];
                            }
                    }
                    SGSF_PT(11);
                    SGSF_PT(12);
                    if (p.want_prev && !HY) {
                        for (int e = lane; e < n * MP; e += 32) sp.Cp[rb * MP + e] = sp.C[rb * MP + e];
                    }
                    __syncwarp();   // every lane has read the rows before any lane writes them
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const int rob = 8 * mt + fr;
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt) {
                            const int q = 8 * nt + 2 * fc;
                            if (rob < n && q < MP) {
                                const int idx = (rb + rob) * MP + q;
                                *reinterpret_cast<double2*>(Cnext + idx) = make_double2(dacc[mt][nt][0], dacc[mt][nt][1]);
                                if constexpr (TC) {
                                    unsigned char* bo = (unsigned char*)sp.Cf + ax * 2048;
#pragma unroll
                                    for (int e = 0; e < 2; ++e) {
                                        const float v = (float)dacc[mt][nt][e], hi = tc::tf32_rna(v);
                                        *reinterpret_cast<float*>(bo + tc::kmajor16_offset(rob, q + e)) = hi;
                                        *reinterpret_cast<float*>(bo + 1024 + tc::kmajor16_offset(rob, q + e)) =
                                            tc::tf32_rna(v - hi);
                                    }
                                } else {
                                    ((T*)sp.Cf)[(ax * MP + q) * NB + rob] = (T)dacc[mt][nt][0];
                                    ((T*)sp.Cf)[(ax * MP + q + 1) * NB + rob] = (T)dacc[mt][nt][1];
                                }
                                if (any_active) {   // commit lam'
                                    const double2 l = *reinterpret_cast<const double2*>(sp.lam + idx);
                                    *reinterpret_cast<double2*>(sp.lam + idx) =
                                        make_double2(l.x - p.rho * gq[mt][nt][0], l.y - p.rho * gq[mt][nt][1]);
                                }
                            }
                        }
                    }
                    if constexpr (TC) {   // this axis' positions of the next iterate, overlapping the check below
                        tc::fence_proxy_async();
                        __syncwarp();
                        // warp-uniform operands (broadcast from lane 0) let the MMA take them as uniform
                        // registers directly instead of a per-lane loop
                        const uint32_t tb_u = __shfl_sync(0xffffffffu, tbase, 0);
                        const int slot_u = __shfl_sync(0xffffffffu, slot, 0), ax_u = __shfl_sync(0xffffffffu, ax, 0);
                        if (tc::elect_one()) {
                            tc::fence_after_sync();
                            tc_issue_axis(tb_u, slot_u, ax_u, sp.Cf);
                            tc::mma_commit(&sp.sh->mbar);
                        }
                    }
                    __syncwarp();
                    SGSF_PT(13);
                }
                prev_active = any_active;
            }
            slot_barrier(bar_id, gsize);
            SGSF_PT(4);
        }
    }
#ifdef SGSF_NEAR_CLOCK
    if (blockIdx.x < 2 && lane == 0)
        printf("NEAR cta %d slot %d warp %d iterations %d near-check cycles per iteration %.0f\n", blockIdx.x, slot, lwarp,
               near_its, (double)near_cyc / (near_its > 0 ? near_its : 1));
#endif
    if constexpr (TC) {   // the last slot to finish frees the TMEM
        tc::fence_before_sync();
        if (lwarp == 0) {
            uint32_t last = 0;
            if (lane == 0) last = atomicAdd(&tmem_info[1], 1u) == (uint32_t)(p.spb - 1);
            if (__shfl_sync(0xffffffffu, last, 0)) {
                tc::fence_after_sync();
                tc::tmem_dealloc(tbase, 256);
            }
        }
    }
#ifdef SGSF_PHASE_TIMING
    if (tid == 0)
        printf("PT block %d iters %d total %.0f T1 %.0f T2 %.0f T3bar %.0f dec %.0f G %.0f MX %.0f "
               "mxG %.0f mxU %.0f mxM %.0f mxP %.0f mxX %.0f mxC %.0f mxE %.0f t1tc %.0f\n", blockIdx.x, pt_iters,
               (double)(pt_acc[0] + pt_acc[1] + pt_acc[2] + pt_acc[3] + pt_acc[4] + pt_acc[5] + pt_acc[6] + pt_acc[8] +
                        pt_acc[9] + pt_acc[10] + pt_acc[11] + pt_acc[12] + pt_acc[13] + pt_acc[14] + pt_acc[15]),
               (double)(pt_acc[5] + pt_acc[15]) / pt_iters, (double)pt_acc[6] / pt_iters, (double)pt_acc[1] / pt_iters,
               (double)pt_acc[2] / pt_iters, (double)pt_acc[3] / pt_iters,
               (double)(pt_acc[4] + pt_acc[0] + pt_acc[8] + pt_acc[9] + pt_acc[10] + pt_acc[11] + pt_acc[12] + pt_acc[13] +
                        pt_acc[14]) / pt_iters,
               (double)pt_acc[8] / pt_iters, (double)pt_acc[9] / pt_iters, (double)pt_acc[10] / pt_iters,
               (double)pt_acc[11] / pt_iters, (double)pt_acc[12] / pt_iters, (double)pt_acc[13] / pt_iters,
               (double)pt_acc[14] / pt_iters, (double)pt_acc[15] / pt_iters);
    if (tid == 0)
        printf("PTW block %d spread %.0f last %d %d %d %d\n", blockIdx.x, (double)pt_spread / pt_iters, pt_lastw[0],
               pt_lastw[1], pt_lastw[2], pt_lastw[3]);
#endif
}

}  // namespace sgsf
