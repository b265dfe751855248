// sf_device.cuh -- per-term device math shared by every kernel.
//
// Spherical block update (reference: kernels/reference.py:13-48,
// _speedups.pyx:18-73).  The reference computes azimuth/polar with atan2,
// the radial factor num/den, and rebuilds the target with sin/cos.  With its
// angle choices the unclamped radial equals the normalised spheroidal radius
//     r = sqrt((dx^2 + dy^2)/a^2 + dz^2/b^2)
// so the target is clamp(r, lo, hi)/r * d: one rsqrt per term.
// Terms with an exactly-zero component go through the reference trig formula
// in FP64 instead: there the reference's cos(pi/2) = 6.1e-17 and
// sin(pi) = 1.2e-16 "leaks" are what breaks the symmetry of head-on
// scenarios, and dropping them changes the trajectory.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace sgsf {

// Reference trig formula in FP64.  Explicit _rn intrinsics keep nvcc from
// contracting into FMAs so the products round like the reference's scalar C.
// This path exists for terms with an exactly-zero component, and there one
// of the two angles is special (0, +-pi/2, +-pi): its sine and cosine are
// the values the library returns for those doubles -- e.g. cos(pi/2) =
// 6.123233995736766e-17, the "leak" that matters -- so only the other angle
// needs atan2 + sincos.
constexpr double kHalfPi = 1.5707963267948966, kPi = 3.141592653589793;
constexpr double kCosHalfPi = 6.123233995736766e-17, kSinPi = 1.2246467991473532e-16;

static __device__ __noinline__ void ref_spherical(double dx, double dy, double dz, double lat, double vert,
                                           double lo, double hi, double* az_o, double* pol_o,
                                           double* rad_o, double* tx, double* ty, double* tz) {
    double az, ca, sa, planar;
    if (dx == 0.0 && dy != 0.0) {   // atan2(+-y, +-0) = +-pi/2
        az = copysign(kHalfPi, dy);
        ca = kCosHalfPi;
        sa = copysign(1.0, dy);
        planar = fabs(dy);
    } else if (dy == 0.0 && dx != 0.0) {   // atan2(+-0, x) = +-0 (x > 0) or +-pi (x < 0)
        if (dx > 0.0) {
            az = copysign(0.0, dy);
            ca = 1.0;
            sa = copysign(0.0, dy);
        } else {
            az = copysign(kPi, dy);
            ca = -1.0;
            sa = copysign(kSinPi, dy);
        }
        planar = fabs(dx);
    } else {
        az = atan2(dy, dx);
        sincos(az, &sa, &ca);
        planar = hypot(dx, dy);
    }
    double pol, sp, cp;
    if (planar == 0.0 && dz == 0.0) {   // the reference's all-zero convention
        pol = kHalfPi;
        sp = 1.0;
        cp = kCosHalfPi;
    } else if (planar == 0.0) {   // atan2(+0, x): 0 for x > 0, pi for x < 0
        if (dz > 0.0) {
            pol = 0.0;
            sp = 0.0;
            cp = 1.0;
        } else {
            pol = kPi;
            sp = kSinPi;
            cp = -1.0;
        }
    } else if (dz == 0.0) {   // atan2(y > 0, +-0) = pi/2
        pol = kHalfPi;
        sp = 1.0;
        cp = kCosHalfPi;
    } else {
        pol = atan2(__ddiv_rn(planar, lat), __ddiv_rn(dz, vert));
        sincos(pol, &sp, &cp);
    }
    double ls = __dmul_rn(lat, sp), vc = __dmul_rn(vert, cp);
    double num = __dadd_rn(__dmul_rn(ls, planar), __dmul_rn(vc, dz));
    double den = __dadd_rn(__dmul_rn(ls, ls), __dmul_rn(vc, vc));
    double rad = __ddiv_rn(num, den);
    if (rad < lo) rad = lo;
    else if (rad > hi) rad = hi;
    double lr = __dmul_rn(__dmul_rn(lat, rad), sp);
    if (az_o) *az_o = az;
    if (pol_o) *pol_o = pol;
    if (rad_o) *rad_o = rad;
    if (tx) *tx = __dmul_rn(lr, ca);
    if (ty) *ty = __dmul_rn(lr, sa);
    if (tz) *tz = __dmul_rn(__dmul_rn(vert, rad), cp);
}

template <typename T> __device__ __forceinline__ T rsq(T q);
template <> __device__ __forceinline__ float rsq<float>(float q) {
    float y;   // MUFU.RSQ, flush-to-zero approximate reciprocal square root (<= 2 ulp)
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(q));
    return y;
}
template <> __device__ __forceinline__ double rsq<double>(double q) { return rsqrt(q); }

template <typename T> __device__ __forceinline__ T fma_t(T a, T b, T c);
template <> __device__ __forceinline__ float fma_t<float>(float a, float b, float c) { return fmaf(a, b, c); }
template <> __device__ __forceinline__ double fma_t<double>(double a, double b, double c) { return fma(a, b, c); }

// Per-family geometry in term precision (+ FP64 originals for the fallback).
template <typename T>
struct Family {
    T lat;      // lateral semiaxis
    T lim;      // lat^2: interior test threshold on q = lat^2 r^2
    T beta;     // lat^2 / vert^2
    double lat64, vert64;
};

template <typename T>
__host__ __device__ inline Family<T> make_family(double lat, double vert) {
    Family<T> f;
    f.lat = (T)lat;
    f.lim = (T)(lat * lat);
    f.beta = (T)((lat * lat) / (vert * vert));
    f.lat64 = lat;
    f.vert64 = vert;
    return f;
}

// Scale factor s of one term: target = s d.  PAIR: radial clamped to
// [1, inf) (clearance); !PAIR: radial clamped to [0, 1] (containment).
// Interior terms get s == 1 exactly, so their residual d - s d is exactly 0.
// `zmin` accumulates min |dx dy dz|: a zero there means some term had an
// exactly-zero component and must be redone on the careful path (the product
// can also underflow to zero, which only sends a term to the careful path).
template <typename T, bool PAIR>
__device__ __forceinline__ T scale_fast(T dx, T dy, T dz, const Family<T>& f, T& zmin) {
    zmin = fmin(zmin, fabs(dx * dy * dz));
    const T q = fma_t<T>(dz * f.beta, dz, fma_t<T>(dy, dy, dx * dx));
    const bool inside = PAIR ? (q >= f.lim) : (q <= f.lim);
    const T s = f.lat * rsq<T>(q);
    return inside ? T(1) : s;
}

// Target of one term with the FP64 reference-formula fallback for terms
// with an exactly-zero component (careful path; involves a call).
template <typename T, bool PAIR>
__device__ __forceinline__ void target(T dx, T dy, T dz, const Family<T>& f, T& tx, T& ty, T& tz) {
    if (dx == T(0) || dy == T(0) || dz == T(0)) {
        double ox, oy, oz;
        ref_spherical((double)dx, (double)dy, (double)dz, f.lat64, f.vert64, PAIR ? 1.0 : 0.0,
                      PAIR ? CUDART_INF : 1.0, nullptr, nullptr, nullptr, &ox, &oy, &oz);
        tx = (T)ox;
        ty = (T)oy;
        tz = (T)oz;
        return;
    }
    T zunused = T(1);
    const T s = scale_fast<T, PAIR>(dx, dy, dz, f, zunused);
    tx = s * dx;
    ty = s * dy;
    tz = s * dz;
}

// (bx, by, bz) - target(dx, dy, dz).  With b == d this is the term's residual
// d - e; with d = d_{k-1}, b = d_k it is the exit residual d_k - e_{k-1}.
// CAREFUL = false never calls out: it only records exactly-zero components in
// zmin (the caller then redoes the whole time step with CAREFUL = true).
template <typename T, bool PAIR, bool CAREFUL>
__device__ __forceinline__ void resid(T dx, T dy, T dz, T bx, T by, T bz, const Family<T>& f, T& zmin, T& rx,
                                      T& ry, T& rz) {
    if (CAREFUL && (dx == T(0) || dy == T(0) || dz == T(0))) {
        T tx, ty, tz;
        target<T, PAIR>(dx, dy, dz, f, tx, ty, tz);
        rx = bx - tx;
        ry = by - ty;
        rz = bz - tz;
        return;
    }
    const T s = scale_fast<T, PAIR>(dx, dy, dz, f, zmin);
    rx = fma_t<T>(-s, dx, bx);
    ry = fma_t<T>(-s, dy, by);
    rz = fma_t<T>(-s, dz, bz);
}

// Generic [lo, hi] version for the unit entry point with non-standard bounds.
template <typename T>
__device__ __forceinline__ void target_generic(T dx, T dy, T dz, const Family<T>& f, double lo, double hi,
                                               T& tx, T& ty, T& tz) {
    if (dx == T(0) || dy == T(0) || dz == T(0)) {
        double ox, oy, oz;
        ref_spherical((double)dx, (double)dy, (double)dz, f.lat64, f.vert64, lo, hi, nullptr, nullptr,
                      nullptr, &ox, &oy, &oz);
        tx = (T)ox;
        ty = (T)oy;
        tz = (T)oz;
        return;
    }
    T q = fma_t<T>(dz * f.beta, dz, fma_t<T>(dy, dy, dx * dx));
    T ir = f.lat * rsq<T>(q);     // 1 / r
    T r = q * ir / f.lat;         // r
    T s = T(1);
    if (r < (T)lo) s = (T)lo * ir;
    else if (r > (T)hi) s = (T)hi * ir;
    tx = s * dx;
    ty = s * dy;
    tz = s * dz;
}

}  // namespace sgsf

namespace sgsf {

// One term of the feasible verdict (check_original_constraints, assembly.py:437-487; margins as
// problem.py:113-137: ((dx^2 + dy^2) / a^2 + dz^2 / b^2) - 1).  Pairs must keep margin >= -tol, workspace
// terms margin <= tol.  The reciprocal form screens; the reference's divisions (exact) decide the terms
// within a few ulps of a threshold and the extremes.  Shared by the standalone verdict kernel and K1's
// fused epilogue, so both give the same bits.
__device__ __forceinline__ void verdict_term(bool pair, double dx, double dy, double dz, double a2, double b2,
                                             double inv_a2, double inv_b2, double tol, double& pmin, double& wmax,
                                             int& pc, int& wc) {
    auto exact = [&]() {
        return __dadd_rn(__dadd_rn(__ddiv_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), a2),
                                   __ddiv_rn(__dmul_rn(dz, dz), b2)), -1.0);
    };
    const double ma = fma(dz * dz, inv_b2, (dx * dx + dy * dy) * inv_a2) - 1.0;
    const double slack = 1e-12 * (1.0 + fabs(ma));
    if (pair) {
        if (ma < pmin + slack) pmin = fmin(pmin, exact());
        if (ma < -tol - slack) ++pc;
        else if (ma <= -tol + slack) pc += (exact() < -tol);
    } else {
        if (ma > wmax - slack) wmax = fmax(wmax, exact());
        if (ma > tol + slack) ++wc;
        else if (ma >= tol - slack) wc += (exact() > tol);
    }
}

}  // namespace sgsf
