// sf_unroll.cuh -- the differentiable safety filter: K unrolled fixed-point iterations in FP64 and
// their reverse (vector-Jacobian) sweep.
//
// The paper trains its initialisation network through an unrolled chain of K fixed-point steps
// z_{k+1} = f_FP(z_k), z = (xi, lambda) (PAPER.md, "Learned Initialization for SF", eq. NN_loss;
// SURVEY 8f item 2, BASELINE config 5).  The reference package has no autodiff; the step itself is
// the reference loop body (solver.py:314-328):
//     E        = Pi(F xi)                                 spherical targets (pairs, workspace + centre)
//     lambda'  = lambda - rho F^T (F xi - E)               solver.py:317-321
//     eta      = rho F^T E + lambda' + xi_bar              solver.py:323-327
//     xi'      = M eta + c                                 KKT solve, M = [K^-1]_11 (assembly.py:186-219)
// written as in K1: xi' = Mm Cbar + Km11 ubar + Md (C - Cbar) + Kd11 (u - ubar) + cconst with
// u = 2 lambda' - lambda + xi_bar.
//
// Reverse step, given the adjoints (xh', lh') of (xi', lambda'):
//     eh  = M^T xh'                 (mean / deviation modes: Km11^T, Kd11^T)
//     lh  = lh' + eh                xi_bar gets eh
//     xh  = rho F^T F eh + rho F^T (J - I)^T F (lh + eh)
// with J the 3x3 Jacobian of a term's target: the identity for interior terms, and for an active
// term (target d / r, r the spheroid radius) J = (1/r)(I - d (D d)^T / r^2).  So, as in the forward,
// only the active terms cost more than the structured F^T F = ((n+1) I - 1 1^T) (x) G.
//
// Layout: one CTA per sample; threads (i, tl) own robot i at step t0 + tl of a window of TW = 256 / n
// steps; every pair is evaluated by both of its robots, so each robot's row accumulates in a fixed
// order (no atomics, deterministic); W^T projections are accumulated per coefficient by owner threads.
#pragma once
#include <cuda_runtime.h>

namespace sgsf {

struct UnrollParams {
    int n, S, m1, batch, iters;
    double rho, lat, vert, ws_lat, ws_vert, cx, cy, cz;
    const double* W;       // S x m1
    const double* Km11;    // m1 x m1 each
    const double* Kd11;
    const double* Mm;
    const double* Md;
    const double* G;       // W^T W
    const double* cconst;  // 3 x n x m1
    const double* xi_bar;  // B x dim
    const double* xi0;     // B x dim
    const double* lam0;    // B x dim
    double* xs;            // B x (iters + 1) x dim: xi_0 .. xi_K (forward output, backward input)
    double* ls;            // B x (iters + 1) x dim: lambda_0 .. lambda_K
    const double* gxs;     // B x (iters + 1) x dim, nullable: dL/dxi_k
    const double* gls;     // nullable: dL/dlambda_k
    double* g_xi_bar;      // B x dim
    double* g_xi0;
    double* g_lam0;
};

size_t unroll_smem_bytes(int n, int S, int m1);
int launch_unroll_forward(const UnrollParams& p, cudaStream_t stream);
int launch_unroll_backward(const UnrollParams& p, cudaStream_t stream);

}  // namespace sgsf
