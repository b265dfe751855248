/*
 * sgsf.h -- C ABI of the B200-native Swarm-Gen safety filter (libsgsf.so).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point that
 * touches the GPU is stream-ordered on the caller's `cudaStream_t` (passed as
 * `void*`, NULL = legacy default stream).  Device buffers are caller-owned.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/swarmfilter):
 *   sgsf_create / sgsf_destroy   SafetyFilter.__init__ + KktFactorization cache   solver.py:232-249,
 *                                assembly.py:154-184, 325-339 (one handle per (problem, degree, rho))
 *   sgsf_solve                   SafetyFilter.batch_solve -> solve (the AM loop)  solver.py:286-407
 *   sgsf_solve_host              same, host buffers in/out (the reference's numpy-in / numpy-out call)
 *   sgsf_verdict                 metrics.feasible_results -> check_original_constraints
 *                                metrics.py:57-69, assembly.py:437-487
 *   sgsf_trajectory              basis.coeffs_to_trajectory                        basis.py:149-160
 *   sgsf_svars                   SolveResult.svars (last spherical step)           solver.py:142-174, 358
 *   sgsf_spherical_project       kernels.spherical_project (backend contract)      kernels/__init__.py:46-50,
 *                                                                                  _speedups.pyx:18-73
 *   sgsf_apply_F / sgsf_apply_FT PairwiseOperator.apply / apply_transpose          assembly.py:285-310
 *   sgsf_kkt_step                KktFactorization.solve                            assembly.py:186-219
 *   sgsf_decoder_forward         the CVAE / VQ-VAE decoder forward pass feeding the SF (no reference code,
 *                                SPEC.md:8; PAPER.md "CVAE / VQ-VAE Network Details")
 *   sgsf_unroll / _backward      K unrolled fixed-point steps and their reverse sweep: the differentiable
 *                                SF of PAPER.md "Learned Initialization for SF" (eq. NN_loss); the step is
 *                                the solve loop body solver.py:314-328 (the reference has no autodiff)
 */
#ifndef SGSF_H
#define SGSF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* whole-call status codes */
#define SGSF_OK              0
#define SGSF_ERR_INVALID     1   /* bad argument / shape            -> DimensionMismatch / ValueError */
#define SGSF_ERR_CUDA        2   /* CUDA runtime error              -> RuntimeError */
#define SGSF_ERR_UNSUPPORTED 3   /* size outside what this build handles (e.g. n > max robots) */
#define SGSF_ERR_SINGULAR    4   /* KKT precompute failed           -> SingularKKT */

/* per-sample status written to outputs.status[b] */
#define SGSF_SAMPLE_OK           0
#define SGSF_SAMPLE_SINGULAR_KKT 1   /* endpoint residual above tol_eq (assembly.py:213-217) */

/* term precision of the iteration (state and xi-step are always FP64) */
#define SGSF_PRECISION_LEAN   0  /* FP32 pair/workspace terms, positions, W^T projection */
#define SGSF_PRECISION_STRICT 1  /* FP64 everywhere */
#define SGSF_PRECISION_HYBRID 2  /* FP32 screening with guard bands, FP64 targets/residuals/state and an FP64
                                    re-evaluation of the stop decision near tol_residual: the FP64 iteration
                                    counts and verdicts at close to lean speed (K1 and K1L) */

typedef struct sgsf_handle_s sgsf_handle_t;

/* FP64 host constants for one (problem, degree, rho); see precompute.py. Row-major. */
typedef struct {
    int n;            /* robots */
    int samples;      /* S = H + 1 */
    int m1;           /* degree + 1 */
    double rho;
    double lat, vert;           /* robot safety spheroid semiaxes a, b */
    double ws_lat, ws_vert;     /* workspace semiaxes a_w, b_w */
    double center[3];           /* workspace centre */
    const double* W;            /* S x m1   value basis */
    const double* Wd;           /* S x m1   velocity basis */
    const double* Wdd;          /* S x m1   acceleration basis */
    const double* B;            /* 6 x m1   endpoint rows (p0 v0 a0 pT vT aT) */
    const double* rhs;          /* 3 x n x 6 */
    const double* PBt;          /* m1 x 6   B^T (B B^T)^-1 */
    const double* Km11;         /* m1 x m1  mean-KKT inverse, top-left */
    const double* Kd11;         /* m1 x m1  deviation-KKT inverse, top-left */
    const double* Mm;           /* m1 x m1  rho Km11 G */
    const double* Md;           /* m1 x m1  rho (n+1) Kd11 G */
    const double* cconst;       /* 3 x n x m1 */
} sgsf_problem_t;

typedef struct {
    int max_iters;
    double tol_residual;
    double tol_eq;
    int early_stop;
    int precision;        /* SGSF_PRECISION_* */
    int want_prev;        /* also write coefficients of iteration K-1 (for svars) */
    int slots_per_block;  /* 0 = auto (smem/thread budget) */
    int grid;             /* 0 = auto (persistent: #SM x CTAs/SM) */
    double verdict_tol;   /* tolerance of outputs->verdict (check_original_constraints, metrics.py:57-69) */
} sgsf_config_t;

/* Verdict outputs (check_original_constraints at tol), device pointers. */
typedef struct {
    uint8_t* ok;              /* B: no violation */
    uint8_t* feasible;        /* B: ok && converged[b] (converged may be NULL -> ok) */
    double* pair_margin_min;  /* B (+inf when n == 1) */
    double* ws_margin_max;    /* B */
    int32_t* pair_viol;       /* B */
    int32_t* ws_viol;         /* B */
} sgsf_verdict_t;

/* Per-sample outputs, device pointers, caller-owned. dim = 3 n m1. */
typedef struct {
    double* coeffs;         /* B x dim */
    double* multipliers;    /* B x dim */
    double* res_inf;        /* B x max_iters (entries >= iterations untouched) */
    double* res_l2;         /* B x max_iters */
    int32_t* iterations;    /* B */
    uint8_t* converged;     /* B */
    double* displacement;   /* B: ||coeffs - xi_bar||_2 */
    int32_t* status;        /* B: SGSF_SAMPLE_* */
    double* eq_err;         /* B: ||A xi - b||_inf of the returned iterate */
    double* coeffs_prev;    /* B x dim, nullable (needs cfg.want_prev) */
    /* nullable: the feasible verdict of the returned iterates at cfg->verdict_tol (sgsf_verdict, launched
       right behind the solve kernel on the same stream); NULL fields are skipped */
    const sgsf_verdict_t* verdict;
} sgsf_outputs_t;


typedef struct {
    void* start;   /* cudaEvent_t recorded just before the main solve kernel (nullable) */
    void* stop;    /* cudaEvent_t recorded just after it */
} sgsf_timing_t;

const char* sgsf_version(void);
const char* sgsf_last_error(void);
/* number of kernels this library has launched since load (evidence for bench.py gpu_launches) */
uint64_t sgsf_launch_count(void);
/* largest n this build solves */
int sgsf_max_robots(void);

int sgsf_create(const sgsf_problem_t* problem, sgsf_handle_t** out);
void sgsf_destroy(sgsf_handle_t* h);

/* bytes of device workspace sgsf_solve needs for `batch` samples (sample queue + longest-first order) */
size_t sgsf_workspace_bytes(int batch);

/*
 * Run the safety filter on a batch.  xi_bar: B x dim (device).  init_mode: B bytes or NULL
 * (0 = boundary projection of xi_bar with zero multipliers, 1 = warm start from xi0/lam0 rows).
 */
int sgsf_solve(sgsf_handle_t* h, int batch, const double* xi_bar, const double* xi0,
               const double* lam0, const uint8_t* init_mode, const sgsf_config_t* cfg,
               sgsf_outputs_t* out, void* workspace, const sgsf_timing_t* timing, void* stream);

/* Same with HOST buffers (pageable or pinned): copies in, solves, verdicts, copies out, syncs. */
int sgsf_solve_host(sgsf_handle_t* h, int batch, const double* xi_bar, const double* xi0,
                    const double* lam0, const uint8_t* init_mode, const sgsf_config_t* cfg,
                    double* coeffs, double* multipliers, double* res_inf, double* res_l2,
                    int32_t* iterations, uint8_t* converged, uint8_t* feasible,
                    double* displacement, int32_t* status, void* stream);

int sgsf_verdict(sgsf_handle_t* h, int batch, const double* coeffs, const uint8_t* converged,
                 double tol, sgsf_verdict_t* out, void* stream);

/* pos/vel/acc: B x n x S x 3 (device); any may be NULL */
int sgsf_trajectory(sgsf_handle_t* h, int batch, const double* coeffs, double* pos, double* vel,
                    double* acc, void* stream);

/* spherical variables of positions C W^T: pair_* B x P x S, ws_* B x n x S (device) */
int sgsf_svars(sgsf_handle_t* h, int batch, const double* coeffs, double* pair_az, double* pair_pol,
               double* pair_rad, double* ws_az, double* ws_pol, double* ws_rad, void* stream);

/*
 * Unit entry point for the spherical block update (kernels contract).  mode:
 *   0 = the solver's lean path (FP32 trig-free target, FP64 trig fallback on zero components)
 *   1 = the solver's strict path (FP64 trig-free target + fallback)
 *   2 = reference trig formula in FP64
 * Angles/radial always come from the FP64 reference formula.  Any output may be NULL.
 */
int sgsf_spherical_project(int count, const double* dx, const double* dy, const double* dz,
                           double lat, double vert, double lo, double hi, int mode,
                           double* az, double* pol, double* rad, double* tx, double* ty, double* tz,
                           void* stream);

/* FP64 operator applications for the step API (tests / step functions). */
int sgsf_apply_F(sgsf_handle_t* h, int batch, const double* xi, double* out, void* stream);
int sgsf_apply_FT(sgsf_handle_t* h, int batch, const double* v, double* out, void* stream);
/* literal coefficient step from eta (3 x n x m1 per sample): C_i = Km11 eta_bar + Kd11 (eta_i - eta_bar) + cconst_i */
int sgsf_kkt_step(sgsf_handle_t* h, int batch, const double* eta, double* out, double* eq_err, void* stream);

/*
 * Differentiable SF (FP64).  sgsf_unroll runs `iters` fixed-point steps z_{k+1} = f(z_k), z = (xi, lambda),
 * from (xi0, lam0) with no early stop, and writes every iterate: xs, ls are B x (iters + 1) x dim (device),
 * row 0 = (xi0, lam0).  sgsf_unroll_backward is its vector-Jacobian product: given dL/dxs and dL/dls
 * (either may be NULL = zero; same shape), it writes dL/dxi_bar, dL/dxi0, dL/dlam0 (B x dim) using the
 * iterates xs of the forward.  Active terms use the Jacobian of the target d / r; interior terms the
 * identity; a zero pair difference (target locally constant) a zero Jacobian.
 */
int sgsf_unroll(sgsf_handle_t* h, int batch, int iters, const double* xi_bar, const double* xi0,
                const double* lam0, double* xs, double* ls, void* stream);
int sgsf_unroll_backward(sgsf_handle_t* h, int batch, int iters, const double* xs, const double* gxs,
                         const double* gls, double* g_xi_bar, double* g_xi0, double* g_lam0, void* stream);

/*
 * Mean pairwise cosine of `count` vectors of length `dim` (device, row-major), optionally centred by the
 * column mean (metrics.mean_pairwise_cosine / diversity_cosine, metrics.py:83-115).  NaN if a (centred)
 * vector is zero.  work: sgsf_cosine_work_doubles(count, dim) doubles (device); result: 1 double (device).
 */
size_t sgsf_cosine_work_doubles(int count, int dim);
int sgsf_pairwise_cosine(int count, int dim, const double* vectors, int center, double* work, double* result,
                         void* stream);

/*
 * Generative decoder forward pass (K4; BASELINE configs 1-3 sample the SF's proposals from a CVAE / VQ-VAE
 * decoder, PAPER.md "CVAE / VQ-VAE Network Details"; the reference has no network code).  Four
 * kernel-3 transposed convolutions of 128 channels (batch norm folded), LeakyReLU or ReLU, a 1x1 head to 3
 * channels and a Linear L -> n (degree + 1) per axis, times `scale`: the coefficient correction to the
 * straight line, B x 3 n (degree + 1), FP64.  Weights are device buffers in the packed layout written by
 * paper_2501_19042_b200.generative.FusedDecoder (sgsf_decoder_pack_bytes(c0) bytes for the 4 layers).
 */
typedef struct {
    int L;               /* latent positions */
    int c0;              /* input channels of the first layer (latent + state features), <= 128 */
    int nm1;             /* n (degree + 1): coefficients per axis */
    int leaky;           /* 1: LeakyReLU(slope), 0: ReLU */
    float slope, scale;
    const void* wpack;   /* the 4 layers' weights, BN folded, tf32 hi / lo, in the kernel's operand layout */
    const float* bias;   /* 4 x 128 folded biases */
    const float* head_w; /* 3 x 128 */
    const float* head_b; /* 3 */
    const float* exp_w;  /* L x nm1: the expansion Linear's weight, transposed */
    const float* exp_b;  /* nm1 */
    int cz;              /* channels read per sample from the input (the latent); the other c0 - cz ... */
    const float* feat;   /* ... come from feat (c0 - cz values, constant over positions and samples), or NULL */
    /* the boundary QP layer fused behind the decoder (projection.py:11-25), all nullable: with base set, the
       output is xi_bar = project(base + correction) instead of the correction */
    const double* base;  /* 3 nm1 straight-line coefficients */
    const double* B6;    /* 6 x m1 endpoint rows */
    const double* PBt;   /* m1 x 6  B^T (B B^T)^-1 */
    const double* rhs;   /* 3 n x 6 endpoint values */
    int n, m1;
} sgsf_decoder_t;
size_t sgsf_decoder_pack_bytes(int c0);
/* h0: B x cz x L float (device): the latent (cz = c0 when feat is NULL); out: B x 3 nm1 double (device) */
int sgsf_decoder_forward(const sgsf_decoder_t* dec, int batch, const float* h0, double* corr, void* stream);
/* test entry point: as sgsf_decoder_forward, also writing each layer's activations (B x 4 x 128 x L floats) to
   dbg, or with raw != 0 the first layer's three tap accumulators in slots 1..3 */
int sgsf_decoder_forward_dbg(const sgsf_decoder_t* dec, int batch, const float* h0, double* corr, float* dbg,
                             int raw, void* stream);
/* FP32 FFMA throughput microbenchmark (roofline denominator); returns TFLOP/s in *tflops */
int sgsf_fp32_peak(double* tflops, double* ms, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SGSF_H */
