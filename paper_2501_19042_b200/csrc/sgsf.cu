// sgsf.cu -- C ABI (include/sgsf.h) over the sm_100a kernels.
//
// One handle per (problem, degree, rho): it owns only immutable device
// constants, like the reference's rho-keyed KKT cache (assembly.py:325-339),
// so it is safe to share across threads and streams.  Every launch is
// stream-ordered on the caller's stream; nothing here synchronises except
// sgsf_solve_host (host buffers in/out) and sgsf_fp32_peak.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sgsf.h"
#include "sf_aux.cuh"
#include "sf_unroll.cuh"
#include "sf_device.cuh"
#include "sf_launch.cuh"
#include "sf_persistent.cuh"

using namespace sgsf;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return fail(SGSF_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

constexpr int kMaxRobots = 64;

}  // namespace

struct sgsf_handle_s {
    int n, S, m1, P;
    double rho, lat, vert, ws_lat, ws_vert, center[3];
    double *W, *Wd, *Wdd, *KMm, *KMd, *Km11, *Kd11, *cconst, *B6, *rhs, *PBt;
    double *Mm, *Md, *G;   // plain m1 x m1 (unrolled solver)
    int device, sm_count;
};

static AuxParams aux_params(const sgsf_handle_t* h) {
    AuxParams a;
    a.n = h->n;
    a.S = h->S;
    a.m1 = h->m1;
    a.P = h->P;
    a.lat = h->lat;
    a.vert = h->vert;
    a.ws_lat = h->ws_lat;
    a.ws_vert = h->ws_vert;
    a.cx = h->center[0];
    a.cy = h->center[1];
    a.cz = h->center[2];
    a.W = h->W;
    a.Wd = h->Wd;
    a.Wdd = h->Wdd;
    a.Km11 = h->Km11;
    a.Kd11 = h->Kd11;
    a.cconst = h->cconst;
    a.B6 = h->B6;
    a.rhs = h->rhs;
    return a;
}

extern "C" {

const char* sgsf_version(void) { return "sgsf 0.1 (sm_100a)"; }
const char* sgsf_last_error(void) { return g_last_error.c_str(); }
uint64_t sgsf_launch_count(void) { return g_launches.load(); }
int sgsf_max_robots(void) { return kMaxRobots; }
// [queue counter | pad to 256 B][score: batch floats][order: batch ints], 256 B aligned
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
size_t sgsf_workspace_bytes(int batch) {
    const size_t b = batch > 0 ? (size_t)batch : 0;
    return 256 + 2 * align256(b * 4);
}

static int upload(double** dst, const double* src, size_t count) {
    if (!src) return fail(SGSF_ERR_INVALID, "null constant pointer");
    CUDA_TRY(cudaMalloc(dst, count * sizeof(double)));
    CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(double), cudaMemcpyHostToDevice));
    return SGSF_OK;
}

void sgsf_destroy(sgsf_handle_t* h) {
    if (!h) return;
    double* ptrs[] = {h->W,  h->Wd,  h->Wdd, h->KMm, h->KMd, h->Km11, h->Kd11,
                      h->cconst, h->B6, h->rhs, h->PBt, h->Mm,  h->Md,  h->G};
    for (double* q : ptrs)
        if (q) cudaFree(q);
    delete h;
}

int sgsf_create(const sgsf_problem_t* pr, sgsf_handle_t** out) {
    if (!pr || !out) return fail(SGSF_ERR_INVALID, "null argument");
    if (pr->n < 1 || pr->samples < 2 || pr->m1 < 2)
        return fail(SGSF_ERR_INVALID, "need n >= 1, samples >= 2, m1 >= 2");
    if (pr->m1 > 16) return fail(SGSF_ERR_UNSUPPORTED, "degree + 1 above 16 is not supported");
    sgsf_handle_t* h = new sgsf_handle_t();
    std::memset(h, 0, sizeof(*h));
    h->n = pr->n;
    h->S = pr->samples;
    h->m1 = pr->m1;
    h->P = pr->n * (pr->n - 1) / 2;
    h->rho = pr->rho;
    h->lat = pr->lat;
    h->vert = pr->vert;
    h->ws_lat = pr->ws_lat;
    h->ws_vert = pr->ws_vert;
    for (int i = 0; i < 3; ++i) h->center[i] = pr->center[i];
    const int m1 = pr->m1, n = pr->n, S = pr->samples;
    std::vector<double> kmm(m1 * 2 * m1), kmd(m1 * 2 * m1);
    for (int q = 0; q < m1; ++q)
        for (int q2 = 0; q2 < m1; ++q2) {
            kmm[q * 2 * m1 + q2] = pr->Mm[q * m1 + q2];
            kmm[q * 2 * m1 + m1 + q2] = pr->Km11[q * m1 + q2];
            kmd[q * 2 * m1 + q2] = pr->Md[q * m1 + q2];
            kmd[q * 2 * m1 + m1 + q2] = pr->Kd11[q * m1 + q2];
        }
    std::vector<double> gram((size_t)m1 * m1, 0.0);   // G = W^T W
    for (int q = 0; q < m1; ++q)
        for (int q2 = 0; q2 < m1; ++q2)
            for (int t = 0; t < S; ++t) gram[q * m1 + q2] += pr->W[t * m1 + q] * pr->W[t * m1 + q2];
    int rc = SGSF_OK;
    if ((rc = upload(&h->W, pr->W, (size_t)S * m1)) || (rc = upload(&h->Wd, pr->Wd, (size_t)S * m1)) ||
        (rc = upload(&h->Wdd, pr->Wdd, (size_t)S * m1)) || (rc = upload(&h->KMm, kmm.data(), kmm.size())) ||
        (rc = upload(&h->KMd, kmd.data(), kmd.size())) || (rc = upload(&h->Km11, pr->Km11, (size_t)m1 * m1)) ||
        (rc = upload(&h->Kd11, pr->Kd11, (size_t)m1 * m1)) ||
        (rc = upload(&h->cconst, pr->cconst, (size_t)3 * n * m1)) || (rc = upload(&h->B6, pr->B, (size_t)6 * m1)) ||
        (rc = upload(&h->rhs, pr->rhs, (size_t)3 * n * 6)) || (rc = upload(&h->PBt, pr->PBt, (size_t)m1 * 6)) ||
        (rc = upload(&h->Mm, pr->Mm, (size_t)m1 * m1)) || (rc = upload(&h->Md, pr->Md, (size_t)m1 * m1)) ||
        (rc = upload(&h->G, gram.data(), gram.size()))) {
        sgsf_destroy(h);
        return rc;
    }
    cudaGetDevice(&h->device);
    cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device);
    *out = h;
    return SGSF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- launch plumbing for K1
namespace sgsf {
int internal_fail(int code, const std::string& msg) { return fail(code, msg); }
void internal_count_launch(int n) { g_launches.fetch_add((uint64_t)n); }
}  // namespace sgsf

extern "C" {

int sgsf_solve(sgsf_handle_t* h, int batch, const double* xi_bar, const double* xi0, const double* lam0,
               const uint8_t* init_mode, const sgsf_config_t* cfg, sgsf_outputs_t* out, void* workspace,
               const sgsf_timing_t* timing, void* stream_) {
    if (!h || !cfg || !out || !workspace) return fail(SGSF_ERR_INVALID, "null argument");
    if (batch < 0) return fail(SGSF_ERR_INVALID, "negative batch");
    if (cfg->max_iters < 1) return fail(SGSF_ERR_INVALID, "max_iters must be >= 1");
    if (!(cfg->tol_residual > 0) || !(cfg->tol_eq > 0)) return fail(SGSF_ERR_INVALID, "tolerances must be positive");
    if (batch == 0) return SGSF_OK;
    if (!xi_bar || !out->coeffs || !out->multipliers || !out->res_inf || !out->res_l2 || !out->iterations ||
        !out->converged || !out->displacement || !out->status || !out->eq_err)
        return fail(SGSF_ERR_INVALID, "null input/output buffer");
    if (init_mode && (!xi0 || !lam0)) return fail(SGSF_ERR_INVALID, "init_mode given without xi0/lam0");
    if (cfg->want_prev && !out->coeffs_prev) return fail(SGSF_ERR_INVALID, "want_prev needs coeffs_prev");
    if (h->n > kMaxRobots) return fail(SGSF_ERR_UNSUPPORTED, "n above sgsf_max_robots() is not supported yet");
    cudaStream_t stream = (cudaStream_t)stream_;

    SolveParams p;
    std::memset(&p, 0, sizeof(p));
    p.n = h->n;
    p.S = h->S;
    p.m1 = h->m1;
    p.batch = batch;
    p.max_iters = cfg->max_iters;
    p.early_stop = cfg->early_stop ? 1 : 0;
    p.want_prev = cfg->want_prev ? 1 : 0;
    p.rho = h->rho;
    p.tol_res = cfg->tol_residual;
    p.tol_eq = cfg->tol_eq;
    p.lat = h->lat;
    p.vert = h->vert;
    p.ws_lat = h->ws_lat;
    p.ws_vert = h->ws_vert;
    p.cx = h->center[0];
    p.cy = h->center[1];
    p.cz = h->center[2];
    p.W = h->W;
    p.KMm = h->KMm;
    p.KMd = h->KMd;
    p.cconst = h->cconst;
    p.B6 = h->B6;
    p.rhs = h->rhs;
    p.PBt = h->PBt;
    p.xi_bar = xi_bar;
    p.xi0 = xi0;
    p.lam0 = lam0;
    p.init_mode = init_mode;
    p.coeffs = out->coeffs;
    p.mult = out->multipliers;
    p.res_inf = out->res_inf;
    p.res_l2 = out->res_l2;
    p.iterations = out->iterations;
    p.converged = out->converged;
    p.displacement = out->displacement;
    p.status = out->status;
    p.eq_err = out->eq_err;
    p.coeffs_prev = out->coeffs_prev;
    p.queue = (int*)workspace;
    CUDA_TRY(cudaMemsetAsync(workspace, 0, sizeof(int), stream));
    const char* no_order = std::getenv("SGSF_NO_ORDER");   // (experiments: index order)
    if (batch > 1 && h->n <= 32 && !(no_order && no_order[0] == '1')) {   // longest-first queue order (sf_order.cuh)
        float* score = (float*)((char*)workspace + 256);
        int* order = (int*)((char*)workspace + 256 + align256((size_t)batch * 4));
        const int rc = launch_order(p, score, order, stream);
        if (rc != SGSF_OK) return rc;
        p.order = order;
    }

    if (cfg->precision < SGSF_PRECISION_LEAN || cfg->precision > SGSF_PRECISION_HYBRID)
        return fail(SGSF_ERR_INVALID, "precision must be SGSF_PRECISION_LEAN, _STRICT or _HYBRID");
    const bool strict = cfg->precision == SGSF_PRECISION_STRICT;
    const int n = h->n;
    const bool wide = h->m1 > 12;
    LaunchInfo li{h->device, h->sm_count};
    int rc = SGSF_OK;
    if (n > 32) {
        rc = launch_large(li, p, cfg, timing, stream, cfg->precision == SGSF_PRECISION_STRICT);
    } else {
#define SGSF_PICK(T, NB, MAXT, TPS)                                                      \
    rc = wide ? launch_persistent<T, NB, 16, MAXT, TPS>(li, p, cfg, timing, stream) \
              : launch_persistent<T, NB, 12, MAXT, TPS>(li, p, cfg, timing, stream)
        if (!strict) {
            if (n <= 4) SGSF_PICK(float, 4, 512, 1);
            else if (n <= 8) SGSF_PICK(float, 8, 384, 1);
            else if (n <= 16) SGSF_PICK(float, 16, 384, 1);
            else SGSF_PICK(float, 32, 256, 2);
        } else {
            if (n <= 4) SGSF_PICK(double, 4, 384, 1);
            else if (n <= 8) SGSF_PICK(double, 8, 256, 1);
            else if (n <= 16) SGSF_PICK(double, 16, 256, 1);
            else SGSF_PICK(double, 32, 256, 2);
        }
#undef SGSF_PICK
        // a K1 slot that does not fit (its two position buffers grow with the horizon: FP64 17..32 robots at
        // H = 100, 17..32 robots past 128 time steps, long horizons in FP64): K1L, one CTA of eight warps per
        // sample with the positions of a step in a per-warp scratch
        if (rc == SGSF_ERR_UNSUPPORTED) rc = launch_large(li, p, cfg, timing, stream, strict);
    }
    // the feasible verdict of the returned iterates, right behind the solve on the same stream (fusing it
    // into K1's per-sample epilogue was exact but slowed the iteration loop: +3% to +15%)
    if (rc != SGSF_OK || !out->verdict) return rc;
    sgsf_verdict_t v = *out->verdict;
    return sgsf_verdict(h, batch, out->coeffs, out->converged, cfg->verdict_tol, &v, stream_);
}

int sgsf_verdict(sgsf_handle_t* h, int batch, const double* coeffs, const uint8_t* converged, double tol,
                 sgsf_verdict_t* out, void* stream) {
    if (!h || !out || (batch > 0 && !coeffs)) return fail(SGSF_ERR_INVALID, "null argument");
    if (batch == 0) return SGSF_OK;
    const int threads = 256;
    const size_t smem = (size_t)(3 * h->n * h->m1 + 3 * h->n * AUX_TCH + AUX_TCH * h->m1) * sizeof(double) +
                        threads * (2 * sizeof(double) + 2 * sizeof(int)) + (size_t)h->P * sizeof(int);
    auto kern = h->m1 <= 12 ? verdict_kernel<12> : (h->m1 <= 16 ? verdict_kernel<16> : verdict_kernel<0>);
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<batch, threads, smem, (cudaStream_t)stream>>>(aux_params(h), batch, coeffs, converged, tol,
                                                                    out->ok, out->feasible, out->pair_margin_min,
                                                                    out->ws_margin_max, out->pair_viol,
                                                                    out->ws_viol);
    g_launches.fetch_add(1);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_trajectory(sgsf_handle_t* h, int batch, const double* coeffs, double* pos, double* vel, double* acc,
                    void* stream) {
    if (!h || (batch > 0 && !coeffs)) return fail(SGSF_ERR_INVALID, "null argument");
    if (batch == 0) return SGSF_OK;
    const size_t total = (size_t)batch * h->n * h->S;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    trajectory_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(aux_params(h), batch, coeffs, pos, vel, acc);
    g_launches.fetch_add(1);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_svars(sgsf_handle_t* h, int batch, const double* coeffs, double* paz, double* ppol, double* prad,
               double* waz, double* wpol, double* wrad, void* stream) {
    if (!h || (batch > 0 && (!coeffs || !waz || !wpol || !wrad))) return fail(SGSF_ERR_INVALID, "null argument");
    if (h->P > 0 && batch > 0 && (!paz || !ppol || !prad)) return fail(SGSF_ERR_INVALID, "null pair output");
    if (batch == 0) return SGSF_OK;
    const size_t smem = (size_t)(3 * h->n * h->m1 + 3 * h->n * AUX_TCH) * sizeof(double);
    CUDA_TRY(cudaFuncSetAttribute(svars_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    svars_kernel<<<batch, 256, smem, (cudaStream_t)stream>>>(aux_params(h), batch, coeffs, paz, ppol, prad, waz,
                                                              wpol, wrad);
    g_launches.fetch_add(1);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_spherical_project(int count, const double* dx, const double* dy, const double* dz, double lat,
                           double vert, double lo, double hi, int mode, double* az, double* pol, double* rad,
                           double* tx, double* ty, double* tz, void* stream) {
    if (count < 0) return fail(SGSF_ERR_INVALID, "negative count");
    if (count == 0) return SGSF_OK;
    if (!dx || !dy || !dz) return fail(SGSF_ERR_INVALID, "null input");
    if (mode < 0 || mode > 2) return fail(SGSF_ERR_INVALID, "mode must be 0, 1 or 2");
    int blocks = (count + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    spherical_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(count, dx, dy, dz, lat, vert, lo, hi, mode, az, pol,
                                                                rad, tx, ty, tz);
    g_launches.fetch_add(1);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_apply_F(sgsf_handle_t* h, int batch, const double* xi, double* out, void* stream) {
    if (!h || (batch > 0 && (!xi || !out))) return fail(SGSF_ERR_INVALID, "null argument");
    if (batch == 0) return SGSF_OK;
    const size_t total = (size_t)batch * 3 * (h->P + h->n) * h->S;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    apply_F_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(aux_params(h), batch, xi, out);
    g_launches.fetch_add(1);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_apply_FT(sgsf_handle_t* h, int batch, const double* v, double* out, void* stream) {
    if (!h || (batch > 0 && (!v || !out))) return fail(SGSF_ERR_INVALID, "null argument");
    if (batch == 0) return SGSF_OK;
    const size_t smem = (size_t)(3 * h->n * AUX_TCH + 3 * h->n * h->m1) * sizeof(double);
    CUDA_TRY(cudaFuncSetAttribute(apply_FT_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    apply_FT_kernel<<<batch, 256, smem, (cudaStream_t)stream>>>(aux_params(h), batch, v, out);
    g_launches.fetch_add(1);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_kkt_step(sgsf_handle_t* h, int batch, const double* eta, double* out, double* eq_err, void* stream) {
    if (!h || (batch > 0 && (!eta || !out))) return fail(SGSF_ERR_INVALID, "null argument");
    if (batch == 0) return SGSF_OK;
    if (h->m1 > KMAX_AUX) return fail(SGSF_ERR_UNSUPPORTED, "degree too large");
    const size_t smem = (size_t)(3 * h->m1 + 3 * h->n) * sizeof(double);
    kkt_step_kernel<<<batch, 128, smem, (cudaStream_t)stream>>>(aux_params(h), batch, eta, out, eq_err);
    g_launches.fetch_add(1);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_solve_host(sgsf_handle_t* h, int batch, const double* xi_bar, const double* xi0, const double* lam0,
                    const uint8_t* init_mode, const sgsf_config_t* cfg, double* coeffs, double* multipliers,
                    double* res_inf, double* res_l2, int32_t* iterations, uint8_t* converged, uint8_t* feasible,
                    double* displacement, int32_t* status, void* stream_) {
    if (!h || !cfg) return fail(SGSF_ERR_INVALID, "null argument");
    if (batch <= 0) return batch == 0 ? SGSF_OK : fail(SGSF_ERR_INVALID, "negative batch");
    cudaStream_t stream = (cudaStream_t)stream_;
    const size_t dim = (size_t)3 * h->n * h->m1, B = (size_t)batch, MI = (size_t)cfg->max_iters;
    // one device arena for inputs + outputs (sizes rounded to 256 B each)
    const size_t sizes[] = {B * dim * 8, init_mode ? B * dim * 8 : 0, init_mode ? B * dim * 8 : 0, init_mode ? B : 0,
                            B * dim * 8, B * dim * 8, B * MI * 8, B * MI * 8, B * 4, B, B * 8, B * 4, B * 8, B,
                            sgsf_workspace_bytes(batch)};
    size_t bytes = 0;
    for (size_t z : sizes) bytes += (z + 255) & ~size_t(255);
    char* arena = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&arena, bytes, stream));
    size_t off = 0;
    auto take = [&](size_t nbytes) {
        char* q = arena + off;
        off += (nbytes + 255) & ~size_t(255);
        return (void*)q;
    };
    double* d_xb = (double*)take(sizes[0]);
    double* d_x0 = init_mode ? (double*)take(sizes[1]) : nullptr;
    double* d_l0 = init_mode ? (double*)take(sizes[2]) : nullptr;
    uint8_t* d_mode = init_mode ? (uint8_t*)take(sizes[3]) : nullptr;
    sgsf_outputs_t o;
    std::memset(&o, 0, sizeof(o));
    o.coeffs = (double*)take(sizes[4]);
    o.multipliers = (double*)take(sizes[5]);
    o.res_inf = (double*)take(sizes[6]);
    o.res_l2 = (double*)take(sizes[7]);
    o.iterations = (int32_t*)take(sizes[8]);
    o.converged = (uint8_t*)take(sizes[9]);
    o.displacement = (double*)take(sizes[10]);
    o.status = (int32_t*)take(sizes[11]);
    o.eq_err = (double*)take(sizes[12]);
    uint8_t* d_feas = (uint8_t*)take(sizes[13]);
    void* ws = take(sizes[14]);
    // every step after the arena allocation goes through one cleanup path: the arena is freed and the stream
    // synchronised whatever fails, and the first error is the one reported
    int rc = SGSF_OK;
    auto step = [&](cudaError_t e, const char* what) {
        if (rc == SGSF_OK && e != cudaSuccess) rc = fail(SGSF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    step(cudaMemcpyAsync(d_xb, xi_bar, B * dim * 8, cudaMemcpyHostToDevice, stream), "H2D xi_bar");
    if (init_mode) {
        step(cudaMemcpyAsync(d_x0, xi0, B * dim * 8, cudaMemcpyHostToDevice, stream), "H2D xi0");
        step(cudaMemcpyAsync(d_l0, lam0, B * dim * 8, cudaMemcpyHostToDevice, stream), "H2D lam0");
        step(cudaMemcpyAsync(d_mode, init_mode, B, cudaMemcpyHostToDevice, stream), "H2D init_mode");
    }
    sgsf_config_t c = *cfg;
    c.want_prev = 0;
    if (!(c.verdict_tol > 0)) c.verdict_tol = 1e-3;   // feasible = converged and the constraints at 1e-3 (metrics.py:57-69)
    sgsf_verdict_t v;
    std::memset(&v, 0, sizeof(v));
    v.feasible = d_feas;
    o.verdict = &v;
    if (rc == SGSF_OK) rc = sgsf_solve(h, batch, d_xb, d_x0, d_l0, d_mode, &c, &o, ws, nullptr, stream);
    if (rc == SGSF_OK) {
        struct {
            void* dst;
            const void* src;
            size_t n;
        } outs[] = {{coeffs, o.coeffs, B * dim * 8}, {multipliers, o.multipliers, B * dim * 8},
                    {res_inf, o.res_inf, B * MI * 8}, {res_l2, o.res_l2, B * MI * 8},
                    {iterations, o.iterations, B * 4}, {converged, o.converged, B}, {feasible, d_feas, B},
                    {displacement, o.displacement, B * 8}, {status, o.status, B * 4}};
        for (auto& c2 : outs)
            if (c2.dst) step(cudaMemcpyAsync(c2.dst, c2.src, c2.n, cudaMemcpyDeviceToHost, stream), "D2H output");
    }
    step(cudaFreeAsync(arena, stream), "free arena");
    step(cudaStreamSynchronize(stream), "synchronize");
    return rc;
}

size_t sgsf_cosine_work_doubles(int count, int dim) {
    return 2 * (size_t)(dim > 0 ? dim : 0) + 2 * (size_t)(count > 0 ? count : 0) + 2;
}

int sgsf_pairwise_cosine(int count, int dim, const double* vectors, int center, double* work, double* result,
                         void* stream_) {
    if (count < 2 || dim < 1 || !vectors || !work || !result)
        return fail(SGSF_ERR_INVALID, "pairwise cosine needs >= 2 vectors of length >= 1 and buffers");
    cudaStream_t stream = (cudaStream_t)stream_;
    double* mean = work;
    double* ssum = mean + dim;
    double* inv = ssum + dim;
    double* u2 = inv + count;
    int* zero = (int*)(u2 + count);
    CUDA_TRY(cudaMemsetAsync(zero, 0, sizeof(int), stream));
    const int blocks = (dim + COS_THREADS - 1) / COS_THREADS;
    if (center) {
        cos_colmean_kernel<<<blocks, COS_THREADS, 0, stream>>>(count, dim, vectors, mean);
        internal_count_launch(1);
    }
    cos_rownorm_kernel<<<count, COS_THREADS, 0, stream>>>(count, dim, vectors, center ? mean : nullptr, inv, u2, zero);
    cos_colsum_kernel<<<blocks, COS_THREADS, 0, stream>>>(count, dim, vectors, center ? mean : nullptr, inv, ssum);
    cos_final_kernel<<<1, COS_THREADS, 0, stream>>>(count, dim, ssum, u2, zero, result);
    internal_count_launch(3);
    CUDA_TRY(cudaGetLastError());
    return SGSF_OK;
}

int sgsf_fp32_peak(double* tflops, double* ms, void* stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    int dev = 0, sms = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    float* sink = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&sink, 16, stream));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    ffma_peak_kernel<<<blocks, threads, 0, stream>>>(sink, 64, 1.0f);   // warm-up
    CUDA_TRY(cudaEventRecord(a, stream));
    ffma_peak_kernel<<<blocks, threads, 0, stream>>>(sink, iters, 1.0f);
    CUDA_TRY(cudaEventRecord(b, stream));
    g_launches.fetch_add(2);
    CUDA_TRY(cudaEventSynchronize(b));
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFreeAsync(sink, stream);
    const double flops = 2.0 * 8.0 * 16.0 * iters * (double)blocks * threads;
    if (ms) *ms = t;
    if (tflops) *tflops = flops / (t * 1e-3) / 1e12;
    return SGSF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- differentiable SF (sf_unroll.cuh)
static sgsf::UnrollParams unroll_params(const sgsf_handle_t* h, int batch, int iters) {
    sgsf::UnrollParams p;
    std::memset(&p, 0, sizeof(p));
    p.n = h->n;
    p.S = h->S;
    p.m1 = h->m1;
    p.batch = batch;
    p.iters = iters;
    p.rho = h->rho;
    p.lat = h->lat;
    p.vert = h->vert;
    p.ws_lat = h->ws_lat;
    p.ws_vert = h->ws_vert;
    p.cx = h->center[0];
    p.cy = h->center[1];
    p.cz = h->center[2];
    p.W = h->W;
    p.Km11 = h->Km11;
    p.Kd11 = h->Kd11;
    p.Mm = h->Mm;
    p.Md = h->Md;
    p.G = h->G;
    p.cconst = h->cconst;
    return p;
}

extern "C" {

int sgsf_unroll(sgsf_handle_t* h, int batch, int iters, const double* xi_bar, const double* xi0,
                const double* lam0, double* xs, double* ls, void* stream) {
    if (!h) return fail(SGSF_ERR_INVALID, "null handle");
    if (batch < 0 || iters < 0) return fail(SGSF_ERR_INVALID, "negative batch or iteration count");
    if (h->n > kMaxRobots) return fail(SGSF_ERR_UNSUPPORTED, "n above sgsf_max_robots() is not supported yet");
    if (batch == 0) return SGSF_OK;
    if (!xi_bar || !xi0 || !lam0 || !xs || !ls) return fail(SGSF_ERR_INVALID, "null input/output buffer");
    sgsf::UnrollParams p = unroll_params(h, batch, iters);
    p.xi_bar = xi_bar;
    p.xi0 = xi0;
    p.lam0 = lam0;
    p.xs = xs;
    p.ls = ls;
    return sgsf::launch_unroll_forward(p, (cudaStream_t)stream);
}

int sgsf_unroll_backward(sgsf_handle_t* h, int batch, int iters, const double* xs, const double* gxs,
                         const double* gls, double* g_xi_bar, double* g_xi0, double* g_lam0, void* stream) {
    if (!h) return fail(SGSF_ERR_INVALID, "null handle");
    if (batch < 0 || iters < 0) return fail(SGSF_ERR_INVALID, "negative batch or iteration count");
    if (h->n > kMaxRobots) return fail(SGSF_ERR_UNSUPPORTED, "n above sgsf_max_robots() is not supported yet");
    if (batch == 0) return SGSF_OK;
    if (!xs || !g_xi_bar || !g_xi0 || !g_lam0) return fail(SGSF_ERR_INVALID, "null input/output buffer");
    sgsf::UnrollParams p = unroll_params(h, batch, iters);
    p.xs = const_cast<double*>(xs);
    p.gxs = gxs;
    p.gls = gls;
    p.g_xi_bar = g_xi_bar;
    p.g_xi0 = g_xi0;
    p.g_lam0 = g_lam0;
    return sgsf::launch_unroll_backward(p, (cudaStream_t)stream);
}

}  // extern "C"
