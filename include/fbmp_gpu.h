/*
 * fbmp_gpu.h -- C ABI of the B200 (sm_100a) blind-pansharpening hot path.
 *
 * This is the drop-in boundary for the reference's C++ entry points (reference paths are
 * relative to /root/reference/proj). Every function takes plain pointers and sizes; there
 * are no torch, CUDA or C++ types in the signatures. The C++ shim in
 * paper_2103_09943_b200/host/ implements the reference's `fbmp::` API on top of these
 * calls (see INTEGRATION.md for the bindings a maintainer would add).
 *
 * Conventions
 *   - Planes are row-major float64; stacks are band-major ([band][row][col]).
 *   - `factor` is the decimation ratio c (= r); HR dims are factor x LR dims.
 *   - Host-pointer calls are synchronous: they upload, compute, download and return.
 *   - `_dev` calls take device pointers (allocated on the context's device) and enqueue on
 *     the context's stream; they return once the result is on the device.
 *   - Return codes mirror the reference error taxonomy (include/fbmp/errors.hpp:8-33):
 *       0 ok, 1 ParamError, 2 DimensionError, 3 NumericalError, 4 CUDA/runtime error.
 *     The message (same text as the reference's exception, including the "channel i: "
 *     prefix of pansharpen.cpp:80-92) is available from fbmp_gpu_last_error() on the
 *     calling thread.
 */
#ifndef FBMP_GPU_H
#define FBMP_GPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum fbmp_status {
    FBMP_OK = 0,
    FBMP_PARAM_ERROR = 1,
    FBMP_DIMENSION_ERROR = 2,
    FBMP_NUMERICAL_ERROR = 3,
    FBMP_RUNTIME_ERROR = 4
};

/* PansharpenParams (pansharpen.hpp:15-26), Laplacian or identity prior. `threads` is accepted for API
 * parity and ignored: all channels of a call are solved concurrently on the device. */
typedef struct fbmp_ps_params {
    double lambda;   /* 2e-4 */
    int radius;      /* 1 */
    double eps;      /* 1e-4 */
    double cg_tol;   /* 5e-5 */
    int cg_max_iter; /* 2000 */
    int threads;     /* 0 */
    int prior;       /* PriorKind: 0 laplacian (default), 1 identity; custom (2) is not provided */
} fbmp_ps_params;

/* KernelEstParams (kernel_estimator.hpp:16-31). init: 0 = dirac, 1 = uniform. */
typedef struct fbmp_ke_params {
    int n;          /* 29 */
    double alpha1;  /* 1.0 */
    double alpha2;  /* 0.006 */
    double mu1, mu2, mu3; /* 100 */
    double rho;     /* 0.5 */
    int t_max;      /* 10000 */
    double th;      /* 1e-5 */
    int init;       /* 0 */
} fbmp_ke_params;

/* SpectralWeightConfig (spectral_weights.hpp:9-14); band_indices are applied by the caller. */
typedef struct fbmp_sw_params {
    int l;               /* 4 */
    double lambda_omega; /* 10 */
    int factor;          /* 2 */
} fbmp_sw_params;

typedef struct fbmp_gpu_ctx fbmp_gpu_ctx;

/* Per-solve statistics of the last pansharpen / blind call on a context. */
typedef struct fbmp_gpu_stats {
    int admm_iters;      /* ADMM iterations of the kernel fit (0 if not run) */
    int cg_iters[64];    /* CG iterations per channel (first 64 channels) */
    double ms_weights, ms_kernel_fit, ms_pansharpen; /* device time of the stages */
    long long cg_channel_iters; /* sum of the CG iterations over all channels of the last solve */
    int n_channels;      /* channels of the last solve (scenes x bands); cg_iters holds the first
                            min(n_channels, 64): fbmp_gpu_ctx_cg_iters returns all of them */
} fbmp_gpu_stats;

void fbmp_gpu_default_ps_params(fbmp_ps_params* p);
void fbmp_gpu_default_ke_params(fbmp_ke_params* p);
void fbmp_gpu_default_sw_params(fbmp_sw_params* p);

/* Context: owns the device workspace, cuFFT plans and the stream. One per host thread. */
int fbmp_gpu_ctx_create(int device, fbmp_gpu_ctx** out);
void fbmp_gpu_ctx_destroy(fbmp_gpu_ctx* ctx);
const char* fbmp_gpu_last_error(void);
int fbmp_gpu_ctx_stats(fbmp_gpu_ctx* ctx, fbmp_gpu_stats* out);
/* Per-channel CG iteration counts of the last solve (all scenes x bands, scene-major) into
 * out[0 .. cap); returns the number of channels (which may exceed cap), or -1 on error. */
int fbmp_gpu_ctx_cg_iters(fbmp_gpu_ctx* ctx, int* out, int cap);
/* The context's cudaStream_t, as an opaque pointer (for device-resident callers). */
void* fbmp_gpu_ctx_stream(fbmp_gpu_ctx* ctx);
/* Number of kernels this library launched on the context so far (instrumentation). */
long long fbmp_gpu_ctx_launches(fbmp_gpu_ctx* ctx);
/* Profiling of the CG loop: when on, CUDA events bracket each CG kernel (graphs are not
 * pipelined). kernel_profile fills 4 entries of total device ms and launch counts for
 * {K_Q (p update + D B p), K_D (B^T U q), K_L (+ lambda L M L p, p.Ap), K_U (axpys + norms)};
 * with the single-kernel operator (env FBMP_KA=4) K_D is empty and K_L holds K_A. */
void fbmp_gpu_ctx_set_profile(fbmp_gpu_ctx* ctx, int on);
/* Precision of the HRMS conjugate-gradient loop (the hot path): 64 (default, the reference's
 * fp64 arithmetic) or 32 (fp32 mode of BASELINE.json's north_star: CG vectors, taps, guide and
 * window maps stored and stenciled in fp32; every dot product, norm and CG scalar in fp64; the
 * kernel fit, guided filter and alias-group solve stay fp64). The fp32 mode needs the specialised
 * operator (radius 1, factor 2 or 4, supported kernel side, images >= 64 x 64, even width) and the
 * single-domain path (not row strips); otherwise the solve fails with FBMP_PARAM. Returns a status. */
int fbmp_gpu_ctx_set_precision(fbmp_gpu_ctx* ctx, int bits);
int fbmp_gpu_ctx_precision(fbmp_gpu_ctx* ctx);
int fbmp_gpu_ctx_kernel_profile(fbmp_gpu_ctx* ctx, double* total_ms, long long* launches);

/* ---- full pipeline ----------------------------------------------------------------------- */

/* pansharpen (pansharpen.hpp:95-96 / pansharpen.cpp:367-424). lrms: N*h*w, pan: H*W,
 * k: n*n taps, out: N*H*W. cg_iters (optional, N ints) receives per-channel CG counts. */
int fbmp_gpu_pansharpen(fbmp_gpu_ctx* ctx, const double* lrms, int N, int h, int w, const double* pan,
                        const double* k, int n, int factor, const fbmp_ps_params* params, double* out,
                        int* cg_iters);

/* l2 + simplex kernel estimate (kernel_estimator.cpp:389-428 through estimate_kernel_plane with
   KernelPrior::l2, :438-455): same scaling and errors as the TGV path; params.n, alpha1, alpha2,
   mu3, rho, t_max, th, init are used. k_out: n*n; iters: ADMM iterations (optional). */
int fbmp_gpu_estimate_kernel_l2_plane(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs,
                                      int factor, const fbmp_ke_params* params, double* k_out, int* iters);
/* TV kernel prior: estimate_kernel_plane with KernelPrior::tv (kernel_estimator.cpp:445-452,
   run_tgv_or_tv(false, ...) :291-387): same scaling, errors and ADMM as the TGV path with p = 0
   and the u-step divided by the scalar symbol alpha1 mu1 |grad|^2 + mu3; alpha2 / mu2 unused.
   state_out / hook_t as fbmp_gpu_estimate_kernel_plane (p, y, L2 stay zero). */
int fbmp_gpu_estimate_kernel_tv_plane(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs,
                                      int factor, const fbmp_ke_params* params, double* k_out, int* iters,
                                      double* state_out, int hook_t);
/* estimate_kernel_tv (kernel_estimator.hpp:120-123): combine_bands(lrms, omega) then the TV fit. */
int fbmp_gpu_estimate_kernel_tv(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w,
                                const double* pan, const double* omega, int factor,
                                const fbmp_ke_params* params, double* k_out, int* iters);
/* estimate_kernel_tgv (kernel_estimator.hpp:114-118): combine_bands(lrms, omega) then the
 * TGV^2 fit. k_out: n*n. iters (optional) receives the ADMM iteration count. */
int fbmp_gpu_estimate_kernel_tgv(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w,
                                 const double* pan, const double* omega, int factor,
                                 const fbmp_ke_params* params, double* k_out, int* iters);

/* estimate_kernel_plane with KernelPrior::tgv2 (kernel_estimator.hpp:109-112). obs: h*w.
 * state_out (optional, 17*n*n: u,p1,p2,x0,x1,y0..y3,z,L1_0,L1_1,L2_0..L2_3,L3) receives the
 * final TgvAdmmState; hook_t >= 0 stops right before the {u,p} solve of iteration hook_t
 * and returns that state (the reference's before_up_solve hook point). */
int fbmp_gpu_estimate_kernel_plane(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs,
                                   int factor, const fbmp_ke_params* params, double* k_out, int* iters,
                                   double* state_out, int hook_t);

/* solve_weights (spectral_weights.hpp:24-25). omega_out: nb doubles. */
int fbmp_gpu_solve_weights(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w,
                           const double* pan, const fbmp_sw_params* cfg, double* omega_out);

/* combine_bands (spectral_weights.hpp:28-29). out: h*w. */
int fbmp_gpu_combine_bands(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w,
                           const double* omega, double* out);

/* SPEC.md:584-591 blind composition (solve_weights on all bands -> estimate_kernel_tgv ->
 * pansharpen). k_out: n*n (n = ke->n), omega_out: N (both optional). */
int fbmp_gpu_blind(fbmp_gpu_ctx* ctx, const double* lrms, int N, int h, int w, const double* pan,
                   const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps, double* out,
                   double* k_out, double* omega_out);

/* Device-resident blind solve (same semantics; all pointers are device pointers). */
int fbmp_gpu_blind_dev(fbmp_gpu_ctx* ctx, const double* d_lrms, int N, int h, int w, const double* d_pan,
                       const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps,
                       double* d_out, double* d_k_out);

/* Channel-sharded blind solve (BASELINE config C3, one rank per GPU): the spectral weights,
 * the kernel fit and the intensity normalisation use all N bands (replicated on every rank,
 * deterministic), only bands [ch0, ch0+nch) are reconstructed. out: nch*H*W. */
int fbmp_gpu_blind_subset(fbmp_gpu_ctx* ctx, const double* lrms, int N, int h, int w, const double* pan,
                          const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps, int ch0,
                          int nch, double* out, double* k_out);

/* Batch of independent scenes (no reference equivalent; BASELINE config C4): S scenes of
 * identical shape, each with its own weights, kernel fit and HRMS solve. */
int fbmp_gpu_blind_batch(fbmp_gpu_ctx* ctx, const double* lrms, int S, int N, int h, int w, const double* pan,
                         const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps,
                         double* out, double* k_out);

/* Device-resident general form: S scenes (all bands; d_out S*N*H*W, d_k_out S*n*n), or one scene
 * (S = 1) with the channel subset [ch0, ch0+nch) (nch = -1: all bands; d_out nch*H*W). */
int fbmp_gpu_blind_batch_dev(fbmp_gpu_ctx* ctx, const double* d_lrms, int S, int N, int h, int w,
                             const double* d_pan, const fbmp_sw_params* sw, const fbmp_ke_params* ke,
                             const fbmp_ps_params* ps, int ch0, int nch, double* d_out, double* d_k_out);

/* Row-strip (multi-GPU) blind solve of one scene (BASELINE config C5 on several GPUs).
 * Inputs (full LRMS / PAN) are replicated on every rank; the spectral weights and the kernel fit
 * run replicated, the CG runs on row strips with an r-halo exchange and two allreduces per
 * iteration (NCCL), the post-processing per channel on rank (channel mod G). With a communicator
 * (fbmp_gpu_ctx_set_comm) the strips are the ranks and vstrips is ignored; without one, vstrips
 * virtual ranks run in this process. d_out (N*H*W) is complete on rank 0. */
int fbmp_gpu_blind_strips_dev(fbmp_gpu_ctx* ctx, const double* d_lrms, int N, int h, int w, const double* d_pan,
                              const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps,
                              int vstrips, double* d_out, double* d_k_out);
/* NCCL bootstrap: rank 0 creates the 128-byte id, the launcher broadcasts it, every rank calls
 * set_comm (collective) on its context. */
int fbmp_gpu_nccl_unique_id(unsigned char* id128);
int fbmp_gpu_ctx_set_comm(fbmp_gpu_ctx* ctx, const unsigned char* id128, int nranks, int rank);

/* ---- unit-level entry points (parity tests) -------------------------------------------- */

/* apply_prior / apply_prior_adjoint (pansharpen.hpp:28-29): circular 5-point Laplacian. */
int fbmp_gpu_apply_prior(fbmp_gpu_ctx* ctx, const double* img, int H, int W, double* out);
/* MattingMatrix::apply(Plane) (pansharpen.hpp:47, :197-202), matrix-free: y = M(guide) x. */
int fbmp_gpu_llp_apply(fbmp_gpu_ctx* ctx, const double* guide, const double* x, int H, int W, int radius,
                       double eps, double* y);
/* B^T U D B p (the data term of pansharpen.cpp:218-223). */
int fbmp_gpu_data_apply(fbmp_gpu_ctx* ctx, const double* p, int H, int W, const double* k, int n, int factor,
                        double* out);
/* The full CG operator A(p) of pansharpen.cpp:218-223 with M built on `guide`. */
int fbmp_gpu_cg_operator(fbmp_gpu_ctx* ctx, const double* guide, const double* p, int H, int W, const double* k,
                         int n, int factor, const fbmp_ps_params* params, double* out);
/* warmstart_cg (pansharpen.hpp:73-75) with M built on `guide` (= L(pan_n) in the pipeline). */
int fbmp_gpu_warmstart_cg(fbmp_gpu_ctx* ctx, const double* x, int h, int w, const double* guide, const double* k,
                          int n, int factor, const fbmp_ps_params* params, int max_iters, int error_on_cap,
                          double* z_out, int* iters, double* final_residual);
/* guided_coeffs + guided_output (pansharpen.hpp:83-84). a_out / c_out optional. */
int fbmp_gpu_guided_filter(fbmp_gpu_ctx* ctx, const double* input, const double* guide, int H, int W, int radius,
                           double eps, double* a_out, double* c_out, double* v_out);
/* guided_output alone (pansharpen.hpp:84). */
int fbmp_gpu_guided_output(fbmp_gpu_ctx* ctx, const double* a, const double* c, const double* guide, int H, int W,
                           int radius, double* out);
/* solve_channel_fft (pansharpen.hpp:90-91). */
int fbmp_gpu_solve_channel_fft(fbmp_gpu_ctx* ctx, const double* x, int h, int w, const double* k, int n,
                               int factor, const double* v, const fbmp_ps_params* params, double* out);
/* Evaluation metrics (metrics.hpp:11-51) of est against ref (N x H x W, band-major), both cropped
   by `crop` pixels (crop_border, metrics.hpp:28-29): `which` selects 1 PSNR (per band into
   psnr_per_band[N] and their mean), 2 regressed PSNR, 4 ERGAS (ratio `factor`), 8 SAM (degrees),
   16 RASE; out[0..4] = psnr_avg, psnr_reg_avg, ergas, sam_deg, rase (NaN when not selected).
   Inputs on the [0, 255] scale as in the reference. Errors as the reference: negative margin
   (param), margin leaving no pixels (dimension), zero reference mean in ERGAS / RASE (numerical). */
int fbmp_gpu_metrics(fbmp_gpu_ctx* ctx, const double* est, const double* ref, int N, int H, int W, int crop,
                     int factor, int which, double* psnr_per_band, double* out);
/* box_mean (ops.hpp:32), circular convolution and its adjoint (ops.hpp:10-15). */
int fbmp_gpu_box_mean(fbmp_gpu_ctx* ctx, const double* img, int H, int W, int radius, double* out);
int fbmp_gpu_convolve(fbmp_gpu_ctx* ctx, const double* img, int H, int W, const double* k, int n, int adjoint,
                      double* out);
/* shrink2 (kernel_estimator.hpp:65): cols is ncols consecutive planes of m samples, in place. */
int fbmp_gpu_shrink2(fbmp_gpu_ctx* ctx, double* cols, int ncols, long long m, double t);
/* project_simplex (kernel_estimator.hpp:68). */
int fbmp_gpu_project_simplex(fbmp_gpu_ctx* ctx, const double* v, int m, double* out);
/* solve_up (kernel_estimator.hpp:78-80) with optional mu3 coupling to anchor (= z - L3).
 * fields: 12 n*n planes x0,x1,y0..y3,L1_0,L1_1,L2_0..L2_3. */
int fbmp_gpu_solve_up(fbmp_gpu_ctx* ctx, const double* fields, int n, const fbmp_ke_params* params,
                      double coupling, const double* anchor, double* u, double* p1, double* p2);
/* E^T E (n^2 x n^2) and E^T f of ObservationSystem (kernel_estimator.cpp:57-71), unscaled. */
int fbmp_gpu_gram(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs, int factor, int n,
                  double* EtE, double* Etf);
/* ObservationSystem::solve_z (kernel_estimator.cpp:79-83) on the device for a Gram matrix from
 * fbmp_gpu_gram: z = (E^T E + mu3 I)^-1 (E^T f + mu3 anchor) (Cholesky, explicit inverse,
 * mat-vec). EtE: n2*n2, Etf / anchor / z_out: n2 (n2 = n*n). FBMP_NUMERICAL if not SPD. */
int fbmp_gpu_solve_z(fbmp_gpu_ctx* ctx, const double* EtE, const double* Etf, int n, double mu3,
                     const double* anchor, double* z_out);
/* ObservationSystem::data_objective (kernel_estimator.cpp:85-87): 0.5 (u'EtE u - 2 u'Etf + ff). */
int fbmp_gpu_data_objective(fbmp_gpu_ctx* ctx, const double* EtE, const double* Etf, int n, double ff,
                            const double* u, double* value);

#ifdef __cplusplus
}
#endif
#endif /* FBMP_GPU_H */
