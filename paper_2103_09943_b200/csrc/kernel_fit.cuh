// kernel_fit.cuh -- device-side entry points of Algorithm 1 (TGV^2 blur-kernel fit) and the
// spectral-weight stage that feeds it.
#pragma once
#include "common.cuh"

namespace fbmp_gpu {

void validate_ps(const fbmp_ps_params& p);
void validate_ke(const fbmp_ke_params& p);

// solve_weights (spectral_weights.cpp:9-53) for S scenes: lrms S*nb*h*w, pan S*H*W,
// omega out S*nb (device). d_status (S ints): 0 ok, 1 singular, 2 residual too large.
void solve_weights_device(Context& ctx, const double* d_lrms, int S, int nb, int h, int w, const double* d_pan,
                          int l, double lambda_omega, int c, double* d_omega, int* d_status);

// combine_bands (spectral_weights.cpp:55-65): out S*h*w.
void combine_bands_device(Context& ctx, const double* d_lrms, int S, int nb, long long p, const double* d_omega,
                          double* d_out);

// PAN statistics for check_degenerate / intensity_scale (kernel_estimator.cpp:269-289):
// stats[s*4 + {0,1,2,3}] = {sum, min, max, max|v|}.
void pan_stats(Context& ctx, const double* d_pan, int S, long long P, double* d_stats);

// Scaled observation system: EtE + mu3 I (n2 x n2), Etf, for pan_n = pan*s, obs_n = obs*s
// (scale per scene in d_s). Returns device pointers inside ctx scratch.
struct ObsSystem {
    int S, n, n2;
    double* M;     // S * n2 * n2 : E^T E + mu3 I (lower triangle meaningful), then Cholesky factor
    double* Etf;   // S * n2
    double* Ginv;  // S * n2 * n2 : (E^T E + mu3 I)^-1 (exactly symmetric)
    double* g;     // S * n2 : Ginv Etf
    int* status;   // S : 0 ok, 1 factorization failed
};
void build_observation(Context& ctx, const double* d_pan, const double* d_obs, int S, int H, int W, int c, int n,
                       double mu3, const double* d_scale, ObsSystem& sys, bool want_inverse, double l2_a1 = 0.0,
                       double l2_a2 = 0.0, bool split = false);
// Cholesky (and the explicit inverse) of sys.M, sys.S systems of side sys.n2; sys.status set on failure
void factor_invert(Context& ctx, ObsSystem& sys, bool want_inverse);
// public ObservationSystem::solve_z / data_objective on a device Gram matrix (kernel_estimator.cpp:79-87)
void solve_z_device(Context& ctx, const double* d_EtE, const double* d_Etf, int n2, double mu3,
                    const double* d_anchor, double* d_z);
void data_objective_device(Context& ctx, const double* d_EtE, const double* d_Etf, const double* d_u, int n2,
                           double ff, double* d_out);
// l2 + simplex kernel estimate of one scene (kernel_estimator.cpp:389-428): device pan / obs, d_k: n*n
void estimate_kernel_l2_device(Context& ctx, const double* d_pan, const double* d_obs, int H, int W, int c,
                               const fbmp_ke_params& prm, double* d_k, int* iters);

// ADMM (kernel_estimator.cpp:291-387). state: S * 17 * n2 (u,p1,p2,x0,x1,y0..y3,z,L1_0,L1_1,
// L2_0..L2_3,L3). If resume_state is null the state is initialised (dirac/uniform). Runs
// until convergence, t_max, or -- when hook_t >= 0 -- the end of the z-step of iteration
// hook_t. info: S * 4 ints {iterations, status, t_stopped, phase} with status 0 ok,
// 1 non-finite u, 2 non-finite z, 3 simplex empty support, 4 stopped at hook.
void admm_device(Context& ctx, const ObsSystem& sys, const fbmp_ke_params& prm, double* d_state,
                 bool init_state, int t_begin, int phase_begin, int hook_t, int* d_info);

// Reference-compatible solve_up (kernel_estimator.cpp:137-241) on the device (one system).
void solve_up_device(Context& ctx, const double* d_fields, int n, const fbmp_ke_params& prm, double coupling,
                     const double* d_anchor, double* d_u, double* d_p1, double* d_p2);
void shrink2_device(Context& ctx, double* d_cols, int ncols, long long m, double t);
void project_simplex_device(Context& ctx, const double* d_v, int m, double* d_out, int* d_status);

// Unscaled Gram (E^T E, E^T f) for the parity tests.
void gram_device(Context& ctx, const double* d_pan, const double* d_obs, int H, int W, int c, int n, double* d_EtE,
                 double* d_Etf);

// Full kernel estimate for S scenes from (pan, obs): writes kernels S*n2 (device) and
// host-side iteration counts; throws the reference's errors. tv: the TV kernel prior
// (KernelPrior::tv, kernel_estimator.cpp:445-452) instead of TGV^2. split: with a communicator on
// the context (C5 row strips), the Gram tiles are split over the ranks (bit-identical result).
void estimate_kernel_device(Context& ctx, const double* d_pan, const double* d_obs, int S, int H, int W, int c,
                            const fbmp_ke_params& prm, double* d_k, std::vector<int>& iters, double* d_state_out,
                            int hook_t, bool tv = false, bool split = false);

// Evaluation metrics (csrc/metrics.cu, metrics.hpp:11-51): device inputs, host outputs.
void metrics_device(Context& ctx, const double* d_est, const double* d_ref, int N, int H, int W, int crop,
                    int factor, int which, double* psnr_per_band, double* out);

}  // namespace fbmp_gpu
