// pansharpen.cuh -- device-side entry points of Algorithm 2 (HRMS reconstruction).
#pragma once
#include "common.cuh"

namespace fbmp_gpu {

// Per-channel CG scalars (pansharpen.cpp:225-256), resident on the device.
struct CgState {
    double rs;        // r.r at the start of the current iteration
    double rhs_norm;  // ||rhs||
    double pp;        // ||p||^2 of the current iteration (K_Q)
    double pAp;       // p.Ap (K_A)
    double alpha;     // rs / pAp (K_A)
    double beta;      // rs_new / rs for the next p update (K_U)
    double zz;        // ||z||^2 after the update (K_U)
    double qq;        // ||q||^2 = p . B^T U D B p of the current iteration (K_Q3; fused K_L / K_DU path)
    double cg_tol;
    int t;            // iteration index
    int done;         // 0 running, 1 converged, 2 non-positive curvature, 3 iteration cap
    int iters;        // operator applications performed (reference's `it + 1`)
    int max_iters;
    unsigned int cnt_init, cnt_q, cnt_a, cnt_u;  // last-block election counters
};

struct PsGeo {
    int H, W, h, w, c, n, C, g;  // C = (n-1)/2, g = ceil(C/c)
    int rw;                       // matting / guided-filter window radius
    double lambda, eps;
    int N;                        // channels in the launch (all scenes)
    int cps;                      // channels per scene: channel ch uses scene ch / cps's
                                  // taps, guide and intensity scale
    int cpc;                      // channels per CTA in the fast K_A (guide tile reuse)
    int dbg;                      // development: bitmask of K_A stages to skip (timing only)
    int identity;                 // 1: identity pansharpening prior (pansharpen.cpp:28-78), 0: Laplacian
    // row-strip domain decomposition (distributed CG, csrc/dist.cu); defaults = whole image:
    int grow0, Hg;                // global row of local row 0 (mod Hg), global height
    int rlo, rhi;                 // local rows owned by this strip: CG dot products sum only these
    double* dred;                 // non-null: kernels publish per-channel LOCAL sums here
                                  //   [0, N): p.Ap; [N + 3 ch + {0,1,2}]: ||p||^2, ||r||^2, ||z||^2
                                  // and leave the CG scalar update to k_dist_* after an allreduce
};

PsGeo make_geo(int N, int h, int w, int c, int n, int rw, double lambda, double eps, int cps = 0);

// Workspace of one batched CG solve (all device pointers, channel-major).
template <class T>
struct CgBuffersT {  // T = double (reference precision) or float (fp32 mode)
    T* z;           // N*P  (output: warm start)
    T* r;           // N*P
    T* p;           // 2*N*P (parity double buffer)
    T* Ap;          // N*P
    T* q;           // N*p  (D B p at the LR points)
    double* part;   // partial sums, 4 * N * max_blocks
    CgState* st;    // N
    int max_blocks;
};
using CgBuffers = CgBuffersT<double>;

// Enqueue the whole CG warm start for N channels sharing `guide` (= L(pan_n)) and taps.
// x: N*h*w (already scaled). Returns after the loop finished (host polls device flags).
void cg_solve(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_guide, const double* d_x,
              CgBuffers& B, int max_iters, double cg_tol, std::vector<CgState>& host_state);
// fp32 mode: the same loop with fp32 vectors (taps, guide, x converted by the caller; the guide
// maps are formed from the fp64 guide), fp64 reductions and CG scalars. Fast path only.
void cg_solve_f32(Context& ctx, const PsGeo& G, const float* d_taps, const double* d_guide64, const float* d_guide,
                  const float* d_x, CgBuffersT<float>& B, int max_iters, double cg_tol,
                  std::vector<CgState>& host_state);
// elementwise fp64 -> fp32 / fp32 -> fp64 copies (fp32 mode staging)
void to_f32(Context& ctx, const double* d_in, long long n, float* d_out);
void to_f64(Context& ctx, const float* d_in, long long n, double* d_out);

// Row-strip decomposition of the CG (csrc/pansharpen.cu, "Row-strip decomposition").
struct StripCg {
    PsGeo G;               // padded strip geometry with grow0 / Hg / rlo / rhi / dred set
    const double* taps;    // n*n
    const double* guide;   // strip of L(pan_n) (H' x W)
    const double* wmu;     // strips of the window statistics (computed on the whole image)
    const double* wg;
    const double* x;       // LR strip (N x H'/c x w), scaled
    CgBuffers B;
    double* dred;          // 4 N (same pointer as G.dred)
};
struct StripComm {
    void* nccl = nullptr;  // ncclComm_t: one strip per rank; null: the strips are virtual ranks
    int nranks = 1, rank = 0;
    int halo = 32;         // rows above and below every strip
};
void cg_solve_strips(Context& ctx, std::vector<StripCg>& strips, const StripComm& comm, int max_iters,
                     double cg_tol, std::vector<CgState>& host_state);

// A(p) (pansharpen.cpp:218-223) for N channels: mode 0 full operator, 1 matting only (M p),
// 2 data term only (B^T U D B p).
void cg_operator_apply(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_guide,
                       const double* d_p, double* d_out, int mode);

// per-scene window statistics of the fast operator: mu_k, g_k = [interior] / (eps/9 + var_k)
void guide_stats(Context& ctx, const PsGeo& G, const double* d_guide, double* mu, double* gk);

// rhs = B^T U x (pansharpen.cpp:225).
void data_rhs(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_x, double* d_out);

// Guided filter (pansharpen.cpp:274-312, called as in :396-399 with input = L(z0) unless
// input_is_plain): v = box(a)*guide + box(c). a_out/c_out optional.
void guided_filter(Context& ctx, int N, int H, int W, int rw, double eps, const double* d_in, int in_is_z0,
                   const double* d_guide, double* d_a, double* d_c, double* d_v, int cps = 0);

// solve_channel_fft (pansharpen.cpp:314-365) for N channels (taps per scene).
// d_scale (device, one per scene, optional): out is multiplied by 1/scale (pansharpen.cpp:401).
void solve_channel_fft(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_x, const double* d_v,
                       const double* d_scale, double* d_out, int* d_flag);

// Elementwise / stencil helpers.
// per-scene 1/max(PAN, LRMS) (pansharpen.cpp:374-376); d_scale: S doubles
void peak_scale(Context& ctx, const double* d_pan, long long P, const double* d_lrms, long long Np, int S,
                double* d_scale);
// out = in * scale[i / per_scale]
void scale_copy(Context& ctx, const double* d_in, long long n, const double* d_scale, long long per_scale,
                double* d_out);
void guided_combine(Context& ctx, const double* d_ab, const double* d_cb, const double* d_g, long long n,
                    double* d_out);
void laplacian_scaled(Context& ctx, const double* d_in, int H, int W, int N, const double* d_scale, double* d_out);
void box_mean(Context& ctx, const double* d_in, int H, int W, int N, int radius, double* d_out);
void convolve(Context& ctx, const double* d_in, int H, int W, const double* d_taps, int n, int adjoint,
              double* d_out);

}  // namespace fbmp_gpu
