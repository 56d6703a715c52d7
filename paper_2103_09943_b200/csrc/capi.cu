// capi.cu -- the C ABI (include/fbmp_gpu.h): context management and the reference-facing
// entry points. Host-pointer calls upload, run the device path and download; there is no
// CPU fallback anywhere in this library.
#include <nccl.h>

#include <cstring>
#include <string>

#include "kernel_fit.cuh"
#include "pansharpen.cuh"

namespace fbmp_gpu {

thread_local std::string g_last_error;

Context::Context(int dev) : device(dev) {
    FBMP_CUDA(cudaSetDevice(dev));
    FBMP_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    cudaDeviceProp prop{};
    FBMP_CUDA(cudaGetDeviceProperties(&prop, dev));
    sm_count = prop.multiProcessorCount;
    if (prop.major < 10)
        throw Failure(FBMP_RUNTIME_ERROR, "fbmp_gpu requires an sm_100 (Blackwell) device; found " +
                                              std::string(prop.name));
}

Context::~Context() {
    cudaSetDevice(device);
    if (nccl) ncclCommDestroy(static_cast<ncclComm_t>(nccl));
    for (auto& kv : plans) cufftDestroy(kv.second);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (auto& e : poll_ev)
        if (e) cudaEventDestroy(e);
    if (pinned_buf) cudaFreeHost(pinned_buf);
    for (auto& a : aux_streams)
        if (a) cudaStreamDestroy(a);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    for (auto& e : copy_ev)
        if (e) cudaEventDestroy(e);
    if (fork_ev) cudaEventDestroy(fork_ev);
    for (auto& e : join_evs)
        if (e) cudaEventDestroy(e);
    ws.clear();
    if (stream) cudaStreamDestroy(stream);
}

void* Context::pinned(size_t bytes) {
    if (bytes > pinned_bytes) {
        if (pinned_buf) {
            FBMP_CUDA(cudaStreamSynchronize(stream));
            FBMP_CUDA(cudaFreeHost(pinned_buf));
            pinned_buf = nullptr;
        }
        const size_t nb = std::max<size_t>(bytes, 64 << 10);
        FBMP_CUDA(cudaMallocHost(&pinned_buf, nb));
        pinned_bytes = nb;
    }
    return pinned_buf;
}

cufftHandle Context::plan(int kind, int rows, int cols, int batch) {
    const auto key = std::make_tuple(kind, rows, cols, batch, 0);
    auto it = plans.find(key);
    if (it != plans.end()) return it->second;
    cufftHandle h;
    int dims[2] = {rows, cols};
    FBMP_CUFFT(cufftPlanMany(&h, 2, dims, nullptr, 1, 0, nullptr, 1, 0, kind == 0 ? CUFFT_D2Z : CUFFT_Z2D, batch));
    FBMP_CUFFT(cufftSetStream(h, stream));
    plans[key] = h;
    return h;
}

void validate_ps(const fbmp_ps_params& p) {  // pansharpen.cpp:96-105 (Laplacian prior)
    if (!(p.lambda > 0)) param_error("pansharpen: lambda must be positive");
    if (p.radius < 1) param_error("pansharpen: radius must be >= 1");
    if (!(p.eps > 0)) param_error("pansharpen: eps must be positive");
    if (!(p.cg_tol > 0)) param_error("pansharpen: cg_tol must be positive");
    if (p.cg_max_iter < 1) param_error("pansharpen: cg_max_iter must be >= 1");
    if (p.threads < 0) param_error("pansharpen: threads must be >= 0");
    if (p.prior == 2) param_error("pansharpen: custom prior requires a kernel");  // pansharpen.cpp:103-104
    if (p.prior != 0 && p.prior != 1)
        param_error("pansharpen: the GPU path implements the Laplacian and identity priors");
}

static void check_kernel(int n, int H, int W) {
    if (n < 1 || n % 2 == 0) param_error("kernel size must be odd and positive");
    if (n > H || n > W) dim_error("kernel larger than image");
}

// Batched HRMS solve on device-resident data (pansharpen.cpp:367-424) for S scenes of N
// channels each: lrms S*N*h*w, pan S*H*W, taps S*n*n, out S*N*H*W.
void pansharpen_device(Context& ctx, const double* d_lrms, int S, int N, int h, int w, const double* d_pan,
                       const double* d_taps, int n, int c, const fbmp_ps_params& prm, double* d_out,
                       std::vector<int>& cg_iters, int ch0 = 0, int nch = -1) {
    validate_ps(prm);
    const int H = h * c, W = w * c;
    if (2 * prm.radius + 1 > std::min(H, W)) dim_error("matting matrix: window larger than image");
    check_kernel(n, H, W);
    const int NS = nch < 0 ? N : nch;  // channels solved per scene (a subset [ch0, ch0+NS) when S == 1)
    if (ch0 < 0 || ch0 + NS > N || (S > 1 && NS != N)) param_error("pansharpen: invalid channel subset");
    const int NC = S * NS;
    const size_t P = static_cast<size_t>(H) * W, p = static_cast<size_t>(h) * w;
    PsGeo G = make_geo(NC, h, w, c, n, prm.radius, prm.lambda, prm.eps, NS);
    G.identity = prm.prior == 1;
    double* scale = ctx.scratch<double>("ps_scale", S);
    double* lpan = ctx.scratch<double>("ps_lpan", P * S);
    double* xn = ctx.scratch<double>("ps_xn", p * NC);
    // normalisation over PAN and ALL bands (pansharpen.cpp:374-376), also for a subset solve
    peak_scale(ctx, d_pan, static_cast<long long>(P), d_lrms, static_cast<long long>(p) * N, S, scale);
    if (G.identity)  // prior.apply(pan_n) (pansharpen.cpp:379): the identity keeps pan_n
        scale_copy(ctx, d_pan, static_cast<long long>(P) * S, scale, static_cast<long long>(P), lpan);
    else
        laplacian_scaled(ctx, d_pan, H, W, S, scale, lpan);
    scale_copy(ctx, d_lrms + static_cast<size_t>(ch0) * p, static_cast<long long>(p) * NC, scale,
               static_cast<long long>(p) * NS, xn);

    CgBuffers B;
    B.z = ctx.scratch<double>("cg_z", P * NC);
    const size_t nbmax = (P / 256 + 64) * 2 + 4096;
    B.part = ctx.scratch<double>("cg_part", 4 * nbmax * NC);
    B.st = ctx.scratch<CgState>("cg_state", NC);
    std::vector<CgState> hs;
    trace("ps: prologue");
    if (ctx.precision == 32) {
        // fp32 mode: the CG vectors, taps, guide and its window maps in fp32; every dot product,
        // norm and CG scalar in fp64. The warm start is widened to fp64 for the guided filter and
        // the alias-group solve, which stay fp64 (once per channel).
        CgBuffersT<float> F;
        F.z = ctx.scratch<float>("cg32_z", P * NC);
        F.r = ctx.scratch<float>("cg32_r", P * NC);
        F.p = ctx.scratch<float>("cg32_p", 2 * P * NC);
        F.Ap = ctx.scratch<float>("cg32_ap", P * NC);
        F.q = ctx.scratch<float>("cg32_q", p * NC);
        F.part = B.part;
        F.st = B.st;
        float* taps32 = ctx.scratch<float>("ps32_taps", static_cast<size_t>(S) * n * n);
        float* lpan32 = ctx.scratch<float>("ps32_lpan", P * S);
        float* xn32 = ctx.scratch<float>("ps32_xn", p * NC);
        to_f32(ctx, d_taps, static_cast<long long>(S) * n * n, taps32);
        to_f32(ctx, lpan, static_cast<long long>(P) * S, lpan32);
        to_f32(ctx, xn, static_cast<long long>(p) * NC, xn32);
        cg_solve_f32(ctx, G, taps32, lpan, lpan32, xn32, F, prm.cg_max_iter, prm.cg_tol, hs);
        to_f64(ctx, F.z, static_cast<long long>(P) * NC, B.z);
    } else {
        B.r = ctx.scratch<double>("cg_r", P * NC);
        B.p = ctx.scratch<double>("cg_p", 2 * P * NC);
        B.Ap = ctx.scratch<double>("cg_ap", P * NC);
        B.q = ctx.scratch<double>("cg_q", p * NC);
        cg_solve(ctx, G, d_taps, lpan, xn, B, prm.cg_max_iter, prm.cg_tol, hs);
    }
    cg_iters.assign(NC, 0);
    for (int i = 0; i < NC; ++i) cg_iters[i] = hs[i].iters;
    if (std::getenv("FBMP_CG_DEBUG"))  // final CG scalars per channel (debugging aid)
        for (int i = 0; i < NC; ++i)
            std::fprintf(stderr, "cg ch %d it %d pp %.17g alpha %.17g zz %.17g rs %.17g\n", i, hs[i].iters, hs[i].pp,
                         hs[i].alpha, hs[i].zz, hs[i].rs);
    for (int i = 0; i < NC; ++i) {  // first failing channel in index order (pansharpen.cpp:421-422)
        const std::string tag = "channel " + std::to_string(ch0 + i % NS) + ": ";
        if (hs[i].done == 2)
            num_error(tag + "warmstart: conjugate gradients hit a non-positive curvature direction");
        if (hs[i].done == 3) {
            // residual of the normal equations, only for the message (pansharpen.cpp:257-262)
            const int sc = i / NS;
            double* az = ctx.scratch<double>("cg_res_az", P);
            double* rhs = ctx.scratch<double>("cg_res_rhs", P);
            PsGeo G1 = make_geo(1, h, w, c, n, prm.radius, prm.lambda, prm.eps);
            G1.identity = G.identity;
            cg_operator_apply(ctx, G1, d_taps + static_cast<size_t>(sc) * n * n, lpan + sc * P, B.z + i * P, az, 0);
            data_rhs(ctx, G1, d_taps + static_cast<size_t>(sc) * n * n, xn + i * p, rhs);
            std::vector<double> a(P), b(P);
            d2h(a.data(), az, P * sizeof(double), ctx.stream);
            d2h(b.data(), rhs, P * sizeof(double), ctx.stream);
            FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
            double s2 = 0.0;
            for (size_t k = 0; k < P; ++k) s2 += (a[k] - b[k]) * (a[k] - b[k]);
            num_error(tag + "warmstart: conjugate gradients did not converge in " + std::to_string(prm.cg_max_iter) +
                      " iterations (residual " + std::to_string(std::sqrt(s2) / hs[i].rhs_norm) + " relative)");
        }
    }
    double* v = ctx.scratch<double>("ps_v", P * NC);
    // guided_coeffs(ch_prior.apply(z0), lpan) (pansharpen.cpp:396-398): L(z0), or z0 itself
    guided_filter(ctx, NC, H, W, prm.radius, prm.eps, B.z, G.identity ? 0 : 1, lpan, nullptr, nullptr, v, NS);
    int* flag = ctx.scratch<int>("ps_flag", NC);
    FBMP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int) * NC, ctx.stream));
    solve_channel_fft(ctx, G, d_taps, xn, v, scale, d_out, flag);
    trace("ps: guided + fft enqueue");
    std::vector<int> hf(NC);
    d2h(hf.data(), flag, sizeof(int) * NC, ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    trace("ps: guided + fft done");
    for (int i = 0; i < NC; ++i)
        if (hf[i])
            num_error("channel " + std::to_string(ch0 + i % NS) +
                      ": solve_channel_fft: alias-group system condition number exceeds 1e14 (prior transfer "
                      "function too small)");
}

namespace {
// dst[p][y][x] = src[p][(r0 + y) mod Hs][x] for y < Hd (row gather with periodic wrap)
__global__ void k_copy_rows(const double* __restrict__ src, int Hs, int W, double* __restrict__ dst, int r0, int Hd,
                            int planes) {
    const long long n = static_cast<long long>(Hd) * W;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n * planes;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long pl = e / n, rem = e - pl * n;
        const int y = static_cast<int>(rem / W), x = static_cast<int>(rem - static_cast<long long>(y) * W);
        int r = (r0 + y) % Hs;
        if (r < 0) r += Hs;
        dst[e] = src[(pl * Hs + r) * W + x];
    }
}
void copy_rows(Context& ctx, const double* src, int Hs, int W, double* dst, int r0, int Hd, int planes) {
    const long long n = static_cast<long long>(Hd) * W * planes;
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 16LL * ctx.sm_count));
    k_copy_rows<<<blocks, 256, 0, ctx.stream>>>(src, Hs, W, dst, r0, Hd, planes);
    ctx.count();
    check_launch();
}
}  // namespace

// HRMS solve of one scene with the CG on row strips: inputs are replicated
// on every rank; with a communicator, rank r owns rows [r H/G, (r+1) H/G); without one, `vstrips`
// virtual ranks run in this process (device copies instead of NCCL -- the same data flow, used by
// the tests on one GPU). The post-processing (guided filter + alias-group FFT solve) needs whole
// planes: the owned rows of z0 are all-gathered per channel and channel c is finished on rank
// c mod G; rank 0 then receives the other channels. d_out: N*H*W (complete on rank 0).
void pansharpen_strips_device(Context& ctx, const double* d_lrms, int N, int h, int w, const double* d_pan,
                              const double* d_taps, int n, int c, const fbmp_ps_params& prm, double* d_out,
                              std::vector<int>& cg_iters, int vstrips) {
    validate_ps(prm);
    if (ctx.precision != 64) param_error("pansharpen: the fp32 mode is not available for row strips");
    if (prm.prior != 0) param_error("pansharpen: row strips implement the Laplacian prior only");
    const int H = h * c, W = w * c;
    if (2 * prm.radius + 1 > std::min(H, W)) dim_error("matting matrix: window larger than image");
    check_kernel(n, H, W);
    const bool dist = ctx.nccl != nullptr;
    const int G = dist ? ctx.nranks : std::max(1, vstrips);
    StripComm comm;
    comm.nccl = ctx.nccl;
    comm.nranks = G;
    comm.rank = dist ? ctx.rank : 0;
    const int halo = comm.halo;
    if (H % G != 0 || (H / G) % std::max(c, 16) != 0 || H / G < halo)
        param_error("strip solve: the PAN height must split into equal strips of >= 32 rows (multiples of 16 and c)");
    const int hloc = H / G, Hp = hloc + 2 * halo;
    const size_t P = static_cast<size_t>(H) * W, p = static_cast<size_t>(h) * w, Pp = static_cast<size_t>(Hp) * W;
    // replicated setup: normalisation, L(pan_n), window statistics, scaled LRMS (whole image)
    double* scale = ctx.scratch<double>("st_scale", 1);
    double* lpan = ctx.scratch<double>("st_lpan", P);
    double* xn = ctx.scratch<double>("st_xn", p * N);
    peak_scale(ctx, d_pan, static_cast<long long>(P), d_lrms, static_cast<long long>(p) * N, 1, scale);
    laplacian_scaled(ctx, d_pan, H, W, 1, scale, lpan);
    scale_copy(ctx, d_lrms, static_cast<long long>(p) * N, scale, static_cast<long long>(p) * N, xn);
    const PsGeo Gf = make_geo(N, h, w, c, n, prm.radius, prm.lambda, prm.eps, N);
    double* wmu = ctx.scratch<double>("st_wmu", P);
    double* wg = ctx.scratch<double>("st_wg", P);
    guide_stats(ctx, Gf, lpan, wmu, wg);
    const int first = dist ? ctx.rank : 0, count = dist ? 1 : G;
    std::vector<StripCg> strips(count);
    const size_t nbmax = (Pp / 256 + 64) * 2 + 4096;
    for (int k = 0; k < count; ++k) {
        const int s = first + k;
        const int grow0 = s * hloc - halo;
        const std::string tag = "st" + std::to_string(k) + "_";
        StripCg& S = strips[k];
        double* gs = ctx.scratch<double>(tag + "guide", Pp);
        double* ms = ctx.scratch<double>(tag + "mu", Pp);
        double* ks = ctx.scratch<double>(tag + "g", Pp);
        double* xs = ctx.scratch<double>(tag + "x", static_cast<size_t>(Hp / c) * w * N);
        copy_rows(ctx, lpan, H, W, gs, grow0, Hp, 1);
        copy_rows(ctx, wmu, H, W, ms, grow0, Hp, 1);
        copy_rows(ctx, wg, H, W, ks, grow0, Hp, 1);
        copy_rows(ctx, xn, h, w, xs, grow0 / c, Hp / c, N);
        S.G = make_geo(N, Hp / c, w, c, n, prm.radius, prm.lambda, prm.eps, N);
        S.G.grow0 = grow0;
        S.G.Hg = H;
        S.G.rlo = halo;
        S.G.rhi = halo + hloc;
        S.dred = ctx.scratch<double>(tag + "red", 4 * static_cast<size_t>(N));
        S.G.dred = S.dred;
        S.taps = d_taps;
        S.guide = gs;
        S.wmu = ms;
        S.wg = ks;
        S.x = xs;
        S.B.z = ctx.scratch<double>(tag + "z", Pp * N);
        S.B.r = ctx.scratch<double>(tag + "r", Pp * N);
        S.B.p = ctx.scratch<double>(tag + "p", 2 * Pp * N);
        S.B.Ap = ctx.scratch<double>(tag + "ap", Pp * N);
        S.B.q = ctx.scratch<double>(tag + "q", static_cast<size_t>(Hp / c) * w * N);
        S.B.part = ctx.scratch<double>(tag + "part", 4 * nbmax * N);
        S.B.st = ctx.scratch<CgState>(tag + "state", N);
    }
    std::vector<CgState> hs;
    trace("strips: prologue");
    cg_solve_strips(ctx, strips, comm, prm.cg_max_iter, prm.cg_tol, hs);
    trace("strips: cg");
    cg_iters.assign(N, 0);
    for (int i = 0; i < N; ++i) cg_iters[i] = hs[i].iters;
    // every rank holds the same CG scalars (the dot products are allreduced), so every rank takes
    // the same branch here; a non-positive curvature fails before the z0 exchange
    for (int i = 0; i < N; ++i)
        if (hs[i].done == 2)
            num_error("channel " + std::to_string(i) +
                      ": warmstart: conjugate gradients hit a non-positive curvature direction");
    // whole z0 planes: owned rows of every strip, in strip order
    double* zf = ctx.scratch<double>("st_zfull", P * N);
    bool any_cap = false;
    for (int i = 0; i < N; ++i) any_cap = any_cap || hs[i].done == 3;  // identical on every rank
    if (dist) {
        // channel ch is post-processed on its owner rank ch mod G: the owned rows of z0 go to the
        // owner only (each rank receives N / G planes instead of N). The error path of a CG that
        // hit its cap needs z0 everywhere (the message's residual): then the planes are all-gathered.
        auto cm = static_cast<ncclComm_t>(ctx.nccl);
        const size_t rows = static_cast<size_t>(hloc) * W;
        const double* own = strips[0].B.z + static_cast<size_t>(halo) * W;
        for (int ch = ctx.rank; ch < N && !any_cap; ch += G)  // this rank's own rows of its channels
            FBMP_CUDA(cudaMemcpyAsync(zf + ch * P + static_cast<size_t>(ctx.rank) * rows, own + ch * Pp,
                                      rows * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
        FBMP_NCCL(ncclGroupStart());
        for (int ch = 0; ch < N; ++ch) {
            if (any_cap) {
                FBMP_NCCL(ncclAllGather(own + ch * Pp, zf + ch * P, rows, ncclDouble, cm, ctx.stream));
                continue;
            }
            const int owner = ch % G;
            if (ctx.rank == owner) {
                for (int r = 0; r < G; ++r)
                    if (r != owner) FBMP_NCCL(ncclRecv(zf + ch * P + r * rows, rows, ncclDouble, r, cm, ctx.stream));
            } else {
                FBMP_NCCL(ncclSend(own + ch * Pp, rows, ncclDouble, owner, cm, ctx.stream));
            }
        }
        FBMP_NCCL(ncclGroupEnd());
    } else {
        for (int k = 0; k < count; ++k)
            for (int ch = 0; ch < N; ++ch)
                FBMP_CUDA(cudaMemcpyAsync(zf + ch * P + static_cast<size_t>(k) * hloc * W,
                                          strips[k].B.z + ch * Pp + static_cast<size_t>(halo) * W,
                                          static_cast<size_t>(hloc) * W * sizeof(double), cudaMemcpyDeviceToDevice,
                                          ctx.stream));
    }
    // CG cap (pansharpen.cpp:257-262): the residual of the normal equations for the message,
    // formed on every rank from the gathered z0 with the single-domain operator, so every rank
    // raises the same error text as the single-domain path
    for (int i = 0; i < N; ++i)
        if (hs[i].done == 3) {
            double* az = ctx.scratch<double>("cg_res_az", P);
            double* rhs = ctx.scratch<double>("cg_res_rhs", P);
            const PsGeo G1 = make_geo(1, h, w, c, n, prm.radius, prm.lambda, prm.eps);
            cg_operator_apply(ctx, G1, d_taps, lpan, zf + i * P, az, 0);
            data_rhs(ctx, G1, d_taps, xn + i * p, rhs);
            std::vector<double> a(P), b(P);
            d2h(a.data(), az, P * sizeof(double), ctx.stream);
            d2h(b.data(), rhs, P * sizeof(double), ctx.stream);
            FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
            double s2 = 0.0;
            for (size_t k = 0; k < P; ++k) s2 += (a[k] - b[k]) * (a[k] - b[k]);
            num_error("channel " + std::to_string(i) + ": warmstart: conjugate gradients did not converge in " +
                      std::to_string(prm.cg_max_iter) + " iterations (residual " +
                      std::to_string(std::sqrt(s2) / hs[i].rhs_norm) + " relative)");
        }
    // post-processing: all channels here (virtual ranks), or the channels c with c mod G == rank
    double* v = ctx.scratch<double>("st_v", P * N);
    int* flag = ctx.scratch<int>("st_flag", N);
    FBMP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int) * N, ctx.stream));
    const PsGeo G1 = make_geo(1, h, w, c, n, prm.radius, prm.lambda, prm.eps, 1);
    if (!dist) {
        guided_filter(ctx, N, H, W, prm.radius, prm.eps, zf, 1, lpan, nullptr, nullptr, v, N);
        solve_channel_fft(ctx, Gf, d_taps, xn, v, scale, d_out, flag);
    } else {
        for (int ch = ctx.rank; ch < N; ch += G) {
            guided_filter(ctx, 1, H, W, prm.radius, prm.eps, zf + ch * P, 1, lpan, nullptr, nullptr, v + ch * P, 1);
            solve_channel_fft(ctx, G1, d_taps, xn + ch * p, v + ch * P, scale, d_out + ch * P, flag + ch);
        }
        auto cm = static_cast<ncclComm_t>(ctx.nccl);  // channels to rank 0
        FBMP_NCCL(ncclGroupStart());
        for (int ch = 0; ch < N; ++ch) {
            const int owner = ch % G;
            if (owner == 0) continue;
            if (ctx.rank == 0) FBMP_NCCL(ncclRecv(d_out + ch * P, P, ncclDouble, owner, cm, ctx.stream));
            if (ctx.rank == owner) FBMP_NCCL(ncclSend(d_out + ch * P, P, ncclDouble, 0, cm, ctx.stream));
        }
        // each channel's condition flag lives on its owner only: combine them so that every rank
        // raises the same "channel i: solve_channel_fft ..." error (or none)
        FBMP_NCCL(ncclAllReduce(flag, flag, N, ncclInt, ncclMax, cm, ctx.stream));
        FBMP_NCCL(ncclGroupEnd());
    }
    std::vector<int> hf(N);
    d2h(hf.data(), flag, sizeof(int) * N, ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    for (int i = 0; i < N; ++i)
        if (hf[i])
            num_error("channel " + std::to_string(i) +
                      ": solve_channel_fft: alias-group system condition number exceeds 1e14 (prior transfer "
                      "function too small)");
}

// SPEC.md:584-591 blind composition for S scenes on device-resident data:
// solve_weights (all bands) -> combine_bands -> estimate_kernel_tgv -> pansharpen.
void blind_device(Context& ctx, const double* d_lrms, int S, int N, int h, int w, const double* d_pan,
                  const fbmp_sw_params& sw, const fbmp_ke_params& ke, const fbmp_ps_params& ps, double* d_out,
                  double* d_k, double* d_omega_out, std::vector<int>& admm_iters, std::vector<int>& cg_iters,
                  int ch0 = 0, int nch = -1, int strips = 0) {
    const int c = sw.factor;
    if (c < 1) param_error("solve_weights: factor must be >= 1");
    if (sw.l < 1) param_error("solve_weights: l must be >= 1");
    if (sw.lambda_omega < 0.0) param_error("solve_weights: lambda_omega must be >= 0");
    validate_ke(ke);
    validate_ps(ps);
    const int H = h * c, W = w * c;
    const long long p = static_cast<long long>(h) * w;
    cudaEvent_t e0, e1, e2, e3;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
    cudaEventRecord(e0, ctx.stream);
    trace("blind: start");
    double* omega = d_omega_out ? d_omega_out : ctx.scratch<double>("bl_omega", static_cast<size_t>(S) * N);
    int* st = ctx.scratch<int>("bl_sw_status", S);
    solve_weights_device(ctx, d_lrms, S, N, h, w, d_pan, sw.l, sw.lambda_omega, c, omega, st);
    double* obs = ctx.scratch<double>("bl_obs", static_cast<size_t>(S) * p);
    combine_bands_device(ctx, d_lrms, S, N, p, omega, obs);
    std::vector<int> hst(S);
    d2h(hst.data(), st, S * sizeof(int), ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    for (int s = 0; s < S; ++s) {
        if (hst[s] == 1)
            num_error("solve_weights: normal matrix is singular (bands linearly dependent and lambda_omega too small)");
        if (hst[s] == 2) num_error("solve_weights: stationarity residual too large (ill-conditioned system)");
    }
    cudaEventRecord(e1, ctx.stream);
    // C5 row strips: the Gram tiles of the kernel fit are split over the ranks (chunk sums
    // all-gathered, bit-identical to one GPU); the rest of the fit is replicated
    const bool strip_path = strips > 0 || ctx.nccl;
    estimate_kernel_device(ctx, d_pan, obs, S, H, W, c, ke, d_k, admm_iters, nullptr, -1, false, strip_path);
    cudaEventRecord(e2, ctx.stream);
    trace("blind: weights + kernel fit");
    if (strip_path) {
        if (S != 1 || nch >= 0) param_error("strip solve: one scene, all bands");
        pansharpen_strips_device(ctx, d_lrms, N, h, w, d_pan, d_k, ke.n, c, ps, d_out, cg_iters, strips);
    } else {
        pansharpen_device(ctx, d_lrms, S, N, h, w, d_pan, d_k, ke.n, c, ps, d_out, cg_iters, ch0, nch);
    }
    cudaEventRecord(e3, ctx.stream);
    cudaEventSynchronize(e3);
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, e0, e1);
    cudaEventElapsedTime(&b, e1, e2);
    cudaEventElapsedTime(&d, e2, e3);
    ctx.stats.ms_weights = a;
    ctx.stats.ms_kernel_fit = b;
    ctx.stats.ms_pansharpen = d;
    ctx.stats.admm_iters = admm_iters.empty() ? 0 : admm_iters[0];
    for (int i = 0; i < 64; ++i) ctx.stats.cg_iters[i] = i < static_cast<int>(cg_iters.size()) ? cg_iters[i] : 0;
    ctx.stats.n_channels = static_cast<int>(cg_iters.size());
    ctx.cg_iters_all = cg_iters;
    ctx.stats.cg_channel_iters = 0;
    for (int it : cg_iters) ctx.stats.cg_channel_iters += it;
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2); cudaEventDestroy(e3);
}

}  // namespace fbmp_gpu

using namespace fbmp_gpu;

struct fbmp_gpu_ctx {
    Context impl;
    explicit fbmp_gpu_ctx(int dev) : impl(dev) {}
};

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return FBMP_OK;
    } catch (const Failure& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return FBMP_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FBMP_RUNTIME_ERROR;
    }
}

// Device copy of a host array in a context scratch slot.
static double* upload(Context& ctx, const std::string& slot, const double* src, size_t count) {
    double* d = ctx.scratch<double>(slot, count ? count : 1);
    if (count) h2d(d, src, count * sizeof(double), ctx.stream);
    return d;
}
static void download(Context& ctx, double* dst, const double* d, size_t count) {
    d2h(dst, d, count * sizeof(double), ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
}
static fbmp_ps_params ps_or_default(const fbmp_ps_params* p) {
    fbmp_ps_params d;
    fbmp_gpu_default_ps_params(&d);
    return p ? *p : d;
}
static fbmp_ke_params ke_or_default(const fbmp_ke_params* p) {
    fbmp_ke_params d;
    fbmp_gpu_default_ke_params(&d);
    return p ? *p : d;
}
static fbmp_sw_params sw_or_default(const fbmp_sw_params* p) {
    fbmp_sw_params d;
    fbmp_gpu_default_sw_params(&d);
    return p ? *p : d;
}

extern "C" {

void fbmp_gpu_default_ps_params(fbmp_ps_params* p) {
    p->lambda = 2e-4;
    p->radius = 1;
    p->eps = 1e-4;
    p->cg_tol = 5e-5;
    p->cg_max_iter = 2000;
    p->threads = 0;
    p->prior = 0;
}
void fbmp_gpu_default_ke_params(fbmp_ke_params* p) {
    p->n = 29;
    p->alpha1 = 1.0;
    p->alpha2 = 0.006;
    p->mu1 = p->mu2 = p->mu3 = 100.0;
    p->rho = 0.5;
    p->t_max = 10000;
    p->th = 1e-5;
    p->init = 0;
}
void fbmp_gpu_default_sw_params(fbmp_sw_params* p) {
    p->l = 4;
    p->lambda_omega = 10.0;
    p->factor = 2;
}

int fbmp_gpu_ctx_create(int device, fbmp_gpu_ctx** out) {
    return guarded([&] { *out = new fbmp_gpu_ctx(device); });
}
void fbmp_gpu_ctx_destroy(fbmp_gpu_ctx* ctx) { delete ctx; }
const char* fbmp_gpu_last_error(void) { return g_last_error.c_str(); }
int fbmp_gpu_ctx_cg_iters(fbmp_gpu_ctx* ctx, int* out, int cap) {
    if (!ctx || (cap > 0 && !out)) {
        g_last_error = "fbmp_gpu_ctx_cg_iters: null argument";
        return -1;
    }
    const auto& v = ctx->impl.cg_iters_all;
    for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) out[i] = v[i];
    return static_cast<int>(v.size());
}

int fbmp_gpu_ctx_stats(fbmp_gpu_ctx* ctx, fbmp_gpu_stats* out) {
    *out = ctx->impl.stats;
    return FBMP_OK;
}
void* fbmp_gpu_ctx_stream(fbmp_gpu_ctx* ctx) { return ctx->impl.stream; }
long long fbmp_gpu_ctx_launches(fbmp_gpu_ctx* ctx) { return ctx->impl.launches; }

int fbmp_gpu_pansharpen(fbmp_gpu_ctx* ctx, const double* lrms, int N, int h, int w, const double* pan,
                        const double* k, int n, int factor, const fbmp_ps_params* params, double* out,
                        int* cg_iters) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_ps_params prm = ps_or_default(params);
        validate_ps(prm);
        if (N < 1) dim_error("multi-band image needs at least one band");
        if (factor < 1) param_error("downsample: factor must be >= 1");
        const size_t p = static_cast<size_t>(h) * w, P = p * factor * factor;
        double* d_l = upload(C, "api_lrms", lrms, p * N);
        double* d_p = upload(C, "api_pan", pan, P);
        double* d_k = upload(C, "api_taps", k, static_cast<size_t>(n) * n);
        double* d_o = C.scratch<double>("api_out", P * N);
        std::vector<int> it;
        pansharpen_device(C, d_l, 1, N, h, w, d_p, d_k, n, factor, prm, d_o, it);
        download(C, out, d_o, P * N);
        for (int i = 0; i < 64; ++i) C.stats.cg_iters[i] = i < N ? it[i] : 0;
        C.stats.n_channels = N;
        C.cg_iters_all = it;
        if (cg_iters)
            for (int i = 0; i < N; ++i) cg_iters[i] = it[i];
    });
}

int fbmp_gpu_apply_prior(fbmp_gpu_ctx* ctx, const double* img, int H, int W, double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const size_t P = static_cast<size_t>(H) * W;
        double* d_i = upload(C, "u_in", img, P);
        double* d_o = C.scratch<double>("u_out", P);
        laplacian_scaled(C, d_i, H, W, 1, nullptr, d_o);
        download(C, out, d_o, P);
    });
}

int fbmp_gpu_llp_apply(fbmp_gpu_ctx* ctx, const double* guide, const double* x, int H, int W, int radius, double eps,
                       double* y) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (radius < 1) param_error("matting matrix: radius must be >= 1");
        if (2 * radius + 1 > std::min(H, W)) dim_error("matting matrix: window larger than image");
        const size_t P = static_cast<size_t>(H) * W;
        double* d_g = upload(C, "u_guide", guide, P);
        double* d_x = upload(C, "u_in", x, P);
        double* d_o = C.scratch<double>("u_out", P);
        double one = 1.0;
        double* d_k = upload(C, "u_taps", &one, 1);
        const PsGeo G = make_geo(1, H, W, 1, 1, radius, 1.0, eps);
        cg_operator_apply(C, G, d_k, d_g, d_x, d_o, 1);
        download(C, y, d_o, P);
    });
}

int fbmp_gpu_data_apply(fbmp_gpu_ctx* ctx, const double* p, int H, int W, const double* k, int n, int factor,
                        double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (factor < 1) param_error("downsample: factor must be >= 1");
        if (H % factor || W % factor) dim_error("downsample: dimensions not divisible by factor");
        check_kernel(n, H, W);
        const size_t P = static_cast<size_t>(H) * W;
        double* d_x = upload(C, "u_in", p, P);
        double* d_k = upload(C, "u_taps", k, static_cast<size_t>(n) * n);
        double* d_o = C.scratch<double>("u_out", P);
        const PsGeo G = make_geo(1, H / factor, W / factor, factor, n, 1, 1.0, 1.0);
        cg_operator_apply(C, G, d_k, nullptr, d_x, d_o, 2);
        download(C, out, d_o, P);
    });
}

int fbmp_gpu_cg_operator(fbmp_gpu_ctx* ctx, const double* guide, const double* p, int H, int W, const double* k,
                         int n, int factor, const fbmp_ps_params* params, double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_ps_params prm = ps_or_default(params);
        if (H % factor || W % factor) dim_error("downsample: dimensions not divisible by factor");
        check_kernel(n, H, W);
        const size_t P = static_cast<size_t>(H) * W;
        double* d_g = upload(C, "u_guide", guide, P);
        double* d_x = upload(C, "u_in", p, P);
        double* d_k = upload(C, "u_taps", k, static_cast<size_t>(n) * n);
        double* d_o = C.scratch<double>("u_out", P);
        validate_ps(prm);
        PsGeo G = make_geo(1, H / factor, W / factor, factor, n, prm.radius, prm.lambda, prm.eps);
        G.identity = prm.prior == 1;
        cg_operator_apply(C, G, d_k, d_g, d_x, d_o, 0);
        download(C, out, d_o, P);
    });
}

int fbmp_gpu_warmstart_cg(fbmp_gpu_ctx* ctx, const double* x, int h, int w, const double* guide, const double* k,
                          int n, int factor, const fbmp_ps_params* params, int max_iters, int error_on_cap,
                          double* z_out, int* iters, double* final_residual) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_ps_params prm = ps_or_default(params);
        const int H = h * factor, W = w * factor;
        check_kernel(n, H, W);
        if (2 * prm.radius + 1 > std::min(H, W)) dim_error("matting matrix: window larger than image");
        const size_t P = static_cast<size_t>(H) * W, p = static_cast<size_t>(h) * w;
        double* d_g = upload(C, "w_guide", guide, P);
        double* d_x = upload(C, "w_x", x, p);
        double* d_k = upload(C, "w_taps", k, static_cast<size_t>(n) * n);
        validate_ps(prm);
        PsGeo G = make_geo(1, h, w, factor, n, prm.radius, prm.lambda, prm.eps);
        G.identity = prm.prior == 1;
        CgBuffers B;
        B.z = C.scratch<double>("cg_z", P);
        B.r = C.scratch<double>("cg_r", P);
        B.p = C.scratch<double>("cg_p", 2 * P);
        B.Ap = C.scratch<double>("cg_ap", P);
        B.q = C.scratch<double>("cg_q", p);
        B.part = C.scratch<double>("cg_part", 4 * ((P / 256 + 64) * 2 + 4096));
        B.st = C.scratch<CgState>("cg_state", 1);
        std::vector<CgState> hs;
        cg_solve(C, G, d_k, d_g, d_x, B, max_iters, prm.cg_tol, hs);
        download(C, z_out, B.z, P);
        if (iters) *iters = hs[0].iters;
        const bool converged = hs[0].done == 1;
        double resid = 0.0;
        if (final_residual || (!converged && error_on_cap)) {
            double* az = C.scratch<double>("cg_res_az", P);
            double* rhs = C.scratch<double>("cg_res_rhs", P);
            cg_operator_apply(C, G, d_k, d_g, B.z, az, 0);
            data_rhs(C, G, d_k, d_x, rhs);
            std::vector<double> a(P), b(P);
            d2h(a.data(), az, P * sizeof(double), C.stream);
            d2h(b.data(), rhs, P * sizeof(double), C.stream);
            FBMP_CUDA(cudaStreamSynchronize(C.stream));
            double s = 0.0;
            for (size_t i = 0; i < P; ++i) s += (a[i] - b[i]) * (a[i] - b[i]);
            resid = std::sqrt(s);
            if (hs[0].rhs_norm == 0.0) resid = 0.0;
        }
        if (final_residual) *final_residual = resid;
        if (hs[0].done == 2) num_error("warmstart: conjugate gradients hit a non-positive curvature direction");
        if (!converged && error_on_cap)
            num_error("warmstart: conjugate gradients did not converge in " + std::to_string(max_iters) +
                      " iterations (residual " + std::to_string(resid / hs[0].rhs_norm) + " relative)");
    });
}

int fbmp_gpu_guided_filter(fbmp_gpu_ctx* ctx, const double* input, const double* guide, int H, int W, int radius,
                           double eps, double* a_out, double* c_out, double* v_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (!(eps > 0)) param_error("guided_coeffs: eps must be positive");
        if (radius < 0) param_error("box_mean: negative radius");
        if (2 * radius + 1 > std::min(H, W)) dim_error("box_mean: window larger than image");
        const size_t P = static_cast<size_t>(H) * W;
        double* d_i = upload(C, "g_in", input, P);
        double* d_g = upload(C, "g_guide", guide, P);
        double* d_a = a_out ? C.scratch<double>("g_a", P) : nullptr;  // coefficient maps only when asked
        double* d_c = c_out ? C.scratch<double>("g_c", P) : nullptr;
        double* d_v = C.scratch<double>("g_v", P);
        guided_filter(C, 1, H, W, radius, eps, d_i, 0, d_g, d_a, d_c, d_v, 1);
        if (a_out) download(C, a_out, d_a, P);
        if (c_out) download(C, c_out, d_c, P);
        if (v_out) download(C, v_out, d_v, P);
    });
}

int fbmp_gpu_guided_output(fbmp_gpu_ctx* ctx, const double* a, const double* c, const double* guide, int H, int W,
                           int radius, double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (radius < 0) param_error("box_mean: negative radius");
        if (2 * radius + 1 > std::min(H, W)) dim_error("box_mean: window larger than image");
        const size_t P = static_cast<size_t>(H) * W;
        double* d_a = upload(C, "g_a", a, P);
        double* d_c = upload(C, "g_c", c, P);
        double* d_g = upload(C, "g_guide", guide, P);
        double* d_ab = C.scratch<double>("g_ab", P);
        double* d_cb = C.scratch<double>("g_cb", P);
        double* d_o = C.scratch<double>("g_v", P);
        box_mean(C, d_a, H, W, 1, radius, d_ab);
        box_mean(C, d_c, H, W, 1, radius, d_cb);
        guided_combine(C, d_ab, d_cb, d_g, static_cast<long long>(P), d_o);  // pansharpen.cpp:306-311
        download(C, out, d_o, P);
    });
}

int fbmp_gpu_solve_channel_fft(fbmp_gpu_ctx* ctx, const double* x, int h, int w, const double* k, int n, int factor,
                               const double* v, const fbmp_ps_params* params, double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_ps_params prm = ps_or_default(params);
        validate_ps(prm);
        const int H = h * factor, W = w * factor;
        check_kernel(n, H, W);
        const size_t P = static_cast<size_t>(H) * W, p = static_cast<size_t>(h) * w;
        double* d_x = upload(C, "f_x", x, p);
        double* d_v = upload(C, "f_v", v, P);
        double* d_k = upload(C, "f_taps", k, static_cast<size_t>(n) * n);
        double* d_o = C.scratch<double>("f_out", P);
        int* flag = C.scratch<int>("f_flag", 1);
        FBMP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), C.stream));
        validate_ps(prm);
        PsGeo G = make_geo(1, h, w, factor, n, prm.radius, prm.lambda, prm.eps);
        G.identity = prm.prior == 1;
        solve_channel_fft(C, G, d_k, d_x, d_v, nullptr, d_o, flag);
        int hf = 0;
        d2h(&hf, flag, sizeof(int), C.stream);
        download(C, out, d_o, P);
        if (hf)
            num_error("solve_channel_fft: alias-group system condition number exceeds 1e14 (prior transfer function "
                      "too small)");
    });
}

int fbmp_gpu_metrics(fbmp_gpu_ctx* ctx, const double* est, const double* ref, int N, int H, int W, int crop,
                     int factor, int which, double* psnr_per_band, double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (N < 1 || H < 1 || W < 1) dim_error("metrics: image shapes differ");
        const size_t n = static_cast<size_t>(N) * H * W;
        double* d_e = upload(C, "met_est", est, n);
        double* d_r = upload(C, "met_ref", ref, n);
        std::vector<double> pb(N);
        metrics_device(C, d_e, d_r, N, H, W, crop, factor, which, pb.data(), out);
        if (psnr_per_band) std::memcpy(psnr_per_band, pb.data(), sizeof(double) * N);
    });
}

int fbmp_gpu_box_mean(fbmp_gpu_ctx* ctx, const double* img, int H, int W, int radius, double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (radius < 0) param_error("box_mean: negative radius");
        if (2 * radius + 1 > std::min(H, W)) dim_error("box_mean: window larger than image");
        const size_t P = static_cast<size_t>(H) * W;
        double* d_i = upload(C, "u_in", img, P);
        double* d_o = C.scratch<double>("u_out", P);
        box_mean(C, d_i, H, W, 1, radius, d_o);
        download(C, out, d_o, P);
    });
}

int fbmp_gpu_convolve(fbmp_gpu_ctx* ctx, const double* img, int H, int W, const double* k, int n, int adjoint,
                      double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (H < 1 || W < 1) dim_error("circular_convolve: empty image");
        check_kernel(n, H, W);
        const size_t P = static_cast<size_t>(H) * W;
        double* d_i = upload(C, "u_in", img, P);
        double* d_k = upload(C, "u_taps", k, static_cast<size_t>(n) * n);
        double* d_o = C.scratch<double>("u_out", P);
        convolve(C, d_i, H, W, d_k, n, adjoint, d_o);
        download(C, out, d_o, P);
    });
}


int fbmp_gpu_solve_weights(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w, const double* pan,
                           const fbmp_sw_params* cfg, double* omega_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_sw_params sw = sw_or_default(cfg);
        const int c = sw.factor;
        if (c < 1) param_error("solve_weights: factor must be >= 1");
        if (sw.l < 1) param_error("solve_weights: l must be >= 1");
        if (sw.lambda_omega < 0.0) param_error("solve_weights: lambda_omega must be >= 0");
        if (nb < 1) dim_error("multi-band image needs at least one band");
        const size_t p = static_cast<size_t>(h) * w, P = p * c * c;
        const int H = h * c, W = w * c;
        if (sw.l + 1 > std::min(h, w) || c * sw.l + 1 > std::min(H, W))  // ops.cpp:132-133
            dim_error("circular_box_blur: window larger than image");
        double* d_l = upload(C, "api_lrms", lrms_subset, p * nb);
        double* d_p = upload(C, "api_pan", pan, P);
        double* d_o = C.scratch<double>("api_omega", nb);
        int* st = C.scratch<int>("api_status", 1);
        solve_weights_device(C, d_l, 1, nb, h, w, d_p, sw.l, sw.lambda_omega, c, d_o, st);
        int hs = 0;
        d2h(&hs, st, sizeof(int), C.stream);
        download(C, omega_out, d_o, nb);
        if (hs == 1)
            num_error("solve_weights: normal matrix is singular (bands linearly dependent and lambda_omega too small)");
        if (hs == 2) num_error("solve_weights: stationarity residual too large (ill-conditioned system)");
    });
}

int fbmp_gpu_combine_bands(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w, const double* omega,
                           double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const size_t p = static_cast<size_t>(h) * w;
        double* d_l = upload(C, "api_lrms", lrms_subset, p * nb);
        double* d_w = upload(C, "api_omega", omega, nb);
        double* d_o = C.scratch<double>("api_obs", p);
        combine_bands_device(C, d_l, 1, nb, static_cast<long long>(p), d_w, d_o);
        download(C, out, d_o, p);
    });
}

static void estimate_plane_host(Context& C, const double* pan, int H, int W, const double* obs, int factor,
                                const fbmp_ke_params& prm, double* k_out, int* iters, double* state_out, int hook_t,
                                bool tv = false) {
    validate_ke(prm);
    if (factor < 1) param_error("build_observation: factor must be >= 1");
    if (H % factor || W % factor) dim_error("build_observation: PAN dimensions must be factor times the observation");
    const size_t P = static_cast<size_t>(H) * W, p = P / (static_cast<size_t>(factor) * factor);
    const int n = prm.n, m = n * n;
    double* d_p = upload(C, "api_pan", pan, P);
    double* d_f = upload(C, "api_obs", obs, p);
    double* d_k = C.scratch<double>("api_k", m);
    double* d_s = state_out ? C.scratch<double>("api_state", static_cast<size_t>(17) * m) : nullptr;
    std::vector<int> it;
    estimate_kernel_device(C, d_p, d_f, 1, H, W, factor, prm, d_k, it, d_s, hook_t, tv);
    download(C, k_out, d_k, m);
    if (d_s) download(C, state_out, d_s, static_cast<size_t>(17) * m);
    if (iters) *iters = it[0];
    C.stats.admm_iters = it[0];
}

int fbmp_gpu_estimate_kernel_plane(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs, int factor,
                                   const fbmp_ke_params* params, double* k_out, int* iters, double* state_out,
                                   int hook_t) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        estimate_plane_host(C, pan, H, W, obs, factor, ke_or_default(params), k_out, iters, state_out, hook_t);
    });
}

int fbmp_gpu_estimate_kernel_tv_plane(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs,
                                      int factor, const fbmp_ke_params* params, double* k_out, int* iters,
                                      double* state_out, int hook_t) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        estimate_plane_host(C, pan, H, W, obs, factor, ke_or_default(params), k_out, iters, state_out, hook_t, true);
    });
}

int fbmp_gpu_estimate_kernel_tv(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w, const double* pan,
                                const double* omega, int factor, const fbmp_ke_params* params, double* k_out,
                                int* iters) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const size_t p = static_cast<size_t>(h) * w;
        std::vector<double> obs(p);
        {
            double* d_l = upload(C, "api_lrms", lrms_subset, p * nb);
            double* d_w = upload(C, "api_omega", omega, nb);
            double* d_o = C.scratch<double>("api_obs2", p);
            combine_bands_device(C, d_l, 1, nb, static_cast<long long>(p), d_w, d_o);
            download(C, obs.data(), d_o, p);
        }
        estimate_plane_host(C, pan, h * factor, w * factor, obs.data(), factor, ke_or_default(params), k_out, iters,
                            nullptr, -1, true);
    });
}

int fbmp_gpu_estimate_kernel_l2_plane(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs,
                                      int factor, const fbmp_ke_params* params, double* k_out, int* iters) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_ke_params prm = ke_or_default(params);
        if (factor < 1) param_error("build_observation: factor must be >= 1");
        if (H % factor || W % factor) dim_error("build_observation: PAN dimensions must be factor times the observation");
        const size_t P = static_cast<size_t>(H) * W, p = P / (static_cast<size_t>(factor) * factor);
        const int m = prm.n * prm.n;
        double* d_p = upload(C, "api_pan", pan, P);
        double* d_f = upload(C, "api_obs", obs, p);
        double* d_k = C.scratch<double>("api_k", m);
        estimate_kernel_l2_device(C, d_p, d_f, H, W, factor, prm, d_k, iters);
        download(C, k_out, d_k, m);
    });
}

int fbmp_gpu_estimate_kernel_tgv(fbmp_gpu_ctx* ctx, const double* lrms_subset, int nb, int h, int w, const double* pan,
                                 const double* omega, int factor, const fbmp_ke_params* params, double* k_out,
                                 int* iters) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const size_t p = static_cast<size_t>(h) * w;
        std::vector<double> obs(p);
        {
            double* d_l = upload(C, "api_lrms", lrms_subset, p * nb);
            double* d_w = upload(C, "api_omega", omega, nb);
            double* d_o = C.scratch<double>("api_obs2", p);
            combine_bands_device(C, d_l, 1, nb, static_cast<long long>(p), d_w, d_o);
            download(C, obs.data(), d_o, p);
        }
        estimate_plane_host(C, pan, h * factor, w * factor, obs.data(), factor, ke_or_default(params), k_out, iters,
                            nullptr, -1);
    });
}

int fbmp_gpu_blind_dev(fbmp_gpu_ctx* ctx, const double* d_lrms, int N, int h, int w, const double* d_pan,
                       const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps, double* d_out,
                       double* d_k_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        std::vector<int> ai, ci;
        blind_device(C, d_lrms, 1, N, h, w, d_pan, sw_or_default(sw), ke_or_default(ke), ps_or_default(ps), d_out,
                     d_k_out, nullptr, ai, ci);
    });
}

int fbmp_gpu_blind_batch_dev(fbmp_gpu_ctx* ctx, const double* d_lrms, int S, int N, int h, int w,
                             const double* d_pan, const fbmp_sw_params* sw, const fbmp_ke_params* ke,
                             const fbmp_ps_params* ps, int ch0, int nch, double* d_out, double* d_k_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (S < 1) param_error("blind: scene count must be >= 1");
        if (nch >= 0 && (S != 1 || ch0 < 0 || nch < 1 || ch0 + nch > N)) param_error("blind: invalid channel subset");
        std::vector<int> ai, ci;
        blind_device(C, d_lrms, S, N, h, w, d_pan, sw_or_default(sw), ke_or_default(ke), ps_or_default(ps), d_out,
                     d_k_out, nullptr, ai, ci, nch >= 0 ? ch0 : 0, nch);
    });
}

int fbmp_gpu_nccl_unique_id(unsigned char* id128) {
    return guarded([&] {
        ncclUniqueId id;
        FBMP_NCCL(ncclGetUniqueId(&id));
        std::memcpy(id128, id.internal, sizeof(id.internal));
    });
}

int fbmp_gpu_ctx_set_comm(fbmp_gpu_ctx* ctx, const unsigned char* id128, int nranks, int rank) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (nranks < 1 || rank < 0 || rank >= nranks) param_error("set_comm: invalid rank / size");
        if (C.nccl) {
            ncclCommDestroy(static_cast<ncclComm_t>(C.nccl));
            C.nccl = nullptr;
        }
        ncclUniqueId id;
        std::memcpy(id.internal, id128, sizeof(id.internal));
        ncclComm_t comm;
        FBMP_NCCL(ncclCommInitRank(&comm, nranks, id, rank));
        C.nccl = comm;
        C.nranks = nranks;
        C.rank = rank;
    });
}

int fbmp_gpu_blind_strips_dev(fbmp_gpu_ctx* ctx, const double* d_lrms, int N, int h, int w, const double* d_pan,
                              const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps,
                              int vstrips, double* d_out, double* d_k_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        std::vector<int> ai, ci;
        blind_device(C, d_lrms, 1, N, h, w, d_pan, sw_or_default(sw), ke_or_default(ke), ps_or_default(ps), d_out,
                     d_k_out, nullptr, ai, ci, 0, -1, std::max(1, vstrips));
    });
}

int fbmp_gpu_blind(fbmp_gpu_ctx* ctx, const double* lrms, int N, int h, int w, const double* pan,
                   const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps, double* out,
                   double* k_out, double* omega_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_sw_params swp = sw_or_default(sw);
        const fbmp_ke_params kep = ke_or_default(ke);
        const int c = swp.factor;
        if (c < 1) param_error("solve_weights: factor must be >= 1");
        const size_t p = static_cast<size_t>(h) * w, P = p * c * c;
        double* d_l = upload(C, "api_lrms", lrms, p * N);
        double* d_p = upload(C, "api_pan", pan, P);
        double* d_o = C.scratch<double>("api_out", P * N);
        double* d_k = C.scratch<double>("api_k", static_cast<size_t>(kep.n) * kep.n);
        double* d_w = C.scratch<double>("api_omega", N);
        std::vector<int> ai, ci;
        // the HRMS planes stream to `out` per channel while the later channels finish
        // (single-domain solves only: the row-strip path gathers the channels on rank 0 first)
        struct Sink {
            Context& c;
            Sink(Context& cc, double* o) : c(cc) { c.host_out = c.nccl ? nullptr : o; }
            ~Sink() {  // no copy into the caller's buffer outlives the call, also on the error path
                c.host_out = nullptr;
                if (c.copy_stream) cudaStreamSynchronize(c.copy_stream);
            }
        } sink(C, out);
        const bool sunk = C.host_out != nullptr;
        blind_device(C, d_l, 1, N, h, w, d_p, swp, kep, ps_or_default(ps), d_o, d_k, d_w, ai, ci);
        FBMP_CUDA(cudaStreamSynchronize(C.stream));
        if (C.copy_stream) FBMP_CUDA(cudaStreamSynchronize(C.copy_stream));
        if (!sunk) download(C, out, d_o, P * N);
        if (k_out) download(C, k_out, d_k, static_cast<size_t>(kep.n) * kep.n);
        if (omega_out) download(C, omega_out, d_w, N);
    });
}

int fbmp_gpu_blind_batch(fbmp_gpu_ctx* ctx, const double* lrms, int S, int N, int h, int w, const double* pan,
                         const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps, double* out,
                         double* k_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_sw_params swp = sw_or_default(sw);
        const fbmp_ke_params kep = ke_or_default(ke);
        const int c = swp.factor;
        if (c < 1) param_error("solve_weights: factor must be >= 1");
        const size_t p = static_cast<size_t>(h) * w, P = p * c * c;
        double* d_l = upload(C, "api_lrms", lrms, p * N * S);
        double* d_p = upload(C, "api_pan", pan, P * S);
        double* d_o = C.scratch<double>("api_out", P * N * S);
        double* d_k = C.scratch<double>("api_k", static_cast<size_t>(kep.n) * kep.n * S);
        std::vector<int> ai, ci;
        blind_device(C, d_l, S, N, h, w, d_p, swp, kep, ps_or_default(ps), d_o, d_k, nullptr, ai, ci);
        download(C, out, d_o, P * N * S);
        if (k_out) download(C, k_out, d_k, static_cast<size_t>(kep.n) * kep.n * S);
    });
}

int fbmp_gpu_shrink2(fbmp_gpu_ctx* ctx, double* cols, int ncols, long long m, double t) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (t < 0) param_error("shrink2: threshold must be non-negative");
        if (ncols < 1 || m < 1) return;
        double* d = upload(C, "u_cols", cols, static_cast<size_t>(ncols) * m);
        shrink2_device(C, d, ncols, m, t);
        download(C, cols, d, static_cast<size_t>(ncols) * m);
    });
}

int fbmp_gpu_project_simplex(fbmp_gpu_ctx* ctx, const double* v, int m, double* out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        double* d_v = upload(C, "u_in", v, m);
        double* d_o = C.scratch<double>("u_out", m);
        int* st = C.scratch<int>("u_status", 1);
        project_simplex_device(C, d_v, m, d_o, st);
        int hs = 0;
        d2h(&hs, st, sizeof(int), C.stream);
        download(C, out, d_o, m);
        if (hs) num_error("project_simplex: empty support (non-finite input?)");
    });
}

int fbmp_gpu_solve_up(fbmp_gpu_ctx* ctx, const double* fields, int n, const fbmp_ke_params* params, double coupling,
                      const double* anchor, double* u, double* p1, double* p2) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_ke_params prm = ke_or_default(params);
        const size_t m = static_cast<size_t>(n) * n;
        double* d_f = upload(C, "u_fields", fields, 12 * m);
        double* d_a = anchor ? upload(C, "u_anchor", anchor, m) : nullptr;
        double* d_u = C.scratch<double>("u_u", m);
        double* d_p1 = C.scratch<double>("u_p1", m);
        double* d_p2 = C.scratch<double>("u_p2", m);
        solve_up_device(C, d_f, n, prm, coupling, d_a, d_u, d_p1, d_p2);
        download(C, u, d_u, m);
        download(C, p1, d_p1, m);
        download(C, p2, d_p2, m);
    });
}

int fbmp_gpu_gram(fbmp_gpu_ctx* ctx, const double* pan, int H, int W, const double* obs, int factor, int n,
                  double* EtE, double* Etf) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (n < 1 || n % 2 == 0) param_error("build_observation: kernel side must be odd");
        if (factor < 1) param_error("build_observation: factor must be >= 1");
        if (H % factor || W % factor) dim_error("build_observation: PAN dimensions must be factor times the observation");
        if (n > std::min(H, W)) dim_error("build_observation: kernel larger than PAN image");
        const size_t P = static_cast<size_t>(H) * W, p = P / (static_cast<size_t>(factor) * factor);
        const size_t n2 = static_cast<size_t>(n) * n;
        double* d_p = upload(C, "api_pan", pan, P);
        double* d_f = upload(C, "api_obs", obs, p);
        double* d_G = C.scratch<double>("api_EtE", n2 * n2);
        double* d_e = C.scratch<double>("api_Etf", n2);
        gram_device(C, d_p, d_f, H, W, factor, n, d_G, d_e);
        download(C, EtE, d_G, n2 * n2);
        download(C, Etf, d_e, n2);
    });
}

int fbmp_gpu_solve_z(fbmp_gpu_ctx* ctx, const double* EtE, const double* Etf, int n, double mu3,
                     const double* anchor, double* z_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        if (n < 1) param_error("build_observation: kernel side must be odd");
        const size_t n2 = static_cast<size_t>(n) * n;
        double* d_G = upload(C, "sz_EtE", EtE, n2 * n2);
        double* d_e = upload(C, "sz_Etf", Etf, n2);
        double* d_a = upload(C, "sz_anchor", anchor, n2);
        double* d_z = C.scratch<double>("sz_z", n2);
        solve_z_device(C, d_G, d_e, static_cast<int>(n2), mu3, d_a, d_z);
        download(C, z_out, d_z, n2);
    });
}

int fbmp_gpu_data_objective(fbmp_gpu_ctx* ctx, const double* EtE, const double* Etf, int n, double ff,
                            const double* u, double* value) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const size_t n2 = static_cast<size_t>(n) * n;
        double* d_G = upload(C, "sz_EtE", EtE, n2 * n2);
        double* d_e = upload(C, "sz_Etf", Etf, n2);
        double* d_u = upload(C, "sz_u", u, n2);
        double* d_v = C.scratch<double>("sz_v", 1);
        data_objective_device(C, d_G, d_e, d_u, static_cast<int>(n2), ff, d_v);
        download(C, value, d_v, 1);
    });
}

int fbmp_gpu_ctx_set_precision(fbmp_gpu_ctx* ctx, int bits) {
    return guarded([&] {
        if (bits != 32 && bits != 64) param_error("precision must be 32 or 64 bits");
        ctx->impl.precision = bits;
    });
}

int fbmp_gpu_ctx_precision(fbmp_gpu_ctx* ctx) { return ctx->impl.precision; }

void fbmp_gpu_ctx_set_profile(fbmp_gpu_ctx* ctx, int on) {
    ctx->impl.profile = on != 0;
    for (int i = 0; i < 4; ++i) {
        ctx->impl.prof_ms[i] = 0.0;
        ctx->impl.prof_n[i] = 0;
    }
}

int fbmp_gpu_ctx_kernel_profile(fbmp_gpu_ctx* ctx, double* total_ms, long long* launches) {
    for (int i = 0; i < 4; ++i) {
        total_ms[i] = ctx->impl.prof_ms[i];
        launches[i] = ctx->impl.prof_n[i];
    }
    return FBMP_OK;
}

int fbmp_gpu_blind_subset(fbmp_gpu_ctx* ctx, const double* lrms, int N, int h, int w, const double* pan,
                          const fbmp_sw_params* sw, const fbmp_ke_params* ke, const fbmp_ps_params* ps, int ch0,
                          int nch, double* out, double* k_out) {
    return guarded([&] {
        Context& C = ctx->impl;
        DeviceGuard dg(C.device);
        const fbmp_sw_params swp = sw_or_default(sw);
        const fbmp_ke_params kep = ke_or_default(ke);
        const int c = swp.factor;
        if (c < 1) param_error("solve_weights: factor must be >= 1");
        if (ch0 < 0 || nch < 1 || ch0 + nch > N) param_error("blind: invalid channel subset");
        const size_t p = static_cast<size_t>(h) * w, P = p * c * c;
        double* d_l = upload(C, "api_lrms", lrms, p * N);
        double* d_p = upload(C, "api_pan", pan, P);
        double* d_o = C.scratch<double>("api_out", P * nch);
        double* d_k = C.scratch<double>("api_k", static_cast<size_t>(kep.n) * kep.n);
        std::vector<int> ai, ci;
        blind_device(C, d_l, 1, N, h, w, d_p, swp, kep, ps_or_default(ps), d_o, d_k, nullptr, ai, ci, ch0, nch);
        download(C, out, d_o, P * nch);
        if (k_out) download(C, k_out, d_k, static_cast<size_t>(kep.n) * kep.n);
    });
}

}  // extern "C"
