// fbmp_api.cpp -- the reference's fbmp:: C++ API (include/fbmp/*.hpp) implemented on the
// B200 C ABI (include/fbmp_gpu.h). Every hot-path entry point (pansharpen, the warm-start CG,
// the matting operator, the guided filter, the alias-group solve, the spectral weights and the
// TGV kernel fit) runs on the GPU; this file only converts types, keeps one device context per
// host thread and rethrows the C ABI status codes as the reference's exception types.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <string>

#include "fbmp/errors.hpp"
#include "fbmp/image.hpp"
#include "fbmp/kernel_estimator.hpp"
#include "fbmp/metrics.hpp"
#include "fbmp/ops.hpp"
#include "fbmp/pansharpen.hpp"
#include "fbmp/spectral_weights.hpp"
#include "fbmp_gpu.h"

namespace fbmp {
namespace {

void check(int status) {
    if (status == FBMP_OK) return;
    const std::string msg = fbmp_gpu_last_error();
    switch (status) {
    case FBMP_PARAM_ERROR: throw ParamError(msg);
    case FBMP_DIMENSION_ERROR: throw DimensionError(msg);
    case FBMP_NUMERICAL_ERROR: throw NumericalError(msg);
    default: throw DeviceError(msg);
    }
}

struct CtxDeleter {
    void operator()(fbmp_gpu_ctx* c) const { fbmp_gpu_ctx_destroy(c); }
};

fbmp_gpu_ctx* ctx() {
    thread_local std::unique_ptr<fbmp_gpu_ctx, CtxDeleter> c;
    if (!c) {
        const char* dev = std::getenv("FBMP_DEVICE");
        fbmp_gpu_ctx* raw = nullptr;
        check(fbmp_gpu_ctx_create(dev ? std::atoi(dev) : 0, &raw));
        c.reset(raw);
    }
    return c.get();
}

fbmp_ps_params to_c(const PansharpenParams& p) {
    return fbmp_ps_params{p.lambda, p.radius, p.eps, p.cg_tol, p.cg_max_iter, p.threads,
                          p.prior == PriorKind::identity ? 1 : (p.prior == PriorKind::custom ? 2 : 0)};
}
fbmp_ke_params to_c(const KernelEstParams& p) {
    return fbmp_ke_params{p.n, p.alpha1, p.alpha2, p.mu1, p.mu2, p.mu3, p.rho, p.t_max, p.th,
                          p.init == KernelInit::dirac ? 0 : 1};
}

std::vector<double> stack(const MultiBandImage& img) {
    std::vector<double> v;
    v.reserve(static_cast<std::size_t>(img.band_count()) * img.height() * img.width());
    for (const Plane& b : img.bands()) v.insert(v.end(), b.data(), b.data() + b.size());
    return v;
}

void require_laplacian(const PansharpenParams& p) {  // the device path: Laplacian and identity priors
    if (p.prior == PriorKind::custom)
        throw ParamError("pansharpen: the GPU path implements the Laplacian and identity priors (no custom prior)");
}

Plane sq(const Plane& a) {
    Plane o = a;
    for (double& v : o.samples()) v *= v;
    return o;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// ops.hpp
// ---------------------------------------------------------------------------------------------
Plane circular_convolve(const Plane& img, const Kernel2D& k) {
    if (img.empty()) throw DimensionError("circular_convolve: empty image");
    Plane out(img.height(), img.width());
    check(fbmp_gpu_convolve(ctx(), img.data(), img.height(), img.width(), k.taps().data(), k.size(), 0, out.data()));
    return out;
}

Plane circular_convolve_adjoint(const Plane& img, const Kernel2D& k) {
    if (img.empty()) throw DimensionError("circular_convolve_adjoint: empty image");
    Plane out(img.height(), img.width());
    check(fbmp_gpu_convolve(ctx(), img.data(), img.height(), img.width(), k.taps().data(), k.size(), 1, out.data()));
    return out;
}

Plane embed_kernel(const Kernel2D& k, int height, int width) {
    if (k.size() > height || k.size() > width) throw DimensionError("kernel larger than image");
    Plane out(height, width);
    const int c = k.center();
    for (int r = 0; r < k.size(); ++r)
        for (int q = 0; q < k.size(); ++q) out(((r - c) % height + height) % height, ((q - c) % width + width) % width) += k(r, q);
    return out;
}

Plane downsample(const Plane& img, int factor) {
    if (factor < 1) throw ParamError("downsample: factor must be >= 1");
    if (img.height() % factor || img.width() % factor) throw DimensionError("downsample: dimensions not divisible by factor");
    Plane out(img.height() / factor, img.width() / factor);
    for (int r = 0; r < out.height(); ++r)
        for (int c = 0; c < out.width(); ++c) out(r, c) = img(r * factor, c * factor);
    return out;
}

Plane upsample_adjoint(const Plane& img, int factor) {
    if (factor < 1) throw ParamError("upsample_adjoint: factor must be >= 1");
    Plane out(img.height() * factor, img.width() * factor);
    for (int r = 0; r < img.height(); ++r)
        for (int c = 0; c < img.width(); ++c) out(r * factor, c * factor) = img(r, c);
    return out;
}

Plane diff_operator(const Plane& img, DiffOp which) {
    if (which == DiffOp::laplacian) {
        Plane out(img.height(), img.width());
        check(fbmp_gpu_apply_prior(ctx(), img.data(), img.height(), img.width(), out.data()));
        return out;
    }
    Plane out(img.height(), img.width());
    for (int r = 0; r < img.height(); ++r)
        for (int c = 0; c < img.width(); ++c)
            out(r, c) = (which == DiffOp::grad_h ? img.at_wrap(r, c + 1) : img.at_wrap(r + 1, c)) - img(r, c);
    return out;
}

Plane diff_adjoint(const Plane& img, DiffOp which) {
    if (which == DiffOp::laplacian) return diff_operator(img, which);  // symmetric stencil
    Plane out(img.height(), img.width());
    for (int r = 0; r < img.height(); ++r)
        for (int c = 0; c < img.width(); ++c)
            out(r, c) = (which == DiffOp::grad_h ? img.at_wrap(r, c - 1) : img.at_wrap(r - 1, c)) - img(r, c);
    return out;
}

Plane box_mean(const Plane& img, int radius) {
    Plane out(img.height(), img.width());
    check(fbmp_gpu_box_mean(ctx(), img.data(), img.height(), img.width(), radius, out.data()));
    return out;
}

Plane circular_box_blur(const Plane& img, int window) {
    if (window < 1) throw ParamError("circular_box_blur: window must be >= 1");
    if (window > std::min(img.height(), img.width())) throw DimensionError("circular_box_blur: window larger than image");
    const int lead = (window - 1) / 2;
    Plane rows(img.height(), img.width()), out(img.height(), img.width());
    for (int r = 0; r < img.height(); ++r)
        for (int c = 0; c < img.width(); ++c) {
            double s = 0.0;
            for (int t = -lead; t < window - lead; ++t) s += img.at_wrap(r, c - t);
            rows(r, c) = s * (1.0 / window);
        }
    for (int r = 0; r < img.height(); ++r)
        for (int c = 0; c < img.width(); ++c) {
            double s = 0.0;
            for (int t = -lead; t < window - lead; ++t) s += rows.at_wrap(r - t, c);
            out(r, c) = s * (1.0 / window);
        }
    return out;
}

// ---------------------------------------------------------------------------------------------
// pansharpen.hpp
// ---------------------------------------------------------------------------------------------
void PansharpenParams::validate() const {
    fbmp_ps_params p = to_c(*this);
    if (!(p.lambda > 0)) throw ParamError("pansharpen: lambda must be positive");
    if (radius < 1) throw ParamError("pansharpen: radius must be >= 1");
    if (!(eps > 0)) throw ParamError("pansharpen: eps must be positive");
    if (!(cg_tol > 0)) throw ParamError("pansharpen: cg_tol must be positive");
    if (cg_max_iter < 1) throw ParamError("pansharpen: cg_max_iter must be >= 1");
    if (threads < 0) throw ParamError("pansharpen: threads must be >= 0");
    if (prior == PriorKind::custom && prior_kernel.size() == 0)
        throw ParamError("pansharpen: custom prior requires a kernel");
}

Plane apply_prior(const Plane& img, const PansharpenParams& params) {
    if (params.prior == PriorKind::identity) return img;
    require_laplacian(params);
    return diff_operator(img, DiffOp::laplacian);
}

Plane apply_prior_adjoint(const Plane& img, const PansharpenParams& params) { return apply_prior(img, params); }

MattingMatrix MattingMatrix::build(const Plane& guide, int radius, double eps) {
    if (radius < 1) throw ParamError("matting matrix: radius must be >= 1");
    if (2 * radius + 1 > std::min(guide.height(), guide.width()))
        throw DimensionError("matting matrix: window larger than image");
    MattingMatrix M;
    M.guide_ = guide;
    M.radius_ = radius;
    M.eps_ = eps;
    M.mean_ = box_mean(guide, radius);
    M.var_ = box_mean(sq(guide), radius);
    for (std::size_t i = 0; i < M.var_.size(); ++i) M.var_.data()[i] -= M.mean_.data()[i] * M.mean_.data()[i];
    return M;
}

MattingMatrix build_matting_matrix(const Plane& guide, int radius, double eps) {
    return MattingMatrix::build(guide, radius, eps);
}

Plane MattingMatrix::apply(const Plane& p) const {
    if (p.height() != height() || p.width() != width()) throw DimensionError("matting matrix: plane shape mismatch");
    Plane y(height(), width());
    check(fbmp_gpu_llp_apply(ctx(), guide_.data(), p.data(), height(), width(), radius_, eps_, y.data()));
    return y;
}

Plane warmstart_cg(const Plane& x_i, const Kernel2D& k, int factor, const MattingMatrix& M,
                   const PansharpenParams& params, int max_iters, bool error_on_cap, double* final_residual) {
    require_laplacian(params);
    if (x_i.height() * factor != M.height() || x_i.width() * factor != M.width())
        throw DimensionError("warmstart: LR channel dimensions must be image/factor");
    fbmp_ps_params p = to_c(params);
    p.radius = M.radius();
    p.eps = M.eps();
    Plane z(M.height(), M.width());
    int iters = 0;
    check(fbmp_gpu_warmstart_cg(ctx(), x_i.data(), x_i.height(), x_i.width(), M.guide().data(), k.taps().data(),
                                k.size(), factor, &p, max_iters, error_on_cap ? 1 : 0, z.data(), &iters,
                                final_residual));
    return z;
}

Plane warmstart_channel(const Plane& x_i, const Plane& pan, const Kernel2D& k, int factor, const MattingMatrix& M,
                        const PansharpenParams& params) {
    params.validate();
    if (pan.height() != M.height() || pan.width() != M.width())
        throw DimensionError("warmstart: matting matrix was not built on the PAN grid");
    return warmstart_cg(x_i, k, factor, M, params, params.cg_max_iter, true);
}

AffineCoeffMaps guided_coeffs(const Plane& input, const Plane& guide, int radius, double eps) {
    if (!input.same_shape(guide)) throw DimensionError("guided_coeffs: shape mismatch");
    if (!(eps > 0)) throw ParamError("guided_coeffs: eps must be positive");
    AffineCoeffMaps m;
    m.a = Plane(input.height(), input.width());
    m.c = Plane(input.height(), input.width());
    check(fbmp_gpu_guided_filter(ctx(), input.data(), guide.data(), input.height(), input.width(), radius, eps,
                                 m.a.data(), m.c.data(), nullptr));
    m.guide_mean = box_mean(guide, radius);
    m.input_mean = box_mean(input, radius);
    m.guide_var = box_mean(sq(guide), radius);
    for (std::size_t i = 0; i < m.guide_var.size(); ++i)
        m.guide_var.data()[i] -= m.guide_mean.data()[i] * m.guide_mean.data()[i];
    return m;
}

Plane guided_output(const AffineCoeffMaps& coeffs, const Plane& guide, int radius) {
    if (!coeffs.a.same_shape(guide)) throw DimensionError("guided_output: shape mismatch");
    Plane out(guide.height(), guide.width());
    check(fbmp_gpu_guided_output(ctx(), coeffs.a.data(), coeffs.c.data(), guide.data(), guide.height(), guide.width(),
                                 radius, out.data()));
    return out;
}

Plane solve_channel_fft(const Plane& x_i, const Kernel2D& k, int factor, const Plane& v,
                        const PansharpenParams& params) {
    params.validate();
    require_laplacian(params);
    if (x_i.height() * factor != v.height() || x_i.width() * factor != v.width())
        throw DimensionError("solve_channel_fft: LR/HR dimensions inconsistent with factor");
    const fbmp_ps_params p = to_c(params);
    Plane z(v.height(), v.width());
    check(fbmp_gpu_solve_channel_fft(ctx(), x_i.data(), x_i.height(), x_i.width(), k.taps().data(), k.size(), factor,
                                     v.data(), &p, z.data()));
    return z;
}

MultiBandImage pansharpen(const MultiBandImage& lrms, const Plane& pan, const Kernel2D& k, int factor,
                          const PansharpenParams& params) {
    params.validate();
    require_laplacian(params);
    if (pan.height() != factor * lrms.height() || pan.width() != factor * lrms.width())
        throw DimensionError("pansharpen: PAN dimensions must be factor times the LRMS dimensions");
    const fbmp_ps_params p = to_c(params);
    const int N = lrms.band_count();
    std::vector<double> in = stack(lrms), out(static_cast<std::size_t>(N) * pan.size());
    check(fbmp_gpu_pansharpen(ctx(), in.data(), N, lrms.height(), lrms.width(), pan.data(), k.taps().data(), k.size(),
                              factor, &p, out.data(), nullptr));
    std::vector<Plane> bands;
    for (int b = 0; b < N; ++b)
        bands.emplace_back(pan.height(), pan.width(),
                           std::vector<double>(out.begin() + static_cast<std::ptrdiff_t>(b * pan.size()),
                                               out.begin() + static_cast<std::ptrdiff_t>((b + 1) * pan.size())));
    return MultiBandImage(std::move(bands));
}

// ---------------------------------------------------------------------------------------------
// spectral_weights.hpp
// ---------------------------------------------------------------------------------------------
SpectralWeights solve_weights(const MultiBandImage& lrms_subset, const Plane& pan, const SpectralWeightConfig& cfg) {
    if (cfg.factor < 1) throw ParamError("solve_weights: factor must be >= 1");
    if (cfg.l < 1) throw ParamError("solve_weights: l must be >= 1");
    if (cfg.lambda_omega < 0.0) throw ParamError("solve_weights: lambda_omega must be >= 0");
    if (pan.height() != cfg.factor * lrms_subset.height() || pan.width() != cfg.factor * lrms_subset.width())
        throw DimensionError("solve_weights: PAN dimensions must be factor times the LRMS dimensions");
    const fbmp_sw_params p{cfg.l, cfg.lambda_omega, cfg.factor};
    std::vector<double> in = stack(lrms_subset);
    SpectralWeights w;
    w.omega.resize(lrms_subset.band_count());
    check(fbmp_gpu_solve_weights(ctx(), in.data(), lrms_subset.band_count(), lrms_subset.height(),
                                 lrms_subset.width(), pan.data(), &p, w.omega.data()));
    return w;
}

Plane combine_bands(const MultiBandImage& lrms_subset, const SpectralWeights& w) {
    if (static_cast<int>(w.omega.size()) != lrms_subset.band_count())
        throw DimensionError("combine_bands: weight count does not match band count");
    std::vector<double> in = stack(lrms_subset);
    Plane out(lrms_subset.height(), lrms_subset.width());
    check(fbmp_gpu_combine_bands(ctx(), in.data(), lrms_subset.band_count(), lrms_subset.height(),
                                 lrms_subset.width(), w.omega.data(), out.data()));
    return out;
}

// ---------------------------------------------------------------------------------------------
// kernel_estimator.hpp
// ---------------------------------------------------------------------------------------------
void KernelEstParams::validate() const {
    if (n < 1 || n % 2 == 0) throw ParamError("kernel estimation: n must be odd and positive");
    if (alpha1 <= 0 || alpha2 <= 0) throw ParamError("kernel estimation: alpha weights must be positive");
    if (mu1 <= 0 || mu2 <= 0 || mu3 <= 0) throw ParamError("kernel estimation: mu penalties must be positive");
    if (!(rho > 0 && rho < (1.0 + std::sqrt(5.0)) / 2.0))
        throw ParamError("kernel estimation: rho must lie in (0, (1+sqrt(5))/2)");
    if (!(th > 0)) throw ParamError("kernel estimation: th must be positive");
    if (t_max < 1) throw ParamError("kernel estimation: t_max must be >= 1");
}

ObservationSystem::ObservationSystem(const Plane& pan, const Plane& observation, int factor, int n, double mu3)
    : n_(n), mu3_(mu3), ff_(dot(observation, observation)) {
    if (n < 1 || n % 2 == 0) throw ParamError("build_observation: kernel side must be odd");
    if (factor < 1) throw ParamError("build_observation: factor must be >= 1");
    if (pan.height() != factor * observation.height() || pan.width() != factor * observation.width())
        throw DimensionError("build_observation: PAN dimensions must be factor times the observation");
    const std::size_t n2 = static_cast<std::size_t>(n) * n;
    EtE_.resize(n2 * n2);
    Etf_.resize(n2);
    check(fbmp_gpu_gram(ctx(), pan.data(), pan.height(), pan.width(), observation.data(), factor, n, EtE_.data(),
                        Etf_.data()));
}

ObservationSystem build_observation(const Plane& pan, const Plane& observation, int factor, int n, double mu3) {
    return ObservationSystem(pan, observation, factor, n, mu3);
}

double ObservationSystem::data_objective(const std::vector<double>& u) const {
    // 0.5 ||E u - f||^2 = 0.5 (u^T E^T E u - 2 u^T E^T f + f^T f), on the device
    if (u.size() != Etf_.size()) throw DimensionError("data_objective: vector length does not match kernel size");
    double v = 0.0;
    check(fbmp_gpu_data_objective(ctx(), EtE_.data(), Etf_.data(), n_, ff_, u.data(), &v));
    return v;
}

std::vector<double> ObservationSystem::solve_z(const std::vector<double>& anchor) const {
    // (E^T E + mu3 I) z = E^T f + mu3 anchor on the device (Cholesky, explicit inverse, mat-vec)
    const std::size_t n2 = Etf_.size();
    if (anchor.size() != n2) throw DimensionError("solve_z: anchor length does not match kernel size");
    std::vector<double> z(n2);
    check(fbmp_gpu_solve_z(ctx(), EtE_.data(), Etf_.data(), n_, mu3_, anchor.data(), z.data()));
    return z;
}

std::vector<Plane> shrink2(std::span<const Plane> columns, double t) {
    if (t < 0) throw ParamError("shrink2: threshold must be non-negative");
    if (columns.empty()) return {};
    for (const Plane& c : columns)
        if (!c.same_shape(columns.front())) throw DimensionError("shrink2: column shape mismatch");
    const std::size_t m = columns.front().size();
    std::vector<double> buf;
    for (const Plane& c : columns) buf.insert(buf.end(), c.data(), c.data() + m);
    check(fbmp_gpu_shrink2(ctx(), buf.data(), static_cast<int>(columns.size()), static_cast<long long>(m), t));
    std::vector<Plane> out;
    for (std::size_t j = 0; j < columns.size(); ++j)
        out.emplace_back(columns[j].height(), columns[j].width(),
                         std::vector<double>(buf.begin() + static_cast<std::ptrdiff_t>(j * m),
                                             buf.begin() + static_cast<std::ptrdiff_t>((j + 1) * m)));
    return out;
}

std::vector<double> project_simplex(const std::vector<double>& v) {
    std::vector<double> out(v.size());
    check(fbmp_gpu_project_simplex(ctx(), v.data(), static_cast<int>(v.size()), out.data()));
    return out;
}

UpSolution solve_up(const std::array<Plane, 2>& x, const std::array<Plane, 4>& y, const std::array<Plane, 2>& L1,
                    const std::array<Plane, 4>& L2, const KernelEstParams& params) {
    const Plane& ref = x[0];
    for (const Plane* p : {&x[1], &y[0], &y[1], &y[2], &y[3], &L1[0], &L1[1], &L2[0], &L2[1], &L2[2], &L2[3]})
        if (!p->same_shape(ref)) throw DimensionError("solve_up: field shape mismatch");
    if (ref.height() != ref.width()) throw DimensionError("solve_up: the device solver takes square fields");
    const int n = ref.height();
    std::vector<double> f;
    for (const Plane* p : {&x[0], &x[1], &y[0], &y[1], &y[2], &y[3], &L1[0], &L1[1], &L2[0], &L2[1], &L2[2], &L2[3]})
        f.insert(f.end(), p->data(), p->data() + p->size());
    const fbmp_ke_params kp = to_c(params);
    UpSolution s{Plane(n, n), Plane(n, n), Plane(n, n)};
    check(fbmp_gpu_solve_up(ctx(), f.data(), n, &kp, 0.0, nullptr, s.u.data(), s.p1.data(), s.p2.data()));
    return s;
}

double estimation_intensity_scale(const Plane& pan, int factor) {
    double m = 0.0;
    for (double v : pan.samples()) m = std::max(m, std::abs(v));
    if (m <= 0.0) throw NumericalError("kernel estimation: PAN image is identically zero");
    const double hw = static_cast<double>(pan.height() / factor) * (pan.width() / factor);
    return std::sqrt(16384.0 / hw) / m;
}

namespace {
TgvAdmmState unpack_state(const std::vector<double>& s, int n, int iterations) {
    const std::size_t m = static_cast<std::size_t>(n) * n;
    auto plane = [&](int f) {
        return Plane(n, n, std::vector<double>(s.begin() + static_cast<std::ptrdiff_t>(f * m),
                                               s.begin() + static_cast<std::ptrdiff_t>((f + 1) * m)));
    };
    TgvAdmmState st;
    st.u = plane(0);
    st.p1 = plane(1);
    st.p2 = plane(2);
    st.x = {plane(3), plane(4)};
    st.y = {plane(5), plane(6), plane(7), plane(8)};
    st.z = plane(9);
    st.L1 = {plane(10), plane(11)};
    st.L2 = {plane(12), plane(13), plane(14), plane(15)};
    st.L3 = plane(16);
    st.iterations = iterations;
    return st;
}
}  // namespace

Kernel2D estimate_kernel_plane(KernelPrior prior, const Plane& pan, const Plane& observation, int factor,
                               const KernelEstParams& params, TgvAdmmState* final_state,
                               const TgvIterHook& before_up_solve) {
    params.validate();
    if (prior == KernelPrior::l2) {  // kernel_estimator.cpp:452-453
        const fbmp_ke_params kp = to_c(params);
        std::vector<double> taps(static_cast<std::size_t>(params.n) * params.n);
        check(fbmp_gpu_estimate_kernel_l2_plane(ctx(), pan.data(), pan.height(), pan.width(), observation.data(), factor,
                                                &kp, taps.data(), nullptr));
        return Kernel2D(params.n, std::move(taps));
    }
    const bool tv = prior == KernelPrior::tv;  // run_tgv_or_tv(false, ...) (kernel_estimator.cpp:450-451)
    const fbmp_ke_params kp = to_c(params);
    auto plane_call = [&](double* taps, int* it, double* st, int hook_t) {
        return tv ? fbmp_gpu_estimate_kernel_tv_plane(ctx(), pan.data(), pan.height(), pan.width(), observation.data(),
                                                      factor, &kp, taps, it, st, hook_t)
                  : fbmp_gpu_estimate_kernel_plane(ctx(), pan.data(), pan.height(), pan.width(), observation.data(),
                                                   factor, &kp, taps, it, st, hook_t);
    };
    const int n = params.n;
    const std::size_t m = static_cast<std::size_t>(n) * n;
    std::vector<double> taps(m), state(17 * m);
    int iters = 0;
    if (before_up_solve) {
        // hook emulation: the device loop stops at the hook point of iteration t and returns
        // the state; the hook sees the same state the reference passes (kernel_estimator.cpp:344)
        int t_final = 0;
        check(plane_call(taps.data(), &t_final, nullptr, -1));
        for (int t = 0; t < t_final; ++t) {
            int tt = 0;
            check(plane_call(taps.data(), &tt, state.data(), t));
            before_up_solve(unpack_state(state, n, t), t);
        }
    }
    check(plane_call(taps.data(), &iters, final_state ? state.data() : nullptr, -1));
    if (final_state) *final_state = unpack_state(state, n, iters);
    return Kernel2D(n, std::move(taps));
}

Kernel2D estimate_kernel_tgv(const MultiBandImage& lrms_subset, const Plane& pan, const SpectralWeights& omega,
                             int factor, const KernelEstParams& params, TgvAdmmState* final_state,
                             const TgvIterHook& before_up_solve) {
    return estimate_kernel_plane(KernelPrior::tgv2, pan, combine_bands(lrms_subset, omega), factor, params,
                                 final_state, before_up_solve);
}

Kernel2D estimate_kernel_tv(const MultiBandImage& lrms_subset, const Plane& pan, const SpectralWeights& omega, int factor,
                            const KernelEstParams& params) {  // kernel_estimator.cpp:466-471
    return estimate_kernel_plane(KernelPrior::tv, pan, combine_bands(lrms_subset, omega), factor, params);
}

Kernel2D estimate_kernel_l2(const MultiBandImage& lrms_subset, const Plane& pan, const SpectralWeights& omega, int factor,
                            const KernelEstParams& params) {  // kernel_estimator.cpp:473-478
    return estimate_kernel_plane(KernelPrior::l2, pan, combine_bands(lrms_subset, omega), factor, params);
}

double tgv_objective(const ObservationSystem& obs, const Plane& u, const Plane& p1, const Plane& p2,
                     const KernelEstParams& params) {
    const double data = obs.data_objective(std::vector<double>(u.data(), u.data() + u.size()));
    const Plane gx = diff_operator(u, DiffOp::grad_h) - p1, gy = diff_operator(u, DiffOp::grad_v) - p2;
    double t1 = 0.0;
    for (std::size_t i = 0; i < gx.size(); ++i) t1 += std::hypot(gx.data()[i], gy.data()[i]);
    const Plane e1 = diff_operator(p1, DiffOp::grad_h), e4 = diff_operator(p2, DiffOp::grad_v);
    const Plane ec = (diff_operator(p1, DiffOp::grad_v) + diff_operator(p2, DiffOp::grad_h)) * 0.5;
    double t2 = 0.0;
    for (std::size_t i = 0; i < e1.size(); ++i) {
        const double c = ec.data()[i];
        t2 += std::sqrt(e1.data()[i] * e1.data()[i] + e4.data()[i] * e4.data()[i] + 2.0 * c * c);
    }
    return data + params.alpha1 * t1 + params.alpha2 * t2;
}

// ---- evaluation metrics (metrics.hpp:11-51) on the device --------------------------------------
Plane crop_border(const Plane& img, int margin) {  // metrics.cpp:46-58 (data movement only)
    if (margin < 0) throw ParamError("crop_border: negative margin");
    if (margin == 0) return img;
    if (2 * margin >= std::min(img.height(), img.width())) throw DimensionError("crop_border: margin leaves no pixels");
    Plane out(img.height() - 2 * margin, img.width() - 2 * margin);
    for (int r = 0; r < out.height(); ++r)
        for (int c = 0; c < out.width(); ++c) out(r, c) = img(r + margin, c + margin);
    return out;
}

MultiBandImage crop_border(const MultiBandImage& img, int margin) {
    std::vector<Plane> bands;
    bands.reserve(img.band_count());
    for (const Plane& b : img.bands()) bands.push_back(crop_border(b, margin));
    return MultiBandImage(std::move(bands));
}

namespace {
std::vector<double> device_metrics(const MultiBandImage& est, const MultiBandImage& ref, int factor, int which,
                                   std::vector<double>* per_band = nullptr) {
    if (est.band_count() != ref.band_count() || est.height() != ref.height() || est.width() != ref.width())
        throw DimensionError("metrics: image shapes differ");
    const std::vector<double> e = stack(est), r = stack(ref);
    std::vector<double> pb(est.band_count()), out(5);
    check(fbmp_gpu_metrics(ctx(), e.data(), r.data(), est.band_count(), est.height(), est.width(), 0, factor, which,
                           pb.data(), out.data()));
    if (per_band) *per_band = pb;
    return out;
}
}  // namespace

std::pair<std::vector<double>, double> psnr_avg(const MultiBandImage& est, const MultiBandImage& ref) {
    std::vector<double> pb;
    const double avg = device_metrics(est, ref, 1, 1, &pb)[0];
    return {pb, avg};
}

double psnr_plane(const Plane& est, const Plane& ref) {
    if (!est.same_shape(ref)) throw DimensionError("metrics: shape mismatch");
    return psnr_avg(MultiBandImage({est}), MultiBandImage({ref})).second;
}

double psnr_reg_avg(const MultiBandImage& est, const MultiBandImage& ref) { return device_metrics(est, ref, 1, 2)[1]; }

double ergas(const MultiBandImage& est, const MultiBandImage& ref, int factor) {
    return device_metrics(est, ref, factor, 4)[2];
}

double sam_deg(const MultiBandImage& est, const MultiBandImage& ref) { return device_metrics(est, ref, 1, 8)[3]; }

double rase(const MultiBandImage& est, const MultiBandImage& ref) { return device_metrics(est, ref, 1, 16)[4]; }


}  // namespace fbmp
