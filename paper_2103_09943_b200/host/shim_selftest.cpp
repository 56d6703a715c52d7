// shim_selftest.cpp -- exercises the fbmp:: C++ API (the drop-in for the reference's headers)
// on the GPU: a few of the reference's own test cases (tests/test_pansharpen.cpp,
// tests/test_kernel_estimator.cpp, tests/test_spectral_weights.cpp) restated, plus a blind
// solve. Prints one line per check; exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>

#include "fbmp/kernel_estimator.hpp"
#include "fbmp/metrics.hpp"
#include "fbmp/ops.hpp"
#include "fbmp/pansharpen.hpp"
#include "fbmp/spectral_weights.hpp"

using namespace fbmp;

static int failures = 0;
static void report(const char* name, bool ok, const std::string& extra = "") {
    std::printf("%s %s %s\n", ok ? "PASS" : "FAIL", name, extra.c_str());
    failures += ok ? 0 : 1;
}
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Plane random_plane(std::mt19937_64& rng, int h, int w, double lo = 0.0, double hi = 1.0) {
    std::uniform_real_distribution<double> d(lo, hi);
    Plane p(h, w);
    for (double& v : p.samples()) v = d(rng);
    return p;
}
static Kernel2D random_kernel(std::mt19937_64& rng, int n) {
    std::uniform_real_distribution<double> d(0.0, 1.0);
    Kernel2D k(n);
    for (double& v : k.taps().samples()) v = d(rng);
    k.normalize();
    return k;
}

int main() {
    std::mt19937_64 rng(2103);
    {  // test_pansharpen.cpp:63-69
        MattingMatrix M = build_matting_matrix(Plane(3, 3, 4.2), 1, 1e-4);
        double err = 0.0;
        for (int j = 0; j < 9; ++j) {
            Plane e(3, 3);
            e.data()[j] = 1.0;
            Plane col = M.apply(e);
            for (int i = 0; i < 9; ++i) err = std::max(err, std::abs(col.data()[i] - ((i == j) - 1.0 / 9.0)));
        }
        report("matting_constant_guide", err < 1e-12);
    }
    {  // test_pansharpen.cpp:113-126
        Plane pan = random_plane(rng, 16, 16);
        PansharpenParams prm;
        prm.cg_tol = 1e-10;
        prm.cg_max_iter = 4000;
        MattingMatrix M = build_matting_matrix(apply_prior(pan, prm), prm.radius, prm.eps);
        Plane z0 = warmstart_channel(Plane(8, 8, 0.37), pan, random_kernel(rng, 5), 2, M, prm);
        double err = 0.0;
        for (double v : z0.samples()) err = std::max(err, std::abs(v - 0.37));
        report("warmstart_constant_channel", err <= 1e-5 * 0.37);
    }
    {  // test_pansharpen.cpp:172-183
        Plane pan = random_plane(rng, 16, 16);
        PansharpenParams prm;
        prm.cg_tol = 1e-14;
        prm.cg_max_iter = 2;
        MattingMatrix M = build_matting_matrix(apply_prior(pan, prm), prm.radius, prm.eps);
        Plane x = random_plane(rng, 8, 8);
        Kernel2D k = random_kernel(rng, 5);
        report("warmstart_cap_error", throws<NumericalError>([&] { warmstart_channel(x, pan, k, 2, M, prm); }));
    }
    {  // test_pansharpen.cpp:405-415
        PansharpenParams prm;
        prm.lambda = 0.0;
        bool ok = throws<ParamError>([&] { prm.validate(); });
        prm = PansharpenParams{};
        prm.prior = PriorKind::custom;
        ok = ok && throws<ParamError>([&] { prm.validate(); });
        report("pansharpen_validation", ok);
    }
    {  // test_kernel_estimator.cpp:153-176
        std::vector<Plane> cols = {Plane(1, 1, 3.0), Plane(1, 1, 4.0)};
        auto out = shrink2(cols, 1.0);
        report("shrink2_kat", std::abs(out[0](0, 0) - 2.4) < 1e-15 && std::abs(out[1](0, 0) - 3.2) < 1e-15);
        auto p = project_simplex({0.5, 0.7});
        report("project_simplex_kat", std::abs(p[0] - 0.4) < 1e-15 && std::abs(p[1] - 0.6) < 1e-15);
    }
    {  // test_kernel_estimator.cpp:297-305
        MultiBandImage lrms({Plane(8, 8, 0.5)});
        SpectralWeights w{{1.0}};
        KernelEstParams prm;
        prm.n = 3;
        report("degenerate_pan", throws<NumericalError>([&] { estimate_kernel_tgv(lrms, Plane(16, 16, 1.0), w, 2, prm); }));
    }
    {  // test_spectral_weights.cpp:143-147
        SpectralWeightConfig cfg;
        cfg.factor = 2;
        cfg.l = 2;
        cfg.lambda_omega = 0.0;
        MultiBandImage lrms({Plane(8, 8, 1.0), Plane(8, 8, 1.0)});
        report("weights_singular", throws<NumericalError>([&] { solve_weights(lrms, Plane(16, 16, 2.0), cfg); }));
    }
    {  // blind composition on a 128 x 128 textured scene, plus the hook
        const int H = 128, c = 4, N = 3, n = 7;
        Plane pan(H, H);
        for (int r = 0; r < H; ++r)
            for (int q = 0; q < H; ++q)
                pan(r, q) = 0.5 + 0.25 * std::sin(0.19 * r) * std::cos(0.23 * q) + 0.2 * ((r / 16 + q / 16) % 2);
        Kernel2D truth(n);
        for (int r = 0; r < n; ++r)
            for (int q = 0; q < n; ++q) truth(r, q) = std::exp(-0.5 * ((r - 3.3) * (r - 3.3) + (q - 2.8) * (q - 2.8)) / 1.7);
        truth.normalize();
        std::vector<Plane> bands;
        for (int b = 0; b < N; ++b) {
            Plane hr = pan * (0.8 + 0.2 * b);
            bands.push_back(downsample(circular_convolve(hr, truth), c));
        }
        MultiBandImage lrms(bands);
        SpectralWeightConfig cfg;
        cfg.factor = c;
        SpectralWeights w = solve_weights(lrms, pan, cfg);
        KernelEstParams kp;
        kp.n = n;
        int hooks = 0;
        TgvAdmmState st;
        kp.t_max = 6;
        Kernel2D k6 = estimate_kernel_tgv(lrms, pan, w, c, kp, &st,
                                          [&](const TgvAdmmState& s, int t) { hooks += (s.z.size() == 49 && t == hooks); });
        report("kernel_hook", hooks == 6 && st.iterations == 6 && k6.in_simplex(1e-9));
        kp.t_max = 10000;
        Kernel2D k = estimate_kernel_tgv(lrms, pan, w, c, kp);
        PansharpenParams prm;
        MultiBandImage out = pansharpen(lrms, pan, k, c, prm);
        bool finite = true;
        for (const Plane& b : out.bands()) finite = finite && b.all_finite();
        report("blind_composition", k.in_simplex(1e-9) && finite && out.band_count() == N && out.height() == H,
               "kernel_sum=" + std::to_string(k.sum()));
        // equal bands give equal outputs (test_pansharpen.cpp:350-361)
        MultiBandImage same({bands[0], bands[0]});
        MultiBandImage o2 = pansharpen(same, pan, k, c, prm);
        bool eq = true;
        for (std::size_t i = 0; i < o2.band(0).size(); ++i) eq = eq && o2.band(0).data()[i] == o2.band(1).data()[i];
        report("equal_bands", eq);
    }
    {  // tests/test_metrics.cpp: crop, identical / offset / affine / scaled cubes, the MSE oracle
        MultiBandImage ref({random_plane(rng, 30, 30, 0.0, 255.0), random_plane(rng, 30, 30, 0.0, 255.0)});
        MultiBandImage est = ref;
        est.band(0)(0, 0) += 50.0;
        MultiBandImage ref1({ref.band(0)}), est1({est.band(0)});  // one band, as the reference's case
        report("metrics_crop", std::isfinite(psnr_avg(est1, ref1).second) &&
                                   std::isinf(psnr_avg(crop_border(est1, 10), crop_border(ref1, 10)).second));
        MultiBandImage off = ref, aff = ref, sc = ref;
        for (int b = 0; b < 2; ++b) {
            off.band(b) += 255.0;
            aff.band(b) *= 0.5;
            aff.band(b) += 3.0;
            sc.band(b) *= 3.0;
        }
        report("metrics_ideal", std::isinf(psnr_avg(ref, ref).second) && std::abs(psnr_avg(off, ref).second) < 1e-12 &&
                                    psnr_reg_avg(aff, ref) > 200.0 && ergas(ref, ref, 4) == 0.0 &&
                                    rase(ref, ref) == 0.0 && std::abs(sam_deg(sc, ref)) < 1e-6);
        double mse = 0.0;
        for (std::size_t i = 0; i < est.band(0).size(); ++i) {
            const double d = est.band(0).data()[i] - ref.band(0).data()[i];
            mse += d * d;
        }
        mse /= est.band(0).size();
        report("metrics_psnr_oracle",
               std::abs(psnr_avg(est, ref).first[0] - 20.0 * std::log10(255.0 / std::sqrt(mse))) < 1e-10);
        report("metrics_errors", throws<DimensionError>([&] { crop_border(ref, 15); }) &&
                                     throws<NumericalError>([&] { ergas(ref, MultiBandImage(2, 30, 30), 4); }));
    }
    {  // ObservationSystem::solve_z / data_objective on the device (kernel_estimator.cpp:79-87):
       // the normal equations hold and 0.5 ||E z - f||^2 >= 0 decreases from the zero kernel
        Plane pan = random_plane(rng, 32, 32), obs = random_plane(rng, 16, 16);
        ObservationSystem sys = build_observation(pan, obs, 2, 5, 3.0);
        const std::size_t n2 = 25;
        std::vector<double> anchor(n2);
        for (double& a : anchor) a = std::uniform_real_distribution<double>(-1.0, 1.0)(rng);
        const std::vector<double> z = sys.solve_z(anchor);
        double res = 0.0, nrm = 0.0;
        for (std::size_t a = 0; a < n2; ++a) {
            double r = 3.0 * z[a] - sys.Etf()[a] - 3.0 * anchor[a];
            for (std::size_t b = 0; b < n2; ++b) r += sys.EtE()[a * n2 + b] * z[b];
            res += r * r;
            nrm += sys.Etf()[a] * sys.Etf()[a];
        }
        const double f0 = sys.data_objective(std::vector<double>(n2, 0.0));
        double ff = 0.0;
        for (double v : obs.samples()) ff += v * v;
        report("solve_z_device", std::sqrt(res) <= 1e-10 * std::sqrt(nrm) && std::abs(f0 - 0.5 * ff) <= 1e-12 * ff &&
                                     sys.data_objective(z) >= 0.0 &&
                                     throws<DimensionError>([&] { sys.solve_z(std::vector<double>(3)); }));
    }
    std::printf("%d failures\n", failures);
    return failures;
}
