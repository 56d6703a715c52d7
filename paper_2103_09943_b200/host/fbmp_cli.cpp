// fbmp_cli.cpp -- command-line front end over the fbmp:: API (the reference's CLI,
// proj/tools/fbmp_main.cpp, is an empty stub; the commands follow SPEC.md:575-591):
//
//   fbmp blind           --lrms L.fbmp --pan P.fbmp --out HRMS.fbmp [--kernel-out K.fbmp]
//                        [--n 29] [--pan-bands 0,1,...] [--l 4] [--lambda-omega 10]
//   fbmp estimate-kernel --lrms L.fbmp --pan P.fbmp --out K.fbmp [--n 29] [--pan-bands ...]
//   fbmp pansharpen      --lrms L.fbmp --pan P.fbmp --kernel K.fbmp --out HRMS.fbmp
//   fbmp metrics         --est E.fbmp --ref R.fbmp [--border 10] [--factor c]   (inputs on [0, 255])
//   fbmp info            --in X.fbmp                                         (height width bands)
//
// The factor is PAN height / LRMS height. Exit codes: 1 usage, parameter or
// dimension error; 2 I/O or format error; 3 numerical error; 4 device error.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "fbmp/errors.hpp"
#include "fbmp/kernel_estimator.hpp"
#include "fbmp/metrics.hpp"
#include "fbmp/pansharpen.hpp"
#include "fbmp/raster_io.hpp"
#include "fbmp/spectral_weights.hpp"

using namespace fbmp;

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::map<std::string, std::string> parse(int argc, char** argv) {
    std::map<std::string, std::string> a;
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc) throw Usage("expected --flag value pairs, got '" + k + "'");
        a[k.substr(2)] = argv[++i];
    }
    return a;
}
std::string need(const std::map<std::string, std::string>& a, const std::string& k) {
    const auto it = a.find(k);
    if (it == a.end()) throw Usage("missing required flag --" + k);
    return it->second;
}
int geti(const std::map<std::string, std::string>& a, const std::string& k, int d) {
    const auto it = a.find(k);
    return it == a.end() ? d : std::atoi(it->second.c_str());
}
double getd(const std::map<std::string, std::string>& a, const std::string& k, double d) {
    const auto it = a.find(k);
    return it == a.end() ? d : std::atof(it->second.c_str());
}

int factor_of(const MultiBandImage& lrms, const Plane& pan) {
    if (lrms.height() < 1 || pan.height() % lrms.height() || pan.width() % lrms.width() ||
        pan.height() / lrms.height() != pan.width() / lrms.width() || pan.height() < lrms.height())
        throw DimensionError("PAN dimensions must be an integer multiple (the same in both axes) of the LRMS");
    return pan.height() / lrms.height();
}

MultiBandImage subset(const MultiBandImage& lrms, const std::map<std::string, std::string>& a) {
    const auto it = a.find("pan-bands");
    if (it == a.end()) return lrms;
    std::vector<Plane> sel;
    std::stringstream ss(it->second);
    for (std::string t; std::getline(ss, t, ',');) {
        const int b = std::atoi(t.c_str());
        if (b < 0 || b >= lrms.band_count()) throw ParamError("pan_bands references missing band " + t);
        sel.push_back(lrms.band(b));
    }
    if (sel.empty()) throw ParamError("pan_bands is empty");
    return MultiBandImage(std::move(sel));
}

Kernel2D fit(const MultiBandImage& lrms, const Plane& pan, int c, const std::map<std::string, std::string>& a) {
    const MultiBandImage sub = subset(lrms, a);
    SpectralWeightConfig sw;
    sw.l = geti(a, "l", 4);
    sw.lambda_omega = getd(a, "lambda-omega", 10.0);
    sw.factor = c;
    const SpectralWeights w = solve_weights(sub, pan, sw);
    KernelEstParams ke;
    ke.n = geti(a, "n", 29);
    return estimate_kernel_tgv(sub, pan, w, c, ke);
}

int run(int argc, char** argv) {
    if (argc < 2) throw Usage("usage: fbmp {blind|estimate-kernel|pansharpen|metrics|info} --flag value ...");
    const std::string cmd = argv[1];
    const auto a = parse(argc, argv);
    if (cmd == "blind" || cmd == "estimate-kernel" || cmd == "pansharpen") {
        const MultiBandImage lrms = load_raster(need(a, "lrms"));
        const MultiBandImage panr = load_raster(need(a, "pan"));
        if (panr.band_count() != 1) throw DimensionError("PAN raster must have one band");
        const Plane& pan = panr.band(0);
        const int c = factor_of(lrms, pan);
        const std::string out = need(a, "out");
        if (cmd == "estimate-kernel") {
            save_kernel(fit(lrms, pan, c, a), out);
            return 0;
        }
        const Kernel2D k = cmd == "blind" ? fit(lrms, pan, c, a) : load_kernel(need(a, "kernel"));
        save_raster(pansharpen(lrms, pan, k, c, PansharpenParams{}), out);
        if (cmd == "blind" && a.count("kernel-out")) save_kernel(k, a.at("kernel-out"));
        return 0;
    }
    if (cmd == "info") {  // header of a raster: height width bands
        const MultiBandImage img = load_raster(need(a, "in"));
        std::printf("%d %d %d\n", img.height(), img.width(), img.band_count());
        return 0;
    }
    if (cmd == "metrics") {
        const MultiBandImage est = load_raster(need(a, "est")), ref = load_raster(need(a, "ref"));
        const int border = geti(a, "border", 10);
        const MultiBandImage e = crop_border(est, border), r = crop_border(ref, border);
        const auto [per, avg] = psnr_avg(e, r);
        std::printf("psnr_avg %.10g\npsnr_reg_avg %.10g\nergas %.10g\nsam_deg %.10g\nrase %.10g\n", avg,
                    psnr_reg_avg(e, r), ergas(e, r, geti(a, "factor", 4)), sam_deg(e, r), rase(e, r));
        for (std::size_t i = 0; i < per.size(); ++i) std::printf("psnr_band_%zu %.10g\n", i, per[i]);
        return 0;
    }
    throw Usage("unknown command '" + cmd + "'");
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const Usage& e) {
        std::fprintf(stderr, "fbmp: %s\n", e.what());
        return 1;
    } catch (const ParamError& e) {
        std::fprintf(stderr, "fbmp: parameter error: %s\n", e.what());
        return 1;
    } catch (const DimensionError& e) {
        std::fprintf(stderr, "fbmp: dimension error: %s\n", e.what());
        return 1;
    } catch (const IoError& e) {
        std::fprintf(stderr, "fbmp: I/O error: %s\n", e.what());
        return 2;
    } catch (const FormatError& e) {
        std::fprintf(stderr, "fbmp: format error: %s\n", e.what());
        return 2;
    } catch (const NumericalError& e) {
        std::fprintf(stderr, "fbmp: numerical error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "fbmp: device error: %s\n", e.what());
        return 4;
    }
}
