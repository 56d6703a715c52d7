// metrics.cu -- on-device evaluation metrics: the reductions behind
// PSNR per band and its mean, regressed (best affine fit) PSNR, ERGAS, SAM and RASE
// (proj/src/metrics.cpp:14-153, proj/include/fbmp/metrics.hpp:11-51), over the border-cropped
// cube (crop_border, metrics.cpp:46-58) without copying the crop.
//
// Every sum is a fixed-order reduction (grid-stride per-thread partial, fixed shuffle tree per
// block, block partials summed in index order by one block), so results do not depend on the
// launch. The reference sums sequentially (image.hpp:50-70); the difference is rounding-level.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernel_fit.cuh"

namespace fbmp_gpu {

namespace {

constexpr int MT = 256;   // threads per block
constexpr int MK = 3;     // sums per band and pass

// pass 0: (e - r)^2, e, r                       (mse_plane :14-22, Plane::mean)
// pass 1: (e - me)^2, (e - me)(r - mr), 0       (psnr_reg_avg :82-93)
// pass 2: (a e + b - r)^2, 0, 0                  (:98-102)
template <int PASS>
__global__ void __launch_bounds__(MT) k_met_sums(const double* __restrict__ est, const double* __restrict__ ref,
                                                 int H, int W, int crop, const double* __restrict__ coef,
                                                 double* __restrict__ part) {
    __shared__ double red[3 * (MT / 32 + 1)];
    const int band = blockIdx.y;
    const int hc = H - 2 * crop, wc = W - 2 * crop;
    const long long Pc = static_cast<long long>(hc) * wc;
    const size_t P = static_cast<size_t>(H) * W;
    const double* e = est + band * P;
    const double* r = ref + band * P;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    if (PASS > 0) {
        c0 = coef[4 * band + 0];
        c1 = coef[4 * band + 1];
        c2 = coef[4 * band + 2];
        c3 = coef[4 * band + 3];
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(MT) + threadIdx.x; i < Pc;
         i += static_cast<long long>(gridDim.x) * MT) {
        const int y = static_cast<int>(i / wc), x = static_cast<int>(i - static_cast<long long>(y) * wc);
        const size_t g = static_cast<size_t>(y + crop) * W + (x + crop);
        const double ev = e[g], rv = r[g];
        if (PASS == 0) {
            const double d = ev - rv;
            s0 += d * d;
            s1 += ev;
            s2 += rv;
        } else if (PASS == 1) {  // c0 = me, c1 = mr
            s0 += (ev - c0) * (ev - c0);
            s1 += (ev - c0) * (rv - c1);
        } else {  // c2 = a, c3 = b
            const double d = c2 * ev + c3 - rv;
            s0 += d * d;
        }
    }
    const double t0 = block_sum<MT>(s0, red);
    const double t1 = PASS < 2 ? block_sum<MT>(s1, red + (MT / 32 + 1)) : 0.0;
    const double t2 = PASS == 0 ? block_sum<MT>(s2, red + 2 * (MT / 32 + 1)) : 0.0;
    if (threadIdx.x == 0) {
        double* o = part + (static_cast<size_t>(band) * gridDim.x + blockIdx.x) * MK;
        o[0] = t0;
        o[1] = t1;
        o[2] = t2;
    }
}

// SAM (sam_deg :120-141): per pixel over bands; zero spectral vectors carry no angle
__global__ void __launch_bounds__(MT) k_met_sam(const double* __restrict__ est, const double* __restrict__ ref, int N,
                                                int H, int W, int crop, double* __restrict__ part) {
    __shared__ double red[2 * (MT / 32 + 1)];
    const int hc = H - 2 * crop, wc = W - 2 * crop;
    const long long Pc = static_cast<long long>(hc) * wc;
    const size_t P = static_cast<size_t>(H) * W;
    double acc = 0.0, cnt = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(MT) + threadIdx.x; i < Pc;
         i += static_cast<long long>(gridDim.x) * MT) {
        const int y = static_cast<int>(i / wc), x = static_cast<int>(i - static_cast<long long>(y) * wc);
        const size_t g = static_cast<size_t>(y + crop) * W + (x + crop);
        double dot = 0.0, ne = 0.0, nr = 0.0;
        for (int b = 0; b < N; ++b) {
            const double ev = est[b * P + g], rv = ref[b * P + g];
            dot += ev * rv;
            ne += ev * ev;
            nr += rv * rv;
        }
        if (ne == 0.0 || nr == 0.0) continue;
        const double cosv = fmin(fmax(dot / sqrt(ne * nr), -1.0), 1.0);
        acc += acos(cosv);
        cnt += 1.0;
    }
    const double t0 = block_sum<MT>(acc, red), t1 = block_sum<MT>(cnt, red + (MT / 32 + 1));
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = t0;
        part[2 * blockIdx.x + 1] = t1;
    }
}

// block partials -> per-band sums, in index order
__global__ void __launch_bounds__(MT) k_met_final(const double* __restrict__ part, int nblk, int k,
                                                  double* __restrict__ out) {
    __shared__ double red[MT / 32 + 1];
    const int band = blockIdx.x, j = blockIdx.y;
    double s = 0.0;
    for (int i = threadIdx.x; i < nblk; i += MT) s += part[(static_cast<size_t>(band) * nblk + i) * k + j];
    const double t = block_sum<MT>(s, red);
    if (threadIdx.x == 0) out[band * k + j] = t;
}

double psnr_from_mse(double mse) {  // metrics.cpp:24-27
    if (mse <= 0.0) return INFINITY;
    return 20.0 * std::log10(255.0 / std::sqrt(mse));
}

}  // namespace

void metrics_device(Context& ctx, const double* d_est, const double* d_ref, int N, int H, int W, int crop,
                    int factor, int which, double* psnr_per_band, double* out) {
    if (crop < 0) param_error("crop_border: negative margin");
    if (2 * crop >= std::min(H, W)) dim_error("crop_border: margin leaves no pixels");
    if (N < 1) dim_error("metrics: image shapes differ");
    if ((which & 4) && factor < 1) param_error("ergas: factor must be >= 1");
    const long long Pc = static_cast<long long>(H - 2 * crop) * (W - 2 * crop);
    const int nblk = static_cast<int>(std::max(1LL, std::min<long long>((Pc + MT - 1) / MT, 4LL * ctx.sm_count)));
    double* part = ctx.scratch<double>("met_part", static_cast<size_t>(N) * nblk * MK);
    double* sums = ctx.scratch<double>("met_sums", static_cast<size_t>(N) * MK);
    double* coef = ctx.scratch<double>("met_coef", static_cast<size_t>(N) * 4);
    std::vector<double> s0(static_cast<size_t>(N) * MK), s1, s2;
    auto run = [&](auto kernel, std::vector<double>& host) {
        kernel<<<dim3(nblk, N), MT, 0, ctx.stream>>>(d_est, d_ref, H, W, crop, coef, part);
        k_met_final<<<dim3(N, MK), MT, 0, ctx.stream>>>(part, nblk, MK, sums);
        ctx.count(2);
        check_launch();
        host.resize(static_cast<size_t>(N) * MK);
        FBMP_CUDA(cudaMemcpyAsync(host.data(), sums, host.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    };
    run(k_met_sums<0>, s0);
    const double np_ = static_cast<double>(Pc);
    std::vector<double> mse(N), me(N), mr(N);
    for (int b = 0; b < N; ++b) {
        mse[b] = s0[b * MK + 0] / np_;
        me[b] = s0[b * MK + 1] / np_;
        mr[b] = s0[b * MK + 2] / np_;
    }
    for (int i = 0; i < 5; ++i) out[i] = NAN;
    if (which & 1) {  // psnr_avg (:66-79)
        double sum = 0.0;
        for (int b = 0; b < N; ++b) {
            psnr_per_band[b] = psnr_from_mse(mse[b]);
            sum += psnr_per_band[b];
        }
        out[0] = sum / N;
    }
    if (which & 2) {  // psnr_reg_avg (:81-105)
        std::vector<double> cf(static_cast<size_t>(N) * 4, 0.0);
        for (int b = 0; b < N; ++b) {
            cf[4 * b] = me[b];
            cf[4 * b + 1] = mr[b];
        }
        FBMP_CUDA(cudaMemcpyAsync(coef, cf.data(), cf.size() * sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
        run(k_met_sums<1>, s1);
        for (int b = 0; b < N; ++b) {
            const double var = s1[b * MK], cov = s1[b * MK + 1];
            double a = 0.0, bb = mr[b];  // constant estimate fits the reference mean
            if (var > 0.0) {
                a = cov / var;
                bb = mr[b] - a * me[b];
            }
            cf[4 * b + 2] = a;
            cf[4 * b + 3] = bb;
        }
        FBMP_CUDA(cudaMemcpyAsync(coef, cf.data(), cf.size() * sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
        run(k_met_sums<2>, s2);
        double sum = 0.0;
        for (int b = 0; b < N; ++b) sum += psnr_from_mse(s2[b * MK] / np_);
        out[1] = sum / N;
    }
    if (which & 4) {  // ergas (:107-118)
        double acc = 0.0;
        for (int b = 0; b < N; ++b) {
            if (mr[b] == 0.0) num_error("ergas: reference band mean is zero");
            const double rmse = std::sqrt(mse[b]);
            acc += (rmse / mr[b]) * (rmse / mr[b]);
        }
        out[2] = 100.0 / factor * std::sqrt(acc / N);
    }
    if (which & 8) {  // sam_deg (:120-141)
        k_met_sam<<<nblk, MT, 0, ctx.stream>>>(d_est, d_ref, N, H, W, crop, part);
        k_met_final<<<dim3(1, 2), MT, 0, ctx.stream>>>(part, nblk, 2, sums);
        ctx.count(2);
        check_launch();
        double h2[2];
        FBMP_CUDA(cudaMemcpyAsync(h2, sums, sizeof(h2), cudaMemcpyDeviceToHost, ctx.stream));
        FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
        out[3] = h2[1] == 0.0 ? 0.0 : h2[0] / h2[1] * 180.0 / M_PI;
    }
    if (which & 16) {  // rase (:143-153)
        double mu = 0.0;
        for (int b = 0; b < N; ++b) mu += mr[b];
        mu /= N;
        if (mu == 0.0) num_error("rase: mean of reference image is zero");
        double acc = 0.0;
        for (int b = 0; b < N; ++b) acc += mse[b];
        out[4] = 100.0 / mu * std::sqrt(acc / N);
    }
}

}  // namespace fbmp_gpu
