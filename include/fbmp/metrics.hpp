// metrics.hpp -- drop-in for the reference's evaluation metrics (proj/include/fbmp/metrics.hpp:11-51):
// the border crop and the PSNR / regressed PSNR / ERGAS / SAM / RASE reductions, computed on the
// GPU (csrc/metrics.cu through fbmp_gpu_metrics). Inputs on the [0, 255] scale. SSIM against the
// PAN, the kernel error and the MetricsReport text/CSV formatting are not part of this library.
#pragma once

#include <utility>
#include <vector>

#include "fbmp/image.hpp"

namespace fbmp {

MultiBandImage crop_border(const MultiBandImage& img, int margin);  // metrics.hpp:28
Plane crop_border(const Plane& img, int margin);                    // metrics.hpp:29

// Per-band 20*log10(255/sqrt(MSE)) and their mean; identical bands report +infinity.
std::pair<std::vector<double>, double> psnr_avg(const MultiBandImage& est, const MultiBandImage& ref);
double psnr_plane(const Plane& est, const Plane& ref);

// Best-affine-fit PSNR averaged over bands (metrics.hpp:36-38).
double psnr_reg_avg(const MultiBandImage& est, const MultiBandImage& ref);

double ergas(const MultiBandImage& est, const MultiBandImage& ref, int factor);
double sam_deg(const MultiBandImage& est, const MultiBandImage& ref);
double rase(const MultiBandImage& est, const MultiBandImage& ref);

}  // namespace fbmp
