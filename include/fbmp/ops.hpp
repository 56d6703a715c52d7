// fbmp/ops.hpp -- image operators of the fbmp:: API (reference: include/fbmp/ops.hpp).
// Convolutions, box means and difference stencils run on the GPU (fbmp_gpu.h); the pure
// index maps (embedding, sampling) are host data movement.
#pragma once

#include "fbmp/image.hpp"

namespace fbmp {

Plane circular_convolve(const Plane& img, const Kernel2D& k);          // centre tap at the origin
Plane circular_convolve_adjoint(const Plane& img, const Kernel2D& k);  // circular correlation
Plane embed_kernel(const Kernel2D& k, int height, int width);          // PSF -> transfer-function layout
Plane downsample(const Plane& img, int factor);                        // keeps (c*i, c*j)
Plane upsample_adjoint(const Plane& img, int factor);                  // zero insertion

enum class DiffOp { grad_h, grad_v, laplacian };
Plane diff_operator(const Plane& img, DiffOp which);  // circular forward differences / 5-point Laplacian
Plane diff_adjoint(const Plane& img, DiffOp which);

Plane box_mean(const Plane& img, int radius);          // clamped (2r+1)^2 window mean
Plane circular_box_blur(const Plane& img, int window);

}  // namespace fbmp
