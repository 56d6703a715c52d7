// fbmp_oracle.cpp -- CPU fp64 restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY. This library is the parity checker for the GPU path: only
// tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / `--impl reference` legs
// may load it. It is never linked into, or called by, the product library.
//
// Why a restatement: the reference (/root/reference/proj) needs Eigen3, FFTW3 and libpng,
// none of which exist in this image, so it cannot be built. This file
// restates, in plain C++17 on raw row-major arrays, every function on the hot path, each
// citing the reference file:line it follows (paths relative to /root/reference/proj).
// Third-party arithmetic is replaced as SURVEY.md §8(c) prescribes:
//   * FFTW c2c (fft_util.cpp:12-62)        -> exact radix-2 / direct DFT, same conventions
//   * Eigen SparseMatrix RowMajor SpMV       -> CSR with the same per-row column order
//   * Eigen SelfAdjointEigenSolver (16x16)   -> cyclic complex Jacobi eigen-solver
//   * Eigen LLT / FullPivLU                  -> Cholesky / Gauss-Jordan with full pivoting
// Pinned by: the reference tests' known answers and oracles (restated in
// tests/test_oracle_kats.py) and an independent numpy/scipy restatement
// (oracle/fbmp_numpy.py), see DESIGN.md "Oracle".
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using cd = std::complex<double>;
using vec = std::vector<double>;
using cvec = std::vector<cd>;
constexpr double kPi = 3.14159265358979323846264338327950288;

// error taxonomy of errors.hpp:8-33 -> status codes 1 param, 2 dimension, 3 numerical
struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void param_error(const std::string& m) { throw Failure(1, m); }
[[noreturn]] void dim_error(const std::string& m) { throw Failure(2, m); }
[[noreturn]] void num_error(const std::string& m) { throw Failure(3, m); }

thread_local std::string g_last_error;

bool trace_cg() {
    static const bool on = std::getenv("FBMP_ORACLE_TRACE") != nullptr;
    return on;
}

// ---- sequential reductions: image.hpp:50-55 (sum), 93-98 (dot), 66-70 (norm) ----------
double seq_dot(const double* a, const double* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
double seq_norm(const double* a, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * a[i];
    return std::sqrt(s);
}
double seq_max(const double* a, size_t n) {
    double m = n ? a[0] : 0.0;
    for (size_t i = 0; i < n; ++i) m = std::max(m, a[i]);
    return m;
}

// ---- 1-D / 2-D DFT with FFTW's c2c conventions (fft_util.cpp:31-62) -------------------
// (a b) for finite operands: the expression std::complex's operator* evaluates before its
// NaN recovery branch (no FMA contraction: -ffp-contract=off), without that branch
inline cd cmul_finite(cd a, cd b) {
    return cd(a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real());
}
class Dft1 {
public:
    explicit Dft1(int n) : n_(n) {
        pow2_ = n > 0 && (n & (n - 1)) == 0;
        tw_.resize(n);
        for (int k = 0; k < n; ++k) {
            const double a = -2.0 * kPi * k / n;
            tw_[k] = cd(std::cos(a), std::sin(a));
        }
        if (pow2_) {
            rev_.resize(n);
            int lg = 0;
            while ((1 << lg) < n) ++lg;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int b = 0; b < lg; ++b)
                    if (i & (1 << b)) r |= 1 << (lg - 1 - b);
                rev_[i] = r;
            }
        }
    }
    // kB adjacent transforms at once (x[i * s + b], b < kB): the same operations per transform as
    // run(), laid out so that the strided column pass of a 2-D FFT touches kB consecutive
    // elements per row (cache blocking only; results are bit-identical to kB calls of run())
    template <int kB>
    void run_block(cd* x, size_t s, int sign, cd* scratch) const {
        const int n = n_;
        if (pow2_) {
            for (int i = 0; i < n; ++i)
                for (int b = 0; b < kB; ++b) scratch[static_cast<size_t>(rev_[i]) * kB + b] = x[i * s + b];
            for (int len = 2; len <= n; len <<= 1) {
                const int half = len >> 1, step = n / len;
                for (int i = 0; i < n; i += len)
                    for (int j = 0; j < half; ++j) {
                        cd w = tw_[j * step];
                        if (sign > 0) w = std::conj(w);
                        cd* lo = scratch + static_cast<size_t>(i + j) * kB;
                        cd* hi = scratch + static_cast<size_t>(i + j + half) * kB;
                        for (int b = 0; b < kB; ++b) {
                            const cd u = lo[b], v = cmul_finite(hi[b], w);
                            lo[b] = u + v;
                            hi[b] = u - v;
                        }
                    }
            }
            for (int i = 0; i < n; ++i)
                for (int b = 0; b < kB; ++b) x[i * s + b] = scratch[static_cast<size_t>(i) * kB + b];
        } else {
            for (int k = 0; k < n; ++k) {
                cd acc[kB];
                for (int b = 0; b < kB; ++b) acc[b] = 0.0;
                for (int j = 0; j < n; ++j) {
                    cd w = tw_[(static_cast<long>(k) * j) % n];
                    if (sign > 0) w = std::conj(w);
                    for (int b = 0; b < kB; ++b) acc[b] += x[j * s + b] * w;
                }
                for (int b = 0; b < kB; ++b) scratch[static_cast<size_t>(k) * kB + b] = acc[b];
            }
            for (int k = 0; k < n; ++k)
                for (int b = 0; b < kB; ++b) x[k * s + b] = scratch[static_cast<size_t>(k) * kB + b];
        }
    }
    // in-place, stride s; sign -1 forward (exp(-i..)), +1 backward (unnormalised)
    void run(cd* x, size_t s, int sign, cd* scratch) const {
        const int n = n_;
        if (pow2_) {
            for (int i = 0; i < n; ++i) scratch[rev_[i]] = x[i * s];
            for (int len = 2; len <= n; len <<= 1) {
                const int half = len >> 1, step = n / len;
                for (int i = 0; i < n; i += len)
                    for (int j = 0; j < half; ++j) {
                        cd w = tw_[j * step];
                        if (sign > 0) w = std::conj(w);
                        const cd u = scratch[i + j], v = cmul_finite(scratch[i + j + half], w);
                        scratch[i + j] = u + v;
                        scratch[i + j + half] = u - v;
                    }
            }
            for (int i = 0; i < n; ++i) x[i * s] = scratch[i];
        } else {
            for (int k = 0; k < n; ++k) {
                cd acc = 0.0;
                for (int j = 0; j < n; ++j) {
                    cd w = tw_[(static_cast<long>(k) * j) % n];
                    if (sign > 0) w = std::conj(w);
                    acc += x[j * s] * w;
                }
                scratch[k] = acc;
            }
            for (int k = 0; k < n; ++k) x[k * s] = scratch[k];
        }
    }

private:
    int n_;
    bool pow2_;
    cvec tw_;
    std::vector<int> rev_;
};

class Fft2 {
public:
    Fft2(int rows, int cols) : r_(rows), c_(cols), dr_(rows), dc_(cols) {
        if (rows < 1 || cols < 1) dim_error("Fft2D: empty grid");
    }
    size_t size() const { return static_cast<size_t>(r_) * c_; }
    void transform(cvec& a, int sign) const {
        constexpr int kB = 16;  // columns per block of the column pass
        cvec scratch(static_cast<size_t>(std::max(r_, c_)) * kB);
        for (int i = 0; i < r_; ++i) dc_.run(a.data() + static_cast<size_t>(i) * c_, 1, sign, scratch.data());
        int j = 0;
        for (; j + kB <= c_; j += kB) dr_.run_block<kB>(a.data() + j, c_, sign, scratch.data());
        for (; j < c_; ++j) dr_.run(a.data() + j, c_, sign, scratch.data());
    }
    cvec forward(const double* in) const {  // fft_util.cpp:31-39
        cvec a(size());
        for (size_t i = 0; i < a.size(); ++i) a[i] = cd(in[i], 0.0);
        transform(a, -1);
        return a;
    }
    vec backward_real(cvec a) const {  // fft_util.cpp:47-56: x 1/(rows*cols), real part
        transform(a, +1);
        const double sc = 1.0 / static_cast<double>(size());
        vec out(size());
        for (size_t i = 0; i < out.size(); ++i) out[i] = a[i].real() * sc;
        return out;
    }

private:
    int r_, c_;
    Dft1 dr_, dc_;
};

// ---- ops.cpp ----------------------------------------------------------------------------
// ops.cpp:9-22: centre tap to (0,0), other taps wrapped
vec embed_kernel(const double* k, int n, int h, int w) {
    if (n > h || n > w) dim_error("kernel larger than image");
    vec out(static_cast<size_t>(h) * w, 0.0);
    const int c = (n - 1) / 2;
    for (int r = 0; r < n; ++r)
        for (int q = 0; q < n; ++q) {
            int rr = (r - c) % h; if (rr < 0) rr += h;
            int cc = (q - c) % w; if (cc < 0) cc += w;
            out[static_cast<size_t>(rr) * w + cc] += k[r * n + q];
        }
    return out;
}

// fft_util.hpp:52-63 / fft_util.cpp:64-85: cached-spectrum circular convolution
struct SpecConv {
    Fft2 fft;
    cvec spec;
    SpecConv(const double* k, int n, int h, int w) : fft(h, w) {
        if (n > h || n > w) dim_error("kernel larger than image");
        vec e = embed_kernel(k, n, h, w);
        spec = fft.forward(e.data());
    }
    vec apply(const double* img, bool adjoint) const {
        cvec a = fft.forward(img);
        for (size_t i = 0; i < a.size(); ++i) a[i] *= adjoint ? std::conj(spec[i]) : spec[i];
        return fft.backward_real(std::move(a));
    }
};

// ops.cpp:36-45
vec downsample(const double* img, int H, int W, int c) {
    if (c < 1) param_error("downsample: factor must be >= 1");
    if (H % c || W % c) dim_error("downsample: dimensions not divisible by factor");
    const int h = H / c, w = W / c;
    vec out(static_cast<size_t>(h) * w);
    for (int r = 0; r < h; ++r)
        for (int q = 0; q < w; ++q) out[static_cast<size_t>(r) * w + q] = img[static_cast<size_t>(r * c) * W + q * c];
    return out;
}
// ops.cpp:47-54
vec upsample_adjoint(const double* img, int h, int w, int c) {
    if (c < 1) param_error("upsample_adjoint: factor must be >= 1");
    const int W = w * c;
    vec out(static_cast<size_t>(h) * c * W, 0.0);
    for (int r = 0; r < h; ++r)
        for (int q = 0; q < w; ++q) out[static_cast<size_t>(r * c) * W + q * c] = img[static_cast<size_t>(r) * w + q];
    return out;
}
// ops.cpp:70-78 (laplacian), 60-69 (forward differences), 87-97 (adjoints)
vec laplacian(const double* x, int h, int w) {
    vec out(static_cast<size_t>(h) * w);
    for (int r = 0; r < h; ++r) {
        const int rm = (r + h - 1) % h, rp = (r + 1) % h;
        for (int c = 0; c < w; ++c) {
            const int cm = (c + w - 1) % w, cp = (c + 1) % w;
            out[static_cast<size_t>(r) * w + c] = 4.0 * x[static_cast<size_t>(r) * w + c] - x[static_cast<size_t>(rm) * w + c] -
                                                  x[static_cast<size_t>(rp) * w + c] - x[static_cast<size_t>(r) * w + cm] -
                                                  x[static_cast<size_t>(r) * w + cp];
        }
    }
    return out;
}
enum Diff { GH = 0, GV = 1, LAP = 2 };
vec diff(const double* x, int h, int w, int which, bool adjoint) {
    if (which == LAP) return laplacian(x, h, w);
    vec out(static_cast<size_t>(h) * w);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            int rr = r, cc = c;
            if (which == GH) cc = adjoint ? (c + w - 1) % w : (c + 1) % w;
            else rr = adjoint ? (r + h - 1) % h : (r + 1) % h;
            out[static_cast<size_t>(r) * w + c] = x[static_cast<size_t>(rr) * w + cc] - x[static_cast<size_t>(r) * w + c];
        }
    return out;
}
// ops.cpp:104-128: clamped-window mean through a summed-area table with a zero guard
vec box_mean(const double* img, int h, int w, int radius) {
    if (radius < 0) param_error("box_mean: negative radius");
    if (2 * radius + 1 > std::min(h, w)) dim_error("box_mean: window larger than image");
    if (radius == 0) return vec(img, img + static_cast<size_t>(h) * w);
    const size_t W1 = static_cast<size_t>(w) + 1;
    vec S((static_cast<size_t>(h) + 1) * W1, 0.0);
    for (int r = 1; r <= h; ++r)
        for (int c = 1; c <= w; ++c)
            S[r * W1 + c] = img[static_cast<size_t>(r - 1) * w + (c - 1)] + S[(r - 1) * W1 + c] + S[r * W1 + c - 1] -
                            S[(r - 1) * W1 + c - 1];
    vec out(static_cast<size_t>(h) * w);
    for (int r = 0; r < h; ++r) {
        const int r0 = std::max(0, r - radius), r1 = std::min(h - 1, r + radius);
        for (int c = 0; c < w; ++c) {
            const int c0 = std::max(0, c - radius), c1 = std::min(w - 1, c + radius);
            const double tot = S[(r1 + 1) * W1 + c1 + 1] - S[r0 * W1 + c1 + 1] - S[(r1 + 1) * W1 + c0] + S[r0 * W1 + c0];
            out[static_cast<size_t>(r) * w + c] = tot / ((r1 - r0 + 1) * (c1 - c0 + 1));
        }
    }
    return out;
}
// ops.cpp:130-155: separable circular box blur, taps at offsets [-lead, window-1-lead]
vec circular_box_blur(const double* img, int h, int w, int window) {
    if (window < 1) param_error("circular_box_blur: window must be >= 1");
    if (window > std::min(h, w)) dim_error("circular_box_blur: window larger than image");
    const int lead = (window - 1) / 2;
    const double gain = 1.0 / window;
    auto at = [&](const double* a, int r, int c) {
        r %= h; if (r < 0) r += h;
        c %= w; if (c < 0) c += w;
        return a[static_cast<size_t>(r) * w + c];
    };
    vec rows(static_cast<size_t>(h) * w), out(static_cast<size_t>(h) * w);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            double s = 0.0;
            for (int t = -lead; t < window - lead; ++t) s += at(img, r, c - t);
            rows[static_cast<size_t>(r) * w + c] = s * gain;
        }
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            double s = 0.0;
            for (int t = -lead; t < window - lead; ++t) s += at(rows.data(), r - t, c);
            out[static_cast<size_t>(r) * w + c] = s * gain;
        }
    return out;
}

// ---- pansharpen.cpp: matting matrix (117-202) ---------------------------------------------
struct Matting {
    int h = 0, w = 0, radius = 0;
    double eps = 0.0;
    vec mean, var;                 // window_mean_ / window_var_ (pansharpen.cpp:128-139)
    std::vector<int64_t> rowptr;   // CSR, columns ascending per row (Eigen RowMajor)
    std::vector<int64_t> col;
    vec val;

    static Matting build(const double* g, int h, int w, int radius, double eps) {
        if (radius < 1) param_error("matting matrix: radius must be >= 1");
        if (2 * radius + 1 > std::min(h, w)) dim_error("matting matrix: window larger than image");
        Matting M;
        M.h = h; M.w = w; M.radius = radius; M.eps = eps;
        const size_t P = static_cast<size_t>(h) * w;
        M.mean = box_mean(g, h, w, radius);
        {
            vec sq(g, g + P);
            for (size_t i = 0; i < P; ++i) sq[i] *= sq[i];
            vec m2 = box_mean(sq.data(), h, w, radius);
            M.var.resize(P);
            for (size_t i = 0; i < P; ++i) M.var[i] = m2[i] - M.mean[i] * M.mean[i];
        }
        const int band = 4 * radius + 1, nw = 2 * radius + 1;
        const double ws = static_cast<double>(nw) * nw;
        vec bands(P * band * band, 0.0);
        auto B = [&](int pr, int pc, int dr, int dc) -> double& {
            const size_t pix = static_cast<size_t>(pr) * w + pc;
            return bands[(pix * band + (dr + 2 * radius)) * band + (dc + 2 * radius)];
        };
        // interior centres only (pansharpen.cpp:152-153); eps/|w| + var (:155)
        for (int kr = radius; kr < h - radius; ++kr)
            for (int kc = radius; kc < w - radius; ++kc) {
                const double mu = M.mean[static_cast<size_t>(kr) * w + kc];
                const double den = eps / ws + M.var[static_cast<size_t>(kr) * w + kc];
                for (int mr = kr - radius; mr <= kr + radius; ++mr)
                    for (int mc = kc - radius; mc <= kc + radius; ++mc) {
                        const double im = g[static_cast<size_t>(mr) * w + mc] - mu;
                        for (int nr = kr - radius; nr <= kr + radius; ++nr)
                            for (int nc = kc - radius; nc <= kc + radius; ++nc) {
                                const double in = g[static_cast<size_t>(nr) * w + nc] - mu;
                                double v = -(1.0 + im * in / den) / ws;
                                if (mr == nr && mc == nc) v += 1.0;
                                B(mr, mc, nr - mr, nc - mc) += v;
                            }
                    }
            }
        // triplets in row order, columns ascending, exact zeros dropped (:176-193)
        M.rowptr.assign(P + 1, 0);
        M.col.reserve(P * band);
        M.val.reserve(P * band);
        for (int pr = 0; pr < h; ++pr)
            for (int pc = 0; pc < w; ++pc) {
                for (int dr = -2 * radius; dr <= 2 * radius; ++dr) {
                    const int nr = pr + dr;
                    if (nr < 0 || nr >= h) continue;
                    for (int dc = -2 * radius; dc <= 2 * radius; ++dc) {
                        const int nc = pc + dc;
                        if (nc < 0 || nc >= w) continue;
                        const double v = B(pr, pc, dr, dc);
                        if (v != 0.0) {
                            M.col.push_back(static_cast<int64_t>(nr) * w + nc);
                            M.val.push_back(v);
                        }
                    }
                }
                M.rowptr[static_cast<size_t>(pr) * w + pc + 1] = static_cast<int64_t>(M.col.size());
            }
        return M;
    }
    // pansharpen.cpp:197-202 (Eigen row-major SpMV: per-row running sum)
    vec apply(const double* x) const {
        const size_t P = static_cast<size_t>(h) * w;
        vec y(P);
        for (size_t r = 0; r < P; ++r) {
            double s = 0.0;
            for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) s += val[k] * x[col[k]];
            y[r] = s;
        }
        return y;
    }
};

struct PsParams {
    double lambda = 2e-4;
    int radius = 1;
    double eps = 1e-4;
    double cg_tol = 5e-5;
    int cg_max_iter = 2000;
    int threads = 0;
    int prior = 0;  // PriorKind: 0 laplacian, 1 identity (pansharpen.cpp:28-78)
};

// pansharpen.cpp:96-105 (laplacian and identity priors)
void validate(const PsParams& p) {
    if (!(p.lambda > 0)) param_error("pansharpen: lambda must be positive");
    if (p.radius < 1) param_error("pansharpen: radius must be >= 1");
    if (!(p.eps > 0)) param_error("pansharpen: eps must be positive");
    if (!(p.cg_tol > 0)) param_error("pansharpen: cg_tol must be positive");
    if (p.cg_max_iter < 1) param_error("pansharpen: cg_max_iter must be >= 1");
    if (p.threads < 0) param_error("pansharpen: threads must be >= 0");
}

std::string fmt_double(double v) { return std::to_string(v); }

// pansharpen.cpp:208-264
vec warmstart_cg(const double* x, int h, int w, const double* k, int n, int factor, const Matting& M,
                 const PsParams& prm, int max_iters, bool error_on_cap, double* final_residual, int* iters_out,
                 int* converged_out) {
    const int H = M.h, W = M.w;
    if (h * factor != H || w * factor != W) dim_error("warmstart: LR channel dimensions must be image/factor");
    const size_t P = static_cast<size_t>(H) * W;
    SpecConv conv(k, n, H, W);
    auto A = [&](const vec& z) {
        vec t = conv.apply(z.data(), false);
        vec d = downsample(t.data(), H, W, factor);
        vec u = upsample_adjoint(d.data(), h, w, factor);
        vec data = conv.apply(u.data(), true);
        // prior.apply_adjoint(M.apply(prior.apply(z))) (pansharpen.cpp:220-221): identity -> M z
        vec l1 = prm.prior == 1 ? z : laplacian(z.data(), H, W);
        vec m = M.apply(l1.data());
        vec l2 = prm.prior == 1 ? m : laplacian(m.data(), H, W);
        for (size_t i = 0; i < P; ++i) l2[i] *= prm.lambda;
        for (size_t i = 0; i < P; ++i) data[i] += l2[i];
        return data;
    };
    vec up = upsample_adjoint(x, h, w, factor);
    vec rhs = conv.apply(up.data(), true);
    const double rhs_norm = seq_norm(rhs.data(), P);
    vec z(P, 0.0);
    if (iters_out) *iters_out = 0;
    if (converged_out) *converged_out = 1;
    if (rhs_norm == 0.0) {
        if (final_residual) *final_residual = 0.0;
        return z;
    }
    vec r = rhs, p = r;
    double rs = seq_dot(r.data(), r.data(), P);
    bool converged = false;
    int it = 0;
    for (; it < max_iters; ++it) {
        vec Ap = A(p);
        const double pAp = seq_dot(p.data(), Ap.data(), P);
        if (!(pAp > 0)) {
            if (std::sqrt(rs) <= 1e-12 * rhs_norm) { converged = true; break; }
            num_error("warmstart: conjugate gradients hit a non-positive curvature direction");
        }
        const double alpha = rs / pAp;
        for (size_t i = 0; i < P; ++i) z[i] += p[i] * alpha;
        for (size_t i = 0; i < P; ++i) r[i] -= Ap[i] * alpha;
        const double step = std::abs(alpha) * seq_norm(p.data(), P);
        const double rs_new = seq_dot(r.data(), r.data(), P);
        if (trace_cg())  // FBMP_ORACLE_TRACE: the stop-test margin of every iteration (debugging aid)
            std::fprintf(stderr, "cg it %d step/(tol |z|) %.17g\n", it + 1,
                         step / (prm.cg_tol * std::max(seq_norm(z.data(), P), 1e-300)));
        if (step <= prm.cg_tol * std::max(seq_norm(z.data(), P), 1e-300)) { converged = true; break; }
        const double beta = rs_new / rs;
        for (size_t i = 0; i < P; ++i) p[i] = r[i] + p[i] * beta;
        rs = rs_new;
    }
    if (iters_out) *iters_out = converged ? it + 1 : it;
    if (converged_out) *converged_out = converged ? 1 : 0;
    vec Az = A(z);
    for (size_t i = 0; i < P; ++i) Az[i] -= rhs[i];
    const double resid = seq_norm(Az.data(), P);
    if (final_residual) *final_residual = resid;
    if (!converged && error_on_cap)
        num_error("warmstart: conjugate gradients did not converge in " + std::to_string(max_iters) +
                  " iterations (residual " + fmt_double(resid / rhs_norm) + " relative)");
    return z;
}

// pansharpen.cpp:274-302
void guided_coeffs(const double* in, const double* g, int h, int w, int radius, double eps, vec& a, vec& c,
                   vec& gmean, vec& gvar, vec& imean) {
    if (!(eps > 0)) param_error("guided_coeffs: eps must be positive");
    const size_t P = static_cast<size_t>(h) * w;
    vec gi(P), gg(P);
    for (size_t i = 0; i < P; ++i) {
        gi[i] = g[i] * in[i];
        gg[i] = g[i] * g[i];
    }
    gmean = box_mean(g, h, w, radius);
    imean = box_mean(in, h, w, radius);
    vec cgi = box_mean(gi.data(), h, w, radius);
    vec cgg = box_mean(gg.data(), h, w, radius);
    gvar.resize(P); a.resize(P); c.resize(P);
    for (size_t i = 0; i < P; ++i) {
        const double mu = gmean[i];
        const double var = cgg[i] - mu * mu;
        const double cov = cgi[i] - mu * imean[i];
        gvar[i] = var;
        a[i] = cov / (var + eps);
        c[i] = imean[i] - a[i] * mu;
    }
}
// pansharpen.cpp:304-312
vec guided_output(const double* a, const double* c, const double* g, int h, int w, int radius) {
    vec ab = box_mean(a, h, w, radius), cb = box_mean(c, h, w, radius);
    const size_t P = static_cast<size_t>(h) * w;
    vec out(P);
    for (size_t i = 0; i < P; ++i) out[i] = ab[i] * g[i] + cb[i];
    return out;
}

// Complex Hermitian eigen-decomposition (cyclic Jacobi), stands in for
// Eigen::SelfAdjointEigenSolver<MatrixXcd> at pansharpen.cpp:353. Eigenvalues ascending.
void herm_eig(int m, std::vector<cd>& A, vec& ev, std::vector<cd>& V) {
    V.assign(static_cast<size_t>(m) * m, 0.0);
    for (int i = 0; i < m; ++i) V[i * m + i] = 1.0;
    auto a = [&](int i, int j) -> cd& { return A[static_cast<size_t>(i) * m + j]; };
    double fro = 0.0;
    for (const cd& v : A) fro += std::norm(v);
    const double skip = 1e-18 * std::sqrt(fro);  // absolute accuracy ~ eps * ||A||, as Eigen's
    for (int sweep = 0; sweep < 60; ++sweep) {
        int rotations = 0;
        for (int p = 0; p < m; ++p)
            for (int q = p + 1; q < m; ++q) {
                const cd apq = a(p, q);
                const double mag = std::abs(apq);
                if (!(mag > skip)) continue;
                ++rotations;
                const double app = a(p, p).real(), aqq = a(q, q).real();
                const cd ph = apq / mag;  // a_pq = |a_pq| e^{i phi}
                const double theta = 0.5 * std::atan2(2.0 * mag, aqq - app);
                const double cs = std::cos(theta), sn = std::sin(theta);
                // rotation G with columns p,q: G_pp = c, G_pq = s*ph, G_qp = -s*conj(ph), G_qq = c
                for (int k = 0; k < m; ++k) {  // A <- A G
                    const cd akp = a(k, p), akq = a(k, q);
                    a(k, p) = cs * akp - sn * std::conj(ph) * akq;
                    a(k, q) = sn * ph * akp + cs * akq;
                }
                for (int k = 0; k < m; ++k) {  // A <- G^H A
                    const cd apk = a(p, k), aqk = a(q, k);
                    a(p, k) = cs * apk - sn * ph * aqk;
                    a(q, k) = sn * std::conj(ph) * apk + cs * aqk;
                }
                for (int k = 0; k < m; ++k) {  // V <- V G
                    const cd vkp = V[static_cast<size_t>(k) * m + p], vkq = V[static_cast<size_t>(k) * m + q];
                    V[static_cast<size_t>(k) * m + p] = cs * vkp - sn * std::conj(ph) * vkq;
                    V[static_cast<size_t>(k) * m + q] = sn * ph * vkp + cs * vkq;
                }
                a(p, q) = 0.0;
                a(q, p) = 0.0;
            }
        if (rotations == 0) break;
    }
    std::vector<int> order(m);
    std::iota(order.begin(), order.end(), 0);
    vec d(m);
    for (int i = 0; i < m; ++i) d[i] = a(i, i).real();
    std::sort(order.begin(), order.end(), [&](int x, int y) { return d[x] < d[y]; });
    ev.resize(m);
    std::vector<cd> V2(V.size());
    for (int j = 0; j < m; ++j) {
        ev[j] = d[order[j]];
        for (int k = 0; k < m; ++k) V2[static_cast<size_t>(k) * m + j] = V[static_cast<size_t>(k) * m + order[j]];
    }
    V.swap(V2);
}

// Complex Hermitian eigen-decomposition by Householder tridiagonalisation and implicit-shift
// QL iterations -- the algorithm of Eigen::SelfAdjointEigenSolver<MatrixXcd> used at
// pansharpen.cpp:353 (the Jacobi solver above is kept for the 3x3 rank test and as a cross-check
// in tests/test_oracle_kats.py). A = V diag(ev) V^H, eigenvalues ascending.
void herm_eig_ql(int n, std::vector<cd>& A, vec& ev, std::vector<cd>& V) {
    auto a = [&](int i, int j) -> cd& { return A[static_cast<size_t>(i) * n + j]; };
    std::vector<cd> Q(static_cast<size_t>(n) * n, 0.0), v(n), p(n), wv(n);
    for (int i = 0; i < n; ++i) Q[static_cast<size_t>(i) * n + i] = 1.0;
    for (int k = 0; k + 2 < n; ++k) {
        double sig = 0.0;
        for (int i = k + 2; i < n; ++i) sig += std::norm(a(i, k));
        if (sig == 0.0) continue;
        const cd x0 = a(k + 1, k);
        const double ax0 = std::abs(x0), xn = std::sqrt(ax0 * ax0 + sig);
        const cd alpha = (ax0 > 0.0 ? -x0 / ax0 : cd(-1.0, 0.0)) * xn;  // -e^{i arg x0} ||x||
        std::fill(v.begin(), v.end(), cd(0.0));
        v[k + 1] = x0 - alpha;
        for (int i = k + 2; i < n; ++i) v[i] = a(i, k);
        double vn = 0.0;
        for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
        const double beta = 2.0 / vn;
        // A <- H A H with H = I - beta v v^H:  p = beta A v, K = beta/2 v^H p, w = p - K v
        for (int i = k; i < n; ++i) {
            cd sacc = 0.0;
            for (int j = k + 1; j < n; ++j) sacc += a(i, j) * v[j];
            p[i] = beta * sacc;
        }
        cd K = 0.0;
        for (int i = k + 1; i < n; ++i) K += std::conj(v[i]) * p[i];
        K *= 0.5 * beta;
        for (int i = k; i < n; ++i) wv[i] = p[i] - K * v[i];
        for (int i = k; i < n; ++i)
            for (int j = k; j < n; ++j) a(i, j) -= v[i] * std::conj(wv[j]) + wv[i] * std::conj(v[j]);
        for (int r = 0; r < n; ++r) {  // Q <- Q H
            cd sacc = 0.0;
            for (int j = k + 1; j < n; ++j) sacc += Q[static_cast<size_t>(r) * n + j] * v[j];
            sacc *= beta;
            for (int j = k + 1; j < n; ++j) Q[static_cast<size_t>(r) * n + j] -= sacc * std::conj(v[j]);
        }
    }
    // T = Q^H A Q is tridiagonal; D = diag(ph) makes its sub-diagonal real: T = D T' D^H
    vec d(n), e(n, 0.0);
    std::vector<cd> ph(n, 1.0);
    for (int i = 0; i < n; ++i) d[i] = a(i, i).real();
    for (int i = 0; i + 1 < n; ++i) {
        const cd off = a(i + 1, i);
        const double m = std::abs(off);
        e[i] = m;
        ph[i + 1] = m > 0.0 ? ph[i] * (off / m) : ph[i];
    }
    // implicit-shift QL on the real tridiagonal T' (e[i] couples i and i+1), Z accumulates
    vec Z(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) Z[static_cast<size_t>(i) * n + i] = 1.0;
    const double eps = std::numeric_limits<double>::epsilon();
    for (int l = 0; l < n; ++l) {
        int iter = 0, m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= eps * dd) break;
            }
            if (m != l) {
                if (iter++ == 60) num_error("herm_eig_ql: no convergence");
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::hypot(g, 1.0);
                g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
                double sn = 1.0, cs = 1.0, pp = 0.0;
                int i;
                for (i = m - 1; i >= l; --i) {
                    double f = sn * e[i];
                    const double b = cs * e[i];
                    e[i + 1] = (r = std::hypot(f, g));
                    if (r == 0.0) {
                        d[i + 1] -= pp;
                        e[m] = 0.0;
                        break;
                    }
                    sn = f / r;
                    cs = g / r;
                    g = d[i + 1] - pp;
                    r = (d[i] - g) * sn + 2.0 * cs * b;
                    d[i + 1] = g + (pp = sn * r);
                    g = cs * r - b;
                    for (int k = 0; k < n; ++k) {
                        f = Z[static_cast<size_t>(k) * n + i + 1];
                        Z[static_cast<size_t>(k) * n + i + 1] = sn * Z[static_cast<size_t>(k) * n + i] + cs * f;
                        Z[static_cast<size_t>(k) * n + i] = cs * Z[static_cast<size_t>(k) * n + i] - sn * f;
                    }
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= pp;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return d[x] < d[y]; });
    ev.resize(n);
    V.assign(static_cast<size_t>(n) * n, 0.0);
    for (int j = 0; j < n; ++j) {
        const int oj = order[j];
        ev[j] = d[oj];
        for (int r = 0; r < n; ++r) {
            cd sacc = 0.0;
            for (int k = 0; k < n; ++k)
                sacc += Q[static_cast<size_t>(r) * n + k] * ph[k] * Z[static_cast<size_t>(k) * n + oj];
            V[static_cast<size_t>(r) * n + j] = sacc;
        }
    }
}

// pansharpen.cpp:56-63 (laplacian transfer function)
std::vector<cd> lap_spectrum(int rows, int cols) {
    std::vector<cd> s(static_cast<size_t>(rows) * cols);
    for (int r = 0; r < rows; ++r) {
        const double cv = std::cos(2.0 * kPi * r / rows);
        for (int c = 0; c < cols; ++c) {
            const double ch = std::cos(2.0 * kPi * c / cols);
            s[static_cast<size_t>(r) * cols + c] = 4.0 - 2.0 * cv - 2.0 * ch;
        }
    }
    return s;
}

// pansharpen.cpp:314-365
// (bench sampling only: rows_limit > 0 solves the alias groups of LR rows [0, rows_limit) and
// t_groups receives the seconds spent in the group loop)
vec solve_channel_fft(const double* x, int h, int w, const double* k, int n, int factor, const double* v, int H, int W,
                      const PsParams& prm, int rows_limit = 0, double* t_groups = nullptr) {
    validate(prm);
    if (h * factor != H || w * factor != W)
        dim_error("solve_channel_fft: LR/HR dimensions inconsistent with factor");
    const int c2 = factor * factor;
    const double lambda = prm.lambda;
    Fft2 fhr(H, W), flr(h, w);
    vec e = embed_kernel(k, n, H, W);
    cvec bhat = fhr.forward(e.data());
    cvec lhat = prm.prior == 1 ? cvec(static_cast<size_t>(H) * W, cd(1.0)) : lap_spectrum(H, W);  // :53-70
    cvec xhat = flr.forward(x);
    cvec vhat = fhr.forward(v);
    cvec zhat(bhat.size());
    std::vector<cd> A(static_cast<size_t>(c2) * c2), V;
    std::vector<cd> rhs(c2), bg(c2), tmp(c2);
    std::vector<size_t> idx(c2);
    vec ev;
    const auto tg0 = std::chrono::steady_clock::now();
    const int kl_end = rows_limit > 0 ? std::min(rows_limit, h) : h;
    for (int kl = 0; kl < kl_end; ++kl)
        for (int ll = 0; ll < w; ++ll) {
            for (int a = 0; a < factor; ++a)
                for (int b = 0; b < factor; ++b)
                    idx[static_cast<size_t>(a) * factor + b] = static_cast<size_t>(kl + a * h) * W + (ll + b * w);
            for (int g = 0; g < c2; ++g) bg[g] = bhat[idx[g]];
            const cd xg = xhat[static_cast<size_t>(kl) * w + ll];
            for (int g = 0; g < c2; ++g) {
                for (int gp = 0; gp < c2; ++gp) A[static_cast<size_t>(g) * c2 + gp] = std::conj(bg[g]) * bg[gp] / static_cast<double>(c2);
                A[static_cast<size_t>(g) * c2 + g] += lambda * std::norm(lhat[idx[g]]);
                rhs[g] = std::conj(bg[g]) * xg + lambda * std::conj(lhat[idx[g]]) * vhat[idx[g]];
            }
            herm_eig_ql(c2, A, ev, V);
            if (!(ev[0] > 0.0) || ev[c2 - 1] > 1e14 * ev[0])
                num_error("solve_channel_fft: alias-group system condition number exceeds 1e14 (prior transfer "
                          "function too small)");
            for (int j = 0; j < c2; ++j) {
                cd s = 0.0;
                for (int g = 0; g < c2; ++g) s += std::conj(V[static_cast<size_t>(g) * c2 + j]) * rhs[g];
                tmp[j] = s / ev[j];
            }
            for (int g = 0; g < c2; ++g) {
                cd s = 0.0;
                for (int j = 0; j < c2; ++j) s += V[static_cast<size_t>(g) * c2 + j] * tmp[j];
                zhat[idx[g]] = s;
            }
        }
    if (t_groups) t_groups[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - tg0).count();
    return fhr.backward_real(std::move(zhat));
}

// pansharpen.cpp:80-92
template <class F>
void annotate(int ch, F&& f) {
    try {
        f();
    } catch (const Failure& e) {
        throw Failure(e.code, "channel " + std::to_string(ch) + ": " + e.what());
    }
}

// pansharpen.cpp:367-424
std::vector<vec> pansharpen(const double* lrms, int N, int h, int w, const double* pan, const double* k, int n,
                            int factor, const PsParams& prm, std::vector<int>* cg_iters) {
    validate(prm);
    const int H = h * factor, W = w * factor;
    const size_t P = static_cast<size_t>(H) * W, p = static_cast<size_t>(h) * w;
    double peak = seq_max(pan, P);
    for (int b = 0; b < N; ++b) peak = std::max(peak, seq_max(lrms + b * p, p));
    const double scale = peak > 0.0 ? 1.0 / peak : 1.0;
    vec pan_n(P);
    for (size_t i = 0; i < P; ++i) pan_n[i] = pan[i] * scale;
    vec lpan = prm.prior == 1 ? pan_n : laplacian(pan_n.data(), H, W);  // prior.apply(pan_n)
    const Matting M = Matting::build(lpan.data(), H, W, prm.radius, prm.eps);
    std::vector<vec> out(N);
    std::vector<std::exception_ptr> errors(N);
    std::vector<int> iters(N, 0);
    std::atomic<int> next{0};
    auto worker = [&]() {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= N) return;
            try {
                annotate(i, [&] {
                    vec xn(p);
                    for (size_t j = 0; j < p; ++j) xn[j] = lrms[i * p + j] * scale;
                    validate(prm);  // warmstart_channel (pansharpen.cpp:266-272)
                    int it = 0, conv = 0;
                    vec z0 = warmstart_cg(xn.data(), h, w, k, n, factor, M, prm, prm.cg_max_iter, true, nullptr, &it,
                                          &conv);
                    iters[i] = it;
                    vec lz = prm.prior == 1 ? z0 : laplacian(z0.data(), H, W);  // ch_prior.apply(z0)
                    vec a, c, gm, gv, im;
                    guided_coeffs(lz.data(), lpan.data(), H, W, prm.radius, prm.eps, a, c, gm, gv, im);
                    vec v = guided_output(a.data(), c.data(), lpan.data(), H, W, prm.radius);
                    vec z = solve_channel_fft(xn.data(), h, w, k, n, factor, v.data(), H, W, prm);
                    const double inv = 1.0 / scale;
                    for (size_t j = 0; j < P; ++j) z[j] *= inv;
                    out[i] = std::move(z);
                });
            } catch (...) {
                errors[i] = std::current_exception();
                return;
            }
        }
    };
    int nt = prm.threads > 0 ? prm.threads : static_cast<int>(std::thread::hardware_concurrency());
    nt = std::clamp(nt, 1, N);
    if (nt == 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
    }
    for (int i = 0; i < N; ++i)
        if (errors[i]) std::rethrow_exception(errors[i]);
    if (cg_iters) *cg_iters = iters;
    return out;
}

// ---- spectral_weights.cpp:9-65 -----------------------------------------------------------
// Gauss-Jordan with full pivoting stands in for Eigen::FullPivLU (rank + solve).
int fullpiv_solve(int n, vec A, vec b, vec& x) {
    std::vector<int> colperm(n);
    std::iota(colperm.begin(), colperm.end(), 0);
    double maxpiv = 0.0;
    int rank = 0;
    for (int k = 0; k < n; ++k) {
        int pr = k, pc = k;
        double best = -1.0;
        for (int i = k; i < n; ++i)
            for (int j = k; j < n; ++j)
                if (std::abs(A[i * n + j]) > best) { best = std::abs(A[i * n + j]); pr = i; pc = j; }
        if (k == 0) maxpiv = best;
        // Eigen's default threshold: |pivot| <= eps * n * max|pivot| counts as zero
        if (best <= maxpiv * 2.220446049250313e-16 * n || best == 0.0) break;
        ++rank;
        if (pr != k) { for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[pr * n + j]); std::swap(b[k], b[pr]); }
        if (pc != k) { for (int i = 0; i < n; ++i) std::swap(A[i * n + k], A[i * n + pc]); std::swap(colperm[k], colperm[pc]); }
        for (int i = k + 1; i < n; ++i) {
            const double f = A[i * n + k] / A[k * n + k];
            for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
            b[i] -= f * b[k];
        }
    }
    if (rank < n) return rank;
    vec y(n);
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < n; ++j) s -= A[i * n + j] * y[j];
        y[i] = s / A[i * n + i];
    }
    x.assign(n, 0.0);
    for (int i = 0; i < n; ++i) x[colperm[i]] = y[i];
    return rank;
}

vec solve_weights(const double* lrms, int nb, int h, int w, const double* pan, int H, int W, int l, double lambda_omega,
                  int c) {
    if (c < 1) param_error("solve_weights: factor must be >= 1");
    if (l < 1) param_error("solve_weights: l must be >= 1");
    if (lambda_omega < 0.0) param_error("solve_weights: lambda_omega must be >= 0");
    if (H != c * h || W != c * w) dim_error("solve_weights: PAN dimensions must be factor times the LRMS dimensions");
    const size_t m = static_cast<size_t>(h) * w;
    std::vector<vec> A(nb);
    for (int i = 0; i < nb; ++i) A[i] = circular_box_blur(lrms + i * m, h, w, l + 1);
    vec hb = circular_box_blur(pan, H, W, c * l + 1);
    vec bvec = downsample(hb.data(), H, W, c);
    vec normal(static_cast<size_t>(nb) * nb), rhs(nb);
    for (int i = 0; i < nb; ++i) {
        for (int j = 0; j < nb; ++j) normal[i * nb + j] = seq_dot(A[i].data(), A[j].data(), m);
        rhs[i] = seq_dot(A[i].data(), bvec.data(), m);
    }
    if (nb > 1)
        for (int i = 0; i < nb; ++i)  // lambda * G^T G, G = first differences
            for (int j = 0; j < nb; ++j) {
                double g = 0.0;
                for (int r = 0; r < nb - 1; ++r) {
                    const double gri = (i == r) ? -1.0 : (i == r + 1 ? 1.0 : 0.0);
                    const double grj = (j == r) ? -1.0 : (j == r + 1 ? 1.0 : 0.0);
                    g += gri * grj;
                }
                normal[i * nb + j] += lambda_omega * g;
            }
    vec omega;
    if (fullpiv_solve(nb, normal, rhs, omega) < nb)
        num_error("solve_weights: normal matrix is singular (bands linearly dependent and lambda_omega too small)");
    double r2 = 0.0;
    for (int i = 0; i < nb; ++i) {
        double s = 0.0;
        for (int j = 0; j < nb; ++j) s += normal[i * nb + j] * omega[j];
        r2 += (s - rhs[i]) * (s - rhs[i]);
    }
    if (!(std::sqrt(r2) <= 1e-8 * seq_norm(rhs.data(), nb) + 1e-12))
        num_error("solve_weights: stationarity residual too large (ill-conditioned system)");
    return omega;
}

vec combine_bands(const double* lrms, int nb, size_t m, const double* omega) {
    vec out(m, 0.0);
    for (int i = 0; i < nb; ++i)
        for (size_t j = 0; j < m; ++j) out[j] += omega[i] * lrms[i * m + j];
    return out;
}

// ---- kernel_estimator.cpp ------------------------------------------------------------------
struct KeParams {
    int n = 29;
    double alpha1 = 1.0, alpha2 = 0.006, mu1 = 100.0, mu2 = 100.0, mu3 = 100.0, rho = 0.5;
    int t_max = 10000;
    double th = 1e-5;
    int init = 0;  // 0 dirac, 1 uniform
    bool with_p = true;  // run_tgv_or_tv's branch: true = TGV^2, false = TV (no p, no y-step)
};

void validate(const KeParams& p) {  // kernel_estimator.cpp:36-45
    if (p.n < 1 || p.n % 2 == 0) param_error("kernel estimation: n must be odd and positive");
    if (p.alpha1 <= 0 || p.alpha2 <= 0) param_error("kernel estimation: alpha weights must be positive");
    if (p.mu1 <= 0 || p.mu2 <= 0 || p.mu3 <= 0) param_error("kernel estimation: mu penalties must be positive");
    const double rho_max = (1.0 + std::sqrt(5.0)) / 2.0;
    if (!(p.rho > 0 && p.rho < rho_max)) param_error("kernel estimation: rho must lie in (0, (1+sqrt(5))/2)");
    if (!(p.th > 0)) param_error("kernel estimation: th must be positive");
    if (p.t_max < 1) param_error("kernel estimation: t_max must be >= 1");
}

// kernel_estimator.cpp:47-83: E (p x n^2), E^T f, E^T E, LLT of E^T E + mu3 I
struct Observation {
    int n = 0;
    double mu3 = 0.0;
    vec Etf, EtE, L;  // L: lower Cholesky factor, row-major n2 x n2
    vec E, f;         // kept for objective evaluation

    Observation(const double* pan, int H, int W, const double* obs, int h, int w, int factor, int n_, double mu3_)
        : n(n_), mu3(mu3_) {
        if (n < 1 || n % 2 == 0) param_error("build_observation: kernel side must be odd");
        if (factor < 1) param_error("build_observation: factor must be >= 1");
        if (H != factor * h || W != factor * w) dim_error("build_observation: PAN dimensions must be factor times the observation");
        if (n > std::min(H, W)) dim_error("build_observation: kernel larger than PAN image");
        const int C = (n - 1) / 2;
        const size_t n2 = static_cast<size_t>(n) * n, p = static_cast<size_t>(h) * w;
        E.resize(p * n2);
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j)
                for (int tr = 0; tr < n; ++tr)
                    for (int tc = 0; tc < n; ++tc) {
                        int rr = (factor * i - (tr - C)) % H; if (rr < 0) rr += H;
                        int cc = (factor * j - (tc - C)) % W; if (cc < 0) cc += W;
                        E[(static_cast<size_t>(i) * w + j) * n2 + tr * n + tc] = pan[static_cast<size_t>(rr) * W + cc];
                    }
        f.assign(obs, obs + p);
        Etf.assign(n2, 0.0);
        EtE.assign(n2 * n2, 0.0);
        for (size_t r = 0; r < p; ++r) {
            const double* e = &E[r * n2];
            for (size_t a = 0; a < n2; ++a) {
                Etf[a] += e[a] * f[r];
                const double ea = e[a];
                double* row = &EtE[a * n2];
                for (size_t b = a; b < n2; ++b) row[b] += ea * e[b];
            }
        }
        for (size_t a = 0; a < n2; ++a)
            for (size_t b = 0; b < a; ++b) EtE[a * n2 + b] = EtE[b * n2 + a];
        L.assign(n2 * n2, 0.0);
        for (size_t j = 0; j < n2; ++j) {
            double d = EtE[j * n2 + j] + mu3;
            for (size_t k = 0; k < j; ++k) d -= L[j * n2 + k] * L[j * n2 + k];
            if (!(d > 0)) num_error("build_observation: factorization of E^T E + mu3 I failed");
            const double ljj = std::sqrt(d);
            L[j * n2 + j] = ljj;
            for (size_t i = j + 1; i < n2; ++i) {
                double s = EtE[i * n2 + j];
                for (size_t k = 0; k < j; ++k) s -= L[i * n2 + k] * L[j * n2 + k];
                L[i * n2 + j] = s / ljj;
            }
        }
    }
    vec solve_z(const double* anchor) const {  // :79-83
        const size_t n2 = static_cast<size_t>(n) * n;
        vec b(n2), y(n2), x(n2);
        for (size_t i = 0; i < n2; ++i) b[i] = Etf[i] + mu3 * anchor[i];
        for (size_t i = 0; i < n2; ++i) {
            double s = b[i];
            for (size_t k = 0; k < i; ++k) s -= L[i * n2 + k] * y[k];
            y[i] = s / L[i * n2 + i];
        }
        for (size_t ii = n2; ii-- > 0;) {
            double s = y[ii];
            for (size_t k = ii + 1; k < n2; ++k) s -= L[k * n2 + ii] * x[k];
            x[ii] = s / L[ii * n2 + ii];
        }
        return x;
    }
    double data_objective(const double* u) const {  // :85-87
        const size_t n2 = static_cast<size_t>(n) * n, p = f.size();
        double s = 0.0;
        for (size_t r = 0; r < p; ++r) {
            double e = -f[r];
            for (size_t a = 0; a < n2; ++a) e += E[r * n2 + a] * u[a];
            s += e * e;
        }
        return 0.5 * s;
    }
};

// kernel_estimator.cpp:94-110
void shrink2(std::vector<vec*> cols, double t) {
    if (t < 0) param_error("shrink2: threshold must be non-negative");
    if (cols.empty()) return;
    const size_t m = cols[0]->size();
    for (size_t i = 0; i < m; ++i) {
        double n2 = 0.0;
        for (vec* c : cols) n2 += (*c)[i] * (*c)[i];
        const double nrm = std::sqrt(n2);
        const double sc = nrm > t ? (nrm - t) / nrm : 0.0;
        for (vec* c : cols) (*c)[i] *= sc;
    }
}

// kernel_estimator.cpp:112-128
vec project_simplex(const double* v, size_t n) {
    vec u(v, v + n);
    std::sort(u.begin(), u.end(), std::greater<>());
    double css = 0.0, tau = 0.0;
    int support = 0;
    for (size_t j = 0; j < n; ++j) {
        css += u[j];
        const double cand = (1.0 - css) / static_cast<double>(j + 1);
        if (u[j] + cand > 0.0) { tau = cand; support = static_cast<int>(j + 1); }
    }
    if (support == 0) num_error("project_simplex: empty support (non-finite input?)");
    vec out(n);
    for (size_t i = 0; i < n; ++i) out[i] = std::max(v[i] + tau, 0.0);
    return out;
}

// 3x3 complex minimum-norm solve for the rank-deficient DC bin (kernel_estimator.cpp:213-225,
// Eigen COD); only reachable through the public solve_up (coupling = 0). Computed through the
// Hermitian eigen-decomposition with a relative rank threshold.
void minnorm3(const cd A[9], const cd b[3], cd x[3]) {
    std::vector<cd> M(A, A + 9), V;
    vec ev;
    herm_eig(3, M, ev, V);
    const double tol = 1e-12 * std::max(std::abs(ev[0]), std::abs(ev[2]));
    for (int i = 0; i < 3; ++i) x[i] = 0.0;
    for (int j = 0; j < 3; ++j) {
        if (std::abs(ev[j]) <= tol) continue;
        cd s = 0.0;
        for (int g = 0; g < 3; ++g) s += std::conj(V[g * 3 + j]) * b[g];
        s /= ev[j];
        for (int g = 0; g < 3; ++g) x[g] += V[g * 3 + j] * s;
    }
}

struct Up { vec u, p1, p2; };

// kernel_estimator.cpp:137-233
Up solve_up_core(const vec x[2], const vec y[4], const vec L1[2], const vec L2[4], const KeParams& prm, int n,
                 double coupling, const vec* anchor) {
    const size_t m = static_cast<size_t>(n) * n;
    const double a1m1 = prm.alpha1 * prm.mu1, a2m2 = prm.alpha2 * prm.mu2;
    vec x1(m), x2(m), y1(m), y2(m), yc(m);
    for (size_t i = 0; i < m; ++i) {
        x1[i] = x[0][i] - L1[0][i];
        x2[i] = x[1][i] - L1[1][i];
        y1[i] = y[0][i] - L2[0][i];
        y2[i] = y[3][i] - L2[3][i];
        yc[i] = (((y[1][i] - L2[1][i]) + y[2][i]) - L2[2][i]) * 0.5;  // Plane ops evaluate left to right
    }
    vec g1 = diff(x1.data(), n, n, GH, true), g2 = diff(x2.data(), n, n, GV, true);
    vec h1 = diff(y1.data(), n, n, GH, true), h2 = diff(yc.data(), n, n, GV, true);
    vec k1 = diff(y2.data(), n, n, GV, true), k2 = diff(yc.data(), n, n, GH, true);
    vec B1(m), B2(m), B3(m);
    for (size_t i = 0; i < m; ++i) {
        B1[i] = (g1[i] + g2[i]) * a1m1;
        B2[i] = (x1[i] * -a1m1) + (h1[i] + h2[i]) * a2m2;
        B3[i] = (x2[i] * -a1m1) + (k1[i] + k2[i]) * a2m2;
    }
    if (coupling > 0.0 && anchor)
        for (size_t i = 0; i < m; ++i) B1[i] += (*anchor)[i] * coupling;
    Fft2 fft(n, n);
    cvec F1 = fft.forward(B1.data()), F2 = fft.forward(B2.data()), F3 = fft.forward(B3.data());
    cvec FU(m), FP1(m), FP2(m), d4(m), d5(m), d6(m), den(m);
    vec d1(m), d2(m), d3(m);
    double maxden = 0.0;
    for (int r = 0; r < n; ++r) {
        const double wv = 2.0 * kPi * r / n;
        const cd dv = cd(std::cos(wv), std::sin(wv)) - 1.0;
        const double av2 = std::norm(dv);
        for (int c = 0; c < n; ++c) {
            const double wh = 2.0 * kPi * c / n;
            const cd dh = cd(std::cos(wh), std::sin(wh)) - 1.0;
            const double ah2 = std::norm(dh);
            const size_t i = static_cast<size_t>(r) * n + c;
            d1[i] = a1m1 * (ah2 + av2) + coupling;
            d2[i] = a1m1 + 0.5 * a2m2 * av2 + a2m2 * ah2;
            d3[i] = a1m1 + 0.5 * a2m2 * ah2 + a2m2 * av2;
            d4[i] = -a1m1 * dh;
            d5[i] = -a1m1 * dv;
            d6[i] = 0.5 * a2m2 * std::conj(dh) * dv;
            den[i] = d1[i] * (d2[i] * d3[i] - std::norm(d6[i])) - std::conj(d4[i]) * (d4[i] * d3[i] - std::conj(d6[i]) * d5[i]) +
                     std::conj(d5[i]) * (d4[i] * d6[i] - cd(d2[i]) * d5[i]);
            maxden = std::max(maxden, std::abs(den[i]));
        }
    }
    const double tol = 1e-12 * maxden;
    for (size_t i = 0; i < m; ++i) {
        const cd b1 = F1[i], b2 = F2[i], b3 = F3[i];
        if (std::abs(den[i]) > tol) {
            const cd nu = b1 * (d2[i] * d3[i] - std::norm(d6[i])) - std::conj(d4[i]) * (b2 * d3[i] - std::conj(d6[i]) * b3) +
                          std::conj(d5[i]) * (b2 * d6[i] - cd(d2[i]) * b3);
            const cd np1 = cd(d1[i]) * (b2 * d3[i] - std::conj(d6[i]) * b3) - b1 * (d4[i] * d3[i] - std::conj(d6[i]) * d5[i]) +
                           std::conj(d5[i]) * (d4[i] * b3 - b2 * d5[i]);
            const cd np2 = cd(d1[i]) * (cd(d2[i]) * b3 - d6[i] * b2) - std::conj(d4[i]) * (d4[i] * b3 - b2 * d5[i]) +
                           b1 * (d4[i] * d6[i] - cd(d2[i]) * d5[i]);
            FU[i] = nu / den[i];
            FP1[i] = np1 / den[i];
            FP2[i] = np2 / den[i];
        } else {
            const cd A[9] = {cd(d1[i]), std::conj(d4[i]), std::conj(d5[i]), d4[i], cd(d2[i]), std::conj(d6[i]),
                             d5[i], d6[i], cd(d3[i])};
            const cd b[3] = {b1, b2, b3};
            cd s[3];
            minnorm3(A, b, s);
            FU[i] = s[0]; FP1[i] = s[1]; FP2[i] = s[2];
        }
    }
    Up out;
    out.u = fft.backward_real(std::move(FU));
    out.p1 = fft.backward_real(std::move(FP1));
    out.p2 = fft.backward_real(std::move(FP2));
    return out;
}

void check_finite(const vec& p, const char* what, int t) {  // kernel_estimator.cpp:28-32
    for (double v : p)
        if (!std::isfinite(v))
            num_error(std::string("kernel estimation diverged: non-finite ") + what + " at iteration " + std::to_string(t));
}

// kernel_estimator.cpp:283-289
double intensity_scale(const double* pan, int H, int W, int factor) {
    double m = 0.0;
    for (size_t i = 0; i < static_cast<size_t>(H) * W; ++i) m = std::max(m, std::abs(pan[i]));
    if (m <= 0.0) num_error("kernel estimation: PAN image is identically zero");
    const double hw = static_cast<double>(H / factor) * (W / factor);
    return std::sqrt(16384.0 / hw) / m;
}

struct AdmmState {  // kernel_estimator.hpp:85-94 (u,p1,p2,x[2],y[4],z,L1[2],L2[4],L3)
    vec f[17];
    int iterations = 0;
};

// kernel_estimator.cpp:269-276, 438-455, 291-387 (TGV^2 branch, with_p = true; TV branch,
// with_p = false: no y-step, u from the scalar symbol d1 of :309-321 / :356-364)
thread_local std::chrono::steady_clock::time_point* g_setup_mark = nullptr;
vec estimate_kernel_plane_tgv(const double* pan, int H, int W, const double* obs, int h, int w, int factor,
                              const KeParams& prm, int* iters_out, AdmmState* final_state, int t_stop_hook = -1) {
    validate(prm);
    const size_t P = static_cast<size_t>(H) * W;
    double mean = 0.0;
    for (size_t i = 0; i < P; ++i) mean += pan[i];
    mean = P ? mean / static_cast<double>(P) : 0.0;
    double dev = 0.0;
    for (size_t i = 0; i < P; ++i) dev = std::max(dev, std::abs(pan[i] - mean));
    if (dev <= 1e-12 * std::max(1.0, std::abs(mean)))
        num_error("kernel estimation: constant PAN image is unidentifiable (E^T E has rank 1)");
    const double s = intensity_scale(pan, H, W, factor);
    vec pan_n(P), obs_n(static_cast<size_t>(h) * w);
    for (size_t i = 0; i < P; ++i) pan_n[i] = pan[i] * s;
    for (size_t i = 0; i < obs_n.size(); ++i) obs_n[i] = obs[i] * s;
    const int n = prm.n;
    const size_t m = static_cast<size_t>(n) * n;
    const Observation O(pan_n.data(), H, W, obs_n.data(), h, w, factor, n, prm.mu3);
    if (g_setup_mark) *g_setup_mark = std::chrono::steady_clock::now();  // bench sampling only

    vec u(m, 0.0);
    if (prm.init == 0) u[static_cast<size_t>((n - 1) / 2) * n + (n - 1) / 2] = 1.0;
    else std::fill(u.begin(), u.end(), 1.0 / (static_cast<double>(n) * n));
    vec z = u, p1(m, 0.0), p2(m, 0.0);
    vec x[2] = {diff(u.data(), n, n, GH, false), diff(u.data(), n, n, GV, false)};
    vec y[4] = {vec(m, 0.0), vec(m, 0.0), vec(m, 0.0), vec(m, 0.0)};
    vec L1[2] = {vec(m, 0.0), vec(m, 0.0)};
    vec L2[4] = {vec(m, 0.0), vec(m, 0.0), vec(m, 0.0), vec(m, 0.0)};
    vec L3(m, 0.0);
    int iters = 0;
    auto symgrad = [&](const vec& a, const vec& b, vec out[4]) {  // :264-267
        vec gv = diff(a.data(), n, n, GV, false), gh = diff(b.data(), n, n, GH, false);
        vec cross(m);
        for (size_t i = 0; i < m; ++i) cross[i] = (gv[i] + gh[i]) * 0.5;
        out[0] = diff(a.data(), n, n, GH, false);
        out[1] = cross;
        out[2] = cross;
        out[3] = diff(b.data(), n, n, GV, false);
    };
    for (int t = 0; t < prm.t_max; ++t) {
        {  // x-step
            vec gh = diff(u.data(), n, n, GH, false), gv = diff(u.data(), n, n, GV, false);
            for (size_t i = 0; i < m; ++i) {
                gh[i] = gh[i] - p1[i] + L1[0][i];
                gv[i] = gv[i] - p2[i] + L1[1][i];
            }
            shrink2({&gh, &gv}, 1.0 / prm.mu1);
            x[0] = std::move(gh);
            x[1] = std::move(gv);
        }
        if (prm.with_p) {  // y-step
            vec ep[4];
            symgrad(p1, p2, ep);
            for (int j = 0; j < 4; ++j)
                for (size_t i = 0; i < m; ++i) ep[j][i] = ep[j][i] + L2[j][i];
            shrink2({&ep[0], &ep[1], &ep[2], &ep[3]}, 1.0 / prm.mu2);
            for (int j = 0; j < 4; ++j) y[j] = std::move(ep[j]);
        }
        {  // z-step
            vec anc(m);
            for (size_t i = 0; i < m; ++i) anc[i] = u[i] + L3[i];
            vec zz = O.solve_z(anc.data());
            z = project_simplex(zz.data(), m);
        }
        if (t == t_stop_hook && final_state) {  // debug: state right before the {u,p} solve
            vec* dst = final_state->f;
            dst[0] = u; dst[1] = p1; dst[2] = p2; dst[3] = x[0]; dst[4] = x[1];
            for (int j = 0; j < 4; ++j) dst[5 + j] = y[j];
            dst[9] = z; dst[10] = L1[0]; dst[11] = L1[1];
            for (int j = 0; j < 4; ++j) dst[12 + j] = L2[j];
            dst[16] = L3;
            final_state->iterations = t;
            if (iters_out) *iters_out = t;
            return z;
        }
        vec anchor(m);
        for (size_t i = 0; i < m; ++i) anchor[i] = z[i] - L3[i];
        Up sol;
        if (prm.with_p) {
            sol = solve_up_core(x, y, L1, L2, prm, n, prm.mu3, &anchor);
            p1 = std::move(sol.p1);
            p2 = std::move(sol.p2);
        } else {  // kernel_estimator.cpp:356-364
            const double a1m1 = prm.alpha1 * prm.mu1;
            vec x1(m), x2(m);
            for (size_t i = 0; i < m; ++i) {
                x1[i] = x[0][i] - L1[0][i];
                x2[i] = x[1][i] - L1[1][i];
            }
            vec g1 = diff(x1.data(), n, n, GH, true), g2 = diff(x2.data(), n, n, GV, true);
            vec B1(m);
            for (size_t i = 0; i < m; ++i) B1[i] = (g1[i] + g2[i]) * a1m1 + anchor[i] * prm.mu3;
            Fft2 fft(n, n);
            cvec FB = fft.forward(B1.data());
            for (int r = 0; r < n; ++r) {  // :309-321
                const double av2 = 2.0 - 2.0 * std::cos(2.0 * M_PI * r / n);
                for (int c = 0; c < n; ++c) {
                    const double ah2 = 2.0 - 2.0 * std::cos(2.0 * M_PI * c / n);
                    FB[static_cast<size_t>(r) * n + c] /= prm.alpha1 * prm.mu1 * (ah2 + av2) + prm.mu3;
                }
            }
            sol.u = fft.backward_real(std::move(FB));
        }
        vec& un = sol.u;
        {  // multipliers
            vec gh = diff(un.data(), n, n, GH, false), gv = diff(un.data(), n, n, GV, false);
            for (size_t i = 0; i < m; ++i) {
                L1[0][i] += (gh[i] - p1[i] - x[0][i]) * prm.rho;
                L1[1][i] += (gv[i] - p2[i] - x[1][i]) * prm.rho;
            }
            if (prm.with_p) {
                vec ep[4];
                symgrad(p1, p2, ep);
                for (int j = 0; j < 4; ++j)
                    for (size_t i = 0; i < m; ++i) L2[j][i] += (ep[j][i] - y[j][i]) * prm.rho;
            }
            for (size_t i = 0; i < m; ++i) L3[i] += (un[i] - z[i]) * prm.rho;
        }
        vec du(m);
        for (size_t i = 0; i < m; ++i) du[i] = u[i] - un[i];
        const double delta = seq_norm(du.data(), m);
        const double scale = std::max(seq_norm(un.data(), m), 1e-300);
        u = std::move(un);
        iters = t + 1;
        check_finite(u, "u", t);
        check_finite(z, "z", t);
        if (delta / scale < prm.th) break;
    }
    if (final_state) {
        vec* dst = final_state->f;
        dst[0] = u; dst[1] = p1; dst[2] = p2; dst[3] = x[0]; dst[4] = x[1];
        for (int j = 0; j < 4; ++j) dst[5 + j] = y[j];
        dst[9] = z; dst[10] = L1[0]; dst[11] = L1[1];
        for (int j = 0; j < 4; ++j) dst[12 + j] = L2[j];
        dst[16] = L3;
        final_state->iterations = iters;
    }
    if (iters_out) *iters_out = iters;
    return z;
}

// kernel_estimator.cpp:243-260
double tgv_objective(const Observation& O, const double* u, const double* p1, const double* p2, const KeParams& prm) {
    const int n = O.n;
    const size_t m = static_cast<size_t>(n) * n;
    const double data = O.data_objective(u);
    vec gh = diff(u, n, n, GH, false), gv = diff(u, n, n, GV, false);
    double tgv1 = 0.0;
    for (size_t i = 0; i < m; ++i) tgv1 += std::hypot(gh[i] - p1[i], gv[i] - p2[i]);
    vec e1 = diff(p1, n, n, GH, false), e4 = diff(p2, n, n, GV, false);
    vec a = diff(p1, n, n, GV, false), b = diff(p2, n, n, GH, false);
    double tgv2 = 0.0;
    for (size_t i = 0; i < m; ++i) {
        const double c = (a[i] + b[i]) * 0.5;
        tgv2 += std::sqrt(e1[i] * e1[i] + e4[i] * e4[i] + 2.0 * c * c);
    }
    return data + prm.alpha1 * tgv1 + prm.alpha2 * tgv2;
}


// Bounded CPU baseline (bench.py): the blind pipeline with the CG loop of every channel
// capped at `cg_cap` iterations (no cap error), timing each stage with steady_clock.
// times: {weights, kernel_fit, matting_build, cg_phase (channels threaded), post_phase}.
void blind_sampled(const double* lrms, int N, int h, int w, const double* pan, int factor, int n, int threads,
                   int cg_cap, int admm_cap, int post_rows, double* times, int* cg_iters_done, int* admm_iters) {
    // times: weights, fit setup (intensity scale, E^T E, Cholesky), ADMM (capped at admm_cap
    // iterations when > 0), matting build, CG (capped at cg_cap per band), post-processing
    // without the alias-group loop, alias-group loop over LR rows [0, post_rows) (all when 0)
    using clk = std::chrono::steady_clock;
    auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
    const int H = h * factor, W = w * factor;
    const size_t P = static_cast<size_t>(H) * W, p = static_cast<size_t>(h) * w;
    auto t0 = clk::now();
    vec om = solve_weights(lrms, N, h, w, pan, H, W, 4, 10.0, factor);
    vec obs = combine_bands(lrms, N, p, om.data());
    auto t1 = clk::now();
    KeParams kp;
    kp.n = n;
    if (admm_cap > 0) kp.t_max = admm_cap;
    clk::time_point ts = t1;
    g_setup_mark = &ts;
    vec k = estimate_kernel_plane_tgv(pan, H, W, obs.data(), h, w, factor, kp, admm_iters, nullptr);
    g_setup_mark = nullptr;
    auto t2 = clk::now();
    PsParams prm;
    double peak = seq_max(pan, P);
    for (int b = 0; b < N; ++b) peak = std::max(peak, seq_max(lrms + b * p, p));
    const double scale = peak > 0.0 ? 1.0 / peak : 1.0;
    vec pan_n(P);
    for (size_t i = 0; i < P; ++i) pan_n[i] = pan[i] * scale;
    vec lpan = laplacian(pan_n.data(), H, W);
    const Matting M = Matting::build(lpan.data(), H, W, prm.radius, prm.eps);
    auto t3 = clk::now();
    std::vector<vec> z0(N), xn(N, vec(p));
    int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    nt = std::clamp(nt, 1, N);
    auto run_phase = [&](auto&& body) {
        std::atomic<int> next{0};
        auto worker = [&] {
            for (int i; (i = next.fetch_add(1)) < N;) body(i);
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
    };
    run_phase([&](int i) {
        for (size_t j = 0; j < p; ++j) xn[i][j] = lrms[i * p + j] * scale;
        int it = 0, cv = 0;
        z0[i] = warmstart_cg(xn[i].data(), h, w, k.data(), n, factor, M, prm, cg_cap, false, nullptr, &it, &cv);
        cg_iters_done[i] = it;
    });
    auto t4 = clk::now();
    vec tg(N, 0.0);
    run_phase([&](int i) {
        vec lz = laplacian(z0[i].data(), H, W);
        vec a, c, gm, gv, im;
        guided_coeffs(lz.data(), lpan.data(), H, W, prm.radius, prm.eps, a, c, gm, gv, im);
        vec v = guided_output(a.data(), c.data(), lpan.data(), H, W, prm.radius);
        vec z = solve_channel_fft(xn[i].data(), h, w, k.data(), n, factor, v.data(), H, W, prm, post_rows, &tg[i]);
    });
    auto t5 = clk::now();
    // the bands run concurrently on nt threads: the wall time of the group loops is the mean
    // per-band loop time x ceil(N / nt) rounds
    double tgm = 0.0;
    for (double x : tg) tgm += x;
    tgm /= N;
    const double rounds = std::ceil(static_cast<double>(N) / nt);
    times[0] = sec(t0, t1);
    times[1] = sec(t1, ts);
    times[2] = sec(ts, t2);
    times[3] = sec(t2, t3);
    times[4] = sec(t3, t4);
    times[5] = std::max(0.0, sec(t4, t5) - tgm * rounds);
    times[6] = tgm * rounds;
}

}  // namespace orc

// =============================================================================================
// extern "C" surface for ctypes (tests / bench only)
// =============================================================================================
using namespace orc;

template <class F>
static int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const Failure& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 4;
    }
}
static void put(const vec& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(double)); }

extern "C" {

const char* orc_last_error() { return g_last_error.c_str(); }

int orc_conv(const double* img, int h, int w, const double* k, int n, int adjoint, double* out) {
    return guard([&] { SpecConv c(k, n, h, w); put(c.apply(img, adjoint != 0), out); });
}
int orc_fft2(const double* in, int h, int w, double* out_interleaved) {
    return guard([&] {
        Fft2 f(h, w);
        cvec a = f.forward(in);
        std::memcpy(out_interleaved, a.data(), a.size() * sizeof(cd));
    });
}
int orc_downsample(const double* img, int H, int W, int c, double* out) {
    return guard([&] { put(downsample(img, H, W, c), out); });
}
int orc_upsample_adjoint(const double* img, int h, int w, int c, double* out) {
    return guard([&] { put(upsample_adjoint(img, h, w, c), out); });
}
int orc_diff(const double* img, int h, int w, int which, int adjoint, double* out) {
    return guard([&] { put(diff(img, h, w, which, adjoint != 0), out); });
}
int orc_box_mean(const double* img, int h, int w, int r, double* out) {
    return guard([&] { put(box_mean(img, h, w, r), out); });
}
int orc_circular_box_blur(const double* img, int h, int w, int window, double* out) {
    return guard([&] { put(circular_box_blur(img, h, w, window), out); });
}
int orc_embed_kernel(const double* k, int n, int h, int w, double* out) {
    return guard([&] { put(embed_kernel(k, n, h, w), out); });
}

void* orc_matting_build(const double* guide, int h, int w, int radius, double eps) {
    Matting* M = nullptr;
    const int st = guard([&] { M = new Matting(Matting::build(guide, h, w, radius, eps)); });
    return st == 0 ? M : nullptr;
}
void orc_matting_free(void* M) { delete static_cast<Matting*>(M); }
int orc_matting_apply(void* M, const double* x, double* y) {
    return guard([&] { put(static_cast<Matting*>(M)->apply(x), y); });
}
long long orc_matting_nnz(void* M) { return static_cast<long long>(static_cast<Matting*>(M)->val.size()); }
int orc_matting_csr(void* M, long long* rowptr, long long* col, double* val) {
    return guard([&] {
        auto* m = static_cast<Matting*>(M);
        for (size_t i = 0; i < m->rowptr.size(); ++i) rowptr[i] = m->rowptr[i];
        for (size_t i = 0; i < m->col.size(); ++i) col[i] = m->col[i];
        put(m->val, val);
    });
}
int orc_matting_stats(void* M, double* mean, double* var) {
    return guard([&] { put(static_cast<Matting*>(M)->mean, mean); put(static_cast<Matting*>(M)->var, var); });
}

// warmstart_cg on a prebuilt matting matrix (pansharpen.hpp:73-75)
int orc_warmstart_cg(const double* x, int h, int w, const double* k, int n, int factor, void* M, double lambda,
                     double cg_tol, int max_iters, int error_on_cap, double* z_out, int* iters, double* final_residual,
                     int* converged, int prior) {
    return guard([&] {
        PsParams p;
        p.lambda = lambda;
        p.cg_tol = cg_tol;
        p.prior = prior;
        put(warmstart_cg(x, h, w, k, n, factor, *static_cast<Matting*>(M), p, max_iters, error_on_cap != 0,
                         final_residual, iters, converged),
            z_out);
    });
}
int orc_guided_coeffs(const double* in, const double* g, int h, int w, int radius, double eps, double* a, double* c,
                      double* gmean, double* gvar, double* imean) {
    return guard([&] {
        vec A, C, GM, GV, IM;
        guided_coeffs(in, g, h, w, radius, eps, A, C, GM, GV, IM);
        put(A, a); put(C, c); put(GM, gmean); put(GV, gvar); put(IM, imean);
    });
}
int orc_guided_output(const double* a, const double* c, const double* g, int h, int w, int radius, double* out) {
    return guard([&] { put(guided_output(a, c, g, h, w, radius), out); });
}
// Hermitian eigen-decomposition (A: n x n complex, interleaved re/im, row-major); method 0 =
// Householder + QL (the alias-group solver), 1 = cyclic Jacobi. V: n x n complex, columns.
int orc_herm_eig(int n, const double* A, int method, double* ev, double* V) {
    return guard([&] {
        std::vector<cd> M(static_cast<size_t>(n) * n), W;
        for (size_t i = 0; i < M.size(); ++i) M[i] = cd(A[2 * i], A[2 * i + 1]);
        vec e;
        if (method == 0)
            herm_eig_ql(n, M, e, W);
        else
            herm_eig(n, M, e, W);
        for (int i = 0; i < n; ++i) ev[i] = e[i];
        for (size_t i = 0; i < W.size(); ++i) {
            V[2 * i] = W[i].real();
            V[2 * i + 1] = W[i].imag();
        }
    });
}
int orc_solve_channel_fft(const double* x, int h, int w, const double* k, int n, int factor, const double* v,
                          double lambda, double* out, int prior) {
    return guard([&] {
        PsParams p;
        p.lambda = lambda;
        p.prior = prior;
        put(solve_channel_fft(x, h, w, k, n, factor, v, h * factor, w * factor, p), out);
    });
}
int orc_pansharpen(const double* lrms, int N, int h, int w, const double* pan, const double* k, int n, int factor,
                   double lambda, int radius, double eps, double cg_tol, int cg_max_iter, int threads, double* out,
                   int* cg_iters, int prior) {
    return guard([&] {
        PsParams p{lambda, radius, eps, cg_tol, cg_max_iter, threads, prior};
        std::vector<int> it;
        auto res = pansharpen(lrms, N, h, w, pan, k, n, factor, p, &it);
        const size_t P = static_cast<size_t>(h) * factor * w * factor;
        for (int b = 0; b < N; ++b) std::memcpy(out + b * P, res[b].data(), P * sizeof(double));
        for (int b = 0; b < N; ++b) cg_iters[b] = it[b];
    });
}
int orc_solve_weights(const double* lrms, int nb, int h, int w, const double* pan, int H, int W, int l,
                      double lambda_omega, int factor, double* omega) {
    return guard([&] { put(solve_weights(lrms, nb, h, w, pan, H, W, l, lambda_omega, factor), omega); });
}
int orc_combine_bands(const double* lrms, int nb, int h, int w, const double* omega, double* out) {
    return guard([&] { put(combine_bands(lrms, nb, static_cast<size_t>(h) * w, omega), out); });
}
int orc_shrink2(double* cols, int ncols, long long m, double t) {
    return guard([&] {
        std::vector<vec> c(ncols);
        std::vector<vec*> ptr;
        for (int j = 0; j < ncols; ++j) { c[j].assign(cols + j * m, cols + (j + 1) * m); ptr.push_back(&c[j]); }
        shrink2(ptr, t);
        for (int j = 0; j < ncols; ++j) std::memcpy(cols + j * m, c[j].data(), m * sizeof(double));
    });
}
int orc_project_simplex(const double* v, long long n, double* out) {
    return guard([&] { put(project_simplex(v, static_cast<size_t>(n)), out); });
}
// fields: x0 x1 y0..y3 L1_0 L1_1 L2_0..L2_3 (12 n x n planes) [+ anchor]
int orc_solve_up(const double* fields, int n, double alpha1, double alpha2, double mu1, double mu2, double coupling,
                 const double* anchor, double* u, double* p1, double* p2) {
    return guard([&] {
        const size_t m = static_cast<size_t>(n) * n;
        auto F = [&](int i) { return vec(fields + i * m, fields + (i + 1) * m); };
        vec x[2] = {F(0), F(1)}, y[4] = {F(2), F(3), F(4), F(5)}, L1[2] = {F(6), F(7)}, L2[4] = {F(8), F(9), F(10), F(11)};
        KeParams prm;
        prm.alpha1 = alpha1; prm.alpha2 = alpha2; prm.mu1 = mu1; prm.mu2 = mu2;
        vec anc;
        if (anchor) anc.assign(anchor, anchor + m);
        Up s = solve_up_core(x, y, L1, L2, prm, n, coupling, anchor ? &anc : nullptr);
        put(s.u, u); put(s.p1, p1); put(s.p2, p2);
    });
}
// E^T E (n2 x n2) and E^T f for a (pan, obs) pair, no scaling
int orc_gram(const double* pan, int H, int W, const double* obs, int factor, int n, double* EtE, double* Etf) {
    return guard([&] {
        Observation O(pan, H, W, obs, H / factor, W / factor, factor, n, 1.0);
        put(O.EtE, EtE); put(O.Etf, Etf);
    });
}
int orc_solve_z(const double* pan, int H, int W, const double* obs, int factor, int n, double mu3,
                const double* anchor, double* z) {
    return guard([&] {
        Observation O(pan, H, W, obs, H / factor, W / factor, factor, n, mu3);
        put(O.solve_z(anchor), z);
    });
}
// TGV^2 estimate from (pan, obs); state_out (17 n x n planes) optional; hook_t >= 0 stops
// right before the {u,p} solve of iteration hook_t and returns that state.
int orc_estimate_kernel_plane(const double* pan, int H, int W, const double* obs, int factor, int n, double alpha1,
                              double alpha2, double mu1, double mu2, double mu3, double rho, int t_max, double th,
                              int init, double* k_out, int* iters, double* state_out, int hook_t) {
    return guard([&] {
        KeParams p;
        p.n = n; p.alpha1 = alpha1; p.alpha2 = alpha2; p.mu1 = mu1; p.mu2 = mu2; p.mu3 = mu3; p.rho = rho;
        p.t_max = t_max; p.th = th; p.init = init;
        AdmmState st;
        vec z = estimate_kernel_plane_tgv(pan, H, W, obs, H / factor, W / factor, factor, p, iters,
                                          state_out ? &st : nullptr, hook_t);
        put(z, k_out);
        if (state_out) {
            const size_t m = static_cast<size_t>(n) * n;
            for (int j = 0; j < 17; ++j) std::memcpy(state_out + j * m, st.f[j].data(), m * sizeof(double));
        }
    });
}
// TV kernel prior (estimate_kernel_plane(KernelPrior::tv, ...), kernel_estimator.cpp:445-452)
int orc_estimate_kernel_plane_tv(const double* pan, int H, int W, const double* obs, int factor, int n, double alpha1,
                                 double mu1, double mu3, double rho, int t_max, double th, int init, double* k_out,
                                 int* iters, double* state_out) {
    return guard([&] {
        KeParams p;
        p.n = n; p.alpha1 = alpha1; p.mu1 = mu1; p.mu3 = mu3; p.rho = rho;
        p.t_max = t_max; p.th = th; p.init = init; p.with_p = false;
        AdmmState st;
        vec z = estimate_kernel_plane_tgv(pan, H, W, obs, H / factor, W / factor, factor, p, iters,
                                          state_out ? &st : nullptr);
        put(z, k_out);
        if (state_out) {
            const size_t m = static_cast<size_t>(n) * n;
            for (int j = 0; j < 17; ++j) std::memcpy(state_out + j * m, st.f[j].data(), m * sizeof(double));
        }
    });
}
int orc_tgv_objective(const double* pan, int H, int W, const double* obs, int factor, int n, double mu3,
                      const double* u, const double* p1, const double* p2, double alpha1, double alpha2,
                      double* value) {
    return guard([&] {
        Observation O(pan, H, W, obs, H / factor, W / factor, factor, n, mu3);
        KeParams p;
        p.n = n; p.alpha1 = alpha1; p.alpha2 = alpha2;
        *value = tgv_objective(O, u, p1, p2, p);
    });
}
double orc_intensity_scale(const double* pan, int H, int W, int factor) {
    double s = 0.0;
    guard([&] { s = intensity_scale(pan, H, W, factor); });
    return s;
}
// SPEC.md:584-591 blind composition on all bands: weights -> TGV kernel -> pansharpen
int orc_blind(const double* lrms, int N, int h, int w, const double* pan, int factor, int n, int l,
              double lambda_omega, int threads, double* out, double* k_out, double* omega_out, int* admm_iters,
              int* cg_iters) {
    return guard([&] {
        const int H = h * factor, W = w * factor;
        vec om = solve_weights(lrms, N, h, w, pan, H, W, l, lambda_omega, factor);
        vec obs = combine_bands(lrms, N, static_cast<size_t>(h) * w, om.data());
        KeParams kp;
        kp.n = n;
        vec k = estimate_kernel_plane_tgv(pan, H, W, obs.data(), h, w, factor, kp, admm_iters, nullptr);
        PsParams pp;
        pp.threads = threads;
        std::vector<int> it;
        auto res = pansharpen(lrms, N, h, w, pan, k.data(), n, factor, pp, &it);
        const size_t P = static_cast<size_t>(H) * W;
        for (int b = 0; b < N; ++b) std::memcpy(out + b * P, res[b].data(), P * sizeof(double));
        for (int b = 0; b < N; ++b) cg_iters[b] = it[b];
        put(k, k_out);
        put(om, omega_out);
    });
}

int orc_blind_sampled(const double* lrms, int N, int h, int w, const double* pan, int factor, int n, int threads,
                      int cg_cap, int admm_cap, int post_rows, double* times, int* cg_iters_done, int* admm_iters) {
    return guard([&] {
        blind_sampled(lrms, N, h, w, pan, factor, n, threads, cg_cap, admm_cap, post_rows, times, cg_iters_done,
                      admm_iters);
    });
}

// E (p x n^2) of ObservationSystem (kernel_estimator.cpp:57-68), for the construction KATs
int orc_observation_matrix(const double* pan, int H, int W, int factor, int n, double* E) {
    return guard([&] {
        std::vector<double> obs(static_cast<size_t>(H / factor) * (W / factor), 0.0);
        Observation O(pan, H, W, obs.data(), H / factor, W / factor, factor, n, 1.0);
        put(O.E, E);
    });
}

}  // extern "C"
