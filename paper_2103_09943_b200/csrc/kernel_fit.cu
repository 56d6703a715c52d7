// kernel_fit.cu -- sm_100a kernels of Algorithm 1 (TGV^2 + simplex blur-kernel fit,
// reference /root/reference/proj/src/kernel_estimator.cpp) and of the spectral-weight stage
// that feeds it (spectral_weights.cpp).
//
//   K_SW    box blurs + normal equations + full-pivot solve of Eq. (8), one block per scene
//   K_GRAM  E^T E through its c-periodic block-Toeplitz structure: only the c^2 (2n-1)^2
//           distinct sums T[rho][d] = sum_x P(x - rho) P(x - rho - d) are formed (E is never
//           materialised); E^T f likewise from PAN patches staged in shared memory
//   K_CHOL  blocked Cholesky of E^T E + mu3 I, explicit symmetric inverse (L^-T L^-1)
//   K_ADMM  the whole ADMM loop in one persistent CTA per scene: all 17 n x n fields live in
//           shared memory, DFTs as small matrix products, simplex projection by ranks;
//           the only global traffic per iteration is the (E^T E + mu3 I)^-1 mat-vec (L2).
#include <cmath>

#include <cooperative_groups.h>

#include "kernel_fit.cuh"
#include <nccl.h>

#include <cstdlib>

namespace fbmp_gpu {

namespace {

constexpr int NT = 256;

inline int grid1d(Context& ctx, long long n, int threads = 256) {
    long long b = (n + threads - 1) / threads;
    const long long cap = static_cast<long long>(ctx.sm_count) * 16;
    return static_cast<int>(std::max(1LL, std::min(b, cap)));
}
template <class K>
void set_smem(K kernel, size_t bytes) {
    FBMP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

// =============================================================================================
// Spectral weights (spectral_weights.cpp:9-53)
// =============================================================================================
// Circular box blur along columns (ops.cpp:139-145) with output decimation dc:
// out[b][r][j] = gain * sum_{t=-lead}^{win-lead-1} in[b][r][(dc*j - t) mod Win]
__global__ void k_blur_h(const double* __restrict__ in, int B, int Hin, int Win, int Wout, int dc, int win,
                         double* __restrict__ out) {
    const int lead = (win - 1) / 2;
    const double gain = 1.0 / win;
    const long long tot = static_cast<long long>(B) * Hin * Wout;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(e % Wout);
        const long long br = e / Wout;
        const double* row = in + br * Win;
        double s = 0.0;
        for (int t = -lead; t < win - lead; ++t) s += row[wrapi(dc * j - t, Win)];
        out[e] = s * gain;
    }
}
// ... and along rows (ops.cpp:146-152) with output decimation dr.
__global__ void k_blur_v(const double* __restrict__ in, int B, int Hin, int W, int Hout, int dr, int win,
                         double* __restrict__ out) {
    const int lead = (win - 1) / 2;
    const double gain = 1.0 / win;
    const long long tot = static_cast<long long>(B) * Hout * W;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(e % W);
        const long long bi = e / W;
        const int i = static_cast<int>(bi % Hout);
        const long long b = bi / Hout;
        const double* col = in + b * static_cast<long long>(Hin) * W + j;
        double s = 0.0;
        for (int t = -lead; t < win - lead; ++t) s += col[static_cast<size_t>(wrapi(dr * i - t, Hin)) * W];
        out[e] = s * gain;
    }
}

// per-block partial dot products: pairs (i<=j) of A columns, then A_i . b
__global__ void __launch_bounds__(NT) k_sw_dots(const double* __restrict__ A, const double* __restrict__ bvec, int nb,
                                                long long p, int nblk, double* __restrict__ part) {
    __shared__ double red[NT / 32 + 1];
    const int s = blockIdx.y;
    const double* As = A + static_cast<size_t>(s) * nb * p;
    const double* bs = bvec + static_cast<size_t>(s) * p;
    const long long chunk = (p + nblk - 1) / nblk;
    const long long lo = blockIdx.x * chunk, hi = std::min(p, lo + chunk);
    const int nv = nb * (nb + 1) / 2 + nb;
    int v = 0;
    for (int i = 0; i < nb; ++i)
        for (int j = i; j <= nb; ++j, ++v) {
            const double* x = As + static_cast<size_t>(i) * p;
            const double* y = j < nb ? As + static_cast<size_t>(j) * p : bs;
            double acc = 0.0;
            for (long long k = lo + threadIdx.x; k < hi; k += NT) acc += x[k] * y[k];
            const double bsum = block_sum<NT>(acc, red);
            if (threadIdx.x == 0) part[(static_cast<size_t>(s) * nblk + blockIdx.x) * nv + v] = bsum;
        }
}

// one block per scene: sum partials, add lambda G^T G, full-pivot solve, stationarity check
__global__ void k_sw_solve(const double* __restrict__ part, int nb, int nblk, double lambda_omega,
                           double* __restrict__ omega, int* __restrict__ status) {
    extern __shared__ double sh[];
    const int s = blockIdx.x;
    const int nv = nb * (nb + 1) / 2 + nb;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        double acc = 0.0;
        for (int b = 0; b < nblk; ++b) acc += part[(static_cast<size_t>(s) * nblk + b) * nv + v];
        sh[v] = acc;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double* N = sh + nv;          // nb*nb
    double* rhs = N + nb * nb;    // nb
    double* A = rhs + nb;         // nb*nb work
    double* bw = A + nb * nb;     // nb
    double* y = bw + nb;          // nb
    int* perm = reinterpret_cast<int*>(y + nb);
    int v = 0;
    for (int i = 0; i < nb; ++i)
        for (int j = i; j <= nb; ++j, ++v) {
            if (j < nb) N[i * nb + j] = N[j * nb + i] = sh[v];
            else rhs[i] = sh[v];
        }
    if (nb > 1)
        for (int i = 0; i < nb; ++i)
            for (int j = 0; j < nb; ++j) {
                double g = 0.0;
                for (int r = 0; r < nb - 1; ++r) {
                    const double gi = (i == r) ? -1.0 : (i == r + 1 ? 1.0 : 0.0);
                    const double gj = (j == r) ? -1.0 : (j == r + 1 ? 1.0 : 0.0);
                    g += gi * gj;
                }
                N[i * nb + j] += lambda_omega * g;
            }
    for (int i = 0; i < nb * nb; ++i) A[i] = N[i];
    for (int i = 0; i < nb; ++i) { bw[i] = rhs[i]; perm[i] = i; }
    double maxpiv = 0.0;
    int rank = 0;
    for (int k = 0; k < nb; ++k) {  // Gauss with full pivoting (stands in for Eigen::FullPivLU)
        int pr = k, pc = k;
        double best = -1.0;
        for (int i = k; i < nb; ++i)
            for (int j = k; j < nb; ++j)
                if (fabs(A[i * nb + j]) > best) { best = fabs(A[i * nb + j]); pr = i; pc = j; }
        if (k == 0) maxpiv = best;
        if (best <= maxpiv * 2.220446049250313e-16 * nb || best == 0.0) break;
        ++rank;
        if (pr != k) {
            for (int j = 0; j < nb; ++j) { const double t = A[k * nb + j]; A[k * nb + j] = A[pr * nb + j]; A[pr * nb + j] = t; }
            const double t = bw[k]; bw[k] = bw[pr]; bw[pr] = t;
        }
        if (pc != k) {
            for (int i = 0; i < nb; ++i) { const double t = A[i * nb + k]; A[i * nb + k] = A[i * nb + pc]; A[i * nb + pc] = t; }
            const int t = perm[k]; perm[k] = perm[pc]; perm[pc] = t;
        }
        for (int i = k + 1; i < nb; ++i) {
            const double f = A[i * nb + k] / A[k * nb + k];
            for (int j = k; j < nb; ++j) A[i * nb + j] -= f * A[k * nb + j];
            bw[i] -= f * bw[k];
        }
    }
    if (rank < nb) { status[s] = 1; return; }
    for (int i = nb - 1; i >= 0; --i) {
        double t = bw[i];
        for (int j = i + 1; j < nb; ++j) t -= A[i * nb + j] * y[j];
        y[i] = t / A[i * nb + i];
    }
    double* om = omega + static_cast<size_t>(s) * nb;
    for (int i = 0; i < nb; ++i) om[perm[i]] = y[i];
    double r2 = 0.0, b2 = 0.0;
    for (int i = 0; i < nb; ++i) {
        double t = 0.0;
        for (int j = 0; j < nb; ++j) t += N[i * nb + j] * om[j];
        r2 += (t - rhs[i]) * (t - rhs[i]);
        b2 += rhs[i] * rhs[i];
    }
    status[s] = (sqrt(r2) <= 1e-8 * sqrt(b2) + 1e-12) ? 0 : 2;
}

__global__ void k_combine(const double* __restrict__ lrms, int S, int nb, long long p, const double* __restrict__ omega,
                          double* __restrict__ out) {
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < S * p;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long s = e / p, j = e - s * p;
        double acc = 0.0;
        for (int i = 0; i < nb; ++i) acc += omega[s * nb + i] * lrms[(s * nb + i) * p + j];
        out[e] = acc;
    }
}

// PAN statistics: {sum, min, max, max|v|} per scene
__global__ void __launch_bounds__(NT) k_stats_partial(const double* __restrict__ pan, long long P, int nblk,
                                                      double* __restrict__ part) {
    __shared__ double red[NT / 32 + 1];
    __shared__ double mn[NT], mx[NT], ma[NT];
    const int s = blockIdx.y;
    const double* ps = pan + static_cast<size_t>(s) * P;
    double sum = 0.0, lo = INFINITY, hi = -INFINITY, am = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(NT) + threadIdx.x; i < P; i += static_cast<long long>(nblk) * NT) {
        const double v = ps[i];
        sum += v;
        lo = fmin(lo, v);
        hi = fmax(hi, v);
        am = fmax(am, fabs(v));
    }
    const double bs = block_sum<NT>(sum, red);
    mn[threadIdx.x] = lo; mx[threadIdx.x] = hi; ma[threadIdx.x] = am;
    __syncthreads();
    for (int o = NT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            mn[threadIdx.x] = fmin(mn[threadIdx.x], mn[threadIdx.x + o]);
            mx[threadIdx.x] = fmax(mx[threadIdx.x], mx[threadIdx.x + o]);
            ma[threadIdx.x] = fmax(ma[threadIdx.x], ma[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* o = part + (static_cast<size_t>(s) * nblk + blockIdx.x) * 4;
        o[0] = bs; o[1] = mn[0]; o[2] = mx[0]; o[3] = ma[0];
    }
}
// one warp per scene (min / max are exact in any order; the sum only feeds the mean of the
// degeneracy test, kernel_estimator.cpp:269-276, whose outcome does not depend on its last bits)
__global__ void k_stats_final(const double* __restrict__ part, int nblk, double* __restrict__ stats) {
    const int s = blockIdx.x, lane = threadIdx.x;
    double sum = 0.0, lo = INFINITY, hi = -INFINITY, am = 0.0;
    for (int b = lane; b < nblk; b += 32) {
        const double* o = part + (static_cast<size_t>(s) * nblk + b) * 4;
        sum += o[0]; lo = fmin(lo, o[1]); hi = fmax(hi, o[2]); am = fmax(am, o[3]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
    }
    if (lane == 0) {
        stats[s * 4 + 0] = sum; stats[s * 4 + 1] = lo; stats[s * 4 + 2] = hi; stats[s * 4 + 3] = am;
    }
}

// =============================================================================================
// K_GRAM
// =============================================================================================
constexpr int TG = 16;  // LR tile side of the Gram kernels

// T[s][rho][d] partials for one LR tile and one sampling phase rho = (rho_r, rho_c):
//   sum_{(i,j) in tile} P(c i - rho_r + C, c j - rho_c + C) * P(c i - rho_r - dr + C, c j - rho_c - dc + C)
// with P = pan * scale (the reference's pan_n, kernel_estimator.cpp:443-444).
__global__ void __launch_bounds__(NT) k_gram_T(const double* __restrict__ pan, const double* __restrict__ scale, int H,
                                               int W, int h, int w, int c, int n, double* __restrict__ part,
                                               int ntiles, int t_lo) {
    extern __shared__ double reg[];
    const int s = blockIdx.z, phase = blockIdx.y, tile = blockIdx.x + t_lo;
    const int rho_r = phase / c, rho_c = phase - rho_r * c;
    const int ntx = (w + TG - 1) / TG;
    const int i0 = (tile / ntx) * TG, j0 = (tile % ntx) * TG;
    const int C = (n - 1) / 2, D = 2 * n - 1, nd = D * D;
    const int SR = c * (TG - 1) + 2 * (n - 1) + 1;
    const int R0 = c * i0 - rho_r + C - (n - 1), C0 = c * j0 - rho_c + C - (n - 1);
    const double sc = scale ? scale[s] : 1.0;
    const double* ps = pan + static_cast<size_t>(s) * H * W;
    for (int e = threadIdx.x; e < SR * SR; e += NT) {
        const int y = e / SR, x = e - y * SR;
        reg[e] = ps[static_cast<size_t>(wrapi(R0 + y, H)) * W + wrapi(C0 + x, W)] * sc;
    }
    __syncthreads();
    const int ni = min(TG, h - i0), nj = min(TG, w - j0);
    double* out = part + ((static_cast<size_t>(s) * ntiles + tile) * c * c + phase) * nd;
    constexpr int K = 8;
    for (int o0 = 0; o0 < nd; o0 += NT * K) {
        double acc[K];
        int off[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            acc[k] = 0.0;
            const int o = o0 + k * NT + threadIdx.x;
            const int dr = o / D - (n - 1), dc = o % D - (n - 1);
            off[k] = (o < nd) ? dr * SR + dc : 0;
        }
        for (int ii = 0; ii < ni; ++ii)
            for (int jj = 0; jj < nj; ++jj) {
                const int cp = (c * ii + n - 1) * SR + c * jj + n - 1;
                const double cv = reg[cp];
#pragma unroll
                for (int k = 0; k < K; ++k) acc[k] = fma(cv, reg[cp - off[k]], acc[k]);
            }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int o = o0 + k * NT + threadIdx.x;
            if (o < nd) out[o] = acc[k];
        }
    }
}

// Same partials, register-blocked: a thread owns one row offset dr and GK consecutive column
// offsets; walking the tile's points along a row, its window of GK region values shifts by c
// columns per point (c new loads, GK FMAs, one broadcast load of the centre value). Every output
// keeps the point order of k_gram_T, so the partials are bit-identical.
constexpr int GK = 12;
constexpr int NTG = 192;  // >= (2n-1) * ceil((2n-1) / GK) for n <= 21
template <int CF>
__global__ void __launch_bounds__(NTG) k_gram_T2(const double* __restrict__ pan, const double* __restrict__ scale,
                                                 int H, int W, int h, int w, int n, double* __restrict__ part,
                                                 int ntiles, int t_lo) {
    constexpr int c = CF;
    extern __shared__ double smg[];
    double* reg = smg + GK;  // GK doubles of slack below the region: the full-tile path loads the
                             // window's padding columns unconditionally (their sums are discarded)
    const int s = blockIdx.z, phase = blockIdx.y, tile = blockIdx.x + t_lo;
    const int rho_r = phase / c, rho_c = phase - rho_r * c;
    const int ntx = (w + TG - 1) / TG;
    const int i0 = (tile / ntx) * TG, j0 = (tile % ntx) * TG;
    const int D = 2 * n - 1, nd = D * D, nblk = (D + GK - 1) / GK;
    const int SR = c * (TG - 1) + 2 * (n - 1) + 1;
    const int R0 = c * i0 - rho_r + (n - 1) / 2 - (n - 1), C0 = c * j0 - rho_c + (n - 1) / 2 - (n - 1);
    const double sc = scale ? scale[s] : 1.0;
    const double* ps = pan + static_cast<size_t>(s) * H * W;
    for (int e = threadIdx.x; e < SR * SR; e += NTG) {
        const int y = e / SR, x = e - y * SR;
        reg[e] = ps[static_cast<size_t>(wrapi(R0 + y, H)) * W + wrapi(C0 + x, W)] * sc;
    }
    __syncthreads();
    const int ni = min(TG, h - i0), nj = min(TG, w - j0);
    double* out = part + ((static_cast<size_t>(s) * ntiles + tile) * c * c + phase) * nd;
    const int rb = threadIdx.x / nblk, blk = threadIdx.x - rb * nblk;
    if (rb >= D) return;
    const int dr = rb - (n - 1), dc0 = blk * GK - (n - 1);
    double acc[GK];
#pragma unroll
    for (int k = 0; k < GK; ++k) acc[k] = 0.0;
    if (nj == TG) {
        // full tile row: the point loop is unrolled, so the c-column window shift is register
        // renaming (each region value is loaded once per row and feeds up to GK / c points);
        // every accumulator keeps the ascending point order of the generic loop below
        for (int ii = 0; ii < ni; ++ii) {
            const double* crow = reg + (c * ii + n - 1) * SR + n - 1;
            const double* wrow = reg + (c * ii + n - 1 - dr) * SR + n - 1 - dc0;
#pragma unroll
            for (int jj = 0; jj < TG; ++jj) {
                const double cv = crow[c * jj];
#pragma unroll
                for (int k = 0; k < GK; ++k) acc[k] = fma(cv, wrow[c * jj - k], acc[k]);
            }
        }
    } else {
    for (int ii = 0; ii < ni; ++ii) {
        const double* crow = reg + (c * ii + n - 1) * SR + n - 1;          // centre values
        const double* wrow = reg + (c * ii + n - 1 - dr) * SR + n - 1 - dc0;  // window row
        double win[GK];
        const int kval = min(GK, n - dc0);  // column offsets beyond n - 1 are padding: never loaded
#pragma unroll
        for (int k = 0; k < GK; ++k) win[k] = k < kval ? wrow[-k] : 0.0;
        for (int jj = 0; jj < nj; ++jj) {
            const double cv = crow[c * jj];
#pragma unroll
            for (int k = 0; k < GK; ++k) acc[k] = fma(cv, win[k], acc[k]);
            // shift by c columns: win[k] <- value at column + c
            const double* nxt = wrow + c * (jj + 1);
            const bool more = jj + 1 < nj;  // no load past the tile's last point
#pragma unroll
            for (int k = GK - 1; k >= 0; --k) win[k] = (k >= c) ? win[k - c] : (more && k < kval ? nxt[-k] : 0.0);
        }
    }
    }
#pragma unroll
    for (int k = 0; k < GK; ++k) {
        const int dc = dc0 + k;
        if (dc <= n - 1) out[(dr + n - 1) * D + dc + n - 1] = acc[k];
    }
}

// E^T f partials: sum_{(i,j) in tile} P(c i - tr + C, c j - tc + C) * f(i, j), f = obs * scale
__global__ void __launch_bounds__(NT) k_gram_etf(const double* __restrict__ pan, const double* __restrict__ obs,
                                                 const double* __restrict__ scale, int H, int W, int h, int w, int c,
                                                 int n, double* __restrict__ part, int ntiles, int t_lo) {
    extern __shared__ double reg[];
    const int s = blockIdx.z, tile = blockIdx.x + t_lo;
    const int ntx = (w + TG - 1) / TG;
    const int i0 = (tile / ntx) * TG, j0 = (tile % ntx) * TG;
    const int C = (n - 1) / 2, n2 = n * n;
    const int SR = c * (TG - 1) + n;
    const int R0 = c * i0 + C - (n - 1), C0 = c * j0 + C - (n - 1);
    const double sc = scale ? scale[s] : 1.0;
    const double* ps = pan + static_cast<size_t>(s) * H * W;
    const double* fs = obs + static_cast<size_t>(s) * h * w;
    double* sf = reg + ((SR * SR + 1) & ~1);
    for (int e = threadIdx.x; e < SR * SR; e += NT) {
        const int y = e / SR, x = e - y * SR;
        reg[e] = ps[static_cast<size_t>(wrapi(R0 + y, H)) * W + wrapi(C0 + x, W)] * sc;
    }
    const int ni = min(TG, h - i0), nj = min(TG, w - j0);
    for (int e = threadIdx.x; e < TG * TG; e += NT) {
        const int a = e / TG, b = e - a * TG;
        sf[e] = (a < ni && b < nj) ? fs[static_cast<size_t>(i0 + a) * w + j0 + b] * sc : 0.0;
    }
    __syncthreads();
    for (int tap = threadIdx.x; tap < n2; tap += NT) {
        const int tr = tap / n, tc = tap - tr * n;
        double acc = 0.0;
        for (int ii = 0; ii < ni; ++ii)
            for (int jj = 0; jj < nj; ++jj)
                acc = fma(reg[(c * ii + n - 1 - tr) * SR + c * jj + n - 1 - tc], sf[ii * TG + jj], acc);
        part[(static_cast<size_t>(s) * ntiles + tile) * n2 + tap] = acc;
    }
}

// Tile partials are reduced in GRAM_CHUNKS fixed, contiguous tile chunks (sequential sums inside a
// chunk, then over the chunks in order). The chunking does not depend on the number of ranks, so a
// C5 fit split over G | GRAM_CHUNKS ranks (each computes whole chunks, the chunk sums are
// all-gathered) is bit-identical to the single-GPU fit.
constexpr int GRAM_CHUNKS = 8;
__host__ __device__ inline int chunk_tile(int k, int ntiles) {
    return static_cast<int>(static_cast<long long>(k) * ntiles / GRAM_CHUNKS);
}
// cp[s][k][v] = sum_{t in chunk k} part[s][t][v] for k in [k0, k1)
__global__ void k_reduce_chunks(const double* __restrict__ part, int S, int ntiles, int nv, int k0, int k1,
                                double* __restrict__ cp) {
    const int nk = k1 - k0;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
         e < static_cast<long long>(S) * nk * nv; e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long s = e / (static_cast<long long>(nk) * nv);
        const long long rem = e - s * nk * nv;
        const int k = k0 + static_cast<int>(rem / nv), v = static_cast<int>(rem - (rem / nv) * nv);
        const double* pp = part + s * ntiles * static_cast<long long>(nv) + v;
        const int t1 = chunk_tile(k + 1, ntiles);
        double acc = 0.0;
        int t = chunk_tile(k, ntiles);
        for (; t + 16 <= t1; t += 16) {  // tile order kept; loads issued 16 ahead of the additions
            double x[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) x[q] = __ldg(pp + static_cast<long long>(t + q) * nv);
#pragma unroll
            for (int q = 0; q < 16; ++q) acc += x[q];
        }
        for (; t < t1; ++t) acc += __ldg(pp + static_cast<long long>(t) * nv);
        cp[(s * GRAM_CHUNKS + k) * nv + v] = acc;
    }
}
// out[s][v] = sum_k cp[s][k][v]
__global__ void k_sum_chunks(const double* __restrict__ cp, int S, int nv, double* __restrict__ out) {
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(S) * nv;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long s = e / nv, v = e - s * nv;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < GRAM_CHUNKS; ++k) acc += cp[(s * GRAM_CHUNKS + k) * nv + v];
        out[e] = acc;
    }
}


// G[(tr,tc),(tr',tc')] = T[tr mod c][tc mod c][tr'-tr][tc'-tc] (+ mu3 on the diagonal)
__global__ void k_gram_expand(const double* __restrict__ T, int S, int c, int n, double mu3, double* __restrict__ M) {
    const int n2 = n * n, D = 2 * n - 1, nd = D * D;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
         e < static_cast<long long>(S) * n2 * n2; e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long s = e / (static_cast<long long>(n2) * n2);
        const int ab = static_cast<int>(e - s * n2 * static_cast<long long>(n2));
        const int a = ab / n2, b = ab - a * n2;
        const int tr = a / n, tc = a - tr * n, tr2 = b / n, tc2 = b - tr2 * n;
        const int phase = (tr % c) * c + (tc % c);
        const int d = (tr2 - tr + n - 1) * D + (tc2 - tc + n - 1);
        double v = T[(s * c * c + phase) * nd + d];
        if (a == b) v += mu3;
        M[e] = v;
    }
}

// =============================================================================================
// K_CHOL: blocked right-looking Cholesky (lower), explicit inverse
// =============================================================================================
constexpr int NBK = 32;

// factor the panel A[K:N, K:K+nb] in shared memory (diagonal block + sub-panel solve)
__global__ void __launch_bounds__(NT) k_potrf_panel(double* __restrict__ M, int N, int K, int* __restrict__ status) {
    // panel columns [K, K+nb): the nb x nb diagonal block is factorised by warp 0 (lane i owns
    // row i, one __syncwarp per column), the rows below by a row-parallel triangular solve
    extern __shared__ double pnl[];
    constexpr int LD = NBK + 1;  // padded row stride
    const int s = blockIdx.x;
    if (status[s]) return;
    double* A = M + static_cast<size_t>(s) * N * N;
    const int nb = min(NBK, N - K), rows = N - K;
    for (int e = threadIdx.x; e < rows * nb; e += NT) {
        const int i = e / nb, j = e - i * nb;
        pnl[i * LD + j] = A[static_cast<size_t>(K + i) * N + K + j];
    }
    __shared__ int fail;
    if (threadIdx.x == 0) fail = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int i = threadIdx.x;
        for (int k = 0; k < nb; ++k) {
            const double d = pnl[k * LD + k];
            if (!(d > 0)) {
                if (i == 0) fail = 1;
                break;
            }
            const double l = sqrt(d);
            __syncwarp();
            if (i == k) pnl[k * LD + k] = l;
            if (i > k && i < nb) pnl[i * LD + k] /= l;
            __syncwarp();
            if (i > k && i < nb) {
                const double lik = pnl[i * LD + k];
                for (int j = k + 1; j <= i; ++j) pnl[i * LD + j] -= lik * pnl[j * LD + k];
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (fail) {
        if (threadIdx.x == 0) status[s] = 1;
        return;
    }
    for (int i = nb + threadIdx.x; i < rows; i += NT) {  // L21 = A21 L11^-T, row by row
        double* row = pnl + i * LD;
        for (int k = 0; k < nb; ++k) {
            double v = row[k];
            for (int j = 0; j < k; ++j) v -= row[j] * pnl[k * LD + j];
            row[k] = v / pnl[k * LD + k];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * nb; e += NT) {
        const int i = e / nb, j = e - i * nb;
        A[static_cast<size_t>(K + i) * N + K + j] = (i >= j) ? pnl[i * LD + j] : 0.0;
    }
}

// trailing update A[I][J] -= L[I][K:K+nb] L[J][K:K+nb]^T for 32x32 lower tiles beyond K+nb
__global__ void __launch_bounds__(NT) k_syrk(double* __restrict__ M, int N, int K, const int* __restrict__ status) {
    __shared__ double LI[NBK][NBK + 1], LJ[NBK][NBK + 1];
    const int s = blockIdx.y;
    if (status[s]) return;
    double* A = M + static_cast<size_t>(s) * N * N;
    const int base = K + NBK;
    const int nt = (N - base + NBK - 1) / NBK;
    // blockIdx.x enumerates lower tiles (ti >= tj)
    int t = blockIdx.x, ti = 0;
    while (t >= ti + 1) { t -= ti + 1; ++ti; }
    const int tj = t;
    if (ti >= nt) return;
    const int r0 = base + ti * NBK, c0 = base + tj * NBK;
    for (int e = threadIdx.x; e < NBK * NBK; e += NT) {
        const int a = e / NBK, b = e - a * NBK;
        LI[a][b] = (r0 + a < N) ? A[static_cast<size_t>(r0 + a) * N + K + b] : 0.0;
        LJ[a][b] = (c0 + a < N) ? A[static_cast<size_t>(c0 + a) * N + K + b] : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < NBK * NBK; e += NT) {
        const int a = e / NBK, b = e - a * NBK;
        const int i = r0 + a, j = c0 + b;
        if (i < N && j < N && j <= i) {
            double acc = 0.0;
#pragma unroll 8
            for (int k = 0; k < NBK; ++k) acc = fma(LI[a][k], LJ[b][k], acc);
            A[static_cast<size_t>(i) * N + j] -= acc;
        }
    }
}

// L^-1 column by column (one warp per column, forward substitution)
__global__ void __launch_bounds__(NT) k_trtri(const double* __restrict__ M, int N, double* __restrict__ Linv,
                                              const int* __restrict__ status) {
    extern __shared__ double ys[];
    const int s = blockIdx.y;
    if (status[s]) return;
    const double* L = M + static_cast<size_t>(s) * N * N;
    double* Li = Linv + static_cast<size_t>(s) * N * N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * (NT / 32) + warp;
    if (j >= N) return;
    double* y = ys + warp * N;
    for (int i = lane; i < N; i += 32) y[i] = 0.0;
    __syncwarp();
    if (lane == 0) y[j] = 1.0 / L[static_cast<size_t>(j) * N + j];
    __syncwarp();
    for (int i = j + 1; i < N; ++i) {
        const double* row = L + static_cast<size_t>(i) * N;
        double acc = 0.0;
        for (int k = j + lane; k < i; k += 32) acc = fma(row[k], y[k], acc);
        acc = warp_sum(acc);
        if (lane == 0) y[i] = -acc / row[i];
        __syncwarp();
    }
    for (int i = lane; i < N; i += 32) Li[static_cast<size_t>(i) * N + j] = y[i];
}

// Same forward substitution with the next row of L in flight while the current one is reduced
// (the chain over rows is latency-bound on L2 loads otherwise). KL = ceil(N / 32) values per lane.
template <int KL>
__global__ void __launch_bounds__(NT) k_trtri_pf(const double* __restrict__ M, int N, double* __restrict__ Linv,
                                                 const int* __restrict__ status) {
    extern __shared__ double ys[];
    const int s = blockIdx.y;
    if (status[s]) return;
    const double* L = M + static_cast<size_t>(s) * N * N;
    double* Li = Linv + static_cast<size_t>(s) * N * N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * (NT / 32) + warp;
    if (j >= N) return;
    double* y = ys + warp * N;
    for (int i = lane; i < N; i += 32) y[i] = 0.0;
    __syncwarp();
    if (lane == 0) y[j] = 1.0 / L[static_cast<size_t>(j) * N + j];
    __syncwarp();
    // row i, columns k = j + lane + 32 t (t < KL)
    double cur[KL], nxt[KL];
    double dcur = 0.0, dnxt = 0.0;
    auto load = [&](int i, double (&v)[KL], double& d) {
        const double* row = L + static_cast<size_t>(i) * N;
#pragma unroll
        for (int t = 0; t < KL; ++t) {
            const int k = j + lane + 32 * t;
            v[t] = k < i ? __ldg(row + k) : 0.0;
        }
        d = __ldg(row + i);
    };
    if (j + 1 < N) load(j + 1, cur, dcur);
    for (int i = j + 1; i < N; ++i) {
        if (i + 1 < N) load(i + 1, nxt, dnxt);
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < KL; ++t) {
            const int k = j + lane + 32 * t;
            if (k < i) acc = fma(cur[t], y[k], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) y[i] = -acc / dcur;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < KL; ++t) cur[t] = nxt[t];
        dcur = dnxt;
    }
    for (int i = lane; i < N; i += 32) Li[static_cast<size_t>(i) * N + j] = y[i];
}

// Ginv[a][b] = sum_k Linv[k][a] Linv[k][b] (a >= b), mirrored -> exactly symmetric
__global__ void __launch_bounds__(NT) k_inv_gram(const double* __restrict__ Linv, int N, double* __restrict__ Ginv,
                                                 const int* __restrict__ status) {
    __shared__ double A_[NBK][NBK + 1], B_[NBK][NBK + 1];
    const int s = blockIdx.y;
    if (status[s]) return;
    const double* Li = Linv + static_cast<size_t>(s) * N * N;
    double* G = Ginv + static_cast<size_t>(s) * N * N;
    int t = blockIdx.x, ti = 0;
    while (t >= ti + 1) { t -= ti + 1; ++ti; }
    const int tj = t;
    const int nt = (N + NBK - 1) / NBK;
    if (ti >= nt) return;
    const int a0 = ti * NBK, b0 = tj * NBK;
    double acc[NBK * NBK / NT];
#pragma unroll
    for (int q = 0; q < NBK * NBK / NT; ++q) acc[q] = 0.0;
    for (int k0 = a0; k0 < N; k0 += NBK) {  // Linv[k][a] = 0 for k < a
        __syncthreads();
        for (int e = threadIdx.x; e < NBK * NBK; e += NT) {
            const int kk = e / NBK, x = e - kk * NBK;
            const int k = k0 + kk;
            A_[kk][x] = (k < N && a0 + x < N) ? Li[static_cast<size_t>(k) * N + a0 + x] : 0.0;
            B_[kk][x] = (k < N && b0 + x < N) ? Li[static_cast<size_t>(k) * N + b0 + x] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NBK * NBK / NT; ++q) {
            const int e = threadIdx.x + q * NT;
            const int a = e / NBK, b = e - a * NBK;
            double v = acc[q];
            for (int kk = 0; kk < NBK; ++kk) v = fma(A_[kk][a], B_[kk][b], v);
            acc[q] = v;
        }
    }
#pragma unroll
    for (int q = 0; q < NBK * NBK / NT; ++q) {
        const int e = threadIdx.x + q * NT;
        const int a = a0 + e / NBK, b = b0 + e % NBK;
        if (a < N && b < N && b <= a) {
            G[static_cast<size_t>(a) * N + b] = acc[q];
            G[static_cast<size_t>(b) * N + a] = acc[q];
        }
    }
}

// =============================================================================================
// K_ADMM
// =============================================================================================
struct AdmmArgs {
    int n, m;
    double alpha1, alpha2, mu1, mu2, mu3, rho, th, coupling;
    int t_max, t_begin, phase_begin, hook_t, init_kind, init_state;
    int cache_symbols;  // 1: per-frequency {u,p} symbols cached in shared memory
    int ginv_global;    // 1: the cluster's mat-vec rows are read from the inverse in global memory
                        //    (L2-resident) instead of a shared-memory slice (large kernels)
    const double* tv_d1;  // TV kernel prior (run_tgv_or_tv(false, ...)): the u-step symbol d1 (n2,
                          // host-evaluated as kernel_estimator.cpp:309-321); null = TGV^2
};

constexpr int NTADMM = 512;
#ifdef FBMP_ADMM_PROF  // phase timers of k_admm (thread 0, clock64), A/B diagnostics only
__device__ long long g_admm_prof[16];
#define APROF_T0 long long _ap_t = clock64(), _ap_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; \
    if (threadIdx.x == 0 && blockIdx.x == 0) for (int _k = 8; _k < 12; ++_k) g_admm_prof[_k] = 0;
#define APROF(k) if (threadIdx.x == 0 && blockIdx.x == 0) { const long long _n = clock64(); _ap_acc[k] += _n - _ap_t; _ap_t = _n; }
#define APROF_END if (threadIdx.x == 0 && blockIdx.x == 0) for (int _k = 0; _k < 8; ++_k) g_admm_prof[_k] = _ap_acc[_k];
// sub-phases of the {u,p} solve (rhs, forward DFT, per-frequency solve, inverse DFT): slots 8..11
#define UPROF_T0 long long _up_t = clock64();
#define UPROF(k) if (threadIdx.x == 0 && blockIdx.x == 0) { const long long _n = clock64(); atomicAdd(reinterpret_cast<unsigned long long*>(&g_admm_prof[8 + k]), static_cast<unsigned long long>(_n - _up_t)); _up_t = _n; }
#else
#define APROF_T0
#define APROF(k)
#define APROF_END
#define UPROF_T0
#define UPROF(k)
#endif
// projection scratch of the sorted (m <= NTADMM) projection; none for the rank-based one
__host__ __device__ constexpr int admm_scratch_doubles(int m) {
    return m <= NTADMM ? (6 * m > 3 * NTADMM ? 6 * m : 3 * NTADMM) : 0;
}
enum { F_U = 0, F_P1, F_P2, F_X0, F_X1, F_Y0, F_Y1, F_Y2, F_Y3, F_Z, F_L10, F_L11, F_L20, F_L21, F_L22, F_L23, F_L3 };

struct AdmmSmem {
    double* f[17];
    double *bz, *zz, *unew, *tmp6;  // tmp6: max(6m, 3 NTADMM) doubles, projection scratch
    double *spec, *rowt;            // 3 complex planes each (6*m doubles)
    double *twc, *tws;              // n
    double* red;
    double* sym = nullptr;          // optional cache of the per-frequency symbols (11*m) + tol
};

// per-frequency symbols of the {u,p} system (kernel_estimator.cpp:175-195):
// {d1, d2, d3, Re d4, Im d4, Re d5, Im d5, Re d6, Im d6, Re den, Im den}
__device__ __forceinline__ void up_symbol(const AdmmSmem& S, int n, int i, double a1m1, double a2m2, double coupling,
                                          double out[11]) {
    const int r = i / n, c = i - r * n;
    const double dvr = S.twc[r] - 1.0, dvi = S.tws[r];
    const double dhr = S.twc[c] - 1.0, dhi = S.tws[c];
    const double av2 = dvr * dvr + dvi * dvi, ah2 = dhr * dhr + dhi * dhi;
    const double d1 = a1m1 * (ah2 + av2) + coupling;
    const double d2 = a1m1 + 0.5 * a2m2 * av2 + a2m2 * ah2;
    const double d3 = a1m1 + 0.5 * a2m2 * ah2 + a2m2 * av2;
    const double d4r = -a1m1 * dhr, d4i = -a1m1 * dhi, d5r = -a1m1 * dvr, d5i = -a1m1 * dvi;
    const double d6r = 0.5 * a2m2 * (dhr * dvr + dhi * dvi), d6i = 0.5 * a2m2 * (dhr * dvi - dhi * dvr);
    // den = d1 (d2 d3 - |d6|^2) - conj(d4)(d4 d3 - conj(d6) d5) + conj(d5)(d4 d6 - d2 d5)
    const double t1 = d1 * (d2 * d3 - (d6r * d6r + d6i * d6i));
    const double ar = d4r * d3 - (d6r * d5r + d6i * d5i), ai = d4i * d3 - (d6r * d5i - d6i * d5r);
    const double br = (d4r * d6r - d4i * d6i) - d2 * d5r, bi = (d4r * d6i + d4i * d6r) - d2 * d5i;
    out[0] = d1; out[1] = d2; out[2] = d3;
    out[3] = d4r; out[4] = d4i; out[5] = d5r; out[6] = d5i; out[7] = d6r; out[8] = d6i;
    out[9] = t1 - (d4r * ar + d4i * ai) + (d5r * br + d5i * bi);
    out[10] = -(d4r * ai - d4i * ar) + (d5r * bi - d5i * br);
}


// interleaved complex planes: element e = (re, im) at doubles [2e, 2e+1] (16-byte aligned)
__device__ __forceinline__ double2 cld2(const double* base, int e) { return reinterpret_cast<const double2*>(base)[e]; }
__device__ __forceinline__ void cst2(double* base, int e, double re, double im) {
    reinterpret_cast<double2*>(base)[e] = make_double2(re, im);
}

// forward 2-D DFT of 3 real n x n planes (src[f]) -> spec (3 interleaved complex planes).
// Real input: only the columns kc <= n/2 of the spectrum are formed (the rest is the Hermitian
// mirror); the {u,p} solve and the inverse use that half only.
// One thread per output bin computes all three fields, sharing twiddles and index updates.
template <int NC>  // NC > 0: the kernel side at compile time (unrolled loops, constant divisors)
__device__ void dft3_forward(const AdmmSmem& S, int n_rt, const double* const src[3]) {
    const int n = NC > 0 ? NC : n_rt;
    const int m = n * n, nh = n / 2 + 1;  // columns 0..n/2 (Nyquist included for even n)
    for (int e = threadIdx.x; e < n * nh; e += blockDim.x) {  // rows: T[r][kc] = sum_c x[r][c] w^(kc c)
        const int r = e / nh, kc = e - r * nh;
        const double *x0 = src[0] + r * n, *x1 = src[1] + r * n, *x2 = src[2] + r * n;
        double re0 = 0.0, im0 = 0.0, re1 = 0.0, im1 = 0.0, re2 = 0.0, im2 = 0.0;
        int idx = 0;
        #pragma unroll
        for (int c = 0; c < n; ++c) {
            const double wc = S.twc[idx], ws = S.tws[idx];
            re0 = fma(x0[c], wc, re0); im0 = fma(-x0[c], ws, im0);
            re1 = fma(x1[c], wc, re1); im1 = fma(-x1[c], ws, im1);
            re2 = fma(x2[c], wc, re2); im2 = fma(-x2[c], ws, im2);
            idx += kc;
            if (idx >= n) idx -= n;
        }
        const int o = r * n + kc;
        cst2(S.rowt, o, re0, im0);
        cst2(S.rowt, m + o, re1, im1);
        cst2(S.rowt, 2 * m + o, re2, im2);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * nh; e += blockDim.x) {  // cols: F[kr][kc] = sum_r T[r][kc] w^(kr r)
        const int kr = e / nh, kc = e - kr * nh;
        double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        int idx = 0;
        #pragma unroll
        for (int r = 0; r < n; ++r) {
            const double wc = S.twc[idx], wsn = -S.tws[idx];
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double2 tv = cld2(S.rowt, f * m + r * n + kc);
                const double tr = tv.x, ti = tv.y;
                acc[f][0] = fma(tr, wc, fma(-ti, wsn, acc[f][0]));
                acc[f][1] = fma(tr, wsn, fma(ti, wc, acc[f][1]));
            }
            idx += kr;
            if (idx >= n) idx -= n;
        }
#pragma unroll
        for (int f = 0; f < 3; ++f) cst2(S.spec, f * m + kr * n + kc, acc[f][0], acc[f][1]);
    }
    __syncthreads();
}

// inverse 2-D DFT of the half spectrum -> dst[f] = Re(.) / m  (fft_util.cpp:47-56): first over kr
// for the columns kc <= (n-1)/2, then the real inverse over kc using the Hermitian mirror:
// x = (Re H[0] + 2 sum_{kc >= 1} Re(H[kc] w^(-kc c))) / m.
template <int NC>
__device__ void dft3_inverse(const AdmmSmem& S, int n_rt, double* const dst[3]) {
    const int n = NC > 0 ? NC : n_rt;
    const int m = n * n, K2 = (n - 1) / 2, nh = n / 2 + 1;
    for (int e = threadIdx.x; e < n * nh; e += blockDim.x) {  // H[r][kc] = sum_kr F[kr][kc] w^(-kr r)
        const int r = e / nh, kc = e - r * nh;
        double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        int idx = 0;
        #pragma unroll
        for (int kr = 0; kr < n; ++kr) {
            const double wc = S.twc[idx], wsn = S.tws[idx];
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double2 fv = cld2(S.spec, f * m + kr * n + kc);
                acc[f][0] = fma(fv.x, wc, fma(-fv.y, wsn, acc[f][0]));
                acc[f][1] = fma(fv.x, wsn, fma(fv.y, wc, acc[f][1]));
            }
            idx += r;
            if (idx >= n) idx -= n;
        }
#pragma unroll
        for (int f = 0; f < 3; ++f) cst2(S.rowt, f * m + r * n + kc, acc[f][0], acc[f][1]);
    }
    __syncthreads();
    const double inv = 1.0 / static_cast<double>(m);
    for (int e = threadIdx.x; e < m; e += blockDim.x) {  // real inverse over kc
        const int r = e / n, c = e - r * n;
        double re[3];
#pragma unroll
        for (int f = 0; f < 3; ++f) re[f] = 0.0;
        int idx = c;
        #pragma unroll
        for (int kc = 1; kc <= K2; ++kc) {
            const double wc = S.twc[idx], ws = S.tws[idx];
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double2 hv = cld2(S.rowt, f * m + r * n + kc);
                re[f] = fma(hv.x, wc, fma(-hv.y, ws, re[f]));
            }
            idx += c;
            if (idx >= n) idx -= n;
        }
        double ny[3] = {0.0, 0.0, 0.0};  // even n: the Nyquist column counts once
        if ((n & 1) == 0) {
            const int ix = (c * (n / 2)) % n;
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double2 hv = cld2(S.rowt, f * m + r * n + n / 2);
                ny[f] = hv.x * S.twc[ix] - hv.y * S.tws[ix];
            }
        }
#pragma unroll
        for (int f = 0; f < 3; ++f) dst[f][e] = (cld2(S.rowt, f * m + r * n).x + 2.0 * re[f] + ny[f]) * inv;
    }
    __syncthreads();
}

// block-wide max of a double (exact), NTADMM threads, warp shuffles + one shared pass
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = red[0];
    for (int w = 1; w < NTADMM / 32; ++w) r = fmax(r, red[w]);
    __syncthreads();
    return r;
}

// {u,p} solve (kernel_estimator.cpp:137-233) on fields in shared memory; writes u -> uout,
// p1 -> p1out, p2 -> p2out. anchor (nullable) already holds z - L3.
template <int NC>
__device__ void up_solve(const AdmmSmem& S, int n_rt, double a1m1, double a2m2, double coupling, const double* x0,
                         const double* x1, const double* y0, const double* y1, const double* y2, const double* y3,
                         const double* L10, const double* L11, const double* L20, const double* L21, const double* L22,
                         const double* L23, const double* anchor, double* uout, double* p1out, double* p2out) {
    const int n = NC > 0 ? NC : n_rt;
    const int m = n * n;
    UPROF_T0
    double* B1 = uout;  // the output planes hold the right-hand sides
    double* B2 = p1out;
    double* B3 = p2out;
    // right-hand sides (kernel_estimator.cpp:151-162), differences of the fields formed inline
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int r = i / n, c = i - r * n;
        const int cl = r * n + (c + n - 1) % n, ru = ((r + n - 1) % n) * n + c;  // left / upper neighbours
        auto x1m = [&](int k) { return x0[k] - L10[k]; };
        auto x2m = [&](int k) { return x1[k] - L11[k]; };
        auto y1m = [&](int k) { return y0[k] - L20[k]; };
        auto y2m = [&](int k) { return y3[k] - L23[k]; };
        auto ycm = [&](int k) { return (((y1[k] - L21[k]) + y2[k]) - L22[k]) * 0.5; };
        const double g1 = x1m(cl) - x1m(i), g2 = x2m(ru) - x2m(i);  // ops.cpp:87-97
        const double h1 = y1m(cl) - y1m(i), h2 = ycm(ru) - ycm(i);
        const double k1 = y2m(ru) - y2m(i), k2 = ycm(cl) - ycm(i);
        double b1 = (g1 + g2) * a1m1;
        if (coupling > 0.0 && anchor) b1 = b1 + anchor[i] * coupling;
        const double b2 = (x1m(i) * -a1m1) + (h1 + h2) * a2m2;
        const double b3 = (x2m(i) * -a1m1) + (k1 + k2) * a2m2;
        B1[i] = b1;
        B2[i] = b2;
        B3[i] = b3;
    }
    __syncthreads();
    UPROF(0)
    const double* src[3] = {B1, B2, B3};
    dft3_forward<NC>(S, n, src);
    UPROF(1)
    double tol;
    if (S.sym) {
        tol = S.sym[11 * m];
    } else {  // max |den| for the singular tolerance (kernel_estimator.cpp:174-197)
        double dmax = 0.0, sy[11];
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            up_symbol(S, n, i, a1m1, a2m2, coupling, sy);
            dmax = fmax(dmax, sqrt(sy[9] * sy[9] + sy[10] * sy[10]));
        }
        tol = 1e-12 * block_max(dmax, S.red);
    }
    const int nh = n / 2 + 1;
    for (int e = threadIdx.x; e < n * nh; e += blockDim.x) {  // half spectrum (real fields)
        const int i = (e / nh) * n + (e % nh);
        double sy[11];
        if (S.sym) {
#pragma unroll
            for (int q = 0; q < 11; ++q) sy[q] = S.sym[q * m + i];
        } else {
            up_symbol(S, n, i, a1m1, a2m2, coupling, sy);
        }
        const double d1 = sy[0], d2 = sy[1], d3 = sy[2];
        // complex helpers
        struct Z { double x, y; };
        auto mul = [](Z a, Z b) { return Z{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; };
        auto cj = [](Z a) { return Z{a.x, -a.y}; };
        auto sub = [](Z a, Z b) { return Z{a.x - b.x, a.y - b.y}; };
        auto add = [](Z a, Z b) { return Z{a.x + b.x, a.y + b.y}; };
        auto rs = [](double s, Z a) { return Z{s * a.x, s * a.y}; };
        const Z d4{sy[3], sy[4]}, d5{sy[5], sy[6]}, d6{sy[7], sy[8]};
        const double n6 = d6.x * d6.x + d6.y * d6.y;
        const Z den{sy[9], sy[10]};
        const double2 s1 = cld2(S.spec, i), s2 = cld2(S.spec, m + i), s3 = cld2(S.spec, 2 * m + i);
        Z b1{s1.x, s1.y}, b2{s2.x, s2.y}, b3{s3.x, s3.y};
        Z fu, fp1, fp2;
        const double aden = sqrt(den.x * den.x + den.y * den.y);
        if (aden > tol) {
            const Z nu = add(sub(rs(d2 * d3 - n6, b1), mul(cj(d4), sub(rs(d3, b2), mul(cj(d6), b3)))),
                             mul(cj(d5), sub(mul(b2, d6), rs(d2, b3))));
            const Z np1 = add(sub(rs(d1, sub(rs(d3, b2), mul(cj(d6), b3))), mul(b1, sub(rs(d3, d4), mul(cj(d6), d5)))),
                              mul(cj(d5), sub(mul(d4, b3), mul(b2, d5))));
            const Z np2 = add(sub(rs(d1, sub(rs(d2, b3), mul(d6, b2))), mul(cj(d4), sub(mul(d4, b3), mul(b2, d5)))),
                              mul(b1, sub(mul(d4, d6), rs(d2, d5))));
            const double dd = den.x * den.x + den.y * den.y;
            auto divz = [&](Z a) { return Z{(a.x * den.x + a.y * den.y) / dd, (a.y * den.x - a.x * den.y) / dd}; };
            fu = divz(nu);
            fp1 = divz(np1);
            fp2 = divz(np2);
        } else {
            // rank-deficient bin (DC with coupling 0): the system is diag(d1, d2, d3) there,
            // whose minimum-norm solution is the pseudo-inverse (kernel_estimator.cpp:213-225)
            const double dtol = 1e-12 * fmax(fabs(d1), fmax(fabs(d2), fabs(d3)));
            fu = fabs(d1) > dtol ? rs(1.0 / d1, b1) : Z{0.0, 0.0};
            fp1 = fabs(d2) > dtol ? rs(1.0 / d2, b2) : Z{0.0, 0.0};
            fp2 = fabs(d3) > dtol ? rs(1.0 / d3, b3) : Z{0.0, 0.0};
        }
        cst2(S.spec, i, fu.x, fu.y);
        cst2(S.spec, m + i, fp1.x, fp1.y);
        cst2(S.spec, 2 * m + i, fp2.x, fp2.y);
    }
    __syncthreads();
    UPROF(2)
    double* dst[3] = {uout, p1out, p2out};
    dft3_inverse<NC>(S, n, dst);
    UPROF(3)
}

// TV u-step (kernel_estimator.cpp:356-364): u = F^-1( F(B1) / d1 ) with
// B1 = (grad_h^T (x0 - L1_0) + grad_v^T (x1 - L1_1)) alpha1 mu1 + anchor mu3. p stays zero, so the
// TGV x-step, y-step and multipliers of k_admm reduce to the TV ones exactly (y = L2 = 0).
template <int NC>
__device__ void tv_solve(const AdmmSmem& S, int n_rt, double a1m1, double mu3, const double* x0, const double* x1,
                         const double* L10, const double* L11, const double* anchor, const double* __restrict__ d1,
                         double* uout, double* scratch) {
    const int n = NC > 0 ? NC : n_rt;
    const int m = n * n;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int r = i / n, c = i - r * n;
        const int cl = r * n + (c + n - 1) % n, ru = ((r + n - 1) % n) * n + c;
        const double g1 = (x0[cl] - L10[cl]) - (x0[i] - L10[i]);  // ops.cpp:87-97
        const double g2 = (x1[ru] - L11[ru]) - (x1[i] - L11[i]);
        uout[i] = (g1 + g2) * a1m1 + anchor[i] * mu3;
    }
    __syncthreads();
    const double* src[3] = {uout, uout, uout};
    dft3_forward<NC>(S, n, src);
    const int nh = n / 2 + 1;
    for (int e = threadIdx.x; e < n * nh; e += blockDim.x) {
        const int i = (e / nh) * n + (e % nh);
        const double2 v = cld2(S.spec, i);
        const double d = __ldg(d1 + i);
        cst2(S.spec, i, v.x / d, v.y / d);
    }
    __syncthreads();
    double* dst[3] = {uout, scratch, scratch};
    dft3_inverse<NC>(S, n, dst);
}

// deterministic block sum for NTADMM threads
__device__ __forceinline__ double admm_sum(double v, double* red) { return block_sum<NTADMM>(v, red); }

// Euclidean projection onto the simplex (kernel_estimator.cpp:112-128) by ranks: element i
// takes the position it would have in a descending sort (ties by index); its cumulative sum
// and candidate threshold follow; tau comes from the largest-rank qualifying element.
__device__ int project_simplex_block(const double* v, double* out, int m, double* red, int* ired) {
    int best_rank = 0;
    double best_tau = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double vi = v[i];
        double css = 0.0;
        int cnt = 0;
        for (int k = 0; k < m; ++k) {
            const double vk = v[k];
            const bool in = vk > vi || (vk == vi && k <= i);
            css += in ? vk : 0.0;
            cnt += in;
        }
        const double cand = (1.0 - css) / static_cast<double>(cnt);
        if (vi + cand > 0.0 && cnt > best_rank) {
            best_rank = cnt;
            best_tau = cand;
        }
    }
    // arg-max of the qualifying rank (ranks are distinct, so the winner is unique)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int orank = __shfl_xor_sync(0xffffffffu, best_rank, o);
        const double otau = __shfl_xor_sync(0xffffffffu, best_tau, o);
        if (orank > best_rank) {
            best_rank = orank;
            best_tau = otau;
        }
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        ired[threadIdx.x >> 5] = best_rank;
        red[threadIdx.x >> 5] = best_tau;
    }
    __syncthreads();
    int support = ired[0];
    double tau = red[0];
    for (int w = 1; w < static_cast<int>(blockDim.x) / 32; ++w)
        if (ired[w] > support) {
            support = ired[w];
            tau = red[w];
        }
    if (support > 0)
        for (int i = threadIdx.x; i < m; i += blockDim.x) out[i] = fmax(v[i] + tau, 0.0);
    __syncthreads();
    return support;
}

// Same projection for m <= NTADMM, in O(log^2) steps: a bitonic sort of (value desc, index asc)
// with one element per thread (partners within a warp by shuffles, across warps through shared
// memory, double-buffered), the cumulative sums in sorted order by a block scan, and the largest
// qualifying position by a block max. scratch: 3 * NTADMM doubles.
__device__ int project_simplex_sorted(const double* v, double* out, int m, double* red, int* ired, double* scratch) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    // values only: equal values are interchangeable in the running sums, so no index tie-break
    double* kv[2] = {scratch, scratch + NTADMM};
    double val = t < m ? v[t] : -INFINITY;
    int buf = 0;
    for (int k = 2; k <= NTADMM; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            double pv;
            if (j >= 32) {
                kv[buf][t] = val;
                __syncthreads();
                pv = kv[buf][t ^ j];
                buf ^= 1;  // the next exchange writes the other buffer: one barrier per stage
            } else {
                pv = __shfl_xor_sync(0xffffffffu, val, j);
            }
            // keep the larger value on the lower position of an ascending block (descending sort)
            const bool want_first = ((t & j) == 0) == ((t & k) == 0);
            const bool own_first = val > pv;
            if (own_first != want_first) val = pv;
        }
    }
    // thread t holds the t-th largest value; inclusive scan in sorted order
    double css = t < m ? val : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, css, o);
        if (lane >= o) css += y;
    }
    if (lane == 31) red[wid] = css;
    __syncthreads();
    if (wid == 0) {
        double x = lane < NTADMM / 32 ? red[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < NTADMM / 32) red[NTADMM / 32 + lane] = x;  // inclusive warp prefixes
    }
    __syncthreads();
    if (wid > 0) css += red[NTADMM / 32 + wid - 1];
    // largest qualifying position (kernel_estimator.cpp:118-124)
    const double cand = (1.0 - css) / static_cast<double>(t + 1);
    const int q = (t < m && val + cand > 0.0) ? t : -1;
    const int wq = __reduce_max_sync(0xffffffffu, q);
    __syncthreads();  // red is reused
    if (lane == 0) ired[wid] = wq;
    __syncthreads();
    int rho = -1;
    for (int w = 0; w < NTADMM / 32; ++w) rho = max(rho, ired[w]);
    if (t == rho) red[0] = cand;
    __syncthreads();
    const double tau = red[0];
    if (rho >= 0)
        for (int i = t; i < m; i += NTADMM) out[i] = fmax(v[i] + tau, 0.0);
    __syncthreads();
    return rho + 1;
}

size_t admm_smem_doubles(int n, int cs = 1, bool ginv_global = false) {
    const size_t m = static_cast<size_t>(n) * n, rp = (m + cs - 1) / cs;
    return static_cast<size_t>(17 + 3 + 6 + 6) * m + admm_scratch_doubles(static_cast<int>(m)) + 2 * n + NTADMM +
           NTADMM / 2 + 4 + 8 + (cs > 1 ? (ginv_global ? 0 : rp * m) + 2 * rp : 0);
}

// CS > 1: the CTAs of a thread-block cluster run the same (deterministic, bit-identical) ADMM
// on one scene; each holds rows [crank*RP, crank*RP+RP) of the symmetric inverse in shared
// memory, computes that slice of the z-step mat-vec, and the slices are all-gathered through
// distributed shared memory (one cluster barrier per iteration, slices double-buffered).
template <int NC>  // NC > 0: kernel side known at compile time (n = 15, 17, 21: the BASELINE configs)
__global__ void __launch_bounds__(NTADMM) k_admm(AdmmArgs A, const double* __restrict__ Ginv_all,
                                                 const double* __restrict__ Etf_all, double* __restrict__ state_all,
                                                 int* __restrict__ info_all, double* __restrict__ k_out, int CS) {
    namespace cg = cooperative_groups;
    extern __shared__ double smem[];
    const int s = blockIdx.x / CS, crank = blockIdx.x - (blockIdx.x / CS) * CS;
    const int n = NC > 0 ? NC : A.n, m = n * n;
    const int RP = (m + CS - 1) / CS, r_lo = min(m, crank * RP), r_hi = min(m, r_lo + RP);
    const double* Ginv = Ginv_all + static_cast<size_t>(s) * m * m;
    const double* Etf = Etf_all + static_cast<size_t>(s) * m;
    double* gstate = state_all + static_cast<size_t>(s) * 17 * m;
    int* info = info_all + s * 4;
    AdmmSmem S;
    double* p = smem;
    for (int f = 0; f < 17; ++f) { S.f[f] = p; p += m; }
    S.bz = p; p += m;
    S.zz = p; p += m;
    S.unew = p; p += m;
    S.tmp6 = p; p += admm_scratch_doubles(m);  // projection scratch (sorted projection only)
    S.spec = p; p += 6 * m;
    S.rowt = p; p += 6 * m;
    S.twc = p; p += n;
    S.tws = p; p += n;
    S.red = p; p += NTADMM;
    int* ired = reinterpret_cast<int*>(p);
    p += NTADMM / 2 + 4;
    const bool gglob = A.ginv_global != 0;
    double* Gs = p;          // CS > 1: rows [r_lo, r_hi) of the inverse (unless gglob)
    p += (CS > 1 && !gglob) ? static_cast<size_t>(RP) * m : 0;
    double* zsl = p;         // CS > 1: 2 x RP mat-vec slice (double-buffered by iteration parity)
    p += (CS > 1) ? 2 * RP : 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const double wv = 2.0 * M_PI * k / n;
        S.twc[k] = cos(wv);
        S.tws[k] = sin(wv);
    }
    if (A.cache_symbols) {  // symbols and singular tolerance are iteration-independent
        S.sym = p;
        __syncthreads();
        double dmax = 0.0, sy[11];
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            up_symbol(S, n, i, A.alpha1 * A.mu1, A.alpha2 * A.mu2, A.coupling, sy);
#pragma unroll
            for (int q = 0; q < 11; ++q) S.sym[q * m + i] = sy[q];
            dmax = fmax(dmax, sqrt(sy[9] * sy[9] + sy[10] * sy[10]));
        }
        const double tol = 1e-12 * block_max(dmax, S.red);
        if (threadIdx.x == 0) S.sym[11 * m] = tol;
    }
    if (CS > 1 && !gglob)
        for (size_t e = threadIdx.x; e < static_cast<size_t>(r_hi - r_lo) * m; e += blockDim.x)
            Gs[e] = __ldg(Ginv + static_cast<size_t>(r_lo) * m + e);
    // field f lives at smem + f m, except u, which alternates with u_new (pointer swap); no
    // pointer array, so nothing is indexed dynamically through local memory
    double* const fb = smem;
    double* Ucur = fb + F_U * m;
    double* Unew = S.unew;
#define FLD(f) ((f) == F_U ? Ucur : fb + (f) * m)
    if (A.init_state) {  // kernel_estimator.cpp:297-307
        const int cc = (n - 1) / 2;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double u0 = A.init_kind == 0 ? (i == cc * n + cc ? 1.0 : 0.0) : 1.0 / (static_cast<double>(n) * n);
            FLD(F_U)[i] = u0;
            FLD(F_Z)[i] = u0;
            for (int f = F_P1; f <= F_L3; ++f)
                if (f != F_Z) FLD(f)[i] = 0.0;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const int r = i / n, c = i - r * n;
            FLD(F_X0)[i] = FLD(F_U)[r * n + (c + 1) % n] - FLD(F_U)[i];
            FLD(F_X1)[i] = FLD(F_U)[((r + 1) % n) * n + c] - FLD(F_U)[i];
        }
    } else {
        for (int e = threadIdx.x; e < 17 * m; e += blockDim.x) FLD(e / m)[e % m] = gstate[e];
    }
    __syncthreads();
    const double a1m1 = A.alpha1 * A.mu1, a2m2 = A.alpha2 * A.mu2;
    const double t1 = 1.0 / A.mu1, t2 = 1.0 / A.mu2;
    int status = 0, iters = A.t_begin, t = A.t_begin;
    int phase = A.phase_begin;
    APROF_T0
    for (; t < A.t_max; ++t) {
        if (phase == 0) {
            // x-step and y-step (kernel_estimator.cpp:325-337), z-step right-hand side (:340)
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const int r = i / n, c = i - r * n;
                const int ir = r * n + (c + 1) % n, id = ((r + 1) % n) * n + c;
                const double* u = FLD(F_U);
                const double* p1 = FLD(F_P1);
                const double* p2 = FLD(F_P2);
                double a0 = ((u[ir] - u[i]) - p1[i]) + FLD(F_L10)[i];
                double a1 = ((u[id] - u[i]) - p2[i]) + FLD(F_L11)[i];
                const double nrm = sqrt(a0 * a0 + a1 * a1);
                const double sc = nrm > t1 ? (nrm - t1) / nrm : 0.0;
                FLD(F_X0)[i] = a0 * sc;
                FLD(F_X1)[i] = a1 * sc;
                const double e0 = p1[ir] - p1[i];
                const double cr = ((p1[id] - p1[i]) + (p2[ir] - p2[i])) * 0.5;
                const double e3 = p2[id] - p2[i];
                const double b0 = e0 + FLD(F_L20)[i], b1 = cr + FLD(F_L21)[i], b2 = cr + FLD(F_L22)[i],
                             b3 = e3 + FLD(F_L23)[i];
                const double nrm2 = sqrt(b0 * b0 + b1 * b1 + b2 * b2 + b3 * b3);
                const double sc2 = nrm2 > t2 ? (nrm2 - t2) / nrm2 : 0.0;
                FLD(F_Y0)[i] = b0 * sc2;
                FLD(F_Y1)[i] = b1 * sc2;
                FLD(F_Y2)[i] = b2 * sc2;
                FLD(F_Y3)[i] = b3 * sc2;
                S.bz[i] = Etf[i] + A.mu3 * (u[i] + FLD(F_L3)[i]);
            }
            __syncthreads();
            APROF(0)
            // z = project_simplex((E^T E + mu3 I)^-1 (E^T f + mu3 (u + L3)))   (:341, :79-83)
            if (CS > 1) {
                double* mine = zsl + (t & 1) * RP;
                const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
                for (int i = r_lo + warp; i < r_hi; i += NTADMM / 32) {
                    double acc = 0.0;
                    if (gglob) {
                        const double* row = Ginv + static_cast<size_t>(i) * m;
                        for (int j = lane; j < m; j += 32) acc = fma(__ldg(row + j), S.bz[j], acc);
                    } else {
                        const double* row = Gs + static_cast<size_t>(i - r_lo) * m;
                        for (int j = lane; j < m; j += 32) acc = fma(row[j], S.bz[j], acc);
                    }
                    acc = warp_sum(acc);
                    if (lane == 0) mine[i - r_lo] = acc;
                }
                cg::this_cluster().sync();
                for (int i = threadIdx.x; i < m; i += blockDim.x) {
                    const int owner = i / RP;
                    const double* rem = cg::this_cluster().map_shared_rank(zsl, owner);
                    S.zz[i] = rem[(t & 1) * RP + (i - owner * RP)];
                }
            } else {
                for (int i = threadIdx.x; i < m; i += blockDim.x) {
                    double a0 = 0.0, a1 = 0.0;
                    int j = 0;
                    for (; j + 1 < m; j += 2) {
                        a0 = fma(__ldg(Ginv + static_cast<size_t>(j) * m + i), S.bz[j], a0);
                        a1 = fma(__ldg(Ginv + static_cast<size_t>(j + 1) * m + i), S.bz[j + 1], a1);
                    }
                    if (j < m) a0 = fma(__ldg(Ginv + static_cast<size_t>(j) * m + i), S.bz[j], a0);
                    S.zz[i] = a0 + a1;
                }
            }
            __syncthreads();
            APROF(1)
            bool finite = true;
            for (int i = threadIdx.x; i < m; i += blockDim.x) finite = finite && isfinite(S.zz[i]);
            if (!__syncthreads_and(finite)) { status = 3; iters = t; break; }
            APROF(2)
            const int support = m <= NTADMM ? project_simplex_sorted(S.zz, FLD(F_Z), m, S.red, ired, S.tmp6)
                                             : project_simplex_block(S.zz, FLD(F_Z), m, S.red, ired);
            APROF(3)
            if (support == 0) { status = 3; iters = t; break; }
            if (t == A.hook_t) { status = 4; break; }
        }
        phase = 0;
        // {u,p}-step with the mu3 tie to z - L3 (:349-355)
        for (int i = threadIdx.x; i < m; i += blockDim.x) S.bz[i] = FLD(F_Z)[i] - FLD(F_L3)[i];
        __syncthreads();
        APROF(4)
        // old p1, p2 are dead after the y-step: the solve writes them in place, u_new separately
        if (A.tv_d1)
            tv_solve<NC>(S, n, a1m1, A.mu3, FLD(F_X0), FLD(F_X1), FLD(F_L10), FLD(F_L11), S.bz, A.tv_d1, Unew, S.zz);
        else
            up_solve<NC>(S, n, a1m1, a2m2, A.coupling, FLD(F_X0), FLD(F_X1), FLD(F_Y0), FLD(F_Y1), FLD(F_Y2), FLD(F_Y3),
                     FLD(F_L10), FLD(F_L11), FLD(F_L20), FLD(F_L21), FLD(F_L22), FLD(F_L23), S.bz, Unew, FLD(F_P1),
                     FLD(F_P2));
        APROF(5)
        // multipliers (:367-373), change of u (:375-376)
        double dd = 0.0, un = 0.0;
        bool fin_u = true, fin_z = true;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const int r = i / n, c = i - r * n;
            const int ir = r * n + (c + 1) % n, id = ((r + 1) % n) * n + c;
            const double* u1 = Unew;
            const double* p1 = FLD(F_P1);
            const double* p2 = FLD(F_P2);
            FLD(F_L10)[i] += (((u1[ir] - u1[i]) - p1[i]) - FLD(F_X0)[i]) * A.rho;
            FLD(F_L11)[i] += (((u1[id] - u1[i]) - p2[i]) - FLD(F_X1)[i]) * A.rho;
            const double e0 = p1[ir] - p1[i];
            const double cr = ((p1[id] - p1[i]) + (p2[ir] - p2[i])) * 0.5;
            const double e3 = p2[id] - p2[i];
            FLD(F_L20)[i] += (e0 - FLD(F_Y0)[i]) * A.rho;
            FLD(F_L21)[i] += (cr - FLD(F_Y1)[i]) * A.rho;
            FLD(F_L22)[i] += (cr - FLD(F_Y2)[i]) * A.rho;
            FLD(F_L23)[i] += (e3 - FLD(F_Y3)[i]) * A.rho;
            FLD(F_L3)[i] += (u1[i] - FLD(F_Z)[i]) * A.rho;
            const double du = FLD(F_U)[i] - u1[i];
            dd += du * du;
            un += u1[i] * u1[i];
            fin_u = fin_u && isfinite(u1[i]);
            fin_z = fin_z && isfinite(FLD(F_Z)[i]);
        }
        const double delta = sqrt(admm_sum(dd, S.red));
        const double scale = fmax(sqrt(admm_sum(un, S.red)), 1e-300);
        const bool all_u = __syncthreads_and(fin_u);
        const bool all_z = __syncthreads_and(fin_z);
        {  // u <- u_new by swapping the buffers (all threads hold the same pointers)
            double* tmp = Ucur;
            Ucur = Unew;
            Unew = tmp;
        }
        iters = t + 1;
        APROF(6)
        if (!all_u) { status = 1; break; }  // check_finite (:379-380)
        if (!all_z) { status = 2; break; }
        if (delta / scale < A.th) { ++t; break; }
    }
    APROF_END
    if (crank == 0) {
        for (int e = threadIdx.x; e < 17 * m; e += blockDim.x) gstate[e] = FLD(e / m)[e % m];
        if (k_out)
            for (int i = threadIdx.x; i < m; i += blockDim.x) k_out[static_cast<size_t>(s) * m + i] = FLD(F_Z)[i];
        if (threadIdx.x == 0) {
            info[0] = iters;
            info[1] = status;
            info[2] = t;
            info[3] = 0;
        }
    }
    if (CS > 1) cg::this_cluster().sync();  // no CTA leaves while a peer may still read its slice
#undef FLD
}

// standalone {u,p} solve for the public solve_up (kernel_estimator.cpp:237-241)
__global__ void __launch_bounds__(NTADMM) k_solve_up(int n, double a1m1, double a2m2, double coupling,
                                                     const double* __restrict__ fields, const double* __restrict__ anchor,
                                                     double* __restrict__ u, double* __restrict__ p1,
                                                     double* __restrict__ p2) {
    extern __shared__ double smem[];
    const int m = n * n;
    AdmmSmem S;
    double* p = smem;
    double* fl[12];
    for (int f = 0; f < 12; ++f) { fl[f] = p; p += m; }
    double* anc = p; p += m;
    double* uo = p; p += m;
    double* p1o = p; p += m;
    double* p2o = p; p += m;
    S.tmp6 = p; p += 6 * m;
    S.spec = p; p += 6 * m;
    S.rowt = p; p += 6 * m;
    S.twc = p; p += n;
    S.tws = p; p += n;
    S.red = p; p += NTADMM;
    for (int e = threadIdx.x; e < 12 * m; e += blockDim.x) fl[e / m][e % m] = fields[e];
    for (int i = threadIdx.x; i < m; i += blockDim.x) anc[i] = anchor ? anchor[i] : 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const double wv = 2.0 * M_PI * k / n;
        S.twc[k] = cos(wv);
        S.tws[k] = sin(wv);
    }
    __syncthreads();
    up_solve<0>(S, n, a1m1, a2m2, coupling, fl[0], fl[1], fl[2], fl[3], fl[4], fl[5], fl[6], fl[7], fl[8], fl[9], fl[10],
             fl[11], anchor ? anc : nullptr, uo, p1o, p2o);
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        u[i] = uo[i];
        p1[i] = p1o[i];
        p2[i] = p2o[i];
    }
}

__global__ void k_shrink2(double* __restrict__ cols, int ncols, long long m, double t) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double n2 = 0.0;
        for (int j = 0; j < ncols; ++j) n2 += cols[j * m + i] * cols[j * m + i];
        const double nrm = sqrt(n2);
        const double sc = nrm > t ? (nrm - t) / nrm : 0.0;
        for (int j = 0; j < ncols; ++j) cols[j * m + i] *= sc;
    }
}

__global__ void __launch_bounds__(NTADMM) k_project(const double* __restrict__ v, int m, double* __restrict__ out,
                                                    int* __restrict__ status) {
    extern __shared__ double sh[];
    double* vs = sh;
    double* os = sh + m;
    double* red = os + m;
    int* ired = reinterpret_cast<int*>(red + NTADMM);
    double* scratch = red + NTADMM + NTADMM / 2 + 4;
    for (int i = threadIdx.x; i < m; i += blockDim.x) vs[i] = v[i];
    __syncthreads();
    const int support = m <= NTADMM ? project_simplex_sorted(vs, os, m, red, ired, scratch)
                                    : project_simplex_block(vs, os, m, red, ired);
    if (threadIdx.x == 0) *status = support == 0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) out[i] = os[i];
}

}  // namespace

// =============================================================================================
// host wrappers
// =============================================================================================
void validate_ke(const fbmp_ke_params& p) {  // kernel_estimator.cpp:36-45
    if (p.n < 1 || p.n % 2 == 0) param_error("kernel estimation: n must be odd and positive");
    if (p.alpha1 <= 0 || p.alpha2 <= 0) param_error("kernel estimation: alpha weights must be positive");
    if (p.mu1 <= 0 || p.mu2 <= 0 || p.mu3 <= 0) param_error("kernel estimation: mu penalties must be positive");
    const double rho_max = (1.0 + std::sqrt(5.0)) / 2.0;
    if (!(p.rho > 0 && p.rho < rho_max)) param_error("kernel estimation: rho must lie in (0, (1+sqrt(5))/2)");
    if (!(p.th > 0)) param_error("kernel estimation: th must be positive");
    if (p.t_max < 1) param_error("kernel estimation: t_max must be >= 1");
}

void solve_weights_device(Context& ctx, const double* d_lrms, int S, int nb, int h, int w, const double* d_pan, int l,
                          double lambda_omega, int c, double* d_omega, int* d_status) {
    const int H = h * c, W = w * c;
    const long long p = static_cast<long long>(h) * w;
    double* t1 = ctx.scratch<double>("sw_t1", static_cast<size_t>(S) * H * w);
    double* bvec = ctx.scratch<double>("sw_b", static_cast<size_t>(S) * p);
    double* t2 = ctx.scratch<double>("sw_t2", static_cast<size_t>(S) * nb * p);
    double* A = ctx.scratch<double>("sw_A", static_cast<size_t>(S) * nb * p);
    const int hwin = c * l + 1, lwin = l + 1;
    k_blur_h<<<grid1d(ctx, static_cast<long long>(S) * H * w), 256, 0, ctx.stream>>>(d_pan, S, H, W, w, c, hwin, t1);
    k_blur_v<<<grid1d(ctx, static_cast<long long>(S) * p), 256, 0, ctx.stream>>>(t1, S, H, w, h, c, hwin, bvec);
    k_blur_h<<<grid1d(ctx, static_cast<long long>(S) * nb * p), 256, 0, ctx.stream>>>(d_lrms, S * nb, h, w, w, 1, lwin, t2);
    k_blur_v<<<grid1d(ctx, static_cast<long long>(S) * nb * p), 256, 0, ctx.stream>>>(t2, S * nb, h, w, h, 1, lwin, A);
    const int nblk = static_cast<int>(std::max(1LL, std::min<long long>(64, (p + 4095) / 4096)));
    const int nv = nb * (nb + 1) / 2 + nb;
    double* part = ctx.scratch<double>("sw_part", static_cast<size_t>(S) * nblk * nv);
    k_sw_dots<<<dim3(nblk, S), NT, 0, ctx.stream>>>(A, bvec, nb, p, nblk, part);
    const size_t sm = (nv + 3 * nb * nb + 4 * nb + nb) * sizeof(double) + 64;
    k_sw_solve<<<S, 64, sm, ctx.stream>>>(part, nb, nblk, lambda_omega, d_omega, d_status);
    ctx.count(6);
    check_launch();
}

void combine_bands_device(Context& ctx, const double* d_lrms, int S, int nb, long long p, const double* d_omega,
                          double* d_out) {
    k_combine<<<grid1d(ctx, S * p), 256, 0, ctx.stream>>>(d_lrms, S, nb, p, d_omega, d_out);
    ctx.count();
    check_launch();
}

void pan_stats(Context& ctx, const double* d_pan, int S, long long P, double* d_stats) {
    const int nblk = static_cast<int>(std::max(1LL, std::min<long long>(256, (P + 8191) / 8192)));
    double* part = ctx.scratch<double>("stats_part", static_cast<size_t>(S) * nblk * 4);
    k_stats_partial<<<dim3(nblk, S), NT, 0, ctx.stream>>>(d_pan, P, nblk, part);
    k_stats_final<<<S, 32, 0, ctx.stream>>>(part, nblk, d_stats);
    ctx.count(2);
    check_launch();
}

static void gram_T_and_etf(Context& ctx, const double* d_pan, const double* d_obs, int S, int H, int W, int c, int n,
                           const double* d_scale, double* T, double* Etf, bool split = false) {
    const int h = H / c, w = W / c;
    const int ntiles = ceil_div(h, TG) * ceil_div(w, TG);
    const int D = 2 * n - 1, nd = D * D, n2 = n * n;
    const int SR = c * (TG - 1) + 2 * (n - 1) + 1;
    const size_t smT = static_cast<size_t>(SR) * SR * sizeof(double);
    if (smT > 227 * 1024) param_error("build_observation: kernel side too large for the device Gram kernel");
    // rank split (C5 strips): rank r computes tile chunks [k0, k1) and the chunk sums
    // are all-gathered; without a communicator (or G not dividing the chunk count) every chunk here
    const bool dist = split && ctx.nccl && ctx.nranks > 1 && GRAM_CHUNKS % ctx.nranks == 0 && S == 1;
    const int G = dist ? ctx.nranks : 1, rk = dist ? ctx.rank : 0;
    const int k0 = rk * GRAM_CHUNKS / G, k1 = (rk + 1) * GRAM_CHUNKS / G;
    const int t_lo = chunk_tile(k0, ntiles), t_hi = chunk_tile(k1, ntiles), nt = t_hi - t_lo;
    double* partT = ctx.scratch<double>("gram_partT", static_cast<size_t>(S) * ntiles * c * c * nd);
    double* cpT = ctx.scratch<double>("gram_cpT", static_cast<size_t>(S) * GRAM_CHUNKS * c * c * nd);
    if (nt > 0) {
        if (D * ((D + GK - 1) / GK) <= NTG && (c == 1 || c == 2 || c == 4)) {  // register-blocked (n <= 21)
            auto fn = c == 4 ? k_gram_T2<4> : c == 2 ? k_gram_T2<2> : k_gram_T2<1>;
            const size_t smT2 = smT + GK * sizeof(double);
            set_smem(fn, smT2);
            fn<<<dim3(nt, c * c, S), NTG, smT2, ctx.stream>>>(d_pan, d_scale, H, W, h, w, n, partT, ntiles, t_lo);
        } else {
            set_smem(k_gram_T, smT);
            k_gram_T<<<dim3(nt, c * c, S), NT, smT, ctx.stream>>>(d_pan, d_scale, H, W, h, w, c, n, partT, ntiles,
                                                                    t_lo);
        }
        ctx.count();
    }
    k_reduce_chunks<<<grid1d(ctx, static_cast<long long>(S) * (k1 - k0) * c * c * nd), 256, 0, ctx.stream>>>(
        partT, S, ntiles, c * c * nd, k0, k1, cpT);
    const int SRf = c * (TG - 1) + n;
    const size_t smF = (static_cast<size_t>((SRf * SRf + 1) & ~1) + TG * TG) * sizeof(double);
    set_smem(k_gram_etf, smF);
    double* partF = ctx.scratch<double>("gram_partF", static_cast<size_t>(S) * ntiles * n2);
    double* cpF = ctx.scratch<double>("gram_cpF", static_cast<size_t>(S) * GRAM_CHUNKS * n2);
    if (nt > 0)
        k_gram_etf<<<dim3(nt, 1, S), NT, smF, ctx.stream>>>(d_pan, d_obs, d_scale, H, W, h, w, c, n, partF, ntiles,
                                                            t_lo);
    k_reduce_chunks<<<grid1d(ctx, static_cast<long long>(S) * (k1 - k0) * n2), 256, 0, ctx.stream>>>(
        partF, S, ntiles, n2, k0, k1, cpF);
    ctx.count(nt > 0 ? 3 : 2);
    check_launch();
    if (dist) {  // every rank receives all chunk sums (S == 1: chunk k's sums are contiguous)
        auto cm = static_cast<ncclComm_t>(ctx.nccl);
        const size_t nT = static_cast<size_t>(GRAM_CHUNKS / G) * c * c * nd, nF = static_cast<size_t>(GRAM_CHUNKS / G) * n2;
        FBMP_NCCL(ncclGroupStart());
        FBMP_NCCL(ncclAllGather(cpT + static_cast<size_t>(k0) * c * c * nd, cpT, nT, ncclDouble, cm, ctx.stream));
        FBMP_NCCL(ncclAllGather(cpF + static_cast<size_t>(k0) * n2, cpF, nF, ncclDouble, cm, ctx.stream));
        FBMP_NCCL(ncclGroupEnd());
    }
    k_sum_chunks<<<grid1d(ctx, static_cast<long long>(S) * c * c * nd), 256, 0, ctx.stream>>>(cpT, S, c * c * nd, T);
    k_sum_chunks<<<grid1d(ctx, static_cast<long long>(S) * n2), 256, 0, ctx.stream>>>(cpF, S, n2, Etf);
    ctx.count(2);
    check_launch();
}

// z = (E^T E + mu3 I)^-1 (E^T f + mu3 anchor) for a Gram matrix given on the device (the public
// ObservationSystem::solve_z, kernel_estimator.cpp:79-83): Cholesky + explicit inverse + mat-vec
__global__ void k_shift_diag(const double* __restrict__ EtE, int n2, double mu3, double* __restrict__ M) {
    const long long NN = static_cast<long long>(n2) * n2;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < NN;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = e / n2;
        M[e] = (e - r * n2 == r) ? EtE[e] + mu3 : EtE[e];
    }
}
__global__ void k_solve_z_apply(const double* __restrict__ Ginv, const double* __restrict__ Etf,
                                const double* __restrict__ anchor, int n2, double mu3, double* __restrict__ z) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n2) return;
    const double* row = Ginv + static_cast<size_t>(warp) * n2;  // symmetric: row = column
    double acc = 0.0;
    for (int j = lane; j < n2; j += 32) acc = fma(row[j], Etf[j] + mu3 * anchor[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) z[warp] = acc;
}
// 0.5 ||E u - f||^2 = 0.5 (u^T E^T E u - 2 u^T E^T f + f^T f) (kernel_estimator.cpp:85-87), one CTA
__global__ void __launch_bounds__(NT) k_data_objective(const double* __restrict__ EtE, const double* __restrict__ Etf,
                                                       const double* __restrict__ u, int n2, double ff,
                                                       double* __restrict__ out) {
    __shared__ double red[2 * (NT / 32 + 1)];
    double q = 0.0, l = 0.0;
    for (int a = threadIdx.x; a < n2; a += NT) {
        double r = 0.0;
        const double* row = EtE + static_cast<size_t>(a) * n2;
        for (int b = 0; b < n2; ++b) r = fma(row[b], u[b], r);
        q = fma(u[a], r, q);
        l = fma(u[a], Etf[a], l);
    }
    const double2 t = block_sum2<NT>(q, l, red);
    if (threadIdx.x == 0) out[0] = 0.5 * (t.x - 2.0 * t.y + ff);
}
void solve_z_device(Context& ctx, const double* d_EtE, const double* d_Etf, int n2, double mu3,
                    const double* d_anchor, double* d_z) {
    ObsSystem sys;
    sys.S = 1;
    sys.n = 0;
    sys.n2 = n2;
    const size_t NN = static_cast<size_t>(n2) * n2;
    sys.M = ctx.scratch<double>("sz_M", NN);
    sys.Ginv = ctx.scratch<double>("sz_Ginv", NN);
    sys.Etf = nullptr;
    sys.g = nullptr;
    sys.status = ctx.scratch<int>("sz_status", 1);
    k_shift_diag<<<grid1d(ctx, static_cast<long long>(NN)), 256, 0, ctx.stream>>>(d_EtE, n2, mu3, sys.M);
    ctx.count();
    factor_invert(ctx, sys, true);
    int hst = 0;
    d2h(&hst, sys.status, sizeof(int), ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    if (hst) num_error("build_observation: factorization of E^T E + mu3 I failed");
    k_solve_z_apply<<<ceil_div(n2 * 32, 256), 256, 0, ctx.stream>>>(sys.Ginv, d_Etf, d_anchor, n2, mu3, d_z);
    ctx.count();
    check_launch();
}
void data_objective_device(Context& ctx, const double* d_EtE, const double* d_Etf, const double* d_u, int n2,
                           double ff, double* d_out) {
    k_data_objective<<<1, NT, 0, ctx.stream>>>(d_EtE, d_Etf, d_u, n2, ff, d_out);
    ctx.count();
    check_launch();
}

void gram_device(Context& ctx, const double* d_pan, const double* d_obs, int H, int W, int c, int n, double* d_EtE,
                 double* d_Etf) {
    const int D = 2 * n - 1;
    double* T = ctx.scratch<double>("gram_T", static_cast<size_t>(c) * c * D * D);
    gram_T_and_etf(ctx, d_pan, d_obs, 1, H, W, c, n, nullptr, T, d_Etf);
    const long long n2 = static_cast<long long>(n) * n;
    k_gram_expand<<<grid1d(ctx, n2 * n2), 256, 0, ctx.stream>>>(T, 1, c, n, 0.0, d_EtE);
    ctx.count();
    check_launch();
}

// l2 kernel prior (kernel_estimator.cpp:394-407): K = E^T E + 2 a1 grad^T grad + (2 a2 + mu3) I, where
// grad^T grad of the circular forward differences is 4 I minus the four periodic neighbours
__global__ void k_add_l2(double* __restrict__ M, int S, int n, double two_a1, double two_a2) {
    const int m = n * n;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(S) * m;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int s = static_cast<int>(e / m), i = static_cast<int>(e - static_cast<long long>(s) * m);
        double* row = M + (static_cast<size_t>(s) * m + i) * m;
        const int r = i / n, c = i - r * n;
        row[i] += 4.0 * two_a1 + two_a2;
        row[r * n + (c + 1) % n] -= two_a1;
        row[r * n + (c + n - 1) % n] -= two_a1;
        row[((r + 1) % n) * n + c] -= two_a1;
        row[((r + n - 1) % n) * n + c] -= two_a1;
    }
}

void build_observation(Context& ctx, const double* d_pan, const double* d_obs, int S, int H, int W, int c, int n,
                       double mu3, const double* d_scale, ObsSystem& sys, bool want_inverse, double l2_a1,
                       double l2_a2, bool split) {
    const int n2 = n * n, D = 2 * n - 1;
    sys.S = S;
    sys.n = n;
    sys.n2 = n2;
    const size_t NN = static_cast<size_t>(n2) * n2;
    sys.M = ctx.scratch<double>("obs_M", S * NN);
    sys.Etf = ctx.scratch<double>("obs_Etf", static_cast<size_t>(S) * n2);
    sys.Ginv = ctx.scratch<double>("obs_Ginv", S * NN);
    sys.g = nullptr;
    sys.status = ctx.scratch<int>("obs_status", S);
    double* T = ctx.scratch<double>("gram_T", static_cast<size_t>(S) * c * c * D * D);
    gram_T_and_etf(ctx, d_pan, d_obs, S, H, W, c, n, d_scale, T, sys.Etf, split);
    k_gram_expand<<<grid1d(ctx, static_cast<long long>(S) * NN), 256, 0, ctx.stream>>>(T, S, c, n, mu3, sys.M);
    ctx.count();
    if (l2_a1 != 0.0 || l2_a2 != 0.0) {
        k_add_l2<<<grid1d(ctx, static_cast<long long>(S) * n2), 256, 0, ctx.stream>>>(sys.M, S, n, 2.0 * l2_a1,
                                                                                       2.0 * l2_a2);
        ctx.count();
    }
    factor_invert(ctx, sys, want_inverse);
}

// Cholesky of sys.M (S systems of side n2, lower triangle) and, if asked, the explicit inverse
// sys.Ginv = L^-T L^-1 (kernel_estimator.cpp:71-76, :79-83)
void factor_invert(Context& ctx, ObsSystem& sys, bool want_inverse) {
    const int S = sys.S, n2 = sys.n2;
    const size_t NN = static_cast<size_t>(n2) * n2;
    FBMP_CUDA(cudaMemsetAsync(sys.status, 0, sizeof(int) * S, ctx.stream));
    const int N = n2;
    const size_t smP = static_cast<size_t>(N) * (NBK + 1) * sizeof(double);
    if (smP > 227 * 1024) param_error("build_observation: kernel side too large for the device Cholesky");
    set_smem(k_potrf_panel, smP);
    for (int K = 0; K < N; K += NBK) {
        k_potrf_panel<<<S, NT, smP, ctx.stream>>>(sys.M, N, K, sys.status);
        ctx.count();
        if (K + NBK < N) {
            const int nt = ceil_div(N - K - NBK, NBK);
            k_syrk<<<dim3(nt * (nt + 1) / 2, S), NT, 0, ctx.stream>>>(sys.M, N, K, sys.status);
            ctx.count();
        }
    }
    check_launch();
    if (!want_inverse) return;
    double* Linv = ctx.scratch<double>("obs_Linv", S * NN);
    const size_t smT = static_cast<size_t>(NT / 32) * N * sizeof(double);
    const int KL = ceil_div(N, 32);
    auto tfn = KL <= 4 ? k_trtri_pf<4> : KL <= 8 ? k_trtri_pf<8> : KL <= 10 ? k_trtri_pf<10> : KL <= 14 ? k_trtri_pf<14>
                                                                                                   : k_trtri_pf<27>;
    set_smem(tfn, smT);
    tfn<<<dim3(ceil_div(N, NT / 32), S), NT, smT, ctx.stream>>>(sys.M, N, Linv, sys.status);
    const int nt = ceil_div(N, NBK);
    k_inv_gram<<<dim3(nt * (nt + 1) / 2, S), NT, 0, ctx.stream>>>(Linv, N, sys.Ginv, sys.status);
    ctx.count(2);
    check_launch();
}

void admm_device(Context& ctx, const ObsSystem& sys, const fbmp_ke_params& prm, double* d_state, bool init_state,
                 int t_begin, int phase_begin, int hook_t, int* d_info, double* d_k, bool tv = false) {
    AdmmArgs A;
    A.tv_d1 = nullptr;
    if (tv) {  // kernel_estimator.cpp:309-321, evaluated on the host as the reference does
        const int n = sys.n;
        std::vector<double> d1(static_cast<size_t>(n) * n);
        for (int r = 0; r < n; ++r) {
            const double av2 = 2.0 - 2.0 * std::cos(2.0 * M_PI * r / n);
            for (int c = 0; c < n; ++c) {
                const double ah2 = 2.0 - 2.0 * std::cos(2.0 * M_PI * c / n);
                d1[static_cast<size_t>(r) * n + c] = prm.alpha1 * prm.mu1 * (ah2 + av2) + prm.mu3;
            }
        }
        double* dd = ctx.scratch<double>("admm_tv_d1", d1.size());
        h2d(dd, d1.data(), d1.size() * sizeof(double), ctx.stream);
        A.tv_d1 = dd;
    }
    A.n = sys.n;
    A.m = sys.n2;
    A.alpha1 = prm.alpha1;
    A.alpha2 = prm.alpha2;
    A.mu1 = prm.mu1;
    A.mu2 = prm.mu2;
    A.mu3 = prm.mu3;
    A.rho = prm.rho;
    A.th = prm.th;
    A.coupling = prm.mu3;
    A.t_max = prm.t_max;
    A.t_begin = t_begin;
    A.phase_begin = phase_begin;
    A.hook_t = hook_t;
    A.init_kind = prm.init;
    A.init_state = init_state ? 1 : 0;
    // cluster size: the smallest power of two whose inverse slice fits next to the ADMM state
    int cs = 1;
    const char* env = std::getenv("FBMP_ADMM_CLUSTER");
    const int cs_max = env ? std::max(1, std::atoi(env)) : 16;
    bool gglob = false;
    if (sys.n2 >= 100) {
        for (int c = 2; c <= cs_max; c *= 2)
            if (admm_smem_doubles(sys.n, c) * sizeof(double) <= 220 * 1024) { cs = c; break; }
        if (cs == 1 && cs_max >= 8) {  // the inverse slice does not fit: read its rows from L2
            gglob = true;
            cs = 8;
        }
    }
    A.ginv_global = gglob ? 1 : 0;
    size_t sm = admm_smem_doubles(sys.n, cs, gglob) * sizeof(double);
    if (sm > 227 * 1024) param_error("kernel estimation: kernel side too large for the device ADMM (n <= 29)");
    const size_t sym_bytes = (11 * static_cast<size_t>(sys.n2) + 2) * sizeof(double);
    A.cache_symbols = sm + sym_bytes <= 225 * 1024 ? 1 : 0;
    if (A.cache_symbols) sm += sym_bytes;
    static const bool generic = std::getenv("FBMP_ADMM_GENERIC") != nullptr;  // A/B: runtime-n kernel
    auto kfn = generic ? k_admm<0>
                       : sys.n == 15 ? k_admm<15> : sys.n == 17 ? k_admm<17> : sys.n == 21 ? k_admm<21> : k_admm<0>;
    set_smem(kfn, sm);
    if (cs > 8) FBMP_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sys.S * cs);
    cfg.blockDim = dim3(NTADMM);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = ctx.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FBMP_CUDA(cudaLaunchKernelEx(&cfg, kfn, A, static_cast<const double*>(sys.Ginv),
                                 static_cast<const double*>(sys.Etf), d_state, d_info, d_k, cs));
    ctx.count();
    check_launch();
#ifdef FBMP_ADMM_PROF
    {
        long long pr[16];
        FBMP_CUDA(cudaMemcpyFromSymbolAsync(pr, g_admm_prof, sizeof(pr), 0, cudaMemcpyDeviceToHost, ctx.stream));
        FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
        std::fprintf(stderr, "admm prof n=%d cs=%d:", sys.n, cs);
        for (int k = 0; k < 7; ++k) std::fprintf(stderr, " %lld", pr[k]);
        std::fprintf(stderr, " | up_solve: rhs %lld fwd %lld solve %lld inv %lld", pr[8], pr[9], pr[10], pr[11]);
        std::fprintf(stderr, "\n");
    }
#endif
}

void admm_device(Context& ctx, const ObsSystem& sys, const fbmp_ke_params& prm, double* d_state, bool init_state,
                 int t_begin, int phase_begin, int hook_t, int* d_info) {
    admm_device(ctx, sys, prm, d_state, init_state, t_begin, phase_begin, hook_t, d_info, nullptr);
}

void solve_up_device(Context& ctx, const double* d_fields, int n, const fbmp_ke_params& prm, double coupling,
                     const double* d_anchor, double* d_u, double* d_p1, double* d_p2) {
    const int m = n * n;
    const size_t sm = (static_cast<size_t>(12 + 4 + 18) * m + 2 * n + NTADMM + 8) * sizeof(double);
    if (sm > 227 * 1024) param_error("solve_up: field size too large for the device solver");
    set_smem(k_solve_up, sm);
    k_solve_up<<<1, NTADMM, sm, ctx.stream>>>(n, prm.alpha1 * prm.mu1, prm.alpha2 * prm.mu2, coupling, d_fields,
                                             d_anchor, d_u, d_p1, d_p2);
    ctx.count();
    check_launch();
}

void shrink2_device(Context& ctx, double* d_cols, int ncols, long long m, double t) {
    k_shrink2<<<grid1d(ctx, m), 256, 0, ctx.stream>>>(d_cols, ncols, m, t);
    ctx.count();
    check_launch();
}

void project_simplex_device(Context& ctx, const double* d_v, int m, double* d_out, int* d_status) {
    const size_t sm = (2 * static_cast<size_t>(m) + 4 * NTADMM + NTADMM / 2 + 4) * sizeof(double);
    if (sm > 227 * 1024) param_error("project_simplex: vector too long for the device projection");
    set_smem(k_project, sm);
    k_project<<<1, NTADMM, sm, ctx.stream>>>(d_v, m, d_out, d_status);
    ctx.count();
    check_launch();
}

void estimate_kernel_device(Context& ctx, const double* d_pan, const double* d_obs, int S, int H, int W, int c,
                            const fbmp_ke_params& prm, double* d_k, std::vector<int>& iters, double* d_state_out,
                            int hook_t, bool tv, bool split) {
    validate_ke(prm);
    const int n = prm.n;
    if (c < 1) param_error("build_observation: factor must be >= 1");
    if (H % c || W % c) dim_error("build_observation: PAN dimensions must be factor times the observation");
    if (n > std::min(H, W)) dim_error("build_observation: kernel larger than PAN image");
    const long long P = static_cast<long long>(H) * W;
    double* stats = ctx.scratch<double>("ke_stats", static_cast<size_t>(S) * 4);
    pan_stats(ctx, d_pan, S, P, stats);
    std::vector<double> hs(static_cast<size_t>(S) * 4);
    d2h(hs.data(), stats, hs.size() * sizeof(double), ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    std::vector<double> scale(S);
    for (int s = 0; s < S; ++s) {  // kernel_estimator.cpp:269-289
        const double mean = hs[s * 4] / static_cast<double>(P);
        const double dev = std::max(hs[s * 4 + 2] - mean, mean - hs[s * 4 + 1]);
        if (dev <= 1e-12 * std::max(1.0, std::abs(mean)))
            num_error("kernel estimation: constant PAN image is unidentifiable (E^T E has rank 1)");
        const double m = hs[s * 4 + 3];
        if (m <= 0.0) num_error("kernel estimation: PAN image is identically zero");
        const double hw = static_cast<double>(H / c) * (W / c);
        scale[s] = std::sqrt(16384.0 / hw) / m;
    }
    double* d_scale = ctx.scratch<double>("ke_scale", S);
    h2d(d_scale, scale.data(), S * sizeof(double), ctx.stream);
    ObsSystem sys;
    build_observation(ctx, d_pan, d_obs, S, H, W, c, n, prm.mu3, d_scale, sys, true, 0.0, 0.0, split);
    const int m = n * n;
    double* state = d_state_out ? d_state_out : ctx.scratch<double>("ke_state", static_cast<size_t>(S) * 17 * m);
    int* info = ctx.scratch<int>("ke_info", static_cast<size_t>(S) * 4);
    admm_device(ctx, sys, prm, state, true, 0, 0, hook_t, info, d_k, tv);
    std::vector<int> hinfo(static_cast<size_t>(S) * 4), hst(S);
    d2h(hinfo.data(), info, hinfo.size() * sizeof(int), ctx.stream);
    d2h(hst.data(), sys.status, S * sizeof(int), ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    iters.assign(S, 0);
    for (int s = 0; s < S; ++s) {
        if (hst[s]) num_error("build_observation: factorization of E^T E + mu3 I failed");
        iters[s] = hinfo[s * 4];
        const int st = hinfo[s * 4 + 1];
        const std::string it = std::to_string(hinfo[s * 4]);
        if (st == 1) num_error("kernel estimation diverged: non-finite u at iteration " + it);
        if (st == 2) num_error("kernel estimation diverged: non-finite z at iteration " + it);
        if (st == 3) num_error("project_simplex: empty support (non-finite input?)");
    }
}

// l2 + simplex ADMM (kernel_estimator.cpp:411-427), one CTA per scene: u' = K^-1 (E^T f + mu3 (z - L)),
// z = project_simplex(u' + L), L += rho (u' - z), stop on ||u - u'|| / max(||u'||, 1e-300) < th.
// K^-1 (explicit, from build_observation) is read from L2; info = {iterations, status}.
__global__ void __launch_bounds__(NTADMM) k_admm_l2(int n, double mu3, double rho, double th, int t_max, int init_kind,
                                                    const double* __restrict__ Kinv_all, const double* __restrict__ Etf_all,
                                                    double* __restrict__ k_out, int* __restrict__ info_all) {
    extern __shared__ double smem[];
    const int s = blockIdx.x, m = n * n;
    const double* Kinv = Kinv_all + static_cast<size_t>(s) * m * m;
    const double* Etf = Etf_all + static_cast<size_t>(s) * m;
    double* u = smem;
    double* z = u + m;
    double* L = z + m;
    double* b = L + m;
    double* un = b + m;
    double* v = un + m;
    double* red = v + m;
    int* ired = reinterpret_cast<int*>(red + NTADMM);
    double* scratch = red + NTADMM + NTADMM / 2 + 4;
    const int cc = (n - 1) / 2;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double u0 = init_kind == 0 ? (i == cc * n + cc ? 1.0 : 0.0) : 1.0 / static_cast<double>(m);
        u[i] = u0;
        z[i] = u0;
        L[i] = 0.0;
    }
    __syncthreads();
    int status = 0, t = 0;
    for (; t < t_max; ++t) {
        for (int i = threadIdx.x; i < m; i += blockDim.x) b[i] = Etf[i] + mu3 * (z[i] - L[i]);
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int i = warp; i < m; i += NTADMM / 32) {  // K^-1 symmetric: row i
            double acc = 0.0;
            for (int j = lane; j < m; j += 32) acc = fma(__ldg(Kinv + static_cast<size_t>(i) * m + j), b[j], acc);
            acc = warp_sum(acc);
            if (lane == 0) un[i] = acc;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) v[i] = un[i] + L[i];
        __syncthreads();
        const int support = m <= NTADMM ? project_simplex_sorted(v, z, m, red, ired, scratch)
                                        : project_simplex_block(v, z, m, red, ired);
        if (support == 0) { status = 3; break; }
        double dd = 0.0, nn = 0.0;
        bool fin = true;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            L[i] += rho * (un[i] - z[i]);
            const double du = u[i] - un[i];
            dd += du * du;
            nn += un[i] * un[i];
            fin = fin && isfinite(un[i]) && isfinite(z[i]);
        }
        const double delta = sqrt(admm_sum(dd, red)) / fmax(sqrt(admm_sum(nn, red)), 1e-300);
        for (int i = threadIdx.x; i < m; i += blockDim.x) u[i] = un[i];
        if (!__syncthreads_and(fin)) { status = 1; break; }
        if (delta < th) { ++t; break; }
    }
    for (int i = threadIdx.x; i < m; i += blockDim.x) k_out[static_cast<size_t>(s) * m + i] = z[i];
    if (threadIdx.x == 0) {
        info_all[2 * s] = t;
        info_all[2 * s + 1] = status;
    }
}

void estimate_kernel_l2_device(Context& ctx, const double* d_pan, const double* d_obs, int H, int W, int c,
                               const fbmp_ke_params& prm, double* d_k, int* iters) {
    validate_ke(prm);
    const int n = prm.n;
    if (c < 1) param_error("build_observation: factor must be >= 1");
    if (H % c || W % c) dim_error("build_observation: PAN dimensions must be factor times the observation");
    if (n > std::min(H, W)) dim_error("build_observation: kernel larger than PAN image");
    const long long P = static_cast<long long>(H) * W;
    double* stats = ctx.scratch<double>("ke_stats", 4);
    pan_stats(ctx, d_pan, 1, P, stats);
    double hs[4];
    d2h(hs, stats, sizeof(hs), ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    const double mean = hs[0] / static_cast<double>(P);  // kernel_estimator.cpp:269-289
    const double dev = std::max(hs[2] - mean, mean - hs[1]);
    if (dev <= 1e-12 * std::max(1.0, std::abs(mean)))
        num_error("kernel estimation: constant PAN image is unidentifiable (E^T E has rank 1)");
    if (hs[3] <= 0.0) num_error("kernel estimation: PAN image is identically zero");
    const double scale = std::sqrt(16384.0 / (static_cast<double>(H / c) * (W / c))) / hs[3];
    double* d_scale = ctx.scratch<double>("ke_scale", 1);
    h2d(d_scale, &scale, sizeof(double), ctx.stream);
    ObsSystem sys;
    build_observation(ctx, d_pan, d_obs, 1, H, W, c, n, prm.mu3, d_scale, sys, true, prm.alpha1, prm.alpha2);
    const int m = n * n;
    int* info = ctx.scratch<int>("ke_info", 2);
    const size_t sm = (6 * static_cast<size_t>(m) + NTADMM + NTADMM / 2 + 4 + admm_scratch_doubles(m)) * sizeof(double);
    if (sm > 227 * 1024) param_error("l2 kernel estimation: kernel side too large for the device solve");
    set_smem(k_admm_l2, sm);
    k_admm_l2<<<1, NTADMM, sm, ctx.stream>>>(n, prm.mu3, prm.rho, prm.th, prm.t_max, prm.init, sys.Ginv, sys.Etf, d_k,
                                             info);
    ctx.count();
    check_launch();
    int hinfo[2], hst = 0;
    d2h(hinfo, info, sizeof(hinfo), ctx.stream);
    d2h(&hst, sys.status, sizeof(int), ctx.stream);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    if (hst) num_error("l2 kernel estimation: normal matrix factorization failed");
    if (hinfo[1] == 1) num_error("l2 kernel estimation diverged at iteration " + std::to_string(hinfo[0]));  // t of the failing iteration (:423)
    if (hinfo[1] == 3) num_error("project_simplex: empty support (non-finite input?)");
    if (iters) *iters = hinfo[0];
}

}  // namespace fbmp_gpu
