// cg_fast.cuh -- specialised CG operator kernels (window radius 1, c in {1,2,4}, images >= 64).
//
// K_Q2: q = D B p with the kernel side N_ and factor CF known at compile time. The HR tile
//       region is split into CF x CF sampling phases in shared memory; every tap becomes an
//       immediate-offset shared load shared by two vertically adjacent LR points (common
//       sub-expressions of the unrolled loop), taps are broadcast reads.
// K_A2: B^T U q + lambda L M L p for all channels of a scene in one CTA (the guide tile and
//       its per-window statistics are loaded once), the matting operator as separable 3x3
//       box sums:  (M s)_m = n_m s_m - box(c1)_m - I_m box(a)_m  with per-window
//       a_k = g_k (box(I s)_k / 9 - mu_k box(s)_k / 9),  c1_k = [k interior](box(s)_k/9 - mu_k a_k),
//       g_k = [k interior] / (eps/9 + var_k)  (pansharpen.cpp:128-164 regrouped), and the data
//       term gathered per sampling phase so that taps are uniform across a warp.
#pragma once
#include "pansharpen.cuh"

namespace fbmp_gpu {
namespace fast {

constexpr int NT = 256;

__host__ __device__ constexpr int pstride(int s) { return s + ((4 - s % 16) + 16) % 16; }

__device__ __forceinline__ int wrap_once(int a, int m) { return a < 0 ? a + m : (a >= m ? a - m : a); }

// ------------------------------------------------------------------------------------------
// per-scene guide statistics (pansharpen.cpp:128-139, :152-155):
//   mu_k = box_mean(I)_k, g_k = 1 / (eps/9 + var_k) on interior centres, 0 elsewhere
// ------------------------------------------------------------------------------------------
__global__ void k_guide_stats(const double* __restrict__ guide, int H, int W, int rw, double eps,
                              double* __restrict__ mu, double* __restrict__ gk) {
    const size_t P = static_cast<size_t>(H) * W;
    const double* I = guide + blockIdx.y * P;
    const double ws = static_cast<double>((2 * rw + 1) * (2 * rw + 1));
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(P);
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(e / W), c = static_cast<int>(e - static_cast<long long>(r) * W);
        double m = 0.0, g = 0.0;
        if (r >= rw && r < H - rw && c >= rw && c < W - rw) {
            double s1 = 0.0, s2 = 0.0;
            for (int dy = -rw; dy <= rw; ++dy)
                for (int dx = -rw; dx <= rw; ++dx) {
                    const double v = I[static_cast<size_t>(r + dy) * W + c + dx];
                    s1 += v;
                    s2 += v * v;
                }
            m = s1 / ws;
            const double var = s2 / ws - m * m;
            g = 1.0 / (eps / ws + var);
        }
        mu[blockIdx.y * P + e] = m;
        gk[blockIdx.y * P + e] = g;
    }
}

// ------------------------------------------------------------------------------------------
// K_Q2
// ------------------------------------------------------------------------------------------
template <int N_, int CF>
struct QGeo {
    static constexpr int C = (N_ - 1) / 2;
    static constexpr int g = (C + CF - 1) / CF;
    static constexpr int TW = 32, TH = 16;
    static constexpr int PW = TW + 2 * g, PH = TH + 2 * g;
    static constexpr int PS = pstride(PW * PH);
    static constexpr int SRW = CF * PW, SRH = CF * PH;
    static constexpr int KOFF = ((N_ * N_ + 1) / 2) * 2;
    static constexpr size_t smem = (KOFF + static_cast<size_t>(CF) * CF * PS) * sizeof(double);
};

template <int N_, int CF, bool CG>
__global__ void __launch_bounds__(NT, 2) k_q2(PsGeo G, const double* __restrict__ taps, const double* __restrict__ src,
                                              double* __restrict__ pbuf, double* __restrict__ q, CgState* st,
                                              double* __restrict__ part, int nblk) {
    using Q = QGeo<N_, CF>;
    __shared__ double red[NT / 32 + 1];
    extern __shared__ double sm[];
    const int ch = blockIdx.y;
    int t = 0;
    double beta = 0.0;
    if (CG) {
        if (st[ch].done) return;
        t = st[ch].t;
        beta = t ? st[ch].beta : 0.0;
    }
    const int H = G.H, W = G.W;
    const size_t P = static_cast<size_t>(H) * W;
    const double* rc = src + ch * P;
    const double* pold = CG ? pbuf + (static_cast<size_t>((t + 1) & 1) * G.N + ch) * P : nullptr;
    double* pnew = CG ? pbuf + (static_cast<size_t>(t & 1) * G.N + ch) * P : nullptr;
    const int ntx = (G.w + Q::TW - 1) / Q::TW;
    const int tyb = blockIdx.x / ntx, txb = blockIdx.x - tyb * ntx;
    const int i0 = tyb * Q::TH, j0 = txb * Q::TW;
    double* sk = sm;
    double* planes = sm + Q::KOFF;
    const double* tp = taps + static_cast<size_t>(ch / G.cps) * N_ * N_;
    for (int e = threadIdx.x; e < N_ * N_; e += NT) sk[e] = tp[e];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int R0 = CF * (i0 - Q::g), C0 = CF * (j0 - Q::g);
    constexpr int own_r0 = CF * Q::g, own_r1 = CF * (Q::g + Q::TH), own_c1 = CF * (Q::g + Q::TW);
    double pp = 0.0;
    // region load: each thread keeps KB elements (r and p_old) in flight before storing
    constexpr int TOT = Q::SRH * Q::SRW;
    constexpr int KB = 8;
    for (int e0 = 0; e0 < TOT; e0 += NT * KB) {
        double vr[KB], vp[KB];
        size_t gi[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int e = e0 + k * NT + threadIdx.x;
            const int rr = e / Q::SRW, cc = e - rr * Q::SRW;
            gi[k] = static_cast<size_t>(wrap_once(R0 + rr, H)) * W + wrap_once(C0 + cc, W);
            if (e < TOT) {
                vr[k] = __ldg(rc + gi[k]);
                if (CG) vp[k] = __ldg(pold + gi[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int e = e0 + k * NT + threadIdx.x;
            if (e >= TOT) break;
            const int rr = e / Q::SRW, cc = e - rr * Q::SRW;
            double v = vr[k];
            if (CG) {
                v = v + vp[k] * beta;  // pansharpen.cpp:254
                if (rr >= own_r0 && rr < own_r1 && cc >= own_r0 && cc < own_c1 && R0 + rr < H && C0 + cc < W) {
                    pnew[gi[k]] = v;
                    pp += v * v;
                }
            }
            planes[((rr % CF) * CF + (cc % CF)) * Q::PS + (rr / CF) * Q::PW + cc / CF] = v;
        }
    }
    __syncthreads();
    // two vertically adjacent LR points per thread: (i0 + 2 warp + {0,1}, j0 + lane)
    const int ti = 2 * warp, tj = lane;
    const double* base = planes + ti * Q::PW + tj;
    double acc0 = 0.0, acc1 = 0.0;
    // Plane row (phase pr, row offset Ir) feeds tap row a0 = CF g - pr - CF Ir of point 0 and
    // a0 + CF of point 1: each row segment is loaded once and used by both points.
    for (int pr = 0; pr < CF; ++pr) {
        const int ir_lo = (CF * Q::g - pr - Q::C + CF - 1) / CF - 1;  // smallest Ir with a0 + CF <= C
        const int ir_hi = (CF * Q::g - pr + Q::C) / CF + 1;           // largest Ir with a0 + CF >= -C
        for (int ir = max(ir_lo, 0); ir <= ir_hi; ++ir) {
            const int a0 = CF * Q::g - pr - CF * ir;
            const bool v0 = a0 >= -Q::C && a0 <= Q::C;
            const bool v1 = a0 + CF >= -Q::C && a0 + CF <= Q::C;
            const double* row = base + pr * CF * Q::PS + ir * Q::PW;
            const double* k0 = sk + (a0 + Q::C) * N_ + Q::C;
            const double* k1 = k0 + CF * N_;
            if (v0 && v1) {
#pragma unroll
                for (int b = -Q::C; b <= Q::C; ++b) {
                    const int cb = CF * Q::g - b;
                    const double v = row[(cb % CF) * Q::PS + cb / CF];
                    acc0 = fma(k0[b], v, acc0);
                    acc1 = fma(k1[b], v, acc1);
                }
            } else if (v0) {
#pragma unroll
                for (int b = -Q::C; b <= Q::C; ++b) {
                    const int cb = CF * Q::g - b;
                    acc0 = fma(k0[b], row[(cb % CF) * Q::PS + cb / CF], acc0);
                }
            } else if (v1) {
#pragma unroll
                for (int b = -Q::C; b <= Q::C; ++b) {
                    const int cb = CF * Q::g - b;
                    acc1 = fma(k1[b], row[(cb % CF) * Q::PS + cb / CF], acc1);
                }
            }
        }
    }
    const int i = i0 + ti, j = j0 + tj;
    double* qc = q + static_cast<size_t>(ch) * G.h * G.w;
    if (j < G.w) {
        if (i < G.h) qc[static_cast<size_t>(i) * G.w + j] = acc0;
        if (i + 1 < G.h) qc[static_cast<size_t>(i + 1) * G.w + j] = acc1;
    }
    if (CG) {
        const double bs = block_sum<NT>(pp, red);
        if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
        if (elect_last_block(&st[ch].cnt_q, nblk)) {
            const double tot = sum_partials<NT>(part + static_cast<size_t>(ch) * nblk, nblk, 1, red);
            if (threadIdx.x == 0) {
                st[ch].pp = tot;
                st[ch].cnt_q = 0;
            }
        }
    }
}

template <int N_, int CF>
inline int q2_blocks(const PsGeo& G) {
    using Q = QGeo<N_, CF>;
    return ((G.w + Q::TW - 1) / Q::TW) * ((G.h + Q::TH - 1) / Q::TH);
}

// ------------------------------------------------------------------------------------------
// K_A2 (radius 1)
// ------------------------------------------------------------------------------------------
namespace a2 {
constexpr int TA = 32;
constexpr int WP = TA + 8;   // p on R+4
constexpr int WI = TA + 6;   // I, s, I*s on R+3
constexpr int WK = TA + 4;   // window stats on R+2
constexpr int WM = TA + 2;   // M s on R+1
constexpr int H1R = WI, H1C = WK;  // first horizontal sums: rows R+3, cols R+2
constexpr int H2R = WK, H2C = WM;  // second: rows R+2, cols R+1
constexpr int MAXN = 21;            // kernel side limit of the fast path
constexpr int O_TAPS = 0;
constexpr int MAXTAP = 442;         // n <= 21
constexpr int O_Q = O_TAPS + MAXTAP;
__host__ __device__ constexpr int maxq(int cf) {  // LR window of the data term
    return ((TA - 1 + (MAXN - 1)) / cf + 2) * ((TA - 1 + (MAXN - 1)) / cf + 2);
}
template <int CF>
struct L {
    static constexpr int O_I = O_Q + ((maxq(CF) + 1) / 2) * 2;
    static constexpr int O_S = O_I + WI * WI;
    static constexpr int O_U = O_S + WI * WI;          // union: [p | Is] -> [a | c1] -> [M]
    static constexpr int U_SIZE = WP * WP + WI * WI;   // 1600 + 1444 >= 2 * WK * WK
    static constexpr int O_H = O_U + U_SIZE;           // horizontal-sum planes / data-term output
    static constexpr int H_SIZE = 2 * H1R * H1C;
    static constexpr int O_MU = O_H + H_SIZE;          // per-window guide statistics (once per tile)
    static constexpr int O_G = O_MU + WK * WK;
    static constexpr int TOTAL = O_G + WK * WK;
    static_assert(U_SIZE >= 2 * WK * WK, "union too small");
    static_assert(H_SIZE >= TA * TA, "output staging too small");
    static constexpr size_t smem = TOTAL * sizeof(double);
};
}  // namespace a2

template <bool CG, int CF>
__global__ void __launch_bounds__(NT, 2) k_apply2(PsGeo G, const double* __restrict__ taps,
                                                  const double* __restrict__ guide, const double* __restrict__ wmu,
                                                  const double* __restrict__ wg, const double* __restrict__ pin,
                                                  const double* __restrict__ q, double* __restrict__ out, CgState* st,
                                                  double* __restrict__ part, int nblk) {
    using namespace a2;
    __shared__ double red[NT / 32 + 1];
    extern __shared__ double sm[];
    const int scene = blockIdx.y;
    const int H = G.H, W = G.W, n = G.n, C = G.C;
    const size_t P = static_cast<size_t>(H) * W;
    const int ntx = (W + TA - 1) / TA;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const int r0 = by * TA, c0 = bx * TA;
    const double* I = guide + scene * P;
    const double* MU = wmu + scene * P;
    const double* GK = wg + scene * P;
    using Lay = L<CF>;
    double* sk = sm + O_TAPS;
    double* sq = sm + O_Q;
    double* sI = sm + Lay::O_I;
    double* sS = sm + Lay::O_S;
    double* sU = sm + Lay::O_U;
    double* sH = sm + Lay::O_H;
    double* sMu = sm + Lay::O_MU;
    double* sG = sm + Lay::O_G;
    const double* tp = taps + static_cast<size_t>(scene) * n * n;
    for (int e = threadIdx.x; e < n * n; e += NT) sk[e] = tp[e];
    for (int e = threadIdx.x; e < WI * WI; e += NT) {
        const int y = e / WI, x = e - y * WI;
        sI[e] = __ldg(I + static_cast<size_t>(wrap_once(r0 - 3 + y, H)) * W + wrap_once(c0 - 3 + x, W));
    }
    for (int e = threadIdx.x; e < WK * WK; e += NT) {
        const int y = e / WK, x = e - y * WK;
        const size_t gi = static_cast<size_t>(wrap_once(r0 - 2 + y, H)) * W + wrap_once(c0 - 2 + x, W);
        sMu[e] = __ldg(MU + gi);
        sG[e] = __ldg(GK + gi);
    }
    // data-term LR window
    const int iq0 = floordiv(r0 - C + CF - 1, CF), jq0 = floordiv(c0 - C + CF - 1, CF);
    const int QH = floordiv(r0 + TA - 1 + C, CF) - iq0 + 1, QW = floordiv(c0 + TA - 1 + C, CF) - jq0 + 1;
    // phase-uniform data-term mapping: item -> (cell column J, 4-cell row block, phase)
    constexpr int CW = TA / CF;            // cells per tile side
    constexpr int RB = CW / 4;             // 4-cell row blocks
    const int it_J = threadIdx.x % CW;
    const int it_rest = threadIdx.x / CW;
    const int it_B = it_rest % RB;
    const int it_ph = it_rest / RB;        // 0 .. CF*CF-1
    const int pr = it_ph / CF, pc = it_ph - pr * CF;
    const int dilo = floordiv(pr - C + CF - 1, CF), dihi = floordiv(pr + C, CF);
    const int djlo = floordiv(pc - C + CF - 1, CF), djhi = floordiv(pc + C, CF);

    for (int chl = 0; chl < G.cps; ++chl) {
        const int ch = scene * G.cps + chl;
        if (CG && st[ch].done) continue;
        const double* p = pin + ch * P;
        if (CG) p = pin + (static_cast<size_t>(st[ch].t & 1) * G.N + ch) * P;
        const double* qc = q + static_cast<size_t>(ch) * G.h * G.w;
        __syncthreads();  // previous channel's readers of the shared buffers are done
        double* sP = sU;
        {
            constexpr int KP = (WP * WP + NT - 1) / NT;
            double v[KP];
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int e = threadIdx.x + k * NT;
                const int y = e / WP, x = e - y * WP;
                if (e < WP * WP)
                    v[k] = __ldg(p + static_cast<size_t>(wrap_once(r0 - 4 + y, H)) * W + wrap_once(c0 - 4 + x, W));
            }
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int e = threadIdx.x + k * NT;
                if (e < WP * WP) sP[e] = v[k];
            }
        }
        for (int e = threadIdx.x; e < QH * QW; e += NT) {
            const int a = e / QW, b = e - a * QW;
            sq[e] = __ldg(qc + static_cast<size_t>(wrapi(iq0 + a, G.h)) * G.w + wrapi(jq0 + b, G.w));
        }
        __syncthreads();
        // own pixels' p (for p.Ap): pixel e = tid + 256 k
        double pown[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int e = threadIdx.x + NT * k;
            pown[k] = sP[(e / TA + 4) * WP + (e % TA) + 4];
        }
        // stage 1: s = L p and I*s on R+3 (ops.cpp:70-78 stencil order)
        double* sIS = sU + WP * WP;
        for (int e = threadIdx.x; e < WI * WI; e += NT) {
            const int y = e / WI + 1, x = e % WI + 1;
            const double v = 4.0 * sP[y * WP + x] - sP[(y - 1) * WP + x] - sP[(y + 1) * WP + x] - sP[y * WP + x - 1] -
                             sP[y * WP + x + 1];
            sS[e] = v;
            sIS[e] = sI[e] * v;
        }
        __syncthreads();
        // stage 2: horizontal 3-sums of s and I*s (rows R+3, cols R+2)
        double* h1 = sH;
        double* h2 = sH + H1R * H1C;
        for (int e = threadIdx.x; e < H1R * H1C; e += NT) {
            const int y = e / H1C, x = e % H1C;
            const int b = y * WI + x;
            h1[e] = sS[b] + sS[b + 1] + sS[b + 2];
            h2[e] = sIS[b] + sIS[b + 1] + sIS[b + 2];
        }
        __syncthreads();
        // stage 3: vertical sums -> per-window a_k, c1_k on R+2
        double* sA = sU;
        double* sC = sU + WK * WK;
        for (int e = threadIdx.x; e < WK * WK; e += NT) {
            const int y = e / WK, x = e % WK;
            const int b = y * H1C + x;
            const double ss = h1[b] + h1[b + H1C] + h1[b + 2 * H1C];
            const double sis = h2[b] + h2[b + H1C] + h2[b + 2 * H1C];
            const double mu = sMu[e], g = sG[e];
            const double xb = ss / 9.0;
            const double a = g * (sis / 9.0 - mu * xb);
            sA[e] = a;
            sC[e] = g != 0.0 ? xb - mu * a : 0.0;
        }
        __syncthreads();
        // stage 4: horizontal 3-sums of a and c1 (rows R+2, cols R+1)
        h1 = sH;
        h2 = sH + H2R * H2C;
        for (int e = threadIdx.x; e < H2R * H2C; e += NT) {
            const int y = e / H2C, x = e % H2C;
            const int b = y * WK + x;
            h1[e] = sA[b] + sA[b + 1] + sA[b + 2];
            h2[e] = sC[b] + sC[b + 1] + sC[b + 2];
        }
        __syncthreads();
        // stage 5: M s on R+1 = n_m s_m - box(c1) - I_m box(a)
        double* sM = sU;
        for (int e = threadIdx.x; e < WM * WM; e += NT) {
            const int y = e / WM, x = e % WM;
            const int b = y * H2C + x;
            const double ba = h1[b] + h1[b + H2C] + h1[b + 2 * H2C];
            const double bc = h2[b] + h2[b + H2C] + h2[b + 2 * H2C];
            const int gr = wrap_once(r0 - 1 + y, H), gc = wrap_once(c0 - 1 + x, W);
            const int nr = min(gr + 1, H - 2) - max(gr - 1, 1) + 1;  // interior window rows covering gr
            const int nc = min(gc + 1, W - 2) - max(gc - 1, 1) + 1;
            const double nm = static_cast<double>(max(nr, 0) * max(nc, 0));
            const int si = (y + 2) * WI + x + 2;
            sM[e] = nm * sS[si] - bc - sI[si] * ba;
        }
        __syncthreads();
        // stage 6a: data term per sampling phase (4 cells per thread along rows) -> sO
        double* sO = sH;
        {
            const int Jc = it_J;
            const int Ic0 = it_B * 4;
            // global LR index of the cell (c0/CF + Jc), row cells (r0/CF + Ic0 + k)
            const int qj0 = c0 / CF + Jc - jq0;
            const int qi0 = r0 / CF + Ic0 - iq0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int di = dilo; di <= dihi; ++di) {
                const double* krow = sk + (CF * di - pr + C) * n + C - pc;
                for (int dj = djlo; dj <= djhi; ++dj) {
                    const double kv = krow[CF * dj];
                    const double* qq = sq + (qi0 + di) * QW + qj0 + dj;
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[k] = fma(kv, qq[k * QW], acc[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sO[((Ic0 + k) * CF + pr) * TA + Jc * CF + pc] = acc[k];
        }
        __syncthreads();
        // stage 6b: t = L(M s), Ap = data + lambda t, p.Ap
        double* oc = out + ch * P;
        double dotp = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int e = threadIdx.x + NT * k;
            const int y = e / TA, x = e % TA;
            const int R = r0 + y, Cc = c0 + x;
            const int m = (y + 1) * WM + x + 1;
            const double tl = 4.0 * sM[m] - sM[m - WM] - sM[m + WM] - sM[m - 1] - sM[m + 1];
            const double val = sO[e] + tl * G.lambda;
            if (R < H && Cc < W) {
                oc[static_cast<size_t>(R) * W + Cc] = val;
                dotp += pown[k] * val;
            }
        }
        if (CG) {
            const double bs = block_sum<NT>(dotp, red);
            if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
            if (elect_last_block(&st[ch].cnt_a, nblk)) {
                const double pAp = sum_partials<NT>(part + static_cast<size_t>(ch) * nblk, nblk, 1, red);
                if (threadIdx.x == 0) {
                    CgState& S = st[ch];
                    S.pAp = pAp;
                    if (!(pAp > 0)) {  // pansharpen.cpp:240-244
                        S.done = (sqrt(S.rs) <= 1e-12 * S.rhs_norm) ? 1 : 2;
                        S.iters = S.t + 1;
                    } else {
                        S.alpha = S.rs / pAp;
                    }
                    S.cnt_a = 0;
                }
            }
        }
    }
}

}  // namespace fast
}  // namespace fbmp_gpu
