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
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

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


// ------------------------------------------------------------------------------------------
// K_A3: K_A2 restructured for shared-memory traffic. Every stage works on a 2 x 4 register
// micro-tile (horizontal and vertical 3-sums fused), I*s is formed on the fly, and the data
// term keeps the thread's zero-padded sampling-phase sub-kernel in registers (N_, CF known
// at compile time; N_ = 0 keeps the generic broadcast-tap loop).
// ------------------------------------------------------------------------------------------
namespace a3 {
constexpr int TA = 32;
constexpr int WP = TA + 8, WI = TA + 6, WK = TA + 4, WM = TA + 2;
template <int CF>
struct L {
    static constexpr int QMAX = a2::maxq(CF);
    static constexpr int O_TAPS = 0;                       // generic path only
    static constexpr int O_I = O_TAPS + a2::MAXTAP;        // guide on R+3
    static constexpr int O_MU = O_I + WI * WI;             // mu_k on R+2
    static constexpr int O_G = O_MU + WK * WK;             // g_k on R+2
    static constexpr int O_S = O_G + WK * WK;              // s on R+3
    static constexpr int O_M = O_S + WI * WI;              // M s on R+1
    static constexpr int O_Q = O_M + WM * WM;              // q window
    static constexpr int O_U = O_Q + ((QMAX + 1) / 2) * 2; // p on R+4 -> (a, c1) on R+2 -> data out
    static constexpr int U_SIZE = 2 * WK * WK;
    static constexpr int TOTAL = O_U + U_SIZE;
    static_assert(U_SIZE >= WP * WP && U_SIZE >= TA * TA, "union too small");
    static constexpr size_t smem = TOTAL * sizeof(double);
};
template <int N_, int CF>
struct DT {  // zero-padded sub-kernel extent of the data term
    static constexpr int C = (N_ - 1) / 2;
    static constexpr int DLO = -(C / CF);
    static constexpr int DHI = (CF - 1 + C) / CF;
    static constexpr int DM = DHI - DLO + 1;
};
}  // namespace a3

template <bool CG, int N_, int CF>
__global__ void __launch_bounds__(NT, 2) k_apply3(PsGeo G, const double* __restrict__ taps,
                                                  const double* __restrict__ guide, const double* __restrict__ wmu,
                                                  const double* __restrict__ wg, const double* __restrict__ pin,
                                                  const double* __restrict__ q, double* __restrict__ out, CgState* st,
                                                  double* __restrict__ part, int nblk) {
    using namespace a3;
    using Lay = L<CF>;
    __shared__ double red[NT / 32 + 1];
    extern __shared__ double sm[];
    const int scene = blockIdx.y;
    const int H = G.H, W = G.W, n = G.n, C = G.C;
    const size_t P = static_cast<size_t>(H) * W;
    const int ntx = (W + TA - 1) / TA;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const int r0 = by * TA, c0 = bx * TA;
    double* sk = sm + Lay::O_TAPS;
    double* sI = sm + Lay::O_I;
    double* sMu = sm + Lay::O_MU;
    double* sG = sm + Lay::O_G;
    double* sS = sm + Lay::O_S;
    double* sM = sm + Lay::O_M;
    double* sq = sm + Lay::O_Q;
    double* sU = sm + Lay::O_U;
    const double* tp = taps + static_cast<size_t>(scene) * n * n;
    {
        const double* I = guide + scene * P;
        const double* MU = wmu + scene * P;
        const double* GK = wg + scene * P;
        if (N_ == 0)
            for (int e = threadIdx.x; e < n * n; e += NT) sk[e] = tp[e];
        constexpr int KI = (WI * WI + NT - 1) / NT, KK = (WK * WK + NT - 1) / NT;
        double vi[KI], vm[KK], vg[KK];
#pragma unroll
        for (int k = 0; k < KI; ++k) {
            const int e = threadIdx.x + k * NT;
            const int y = e / WI, x = e - y * WI;
            if (e < WI * WI) vi[k] = __ldg(I + static_cast<size_t>(wrap_once(r0 - 3 + y, H)) * W + wrap_once(c0 - 3 + x, W));
        }
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            const int e = threadIdx.x + k * NT;
            const int y = e / WK, x = e - y * WK;
            const size_t gi = static_cast<size_t>(wrap_once(r0 - 2 + y, H)) * W + wrap_once(c0 - 2 + x, W);
            if (e < WK * WK) {
                vm[k] = __ldg(MU + gi);
                vg[k] = __ldg(GK + gi);
            }
        }
#pragma unroll
        for (int k = 0; k < KI; ++k)
            if (threadIdx.x + k * NT < WI * WI) sI[threadIdx.x + k * NT] = vi[k];
#pragma unroll
        for (int k = 0; k < KK; ++k)
            if (threadIdx.x + k * NT < WK * WK) {
                sMu[threadIdx.x + k * NT] = vm[k];
                sG[threadIdx.x + k * NT] = vg[k];
            }
    }
    // data-term work item: (cell column, 4-cell row block, sampling phase)
    constexpr int CW = TA / CF, RB = CW / 4;
    const int it_J = threadIdx.x % CW;
    const int it_rest = threadIdx.x / CW;
    const int it_B = it_rest % RB;
    const int it_ph = it_rest / RB;
    const int pr = it_ph / CF, pc = it_ph - pr * CF;
    using D = a3::DT<(N_ > 0 ? N_ : 1), CF>;
    constexpr int DM = N_ > 0 ? D::DM : 1;
    double kreg[DM][DM];
    if (N_ > 0) {
#pragma unroll
        for (int a = 0; a < DM; ++a)
#pragma unroll
            for (int b = 0; b < DM; ++b) {
                const int tr = CF * (a + D::DLO) - pr + D::C, tc = CF * (b + D::DLO) - pc + D::C;
                kreg[a][b] = (tr >= 0 && tr < N_ && tc >= 0 && tc < N_) ? __ldg(tp + tr * N_ + tc) : 0.0;
            }
    }
    const int iq0 = floordiv(r0 - C + CF - 1, CF), jq0 = floordiv(c0 - C + CF - 1, CF);
    const int QH = floordiv(r0 + TA - 1 + C, CF) - iq0 + 1, QW = floordiv(c0 + TA - 1 + C, CF) - jq0 + 1;
    const int dilo = floordiv(pr - C + CF - 1, CF), dihi = floordiv(pr + C, CF);
    const int djlo = floordiv(pc - C + CF - 1, CF), djhi = floordiv(pc + C, CF);
    // micro-tile coordinates (2 rows x 4 cols per thread)
    const int mt_y = 2 * (threadIdx.x / 10), mt_x = 4 * (threadIdx.x % 10);

    for (int chl = 0; chl < G.cps; ++chl) {
        const int ch = scene * G.cps + chl;
        if (CG && st[ch].done) continue;
        const double* p = pin + ch * P;
        if (CG) p = pin + (static_cast<size_t>(st[ch].t & 1) * G.N + ch) * P;
        const double* qc = q + static_cast<size_t>(ch) * G.h * G.w;
        __syncthreads();  // previous channel finished with the shared buffers
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
            for (int k = 0; k < KP; ++k)
                if (threadIdx.x + k * NT < WP * WP) sP[threadIdx.x + k * NT] = v[k];
        }
        for (int e = threadIdx.x; e < QH * QW; e += NT) {
            const int a = e / QW, b = e - a * QW;
            sq[e] = __ldg(qc + static_cast<size_t>(wrapi(iq0 + a, G.h)) * G.w + wrapi(jq0 + b, G.w));
        }
        __syncthreads();
        // own pixels' p for p.Ap, in the S5 mapping (row tid/8, columns 4 (tid%8) + j)
        double pown[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) pown[j] = sP[(threadIdx.x / 8 + 4) * WP + 4 * (threadIdx.x % 8) + j + 4];
        // S1: s = L p on R+3 (micro-tile 2 x 4; 19 x 10 tiles)
        if (threadIdx.x < 190) {
            double pv[4][6];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 6; ++j) pv[i][j] = sP[(mt_y + i) * WP + mt_x + j];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int y = mt_y + i, x = mt_x + j;
                    if (y < WI && x < WI)  // ops.cpp:70-78 stencil order
                        sS[y * WI + x] = 4.0 * pv[i + 1][j + 1] - pv[i][j + 1] - pv[i + 2][j + 1] - pv[i + 1][j] -
                                         pv[i + 1][j + 2];
                }
        }
        __syncthreads();
        // S2: per-window a_k, c1_k on R+2 (micro-tile 2 x 4; 18 x 9 tiles)
        double* sA = sU;
        double* sC = sU + WK * WK;
        if (threadIdx.x < 162) {
            const int wy = 2 * (threadIdx.x / 9), wx = 4 * (threadIdx.x % 9);
            double hs[4][4], hi[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double sv[6], iv[6];
#pragma unroll
                for (int j = 0; j < 6; ++j) {
                    const int o = (wy + i) * WI + wx + j;
                    sv[j] = (wy + i < WI && wx + j < WI) ? sS[o] : 0.0;
                    iv[j] = (wy + i < WI && wx + j < WI) ? sI[o] * sv[j] : 0.0;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    hs[i][j] = sv[j] + sv[j + 1] + sv[j + 2];
                    hi[i][j] = iv[j] + iv[j + 1] + iv[j + 2];
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int y = wy + i, x = wx + j;
                    if (y < WK && x < WK) {
                        const double ss = hs[i][j] + hs[i + 1][j] + hs[i + 2][j];
                        const double sis = hi[i][j] + hi[i + 1][j] + hi[i + 2][j];
                        const double mu = sMu[y * WK + x], g = sG[y * WK + x];
                        const double xb = ss / 9.0;
                        const double a = g * (sis / 9.0 - mu * xb);
                        sA[y * WK + x] = a;
                        sC[y * WK + x] = g != 0.0 ? xb - mu * a : 0.0;
                    }
                }
        }
        __syncthreads();
        // S3: M s on R+1 = n_m s_m - box(c1) - I_m box(a) (micro-tile 2 x 4; 17 x 9 tiles)
        if (threadIdx.x < 153) {
            const int my = 2 * (threadIdx.x / 9), mx = 4 * (threadIdx.x % 9);
            double ha[4][4], hc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double av[6], cv[6];
#pragma unroll
                for (int j = 0; j < 6; ++j) {
                    const int o = (my + i) * WK + mx + j;
                    const bool ok = my + i < WK && mx + j < WK;
                    av[j] = ok ? sA[o] : 0.0;
                    cv[j] = ok ? sC[o] : 0.0;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    ha[i][j] = av[j] + av[j + 1] + av[j + 2];
                    hc[i][j] = cv[j] + cv[j + 1] + cv[j + 2];
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int y = my + i;
                const int gr = wrap_once(r0 - 1 + y, H);
                const int nr = max(min(gr + 1, H - 2) - max(gr - 1, 1) + 1, 0);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int x = mx + j;
                    if (y < WM && x < WM) {
                        const double ba = ha[i][j] + ha[i + 1][j] + ha[i + 2][j];
                        const double bc = hc[i][j] + hc[i + 1][j] + hc[i + 2][j];
                        const int gc = wrap_once(c0 - 1 + x, W);
                        const int nc = max(min(gc + 1, W - 2) - max(gc - 1, 1) + 1, 0);
                        const int si = (y + 2) * WI + x + 2;
                        sM[y * WM + x] = static_cast<double>(nr * nc) * sS[si] - bc - sI[si] * ba;
                    }
                }
            }
        }
        __syncthreads();
        // S4: data term per sampling phase -> sO (4 cells along rows per thread)
        double* sO = sU;
        {
            const int Jc = it_J, Ic0 = it_B * 4;
            const int qj0 = c0 / CF + Jc - jq0, qi0 = r0 / CF + Ic0 - iq0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (N_ > 0) {
#pragma unroll
                for (int m = 0; m < DM + 3; ++m) {
                    double qv[DM];
                    const double* qrow = sq + (qi0 + D::DLO + m) * QW + qj0 + D::DLO;
#pragma unroll
                    for (int b = 0; b < DM; ++b) qv[b] = qrow[b];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int a = m - k;
                        if (a >= 0 && a < DM) {
#pragma unroll
                            for (int b = 0; b < DM; ++b) acc[k] = fma(kreg[a][b], qv[b], acc[k]);
                        }
                    }
                }
            } else {
                for (int di = dilo; di <= dihi; ++di) {
                    const double* krow = sk + (CF * di - pr + C) * n + C - pc;
                    for (int dj = djlo; dj <= djhi; ++dj) {
                        const double kv = krow[CF * dj];
                        const double* qq = sq + (qi0 + di) * QW + qj0 + dj;
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[k] = fma(kv, qq[k * QW], acc[k]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sO[((Ic0 + k) * CF + pr) * TA + Jc * CF + pc] = acc[k];
        }
        __syncthreads();
        // S5: t = L(M s), Ap = data + lambda t, p.Ap (1 x 4 per thread)
        double* oc = out + ch * P;
        double dotp = 0.0;
        {
            const int y = threadIdx.x / 8, x0 = 4 * (threadIdx.x % 8);
            double mv[3][6];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 6; ++j) mv[i][j] = sM[(y + i) * WM + x0 + j];
            const int R = r0 + y;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double tl = 4.0 * mv[1][j + 1] - mv[0][j + 1] - mv[2][j + 1] - mv[1][j] - mv[1][j + 2];
                const double val = sO[y * TA + x0 + j] + tl * G.lambda;
                const int Cc = c0 + x0 + j;
                if (R < H && Cc < W) {
                    oc[static_cast<size_t>(R) * W + Cc] = val;
                    dotp += pown[j] * val;
                }
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


// ------------------------------------------------------------------------------------------
// K_A4: K_A3 with conflict-free column strips. Every stage maps lanes to consecutive columns
// and walks a strip of rows with the vertical 3-sums in a register sliding window, so each
// shared load is a stride-1 (conflict-free) warp access and reused vertically.
// ------------------------------------------------------------------------------------------
namespace a4 {
constexpr int TA = 32;
constexpr int WP = TA + 8, WI = TA + 6, WK = TA + 4, WM = TA + 2;
// stage strips over column PAIRS: S1 19 x 13 strips x 3 rows, S2 18 x 14 x 3, S3 17 x 15 x 3,
// S5 16 x 16 x 2
static_assert(19 * 13 <= NT && 18 * 14 <= NT && 17 * 15 <= NT && 16 * 16 == NT && TA == 32, "strips");
template <int CF>
struct L {
    static constexpr int QMAX = a2::maxq(CF);
    static constexpr int O_TAPS = 0;
    static constexpr int O_I = O_TAPS + a2::MAXTAP;        // guide on R+3
    static constexpr int O_MU = O_I + WI * WI;             // mu_k on R+2
    static constexpr int O_G = O_MU + WK * WK;             // g_k on R+2
    static constexpr int O_S = O_G + WK * WK;              // s on R+3
    static constexpr int O_M = O_S + WI * WI;              // I*s on R+3, then M s on R+1
    static constexpr int O_Q = O_M + WI * WI;              // q window
    static constexpr int QWMAX = (TA - 1 + 2 * (a2::MAXN / 2)) / CF + 2;
    static constexpr int QWP = QWMAX + ((8 - QWMAX % 16) + 16) % 16;   // row stride == 8 (mod 16)
    static constexpr int O_U = O_Q + QWP * QWMAX;          // p on R+4 -> (a, c1) on R+2
    static constexpr int U_SIZE = 2 * WK * WK;
    static constexpr int O_O = O_U + U_SIZE;               // data term out (TA x TA)
    static constexpr int TOTAL = O_O + TA * TA;
    static_assert(U_SIZE >= WP * WP, "union too small");
    static_assert(O_I % 2 == 0 && O_MU % 2 == 0 && O_G % 2 == 0 && O_S % 2 == 0 && O_M % 2 == 0 &&
                  O_Q % 2 == 0 && O_U % 2 == 0 && O_O % 2 == 0 && WK * WK % 2 == 0, "16-byte pair alignment");
    static constexpr size_t smem = TOTAL * sizeof(double);
};
}  // namespace a4

template <bool CG, int N_, int CF>
__global__ void __launch_bounds__(NT, 2) k_apply4(PsGeo G, const double* __restrict__ taps,
                                                  const double* __restrict__ guide, const double* __restrict__ wmu,
                                                  const double* __restrict__ wg, const double* __restrict__ pin,
                                                  const double* __restrict__ q, double* __restrict__ out, CgState* st,
                                                  double* __restrict__ part, int nblk) {
    using namespace a4;
    using Lay = a4::L<CF>;
    __shared__ double red[NT / 32 + 1];
    extern __shared__ double sm[];
    // blockIdx.y = scene * cgroups + group: the CTA handles channels [group*cpc, group*cpc+cpc)
    const int cgroups = (G.cps + G.cpc - 1) / G.cpc;
    const int scene = blockIdx.y / cgroups, group = blockIdx.y - scene * cgroups;
    const int H = G.H, W = G.W, n = G.n, C = G.C;
    const size_t P = static_cast<size_t>(H) * W;
    const int ntx = (W + TA - 1) / TA;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const int r0 = by * TA, c0 = bx * TA;
    double* sk = sm + Lay::O_TAPS;
    double* sI = sm + Lay::O_I;
    double* sMu = sm + Lay::O_MU;
    double* sG = sm + Lay::O_G;
    double* sS = sm + Lay::O_S;
    double* sIS = sm + Lay::O_M;
    double* sM = sm + Lay::O_M;
    double* sq = sm + Lay::O_Q;
    double* sU = sm + Lay::O_U;
    const double* tp = taps + static_cast<size_t>(scene) * n * n;
    // data term: output u = 128 warp + 32 k + lane (k = 0..3) -> (sampling phase, cell); the
    // phase is uniform across a warp, so taps are broadcast reads
    constexpr int CPR = TA / CF, CPP = CPR * CPR;  // cells per row / per phase
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int iq0 = floordiv(r0 - C + CF - 1, CF), jq0 = floordiv(c0 - C + CF - 1, CF);
    const int QH = floordiv(r0 + TA - 1 + C, CF) - iq0 + 1, QW = floordiv(c0 + TA - 1 + C, CF) - jq0 + 1;
    constexpr int QS = Lay::QWP;  // padded row stride of the q window
    using D = a3::DT<(N_ > 0 ? N_ : 1), CF>;
    constexpr int DM = N_ > 0 ? D::DM : 1;
    const int ch_lo = group * G.cpc, ch_hi = min(G.cps, group * G.cpc + G.cpc);
    constexpr int KP = (WP * WP + NT - 1) / NT;
    const int QN = QH * QW;
    constexpr int KQ = (Lay::QWMAX * Lay::QWMAX + NT - 1) / NT;
    double pf_p[KP], pf_q[KQ];
    // issue the loads of channel `chl`'s p (R+4) and q windows into registers
    auto prefetch = [&](int chl) {
        const int ch = scene * G.cps + chl;
        const double* pp = pin + ch * P;
        if (CG) pp = pin + (static_cast<size_t>(st[ch].t & 1) * G.N + ch) * P;
        const double* qc = q + static_cast<size_t>(ch) * G.h * G.w;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const int e = threadIdx.x + k * NT;
            const int y = e / WP, x = e - y * WP;
            pf_p[k] = 0.0;
            if (e < WP * WP && !(G.dbg & 32))
                pf_p[k] = __ldg(pp + static_cast<size_t>(wrap_once(r0 - 4 + y, H)) * W + wrap_once(c0 - 4 + x, W));
        }
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
            const int e = threadIdx.x + k * NT;
            if (e < QN) {
                const int a = e / QW, b = e - a * QW;
                pf_q[k] = __ldg(qc + static_cast<size_t>(wrapi(iq0 + a, G.h)) * G.w + wrapi(jq0 + b, G.w));
            }
        }
    };
    auto next_active = [&](int chl) {
        while (chl < ch_hi && CG && st[scene * G.cps + chl].done) ++chl;
        return chl;
    };
    const double* I = guide + scene * P;
    const double* MU = wmu + scene * P;
    const double* GK = wg + scene * P;
    for (int e = threadIdx.x; e < n * n; e += NT) sk[e] = tp[e];
    constexpr int KI = (WI * WI + NT - 1) / NT, KK = (WK * WK + NT - 1) / NT;
    double vi[KI], vm[KK], vg[KK];
#pragma unroll
    for (int k = 0; k < KI; ++k) {
        const int e = threadIdx.x + k * NT;
        const int y = e / WI, x = e - y * WI;
        if (e < WI * WI) vi[k] = __ldg(I + static_cast<size_t>(wrap_once(r0 - 3 + y, H)) * W + wrap_once(c0 - 3 + x, W));
    }
#pragma unroll
    for (int k = 0; k < KK; ++k) {
        const int e = threadIdx.x + k * NT;
        const int y = e / WK, x = e - y * WK;
        const size_t gi = static_cast<size_t>(wrap_once(r0 - 2 + y, H)) * W + wrap_once(c0 - 2 + x, W);
        if (e < WK * WK) {
            vm[k] = __ldg(MU + gi);
            vg[k] = __ldg(GK + gi);
        }
    }
    int cur = next_active(ch_lo);
    if (cur < ch_hi) prefetch(cur);  // first channel's p / q in flight with the guide tile
#pragma unroll
    for (int k = 0; k < KI; ++k)
        if (threadIdx.x + k * NT < WI * WI) sI[threadIdx.x + k * NT] = vi[k];
#pragma unroll
    for (int k = 0; k < KK; ++k)
        if (threadIdx.x + k * NT < WK * WK) {
            sMu[threadIdx.x + k * NT] = vm[k];
            sG[threadIdx.x + k * NT] = vg[k];
        }

    for (int chl = cur; chl < ch_hi; chl = cur) {
        const int ch = scene * G.cps + chl;
        __syncthreads();  // previous channel finished with the shared buffers
        double* sP = sU;
#pragma unroll
        for (int k = 0; k < KP; ++k)
            if (threadIdx.x + k * NT < WP * WP) sP[threadIdx.x + k * NT] = pf_p[k];
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
            const int e = threadIdx.x + k * NT;
            if (e < QN) {
                const int a = e / QW, b = e - a * QW;
                sq[a * QS + b] = pf_q[k];
            }
        }
        cur = next_active(chl + 1);
        if (cur < ch_hi) prefetch(cur);  // in flight during this channel's stages
        __syncthreads();
        // own pixels' p for p.Ap in the S5 mapping (column pair 2 (tid % 16), rows 2 (tid / 16) + {0,1})
        double2 pown[2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
            pown[i] = ld2(sP + (2 * (threadIdx.x >> 4) + i + 4) * WP + 2 * (threadIdx.x & 15) + 4);
        // S4: data term (needs only q; writes its own buffer, so it runs before S1 without a barrier)
        double* sO = sm + Lay::O_O;
        if (N_ > 0 && !(G.dbg & 1)) {
            // thread = (phase, cell column, 4 cell rows); zero-padded phase sub-kernel in registers,
            // q rows slide through registers (each q value loaded once per thread)
            constexpr int CW4 = TA / CF, RB4 = CW4 / 4;
            const int Jc = threadIdx.x % CW4;
            const int rest = threadIdx.x / CW4;
            const int Ic0 = (rest % RB4) * 4;
            const int ph = rest / RB4;
            const int pr = ph / CF, pc = ph - pr * CF;
            double kreg[DM][DM];
#pragma unroll
            for (int a = 0; a < DM; ++a)
#pragma unroll
                for (int b = 0; b < DM; ++b) {
                    const int tr = CF * (a + D::DLO) - pr + D::C, tc = CF * (b + D::DLO) - pc + D::C;
                    kreg[a][b] = (tr >= 0 && tr < N_ && tc >= 0 && tc < N_) ? sk[tr * N_ + tc] : 0.0;
                }
            const double* qb = sq + (r0 / CF + Ic0 - iq0 + D::DLO) * QS + (c0 / CF + Jc - jq0 + D::DLO);
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int m = 0; m < DM + 3; ++m) {
                double qv[DM];
#pragma unroll
                for (int b = 0; b < DM; ++b) qv[b] = qb[m * QS + b];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int a = m - k;
                    if (a >= 0 && a < DM) {
#pragma unroll
                        for (int b = 0; b < DM; ++b) acc[k] = fma(kreg[a][b], qv[b], acc[k]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sO[((Ic0 + k) * CF + pr) * TA + Jc * CF + pc] = acc[k];
        } else if (!(G.dbg & 1)) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int u = 128 * warp + 32 * k + lane;
                const int ph = u / CPP, cell = u - ph * CPP;
                const int pr = ph / CF, pc = ph - pr * CF;
                const int ci = cell / CPR, cj = cell - ci * CPR;
                const int dilo = floordiv(pr - C + CF - 1, CF), dihi = floordiv(pr + C, CF);
                const int djlo = floordiv(pc - C + CF - 1, CF), djhi = floordiv(pc + C, CF);
                const double* qb = sq + (r0 / CF + ci - iq0) * QS + (c0 / CF + cj - jq0);
                double acc = 0.0;
                for (int di = dilo; di <= dihi; ++di) {
                    const double* krow = sk + (CF * di - pr + C) * n + C - pc;
                    const double* qrow = qb + di * QS;
                    for (int dj = djlo; dj <= djhi; ++dj) acc = fma(krow[CF * dj], qrow[dj], acc);
                }
                sO[(ci * CF + pr) * TA + cj * CF + pc] = acc;
            }
        }
        // S1-S3 and S5 work on column PAIRS (16-byte shared accesses, conflict-free) and walk short
        // strips of rows with the vertical 3-sums in a register sliding window.
        // S1: s = L p and I*s on R+3
        if (threadIdx.x < 19 * 13 && !(G.dbg & 2)) {
            const int xp = 2 * (threadIdx.x % 19), y0 = 3 * (threadIdx.x / 19);
            double2 a0 = ld2(sP + y0 * WP + xp), a1 = ld2(sP + y0 * WP + xp + 2);        // p rows y, y+1
            double2 b0 = ld2(sP + (y0 + 1) * WP + xp), b1 = ld2(sP + (y0 + 1) * WP + xp + 2);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int y = y0 + i;
                if (y < WI) {
                    const double2 e0 = ld2(sP + (y + 2) * WP + xp), e1 = ld2(sP + (y + 2) * WP + xp + 2);
                    // outputs at p columns xp+1, xp+2 (ops.cpp:70-78 operation order)
                    const double v0 = 4.0 * b0.y - a0.y - e0.y - b0.x - b1.x;
                    const double v1 = 4.0 * b1.x - a1.x - e1.x - b0.y - b1.y;
                    const double2 iv = ld2(sI + y * WI + xp);
                    st2(sS + y * WI + xp, make_double2(v0, v1));
                    st2(sIS + y * WI + xp, make_double2(iv.x * v0, iv.y * v1));
                    a0 = b0; a1 = b1; b0 = e0; b1 = e1;
                }
            }
        }
        __syncthreads();
        // S2: per-window a_k, c1_k on R+2 from 3x3 sums of s and I*s
        double* sA = sU;
        double* sC = sU + WK * WK;
        if (threadIdx.x < 18 * 14 && !(G.dbg & 4)) {
            const int xp = 2 * (threadIdx.x % 18), y0 = 3 * (threadIdx.x / 18);
            auto hpair = [&](const double* a, int y) {  // horizontal 3-sums at columns xp, xp+1
                const double2 u = ld2(a + y * WI + xp), v = ld2(a + y * WI + xp + 2);
                return make_double2(u.x + u.y + v.x, u.y + v.x + v.y);
            };
            double2 s0 = hpair(sS, y0), s1 = hpair(sS, y0 + 1);
            double2 i0 = hpair(sIS, y0), i1 = hpair(sIS, y0 + 1);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int y = y0 + i;
                if (y < WK) {
                    const double2 s2 = hpair(sS, y + 2), i2 = hpair(sIS, y + 2);
                    const double2 mu = ld2(sMu + y * WK + xp), g = ld2(sG + y * WK + xp);
                    double2 a, c;
                    {
                        const double xb = (s0.x + s1.x + s2.x) * (1.0 / 9.0);  // box mean, no fp64 division
                        a.x = g.x * ((i0.x + i1.x + i2.x) * (1.0 / 9.0) - mu.x * xb);
                        c.x = g.x != 0.0 ? xb - mu.x * a.x : 0.0;
                    }
                    {
                        const double xb = (s0.y + s1.y + s2.y) * (1.0 / 9.0);
                        a.y = g.y * ((i0.y + i1.y + i2.y) * (1.0 / 9.0) - mu.y * xb);
                        c.y = g.y != 0.0 ? xb - mu.y * a.y : 0.0;
                    }
                    st2(sA + y * WK + xp, a);
                    st2(sC + y * WK + xp, c);
                    s0 = s1; s1 = s2; i0 = i1; i1 = i2;
                }
            }
        }
        __syncthreads();
        // S3: M s on R+1 = n_m s_m - box(c1) - I_m box(a)
        if (threadIdx.x < 17 * 15 && !(G.dbg & 8)) {
            const int xp = 2 * (threadIdx.x % 17), y0 = 3 * (threadIdx.x / 17);
            auto hpair = [&](const double* a, int y) {
                const double2 u = ld2(a + y * WK + xp), v = ld2(a + y * WK + xp + 2);
                return make_double2(u.x + u.y + v.x, u.y + v.x + v.y);
            };
            double2 a0 = hpair(sA, y0), a1 = hpair(sA, y0 + 1);
            double2 k0 = hpair(sC, y0), k1 = hpair(sC, y0 + 1);
            const int gc0 = wrap_once(c0 - 1 + xp, W), gc1 = wrap_once(c0 + xp, W);
            const int nc0 = max(min(gc0 + 1, W - 2) - max(gc0 - 1, 1) + 1, 0);
            const int nc1 = max(min(gc1 + 1, W - 2) - max(gc1 - 1, 1) + 1, 0);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int y = y0 + i;
                if (y < WM) {
                    const double2 a2v = hpair(sA, y + 2), k2 = hpair(sC, y + 2);
                    const int gr = wrap_once(r0 - 1 + y, H);
                    const int nr = max(min(gr + 1, H - 2) - max(gr - 1, 1) + 1, 0);
                    const double2 sv = ld2(sS + (y + 2) * WI + xp + 2), iv = ld2(sI + (y + 2) * WI + xp + 2);
                    double2 m;
                    m.x = static_cast<double>(nr * nc0) * sv.x - (k0.x + k1.x + k2.x) - iv.x * (a0.x + a1.x + a2v.x);
                    m.y = static_cast<double>(nr * nc1) * sv.y - (k0.y + k1.y + k2.y) - iv.y * (a0.y + a1.y + a2v.y);
                    st2(sM + y * WM + xp, m);  // sM aliases I*s: dead after S2, not read here
                    a0 = a1; a1 = a2v; k0 = k1; k1 = k2;
                }
            }
        }
        __syncthreads();
        // S5: t = L(M s), Ap = data + lambda t, p.Ap
        double* oc = out + ch * P;
        double dotp = 0.0;
        if (!(G.dbg & 16)) {
            const int xp = 2 * (threadIdx.x & 15), y0 = 2 * (threadIdx.x >> 4);
            double2 a0 = ld2(sM + y0 * WM + xp), a1 = ld2(sM + y0 * WM + xp + 2);
            double2 b0 = ld2(sM + (y0 + 1) * WM + xp), b1 = ld2(sM + (y0 + 1) * WM + xp + 2);
            const int Cc = c0 + xp;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int y = y0 + i;
                const double2 e0 = ld2(sM + (y + 2) * WM + xp), e1 = ld2(sM + (y + 2) * WM + xp + 2);
                const double t0 = 4.0 * b0.y - a0.y - e0.y - b0.x - b1.x;
                const double t1 = 4.0 * b1.x - a1.x - e1.x - b0.y - b1.y;
                const double2 dv = ld2(sO + y * TA + xp);
                const double2 val = make_double2(dv.x + t0 * G.lambda, dv.y + t1 * G.lambda);
                a0 = b0; a1 = b1; b0 = e0; b1 = e1;
                const int R = r0 + y;
                if (R < H && Cc + 1 < W && !(W & 1)) {
                    *reinterpret_cast<double2*>(oc + static_cast<size_t>(R) * W + Cc) = val;
                    dotp += pown[i].x * val.x + pown[i].y * val.y;
                } else if (R < H) {
                    if (Cc < W) {
                        oc[static_cast<size_t>(R) * W + Cc] = val.x;
                        dotp += pown[i].x * val.x;
                    }
                    if (Cc + 1 < W) {
                        oc[static_cast<size_t>(R) * W + Cc + 1] = val.y;
                        dotp += pown[i].y * val.y;
                    }
                }
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
