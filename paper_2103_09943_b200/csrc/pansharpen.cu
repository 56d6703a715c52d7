// pansharpen.cu -- sm_100a kernels of Algorithm 2 (per-channel HRMS estimation under the
// local Laplacian prior), reference /root/reference/proj/src/pansharpen.cpp.
//
// Hot loop (pansharpen.cpp:237-256) per CG iteration, all channels of a scene batched in
// grid.y, three kernels, scalars resident on the device:
//   K_Q  p <- r + beta p (fused on load), q = D B p at the LR points          (north-star b)
//   K_A  Ap = B^T U q + lambda L M L p, matrix-free matting operator          (north-star a)
//   K_U  z += alpha p, r -= alpha Ap, ||r||^2, ||z||^2, stop test             (north-star c)
// Reductions are deterministic: fixed per-block trees, per-block partials, and a fixed-order
// final sum in the last block to finish (threadfence reduction); no floating-point atomics.
#include <cmath>
#include <cstdlib>

#include "pansharpen.cuh"
#include <nccl.h>

#include "cg_fast.cuh"

namespace fbmp_gpu {

PsGeo make_geo(int N, int h, int w, int c, int n, int rw, double lambda, double eps, int cps) {
    PsGeo G;
    G.N = N;
    G.cps = cps > 0 ? cps : N;
    const char* env = std::getenv("FBMP_KA_CPC");
    // channels per K_D CTA: all of the scene's, except on small images where fewer tiles than SMs
    // would leave the GPU idle (C1: 64 tiles -> 2 channels per CTA, 7.90 -> 7.71 ms; same bits)
    const long long tiles = static_cast<long long>((h * c + 31) / 32) * ((w * c + 31) / 32) * ((N + G.cps - 1) / G.cps);
    const int cpc_def = tiles < 128 ? std::min(2, G.cps) : G.cps;
    G.cpc = std::min(env ? std::max(1, std::atoi(env)) : cpc_def, fast::a4::MAXCPC);
    const char* dbg = std::getenv("FBMP_KA_DBG");
    G.dbg = dbg ? std::atoi(dbg) : 0;
    G.h = h; G.w = w; G.c = c;
    G.H = h * c; G.W = w * c;
    G.n = n; G.C = (n - 1) / 2;
    G.g = (G.C + c - 1) / c;
    G.rw = rw;
    G.lambda = lambda;
    G.eps = eps;
    G.grow0 = 0;
    G.Hg = G.H;
    G.rlo = 0;
    G.rhi = G.H;
    G.dred = nullptr;
    G.identity = 0;
    return G;
}

namespace {

constexpr int TQ = 16;            // K_Q LR tile side
constexpr int NTQ = TQ * TQ;      // threads per K_Q block
constexpr int TA = 32;            // K_A / K_GF HR tile side
constexpr int NTA = 256;          // threads per K_A block
constexpr int NTU = 256;          // threads per K_U block
#ifndef FBMP_UPT
#define FBMP_UPT 8
#endif
constexpr int UPT = FBMP_UPT;     // elements per thread in K_U
// fp32 K_U: twice the elements per thread (float4 runs), so a thread keeps as many bytes in flight
template <class T>
constexpr int upt() { return sizeof(T) == 8 ? UPT : 2 * UPT; }

__host__ __device__ inline int plane_stride(int pw) {  // >= pw*pw and == 4 (mod 16)
    const int s = pw * pw;
    return s + ((4 - s % 16) + 16) % 16;
}

// ------------------------------------------------------------------------------------------
// K_Q: q = D B p at the LR points of a TQ x TQ LR tile (+ fused p update in CG mode).
// The HR region (tile footprint + halo c*g >= C) is staged in shared memory split into
// c x c sampling phases so that lanes reading consecutive LR columns hit consecutive words.
// ------------------------------------------------------------------------------------------
template <bool CG>
__global__ void __launch_bounds__(NTQ) k_q(PsGeo G, const double* __restrict__ taps, const double* __restrict__ src,
                                           double* __restrict__ pbuf, double* __restrict__ q, CgState* st,
                                           double* __restrict__ part, int nblk) {
    __shared__ double red[NTQ / 32 + 1];
    extern __shared__ double sm[];
    const int ch = blockIdx.y;
    int t = 0;
    double beta = 0.0;
    if (CG) {
        if (st[ch].done) return;
        t = st[ch].t;
        beta = t ? st[ch].beta : 0.0;
    }
    const int c = G.c, n = G.n, C = G.C, g = G.g;
    const size_t P = static_cast<size_t>(G.H) * G.W;
    const double* rc = src + ch * P;
    const double* pold = CG ? pbuf + (static_cast<size_t>((t + 1) & 1) * G.N + ch) * P : nullptr;
    double* pnew = CG ? pbuf + (static_cast<size_t>(t & 1) * G.N + ch) * P : nullptr;

    const int ntx = (G.w + TQ - 1) / TQ;
    const int tyb = blockIdx.x / ntx, txb = blockIdx.x - tyb * ntx;
    const int i0 = tyb * TQ, j0 = txb * TQ;
    const int PW = TQ + 2 * g, PS = plane_stride(PW), SR = c * PW;
    double* sk = sm;
    double* planes = sm + ((n * n + 1) & ~1);
    const double* tp = taps + static_cast<size_t>(ch / G.cps) * n * n;
    for (int e = threadIdx.x; e < n * n; e += NTQ) sk[e] = tp[e];

    const int R0 = c * (i0 - g), C0 = c * (j0 - g);
    double pp = 0.0;
    for (int e = threadIdx.x; e < SR * SR; e += NTQ) {
        const int rr = e / SR, cc = e - rr * SR;
        const int R = wrapi(R0 + rr, G.H), Cc = wrapi(C0 + cc, G.W);
        const size_t gi = static_cast<size_t>(R) * G.W + Cc;
        double v = __ldg(rc + gi);
        if (CG) {
            v = v + __ldg(pold + gi) * beta;  // pansharpen.cpp:254  p = r + p * beta
            const int orr = rr - c * g, occ = cc - c * g;
            if (orr >= 0 && orr < c * TQ && occ >= 0 && occ < c * TQ && R0 + rr < G.H && C0 + cc < G.W) {
                pnew[gi] = v;
                pp += v * v;
            }
        }
        planes[((rr % c) * c + (cc % c)) * PS + (rr / c) * PW + cc / c] = v;
    }
    __syncthreads();

    const int ti = threadIdx.x / TQ, tj = threadIdx.x - ti * TQ;
    const int i = i0 + ti, j = j0 + tj;
    if (i < G.h && j < G.w) {
        double acc = 0.0;
        for (int a = -C; a <= C; ++a) {  // (B p)(ci,cj) = sum_ab k[a+C][b+C] p(ci-a, cj-b)
            const int rr = c * (ti + g) - a;
            const double* base = planes + (rr % c) * c * PS + (rr / c) * PW;
            const double* krow = sk + (a + C) * n;
            const int cc0 = c * (tj + g) - C;
            int pc = cc0 % c, J = cc0 / c;
            for (int b = C; b >= -C; --b) {
                acc = fma(krow[b + C], base[pc * PS + J], acc);
                if (++pc == c) { pc = 0; ++J; }
            }
        }
        q[static_cast<size_t>(ch) * G.h * G.w + static_cast<size_t>(i) * G.w + j] = acc;
    }
    if (CG) {
        const double bs = block_sum<NTQ>(pp, red);
        if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
        if (elect_last_block(&st[ch].cnt_q, nblk)) {
            const double tot = sum_partials<NTQ>(part + static_cast<size_t>(ch) * nblk, nblk, 1, red);
            if (threadIdx.x == 0) {
                st[ch].pp = tot;
                st[ch].cnt_q = 0;
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// K_A: out = B^T U q (+) lambda * L M L p on a TA x TA HR tile.
// MODE 0: full CG operator (pansharpen.cpp:218-223); 1: M p only (:197-202); 2: data term only.
// The matting operator is applied matrix-free (pansharpen.cpp:155-164 regrouped per window):
//   (M s)_m = sum_{interior k with m in w_k} [ s_m - mean_k(s) - (I_m - mu_k) a_k ],
//   a_k = mean_k((I - mu_k) s) / (eps/|w| + var_k),
// with mu_k, var_k recomputed in-tile from the guide I (no per-scene maps are read).
// ------------------------------------------------------------------------------------------
struct ApplyLayout {
    int hp, hI, hs, hwin, hM;  // halos of p, I, s, window stats, M s
    int iq0, jq0, QH, QW;      // LR q window
    int off_q, off_p, off_I, off_s, off_x, off_a, off_mu, off_w, off_M, total;
};

__host__ __device__ inline ApplyLayout apply_layout(const PsGeo& G, int mode, int r0, int c0) {
    ApplyLayout L{};
    const int rw = G.rw;
    const int e = mode == 0 ? 1 : 0;
    L.hM = e;
    L.hwin = rw + e;
    L.hs = 2 * rw + e;
    L.hI = 2 * rw + e;
    L.hp = mode == 2 ? 0 : L.hs + e;
    const int c = G.c, C = G.C;
    // LR rows whose c-multiple lies within C of the tile rows
    auto fdiv = [](int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
    L.iq0 = fdiv(r0 - C + c - 1, c);
    L.jq0 = fdiv(c0 - C + c - 1, c);
    L.QH = fdiv(r0 + TA - 1 + C, c) - L.iq0 + 1;
    L.QW = fdiv(c0 + TA - 1 + C, c) - L.jq0 + 1;
    int o = 0;
    auto take = [&](int cnt) { const int at = o; o += (cnt + 1) & ~1; return at; };
    const int n2 = G.n * G.n;
    const int dq = (TA - 1 + 2 * C) / c + 2;  // upper bound of QH / QW for any tile origin
    take(n2);  // taps at offset 0
    L.off_q = take(dq * dq);
    if (mode != 2) {
        const int sp = TA + 2 * L.hp, sI = TA + 2 * L.hI, ss = TA + 2 * L.hs, sw = TA + 2 * L.hwin,
                  sM = TA + 2 * L.hM;
        L.off_p = take(sp * sp);
        L.off_I = take(sI * sI);
        L.off_s = mode == 0 ? take(ss * ss) : L.off_p;
        L.off_x = take(sw * sw);
        L.off_a = take(sw * sw);
        L.off_mu = take(sw * sw);
        L.off_w = take(sw * sw);
        L.off_M = take(sM * sM);
    }
    L.total = o;
    return L;
}

template <int MODE, bool CG>
__global__ void __launch_bounds__(NTA) k_apply(PsGeo G, const double* __restrict__ taps,
                                               const double* __restrict__ guide, const double* __restrict__ pin,
                                               const double* __restrict__ q, double* __restrict__ out, CgState* st,
                                               double* __restrict__ part, int nblk) {
    __shared__ double red[NTA / 32 + 1];
    extern __shared__ double sm[];
    const int ch = blockIdx.y;
    const size_t P = static_cast<size_t>(G.H) * G.W;
    const double* p = pin + ch * P;
    int t = 0;
    if (CG) {
        if (st[ch].done) return;
        t = st[ch].t;
        p = pin + (static_cast<size_t>(t & 1) * G.N + ch) * P;
    }
    const int ntx = (G.W + TA - 1) / TA;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const int r0 = by * TA, c0 = bx * TA;
    const ApplyLayout L = apply_layout(G, MODE, r0, c0);
    const int H = G.H, W = G.W, c = G.c, n = G.n, C = G.C, rw = G.rw;
    double* sk = sm;
    double* sq = sm + L.off_q;
    const double* tp = taps + static_cast<size_t>(ch / G.cps) * n * n;
    if (guide) guide += static_cast<size_t>(ch / G.cps) * P;
    for (int e = threadIdx.x; e < n * n; e += NTA) sk[e] = tp[e];
    if (MODE != 1) {
        const double* qc = q + static_cast<size_t>(ch) * G.h * G.w;
        for (int e = threadIdx.x; e < L.QH * L.QW; e += NTA) {
            const int a = e / L.QW, b = e - a * L.QW;
            sq[e] = __ldg(qc + static_cast<size_t>(wrapi(L.iq0 + a, G.h)) * G.w + wrapi(L.jq0 + b, G.w));
        }
    }
    const int SPW = TA + 2 * L.hp, SIW = TA + 2 * L.hI, SSW = TA + 2 * L.hs, SWW = TA + 2 * L.hwin,
              SMW = TA + 2 * L.hM;
    double *sp = sm + L.off_p, *sI = sm + L.off_I, *ss = sm + L.off_s;
    double *sx = sm + L.off_x, *sa = sm + L.off_a, *smu = sm + L.off_mu, *swt = sm + L.off_w, *sM = sm + L.off_M;
    if (MODE != 2) {
        for (int e = threadIdx.x; e < SPW * SPW; e += NTA) {
            const int y = e / SPW, x = e - y * SPW;
            sp[e] = __ldg(p + static_cast<size_t>(wrapi(r0 - L.hp + y, H)) * W + wrapi(c0 - L.hp + x, W));
        }
        for (int e = threadIdx.x; e < SIW * SIW; e += NTA) {
            const int y = e / SIW, x = e - y * SIW;
            sI[e] = __ldg(guide + static_cast<size_t>(wrapi(r0 - L.hI + y, H)) * W + wrapi(c0 - L.hI + x, W));
        }
        __syncthreads();
        if (MODE == 0) {  // s = L p on R + hs (ops.cpp:70-78 stencil order)
            for (int e = threadIdx.x; e < SSW * SSW; e += NTA) {
                const int y = e / SSW + 1, x = e % SSW + 1;
                ss[e] = 4.0 * sp[y * SPW + x] - sp[(y - 1) * SPW + x] - sp[(y + 1) * SPW + x] - sp[y * SPW + x - 1] -
                        sp[y * SPW + x + 1];
            }
            __syncthreads();
        }
        // per-window statistics on R + hwin
        const double ws = static_cast<double>((2 * rw + 1) * (2 * rw + 1));
        const int oI = L.hI - L.hwin, oS = L.hs - L.hwin;
        for (int e = threadIdx.x; e < SWW * SWW; e += NTA) {
            const int y = e / SWW, x = e - y * SWW;
            const int gr = wrapi(r0 - L.hwin + y, H), gc = wrapi(c0 - L.hwin + x, W);
            double xb = 0.0, a = 0.0, mu = 0.0, wt = 0.0;
            if (gr >= rw && gr < H - rw && gc >= rw && gc < W - rw) {  // interior centre (:152-153)
                double s1 = 0.0, s2 = 0.0, sx_ = 0.0;
                for (int dy = -rw; dy <= rw; ++dy)
                    for (int dx = -rw; dx <= rw; ++dx) {
                        const double iv = sI[(y + oI + dy) * SIW + x + oI + dx];
                        s1 += iv;
                        s2 += iv * iv;
                        sx_ += ss[(y + oS + dy) * SSW + x + oS + dx];
                    }
                mu = s1 / ws;
                const double var = s2 / ws - mu * mu;
                const double den = G.eps / ws + var;  // pansharpen.cpp:155
                double sc = 0.0;
                for (int dy = -rw; dy <= rw; ++dy)
                    for (int dx = -rw; dx <= rw; ++dx)
                        sc += (sI[(y + oI + dy) * SIW + x + oI + dx] - mu) * ss[(y + oS + dy) * SSW + x + oS + dx];
                xb = sx_ / ws;
                a = (sc / ws) / den;
                wt = 1.0;
            }
            sx[e] = xb;
            sa[e] = a;
            smu[e] = mu;
            swt[e] = wt;
        }
        __syncthreads();
        // M s on R + hM
        const int oW = L.hwin - L.hM, oSM = L.hs - L.hM, oIM = L.hI - L.hM;
        for (int e = threadIdx.x; e < SMW * SMW; e += NTA) {
            const int y = e / SMW, x = e - y * SMW;
            const double sv = ss[(y + oSM) * SSW + x + oSM];
            const double iv = sI[(y + oIM) * SIW + x + oIM];
            double acc = 0.0;
            for (int dy = -rw; dy <= rw; ++dy)
                for (int dx = -rw; dx <= rw; ++dx) {
                    const int k = (y + oW + dy) * SWW + x + oW + dx;
                    acc += swt[k] * sv - sx[k] - (iv - smu[k]) * sa[k];
                }
            sM[e] = acc;
        }
    }
    __syncthreads();

    double* oc = out + ch * P;
    double dotp = 0.0;
    const int tx = threadIdx.x & 31, ty0 = threadIdx.x >> 5;
    for (int ty = ty0; ty < TA; ty += NTA / 32) {
        const int R = r0 + ty, Cc = c0 + tx;
        if (R >= H || Cc >= W) continue;
        double val = 0.0;
        if (MODE != 1) {  // data term: sum over LR points within C of (R, Cc)
            const int ilo = floordiv(R - C + c - 1, c), ihi = floordiv(R + C, c);
            const int jlo = floordiv(Cc - C + c - 1, c), jhi = floordiv(Cc + C, c);
            double acc = 0.0;
            for (int i = ilo; i <= ihi; ++i) {
                const double* krow = sk + (c * i - R + C) * n + C - Cc;
                const double* qrow = sq + (i - L.iq0) * L.QW - L.jq0;
                for (int j = jlo; j <= jhi; ++j) acc = fma(krow[c * j], qrow[j], acc);
            }
            val = acc;
        }
        if (MODE == 0) {
            const int y = ty + 1, x = tx + 1;
            const double tl = 4.0 * sM[y * SMW + x] - sM[(y - 1) * SMW + x] - sM[(y + 1) * SMW + x] -
                              sM[y * SMW + x - 1] - sM[y * SMW + x + 1];
            val = val + tl * G.lambda;
        } else if (MODE == 1) {
            val = sM[ty * SMW + tx];
        }
        oc[static_cast<size_t>(R) * W + Cc] = val;
        if (CG) dotp += sp[(ty + L.hp) * SPW + tx + L.hp] * val;
    }
    if (CG) {
        const double bs = block_sum<NTA>(dotp, red);
        if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
        if (elect_last_block(&st[ch].cnt_a, nblk)) {
            const double pAp = sum_partials<NTA>(part + static_cast<size_t>(ch) * nblk, nblk, 1, red);
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

// ------------------------------------------------------------------------------------------
// K_U: z += alpha p, r -= alpha Ap, ||r||^2, ||z||^2 and the relative-step stop test
// (pansharpen.cpp:245-255).
// ------------------------------------------------------------------------------------------
template <class T = double>
__global__ void __launch_bounds__(NTU) k_update(PsGeo G, T* __restrict__ z, T* __restrict__ r,
                                                const T* __restrict__ pbuf, const T* __restrict__ Ap,
                                                CgState* st, double* __restrict__ part, int nblk) {
    using V = fast::v2<T>;
    __shared__ double red[2 * (NTU / 32 + 1)];
    const int ch = blockIdx.y;
    // t and z, r, p are not written by K_A (the predecessor): read them before pdl_wait so the
    // loads overlap K_A's tail; done may still be set by K_A (pAp <= 0) and is re-checked
    if (__syncthreads_or(st[ch].done)) return;  // uniform: the reductions below stay convergent
    const int t = st[ch].t;
    const size_t P = static_cast<size_t>(G.H) * G.W;
    const T* pc = pbuf + (static_cast<size_t>(t & 1) * G.N + ch) * P;
    T* zc = z + ch * P;
    T* rc = r + ch * P;
    const T* ac = Ap + ch * P;
    double rr = 0.0, zz = 0.0;
    constexpr int EPT = upt<T>();
    const size_t base = static_cast<size_t>(blockIdx.x) * NTU * EPT;
    const size_t own_lo = static_cast<size_t>(G.rlo) * G.W, own_hi = static_cast<size_t>(G.rhi) * G.W;
    // the whole block's range is owned (always, unless the CG runs on a row strip)
    const bool all_owned = base >= own_lo && base + static_cast<size_t>(NTU) * EPT <= own_hi;
    if constexpr (!std::is_same<T, double>::value) {
        if ((P & 3) == 0) {  // fp32: 16-byte runs of four elements, fp64 sums
            constexpr int KV = EPT / 4;
            const size_t nv = P / 4;
            float4 pv[KV], av[KV], zv[KV], rv[KV];
#pragma unroll
            for (int k = 0; k < KV; ++k) {
                const size_t vi = base / 4 + static_cast<size_t>(k) * NTU + threadIdx.x;
                if (vi < nv) {
                    pv[k] = __ldcs(reinterpret_cast<const float4*>(pc) + vi);
                    zv[k] = __ldcs(reinterpret_cast<const float4*>(zc) + vi);
                    rv[k] = __ldcs(reinterpret_cast<const float4*>(rc) + vi);
                }
            }
            pdl_wait();
            pdl_trigger();
            if (__syncthreads_or(st[ch].done)) return;
            const float alpha = static_cast<float>(st[ch].alpha);
#pragma unroll
            for (int k = 0; k < KV; ++k) {
                const size_t vi = base / 4 + static_cast<size_t>(k) * NTU + threadIdx.x;
                if (vi < nv) av[k] = __ldcs(reinterpret_cast<const float4*>(ac) + vi);
            }
#pragma unroll
            for (int k = 0; k < KV; ++k) {
                const size_t vi = base / 4 + static_cast<size_t>(k) * NTU + threadIdx.x;
                if (vi < nv) {
                    float* zf = &zv[k].x;
                    float* rf = &rv[k].x;
                    const float* pf = &pv[k].x;
                    const float* af = &av[k].x;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        zf[u] = zf[u] + pf[u] * alpha;
                        rf[u] = rf[u] - af[u] * alpha;
                        const bool o = all_owned || (4 * vi + u >= own_lo && 4 * vi + u < own_hi);
                        const double rx = rf[u], zx = zf[u];
                        rr += o ? rx * rx : 0.0;
                        zz += o ? zx * zx : 0.0;
                    }
                    __stcs(reinterpret_cast<float4*>(zc) + vi, zv[k]);
                    __stcs(reinterpret_cast<float4*>(rc) + vi, rv[k]);
                }
            }
            goto reduce;
        }
    }
    if ((P & 1) == 0) {
        constexpr int KV = EPT / 2;
        const size_t nv = P / 2;
        V pv[KV], av[KV], zv[KV], rv[KV];
#pragma unroll
        for (int k = 0; k < KV; ++k) {
            const size_t vi = base / 2 + static_cast<size_t>(k) * NTU + threadIdx.x;
            if (vi < nv) {
                pv[k] = __ldcs(reinterpret_cast<const V*>(pc) + vi);
                zv[k] = __ldcs(reinterpret_cast<const V*>(zc) + vi);
                rv[k] = __ldcs(reinterpret_cast<const V*>(rc) + vi);
            }
        }
        pdl_wait();
        pdl_trigger();
        if (__syncthreads_or(st[ch].done)) return;
        const T alpha = static_cast<T>(st[ch].alpha);
#pragma unroll
        for (int k = 0; k < KV; ++k) {
            const size_t vi = base / 2 + static_cast<size_t>(k) * NTU + threadIdx.x;
            if (vi < nv) av[k] = __ldcs(reinterpret_cast<const V*>(ac) + vi);
        }
#pragma unroll
        for (int k = 0; k < KV; ++k) {
            const size_t vi = base / 2 + static_cast<size_t>(k) * NTU + threadIdx.x;
            if (vi < nv) {
                zv[k].x = zv[k].x + pv[k].x * alpha; zv[k].y = zv[k].y + pv[k].y * alpha;
                rv[k].x = rv[k].x - av[k].x * alpha; rv[k].y = rv[k].y - av[k].y * alpha;
                __stcs(reinterpret_cast<V*>(zc) + vi, zv[k]);
                __stcs(reinterpret_cast<V*>(rc) + vi, rv[k]);
                // owned rows only (all, unless the CG runs on a row strip); selects keep the
                // whole-image sums bit-identical to the plain x^2 + y^2 accumulation
                const bool ox = all_owned || (2 * vi >= own_lo && 2 * vi < own_hi);
                const bool oy = all_owned || (2 * vi + 1 >= own_lo && 2 * vi + 1 < own_hi);
                if constexpr (std::is_same<T, double>::value) {
                    rr += (ox ? rv[k].x * rv[k].x : 0.0) + (oy ? rv[k].y * rv[k].y : 0.0);
                    zz += (ox ? zv[k].x * zv[k].x : 0.0) + (oy ? zv[k].y * zv[k].y : 0.0);
                } else {  // fp32 vectors, fp64 sums
                    const double rx = rv[k].x, ry = rv[k].y, zx = zv[k].x, zy = zv[k].y;
                    rr += (ox ? rx * rx : 0.0) + (oy ? ry * ry : 0.0);
                    zz += (ox ? zx * zx : 0.0) + (oy ? zy * zy : 0.0);
                }
            }
        }
    } else {
        pdl_wait();
        pdl_trigger();
        if (__syncthreads_or(st[ch].done)) return;
        const T alpha = static_cast<T>(st[ch].alpha);
        for (int k = 0; k < EPT; ++k) {
            const size_t i = base + static_cast<size_t>(k) * NTU + threadIdx.x;
            if (i >= P) break;
            const T zv = zc[i] + pc[i] * alpha;
            const T rv = rc[i] - ac[i] * alpha;
            zc[i] = zv;
            rc[i] = rv;
            if (all_owned || (i >= own_lo && i < own_hi)) {
                rr += static_cast<double>(rv) * static_cast<double>(rv);
                zz += static_cast<double>(zv) * static_cast<double>(zv);
            }
        }
    }
reduce:
    const double2 bs = block_sum2<NTU>(rr, zz, red);
    if (threadIdx.x == 0) {
        part[(static_cast<size_t>(ch) * nblk + blockIdx.x) * 2] = bs.x;
        part[(static_cast<size_t>(ch) * nblk + blockIdx.x) * 2 + 1] = bs.y;
    }
    if (elect_last_block(&st[ch].cnt_u, nblk)) {
        const double2 tot = sum_partials2<NTU>(part + static_cast<size_t>(ch) * nblk * 2, nblk, red);
        const double rs_new = tot.x, zsq = tot.y;
        if (threadIdx.x == 0 && G.dred) {  // distributed: publish the local sums only
            G.dred[G.N + 3 * ch + 1] = rs_new;
            G.dred[G.N + 3 * ch + 2] = zsq;
            st[ch].cnt_u = 0;
        } else if (threadIdx.x == 0) {
            CgState& S = st[ch];
            const double step = fabs(S.alpha) * sqrt(S.pp);
            S.zz = zsq;
            if (step <= S.cg_tol * fmax(sqrt(zsq), 1e-300)) {
                S.done = 1;
                S.iters = t + 1;
            } else {
                S.beta = rs_new / S.rs;
                S.rs = rs_new;
                S.t = t + 1;
                if (S.t >= S.max_iters) {
                    S.done = 3;
                    S.iters = S.max_iters;
                }
            }
            S.cnt_u = 0;
        }
    }
}

// CG initialisation after rhs = B^T U x has been written to r by K_D (pansharpen.cpp:225-235):
// z = 0, p_old = 0, rs = ||rhs||^2 over the owned rows, state reset.
template <class T = double>
__global__ void __launch_bounds__(NTU) k_cg_init(PsGeo G, const T* __restrict__ r, T* __restrict__ z,
                                                 T* __restrict__ p1, CgState* st, double* __restrict__ part,
                                                 int nblk, int max_iters, double cg_tol) {
    __shared__ double red[NTU / 32 + 1];
    const int ch = blockIdx.y;
    const size_t P = static_cast<size_t>(G.H) * G.W;
    const T* rc = r + ch * P;
    T* zc = z + ch * P;
    T* pc = p1 + ch * P;
    const size_t own_lo = static_cast<size_t>(G.rlo) * G.W, own_hi = static_cast<size_t>(G.rhi) * G.W;
    double ss = 0.0;
    const size_t base = static_cast<size_t>(blockIdx.x) * NTU * UPT;
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        const size_t i = base + static_cast<size_t>(k) * NTU + threadIdx.x;
        if (i < P) {
            const double v = rc[i];
            zc[i] = T(0);
            pc[i] = T(0);
            ss += (i >= own_lo && i < own_hi) ? v * v : 0.0;
        }
    }
    const double bs = block_sum<NTU>(ss, red);
    if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
    if (elect_last_block(&st[ch].cnt_init, nblk)) {
        const double tot = sum_partials<NTU>(part + static_cast<size_t>(ch) * nblk, nblk, 1, red);
        if (threadIdx.x == 0 && G.dred) {  // distributed: publish the local sum only
            G.dred[G.N + 3 * ch + 1] = tot;
            st[ch].cnt_init = 0;
        } else if (threadIdx.x == 0) {
            CgState& S = st[ch];
            S.rs = tot;
            S.rhs_norm = sqrt(tot);
            S.pp = S.pAp = S.alpha = S.beta = S.zz = S.qq = 0.0;
            S.cg_tol = cg_tol;
            S.t = 0;
            S.iters = 0;
            S.max_iters = max_iters;
            S.done = (S.rhs_norm == 0.0) ? 1 : (max_iters <= 0 ? 3 : 0);
            S.cnt_q = S.cnt_a = S.cnt_u = 0;
            S.cnt_init = 0;
        }
    }
}

// ------------------------------------------------------------------------------------------
// rhs = B^T U x and CG initialisation (pansharpen.cpp:225-235).
// ------------------------------------------------------------------------------------------
template <bool CG>
__global__ void __launch_bounds__(NTA) k_rhs(PsGeo G, const double* __restrict__ taps, const double* __restrict__ x,
                                             double* __restrict__ rhs, double* __restrict__ z, double* __restrict__ p1,
                                             CgState* st, double* __restrict__ part, int nblk, int max_iters,
                                             double cg_tol) {
    __shared__ double red[NTA / 32 + 1];
    extern __shared__ double sk[];
    const int ch = blockIdx.y;
    const int H = G.H, W = G.W, c = G.c, n = G.n, C = G.C;
    const double* tp = taps + static_cast<size_t>(ch / G.cps) * n * n;
    for (int e = threadIdx.x; e < n * n; e += NTA) sk[e] = tp[e];
    __syncthreads();
    const int ntx = (W + TA - 1) / TA;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const size_t P = static_cast<size_t>(H) * W;
    const double* xc = x + static_cast<size_t>(ch) * G.h * G.w;
    double ss = 0.0;
    const int tx = threadIdx.x & 31;
    for (int ty = threadIdx.x >> 5; ty < TA; ty += NTA / 32) {
        const int R = by * TA + ty, Cc = bx * TA + tx;
        if (R >= H || Cc >= W) continue;
        const int ilo = floordiv(R - C + c - 1, c), ihi = floordiv(R + C, c);
        const int jlo = floordiv(Cc - C + c - 1, c), jhi = floordiv(Cc + C, c);
        double acc = 0.0;
        for (int i = ilo; i <= ihi; ++i) {
            const double* krow = sk + (c * i - R + C) * n + C - Cc;
            const double* xrow = xc + static_cast<size_t>(wrapi(i, G.h)) * G.w;
            for (int j = jlo; j <= jhi; ++j) acc = fma(krow[c * j], __ldg(xrow + wrapi(j, G.w)), acc);
        }
        const size_t gi = ch * P + static_cast<size_t>(R) * W + Cc;
        rhs[gi] = acc;
        if (CG) {
            z[gi] = 0.0;
            p1[gi] = 0.0;
            if (R >= G.rlo && R < G.rhi) ss += acc * acc;
        }
    }
    if (CG) {
        const double bs = block_sum<NTA>(ss, red);
        if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
        if (elect_last_block(&st[ch].cnt_init, nblk)) {
            const double tot = sum_partials<NTA>(part + static_cast<size_t>(ch) * nblk, nblk, 1, red);
            if (threadIdx.x == 0 && G.dred) {  // distributed: publish the local sum only
                G.dred[G.N + 3 * ch + 1] = tot;
                st[ch].cnt_init = 0;
            } else if (threadIdx.x == 0) {
                CgState& S = st[ch];
                S.rs = tot;
                S.rhs_norm = sqrt(tot);
                S.pp = S.pAp = S.alpha = S.beta = S.zz = S.qq = 0.0;
                S.cg_tol = cg_tol;
                S.t = 0;
                S.iters = 0;
                S.max_iters = max_iters;
                S.done = (S.rhs_norm == 0.0) ? 1 : (max_iters <= 0 ? 3 : 0);
                S.cnt_q = S.cnt_a = S.cnt_u = 0;
                S.cnt_init = 0;
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// Guided filter (pansharpen.cpp:274-312), clamped windows (ops.cpp:104-128).
// input = L(z0) when in_is_z0 (pansharpen.cpp:396-398), else the input plane itself.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTA) k_guided(int H, int W, int rw, double eps, int cps, const double* __restrict__ in,
                                                int in_is_z0, const double* __restrict__ guide,
                                                double* __restrict__ aout, double* __restrict__ cout,
                                                double* __restrict__ vout) {
    extern __shared__ double sm[];
    const int ch = blockIdx.y;
    const size_t P = static_cast<size_t>(H) * W;
    const double* ic = in + ch * P;
    guide += static_cast<size_t>(ch / cps) * P;
    const int ntx = (W + TA - 1) / TA;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const int r0 = by * TA, c0 = bx * TA;
    const int hz = 2 * rw + (in_is_z0 ? 1 : 0), hin = 2 * rw, hac = rw;
    const int SZ = TA + 2 * hz, SN = TA + 2 * hin, SA = TA + 2 * hac;
    double* sz = sm;
    double* sin_ = in_is_z0 ? sz + ((SZ * SZ + 1) & ~1) : sz;
    double* sI = sin_ + ((SN * SN + 1) & ~1);
    double* sa = sI + ((SN * SN + 1) & ~1);
    double* sc = sa + ((SA * SA + 1) & ~1);
    for (int e = threadIdx.x; e < SZ * SZ; e += NTA) {
        const int y = e / SZ, x = e - y * SZ;
        sz[e] = __ldg(ic + static_cast<size_t>(wrapi(r0 - hz + y, H)) * W + wrapi(c0 - hz + x, W));
    }
    for (int e = threadIdx.x; e < SN * SN; e += NTA) {
        const int y = e / SN, x = e - y * SN;
        sI[e] = __ldg(guide + static_cast<size_t>(wrapi(r0 - hin + y, H)) * W + wrapi(c0 - hin + x, W));
    }
    __syncthreads();
    if (in_is_z0) {
        for (int e = threadIdx.x; e < SN * SN; e += NTA) {
            const int y = e / SN + 1, x = e % SN + 1;
            sin_[e] = 4.0 * sz[y * SZ + x] - sz[(y - 1) * SZ + x] - sz[(y + 1) * SZ + x] - sz[y * SZ + x - 1] -
                      sz[y * SZ + x + 1];
        }
        __syncthreads();
    }
    // a, c on R + rw (only in-image positions are ever consumed)
    for (int e = threadIdx.x; e < SA * SA; e += NTA) {
        const int y = e / SA, x = e - y * SA;
        const int gr = r0 - hac + y, gc = c0 - hac + x;
        double a = 0.0, cc = 0.0;
        if (gr >= 0 && gr < H && gc >= 0 && gc < W) {
            const int ra = max(0, gr - rw), rb = min(H - 1, gr + rw);
            const int ca = max(0, gc - rw), cb = min(W - 1, gc + rw);
            double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
            for (int yy = ra; yy <= rb; ++yy)
                for (int xx = ca; xx <= cb; ++xx) {
                    const int li = (yy - r0 + hin) * SN + (xx - c0 + hin);
                    const double gv = sI[li], iv = sin_[li];
                    s1 += gv;
                    s2 += iv;
                    s3 += gv * iv;
                    s4 += gv * gv;
                }
            const double cnt = static_cast<double>((rb - ra + 1) * (cb - ca + 1));
            const double mu = s1 / cnt, im = s2 / cnt, cgi = s3 / cnt, cgg = s4 / cnt;
            const double var = cgg - mu * mu;
            const double cov = cgi - mu * im;
            a = cov / (var + eps);
            cc = im - a * mu;
        }
        sa[e] = a;
        sc[e] = cc;
    }
    __syncthreads();
    const int tx = threadIdx.x & 31;
    for (int ty = threadIdx.x >> 5; ty < TA; ty += NTA / 32) {
        const int R = r0 + ty, Cc = c0 + tx;
        if (R >= H || Cc >= W) continue;
        const int ra = max(0, R - rw), rb = min(H - 1, R + rw);
        const int ca = max(0, Cc - rw), cb = min(W - 1, Cc + rw);
        double s1 = 0.0, s2 = 0.0;
        for (int yy = ra; yy <= rb; ++yy)
            for (int xx = ca; xx <= cb; ++xx) {
                const int li = (yy - r0 + hac) * SA + (xx - c0 + hac);
                s1 += sa[li];
                s2 += sc[li];
            }
        const double cnt = static_cast<double>((rb - ra + 1) * (cb - ca + 1));
        const double gv = sI[(ty + hin) * SN + tx + hin];
        const size_t gi = ch * P + static_cast<size_t>(R) * W + Cc;
        vout[gi] = (s1 / cnt) * gv + s2 / cnt;
        if (aout) aout[gi] = sa[(ty + hac) * SA + tx + hac];
        if (cout) cout[gi] = sc[(ty + hac) * SA + tx + hac];
    }
}

// ------------------------------------------------------------------------------------------
// Guided filter, tiled and separable (pansharpen.cpp:274-312, box_mean = ops.cpp:104-128 with
// clamped windows). One CTA per (32 x 32 output tile, channel); the radius is a template
// parameter, so every staged region has compile-time extents and all passes are flattened
// element loops over the 256 threads (no partially filled warps, constant divisors). Box sums
// are separable: row sums over the clamped column range, then column sums over the clamped row
// range (out-of-image taps contribute exact zeros; the count is the clamped window's size). The
// input is L(z0) from a z0 tile with a one-pixel larger halo (Z0), else the plane itself.
// Requires H, W >= tile + halo (wrap1).
// ------------------------------------------------------------------------------------------
constexpr int GTW = 32, GTH = 32, GNT = 256;
__device__ __forceinline__ int wrap1(int a, int m) {  // valid for -m <= a < 2m
    a += a < 0 ? m : 0;
    return a >= m ? a - m : a;
}
template <int RW, bool Z0>
struct GfLay {
    static constexpr int HZ = 2 * RW + (Z0 ? 1 : 0), HIN = 2 * RW, HAC = RW;
    static constexpr int NR = GTH + 2 * HIN, NC = GTW + 2 * HIN, AR = GTH + 2 * HAC, AC = GTW + 2 * HAC;
    static constexpr int ZR = GTH + 2 * HZ, ZC = GTW + 2 * HZ;
    static constexpr int HS = (4 * NR * AC > ZR * ZC) ? 4 * NR * AC : ZR * ZC;  // row sums | z0 tile
    static constexpr size_t bytes = (2 * static_cast<size_t>(NR) * NC + 2 * static_cast<size_t>(AR) * AC + HS) *
                                    sizeof(double);
};
template <int RW, bool Z0>
__global__ void __launch_bounds__(GNT) k_guided2(int H, int W, double eps, int cps, const double* __restrict__ in,
                                                 const double* __restrict__ guide, double* __restrict__ aout,
                                                 double* __restrict__ cout, double* __restrict__ vout) {
    using L = GfLay<RW, Z0>;
    constexpr int NR = L::NR, NC = L::NC, AR = L::AR, AC = L::AC, ZR = L::ZR, ZC = L::ZC;
    constexpr int HIN = L::HIN, HAC = L::HAC, HZ = L::HZ;
    extern __shared__ double sm[];
    const int ch = blockIdx.y;
    const size_t P = static_cast<size_t>(H) * W;
    const int ntx = (W + GTW - 1) / GTW;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const int r0 = by * GTH, c0 = bx * GTW;
    double* sI = sm;                 // guide, NR x NC
    double* sIn = sI + NR * NC;      // filter input, NR x NC
    double* sa = sIn + NR * NC;      // a, AR x AC
    double* sc = sa + AR * AC;       // c
    double* rs = sc + AR * AC;       // 4 row-sum planes NR x AC (then 2 planes AR x GTW)
    double* sZ = rs;                 // z0 tile (dead before the row sums are formed)
    const int t = threadIdx.x;
    const double* gs = guide + static_cast<size_t>(ch / cps) * P;
    const double* ic = in + static_cast<size_t>(ch) * P;
    for (int e = t; e < NR * NC; e += GNT) {
        const int y = e / NC, x = e - y * NC;
        sI[e] = __ldg(gs + static_cast<size_t>(wrap1(r0 - HIN + y, H)) * W + wrap1(c0 - HIN + x, W));
    }
    if (Z0) {
        for (int e = t; e < ZR * ZC; e += GNT) {
            const int y = e / ZC, x = e - y * ZC;
            sZ[e] = __ldg(ic + static_cast<size_t>(wrap1(r0 - HZ + y, H)) * W + wrap1(c0 - HZ + x, W));
        }
        __syncthreads();
        for (int e = t; e < NR * NC; e += GNT) {
            const int y = e / NC, x = e - y * NC;
            const double* z = sZ + (y + 1) * ZC + x + 1;  // ops.cpp:70-78 order
            sIn[e] = 4.0 * z[0] - z[-ZC] - z[ZC] - z[-1] - z[1];
        }
    } else {
        for (int e = t; e < NR * NC; e += GNT) {
            const int y = e / NC, x = e - y * NC;
            sIn[e] = __ldg(ic + static_cast<size_t>(wrap1(r0 - HIN + y, H)) * W + wrap1(c0 - HIN + x, W));
        }
    }
    __syncthreads();
    // guided_coeffs (pansharpen.cpp:274-301): row sums of I, I^2, in, I in over the clamped columns
    // of A-region column x (staging columns x + RW + k, k in [-RW, RW]; out-of-image taps add 0)
    for (int e = t; e < NR * AC; e += GNT) {
        const int y = e / AC, x = e - y * AC;
        const int gc = c0 - HAC + x;
        double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
        for (int k = -RW; k <= RW; ++k) {
            const bool ok = gc + k >= 0 && gc + k < W;
            const double gv = ok ? sI[y * NC + x + RW + k] : 0.0;
            const double iv = ok ? sIn[y * NC + x + RW + k] : 0.0;
            s1 += gv;
            s2 += iv;
            s3 += gv * iv;
            s4 += gv * gv;
        }
        rs[e] = s1;
        rs[NR * AC + e] = s2;
        rs[2 * NR * AC + e] = s3;
        rs[3 * NR * AC + e] = s4;
    }
    __syncthreads();
    for (int e = t; e < AR * AC; e += GNT) {
        const int y = e / AC, x = e - y * AC;
        const int gr = r0 - HAC + y, gc = c0 - HAC + x;
        double a = 0.0, cc = 0.0;
        if (gr >= 0 && gr < H && gc >= 0 && gc < W) {
            double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
            for (int k = -RW; k <= RW; ++k) {
                if (gr + k < 0 || gr + k >= H) continue;
                const int o = (y + RW + k) * AC + x;
                s1 += rs[o];
                s2 += rs[NR * AC + o];
                s3 += rs[2 * NR * AC + o];
                s4 += rs[3 * NR * AC + o];
            }
            const int nr = min(H - 1, gr + RW) - max(0, gr - RW) + 1, nc = min(W - 1, gc + RW) - max(0, gc - RW) + 1;
            const double inv = 1.0 / static_cast<double>(nr * nc);  // one division per window
            const double mu = s1 * inv, im = s2 * inv, cgi = s3 * inv, cgg = s4 * inv;
            const double var = cgg - mu * mu;  // pansharpen.cpp:293-298
            const double cov = cgi - mu * im;
            a = cov / (var + eps);
            cc = im - a * mu;
        }
        sa[e] = a;
        sc[e] = cc;
    }
    __syncthreads();
    // guided_output (pansharpen.cpp:304-312): row sums of a, c over the clamped columns
    double* ra = rs;
    double* rc = rs + AR * GTW;
    for (int e = t; e < AR * GTW; e += GNT) {
        const int y = e / GTW, x = e - y * GTW;
        const int gc = c0 + x;
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = -RW; k <= RW; ++k) {
            const bool ok = gc + k >= 0 && gc + k < W;
            s1 += ok ? sa[y * AC + x + RW + k] : 0.0;
            s2 += ok ? sc[y * AC + x + RW + k] : 0.0;
        }
        ra[e] = s1;
        rc[e] = s2;
    }
    __syncthreads();
    for (int e = t; e < GTH * GTW; e += GNT) {
        const int y = e / GTW, x = e - y * GTW;
        const int R = r0 + y, Cc = c0 + x;
        if (R >= H || Cc >= W) continue;
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = -RW; k <= RW; ++k) {
            if (R + k < 0 || R + k >= H) continue;
            s1 += ra[(y + RW + k) * GTW + x];
            s2 += rc[(y + RW + k) * GTW + x];
        }
        const int nr = min(H - 1, R + RW) - max(0, R - RW) + 1, nc = min(W - 1, Cc + RW) - max(0, Cc - RW) + 1;
        const double inv = 1.0 / static_cast<double>(nr * nc);
        const double gv = sI[(y + HIN) * NC + x + HIN];
        const size_t gi = static_cast<size_t>(ch) * P + static_cast<size_t>(R) * W + Cc;
        vout[gi] = (s1 * inv) * gv + s2 * inv;
        if (aout) aout[gi] = sa[(y + HAC) * AC + x + HAC];
        if (cout) cout[gi] = sc[(y + HAC) * AC + x + HAC];
    }
}

// ------------------------------------------------------------------------------------------
// Guided filter by row streaming (radius 1; pansharpen.cpp:274-312 with box_mean's clamped
// windows, ops.cpp:104-128): the K_L scheme. One warp per CTA owns a band of 56 output columns
// (lane = column pair, 4 halo columns each side, periodic like the loads) and walks a strip of
// rows; per input row Y it forms, all in registers, in = L(z0) at Y-1 (periodic, ops.cpp:70-78
// order), the clamped row sums of I, in, I in, I^2 at Y-1, the window means and a, c at Y-2,
// the clamped row sums of a, c at Y-2, and v = mean(a) I + mean(c) at Y-3. Out-of-image columns
// and rows contribute exact zeros; counts are the clamped window sizes. z0 and I rows stream by
// cp.async (ring of GS_NB steps); the scene's I rows are shared by its channels through L2
// (channel-fastest CTA order).
// ------------------------------------------------------------------------------------------
constexpr int GS_BAND = 56, GS_HALO = 4, GS_NB = 4;
template <bool Z0>
__global__ void __launch_bounds__(32, 12) k_guided3(int H, int W, double eps, int N, int cps, int kstrips, int R,
                                                    const double* __restrict__ in, const double* __restrict__ guide,
                                                    double* __restrict__ vout) {
    using V = double2;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x;
    const int ch = blockIdx.x % N, item = blockIdx.x / N;
    const int band = item / kstrips, strip = item - band * kstrips;
    const size_t P = static_cast<size_t>(H) * W;
    const int c0 = band * GS_BAND, r0 = strip * R, r1 = min(H, r0 + R);
    if (r0 >= H) return;
    const int ox = c0 - GS_HALO + 2 * lane;                 // unwrapped column of .x
    const int X = fast::wrap_once(ox, W);
    const double* zc = in + static_cast<size_t>(ch) * P + X;
    const double* I = guide + static_cast<size_t>(ch / cps) * P + X;
    double* vc = vout + static_cast<size_t>(ch) * P + X;
    const bool writer = lane >= GS_HALO / 2 && lane < (GS_HALO + GS_BAND) / 2 && ox < W;
    // column validity (clamped windows) of the pair and of its horizontal neighbours
    const double vxl = ox - 1 >= 0 && ox - 1 < W ? 1.0 : 0.0, vx0 = ox >= 0 && ox < W ? 1.0 : 0.0;
    const double vx1 = ox + 1 >= 0 && ox + 1 < W ? 1.0 : 0.0, vxr = ox + 2 >= 0 && ox + 2 < W ? 1.0 : 0.0;
    // clamped column counts of the pair's windows
    const int nc0 = min(W - 1, ox + 1) - max(0, ox - 1) + 1, nc1 = min(W - 1, ox + 2) - max(0, ox) + 1;
    // 1 / window size for interior rows (3 rows), per lane; border rows take the general division
    const double i30 = 1.0 / static_cast<double>(3 * nc0), i31 = 1.0 / static_cast<double>(3 * nc1);
    __shared__ V ring[GS_NB][2][32];  // z(Y), I(Y-1)
    auto back = [&](int r, int k) { int q = r - k; while (q < 0) q += H; return q; };
    auto adv = [&](int o) { return o + W == static_cast<int>(P) ? 0 : o + W; };
    const int y0 = r0 - 3;                                   // unwrapped input row of step 0
    const int yA = back(y0 + H, 0) % H;
    int io0 = yA * W, io1 = back(yA, 1) * W, o3 = back(yA, 3) * W;
    const int steps = (r1 - r0) + 6;
    auto issue = [&](int slot) {
        fast::cp_async_pair(&ring[slot][0][lane], zc + io0);
        fast::cp_async_pair(&ring[slot][1][lane], I + io1);
        io0 = adv(io0);
        io1 = adv(io1);
    };
#pragma unroll
    for (int j = 0; j < GS_NB - 1; ++j) {
        if (j < steps) issue(j);
        fast::cp_async_commit();
    }
    V zm1 = {0, 0}, zm2 = {0, 0};                 // z(Y-1), z(Y-2)
    V Im2 = {0, 0}, Im3 = {0, 0};                 // I(Y-2), I(Y-3)
    V S1a = {0, 0}, S1b = {0, 0}, S2a = {0, 0}, S2b = {0, 0}, S3a = {0, 0}, S3b = {0, 0}, S4a = {0, 0}, S4b = {0, 0};
    V Aa = {0, 0}, Ab = {0, 0}, Ca = {0, 0}, Cb = {0, 0};  // row sums of a, c at Y-4, Y-3
#pragma unroll 2
    for (int st = 0; st < steps; ++st) {
        if (st + GS_NB - 1 < steps) issue((st + GS_NB - 1) % GS_NB);
        fast::cp_async_commit();
        fast::cp_async_wait<GS_NB - 1>();
        const int slot = st % GS_NB;
        const V z0 = ring[slot][0][lane], Im1 = ring[slot][1][lane];
        const int y1 = y0 + st - 1, y2 = y0 + st - 2, y3 = y0 + st - 3;  // unwrapped rows of the stages
        // in(Y-1)
        V in1;
        if (Z0) {
            const double zL = __shfl_up_sync(FULL, zm1.y, 1), zR = __shfl_down_sync(FULL, zm1.x, 1);
            in1.x = 4.0 * zm1.x - zm2.x - z0.x - zL - zm1.y;
            in1.y = 4.0 * zm1.y - zm2.y - z0.y - zm1.x - zR;
        } else {
            in1 = zm1;
        }
        // clamped row sums at Y-1 (rows outside the image count as zero)
        const double rv1 = y1 >= 0 && y1 < H ? 1.0 : 0.0;
        V s1n, s2n, s3n, s4n;
        {
            const double gx = Im1.x * vx0, gy = Im1.y * vx1, ix = in1.x * vx0, iy = in1.y * vx1;
            const double gL = __shfl_up_sync(FULL, Im1.y, 1) * vxl, gR = __shfl_down_sync(FULL, Im1.x, 1) * vxr;
            const double iL = __shfl_up_sync(FULL, in1.y, 1) * vxl, iR = __shfl_down_sync(FULL, in1.x, 1) * vxr;
            s1n = make_double2((gL + gx + gy) * rv1, (gx + gy + gR) * rv1);
            s2n = make_double2((iL + ix + iy) * rv1, (ix + iy + iR) * rv1);
            s3n = make_double2((gL * iL + gx * ix + gy * iy) * rv1, (gx * ix + gy * iy + gR * iR) * rv1);
            s4n = make_double2((gL * gL + gx * gx + gy * gy) * rv1, (gx * gx + gy * gy + gR * gR) * rv1);
        }
        // window means and a, c at Y-2 (pansharpen.cpp:285-301); outside the image a = c = 0
        V a2, c2;
        {
            const int nr = min(H - 1, y2 + 1) - max(0, y2 - 1) + 1;
            const bool rin = y2 >= 0 && y2 < H;
            const double inv0 = nr == 3 ? i30 : 1.0 / static_cast<double>(nr * nc0);
            const double inv1 = nr == 3 ? i31 : 1.0 / static_cast<double>(nr * nc1);
            {
                const double mu = (S1a.x + S1b.x + s1n.x) * inv0, im = (S2a.x + S2b.x + s2n.x) * inv0;
                const double cgi = (S3a.x + S3b.x + s3n.x) * inv0, cgg = (S4a.x + S4b.x + s4n.x) * inv0;
                const double var = cgg - mu * mu, cov = cgi - mu * im;
                const double a = cov / (var + eps);
                const bool ok = rin && vx0 != 0.0;
                a2.x = ok ? a : 0.0;
                c2.x = ok ? im - a * mu : 0.0;
            }
            {
                const double mu = (S1a.y + S1b.y + s1n.y) * inv1, im = (S2a.y + S2b.y + s2n.y) * inv1;
                const double cgi = (S3a.y + S3b.y + s3n.y) * inv1, cgg = (S4a.y + S4b.y + s4n.y) * inv1;
                const double var = cgg - mu * mu, cov = cgi - mu * im;
                const double a = cov / (var + eps);
                const bool ok = rin && vx1 != 0.0;
                a2.y = ok ? a : 0.0;
                c2.y = ok ? im - a * mu : 0.0;
            }
        }
        // clamped row sums of a, c at Y-2 (out-of-image a, c are already zero)
        V An, Cn;
        {
            const double aL = __shfl_up_sync(FULL, a2.y, 1), aR = __shfl_down_sync(FULL, a2.x, 1);
            const double cL = __shfl_up_sync(FULL, c2.y, 1), cR = __shfl_down_sync(FULL, c2.x, 1);
            An = make_double2(aL + a2.x + a2.y, a2.x + a2.y + aR);
            Cn = make_double2(cL + c2.x + c2.y, c2.x + c2.y + cR);
        }
        // v at Y-3 (guided_output, pansharpen.cpp:304-312)
        if (st >= 6 && writer) {
            const int nr = min(H - 1, y3 + 1) - max(0, y3 - 1) + 1;
            const double inv0 = nr == 3 ? i30 : 1.0 / static_cast<double>(nr * nc0);
            const double inv1 = nr == 3 ? i31 : 1.0 / static_cast<double>(nr * nc1);
            const double ax = (Aa.x + Ab.x + An.x) * inv0, cx = (Ca.x + Cb.x + Cn.x) * inv0;
            const double ay = (Aa.y + Ab.y + An.y) * inv1, cy = (Ca.y + Cb.y + Cn.y) * inv1;
            *reinterpret_cast<V*>(vc + o3) = make_double2(ax * Im3.x + cx, ay * Im3.y + cy);
        }
        o3 = adv(o3);
        zm2 = zm1; zm1 = z0;
        Im3 = Im2; Im2 = Im1;
        S1a = S1b; S1b = s1n; S2a = S2b; S2b = s2n; S3a = S3b; S3b = s3n; S4a = S4b; S4b = s4n;
        Aa = Ab; Ab = An; Ca = Cb; Cb = Cn;
    }
}

// ------------------------------------------------------------------------------------------
// Alias-group direct solve (pansharpen.cpp:337-363): one thread per LR frequency (kl, ll).
// The c^2 x c^2 system A = diag(D) + u u^H / c^2 (D = lambda |L^|^2, u = conj(b^)) is solved in
// closed form, eliminating through the coordinate j with the smallest D (the one that can be
// ~0 near DC), which keeps the solve stable where Sherman-Morrison would cancel. The
// eigenvalue-ratio test of :353-357 uses the exact extremal eigenvalues of the rank-one
// update (secular equation) whenever the cheap interlacing bound is inconclusive.
// ------------------------------------------------------------------------------------------
struct cplx {
    double x, y;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ cplx cconj(cplx a) { return {a.x, -a.y}; }
__device__ __forceinline__ double cnorm(cplx a) { return a.x * a.x + a.y * a.y; }

__device__ __forceinline__ cplx half_lookup(const double2* X, int R, int Cc, int H, int W) {
    const int WH = W / 2 + 1;
    if (Cc < WH) {
        const double2 v = X[static_cast<size_t>(R) * WH + Cc];
        return {v.x, v.y};
    }
    const double2 v = X[static_cast<size_t>((H - R) % H) * WH + (W - Cc)];
    return {v.x, -v.y};
}

// smallest root of c2 + sum |u_g|^2/(D_g - x) in (lo, hi), by bisection
__device__ __forceinline__ double secular_root(int m, const double* D, const double* u2, double c2, double lo,
                                            double hi) {
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (!(mid > lo && mid < hi)) break;
        double f = c2;
        for (int g = 0; g < m; ++g)
            if (u2[g] > 0.0) f += u2[g] / (D[g] - mid);
        if (f > 0.0) hi = mid;
        else lo = mid;
    }
    return 0.5 * (lo + hi);
}

__device__ __forceinline__ bool alias_condition_ok(int m, const double* D, const double* u2, double c2) {
    double dmin_all = INFINITY, dmax_all = -INFINITY;
    double dmin_u = INFINITY, d2_u = INFINITY, dmax_u = -INFINITY, unorm = 0.0;
    int mult_min = 0;
    double min_defl = INFINITY, max_defl = -INFINITY;
    for (int g = 0; g < m; ++g) {
        dmin_all = fmin(dmin_all, D[g]);
        dmax_all = fmax(dmax_all, D[g]);
        if (u2[g] > 0.0) {
            unorm += u2[g];
            dmax_u = fmax(dmax_u, D[g]);
            if (D[g] < dmin_u) { d2_u = dmin_u; dmin_u = D[g]; mult_min = 1; }
            else if (D[g] == dmin_u) { ++mult_min; }
            else if (D[g] < d2_u) d2_u = D[g];
        } else {
            min_defl = fmin(min_defl, D[g]);
            max_defl = fmax(max_defl, D[g]);
        }
    }
    const double ub_max = dmax_all + unorm / c2;
    if (dmin_all > 0.0 && ub_max <= 1e14 * dmin_all) return true;
    double ev_min = min_defl, ev_max = max_defl;
    if (unorm > 0.0) {
        double r;
        if (mult_min >= 2) r = dmin_u;
        else if (!(d2_u < INFINITY)) r = dmin_u + unorm / c2;
        else r = secular_root(m, D, u2, c2, dmin_u, d2_u);
        ev_min = fmin(ev_min, r);
        const double top = secular_root(m, D, u2, c2, dmax_u, dmax_u + unorm / c2 * (1.0 + 1e-12) + 1e-300);
        ev_max = fmax(ev_max, top);
    }
    return (ev_min > 0.0) && !(ev_max > 1e14 * ev_min);
}

// cos(2 pi R / H) for R < H, then cos(2 pi C / W) for C < W: the Laplacian symbol's factors,
// evaluated once per solve instead of 2 c^2 times per alias group (same expression, same bits)
__global__ void k_cos_tables(int H, int W, double* __restrict__ tab) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H + W; i += gridDim.x * blockDim.x)
        tab[i] = i < H ? cos(2.0 * M_PI * i / H) : cos(2.0 * M_PI * (i - H) / W);
}

// ------------------------------------------------------------------------------------------
// Alias-group solve, one 16-lane group per alias group (factor c <= 4, m = c^2 <= 16 members):
// lane g of the group owns member g (its D, u = conj(b^), rhs live in registers; nothing is
// indexed dynamically, so there is no local-memory frame). The group loops over the channels of
// its scene: b^ and the Laplacian symbol are loaded once for all of them. Sums over the members
// (sigma's numerator/denominator, u^H z) are xor-butterflies, identical on every lane.
// Same closed form as k_alias; the rare inconclusive interlacing bound goes to the exact
// secular-equation check, evaluated by the whole group (alias_condition_grp).
// ------------------------------------------------------------------------------------------
constexpr int AG = 16;          // lanes per alias group
constexpr int AG_NT = 128;      // threads per CTA (8 groups)
// group reductions over the 16 lanes of an alias group (gm = the group's lane mask)
__device__ __forceinline__ double grp_sum(unsigned gm, double v) {
#pragma unroll
    for (int o = 1; o < AG; o <<= 1) v += __shfl_xor_sync(gm, v, o, AG);
    return v;
}
__device__ __forceinline__ double grp_max(unsigned gm, double v) {
#pragma unroll
    for (int o = 1; o < AG; o <<= 1) v = fmax(v, __shfl_xor_sync(gm, v, o, AG));
    return v;
}
__device__ __forceinline__ double grp_min(unsigned gm, double v) {
#pragma unroll
    for (int o = 1; o < AG; o <<= 1) v = fmin(v, __shfl_xor_sync(gm, v, o, AG));
    return v;
}
// smallest root of c2 + sum_g |u_g|^2 / (D_g - x) in (lo, hi) by bisection; each lane holds one
// member's term, the sum is a group butterfly (identical on all lanes, so every lane takes the
// same branch)
__device__ double secular_root_grp(unsigned gm, bool uu, double D, double u2, double c2, double lo, double hi) {
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (!(mid > lo && mid < hi)) break;
        const double f = c2 + grp_sum(gm, uu ? u2 / (D - mid) : 0.0);
        if (f > 0.0) hi = mid;
        else lo = mid;
    }
    return 0.5 * (lo + hi);
}
// pansharpen.cpp:353-357 for a group whose cheap interlacing bound was inconclusive: the exact
// extremal eigenvalues of diag(D) + u u^H / c^2 (deflated members and the secular equation),
// as alias_condition_ok, with the member loops as group reductions
__device__ bool alias_condition_grp(unsigned gm, bool mem, double D, double u2, double c2, double unorm) {
    const bool uu = mem && u2 > 0.0;
    const double dmin_u = grp_min(gm, uu ? D : INFINITY);
    const double mult_min = grp_sum(gm, (uu && D == dmin_u) ? 1.0 : 0.0);
    const double d2_u = grp_min(gm, (uu && D > dmin_u) ? D : INFINITY);
    const double dmax_u = grp_max(gm, uu ? D : -INFINITY);
    double ev_min = grp_min(gm, (mem && !uu) ? D : INFINITY);
    double ev_max = grp_max(gm, (mem && !uu) ? D : -INFINITY);
    if (unorm > 0.0) {
        double r;
        if (mult_min >= 2.0) r = dmin_u;
        else if (!(d2_u < INFINITY)) r = dmin_u + unorm / c2;
        else r = secular_root_grp(gm, uu, D, u2, c2, dmin_u, d2_u);
        ev_min = fmin(ev_min, r);
        const double top = secular_root_grp(gm, uu, D, u2, c2, dmax_u, dmax_u + unorm / c2 * (1.0 + 1e-12) + 1e-300);
        ev_max = fmax(ev_max, top);
    }
    return (ev_min > 0.0) && !(ev_max > 1e14 * ev_min);
}
// 1/x to within an ulp: MUFU seed + two Newton steps, inline (no IEEE division subroutine call)
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__global__ void __launch_bounds__(AG_NT) k_alias16(int H, int W, int h, int w, int c, int N, int cps, int identity,
                                                   double lambda, const double2* __restrict__ Bh,
                                                   const double2* __restrict__ Xh, const double2* __restrict__ Vh,
                                                   double2* __restrict__ Zh, const double* __restrict__ cosHW,
                                                   int* __restrict__ flag) {
    const int g = threadIdx.x & (AG - 1);
    const unsigned gm = 0xffffu << (threadIdx.x & AG);  // this group's half of the warp
    const int gid = static_cast<int>(blockIdx.x) * (AG_NT / AG) + static_cast<int>(threadIdx.x / AG);  // h w < 2^31
    const bool live = gid < h * w;   // uniform over the group
    const int kl = live ? gid / w : 0, ll = live ? gid - kl * w : 0;
    const int m = c * c;
    const bool mem = live && g < m;
    const double c2 = static_cast<double>(m);
    const int scene = blockIdx.y;
    const size_t HS = static_cast<size_t>(H) * (W / 2 + 1), LS = static_cast<size_t>(h) * (w / 2 + 1);
    const int WH = W / 2 + 1;
    const int a = mem ? g / c : 0, b = mem ? g - (g / c) * c : 0;
    const int R = kl + a * h, Cc = ll + b * w;
    // half-spectrum index of member (R, Cc) and whether it is read through Hermitian symmetry
    const bool mirror = Cc >= WH;
    const size_t hidx = mirror ? static_cast<size_t>((H - R) % H) * WH + (W - Cc) : static_cast<size_t>(R) * WH + Cc;
    double D = INFINITY, lh = 0.0;
    cplx u = {0.0, 0.0};
    if (mem) {
        const double2 bv = __ldg(Bh + static_cast<size_t>(scene) * HS + hidx);
        u = {bv.x, mirror ? bv.y : -bv.y};  // conj(b^)
        lh = identity ? 1.0 : 4.0 - 2.0 * __ldg(cosHW + R) - 2.0 * __ldg(cosHW + H + Cc);  // pansharpen.cpp:53-70
        D = lambda * (lh * lh);
    }
    const double u2 = mem ? cnorm(u) : 0.0;
    const double rD = mem ? rcp_nr(D) : 0.0;  // reciprocals: no division subroutine calls
    // jmin = first member with the smallest D (the sequential strict-< scan of k_alias)
    double dmin = D;
    int jmin = mem ? g : AG;
#pragma unroll
    for (int o = 1; o < AG; o <<= 1) {
        const double od = __shfl_xor_sync(gm, dmin, o, AG);
        const int oj = __shfl_xor_sync(gm, jmin, o, AG);
        if (od < dmin || (od == dmin && oj < jmin)) { dmin = od; jmin = oj; }
    }
    const bool isj = mem && g == jmin;
    // condition test (pansharpen.cpp:353-357): cheap interlacing bound, exact check if inconclusive
    const double dmax_all = grp_max(gm, mem ? D : -INFINITY);
    const double unorm = grp_sum(gm, u2 > 0.0 ? u2 : 0.0);
    bool ok = dmin > 0.0 && dmax_all + unorm / c2 <= 1e14 * dmin;
    if (live && !ok) ok = alias_condition_grp(gm, mem, D, u2, c2, unorm);  // group-uniform branch
    const double Dj = dmin;
    const double u2j = __shfl_sync(gm, u2, jmin & (AG - 1), AG);
    const int ch1 = min(N, (scene + 1) * cps);
    for (int ch = scene * cps; ch < ch1; ++ch) {
        if (live && !ok && g == 0) atomicExch(flag + ch, 1);
        cplx rhs = {0.0, 0.0};
        if (live) {
            const double2 xv = __ldg(Xh + ch * LS + (ll < w / 2 + 1 ? static_cast<size_t>(kl) * (w / 2 + 1) + ll
                                                               : static_cast<size_t>((h - kl) % h) * (w / 2 + 1) + (w - ll)));
            const cplx xg = {xv.x, ll < w / 2 + 1 ? xv.y : -xv.y};
            if (mem) {
                const double2 vv2 = __ldg(Vh + ch * HS + hidx);
                const cplx vv = {vv2.x, mirror ? -vv2.y : vv2.y};
                const cplx ux = cmul(u, xg);
                rhs = {ux.x + lambda * lh * vv.x, ux.y + lambda * lh * vv.y};
            }
        }
        // sigma = u^H z / c^2 from the D_j-scaled secular identity (exact for D_j = 0)
        const cplx t = cmul(cconj(u), rhs);
        const double ratio = isj ? 1.0 : (mem ? Dj * rD : 0.0);
        const double num_x = grp_sum(gm, t.x * ratio), num_y = grp_sum(gm, t.y * ratio);
        const double den = c2 * Dj + grp_sum(gm, mem ? u2 * ratio : 0.0);
        const double rden = rcp_nr(den);
        const cplx sigma = {num_x * rden, num_y * rden};
        const cplx us = cmul(u, sigma);
        cplx zg = {0.0, 0.0};
        if (mem && !isj) zg = {(rhs.x - us.x) * rD, (rhs.y - us.y) * rD};
        const cplx tz = cmul(cconj(u), zg);
        const double zs_x = grp_sum(gm, tz.x), zs_y = grp_sum(gm, tz.y);
        if (isj) {
            if (u2j < c2 * Dj) {
                zg = {(rhs.x - us.x) * rD, (rhs.y - us.y) * rD};  // rD = 1 / Dj on this lane
            } else {
                const cplx s = {c2 * sigma.x - zs_x, c2 * sigma.y - zs_y};
                const double ru = rcp_nr(u2j);
                zg = {(s.x * u.x - s.y * u.y) * ru, (s.y * u.x + s.x * u.y) * ru};  // s / conj(u) = s u / |u|^2
            }
        }
        if (mem && !mirror) Zh[ch * HS + hidx] = make_double2(zg.x, zg.y);
    }
}

template <int CM>
__global__ void __launch_bounds__(128) k_alias(int H, int W, int h, int w, int c, int cps, int identity, double lambda,
                                               const double2* __restrict__ Bh, const double2* __restrict__ Xh,
                                               const double2* __restrict__ Vh, double2* __restrict__ Zh,
                                               const double* __restrict__ cosHW, int* __restrict__ flag) {
    constexpr int M = CM * CM;
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= h * w) return;
    const int ch = blockIdx.y;
    const int kl = gid / w, ll = gid - kl * w;
    const int m = c * c;
    const double c2 = static_cast<double>(m);
    const size_t HS = static_cast<size_t>(H) * (W / 2 + 1), LS = static_cast<size_t>(h) * (w / 2 + 1);
    const double2* V = Vh + ch * HS;
    double2* Z = Zh + ch * HS;
    Bh += static_cast<size_t>(ch / cps) * HS;
    const cplx xg = half_lookup(Xh + ch * LS, kl, ll, h, w);
    double D[M], u2[M];
    cplx u[M], rhs[M];
    int jmin = 0;
    for (int a = 0; a < c; ++a)
        for (int b = 0; b < c; ++b) {
            const int g = a * c + b;
            const int R = kl + a * h, Cc = ll + b * w;
            const cplx bv = half_lookup(Bh, R, Cc, H, W);
            const cplx vv = half_lookup(V, R, Cc, H, W);
            const double lh = identity ? 1.0 : 4.0 - 2.0 * __ldg(cosHW + R) - 2.0 * __ldg(cosHW + H + Cc);  // :53-70
            D[g] = lambda * (lh * lh);
            u[g] = cconj(bv);
            u2[g] = cnorm(u[g]);
            const cplx ux = cmul(u[g], xg);
            rhs[g] = {ux.x + lambda * lh * vv.x, ux.y + lambda * lh * vv.y};
            if (D[g] < D[jmin]) jmin = g;
        }
    if (!alias_condition_ok(m, D, u2, c2)) atomicExch(flag + ch, 1);
    // sigma = u^H z / c^2 from the D_j-scaled secular identity (exact for D_j = 0)
    const double Dj = D[jmin];
    cplx num = cmul(cconj(u[jmin]), rhs[jmin]);
    double den = c2 * Dj + u2[jmin];
    for (int g = 0; g < m; ++g) {
        if (g == jmin) continue;
        const double ratio = Dj / D[g];
        const cplx t = cmul(cconj(u[g]), rhs[g]);
        num.x += t.x * ratio;
        num.y += t.y * ratio;
        den += u2[g] * ratio;
    }
    const cplx sigma = {num.x / den, num.y / den};
    cplx zsum = {0.0, 0.0};
    cplx zg[M];
    for (int g = 0; g < m; ++g) {
        if (g == jmin) continue;
        const cplx us = cmul(u[g], sigma);
        zg[g] = {(rhs[g].x - us.x) / D[g], (rhs[g].y - us.y) / D[g]};
        const cplx t = cmul(cconj(u[g]), zg[g]);
        zsum.x += t.x;
        zsum.y += t.y;
    }
    if (u2[jmin] < c2 * Dj) {
        const cplx us = cmul(u[jmin], sigma);
        zg[jmin] = {(rhs[jmin].x - us.x) / Dj, (rhs[jmin].y - us.y) / Dj};
    } else {
        const cplx s = {c2 * sigma.x - zsum.x, c2 * sigma.y - zsum.y};
        const cplx uc = cconj(u[jmin]);
        const double d = u2[jmin];
        zg[jmin] = {(s.x * uc.x + s.y * uc.y) / d, (s.y * uc.x - s.x * uc.y) / d};
    }
    const int WH = W / 2 + 1;
    for (int a = 0; a < c; ++a)
        for (int b = 0; b < c; ++b) {
            const int Cc = ll + b * w;
            if (Cc < WH) {
                const int R = kl + a * h;
                const cplx v = zg[a * c + b];
                Z[static_cast<size_t>(R) * WH + Cc] = make_double2(v.x, v.y);
            }
        }
}

// out = (z_raw * (1/(H W))) * (1/scale)   (fft_util.cpp:47-56 then pansharpen.cpp:401)
__global__ void k_unscale(const double* __restrict__ zr, long long n, double inv_n, const double* __restrict__ dscale,
                          long long per_scale, double* __restrict__ out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double inv = dscale ? 1.0 / dscale[i / per_scale] : 1.0;
        out[i] = (zr[i] * inv_n) * inv;
    }
}

// ops.cpp:9-22 embed_kernel
// n <= H, W (checked by the callers): the taps land on distinct positions of the zeroed plane,
// so each is stored once (= 0 + tap, the reference's accumulation)
__global__ void k_embed(const double* __restrict__ taps, int n, int H, int W, double* __restrict__ out) {
    taps += static_cast<size_t>(blockIdx.x) * n * n;
    out += static_cast<size_t>(blockIdx.x) * H * W;
    const int C = (n - 1) / 2;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int r = e / n, q = e - r * n;
        const int rr = wrapi(r - C, H), cc = wrapi(q - C, W);
        out[static_cast<size_t>(rr) * W + cc] = 0.0 + taps[e];
    }
}

// ---- small helpers ---------------------------------------------------------------------------
__global__ void k_max_partial(const double* __restrict__ a, long long n, const double* __restrict__ b, long long nb,
                              double* __restrict__ part) {
    __shared__ double sh[256];
    a += blockIdx.y * n;
    b += blockIdx.y * nb;
    part += static_cast<size_t>(blockIdx.y) * gridDim.x;
    double m = -INFINITY;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n + nb; i += gridDim.x * 256LL)
        m = fmax(m, i < n ? a[i] : b[i - n]);
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_peak_final(const double* __restrict__ part, int nb, double* __restrict__ scale) {
    double m = -INFINITY;  // one warp per scene (max is exact in any order)
    for (int i = threadIdx.x; i < nb; i += 32) m = fmax(m, part[static_cast<size_t>(blockIdx.x) * nb + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) scale[blockIdx.x] = m > 0.0 ? 1.0 / m : 1.0;  // pansharpen.cpp:374-376
}
__global__ void k_scale_copy(const double* __restrict__ in, long long n, const double* __restrict__ s,
                             long long per, double* __restrict__ out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = in[i] * s[i / per];
}
__global__ void k_guided_combine(const double* __restrict__ ab, const double* __restrict__ cb,
                                 const double* __restrict__ g, long long n, double* __restrict__ out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = ab[i] * g[i] + cb[i];  // pansharpen.cpp:309-310
}
// L(in * s) with the reference's rounding: pan_n = pan * scale first (pansharpen.cpp:378-380)
__global__ void k_lap_scaled(const double* __restrict__ in, int H, int W, const double* __restrict__ s,
                             double* __restrict__ out) {
    const double sc = s ? s[blockIdx.y] : 1.0;
    const size_t P = static_cast<size_t>(H) * W;
    const double* ic = in + blockIdx.y * P;
    double* oc = out + blockIdx.y * P;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < static_cast<long long>(P);
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / W), c = static_cast<int>(i - static_cast<long long>(r) * W);
        const int rm = (r + H - 1) % H, rp = (r + 1) % H, cm = (c + W - 1) % W, cp = (c + 1) % W;
        const double x0 = __dmul_rn(ic[i], sc);
        const double xn = __dmul_rn(ic[static_cast<size_t>(rm) * W + c], sc);
        const double xs = __dmul_rn(ic[static_cast<size_t>(rp) * W + c], sc);
        const double xw = __dmul_rn(ic[static_cast<size_t>(r) * W + cm], sc);
        const double xe = __dmul_rn(ic[static_cast<size_t>(r) * W + cp], sc);
        double v = __dmul_rn(4.0, x0);
        v = __dsub_rn(v, xn);
        v = __dsub_rn(v, xs);
        v = __dsub_rn(v, xw);
        v = __dsub_rn(v, xe);
        oc[i] = v;
    }
}
__global__ void k_box_mean(const double* __restrict__ in, int H, int W, int rad, double* __restrict__ out) {
    const size_t P = static_cast<size_t>(H) * W;
    const double* ic = in + blockIdx.y * P;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < static_cast<long long>(P);
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / W), c = static_cast<int>(i - static_cast<long long>(r) * W);
        const int ra = max(0, r - rad), rb = min(H - 1, r + rad), ca = max(0, c - rad), cb = min(W - 1, c + rad);
        double s = 0.0;
        for (int y = ra; y <= rb; ++y)
            for (int x = ca; x <= cb; ++x) s += ic[static_cast<size_t>(y) * W + x];
        out[blockIdx.y * P + i] = s / static_cast<double>((rb - ra + 1) * (cb - ca + 1));
    }
}
__global__ void k_convolve(const double* __restrict__ in, int H, int W, const double* __restrict__ taps, int n,
                           int adjoint, double* __restrict__ out) {
    const int C = (n - 1) / 2;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
         i < static_cast<long long>(H) * W; i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / W), c = static_cast<int>(i - static_cast<long long>(r) * W);
        double s = 0.0;
        for (int a = -C; a <= C; ++a)
            for (int b = -C; b <= C; ++b) {
                const int rr = adjoint ? r + a : r - a, cc = adjoint ? c + b : c - b;
                s += taps[(a + C) * n + b + C] * in[static_cast<size_t>(wrapi(rr, H)) * W + wrapi(cc, W)];
            }
        out[i] = s;
    }
}

inline int grid1d(Context& ctx, long long n, int threads = 256) {
    long long b = (n + threads - 1) / threads;
    const long long cap = static_cast<long long>(ctx.sm_count) * 16;
    return static_cast<int>(std::max(1LL, std::min(b, cap)));
}

size_t q_smem(const PsGeo& G) {
    const int PW = TQ + 2 * G.g;
    return (static_cast<size_t>((G.n * G.n + 1) & ~1) + static_cast<size_t>(G.c) * G.c * plane_stride(PW)) *
           sizeof(double);
}
size_t a_smem(const PsGeo& G, int mode) { return static_cast<size_t>(apply_layout(G, mode, 0, 0).total) * sizeof(double); }

template <class K>
void set_smem(K kernel, size_t bytes) {
    FBMP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

void check_smem(size_t bytes, const char* what) {
    if (bytes > 227 * 1024)
        param_error(std::string(what) + ": problem parameters need more shared memory than an SM provides");
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// fast-path dispatch (cg_fast.cuh): radius 1, c in {1,2,4}, n <= 21, images >= 64 x 64
// ---------------------------------------------------------------------------------------------
bool fast_ok(const PsGeo& G) {
    return G.rw == 1 && (G.c == 1 || G.c == 2 || G.c == 4) && G.n <= fast::a4::MAXN && G.H >= 64 && G.W >= 64 &&
           std::getenv("FBMP_DISABLE_FAST") == nullptr;
}

template <class T>
using QFnT = void (*)(PsGeo, const T*, const T*, T*, T*, CgState*, double*, int);
template <class T>
struct QLaunchT {
    QFnT<T> fn = nullptr;
    size_t smem = 0;
    int nblk = 0;
    int threads = 0;
    bool streaming = false;  // K_Q3
};
using QLaunch = QLaunchT<double>;
// K_Q2's shared memory for storage type T (QGeo counts doubles)
template <int N_, int CF, int MJ, class T>
constexpr size_t q2_smem() { return fast::QGeo<N_, CF, MJ>::smem / sizeof(double) * sizeof(T); }
template <int N_, int CF, bool CG, class T = double>
QLaunchT<T> q2_make(const PsGeo& G) {
    QLaunchT<T> L;
    // narrow images (C1: 64 LR columns) are latency-bound: 1 LR column per lane gives 4x the CTAs
    // (the per-output summation order does not depend on MJ). Env FBMP_KQ2_MJ overrides.
    static const int mj_env = std::getenv("FBMP_KQ2_MJ") ? std::atoi(std::getenv("FBMP_KQ2_MJ")) : 0;
    const int mj = mj_env ? mj_env : (CF == 4 && G.w <= 64 ? 1 : 4);
    if (mj == 1) {
        L.fn = fast::k_q2<N_, CF, CG, 1, T>;
        L.smem = q2_smem<N_, CF, 1, T>();
        L.nblk = fast::q2_blocks<N_, CF, 1>(G);
        L.threads = fast::QGeo<N_, CF, 1>::NTH;
    } else if (mj == 2) {
        L.fn = fast::k_q2<N_, CF, CG, 2, T>;
        L.smem = q2_smem<N_, CF, 2, T>();
        L.nblk = fast::q2_blocks<N_, CF, 2>(G);
        L.threads = fast::QGeo<N_, CF, 2>::NTH;
    } else {
        L.fn = fast::k_q2<N_, CF, CG, 4, T>;
        L.smem = q2_smem<N_, CF, 4, T>();
        L.nblk = fast::q2_blocks<N_, CF>(G);
        L.threads = fast::QGeo<N_, CF>::NTH;
    }
    return L;
}
// K_Q3 strip plan: LR-row strips of SR rows per band. Large problems take the tallest SR in
// {128, 64, 32} that still gives >= 4 waves (halo overhead 2g/SR); small ones one wave of CTAs
// (occupancy from the runtime), floored at 4 rows. Env FBMP_KQ3_SR overrides.
template <int N_, bool CG, class T = double>
QLaunchT<T> q3_make(const PsGeo& G) {
    constexpr int MJ = 2;
    using Q = fast::q3::Geo<N_, MJ, T>;
    QLaunchT<T> L;
    L.fn = fast::k_q3<N_, MJ, CG, T>;
    L.smem = Q::smem;
    L.threads = fast::q3::NTH;
    L.streaming = true;
    static int sms = 0, per_sm = 0;
    if (!sms) {
        int dev = 0;
        FBMP_CUDA(cudaGetDevice(&dev));
        FBMP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    set_smem(L.fn, L.smem);
    FBMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.fn, L.threads, L.smem));
    const int nbands = ceil_div(G.w, Q::TWL);
    const long long slots = static_cast<long long>(sms) * std::max(per_sm, 1);
    int SR;
    if (const char* e = std::getenv("FBMP_KQ3_SR")) {
        SR = std::max(1, std::atoi(e));
    } else if (static_cast<long long>(nbands) * ceil_div(G.h, 32) * G.N >= 4 * slots) {
        // at least four waves: the tallest strip that keeps them (C5: 128 rows, 16 % faster than 32)
        SR = 32;
        for (int cand : {128, 64})
            if (static_cast<long long>(nbands) * ceil_div(G.h, cand) * G.N >= 4 * slots) {
                SR = cand;
                break;
            }
    } else {
        const long long per = std::max(1LL, slots / (static_cast<long long>(nbands) * G.N));
        SR = std::max(4, ceil_div(G.h, static_cast<int>(std::min<long long>(per, G.h))));
    }
    const int nstrips = ceil_div(G.h, std::min(SR, G.h));
    L.nblk = nbands * nstrips;
    return L;
}
bool q3_ok(const PsGeo& G) {
    // K_Q3 from LR width 128 (C2..C5); narrower images keep the tile kernel (env FBMP_KQ3_MINW)
    static const bool off = std::getenv("FBMP_KQ") && std::atoi(std::getenv("FBMP_KQ")) == 2;
    static const int minw = std::getenv("FBMP_KQ3_MINW") ? std::atoi(std::getenv("FBMP_KQ3_MINW")) : 128;
    return !off && G.c == 4 && G.w >= std::max(64, minw) && G.W % 4 == 0;
}

template <bool CG, class T = double>
QLaunchT<T> q2_select(const PsGeo& G) {
    if (!fast_ok(G)) return {};
    if (G.c == 4 && q3_ok(G)) {
        switch (G.n) {
        case 21: return q3_make<21, CG, T>(G);
        case 17: return q3_make<17, CG, T>(G);
        case 15: return q3_make<15, CG, T>(G);
        case 7: return q3_make<7, CG, T>(G);
        default: break;
        }
    }
    if (G.c == 4) {
        switch (G.n) {
        case 21: return q2_make<21, 4, CG, T>(G);
        case 17: return q2_make<17, 4, CG, T>(G);
        case 15: return q2_make<15, 4, CG, T>(G);
        case 7: return q2_make<7, 4, CG, T>(G);
        default: break;
        }
    } else if (G.c == 2) {
        switch (G.n) {
        case 5: return q2_make<5, 2, CG, T>(G);
        case 3: return q2_make<3, 2, CG, T>(G);
        default: break;
        }
    }
    return {};
}

// per-scene (mu_k, g_k) maps for the fast K_A (formed in fp64, stored as T)
template <class T>
void guide_stats_t(Context& ctx, const PsGeo& G, const double* d_guide, T* mu, T* gk) {
    const int S = (G.N + G.cps - 1) / G.cps;
    fast::k_guide_stats<<<dim3(grid1d(ctx, static_cast<long long>(G.H) * G.W), S), 256, 0, ctx.stream>>>(
        d_guide, G.H, G.W, G.rw, G.eps, mu, gk);
    ctx.count();
    check_launch();
}
void guide_stats(Context& ctx, const PsGeo& G, const double* d_guide, double* mu, double* gk) {
    guide_stats_t<double>(ctx, G, d_guide, mu, gk);
}

using AFn = void (*)(PsGeo, const double*, const double*, const double*, const double*, const double*,
                     const double*, double*, CgState*, double*, int);
template <bool CG>
std::pair<AFn, size_t> apply3_select(const PsGeo& G) {
    if (G.c == 4) {
        const size_t sm = fast::a4::L<4>::smem;
        switch (G.n) {
        case 21: return {fast::k_apply4<CG, 21, 4>, sm};
        case 17: return {fast::k_apply4<CG, 17, 4>, sm};
        case 15: return {fast::k_apply4<CG, 15, 4>, sm};
        case 7: return {fast::k_apply4<CG, 7, 4>, sm};
        default: return {fast::k_apply4<CG, 0, 4>, sm};
        }
    }
    if (G.c == 2) return {fast::k_apply4<CG, 0, 2>, fast::a4::L<2>::smem};
    return {fast::k_apply4<CG, 0, 1>, fast::a4::L<1>::smem};
}

// K_D + K_L (the default CG operator; env FBMP_KA=4 selects the single-kernel K_A)
struct LlpPlan {
    int nb = 0, k = 1, R = 0, ctas = 0;
    bool pairs = false;  // k_llp2 (column pairs; W even)
    bool quads = false;  // k_llp4f (fp32 mode, four columns per lane; W % 4 == 0)
};
inline bool use_llp() {
    static const bool on = !(std::getenv("FBMP_KA") && std::atoi(std::getenv("FBMP_KA")) == 4);
    return on;
}
// Strip height: minimise rounds x (R + 8) (a warp's steps, 8 = pipeline warm-up rows) over the
// resident warp slots; R is a multiple of the partial row block.
template <class T = double>
LlpPlan llp_plan(Context& ctx, const PsGeo& G) {
    static int per_sm[3] = {0, 0, 0};
    LlpPlan L;
    static const bool no_pairs = std::getenv("FBMP_KL1") != nullptr;
    static const bool no_quads = std::getenv("FBMP_KL_NOQUAD") != nullptr;  // A/B: fp32 on k_llp2
    L.pairs = (G.W % 2 == 0) && (!no_pairs || !std::is_same<T, double>::value);
    L.quads = !std::is_same<T, double>::value && G.W % 4 == 0 && !no_quads && !G.identity;
    int& ps = per_sm[L.quads ? 2 : (L.pairs ? 1 : 0)];
    if (!ps) {
        int blocks = 0;
        if (L.quads)
            FBMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fast::k_llp4f<true>, fast::kl::NTL, 0));
        else if (L.pairs)
            FBMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fast::k_llp2<true, T>, fast::kl::NTL, 0));
        else
            FBMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fast::k_llp<true>, fast::kl::NTL, 0));
        ps = std::max(1, std::min(blocks, 32)) * (fast::kl::NTL / 32);
    }
    const long long slots = static_cast<long long>(ps) * ctx.sm_count;
    L.nb = ceil_div(G.W, L.quads ? fast::kl::BAND4 : (L.pairs ? fast::kl::BAND2 : fast::kl::BAND));
    const long long bc = static_cast<long long>(L.nb) * G.N;
    long long best = -1;
    for (int k = 1; k <= ceil_div(G.H, fast::kl::RB); ++k) {
        const int R = ceil_div(ceil_div(G.H, k), fast::kl::RB) * fast::kl::RB;
        const int ke = ceil_div(G.H, R);
        const long long items = bc * ke, rounds = (items + slots - 1) / slots;
        const long long cost = rounds * (R + 8);
        if (best < 0 || cost < best) {
            best = cost;
            L.k = ke;
            L.R = R;
        }
    }
    L.ctas = L.nb * L.k;
    return L;
}
template <bool CG, class T = double>
std::pair<void (*)(PsGeo, const T*, const T*, T*, const CgState*), size_t> dterm_select(const PsGeo& G) {
    constexpr size_t sc = sizeof(T);  // dterm_smem counts doubles
    if (G.c == 4) {
        const size_t sm = fast::kl::dterm_smem<4>(G.cpc) / 8 * sc;  // register-tap variants hold every channel's window
        switch (G.n) {
        case 21: return {fast::k_dterm<CG, 21, 4, T>, sm};
        case 17: return {fast::k_dterm<CG, 17, 4, T>, sm};
        case 15: return {fast::k_dterm<CG, 15, 4, T>, sm};
        case 7: return {fast::k_dterm<CG, 7, 4, T>, sm};
        default: return {fast::k_dterm<CG, 0, 4, T>, fast::kl::dterm_smem<4>() / 8 * sc};
        }
    }
    if (G.c == 2) return {fast::k_dterm<CG, 0, 2, T>, fast::kl::dterm_smem<2>() / 8 * sc};
    return {fast::k_dterm<CG, 0, 1, T>, fast::kl::dterm_smem<1>() / 8 * sc};
}
template <bool CG, class T = double>
void launch_llp(Context& ctx, const PsGeo& G, const T* taps, const T* guide, const T* mu,
                const T* gk, const T* p, const T* q, T* out, CgState* st, double* part,
                bool pdl = false, cudaEvent_t between = nullptr) {
    const int S = (G.N + G.cps - 1) / G.cps;
    const int nba = ceil_div(G.W, fast::a4::TA) * ceil_div(G.H, fast::a4::TA);
    const int groups = (G.cps + G.cpc - 1) / G.cpc;
    const auto fd = dterm_select<CG, T>(G);
    if (pdl)
        launch_pdl(fd.first, dim3(nba, S * groups), dim3(fast::NT), fd.second, ctx.stream, G, taps, q, out,
                   static_cast<const CgState*>(st));
    else
        fd.first<<<dim3(nba, S * groups), fast::NT, fd.second, ctx.stream>>>(G, taps, q, out, st);
    if (between) FBMP_CUDA(cudaEventRecordWithFlags(between, ctx.stream, cudaEventRecordExternal));
    const LlpPlan L = llp_plan<T>(ctx, G);
    if (G.identity) {  // identity prior: M without the Laplacians (pair kernel only)
        if (!L.pairs) param_error("pansharpen: the identity prior on the device needs an even image width");
        fast::k_llp2<CG, T, false><<<dim3(L.ctas * G.N), fast::kl::NTL, 0, ctx.stream>>>(G, guide, mu, gk, p, out, st,
                                                                                         part, L.nb, L.k, L.R);
        return;
    }
    if constexpr (!std::is_same<T, double>::value) {
        if (L.quads) {
            fast::k_llp4f<CG><<<dim3(L.ctas * G.N), fast::kl::NTL, 0, ctx.stream>>>(G, guide, mu, gk, p, out, st, part,
                                                                                    L.nb, L.k, L.R);
            return;
        }
    }
    // env FBMP_PDL_KL=1: K_L also by programmatic dependent launch (its CTAs start while K_D drains)
    static const bool pdl_kl = std::getenv("FBMP_PDL_KL") && std::atoi(std::getenv("FBMP_PDL_KL")) == 1;
    if (L.pairs && pdl && pdl_kl) {
        launch_pdl(fast::k_llp2<CG, T>, dim3(L.ctas * G.N), dim3(fast::kl::NTL), 0, ctx.stream, G, guide, mu, gk, p,
                   out, st, part, L.nb, L.k, L.R);
    } else if (L.pairs) {
        fast::k_llp2<CG, T><<<dim3(L.ctas * G.N), fast::kl::NTL, 0, ctx.stream>>>(G, guide, mu, gk, p, out, st, part,
                                                                                  L.nb, L.k, L.R);
    } else {
        if constexpr (std::is_same<T, double>::value)
            fast::k_llp<CG><<<dim3(L.ctas * G.N), fast::kl::NTL, 0, ctx.stream>>>(G, guide, mu, gk, p, out, st, part,
                                                                                  L.nb, L.k, L.R);
        else
            param_error("pansharpen: the fp32 mode needs an even image width");
    }
}

// Fused CG path (K_Q3 -> K_L without d -> K_DU): p.Ap = ||q||^2 + lambda p.(L M L p), and the
// data term is formed inside the update kernel, so d and Ap never touch HBM (11 planes per
// channel-iteration). Needs the streaming K_Q3 (it sums ||q||^2), the pair / quad K_L
// and image sides that are multiples of the 32 x 32 tile. Env FBMP_DU=0 keeps K_D + K_L + K_U.
template <class T>
using DuFn = void (*)(PsGeo, const T*, const T*, const T*, T*, T*, const T*, CgState*, double*, int);
template <class T>
DuFn<T> du_select(const PsGeo& G) {
    static const bool off = std::getenv("FBMP_DU") && std::atoi(std::getenv("FBMP_DU")) == 0;
    if (off || G.c != 4 || G.H % fast::du::TH || G.W % fast::du::TW || !use_llp() || G.N > fast::du::MAXCH)
        return nullptr;
    // row strips: K_DU sums whole tiles, K_Q3 whole LR rows
    if (G.dred && (G.rlo % fast::du::TH || G.rhi % fast::du::TH)) return nullptr;
    switch (G.n) {
    case 21: return fast::k_du<21, T>;
    case 17: return fast::k_du<17, T>;
    case 15: return fast::k_du<15, T>;
    case 7: return fast::k_du<7, T>;
    default: return nullptr;
    }
}
// K_L of the fused path: w = L M L p into `out`, p.Ap = qq + lambda p.w
template <class T>
void launch_llp_w(Context& ctx, const PsGeo& G, const T* guide, const T* mu, const T* gk, const T* p, T* out,
                  CgState* st, double* part, bool pdl) {
    const LlpPlan L = llp_plan<T>(ctx, G);
    const dim3 grid(L.ctas * G.N), blk(fast::kl::NTL);
    auto go = [&](auto fn) {
        if (pdl)
            launch_pdl(fn, grid, blk, 0, ctx.stream, G, guide, mu, gk, p, out, st, part, L.nb, L.k, L.R);
        else
            fn<<<grid, blk, 0, ctx.stream>>>(G, guide, mu, gk, p, out, st, part, L.nb, L.k, L.R);
    };
    if (G.identity) {
        go(fast::k_llp2<true, T, false, false>);
        return;
    }
    if constexpr (!std::is_same<T, double>::value) {
        if (L.quads) {
            go(fast::k_llp4f<true, false>);
            return;
        }
    }
    go(fast::k_llp2<true, T, true, false>);
}

// rhs = B^T U x into r through K_D, then the CG initialisation (fast path; k_rhs otherwise)
template <class T = double>
void launch_rhs_init(Context& ctx, const PsGeo& G, const T* taps, const T* x, CgBuffersT<T>& B, double* part,
                     int max_iters, double cg_tol) {
    const int S = (G.N + G.cps - 1) / G.cps;
    const int nba = ceil_div(G.W, fast::a4::TA) * ceil_div(G.H, fast::a4::TA);
    const int groups = (G.cps + G.cpc - 1) / G.cpc;
    const auto fd = dterm_select<false, T>(G);
    set_smem(fd.first, fd.second);
    fd.first<<<dim3(nba, S * groups), fast::NT, fd.second, ctx.stream>>>(G, taps, x, B.r, nullptr);
    const size_t P = static_cast<size_t>(G.H) * G.W;
    const int nbu = static_cast<int>((P + static_cast<size_t>(NTU) * UPT - 1) / (static_cast<size_t>(NTU) * UPT));
    k_cg_init<T><<<dim3(nbu, G.N), NTU, 0, ctx.stream>>>(G, B.r, B.z, B.p + static_cast<size_t>(G.N) * P, B.st, part,
                                                        nbu, max_iters, cg_tol);
    ctx.count(2);
    check_launch();
}

template <bool CG, class T = double>
void launch_apply2(Context& ctx, const PsGeo& G, const T* taps, const T* guide, const T* mu,
                   const T* gk, const T* p, const T* q, T* out, CgState* st, double* part,
                   bool pdl = false, cudaEvent_t between = nullptr) {
    const int S = (G.N + G.cps - 1) / G.cps;
    const int nba = ceil_div(G.W, fast::a4::TA) * ceil_div(G.H, fast::a4::TA);
    const int groups = (G.cps + G.cpc - 1) / G.cpc;
    if (use_llp() || !std::is_same<T, double>::value) {
        launch_llp<CG, T>(ctx, G, taps, guide, mu, gk, p, q, out, st, part, pdl, between);
        return;
    }
    if constexpr (std::is_same<T, double>::value) {
        if (between) FBMP_CUDA(cudaEventRecordWithFlags(between, ctx.stream, cudaEventRecordExternal));
        const auto fs = apply3_select<CG>(G);
        if (pdl)
            launch_pdl(fs.first, dim3(nba, S * groups), dim3(fast::NT), fs.second, ctx.stream, G, taps, guide, mu, gk,
                       p, q, out, st, part, nba);
        else
            fs.first<<<dim3(nba, S * groups), fast::NT, fs.second, ctx.stream>>>(G, taps, guide, mu, gk, p, q, out, st,
                                                                                  part, nba);
    }
}

template <bool CG, class T = double>
void prepare_apply2(const PsGeo& G) {
    if (use_llp() || !std::is_same<T, double>::value) {
        const auto fd = dterm_select<CG, T>(G);
        set_smem(fd.first, fd.second);
        return;
    }
    const auto fs = apply3_select<CG>(G);
    set_smem(fs.first, fs.second);
}

// =============================================================================================
// host wrappers
// =============================================================================================
void data_rhs(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_x, double* d_out) {
    const int nb = ceil_div(G.W, TA) * ceil_div(G.H, TA);
    const size_t sm = static_cast<size_t>(G.n) * G.n * sizeof(double);
    set_smem(k_rhs<false>, sm);
    k_rhs<false><<<dim3(nb, G.N), NTA, sm, ctx.stream>>>(G, d_taps, d_x, d_out, nullptr, nullptr, nullptr, nullptr,
                                                         nb, 0, 0.0);
    ctx.count();
    check_launch();
}

void cg_operator_apply(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_guide, const double* d_p,
                       double* d_out, int mode) {
    const int nbq = ceil_div(G.w, TQ) * ceil_div(G.h, TQ);
    const int nba = ceil_div(G.W, TA) * ceil_div(G.H, TA);
    double* q = ctx.scratch<double>("op_q", static_cast<size_t>(G.N) * G.h * G.w);
    if (mode != 1) {
        const QLaunch ql = q2_select<false>(G);
        if (ql.fn) {
            set_smem(ql.fn, ql.smem);
            ql.fn<<<dim3(ql.nblk, G.N), ql.threads, ql.smem, ctx.stream>>>(G, d_taps, d_p, nullptr, q, nullptr, nullptr,
                                                                          ql.nblk);
        } else {
            const size_t sq = q_smem(G);
            check_smem(sq, "cg operator");
            set_smem(k_q<false>, sq);
            k_q<false><<<dim3(nbq, G.N), NTQ, sq, ctx.stream>>>(G, d_taps, d_p, nullptr, q, nullptr, nullptr, nbq);
        }
        ctx.count();
        check_launch();
    }
    if (mode == 0 && fast_ok(G)) {
        const size_t P = static_cast<size_t>(G.H) * G.W;
        const int S = (G.N + G.cps - 1) / G.cps;
        double* mu = ctx.scratch<double>("op_wmu", P * S);
        double* gk = ctx.scratch<double>("op_wg", P * S);
        guide_stats(ctx, G, d_guide, mu, gk);
        prepare_apply2<false>(G);
        launch_apply2<false>(ctx, G, d_taps, d_guide, mu, gk, d_p, q, d_out, nullptr, nullptr);
        ctx.count();
        check_launch();
        return;
    }
    if (G.identity && mode != 1) param_error("cg operator: the identity prior needs the specialised operator");
    const size_t sa = a_smem(G, mode);
    check_smem(sa, "cg operator");
    if (mode == 0) {
        set_smem(k_apply<0, false>, sa);
        k_apply<0, false><<<dim3(nba, G.N), NTA, sa, ctx.stream>>>(G, d_taps, d_guide, d_p, q, d_out, nullptr, nullptr, nba);
    } else if (mode == 1) {
        set_smem(k_apply<1, false>, sa);
        k_apply<1, false><<<dim3(nba, G.N), NTA, sa, ctx.stream>>>(G, d_taps, d_guide, d_p, q, d_out, nullptr, nullptr, nba);
    } else {
        set_smem(k_apply<2, false>, sa);
        k_apply<2, false><<<dim3(nba, G.N), NTA, sa, ctx.stream>>>(G, d_taps, d_guide, d_p, q, d_out, nullptr, nullptr, nba);
    }
    ctx.count();
    check_launch();
}

// The CG loop for storage type T: double, or float (fp32 mode: fast path only; the guide maps
// are formed in fp64 from d_guide64 and stored as T, d_guide is the T copy K_L streams).
template <class T>
void cg_solve_t(Context& ctx, const PsGeo& G, const T* d_taps, const double* d_guide64, const T* d_guide, const T* d_x,
                CgBuffersT<T>& B, int max_iters, double cg_tol, std::vector<CgState>& host_state) {
    constexpr bool F64 = std::is_same<T, double>::value;
    const int N = G.N;
    const QLaunchT<T> q2 = q2_select<true, T>(G);
    const bool fastA = fast_ok(G);
    if (!F64 && !(fastA && q2.fn))
        param_error("pansharpen: the fp32 mode needs the specialised operator (radius 1, factor 2 or 4 with a "
                    "supported kernel side, images >= 64 x 64)");
    if (G.identity && !(fastA && use_llp()))
        param_error("pansharpen: the identity prior on the device needs the specialised operator (radius 1, "
                    "factor 1, 2 or 4, images >= 64 x 64)");
    const int nbq = q2.fn ? q2.nblk : ceil_div(G.w, TQ) * ceil_div(G.h, TQ);
    const int nba = fastA ? ceil_div(G.W, fast::a4::TA) * ceil_div(G.H, fast::a4::TA) : ceil_div(G.W, TA) * ceil_div(G.H, TA);
    const size_t P = static_cast<size_t>(G.H) * G.W;
    const int nbu = static_cast<int>((P + static_cast<size_t>(NTU) * upt<T>() - 1) / (static_cast<size_t>(NTU) * upt<T>()));
    const size_t sq = q2.fn ? q2.smem : q_smem(G), sa = a_smem(G, 0), sr = static_cast<size_t>(G.n) * G.n * sizeof(double);
    check_smem(sq, "warmstart");
    if (!fastA) check_smem(sa, "warmstart");
    if (q2.fn) set_smem(q2.fn, q2.smem);
    if constexpr (F64) {
        if (!q2.fn) set_smem(k_q<true>, sq);
        if (!fastA) set_smem(k_apply<0, true>, sa);
        set_smem(k_rhs<true>, sr);
    }
    if (fastA) prepare_apply2<true, T>(G);
    T* wmu = nullptr;
    T* wg = nullptr;
    if (fastA) {
        const int S = (G.N + G.cps - 1) / G.cps;
        wmu = ctx.scratch<T>("cg_wmu", P * S);
        wg = ctx.scratch<T>("cg_wg", P * S);
        guide_stats_t<T>(ctx, G, d_guide64, wmu, wg);
    }
    double* part_init = B.part;
    double* part_q = part_init + static_cast<size_t>(N) * nba;
    // K_Q3 also publishes ||q||^2 partials per (LR row, 64-column band) behind its ||p||^2 partials
    const size_t nqseg = static_cast<size_t>(G.h) * ceil_div(G.w, 64);
    double* part_a = part_q + static_cast<size_t>(N) * (nbq + nqseg);
    const int nbA = fastA && use_llp() ? std::max(nba, ceil_div(G.W, fast::kl::BAND) * ceil_div(G.H, fast::kl::RB)) : nba;  // >= k_llp2's
    double* part_u = part_a + static_cast<size_t>(N) * nbA;
    // fused path: K_Q3 -> K_L (w, p.Ap from ||q||^2) -> K_DU (data term + update)
    const DuFn<T> du = fastA && q2.fn && q2.streaming && llp_plan<T>(ctx, G).pairs ? du_select<T>(G) : nullptr;
    const size_t sdu = du ? fast::du::smem<T>() : 0;
    int du_ctas = 0;  // persistent K_DU: one CTA per resident slot
    if (du) {
        set_smem(du, sdu);
        int per_sm = 0;
        FBMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, du, fast::du::NTD, sdu));
        static const int du_env = std::getenv("FBMP_DU_PER_SM") ? std::atoi(std::getenv("FBMP_DU_PER_SM")) : 0;
        if (du_env > 0) per_sm = std::min(per_sm, du_env);
        du_ctas = std::max(1, per_sm) * ctx.sm_count;
    }
    const int ntile_du = (G.W / fast::du::TW) * (G.H / fast::du::TH);
    const int nbU = du ? std::max(nbu, ntile_du) : nbu;  // K_DU publishes one (rr, zz) pair per tile
    // counters must start at zero
    FBMP_CUDA(cudaMemsetAsync(B.st, 0, sizeof(CgState) * N, ctx.stream));
    if (fastA && (use_llp() || !F64)) {
        launch_rhs_init<T>(ctx, G, d_taps, d_x, B, part_init, max_iters, cg_tol);
    } else if constexpr (F64) {
        k_rhs<true><<<dim3(nba, N), NTA, sr, ctx.stream>>>(G, d_taps, d_x, B.r, B.z, B.p + static_cast<size_t>(N) * P,
                                                           B.st, part_init, nba, max_iters, cg_tol);
        ctx.count();
        check_launch();
    }

    // One CUDA graph holds `chunk` iterations (3 kernels each); kernels of finished channels
    // exit at their first instruction, so the host only polls the flags between graphs.
    // In profile mode event records bracket every kernel and graphs are not pipelined.
    const int chunk = 8;
    const bool prof = ctx.profile;
    // programmatic dependent launch per CG kernel (bit 0 K_Q, 1 K_A, 2 K_U; env FBMP_PDL).
    // PDL on all three launches: C2 (K_Q3) 19.74 -> 19.44 ms, C1 (one-column K_Q2) 8.01 -> 7.92 ms,
    // C3/C4 neutral. (With the four-column K_Q2 it cost C1 5.5 %.)
    static const int pdl_env = std::getenv("FBMP_PDL") ? std::atoi(std::getenv("FBMP_PDL")) : -1;
    const int pdl_mask = pdl_env >= 0 ? pdl_env : 7;
    constexpr int EV = 5;  // profile events per iteration: K_Q | K_D | K_L (or K_A) | K_U
    std::vector<cudaEvent_t> pev(prof ? chunk * EV : 0);
    for (auto& e : pev) FBMP_CUDA(cudaEventCreate(&e));
    // the chunk graph depends only on geometry, buffers and launch shapes: cache it in the context
    std::string key;
    {
        const void* ptrs[] = {d_taps, d_guide, wmu, wg, B.r, B.p, B.q, B.Ap, B.st, B.z, part_q, part_a, part_u,
                              reinterpret_cast<const void*>(q2.fn), reinterpret_cast<const void*>(du)};
        const long long dims[] = {nbq, nba, nbu, static_cast<long long>(sq), fastA ? 1 : 0, chunk,
                                  static_cast<long long>(sizeof(T))};
        key.append(reinterpret_cast<const char*>(&G), sizeof(G));
        key.append(reinterpret_cast<const char*>(ptrs), sizeof(ptrs));
        key.append(reinterpret_cast<const char*>(dims), sizeof(dims));
    }
    // channel groups: the chunk graph holds two independent CG chains on two streams (fork / join
    // inside the graph), so the kernels of one half of the channels overlap the tails (and, between
    // the memory-bound K_DU and the latency-bound K_Q3 / K_L, the idle resources) of the other
    // half's. On by default for a single scene with the fused chain (measured, same bits: C2 16.85 ->
    // 16.13 ms, C3 84.1 -> 80.0 ms, C5 1203 -> 1180 ms, C1 7.34 -> 7.24 ms); off for scene batches
    // (C4: 205 -> 255 ms, the batch already fills the GPU). Env FBMP_CG_GROUPS = 1 / 2 overrides.
    static const int groups_env = std::getenv("FBMP_CG_GROUPS") ? std::atoi(std::getenv("FBMP_CG_GROUPS")) : 0;
    const int S_sc = (G.N + G.cps - 1) / G.cps;
    int ngrp = 1;
    const bool grp_ok = !prof && fastA && q2.fn && use_llp() && (S_sc >= 2 || (S_sc == 1 && N >= 2));
    if (grp_ok && (groups_env >= 2 || (groups_env == 0 && S_sc == 1)))
        ngrp = std::min({std::max(groups_env, 2), 4, S_sc >= 2 ? S_sc : N});
    struct Grp {
        PsGeo G;
        int c0 = 0;
        const T *taps, *guide, *mu, *g;
        CgBuffersT<T> B;
        double *pq, *pa, *pu;
    };
    std::vector<Grp> grp(ngrp);
    {
        const size_t per_ch = static_cast<size_t>(nba) + nbq + nqseg + nbA + 2 * static_cast<size_t>(nbU);
        for (int gi = 0; gi < ngrp; ++gi) {
            Grp& R = grp[gi];
            int c0, c1;
            if (ngrp == 1) {
                c0 = 0;
                c1 = N;
            } else if (S_sc >= 2) {  // whole scenes
                const int s0 = gi * S_sc / ngrp, s1 = (gi + 1) * S_sc / ngrp;
                c0 = s0 * G.cps;
                c1 = std::min(N, s1 * G.cps);
            } else {
                c0 = gi * N / ngrp;
                c1 = (gi + 1) * N / ngrp;
            }
            const int ng = c1 - c0, s0 = c0 / G.cps;
            R.c0 = c0;
            R.G = G;
            R.G.N = ng;
            if (S_sc == 1 && ngrp > 1) {
                R.G.cps = ng;
                R.G.cpc = std::min(G.cpc, ng);
            }
            R.taps = d_taps + static_cast<size_t>(s0) * G.n * G.n;
            R.guide = d_guide + static_cast<size_t>(s0) * P;
            R.mu = wmu ? wmu + static_cast<size_t>(s0) * P : nullptr;
            R.g = wg ? wg + static_cast<size_t>(s0) * P : nullptr;
            R.B = B;
            R.B.z = B.z + c0 * P;
            R.B.r = B.r + c0 * P;
            R.B.Ap = B.Ap + c0 * P;
            R.B.p = B.p + 2 * c0 * P;  // group-local parity double buffer (ng planes each)
            R.B.q = B.q + static_cast<size_t>(c0) * G.h * G.w;
            R.B.st = B.st + c0;
            if (ngrp == 1) {
                R.pq = part_q;
                R.pa = part_a;
                R.pu = part_u;
            } else {
                double* base = B.part + c0 * per_ch;
                R.pq = base;
                R.pa = R.pq + static_cast<size_t>(ng) * (nbq + nqseg);
                R.pu = R.pa + static_cast<size_t>(ng) * nbA;
            }
        }
        // k_rhs zeroed p_old in the whole-launch layout; the group layout needs the same zeros
        if (ngrp > 1) FBMP_CUDA(cudaMemsetAsync(B.p, 0, 2 * P * N * sizeof(T), ctx.stream));
    }
    key.append(reinterpret_cast<const char*>(&ngrp), sizeof(ngrp));
    trace("cg: setup");
    cudaGraphExec_t exec = nullptr;
    auto cached = prof ? ctx.graphs.end() : ctx.graphs.find(key);
    if (cached != ctx.graphs.end()) {
        exec = cached->second;
    } else {
        cudaGraph_t graph;
        cudaStream_t main = ctx.stream;
        for (int a = 0; a + 1 < ngrp; ++a)
            if (!ctx.aux_streams[a]) {
                FBMP_CUDA(cudaStreamCreateWithFlags(&ctx.aux_streams[a], cudaStreamNonBlocking));
                FBMP_CUDA(cudaEventCreateWithFlags(&ctx.join_evs[a], cudaEventDisableTiming));
            }
        if (ngrp > 1 && !ctx.fork_ev) FBMP_CUDA(cudaEventCreateWithFlags(&ctx.fork_ev, cudaEventDisableTiming));
        FBMP_CUDA(cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal));
        if (ngrp > 1) {
            FBMP_CUDA(cudaEventRecord(ctx.fork_ev, main));
            for (int a = 0; a + 1 < ngrp; ++a) FBMP_CUDA(cudaStreamWaitEvent(ctx.aux_streams[a], ctx.fork_ev, 0));
        }
        for (int gi = 0; gi < ngrp; ++gi) {
            Grp& R = grp[gi];
            const int Ng = R.G.N;
            ctx.stream = gi == 0 ? main : ctx.aux_streams[gi - 1];  // launch helpers enqueue on ctx.stream
            for (int it = 0; it < chunk; ++it) {
                if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 0], ctx.stream, cudaEventRecordExternal));
                if (q2.fn && (pdl_mask & 1))
                    launch_pdl(q2.fn, dim3(nbq, Ng), dim3(q2.threads), sq, ctx.stream, R.G, R.taps, R.B.r, R.B.p, R.B.q,
                               R.B.st, R.pq, nbq);
                else if (q2.fn)
                    q2.fn<<<dim3(nbq, Ng), q2.threads, sq, ctx.stream>>>(R.G, R.taps, R.B.r, R.B.p, R.B.q, R.B.st, R.pq,
                                                                         nbq);
                else if constexpr (F64)
                    k_q<true><<<dim3(nbq, Ng), NTQ, sq, ctx.stream>>>(R.G, R.taps, R.B.r, R.B.p, R.B.q, R.B.st, R.pq,
                                                                       nbq);
                if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 1], ctx.stream, cudaEventRecordExternal));
                if (du) {
                    if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 2], ctx.stream, cudaEventRecordExternal));
                    launch_llp_w<T>(ctx, R.G, R.guide, R.mu, R.g, R.B.p, R.B.Ap, R.B.st, R.pa, (pdl_mask & 2) != 0);
                    if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 3], ctx.stream, cudaEventRecordExternal));
                    if (pdl_mask & 4)
                        launch_pdl(du, dim3(du_ctas), dim3(fast::du::NTD), sdu, ctx.stream, R.G, R.taps, R.B.q, R.B.Ap, R.B.z,
                                   R.B.r, R.B.p, R.B.st, R.pu, ntile_du);
                    else
                        du<<<dim3(du_ctas), fast::du::NTD, sdu, ctx.stream>>>(R.G, R.taps, R.B.q, R.B.Ap, R.B.z, R.B.r, R.B.p,
                                                                        R.B.st, R.pu, ntile_du);
                    if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 4], ctx.stream, cudaEventRecordExternal));
                    continue;
                }
                if (fastA) {
                    launch_apply2<true, T>(ctx, R.G, R.taps, R.guide, R.mu, R.g, R.B.p, R.B.q, R.B.Ap, R.B.st, R.pa,
                                           (pdl_mask & 2) != 0, prof ? pev[it * EV + 2] : nullptr);
                } else if constexpr (F64) {
                    if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 2], ctx.stream, cudaEventRecordExternal));
                    k_apply<0, true><<<dim3(nba, Ng), NTA, sa, ctx.stream>>>(R.G, R.taps, R.guide, R.B.p, R.B.q,
                                                                              R.B.Ap, R.B.st, R.pa, nba);
                }
                if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 3], ctx.stream, cudaEventRecordExternal));
                if (pdl_mask & 4)
                    launch_pdl(k_update<T>, dim3(nbu, Ng), dim3(NTU), 0, ctx.stream, R.G, R.B.z, R.B.r, R.B.p, R.B.Ap,
                               R.B.st, R.pu, nbu);
                else
                    k_update<T><<<dim3(nbu, Ng), NTU, 0, ctx.stream>>>(R.G, R.B.z, R.B.r, R.B.p, R.B.Ap, R.B.st, R.pu,
                                                                       nbu);
                if (prof) FBMP_CUDA(cudaEventRecordWithFlags(pev[it * EV + 4], ctx.stream, cudaEventRecordExternal));
            }
        }
        ctx.stream = main;
        if (ngrp > 1) {
            for (int a = 0; a + 1 < ngrp; ++a) {
                FBMP_CUDA(cudaEventRecord(ctx.join_evs[a], ctx.aux_streams[a]));
                FBMP_CUDA(cudaStreamWaitEvent(main, ctx.join_evs[a], 0));
            }
        }
        FBMP_CUDA(cudaStreamEndCapture(main, &graph));
        FBMP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        if (!prof) {
            if (ctx.graphs.size() >= 16) {
                for (auto& kv : ctx.graphs) cudaGraphExecDestroy(kv.second);
                ctx.graphs.clear();
            }
            ctx.graphs.emplace(key, exec);
        }
    }
    trace("cg: graph");

    CgState* pinned = static_cast<CgState*>(ctx.pinned(sizeof(CgState) * N * 2));
    cudaEvent_t* ev = ctx.poll_ev;
    for (int i = 0; i < 2; ++i)
        if (!ev[i]) FBMP_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    trace("cg: pinned + events");
    auto all_done = [&](const CgState* s) {
        for (int i = 0; i < N; ++i)
            if (!s[i].done) return false;
        return true;
    };
    auto launch = [&](int slot) {
        FBMP_CUDA(cudaGraphLaunch(exec, ctx.stream));
        ctx.count((fastA && !du && (use_llp() || !F64) ? 4 : 3) * chunk * ngrp);  // kernel nodes of one chunk graph
        FBMP_CUDA(cudaMemcpyAsync(pinned + slot * N, B.st, sizeof(CgState) * N, cudaMemcpyDeviceToHost, ctx.stream));
        FBMP_CUDA(cudaEventRecord(ev[slot], ctx.stream));
    };
    const long long max_graphs = static_cast<long long>(max_iters) / chunk + 4;
    int k = 0;
    if (prof) {
        // iterations with at least one active channel = max over channels of iters
        for (long long g = 0; g <= max_graphs; ++g) {
            launch(0);
            FBMP_CUDA(cudaEventSynchronize(ev[0]));
            int active_iters = 0;
            for (int i = 0; i < N; ++i) active_iters = std::max(active_iters, pinned[i].done ? pinned[i].iters : pinned[i].t);
            for (int it = 0; it < chunk; ++it) {
                if (g * chunk + it >= active_iters) break;
                for (int kk = 0; kk < EV - 1; ++kk) {
                    if (du && kk == 1) continue;  // fused path: no K_D launch (the slot is an empty event pair)
                    float ms = 0.f;
                    FBMP_CUDA(cudaEventElapsedTime(&ms, pev[it * EV + kk], pev[it * EV + kk + 1]));
                    ctx.prof_ms[kk] += ms;
                    ctx.prof_n[kk] += 1;
                }
            }
            if (all_done(pinned)) break;
        }
    } else {
        launch(0);
        launch(1);
        for (long long guard = 0;; ++guard) {
            const int slot = k & 1;
            FBMP_CUDA(cudaEventSynchronize(ev[slot]));
            if (all_done(pinned + slot * N) || guard > max_graphs) break;
            launch(slot);
            ++k;
        }
    }
    trace("cg: iterate");
    for (auto& e : pev) cudaEventDestroy(e);
    FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
    host_state.resize(N);
    FBMP_CUDA(cudaMemcpy(host_state.data(), B.st, sizeof(CgState) * N, cudaMemcpyDeviceToHost));
    if (prof) cudaGraphExecDestroy(exec);
    trace("cg: teardown");
}

void cg_solve(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_guide, const double* d_x,
              CgBuffers& B, int max_iters, double cg_tol, std::vector<CgState>& host_state) {
    cg_solve_t<double>(ctx, G, d_taps, d_guide, d_guide, d_x, B, max_iters, cg_tol, host_state);
}

void cg_solve_f32(Context& ctx, const PsGeo& G, const float* d_taps, const double* d_guide64, const float* d_guide,
                  const float* d_x, CgBuffersT<float>& B, int max_iters, double cg_tol,
                  std::vector<CgState>& host_state) {
    cg_solve_t<float>(ctx, G, d_taps, d_guide64, d_guide, d_x, B, max_iters, cg_tol, host_state);
}

namespace {
template <class A, class B>
__global__ void k_convert(const A* __restrict__ in, long long n, B* __restrict__ out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = static_cast<B>(in[i]);
}
}  // namespace
void to_f32(Context& ctx, const double* d_in, long long n, float* d_out) {
    k_convert<double, float><<<grid1d(ctx, n), 256, 0, ctx.stream>>>(d_in, n, d_out);
    ctx.count();
    check_launch();
}
void to_f64(Context& ctx, const float* d_in, long long n, double* d_out) {
    k_convert<float, double><<<grid1d(ctx, n), 256, 0, ctx.stream>>>(d_in, n, d_out);
    ctx.count();
    check_launch();
}

void guided_filter(Context& ctx, int N, int H, int W, int rw, double eps, const double* d_in, int in_is_z0,
                   const double* d_guide, double* d_a, double* d_c, double* d_v, int cps) {
    const int nb = ceil_div(W, TA) * ceil_div(H, TA);
    const int hz = 2 * rw + (in_is_z0 ? 1 : 0), SZ = TA + 2 * hz, SN = TA + 4 * rw, SA = TA + 2 * rw;
    const size_t sm = (static_cast<size_t>((SZ * SZ + 1) & ~1) + (in_is_z0 ? ((SN * SN + 1) & ~1) : 0) +
                       ((SN * SN + 1) & ~1) + 2 * ((SA * SA + 1) & ~1)) * sizeof(double);
    const int hz2 = 2 * rw + (in_is_z0 ? 1 : 0);
    static const bool tiled = std::getenv("FBMP_GF_TILED") != nullptr;  // A/B: the tiled k_guided2
    if (rw == 1 && !tiled && !d_a && !d_c && W % 2 == 0 && H >= 16 && W >= 64) {
        // row streaming: strips of R rows per (band, channel) item, enough items to fill the SMs
        const int nb = ceil_div(W, GS_BAND);
        const long long slots = static_cast<long long>(ctx.sm_count) * 12;  // warps the registers allow
        const int k = static_cast<int>(std::max(1LL, std::min<long long>(ceil_div(H, 16),
                                                                          slots / std::max(1, nb * N))));
        const int R = ceil_div(H, k), kstrips = ceil_div(H, R);
        const int cpsv = cps > 0 ? cps : N;
        if (in_is_z0)
            k_guided3<true><<<nb * kstrips * N, 32, 0, ctx.stream>>>(H, W, eps, N, cpsv, kstrips, R, d_in, d_guide,
                                                                     d_v);
        else
            k_guided3<false><<<nb * kstrips * N, 32, 0, ctx.stream>>>(H, W, eps, N, cpsv, kstrips, R, d_in, d_guide,
                                                                      d_v);
    } else if (rw == 1 && H >= GTH + hz2 && W >= GTW + hz2) {  // wrap1's range
        const int cpsv = cps > 0 ? cps : N;
        const dim3 grid(ceil_div(W, GTW) * ceil_div(H, GTH), N);
        if (in_is_z0) {
            set_smem(k_guided2<1, true>, GfLay<1, true>::bytes);
            k_guided2<1, true><<<grid, GNT, GfLay<1, true>::bytes, ctx.stream>>>(H, W, eps, cpsv, d_in, d_guide, d_a,
                                                                                 d_c, d_v);
        } else {
            set_smem(k_guided2<1, false>, GfLay<1, false>::bytes);
            k_guided2<1, false><<<grid, GNT, GfLay<1, false>::bytes, ctx.stream>>>(H, W, eps, cpsv, d_in, d_guide,
                                                                                   d_a, d_c, d_v);
        }
    } else {
        check_smem(sm, "guided filter");
        set_smem(k_guided, sm);
        k_guided<<<dim3(nb, N), NTA, sm, ctx.stream>>>(H, W, rw, eps, cps > 0 ? cps : N, d_in, in_is_z0, d_guide,
                                                       d_a, d_c, d_v);
    }
    ctx.count();
    check_launch();
}

void solve_channel_fft(Context& ctx, const PsGeo& G, const double* d_taps, const double* d_x, const double* d_v,
                       const double* d_scale, double* d_out, int* d_flag) {
    const int N = G.N, H = G.H, W = G.W, h = G.h, w = G.w, S = (G.N + G.cps - 1) / G.cps;
    if (G.c > 8) param_error("solve_channel_fft: factor > 8 is not supported by the device solver");
    const size_t P = static_cast<size_t>(H) * W;
    const size_t HS = static_cast<size_t>(H) * (W / 2 + 1), LS = static_cast<size_t>(h) * (w / 2 + 1);
    double* emb = ctx.scratch<double>("fft_emb", P * S);
    double2* bh = ctx.scratch<double2>("fft_bh", HS * S);
    double2* vh = ctx.scratch<double2>("fft_vh", HS * N);
    double2* zh = ctx.scratch<double2>("fft_zh", HS * N);
    double2* xh = ctx.scratch<double2>("fft_xh", LS * N);
    double* zr = ctx.scratch<double>("fft_zr", P * N);
    FBMP_CUDA(cudaMemsetAsync(emb, 0, P * S * sizeof(double), ctx.stream));
    k_embed<<<S, 256, 0, ctx.stream>>>(d_taps, G.n, H, W, emb);
    ctx.count();
    FBMP_CUFFT(cufftExecD2Z(ctx.plan(0, H, W, S), emb, reinterpret_cast<cufftDoubleComplex*>(bh)));
    FBMP_CUFFT(cufftExecD2Z(ctx.plan(0, H, W, N), const_cast<double*>(d_v), reinterpret_cast<cufftDoubleComplex*>(vh)));
    FBMP_CUFFT(cufftExecD2Z(ctx.plan(0, h, w, N), const_cast<double*>(d_x), reinterpret_cast<cufftDoubleComplex*>(xh)));
    double* cosHW = ctx.scratch<double>("fft_cos", static_cast<size_t>(H) + W);
    k_cos_tables<<<ceil_div(H + W, 256), 256, 0, ctx.stream>>>(H, W, cosHW);
    if (G.c <= 4) {
        const dim3 grid(ceil_div(static_cast<long long>(h) * w * AG, AG_NT), S);
        k_alias16<<<grid, AG_NT, 0, ctx.stream>>>(H, W, h, w, G.c, N, G.cps, G.identity, G.lambda, bh, xh, vh, zh,
                                                  cosHW, d_flag);
    } else {
        const int nthreads = 128;
        const dim3 grid(ceil_div(static_cast<long long>(h) * w, nthreads), N);
        k_alias<8><<<grid, nthreads, 0, ctx.stream>>>(H, W, h, w, G.c, G.cps, G.identity, G.lambda, bh, xh, vh, zh,
                                                       cosHW, d_flag);
    }
    ctx.count(2);
    check_launch();
    if (ctx.host_out && N > 1) {
        // per channel: inverse FFT, unscale, then the plane's D2H on the copy stream overlaps the
        // next channel's FFT (the same cuFFT plan kind with batch 1: the same per-plane result)
        if (!ctx.copy_stream) {
            FBMP_CUDA(cudaStreamCreateWithFlags(&ctx.copy_stream, cudaStreamNonBlocking));
            for (auto& e : ctx.copy_ev) FBMP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        for (int ch = 0; ch < N; ++ch) {
            FBMP_CUFFT(cufftExecZ2D(ctx.plan(1, H, W, 1), reinterpret_cast<cufftDoubleComplex*>(zh + ch * HS),
                                    zr + ch * P));
            k_unscale<<<grid1d(ctx, static_cast<long long>(P)), 256, 0, ctx.stream>>>(
                zr + ch * P, static_cast<long long>(P), 1.0 / static_cast<double>(P),
                d_scale ? d_scale + ch / G.cps : nullptr, static_cast<long long>(P), d_out + ch * P);
            ctx.count();
            cudaEvent_t e = ctx.copy_ev[ch & 1];
            FBMP_CUDA(cudaEventRecord(e, ctx.stream));
            FBMP_CUDA(cudaStreamWaitEvent(ctx.copy_stream, e, 0));
            FBMP_CUDA(cudaMemcpyAsync(ctx.host_out + ch * P, d_out + ch * P, P * sizeof(double),
                                      cudaMemcpyDeviceToHost, ctx.copy_stream));
        }
        check_launch();
        return;
    }
    FBMP_CUFFT(cufftExecZ2D(ctx.plan(1, H, W, N), reinterpret_cast<cufftDoubleComplex*>(zh), zr));
    k_unscale<<<grid1d(ctx, static_cast<long long>(P) * N), 256, 0, ctx.stream>>>(
        zr, static_cast<long long>(P) * N, 1.0 / static_cast<double>(P), d_scale, static_cast<long long>(P) * G.cps,
        d_out);
    ctx.count();
    check_launch();
    if (ctx.host_out) {  // one channel: a plain download after the solve
        FBMP_CUDA(cudaMemcpyAsync(ctx.host_out, d_out, P * N * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    }
}

void peak_scale(Context& ctx, const double* d_pan, long long P, const double* d_lrms, long long Np, int S,
                double* d_scale) {
    const int nb = std::min(grid1d(ctx, P + Np), 512);
    double* part = ctx.scratch<double>("peak_part", static_cast<size_t>(nb) * S);
    k_max_partial<<<dim3(nb, S), 256, 0, ctx.stream>>>(d_pan, P, d_lrms, Np, part);
    k_peak_final<<<S, 32, 0, ctx.stream>>>(part, nb, d_scale);
    ctx.count(2);
    check_launch();
}

void scale_copy(Context& ctx, const double* d_in, long long n, const double* d_scale, long long per, double* d_out) {
    k_scale_copy<<<grid1d(ctx, n), 256, 0, ctx.stream>>>(d_in, n, d_scale, per, d_out);
    ctx.count();
    check_launch();
}

void guided_combine(Context& ctx, const double* d_ab, const double* d_cb, const double* d_g, long long n,
                    double* d_out) {
    k_guided_combine<<<grid1d(ctx, n), 256, 0, ctx.stream>>>(d_ab, d_cb, d_g, n, d_out);
    ctx.count();
    check_launch();
}

void laplacian_scaled(Context& ctx, const double* d_in, int H, int W, int N, const double* d_scale, double* d_out) {
    k_lap_scaled<<<dim3(grid1d(ctx, static_cast<long long>(H) * W), N), 256, 0, ctx.stream>>>(d_in, H, W, d_scale,
                                                                                              d_out);
    ctx.count();
    check_launch();
}

void box_mean(Context& ctx, const double* d_in, int H, int W, int N, int radius, double* d_out) {
    k_box_mean<<<dim3(grid1d(ctx, static_cast<long long>(H) * W), N), 256, 0, ctx.stream>>>(d_in, H, W, radius, d_out);
    ctx.count();
    check_launch();
}

void convolve(Context& ctx, const double* d_in, int H, int W, const double* d_taps, int n, int adjoint, double* d_out) {
    k_convolve<<<grid1d(ctx, static_cast<long long>(H) * W), 256, 0, ctx.stream>>>(d_in, H, W, d_taps, n, adjoint,
                                                                                   d_out);
    ctx.count();
    check_launch();
}


// =============================================================================================
// Row-strip decomposition of the CG (SURVEY.md 8(e), config C5 on several GPUs)
// =============================================================================================
// Every strip holds its rows plus `halo` rows above and below (periodic in the global image);
// the CG kernels run unchanged on the padded strip, so rows near the padded edges see wrapped
// garbage -- the halo (>= the operator's dependency depth, 32 rows) keeps it out of the owned
// rows. Dot products sum owned rows only and are combined across strips by an allreduce; the
// CG scalars are then updated by k_dist_* on every strip identically. Per iteration the only
// data exchanged is the halo of r (p_new is recomputed in the halo from r and p_old, both valid
// there). With a communicator the strips are the ranks (NCCL allreduce / send-recv over
// NVLink); without one, the strips are virtual ranks of this process (device copies and an
// in-order sum), which is how the decomposition is tested on one GPU.
namespace {

__global__ void k_dist_sum(double* const* reds, int S, int off, int n) {  // loopback allreduce
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < S; ++k) s += reds[k][off + i];  // strip (rank) order, like a ring sum
        for (int k = 0; k < S; ++k) reds[k][off + i] = s;
    }
}

__global__ void k_dist_init(CgState* st, const double* __restrict__ dred, int N, int max_iters, double cg_tol) {
    const int ch = blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= N) return;
    CgState& S = st[ch];
    const double tot = dred[N + 3 * ch + 1];
    S.rs = tot;
    S.rhs_norm = sqrt(tot);
    S.pp = S.pAp = S.alpha = S.beta = S.zz = S.qq = 0.0;
    S.cg_tol = cg_tol;
    S.t = 0;
    S.iters = 0;
    S.max_iters = max_iters;
    S.done = (S.rhs_norm == 0.0) ? 1 : (max_iters <= 0 ? 3 : 0);
    S.cnt_q = S.cnt_a = S.cnt_u = S.cnt_init = 0;
}

__global__ void k_dist_alpha(CgState* st, const double* __restrict__ dred, int N) {  // pansharpen.cpp:236-244
    const int ch = blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= N || st[ch].done) return;
    CgState& S = st[ch];
    const double pAp = dred[ch];
    S.pAp = pAp;
    if (!(pAp > 0)) {
        S.done = (sqrt(S.rs) <= 1e-12 * S.rhs_norm) ? 1 : 2;
        S.iters = S.t + 1;
    } else {
        S.alpha = S.rs / pAp;
    }
}

__global__ void k_dist_beta(CgState* st, const double* __restrict__ dred, int N) {  // pansharpen.cpp:245-255
    const int ch = blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= N || st[ch].done) return;
    CgState& S = st[ch];
    const double pp = dred[N + 3 * ch], rs_new = dred[N + 3 * ch + 1], zsq = dred[N + 3 * ch + 2];
    S.pp = pp;
    S.zz = zsq;
    const double step = fabs(S.alpha) * sqrt(pp);
    if (step <= S.cg_tol * fmax(sqrt(zsq), 1e-300)) {
        S.done = 1;
        S.iters = S.t + 1;
    } else {
        S.beta = rs_new / S.rs;
        S.rs = rs_new;
        S.t = S.t + 1;
        if (S.t >= S.max_iters) {
            S.done = 3;
            S.iters = S.max_iters;
        }
    }
}

}  // namespace

void cg_solve_strips(Context& ctx, std::vector<StripCg>& SS, const StripComm& comm, int max_iters, double cg_tol,
                     std::vector<CgState>& host_state) {
    const int NS = static_cast<int>(SS.size());
    if (NS < 1) param_error("cg_solve_strips: no strips");
    const PsGeo& G0 = SS[0].G;
    const int N = G0.N, halo = comm.halo;
    if (!fast_ok(G0) || !use_llp()) param_error("distributed CG: needs the fast operator path (radius 1, c in {1,2,4})");
    const size_t P = static_cast<size_t>(G0.H) * G0.W;
    const int W = G0.W, Hp = G0.H;
    const QLaunch q2 = q2_select<true>(G0);
    if (!q2.fn) param_error("distributed CG: kernel side without a specialised K_Q");
    const int nbq = q2.nblk;
    const int nba = ceil_div(G0.W, fast::a4::TA) * ceil_div(G0.H, fast::a4::TA);
    const int nbu = static_cast<int>((P + static_cast<size_t>(NTU) * UPT - 1) / (static_cast<size_t>(NTU) * UPT));
    const int nbA = std::max(nba, ceil_div(G0.W, fast::kl::BAND) * ceil_div(G0.H, fast::kl::RB));
    const size_t sr = static_cast<size_t>(G0.n) * G0.n * sizeof(double);
    set_smem(q2.fn, q2.smem);
    prepare_apply2<true>(G0);
    set_smem(k_rhs<true>, sr);
    // fused chain (K_Q3 -> K_L without d -> K_DU) when every strip qualifies: the strips publish their
    // shares of ||q||^2 + lambda p.w, ||r||^2, ||z||^2 and the k_dist_* kernels close the iteration
    DuFn<double> du = q2.streaming && llp_plan<double>(ctx, G0).pairs ? du_select<double>(G0) : nullptr;
    for (auto& S : SS)
        if (du && du_select<double>(S.G) != du) du = nullptr;
    const size_t sdu = du ? fast::du::smem<double>() : 0;
    const int ntile_du = (G0.W / fast::du::TW) * (G0.H / fast::du::TH);
    int du_ctas = 0;
    if (du) {
        set_smem(du, sdu);
        int per_sm = 0;
        FBMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, du, fast::du::NTD, sdu));
        du_ctas = std::max(1, per_sm) * ctx.sm_count;
    }
    double** d_reds = ctx.scratch<double*>("dist_reds", NS);
    {
        std::vector<double*> h(NS);
        for (int k = 0; k < NS; ++k) h[k] = SS[k].dred;
        FBMP_CUDA(cudaMemcpyAsync(d_reds, h.data(), sizeof(double*) * NS, cudaMemcpyHostToDevice, ctx.stream));
    }
    auto parts = [&](StripCg& S, double*& pi, double*& pq, double*& pa, double*& pu) {
        pi = S.B.part;
        pq = pi + static_cast<size_t>(N) * nba;
        pa = pq + static_cast<size_t>(N) * (nbq + static_cast<size_t>(S.G.h) * ceil_div(S.G.w, 64));  // K_Q3: ||p||^2, ||q||^2 partials
        pu = pa + static_cast<size_t>(N) * nbA;
    };
    auto allreduce = [&](int off, int n) {
        if (comm.nccl) {
            for (auto& S : SS)
                FBMP_NCCL(ncclAllReduce(S.dred + off, S.dred + off, n, ncclDouble, ncclSum,
                                        static_cast<ncclComm_t>(comm.nccl), ctx.stream));
        } else {
            k_dist_sum<<<1, 128, 0, ctx.stream>>>(d_reds, NS, off, n);
            ctx.count();
        }
    };
    // halo of r: top halo <- the neighbour above's last owned rows, bottom <- the one below's first
    auto exchange_r = [&]() {
        const size_t hb = static_cast<size_t>(halo) * W * sizeof(double);
        const int hloc = Hp - 2 * halo;
        if (comm.nccl) {
            auto cm = static_cast<ncclComm_t>(comm.nccl);
            const int up = (comm.rank + comm.nranks - 1) % comm.nranks, dn = (comm.rank + 1) % comm.nranks;
            double* r = SS[0].B.r;
            FBMP_NCCL(ncclGroupStart());
            // per peer, sends and receives match in issue order: the downward flow (my last owned
            // rows -> the top halo below) is issued before the upward flow, so the pairing is right
            // also when up == dn (2 ranks) or up == dn == me (1 rank: the periodic wrap)
            for (int c = 0; c < N; ++c) {
                double* pl = r + c * P;
                FBMP_NCCL(ncclSend(pl + static_cast<size_t>(hloc) * W, halo * W, ncclDouble, dn, cm, ctx.stream));
                FBMP_NCCL(ncclRecv(pl, halo * W, ncclDouble, up, cm, ctx.stream));
                FBMP_NCCL(ncclSend(pl + static_cast<size_t>(halo) * W, halo * W, ncclDouble, up, cm, ctx.stream));
                FBMP_NCCL(ncclRecv(pl + static_cast<size_t>(halo + hloc) * W, halo * W, ncclDouble, dn, cm,
                                   ctx.stream));
            }
            FBMP_NCCL(ncclGroupEnd());
        } else {
            for (int k = 0; k < NS; ++k) {
                const StripCg& A = SS[(k + NS - 1) % NS];  // above
                const StripCg& Bl = SS[(k + 1) % NS];      // below
                for (int c = 0; c < N; ++c) {
                    double* pl = SS[k].B.r + c * P;
                    FBMP_CUDA(cudaMemcpyAsync(pl, A.B.r + c * P + static_cast<size_t>(hloc) * W, hb,
                                              cudaMemcpyDeviceToDevice, ctx.stream));
                    FBMP_CUDA(cudaMemcpyAsync(pl + static_cast<size_t>(halo + hloc) * W,
                                              Bl.B.r + c * P + static_cast<size_t>(halo) * W, hb,
                                              cudaMemcpyDeviceToDevice, ctx.stream));
                }
            }
        }
    };
    // init: rhs = B^T U x (r), z = 0, p_old = 0; rs = ||rhs||^2 over all owned rows
    for (auto& S : SS) {
        FBMP_CUDA(cudaMemsetAsync(S.B.st, 0, sizeof(CgState) * N, ctx.stream));
        double *pi, *pq, *pa, *pu;
        parts(S, pi, pq, pa, pu);
        launch_rhs_init(ctx, S.G, S.taps, S.x, S.B, pi, max_iters, cg_tol);
    }
    allreduce(N, 3 * N);
    for (auto& S : SS) {
        k_dist_init<<<ceil_div(N, 64), 64, 0, ctx.stream>>>(S.B.st, S.dred, N, max_iters, cg_tol);
        ctx.count();
    }
    exchange_r();
    CgState* pinned = static_cast<CgState*>(ctx.pinned(sizeof(CgState) * N));
    const int chunk = 8;
    for (long long it = 0; it <= static_cast<long long>(max_iters) + chunk; it += chunk) {
        for (int j = 0; j < chunk; ++j) {
            for (auto& S : SS) {
                double *pi, *pq, *pa, *pu;
                parts(S, pi, pq, pa, pu);
                q2.fn<<<dim3(nbq, N), q2.threads, q2.smem, ctx.stream>>>(S.G, S.taps, S.B.r, S.B.p, S.B.q, S.B.st, pq, nbq);
                ctx.count();
                if (du) {
                    launch_llp_w<double>(ctx, S.G, S.guide, S.wmu, S.wg, S.B.p, S.B.Ap, S.B.st, pa, false);
                    ctx.count();
                } else {
                    launch_apply2<true>(ctx, S.G, S.taps, S.guide, S.wmu, S.wg, S.B.p, S.B.q, S.B.Ap, S.B.st, pa);
                    ctx.count(2);
                }
            }
            allreduce(0, N);
            for (auto& S : SS) {
                k_dist_alpha<<<ceil_div(N, 64), 64, 0, ctx.stream>>>(S.B.st, S.dred, N);
                double *pi, *pq, *pa, *pu;
                parts(S, pi, pq, pa, pu);
                if (du)
                    du<<<dim3(du_ctas), fast::du::NTD, sdu, ctx.stream>>>(S.G, S.taps, S.B.q, S.B.Ap, S.B.z, S.B.r, S.B.p,
                                                                         S.B.st, pu, ntile_du);
                else
                    k_update<<<dim3(nbu, N), NTU, 0, ctx.stream>>>(S.G, S.B.z, S.B.r, S.B.p, S.B.Ap, S.B.st, pu, nbu);
                ctx.count(2);
            }
            allreduce(N, 3 * N);
            for (auto& S : SS) {
                k_dist_beta<<<ceil_div(N, 64), 64, 0, ctx.stream>>>(S.B.st, S.dred, N);
                ctx.count();
            }
            exchange_r();
        }
        check_launch();
        FBMP_CUDA(cudaMemcpyAsync(pinned, SS[0].B.st, sizeof(CgState) * N, cudaMemcpyDeviceToHost, ctx.stream));
        FBMP_CUDA(cudaStreamSynchronize(ctx.stream));
        bool all = true;
        for (int i = 0; i < N; ++i) all = all && pinned[i].done;
        if (all) break;
    }
    host_state.assign(pinned, pinned + N);
}

}  // namespace fbmp_gpu
