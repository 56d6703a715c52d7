// cg_fast.cuh -- specialised CG operator kernels (window radius 1, c in {1,2,4}, images >= 64).
//
// K_Q2: q = D B p with the kernel side N_ and factor CF known at compile time. The HR tile
//       region is split into CF x CF sampling phases in shared memory; every tap becomes an
//       immediate-offset shared load shared by two vertically adjacent LR points (common
//       sub-expressions of the unrolled loop), taps are broadcast reads.
// K_A:  B^T U q + lambda L M L p for all channels of a scene in one CTA (the guide tile and
//       its per-window statistics are loaded once), the matting operator as separable 3x3
//       box sums:  (M s)_m = n_m s_m - box(c1)_m - I_m box(a)_m  with per-window
//       a_k = g_k (box(I s)_k / 9 - mu_k box(s)_k / 9),  c1_k = [k interior](box(s)_k/9 - mu_k a_k),
//       g_k = [k interior] / (eps/9 + var_k)  (pansharpen.cpp:128-164 regrouped), and the data
//       term gathered per sampling phase so that taps are uniform across a warp.
#pragma once
#include <type_traits>

#include "pansharpen.cuh"

#ifndef FBMP_KQ_KB
#define FBMP_KQ_KB 4  // K_Q: CF-wide runs of r and p_old in flight per thread
#endif

namespace fbmp_gpu {
namespace fast {

constexpr int NT = 256;

__host__ __device__ constexpr int pstride(int s) { return s + ((4 - s % 16) + 16) % 16; }
__host__ __device__ constexpr int cfloordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ int wrap_once(int a, int m) { return a < 0 ? a + m : (a >= m ? a - m : a); }
// Storage / arithmetic type T of the CG vectors: double (the reference precision) or float (the
// fp32 mode: vectors, guide maps and stencils in fp32, every reduction and CG scalar in fp64).
template <class T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <class T> using v2 = typename Vec2<T>::type;
__device__ __forceinline__ double2 mk2(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2 mk2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
// CF-wide runs of T (read-only path for loads)
struct double4_t {
    double2 a, b;
};
template <class T, int CF> struct RunT;
template <> struct RunT<double, 4> { using type = double4_t; };
template <> struct RunT<double, 2> { using type = double2; };
template <> struct RunT<double, 1> { using type = double; };
template <> struct RunT<float, 4> { using type = float4; };
template <> struct RunT<float, 2> { using type = float2; };
template <> struct RunT<float, 1> { using type = float; };
template <class V, class T>
__device__ __forceinline__ V ldv(const T* p);
template <>
__device__ __forceinline__ double ldv<double, double>(const double* p) { return __ldg(p); }
template <>
__device__ __forceinline__ double2 ldv<double2, double>(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
template <>
__device__ __forceinline__ double4_t ldv<double4_t, double>(const double* p) {
    return {__ldg(reinterpret_cast<const double2*>(p)), __ldg(reinterpret_cast<const double2*>(p) + 1)};
}
template <>
__device__ __forceinline__ float ldv<float, float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float2 ldv<float2, float>(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
template <>
__device__ __forceinline__ float4 ldv<float4, float>(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void unpack(double x, double* v) { v[0] = x; }
__device__ __forceinline__ void unpack(double2 x, double* v) { v[0] = x.x; v[1] = x.y; }
__device__ __forceinline__ void unpack(double4_t x, double* v) { v[0] = x.a.x; v[1] = x.a.y; v[2] = x.b.x; v[3] = x.b.y; }
__device__ __forceinline__ void unpack(float x, float* v) { v[0] = x; }
__device__ __forceinline__ void unpack(float2 x, float* v) { v[0] = x.x; v[1] = x.y; }
__device__ __forceinline__ void unpack(float4 x, float* v) { v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; }
template <int K, class T>
__device__ __forceinline__ void stv(T* p, const T (&v)[K]) {
    if constexpr (K == 1) {
        *p = v[0];
    } else if constexpr (K == 4 && std::is_same<T, float>::value) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int u = 0; u < K; u += 2) st2(p + u, mk2(v[u], v[u + 1]));
    }
}

// ------------------------------------------------------------------------------------------
// per-scene guide statistics (pansharpen.cpp:128-139, :152-155):
//   mu_k = box_mean(I)_k, g_k = 1 / (eps/9 + var_k) on interior centres, 0 elsewhere
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_guide_stats(const double* __restrict__ guide, int H, int W, int rw, double eps,
                              T* __restrict__ mu, T* __restrict__ gk) {
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
        mu[blockIdx.y * P + e] = static_cast<T>(m);
        gk[blockIdx.y * P + e] = static_cast<T>(g);
    }
}

// ------------------------------------------------------------------------------------------
// K_Q2
// ------------------------------------------------------------------------------------------
template <int N_, int CF, int MJ_ = 4>
struct QGeo {
    static constexpr int C = (N_ - 1) / 2;
    static constexpr int g = (C + CF - 1) / CF;
    static constexpr int NTH = 128;                        // 4 warps
    static constexpr int MJ = MJ_;                         // LR columns per thread
    static constexpr int TH = 32, TW = MJ * (NTH / 32);    // lane = LR row, warp = 4 LR columns
    static constexpr int PW = TW + 2 * g, PH = TH + 2 * g; // phase-plane extent (LR)
    static constexpr int PWS = PW | 1;                     // odd row stride: lanes (rows) hit distinct banks
    static constexpr int PS = pstride(PWS * PH);
    static constexpr int SRW = CF * PW, SRH = CF * PH;
    static constexpr int KOFF = ((N_ * N_ + 1) / 2) * 2;
    static constexpr size_t smem = (KOFF + static_cast<size_t>(CF) * CF * PS) * sizeof(double);
};

// K_Q: p = r + beta p_old (pansharpen.cpp:254) and q = D B p (pansharpen.cpp:218-223, first
// half) at every LR point, plus ||p||^2. The HR region of the tile (+ halo) is split into CF x CF
// sampling-phase planes in shared memory; tap (a, b) of LR point (i, j) reads plane
// ((CF g - a) mod CF, (CF g - b) mod CF) at (i + (CF g - a) div CF, j + (CF g - b) div CF).
// A lane owns one LR row and MJ consecutive LR columns: every plane value loaded feeds up to MJ
// points and every (broadcast) tap MJ FMAs.
template <int N_, int CF, bool CG, int MJ_ = 4, class T = double>
__global__ void __launch_bounds__(QGeo<N_, CF, MJ_>::NTH, 3) k_q2(PsGeo G, const T* __restrict__ taps,
                                                             const T* __restrict__ src,
                                                             T* __restrict__ pbuf, T* __restrict__ q,
                                                             CgState* st, double* __restrict__ part, int nblk) {
    using Q = QGeo<N_, CF, MJ_>;
    constexpr int NQ = Q::NTH;
    __shared__ double red[NQ / 32 + 1];
    extern __shared__ __align__(16) unsigned char smraw[];
    T* sm = reinterpret_cast<T*>(smraw);
    const int ch = blockIdx.y;
    const T* tp = taps + static_cast<size_t>(ch / G.cps) * N_ * N_;
    T* sk = sm;
    for (int e = threadIdx.x; e < N_ * N_; e += NQ) sk[e] = tp[e];
    int t = 0;
    T beta = 0;
    if (CG) {
        pdl_wait();  // r, beta and the flags come from K_U
        pdl_trigger();
        if (st[ch].done) return;
        t = st[ch].t;
        beta = t ? static_cast<T>(st[ch].beta) : T(0);
    }
    const int H = G.H, W = G.W;
    const size_t P = static_cast<size_t>(H) * W;
    const T* rc = src + ch * P;
    const T* pold = CG ? pbuf + (static_cast<size_t>((t + 1) & 1) * G.N + ch) * P : nullptr;
    T* pnew = CG ? pbuf + (static_cast<size_t>(t & 1) * G.N + ch) * P : nullptr;
    const int ntx = (G.w + Q::TW - 1) / Q::TW;
    const int tyb = blockIdx.x / ntx, txb = blockIdx.x - tyb * ntx;
    const int i0 = tyb * Q::TH, j0 = txb * Q::TW;
    T* planes = sm + Q::KOFF;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int R0 = CF * (i0 - Q::g), C0 = CF * (j0 - Q::g);
    constexpr int own_r0 = CF * Q::g, own_r1 = CF * (Q::g + Q::TH);
    double pp = 0.0;
    // region load in runs of CF consecutive HR columns (one LR column, all column phases): the
    // run start is a multiple of CF in a row of W = w CF, so a run never wraps and its loads and
    // stores are CF-wide vectors; each thread keeps KB runs of r and p_old in flight
    using VT = typename RunT<T, CF>::type;
    constexpr int RUNS = Q::SRH * Q::PW;
    constexpr int KB = FBMP_KQ_KB;
    for (int e0 = 0; e0 < RUNS; e0 += NQ * KB) {
        VT vr[KB], vp[KB];
        size_t gi[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int e = e0 + k * NQ + threadIdx.x;
            const int rr = e / Q::PW, jc = e - rr * Q::PW;
            gi[k] = static_cast<size_t>(wrap_once(R0 + rr, H)) * W + wrap_once(C0 + CF * jc, W);
            if (e < RUNS) {
                vr[k] = ldv<VT, T>(rc + gi[k]);
                if (CG) vp[k] = ldv<VT, T>(pold + gi[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int e = e0 + k * NQ + threadIdx.x;
            if (e >= RUNS) break;
            const int rr = e / Q::PW, jc = e - rr * Q::PW;
            T v[CF];
            unpack(vr[k], v);
            if (CG) {
                T o[CF];
                unpack(vp[k], o);
#pragma unroll
                for (int u = 0; u < CF; ++u) v[u] = v[u] + o[u] * beta;  // pansharpen.cpp:254
                if (rr >= own_r0 && rr < own_r1 && jc >= Q::g && jc < Q::g + Q::TW && R0 + rr < H && C0 + CF * jc < W) {
                    stv(pnew + gi[k], v);
                    if (R0 + rr >= G.rlo && R0 + rr < G.rhi) {  // rows owned by this strip
#pragma unroll
                        for (int u = 0; u < CF; ++u) pp += static_cast<double>(v[u]) * v[u];
                    }
                }
            }
            T* pl = planes + ((rr % CF) * CF) * Q::PS + (rr / CF) * Q::PWS + jc;
#pragma unroll
            for (int u = 0; u < CF; ++u) pl[u * Q::PS] = v[u];
        }
    }
    __syncthreads();
    // points (i0 + lane, j0 + MJ warp + m), m < MJ
    constexpr int MJ = Q::MJ;
    const T* base = planes + lane * Q::PWS + MJ * warp;
    T acc[MJ];
#pragma unroll
    for (int m = 0; m < MJ; ++m) acc[m] = 0;
    constexpr int G4 = CF * Q::g;
    constexpr int JMAX = (G4 + Q::C) / CF + 1;
#pragma unroll
    for (int a = -Q::C; a <= Q::C; ++a) {
        const int ra = G4 - a;  // >= 0; constants once unrolled
        const int pr = ra % CF, ir = ra / CF;
        const T* krow = sk + (a + Q::C) * N_ + Q::C;
#pragma unroll
        for (int pc = 0; pc < CF; ++pc) {
            // column offsets jo with tap b = G4 - pc - CF jo in [-C, C]
            const int jlo = (G4 - pc - Q::C + CF - 1) / CF, jhi = (G4 - pc + Q::C) / CF;  // G4 - pc - C > -CF
            const T* prow = base + (pr * CF + pc) * Q::PS + ir * Q::PWS;
            T v[JMAX + MJ];
#pragma unroll
            for (int x = 0; x < JMAX + MJ; ++x)
                if (x >= jlo && x <= jhi + MJ - 1) v[x] = prow[x];
#pragma unroll
            for (int jo = 0; jo < JMAX; ++jo) {
                if (jo >= jlo && jo <= jhi) {
                    const T kv = krow[G4 - pc - CF * jo];
#pragma unroll
                    for (int m = 0; m < MJ; ++m) acc[m] = fma(kv, v[jo + m], acc[m]);
                }
            }
        }
    }
    const int i = i0 + lane;
    T* qc = q + static_cast<size_t>(ch) * G.h * G.w;
    if (i < G.h) {
#pragma unroll
        for (int m = 0; m < MJ; ++m) {
            const int j = j0 + MJ * warp + m;
            if (j < G.w) qc[static_cast<size_t>(i) * G.w + j] = acc[m];
        }
    }
    if (CG) {
        const double bs = block_sum<NQ>(pp, red);
        if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
        if (elect_last_block(&st[ch].cnt_q, nblk)) {
            const double tot = sum_partials<NQ>(part + static_cast<size_t>(ch) * nblk, nblk, 1, red);
            if (threadIdx.x == 0) {
                if (G.dred) G.dred[G.N + 3 * ch] = tot;
                else st[ch].pp = tot;
                st[ch].cnt_q = 0;
            }
        }
    }
}

template <int N_, int CF, int MJ_ = 4>
inline int q2_blocks(const PsGeo& G) {
    using Q = QGeo<N_, CF, MJ_>;
    return ((G.w + Q::TW - 1) / Q::TW) * ((G.h + Q::TH - 1) / Q::TH);
}

// ------------------------------------------------------------------------------------------
// K_Q3 (factor 4): the same q = D B p (+ p update, ||p||^2) as K_Q2, streamed by HR rows.
//
// q(i, j) = sum_{a, b in [-C, C]} k[a + C][b + C] p(4i - a, 4j - b). HR row y = 4s + w (superrow
// s, phase w) feeds the LR rows i = s + d with a = 4d - w in [-C, C] (4 or 5 of them), each by a
// horizontal 17-tap (n-tap) product. A CTA owns a band of TWL = 32 MJ LR columns and a strip of
// LR rows; warp w owns the HR rows of phase w and keeps the partial sums of its open LR rows in
// registers, so an HR row is read from HBM once per band and never revisited. Rows arrive by
// TMA bulk copies (one elected lane, mbarrier per ring slot, D rows ahead); the lane computes
// p = r + beta p_old on the staged row, writes the owned part of p, and splits the row into four
// column-phase planes in shared memory, from which it reads its MJ columns' windows with 16-byte
// loads. A finished LR row is the sum of the four warps' partials (fixed order), formed after the
// superrow's block barrier. Shared memory per CTA ~72 KB (n = 17, MJ = 2, D = 3) against K_Q2's
// 99 KB, and the strip height is chosen by the host to fill the SMs.
// ------------------------------------------------------------------------------------------
#ifndef FBMP_KQ3_D
#define FBMP_KQ3_D 3
#endif
#ifndef FBMP_KQ3_PCU
#define FBMP_KQ3_PCU 2
#endif
#ifndef FBMP_KQ3_MINB
#define FBMP_KQ3_MINB 3  // CTAs per SM the register budget is sized for
#endif
namespace q3 {
constexpr int KQ3_PCU = FBMP_KQ3_PCU;  // unroll of the column-phase loop
constexpr int NW = 4;  // warps per CTA = HR row phases
constexpr int NTH = 32 * NW;
template <int N_, int MJ, class T = double>
struct Geo {
    static constexpr int C = (N_ - 1) / 2;
    static constexpr int g = (C + 3) / 4;             // ceil(C / 4)
    static constexpr int gp = C / 4;                  // floor(C / 4)
    static constexpr int TWL = 32 * MJ;               // LR columns per band
    static constexpr int JW = TWL + 2 * g;            // phase-plane width (LR units)
    static constexpr int RW = 4 * JW;                 // HR columns of a staged row
    static constexpr int NV = MJ + g + gp;            // plane values a lane reads per phase
    static constexpr int NVP = (NV + 1) & ~1;         // rounded up to 16-byte pairs
    static constexpr int PLS = (JW + 1) & ~1;         // plane stride (>= the NVP over-read)
    static constexpr int D = FBMP_KQ3_D;              // ring depth (rows per warp)
    static constexpr int K = g + 2 <= 4 ? 4 : 8;      // partial-row slots (>= g + 2, power of 2)
    // per-warp tap tables tt[pc][u + g][d - DMIN] (zero where |b| > C or d is out of range): the
    // FMA loop reads them at constant offsets, two taps per 16-byte load
    static constexpr int NU = g + gp + 1;
    static constexpr int NAP = ((((3 + C) / 4) + ((C) / 4) + 1) + 1) & ~1;  // >= max_w NA, even
    static constexpr int TT = 4 * NU * NAP;
    static constexpr int O_TT = 0;                        // NW x TT
    static constexpr int O_RING = NW * TT;                // NW x D x {r, p_old} x RW
    static constexpr int O_PL = O_RING + NW * D * 2 * RW; // NW x 4 x PLS
    static constexpr int O_SLOT = O_PL + NW * 4 * PLS;    // K x NW x TWL (the raw n x n taps until
                                                          // the tables are built)
    static constexpr int O_BAR = sizeof(T) == 8 ? O_SLOT + K * NW * TWL  // NW x D mbarriers (8-byte aligned)
                                                : (O_SLOT + K * NW * TWL + 1) & ~1;
    static constexpr size_t smem = static_cast<size_t>(O_BAR) * sizeof(T) + static_cast<size_t>(NW * D) * 8;
    static_assert(N_ * N_ <= K * NW * TWL, "raw taps fit in the partial-row slots");
    static_assert(TWL - MJ + NVP <= PLS, "plane over-read");
};

__device__ __forceinline__ unsigned int saddr(const void* p) {
    return static_cast<unsigned int>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned int bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned int parity) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}\n" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
template <class T>
__device__ __forceinline__ void bulk_g2s(T* dst, const T* src, unsigned int bytes, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(b))
                 : "memory");
}

template <class T>
struct Args {
    const T* rc;    // r (CG) or p (operator) plane of the channel
    const T* pold;  // p_old plane (CG)
    T* pnew;        // p plane written (CG)
    T* qc;          // q plane of the channel
    double* qrow;   // ||q||^2 partials of the channel's (LR row, band) segments, at this band
    int nbands;
    T beta;
    int H, W, h, w, rlo, rhi;
    int i0, i1, j0;      // strip rows [i0, i1), band origin
    int s0, s1;          // superrows
};

// one warp's stream of HR rows y = 4 s + WP, s in [s0, s1)
template <int N_, int MJ, bool CG, int WP, class T>
__device__ __forceinline__ double rows(const Args<T>& A, const T* sk, T* tt, T* ring, T* pl,
                                       T* slots, unsigned long long* bar, int lane, int warp, double& qq) {
    using Q = Geo<N_, MJ, T>;
    constexpr int C = Q::C, g = Q::g, gp = Q::gp, RW = Q::RW, PLS = Q::PLS, TWL = Q::TWL, D = Q::D, K = Q::K;
    constexpr int DMIN = -((C - WP) / 4);  // ceil((WP - C) / 4)
    constexpr int DMAX = (WP + C) / 4;
    constexpr int NA = DMAX - DMIN + 1;
    const int H = A.H, W = A.W;
    const int col0 = 4 * (A.j0 - g);
    const unsigned int row_bytes = (CG ? 2u : 1u) * RW * sizeof(T);
    const int yo0 = 4 * A.i0, yo1 = min(4 * A.i1, H);
    const int xo_hi = min(4 * TWL, W - 4 * A.j0);
    // the column split of a staged row at the periodic wrap is the same for every row (at most
    // three pieces): lane k < ncp issues copy k = (array, piece) of every row, so a row's copies
    // go out in parallel; the staged rows are consecutive superrows, so the image row advances
    // by 4 (mod H) per issue
    int ncp = 0;
    const T* csrc = nullptr;
    unsigned int cdst = 0, cbytes = 0;
    {
        int start = col0 % W;
        if (start < 0) start += W;
        int off = 0;
        for (int rem = RW, np_ = 0; rem > 0 && np_ < 3; ++np_) {
            const int len = min(rem, W - start);
#pragma unroll
            for (int a = 0; a < (CG ? 2 : 1); ++a) {
                const int k = a * 3 + np_;
                if (lane == k) {
                    csrc = (a == 0 ? A.rc : A.pold) + start;
                    cdst = saddr(ring + a * RW + off);
                    cbytes = static_cast<unsigned int>(len) * sizeof(T);
                }
            }
            ncp = np_ + 1;
            off += len;
            rem -= len;
            start = 0;
        }
    }
    const bool copier = lane < 3 * (CG ? 2 : 1) && (lane % 3) < ncp;
    const unsigned int bar0 = saddr(bar);
    int yw_next = (4 * A.s0 + WP) % H;  // image row of the next staged superrow
    if (yw_next < 0) yw_next += H;
    auto issue = [&](int slot) {  // warp-collective
        const unsigned int b = bar0 + slot * 8u;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(row_bytes) : "memory");
        if (copier)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             cdst + static_cast<unsigned int>(slot * 2 * RW * sizeof(T))),
                         "l"(csrc + static_cast<size_t>(yw_next) * W), "r"(cbytes), "r"(b)
                         : "memory");
        yw_next += 4;
        if (yw_next >= H) yw_next -= H;
    };
    for (int k = 0; k < D; ++k)
        if (A.s0 + k < A.s1) issue(k);
    // the warp's tap table (built while the first rows are in flight)
    for (int e = lane; e < Q::TT; e += 32) {
        const int pc = e / (Q::NU * Q::NAP), ui = (e / Q::NAP) % Q::NU, dd = e % Q::NAP;
        const int d = DMIN + dd, b = -(4 * (ui - g) + pc);
        tt[e] = (d <= DMAX && b >= -C && b <= C) ? sk[(4 * d - WP + C) * N_ + (b + C)] : T(0);
    }
    __syncthreads();  // every table is built: the raw taps' space goes to the partial-row slots
    T acc[NA][MJ];
#pragma unroll
    for (int d = 0; d < NA; ++d)
#pragma unroll
        for (int m = 0; m < MJ; ++m) acc[d][m] = 0;
    double pp = 0.0;
    const T* plb = pl + MJ * lane;
    for (int s = A.s0; s < A.s1; ++s) {
        const int k = s - A.s0;
        const int slot = k % D;
        mbar_wait(bar + slot, static_cast<unsigned int>((k / D) & 1));
        const int y = 4 * s + WP;
        const T* rr = ring + slot * 2 * RW;
        // p = r + beta p_old on the staged row; owned part -> p, all of it -> phase planes
        {
            const bool own_row = CG && y >= yo0 && y < yo1;
            const bool dot_row = own_row && y >= A.rlo && y < A.rhi;
            T* prow = nullptr;
            if (CG) prow = A.pnew + static_cast<size_t>(own_row ? y : 0) * W + 4 * A.j0 - 4 * g;
            // all ring loads first: the plane / p stores below cannot be proven disjoint from the
            // ring, so loads left inside the loop would wait for every preceding store
            constexpr int NKK = (RW + 63) / 64;
            v2<T> vv[NKK], oo[NKK];
#pragma unroll
            for (int kk = 0; kk < NKK; ++kk) {
                const int e = 2 * lane + 64 * kk;
                if (e < RW) {
                    vv[kk] = ld2(rr + e);
                    if (CG) oo[kk] = ld2(rr + RW + e);
                }
            }
#pragma unroll
            for (int kk = 0; kk < NKK; ++kk) {
                const int e = 2 * lane + 64 * kk;
                if (e < RW) {
                    v2<T> v = vv[kk];
                    if (CG) {
                        const v2<T> o = oo[kk];
                        v.x = v.x + o.x * A.beta;  // pansharpen.cpp:254
                        v.y = v.y + o.y * A.beta;
                        const int xr = e - 4 * g;
                        if (own_row && xr >= 0 && xr < xo_hi) {
                            st2(prow + e, v);
                            if (dot_row) {
                                pp += static_cast<double>(v.x) * static_cast<double>(v.x);
                                pp += static_cast<double>(v.y) * static_cast<double>(v.y);
                            }
                        }
                    }
                    pl[(e & 3) * PLS + (e >> 2)] = v.x;
                    pl[((e & 3) + 1) * PLS + (e >> 2)] = v.y;
                }
            }
        }
        __syncwarp();
        if (s + D < A.s1) {  // the slot is free again: stage the row D superrows ahead
            fence_proxy_async();
            issue(slot);
        }
        // contributions of row y to LR rows s + d, d in [DMIN, DMAX]: for every accumulator the
        // (pc, u) order is ascending; the zero taps of the table (|b| > C) add exact zeros
#pragma unroll KQ3_PCU
        for (int pc = 0; pc < 4; ++pc) {
            T v[Q::NVP];
#pragma unroll
            for (int o = 0; o < Q::NVP; o += 2) {
                const v2<T> t2 = ld2(plb + pc * PLS + o);
                v[o] = t2.x;
                v[o + 1] = t2.y;
            }
            const T* tpc = tt + pc * (Q::NU * Q::NAP);
#pragma unroll
            for (int ui = 0; ui < Q::NU; ++ui) {
                T kv[Q::NAP];
#pragma unroll
                for (int dd = 0; dd < NA; dd += 2) {
                    const v2<T> k2 = ld2(tpc + ui * Q::NAP + dd);
                    kv[dd] = k2.x;
                    kv[dd + 1] = k2.y;
                }
#pragma unroll
                for (int dd = 0; dd < NA; ++dd)
#pragma unroll
                    for (int m = 0; m < MJ; ++m) acc[dd][m] = fma(kv[dd], v[m + ui], acc[dd][m]);
            }
        }
        // LR row s + DMIN is complete for this warp: publish its partial, shift the window
        {
            T* sl = slots + ((s + DMIN) & (K - 1)) * (NW * TWL) + WP * TWL + MJ * lane;
#pragma unroll
            for (int m = 0; m < MJ; m += 2) st2(sl + m, mk2(acc[0][m], acc[0][m + 1]));
#pragma unroll
            for (int d = 0; d + 1 < NA; ++d)
#pragma unroll
                for (int m = 0; m < MJ; ++m) acc[d][m] = acc[d + 1][m];
#pragma unroll
            for (int m = 0; m < MJ; ++m) acc[NA - 1][m] = 0;
        }
        __syncthreads();
        // LR row s - g has all four partials
        const int i = s - g;
        if (warp == (s & 3) && i >= A.i0 && i < A.i1) {
            const T* sb = slots + (i & (K - 1)) * (NW * TWL) + MJ * lane;
            const int j = A.j0 + MJ * lane;
#pragma unroll
            for (int m = 0; m < MJ; m += 2) {
                const v2<T> a0 = ld2(sb + m), a1 = ld2(sb + TWL + m), a2 = ld2(sb + 2 * TWL + m),
                            a3 = ld2(sb + 3 * TWL + m);
                const v2<T> val = mk2(((a0.x + a1.x) + a2.x) + a3.x, ((a0.y + a1.y) + a2.y) + a3.y);
                if (j + m + 1 < A.w) {
                    st2(A.qc + static_cast<size_t>(i) * A.w + j + m, val);
                    // ||q||^2 = p . B^T U D B p (the data part of p.Ap on the fused K_L / K_DU path)
                    if (CG) qq += static_cast<double>(val.x) * static_cast<double>(val.x) +
                                  static_cast<double>(val.y) * static_cast<double>(val.y);
                } else if (j + m < A.w) {
                    A.qc[static_cast<size_t>(i) * A.w + j + m] = val.x;
                    if (CG) qq += static_cast<double>(val.x) * static_cast<double>(val.x);
                }
            }
            if (CG) {  // one partial per (LR row, band): the ||q||^2 tree does not depend on the strips
                const double rq = warp_sum(qq);
                if (lane == 0) A.qrow[static_cast<size_t>(i) * A.nbands] = rq;
                qq = 0.0;
            }
        }
    }
    return pp;
}
}  // namespace q3

template <int N_, int MJ, bool CG, class T = double>
__global__ void __launch_bounds__(q3::NTH, FBMP_KQ3_MINB) k_q3(PsGeo G, const T* __restrict__ taps,
                                                   const T* __restrict__ src, T* __restrict__ pbuf,
                                                   T* __restrict__ q, CgState* st, double* __restrict__ part,
                                                   int nblk) {
    using Q = q3::Geo<N_, MJ, T>;
    __shared__ double red[2 * (q3::NW + 1)];
    extern __shared__ __align__(16) unsigned char smraw[];
    T* sm = reinterpret_cast<T*>(smraw);
    const int ch = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T* tp = taps + static_cast<size_t>(ch / G.cps) * N_ * N_;
    T* sk = sm + Q::O_SLOT;  // raw taps (the partial-row slots take over after the tables)
    for (int e = threadIdx.x; e < N_ * N_; e += q3::NTH) sk[e] = tp[e];
    q3::Args<T> A;
    A.beta = 0;
    int t = 0;
    if (CG) {
        pdl_wait();  // r, beta and the flags come from K_U
        pdl_trigger();
        if (st[ch].done) return;
        t = st[ch].t;
        A.beta = t ? static_cast<T>(st[ch].beta) : T(0);
    }
    A.H = G.H;
    A.W = G.W;
    A.h = G.h;
    A.w = G.w;
    A.rlo = G.rlo;
    A.rhi = G.rhi;
    const size_t P = static_cast<size_t>(G.H) * G.W;
    A.rc = src + ch * P;
    A.pold = CG ? pbuf + (static_cast<size_t>((t + 1) & 1) * G.N + ch) * P : nullptr;
    A.pnew = CG ? pbuf + (static_cast<size_t>(t & 1) * G.N + ch) * P : nullptr;
    A.qc = q + static_cast<size_t>(ch) * G.h * G.w;
    const int nbands = (G.w + Q::TWL - 1) / Q::TWL;
    const int nstrips = nblk / nbands;
    const int SR = (G.h + nstrips - 1) / nstrips;
    const int band = blockIdx.x % nbands, strip = blockIdx.x / nbands;
    A.j0 = band * Q::TWL;
    A.nbands = nbands;
    A.qrow = part + static_cast<size_t>(G.N) * nblk + static_cast<size_t>(ch) * G.h * nbands + band;
    A.i0 = strip * SR;
    A.i1 = min(A.i0 + SR, G.h);
    A.s0 = A.i0 - Q::g;
    A.s1 = A.i1 + Q::g;
    if (A.i1 <= A.i0) A.s1 = A.s0;  // empty strip: no rows, still counted in the p.p election
    T* ring = sm + Q::O_RING + warp * (Q::D * 2 * Q::RW);
    T* pl = sm + Q::O_PL + warp * 4 * Q::PLS;
    T* slots = sm + Q::O_SLOT;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + Q::O_BAR) + warp * Q::D;
    if (lane == 0) {
        for (int k = 0; k < Q::D; ++k) q3::mbar_init(bar + k, 1);
        q3::mbar_fence_init();
    }
    __syncthreads();  // taps and barriers
    T* tt = sm + Q::O_TT + warp * Q::TT;
    double pp, qq = 0.0;
    switch (warp) {
    case 0: pp = q3::rows<N_, MJ, CG, 0, T>(A, sk, tt, ring, pl, slots, bar, lane, warp, qq); break;
    case 1: pp = q3::rows<N_, MJ, CG, 1, T>(A, sk, tt, ring, pl, slots, bar, lane, warp, qq); break;
    case 2: pp = q3::rows<N_, MJ, CG, 2, T>(A, sk, tt, ring, pl, slots, bar, lane, warp, qq); break;
    default: pp = q3::rows<N_, MJ, CG, 3, T>(A, sk, tt, ring, pl, slots, bar, lane, warp, qq); break;
    }
    if (CG) {
        // ||p||^2 partials at part[ch][blk]; ||q||^2 partials per (LR row, band) behind them
        const double bs = block_sum<q3::NTH>(pp, red);
        if (threadIdx.x == 0) part[static_cast<size_t>(ch) * nblk + blockIdx.x] = bs;
        if (elect_last_block(&st[ch].cnt_q, nblk)) {
            const int nseg = G.h * nbands;
            const double* pq2 = part + static_cast<size_t>(G.N) * nblk + static_cast<size_t>(ch) * nseg;
            double s0 = 0.0, s1 = 0.0;
            for (int i = threadIdx.x; i < nblk; i += q3::NTH) s0 += __ldcg(part + static_cast<size_t>(ch) * nblk + i);
            // (row strips: the segments of the owned LR rows only; every strip tiles them the same way)
            const int seg_lo = G.dred ? (G.rlo / 4) * nbands : 0, seg_hi = G.dred ? min(nseg, (G.rhi / 4) * nbands) : nseg;
            for (int i = seg_lo + threadIdx.x; i < seg_hi; i += q3::NTH) s1 += __ldcg(pq2 + i);
            const double2 tot = block_sum2<q3::NTH>(s0, s1, red);
            if (threadIdx.x == 0) {
                if (G.dred) G.dred[G.N + 3 * ch] = tot.x;
                else st[ch].pp = tot.x;
                st[ch].qq = tot.y;
                st[ch].cnt_q = 0;
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// K_A (radius 1): one CTA = one 32 x 32 output tile x the channels [group*cpc, +cpc) of a scene
// ------------------------------------------------------------------------------------------
namespace a4 {
constexpr int TA = 32;
constexpr int MAXN = 21;      // kernel side limit of the fast path
constexpr int MAXTAP = 442;   // n <= 21, even
constexpr int MAXCPC = 32;    // channels per CTA (per-channel warp partials of p.Ap)
// region widths: p on R+4, I / s / I*s on R+3, window statistics on R+2, M s on R+1
constexpr int RP = TA + 8, RI = TA + 6, RK = TA + 4, RM = TA + 2;
// padded row strides (even: 16-byte column pairs). tools/bank_sim.py: with the stage thread
// maps below they make the 128-bit accesses of S1, S3, S5 conflict-free (S2 keeps 1.3x).
constexpr int SP = 50, SI = 50, SK = 38, SMS = 38, SO = TA;
template <int N_, int CF>
struct DT {  // zero-padded sub-kernel extent of the data term
    static constexpr int C = (N_ - 1) / 2;
    static constexpr int DLO = -(C / CF);
    static constexpr int DHI = (CF - 1 + C) / CF;
    static constexpr int DM = DHI - DLO + 1;
};
__host__ __device__ constexpr int qwmax(int cf) { return (TA - 1 + 2 * (MAXN / 2)) / cf + 2; }
template <int CF>
struct L {
    static constexpr int QWMAX = qwmax(CF);
    static constexpr int QWP = QWMAX + ((8 - QWMAX % 16) + 16) % 16;   // q row stride
    static constexpr int O_TAPS = 0;
    static constexpr int O_I = O_TAPS + MAXTAP;             // guide on R+3
    static constexpr int O_MU = O_I + RI * SI;              // mu_k on R+2
    static constexpr int O_G = O_MU + RK * SK;              // g_k on R+2
    static constexpr int O_S = O_G + RK * SK;               // s on R+3
    static constexpr int O_M = O_S + RI * SI;               // I*s on R+3, then M s on R+1
    static constexpr int O_Q = O_M + RI * SI;               // q window
    static constexpr int O_U = O_Q + ((QWP * QWMAX + 1) / 2) * 2;  // p on R+4 -> (a, c1) on R+2
    static constexpr int U_SIZE = (RP * SP > 2 * RK * SK) ? RP * SP : 2 * RK * SK;
    static constexpr int O_O = O_U + U_SIZE;                // data term (TA x TA)
    static constexpr int TOTAL = O_O + TA * SO;
    static_assert(RM * SMS <= RI * SI, "M s must fit in the I*s buffer");
    static_assert(O_I % 2 == 0 && O_MU % 2 == 0 && O_G % 2 == 0 && O_S % 2 == 0 && O_M % 2 == 0 &&
                  O_Q % 2 == 0 && O_U % 2 == 0 && O_O % 2 == 0 && (RK * SK) % 2 == 0, "16-byte pair alignment");
    static constexpr size_t smem = TOTAL * sizeof(double);
};
// stage thread maps over column PAIRS: S1 19 pairs x 13 strips x 3 rows, S2 18 x 14 x 3,
// S3 17 x 15 x 3, S5 16 x 16 x 2
static_assert(19 * 13 <= NT && 18 * 14 <= NT && 17 * 15 <= NT && 16 * 16 == NT && TA == 32, "stage maps");
}  // namespace a4

// K_A: Ap = B^T U q + lambda L M L p and, for CG, p.Ap (pansharpen.cpp:218-223, :236-239).
// Per channel: S4 data term, S1 s = L p and I s, S2 window coefficients (a, c1), S3 M s,
// S5 t = L M s and the output. The p.Ap partials of all channels are published once at the end
// of the CTA (one fence, one arrival per channel); the last CTA of a channel reduces them.
template <bool CG, int N_, int CF>
__global__ void __launch_bounds__(NT, 2) k_apply4(PsGeo G, const double* __restrict__ taps,
                                                  const double* __restrict__ guide, const double* __restrict__ wmu,
                                                  const double* __restrict__ wg, const double* __restrict__ pin,
                                                  const double* __restrict__ q, double* __restrict__ out, CgState* st,
                                                  double* __restrict__ part, int nblk) {
    using namespace a4;
    using Lay = a4::L<CF>;
    static_assert(N_ == 0 || CF == 4, "register data term is specialised for factor 4");
    __shared__ double red[NT / 32 + 1];
    __shared__ double wsum[CG ? MAXCPC : 1][NT / 32];
    __shared__ unsigned int last_mask;
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
    double* sO = sm + Lay::O_O;
    const double* tp = taps + static_cast<size_t>(scene) * n * n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int iq0 = floordiv(r0 - C + CF - 1, CF), jq0 = floordiv(c0 - C + CF - 1, CF);
    const int QH = floordiv(r0 + TA - 1 + C, CF) - iq0 + 1, QW = floordiv(c0 + TA - 1 + C, CF) - jq0 + 1;
    constexpr int QS = Lay::QWP;
    using D = DT<(N_ > 0 ? N_ : 1), CF>;
    constexpr int DM = N_ > 0 ? D::DM : 1;
    const int ch_lo = group * G.cpc, ch_hi = min(G.cps, group * G.cpc + G.cpc);
    constexpr int KP = (RP * RP + NT - 1) / NT;
    const int QN = QH * QW;
    constexpr int KQ = (Lay::QWMAX * Lay::QWMAX + NT - 1) / NT;
    double pf_p[KP], pf_q[KQ];
    if (CG && threadIdx.x == 0) last_mask = 0u;
    // per-channel flags of the group, one load per lane (every warp keeps its own copy): done and
    // t are written by K_U and by this kernel's own final election only, so they are stable here
    // and can be read before pdl_wait
    unsigned int active = ch_hi - ch_lo >= 32 ? 0xffffffffu : (1u << (ch_hi - ch_lo)) - 1u;
    int tpar = 0;
    if (CG) {
        const bool mine = lane < ch_hi - ch_lo;
        const CgState* sl = st + scene * G.cps + ch_lo + (mine ? lane : 0);
        const int dn = mine ? sl->done : 1;
        tpar = mine ? (sl->t & 1) : 0;
        active = __ballot_sync(0xffffffffu, !dn);
    }
    // issue the loads of channel `chl`'s p (R+4) and q windows into registers
    auto prefetch = [&](int chl) {
        const int ch = scene * G.cps + chl;
        const double* pp = pin + ch * P;
        if (CG) pp = pin + (static_cast<size_t>(__shfl_sync(0xffffffffu, tpar, chl - ch_lo)) * G.N + ch) * P;
        const double* qc = q + static_cast<size_t>(ch) * G.h * G.w;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const int e = threadIdx.x + k * NT;
            const int y = e / RP, x = e - y * RP;
            pf_p[k] = 0.0;
            if (e < RP * RP && !(G.dbg & 32))
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
        const unsigned int rest = chl - ch_lo < 32 ? active >> (chl - ch_lo) : 0u;
        return rest ? chl + __ffs(rest) - 1 : ch_hi;
    };
    const double* I = guide + scene * P;
    const double* MU = wmu + scene * P;
    const double* GK = wg + scene * P;
    for (int e = threadIdx.x; e < n * n; e += NT) sk[e] = tp[e];
    constexpr int KI = (RI * RI + NT - 1) / NT, KK = (RK * RK + NT - 1) / NT;
    double vi[KI], vm[KK], vg[KK];
#pragma unroll
    for (int k = 0; k < KI; ++k) {
        const int e = threadIdx.x + k * NT;
        const int y = e / RI, x = e - y * RI;
        if (e < RI * RI) vi[k] = __ldg(I + static_cast<size_t>(wrap_once(r0 - 3 + y, H)) * W + wrap_once(c0 - 3 + x, W));
    }
#pragma unroll
    for (int k = 0; k < KK; ++k) {
        const int e = threadIdx.x + k * NT;
        const int y = e / RK, x = e - y * RK;
        const size_t gi = static_cast<size_t>(wrap_once(r0 - 2 + y, H)) * W + wrap_once(c0 - 2 + x, W);
        if (e < RK * RK) {
            vm[k] = __ldg(MU + gi);
            vg[k] = __ldg(GK + gi);
        }
    }
    if (CG) {  // guide and taps are not written by K_Q: their loads overlap K_Q's tail
        pdl_wait();
        pdl_trigger();
    }
    int cur = next_active(ch_lo);
    if (cur < ch_hi) prefetch(cur);  // first channel's p / q in flight with the guide tile
#pragma unroll
    for (int k = 0; k < KI; ++k) {
        const int e = threadIdx.x + k * NT;
        const int y = e / RI, x = e - y * RI;
        if (e < RI * RI) sI[y * SI + x] = vi[k];
    }
#pragma unroll
    for (int k = 0; k < KK; ++k) {
        const int e = threadIdx.x + k * NT;
        const int y = e / RK, x = e - y * RK;
        if (e < RK * RK) {
            sMu[y * SK + x] = vm[k];
            sG[y * SK + x] = vg[k];
        }
    }

    unsigned int processed = 0u;  // local channels this CTA applied the operator to
    for (int chl = cur; chl < ch_hi; chl = cur) {
        const int ch = scene * G.cps + chl;
        __syncthreads();  // previous channel finished with the shared buffers
        double* sP = sU;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const int e = threadIdx.x + k * NT;
            const int y = e / RP, x = e - y * RP;
            if (e < RP * RP) sP[y * SP + x] = pf_p[k];
        }
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
        // own pixels' p for p.Ap in the S5 map (column pair 2 (tid % 16), rows 2 (tid / 16) + {0,1})
        double2 pown[2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
            pown[i] = ld2(sP + (2 * (threadIdx.x >> 4) + i + 4) * SP + 2 * (threadIdx.x & 15) + 4);
        // S4: data term (needs only q; writes its own buffer, so it runs before S1 without a barrier)
        if (N_ > 0 && !(G.dbg & 1)) {
            // thread = (column phase pc, cell column Jc, 4 cell rows, row phase pr): a warp covers
            // 32 consecutive output columns (conflict-free stores; q loads shared by the 4 pc lanes);
            // the zero-padded phase sub-kernel sits in registers, q rows slide through registers
            constexpr int CW4 = TA / CF, RB4 = CW4 / 4;
            const int pc = threadIdx.x % CF;
            const int Jc = (threadIdx.x / CF) % CW4;
            const int rest = threadIdx.x / (CF * CW4);
            const int Ic0 = (rest % RB4) * 4;
            const int pr = rest / RB4;
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
            for (int k = 0; k < 4; ++k) sO[((Ic0 + k) * CF + pr) * SO + Jc * CF + pc] = acc[k];
        } else if (!(G.dbg & 1)) {
            // generic taps: output u = 128 warp + 32 k + lane -> (sampling phase, cell); the phase
            // is uniform across a warp, so taps are broadcast reads
            constexpr int CPR = TA / CF, CPP = CPR * CPR;  // cells per row / per phase
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
                sO[(ci * CF + pr) * SO + cj * CF + pc] = acc;
            }
        }
        // S1-S3 and S5 work on column PAIRS (16-byte shared accesses, conflict-free) and walk short
        // strips of rows with the vertical 3-sums in a register sliding window.
        // S1: s = L p and I*s on R+3
        if (threadIdx.x < 19 * 13 && !(G.dbg & 2)) {
            const int xp = 2 * (threadIdx.x % 19), y0 = 3 * (threadIdx.x / 19);
            double2 a0 = ld2(sP + y0 * SP + xp), a1 = ld2(sP + y0 * SP + xp + 2);        // p rows y, y+1
            double2 b0 = ld2(sP + (y0 + 1) * SP + xp), b1 = ld2(sP + (y0 + 1) * SP + xp + 2);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int y = y0 + i;
                if (y < RI) {
                    const double2 e0 = ld2(sP + (y + 2) * SP + xp), e1 = ld2(sP + (y + 2) * SP + xp + 2);
                    // outputs at p columns xp+1, xp+2 (ops.cpp:70-78 operation order)
                    const double v0 = 4.0 * b0.y - a0.y - e0.y - b0.x - b1.x;
                    const double v1 = 4.0 * b1.x - a1.x - e1.x - b0.y - b1.y;
                    const double2 iv = ld2(sI + y * SI + xp);
                    st2(sS + y * SI + xp, make_double2(v0, v1));
                    st2(sIS + y * SI + xp, make_double2(iv.x * v0, iv.y * v1));
                    a0 = b0; a1 = b1; b0 = e0; b1 = e1;
                }
            }
        }
        __syncthreads();
        // S2: per-window a_k, c1_k on R+2 from 3x3 sums of s and I*s
        double* sA = sU;
        double* sC = sU + RK * SK;
        if (threadIdx.x < 18 * 14 && !(G.dbg & 4)) {
            const int xp = 2 * (threadIdx.x % 18), y0 = 3 * (threadIdx.x / 18);
            auto hpair = [&](const double* a, int y) {  // horizontal 3-sums at columns xp, xp+1
                const double2 u = ld2(a + y * SI + xp), v = ld2(a + y * SI + xp + 2);
                return make_double2(u.x + u.y + v.x, u.y + v.x + v.y);
            };
            double2 s0 = hpair(sS, y0), s1 = hpair(sS, y0 + 1);
            double2 i0 = hpair(sIS, y0), i1 = hpair(sIS, y0 + 1);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int y = y0 + i;
                if (y < RK) {
                    const double2 s2 = hpair(sS, y + 2), i2 = hpair(sIS, y + 2);
                    const double2 mu = ld2(sMu + y * SK + xp), g = ld2(sG + y * SK + xp);
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
                    st2(sA + y * SK + xp, a);
                    st2(sC + y * SK + xp, c);
                    s0 = s1; s1 = s2; i0 = i1; i1 = i2;
                }
            }
        }
        __syncthreads();
        // S3: M s on R+1 = n_m s_m - box(c1) - I_m box(a)
        if (threadIdx.x < 17 * 15 && !(G.dbg & 8)) {
            const int xp = 2 * (threadIdx.x % 17), y0 = 3 * (threadIdx.x / 17);
            auto hpair = [&](const double* a, int y) {
                const double2 u = ld2(a + y * SK + xp), v = ld2(a + y * SK + xp + 2);
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
                if (y < RM) {
                    const double2 a2v = hpair(sA, y + 2), k2 = hpair(sC, y + 2);
                    const int gr = wrap_once(r0 - 1 + y, H);
                    const int nr = max(min(gr + 1, H - 2) - max(gr - 1, 1) + 1, 0);
                    const double2 sv = ld2(sS + (y + 2) * SI + xp + 2), iv = ld2(sI + (y + 2) * SI + xp + 2);
                    double2 m;
                    m.x = static_cast<double>(nr * nc0) * sv.x - (k0.x + k1.x + k2.x) - iv.x * (a0.x + a1.x + a2v.x);
                    m.y = static_cast<double>(nr * nc1) * sv.y - (k0.y + k1.y + k2.y) - iv.y * (a0.y + a1.y + a2v.y);
                    st2(sM + y * SMS + xp, m);  // sM aliases I*s: dead after S2, not read here
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
            double2 a0 = ld2(sM + y0 * SMS + xp), a1 = ld2(sM + y0 * SMS + xp + 2);
            double2 b0 = ld2(sM + (y0 + 1) * SMS + xp), b1 = ld2(sM + (y0 + 1) * SMS + xp + 2);
            const int Cc = c0 + xp;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int y = y0 + i;
                const double2 e0 = ld2(sM + (y + 2) * SMS + xp), e1 = ld2(sM + (y + 2) * SMS + xp + 2);
                const double t0 = 4.0 * b0.y - a0.y - e0.y - b0.x - b1.x;
                const double t1 = 4.0 * b1.x - a1.x - e1.x - b0.y - b1.y;
                const double2 dv = ld2(sO + y * SO + xp);
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
            dotp = warp_sum(dotp);
            if (lane == 0) wsum[chl - ch_lo][warp] = dotp;
            processed |= 1u << (chl - ch_lo);
        }
    }
    if (CG) {
        // publish the block partial of every processed channel; the last arrival reduces it
        __syncthreads();
        const int li = threadIdx.x;
        if (li < ch_hi - ch_lo && ((processed >> li) & 1u)) {
            const int ch = scene * G.cps + ch_lo + li;
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) s += wsum[li][w];
            part[static_cast<size_t>(ch) * nblk + blockIdx.x] = s;
            __threadfence();  // publish the partial before the arrival is counted
            if (atomicAdd(&st[ch].cnt_a, 1u) == static_cast<unsigned int>(nblk) - 1u) {
                __threadfence();
                atomicOr(&last_mask, 1u << li);
            }
        }
        __syncthreads();
        unsigned int mask = last_mask;
        while (mask) {
            const int li2 = __ffs(mask) - 1;
            mask &= mask - 1u;
            const int ch = scene * G.cps + ch_lo + li2;
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

// ------------------------------------------------------------------------------------------
// K_D + K_L: the CG operator split into the data term (tile kernel) and the matting term
// (register-streaming kernel).
//
// K_D: d = B^T U q for all channels of a scene, one CTA per 32 x 32 HR tile (the q window and
//      taps in shared memory, the K_A register-blocked gather), written to the output plane.
// K_L: out = d + lambda L M L p (pansharpen.cpp:218-223) and p.out. One warp owns a band of 24
//      output columns (lanes = 32 consecutive columns incl. a 4-column halo on each side) and
//      walks down a strip of rows; the vertical 3-point stencils keep their rows in registers
//      and the horizontal neighbours come from lane shuffles, so the five operator stages
//      (s = L p, I s, window coefficients (a, c1), M s, L M s) run without shared memory or
//      block barriers. Per output row the warp issues 6 coalesced row loads and 24 32-bit
//      shuffles; the p.out partials are reduced per CTA and the last CTA of a channel forms
//      p.Ap (same state update as K_A).
// ------------------------------------------------------------------------------------------
#ifndef FBMP_KD_MINB
#define FBMP_KD_MINB 2  // K_D CTAs per SM the register budget is sized for
#endif
namespace kl {
template <int CF>
constexpr size_t dterm_smem(int windows = 2) {  // taps | q windows (2 alternating, or one per channel)
    return (a4::MAXTAP + static_cast<size_t>(windows < 2 ? 2 : windows) * a4::L<CF>::QWP * a4::L<CF>::QWMAX) *
           sizeof(double);
}
constexpr int NTL = 32;           // one warp per CTA: every loop bound derives from blockIdx, so
                                  // the compiler sees a convergent warp and emits plain SHFLs
constexpr int BAND = 24;          // output columns per warp
constexpr int HALO = 4;           // L M L has radius 4
constexpr int RB = 16;            // rows per p.out partial (strip heights are multiples of RB, so
                                  // the reduction tree does not depend on the strip partition)
}  // namespace kl

template <bool CG, int N_, int CF, class T = double>
__global__ void __launch_bounds__(NT, FBMP_KD_MINB) k_dterm(PsGeo G, const T* __restrict__ taps, const T* __restrict__ q,
                                                 T* __restrict__ out, const CgState* __restrict__ st) {
    using namespace a4;
    using Lay = a4::L<CF>;
    static_assert(N_ == 0 || CF == 4, "register data term is specialised for factor 4");
    extern __shared__ __align__(16) unsigned char smraw[];   // taps | q window: dterm_smem<CF>()
    T* sm = reinterpret_cast<T*>(smraw);
    const int cgroups = (G.cps + G.cpc - 1) / G.cpc;
    const int scene = blockIdx.y / cgroups, group = blockIdx.y - scene * cgroups;
    const int H = G.H, W = G.W, n = G.n, C = G.C;
    const size_t P = static_cast<size_t>(H) * W;
    const int ntx = (W + TA - 1) / TA;
    const int by = blockIdx.x / ntx, bx = blockIdx.x - by * ntx;
    const int r0 = by * TA, c0 = bx * TA;
    T* sk = sm + Lay::O_TAPS;
    T* sq = sm + MAXTAP;   // q window right after the taps
    const T* tp = taps + static_cast<size_t>(scene) * n * n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int iq0 = floordiv(r0 - C + CF - 1, CF), jq0 = floordiv(c0 - C + CF - 1, CF);
    const int QH = floordiv(r0 + TA - 1 + C, CF) - iq0 + 1, QW = floordiv(c0 + TA - 1 + C, CF) - jq0 + 1;
    constexpr int QS = Lay::QWP;
    using D = DT<(N_ > 0 ? N_ : 1), CF>;
    constexpr int DM = N_ > 0 ? D::DM : 1;
    const int ch_lo = group * G.cpc, ch_hi = min(G.cps, group * G.cpc + G.cpc);
    for (int e = threadIdx.x; e < n * n; e += NT) sk[e] = tp[e];
    unsigned int active = ch_hi - ch_lo >= 32 ? 0xffffffffu : (1u << (ch_hi - ch_lo)) - 1u;
    if (CG) {
        pdl_wait();  // q and the flags come from K_Q
        pdl_trigger();
        const bool mine = lane < ch_hi - ch_lo;
        const int dn = mine ? st[scene * G.cps + ch_lo + lane].done : 1;
        active = __ballot_sync(0xffffffffu, !dn);
    }
    const int QN = QH * QW;
    if constexpr (N_ > 0) {
        // register taps: the q windows of all active channels of the group go to shared memory
        // at once (one barrier), then every thread applies its phase sub-kernel, loaded once, to
        // each channel
        constexpr int QSZ = Lay::QWP * Lay::QWMAX;
        const int na = __popc(active);
        const bool all_active = na == ch_hi - ch_lo;
        // the window has the same extent for every tile (origins are multiples of CF): constant
        // divisors, and its rows / columns wrap at most once
        constexpr int QWC = cfloordiv(TA - 1 + D::C, CF) - cfloordiv(CF - 1 - D::C, CF) + 1;
        constexpr int QNC = QWC * QWC;
        for (int e = threadIdx.x; e < na * QNC; e += NT) {
            const int c = e / QNC, r = e - c * QNC;
            const int a = r / QWC, b = r - a * QWC;
            // c-th active channel (all of them unless some channel of the group has converged)
            const int chl = ch_lo + (all_active ? c : static_cast<int>(__fns(active, 0, c + 1)));
            const T* qc = q + static_cast<size_t>(scene * G.cps + chl) * G.h * G.w;
            sq[c * QSZ + a * QS + b] =
                __ldg(qc + static_cast<size_t>(wrap_once(iq0 + a, G.h)) * G.w + wrap_once(jq0 + b, G.w));
        }
        __syncthreads();
        constexpr int CW4 = TA / CF, RB4 = CW4 / 4;
        const int pc = threadIdx.x % CF;
        const int Jc = (threadIdx.x / CF) % CW4;
        const int rest = threadIdx.x / (CF * CW4);
        const int Ic0 = (rest % RB4) * 4;
        const int pr = rest / RB4;
        T kreg[DM][DM];
#pragma unroll
        for (int a = 0; a < DM; ++a)
#pragma unroll
            for (int b = 0; b < DM; ++b) {
                const int tr = CF * (a + D::DLO) - pr + D::C, tc = CF * (b + D::DLO) - pc + D::C;
                kreg[a][b] = (tr >= 0 && tr < N_ && tc >= 0 && tc < N_) ? sk[tr * N_ + tc] : T(0);
            }
        const int qoff = (r0 / CF + Ic0 - iq0 + D::DLO) * QS + (c0 / CF + Jc - jq0 + D::DLO);
        const int Cc = c0 + Jc * CF + pc;
        // two channels per pass: independent FMA chains interleave (each output keeps its own
        // summation order)
        unsigned int m = active;
        for (int c = 0; m; c += 2) {
            const int chA = ch_lo + __ffs(m) - 1;
            m &= m - 1u;
            const bool two = m != 0u;
            const int chB = two ? ch_lo + __ffs(m) - 1 : chA;
            if (two) m &= m - 1u;
            const T* qa = sq + c * QSZ + qoff;
            const T* qb2 = sq + (two ? c + 1 : c) * QSZ + qoff;
            T acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
            for (int mm = 0; mm < DM + 3; ++mm) {
                T qv[2][DM];
#pragma unroll
                for (int b = 0; b < DM; ++b) {
                    qv[0][b] = qa[mm * QS + b];
                    qv[1][b] = qb2[mm * QS + b];
                }
                // b outer, output row k inner: consecutive FMAs go to 8 different accumulators,
                // each accumulator still sees (mm, b) in ascending order
#pragma unroll
                for (int b = 0; b < DM; ++b)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int a = mm - k;
                        if (a >= 0 && a < DM) {
                            acc[0][k] = fma(kreg[a][b], qv[0][b], acc[0][k]);
                            acc[1][k] = fma(kreg[a][b], qv[1][b], acc[1][k]);
                        }
                    }
            }
            T* oa = out + (scene * G.cps + chA) * P;
            T* ob = out + (scene * G.cps + chB) * P;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int R = r0 + (Ic0 + k) * CF + pr;
                if (R < H && Cc < W) {
                    oa[static_cast<size_t>(R) * W + Cc] = acc[0][k];
                    if (two) ob[static_cast<size_t>(R) * W + Cc] = acc[1][k];
                }
            }
        }
        return;
    }
    constexpr int KQ = (Lay::QWMAX * Lay::QWMAX + NT - 1) / NT;
    T pf[KQ];
    // the next channel's q window is loaded into registers while the current one is computed;
    // the shared window alternates between two buffers (one barrier per channel)
    auto prefetch = [&](int chl) {
        const T* qc = q + static_cast<size_t>(scene * G.cps + chl) * G.h * G.w;
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
            const int e = threadIdx.x + k * NT;
            if (e < QN) {
                const int a = e / QW, b = e - a * QW;
                pf[k] = __ldg(qc + static_cast<size_t>(wrapi(iq0 + a, G.h)) * G.w + wrapi(jq0 + b, G.w));
            }
        }
    };
    int nxt = active ? ch_lo + __ffs(active) - 1 : -1;
    if (nxt >= 0) prefetch(nxt);
    int buf = 0;
    while (nxt >= 0) {
        const int chl = nxt;
        active &= active - 1u;
        const int ch = scene * G.cps + chl;
        T* sqb = sq + buf * (Lay::QWP * Lay::QWMAX);
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
            const int e = threadIdx.x + k * NT;
            if (e < QN) {
                const int a = e / QW, b = e - a * QW;
                sqb[a * QS + b] = pf[k];
            }
        }
        nxt = active ? ch_lo + __ffs(active) - 1 : -1;
        if (nxt >= 0) prefetch(nxt);
        __syncthreads();  // window (and taps) in; the other buffer is free for the next channel
        buf ^= 1;
        T* oc = out + ch * P;
        if (N_ > 0) {
            constexpr int CW4 = TA / CF, RB4 = CW4 / 4;
            const int pc = threadIdx.x % CF;
            const int Jc = (threadIdx.x / CF) % CW4;
            const int rest = threadIdx.x / (CF * CW4);
            const int Ic0 = (rest % RB4) * 4;
            const int pr = rest / RB4;
            T kreg[DM][DM];
#pragma unroll
            for (int a = 0; a < DM; ++a)
#pragma unroll
                for (int b = 0; b < DM; ++b) {
                    const int tr = CF * (a + D::DLO) - pr + D::C, tc = CF * (b + D::DLO) - pc + D::C;
                    kreg[a][b] = (tr >= 0 && tr < N_ && tc >= 0 && tc < N_) ? sk[tr * N_ + tc] : T(0);
                }
            const T* qb = sqb + (r0 / CF + Ic0 - iq0 + D::DLO) * QS + (c0 / CF + Jc - jq0 + D::DLO);
            T acc[4] = {0, 0, 0, 0};
#pragma unroll
            for (int m = 0; m < DM + 3; ++m) {
                T qv[DM];
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
            const int Cc = c0 + Jc * CF + pc;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int R = r0 + (Ic0 + k) * CF + pr;
                if (R < H && Cc < W) oc[static_cast<size_t>(R) * W + Cc] = acc[k];
            }
        } else {
            constexpr int CPR = TA / CF, CPP = CPR * CPR;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int u = 128 * warp + 32 * k + lane;
                const int ph = u / CPP, cell = u - ph * CPP;
                const int pr = ph / CF, pc = ph - pr * CF;
                const int ci = cell / CPR, cj = cell - ci * CPR;
                const int dilo = floordiv(pr - C + CF - 1, CF), dihi = floordiv(pr + C, CF);
                const int djlo = floordiv(pc - C + CF - 1, CF), djhi = floordiv(pc + C, CF);
                const T* qb = sqb + (r0 / CF + ci - iq0) * QS + (c0 / CF + cj - jq0);
                T acc = 0;
                for (int di = dilo; di <= dihi; ++di) {
                    const T* krow = sk + (CF * di - pr + C) * n + C - pc;
                    const T* qrow = qb + di * QS;
                    for (int dj = djlo; dj <= djhi; ++dj) acc = fma(krow[CF * dj], qrow[dj], acc);
                }
                const int R = r0 + ci * CF + pr, Cc = c0 + cj * CF + pc;
                if (R < H && Cc < W) oc[static_cast<size_t>(R) * W + Cc] = acc;
            }
        }
    }
}

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    const unsigned int s = static_cast<unsigned int>(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// one lane's column pair of a row: 16 bytes (double) through L2 only, 8 bytes (float) through L1
__device__ __forceinline__ void cp_async_pair(double2* sdst, const double* gsrc) { cp_async16(sdst, gsrc); }
__device__ __forceinline__ void cp_async_pair(float2* sdst, const float* gsrc) {
    const unsigned int s = static_cast<unsigned int>(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}

// ------------------------------------------------------------------------------------------
// K_DU (fused CG path, factor 4, image sides multiples of 32): the data term and the CG update in
// one pass. d = B^T U q is formed per 32 x 32 HR tile with K_D's gather (q window in shared
// memory, phase sub-kernel in registers, 4 cell rows per thread) and consumed in registers:
// Ap = d + lambda w (w = L M L p from K_L), z += alpha p, r -= alpha Ap (pansharpen.cpp:245-247),
// ||r||^2, ||z||^2 and the relative-step stop test (:248-255). d and Ap are never written: the
// iteration moves the 11 planes of SURVEY 8(d) and nothing else.
//
// Persistent: the work units are (active channel, tile), channel-major; CTA b owns a contiguous
// range of them, so it builds its phase sub-kernel once per scene and pays no per-tile prologue.
// A unit's q window and the z, r, p, w values of every thread's own four outputs stream into a
// ring of NST shared-memory stages by cp.async, NST - 1 units ahead of their use, which keeps the
// HBM loads in flight under the FP64 gather; one block barrier per unit publishes the window.
// Every unit writes its (||r||^2, ||z||^2) partial to part[(ch, tile)]; the last CTA to arrive
// on a channel sums the tiles in a fixed order, so the result does not depend on the partition.
// ------------------------------------------------------------------------------------------
#ifndef FBMP_DU_NST
#define FBMP_DU_NST 3
#endif
namespace du {
#ifndef FBMP_DU_NT
#define FBMP_DU_NT 256
#endif
constexpr int NST = FBMP_DU_NST;             // ring depth
constexpr int NTD = FBMP_DU_NT;              // threads per CTA: 256 (32 x 32 tiles, 2 CTAs/SM) or 128 (32 x 16, 4 CTAs/SM)
constexpr int TW = 32, TH = NTD / 8;         // HR tile of a unit (64 x 16 with 256 threads measured equal at C2, 2.5 % slower at C5)
constexpr int WIN = 208;                     // q window slots of a stage (>= 21 x 9, 16-byte multiple)
constexpr int STG = WIN + 4 * TW * TH;       // elements per stage: window | z, r, p, w tiles
constexpr int MAXCH = 512;                   // channels per launch (active-channel tables)
template <class T>
constexpr size_t smem() {
    return (static_cast<size_t>(NST) * STG * sizeof(T) + 15) / 16 * 16 + 2 * (NTD / 32) * 2 * sizeof(double) +
           MAXCH * (sizeof(T) + 2 * sizeof(short));
}
// one element to the 32-bit shared address sdst + OFF elements
template <class T, int OFF>
__device__ __forceinline__ void cp_async_elem(unsigned int sdst, const T* gsrc) {
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0 + %2], [%1], 8;\n" ::"r"(sdst), "l"(gsrc), "n"(OFF * 8) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0 + %2], [%1], 4;\n" ::"r"(sdst), "l"(gsrc), "n"(OFF * 4) : "memory");
}
// 16 bytes through L2 only to the 32-bit shared address sdst + OFFB bytes
template <int OFFB, class T>
__device__ __forceinline__ void cp_async_chunk(unsigned int sdst, const T* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0 + %2], [%1], 16;\n" ::"r"(sdst), "l"(gsrc), "n"(OFFB) : "memory");
}
}  // namespace du

template <int N_, class T = double>
__global__ void __launch_bounds__(du::NTD, 512 / du::NTD) k_du(PsGeo G, const T* __restrict__ taps, const T* __restrict__ q,
                                              const T* __restrict__ wv, T* __restrict__ z, T* __restrict__ r,
                                              const T* __restrict__ pbuf, CgState* st, double* __restrict__ part,
                                              int ntile) {
    using namespace a4;
    constexpr int NT = du::NTD;  // (shadows the 256 threads of the tile kernels)
    constexpr int CF = 4;
    using D = DT<N_, CF>;
    constexpr int DM = D::DM;
    constexpr int TW = du::TW, TH = du::TH;
    constexpr int QLO = cfloordiv(CF - 1 - D::C, CF);
    constexpr int QWC = cfloordiv(TW - 1 + D::C, CF) - QLO + 1;  // window columns
    constexpr int QWR = cfloordiv(TH - 1 + D::C, CF) - QLO + 1;  // window rows
    constexpr int QNC = QWC * QWR;
    static_assert(QNC <= du::WIN && QNC <= NT, "q window");
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ double red[2 * (NT / 32 + 1)];
    __shared__ int s_nact, s_last;
    T* stg = reinterpret_cast<T*>(smraw);
    double* wred = reinterpret_cast<double*>(smraw + (static_cast<size_t>(du::NST) * du::STG * sizeof(T) + 15) / 16 * 16);
    T* s_alpha = reinterpret_cast<T*>(wred + 2 * (NT / 32) * 2);
    short* s_act = reinterpret_cast<short*>(s_alpha + du::MAXCH);
    short* s_par = s_act + du::MAXCH;
    const int W = G.W, n = G.n;
    const size_t P = static_cast<size_t>(G.H) * W, pl = static_cast<size_t>(G.h) * G.w;
    const int ntx = W / TW, nty = G.H / TH;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the thread's four outputs of a tile (CF rows apart) and its phase
    constexpr int CW4 = TW / CF, RB4 = TH / CF / 4;
    static_assert(CF * CW4 * RB4 * CF == NT, "one thread per (column, row phase, group of 4 cell rows)");
    const int pc = threadIdx.x % CF;
    const int Jc = (threadIdx.x / CF) % CW4;
    const int rest = threadIdx.x / (CF * CW4);
    const int Ic0 = (rest % RB4) * 4;
    const int pr = rest / RB4;
    const int toff = (Ic0 * CF + pr) * W + Jc * CF + pc;  // within the tile (element indices of a plane fit 31 bits)
    const int rstep = CF * W;
    const int qoff = (Ic0 + D::DLO - QLO) * QWC + (Jc + D::DLO - QLO);
    const int wa = threadIdx.x / QWC, wb = threadIdx.x - wa * QWC;  // window element copied by this thread
    const T lam = static_cast<T>(G.lambda);
    // 32-bit shared addresses of the thread's slots of stage 0
    const unsigned int s_win = static_cast<unsigned int>(__cvta_generic_to_shared(stg + threadIdx.x));
    // the thread's 16-byte chunks of a staged tile: column chunk threadIdx % CPR of the rows
    // threadIdx / CPR + h CROWS
    constexpr int EPC = 16 / sizeof(T), CPR = TW / EPC, CROWS = NT / CPR, CPASS = TH / CROWS;
    static_assert(CPASS * CROWS == TH && CPASS >= 1, "chunk passes");
    const int ce = (threadIdx.x / CPR) * W + (threadIdx.x % CPR) * EPC;  // element offset within the tile
    const unsigned int s_chk = static_cast<unsigned int>(
        __cvta_generic_to_shared(stg + du::WIN + (threadIdx.x / CPR) * TW + (threadIdx.x % CPR) * EPC));
    constexpr unsigned int STGB = du::STG * sizeof(T);
    pdl_wait();  // w, alpha and the flags come from K_L
    pdl_trigger();
    // active channels (ascending), their p parity and alpha
    if (warp == 0) {
        int na = 0;
        for (int base = 0; base < G.N; base += 32) {
            const int c = base + lane;
            const bool on = c < G.N && st[c].done == 0;
            const unsigned int mk = __ballot_sync(0xffffffffu, on);
            if (on) {
                const int pos = na + __popc(mk & ((1u << lane) - 1u));
                s_act[pos] = static_cast<short>(c);
                s_par[pos] = static_cast<short>(st[c].t & 1);
                s_alpha[pos] = static_cast<T>(st[c].alpha);
            }
            na += __popc(mk);
        }
        if (lane == 0) s_nact = na;
    }
    __syncthreads();
    const int nact = s_nact;
    if (nact == 0) return;
    // CTA b owns the contiguous units [b per, (b + 1) per): consecutive tiles of a tile row, so the
    // units in flight continue the same DRAM rows (measured: interleaving the CTAs' units over the
    // image is 7-10 % slower)
    const long long U = static_cast<long long>(nact) * ntile;
    const int per = static_cast<int>((U + gridDim.x - 1) / gridDim.x);
    const long long a0 = static_cast<long long>(blockIdx.x) * per;
    const int nu = a0 >= U ? 0 : static_cast<int>(min(static_cast<long long>(per), U - a0));
    // unit cursors (channel index, tile column / row, element offset of the tile origin), advanced
    // without divisions; one for the copies being issued, one for the unit being consumed
    struct Cursor {
        int k, bx, by, eoff;
    };
    auto advance = [&](Cursor& c) {
        c.eoff += TW;
        if (++c.bx == ntx) {
            c.bx = 0;
            c.eoff += (TH - 1) * W;
            if (++c.by == nty) {
                c.by = 0;
                c.eoff = 0;
                ++c.k;
            }
        }
    };
    Cursor ci;
    {
        ci.k = static_cast<int>(a0 / ntile);
        const int t0 = static_cast<int>(a0 - static_cast<long long>(ci.k) * ntile);
        ci.by = t0 / ntx;
        ci.bx = t0 - ci.by * ntx;
        ci.eoff = ci.by * TH * W + ci.bx * TW;
    }
    Cursor cc = ci;
    auto issue = [&](int stage) {  // the unit at cursor ci -> stage
        const int ch = s_act[ci.k];
        const unsigned int so = static_cast<unsigned int>(stage) * STGB;
        if (threadIdx.x < QNC) {
            const int iq0 = ci.by * (TH / CF) + QLO, jq0 = ci.bx * (TW / CF) + QLO;
            const T* src = q + static_cast<size_t>(ch) * pl + wrap_once(iq0 + wa, G.h) * G.w + wrap_once(jq0 + wb, G.w);
            du::cp_async_elem<T, 0>(s_win + so, src);
        }
        // z, r, p, w tiles as 16-byte chunks through L2 only (cp.async.cg: copies through L1 are
        // limited by the few L1 lines left beside 220 KB of shared memory); the block barrier that
        // publishes the window publishes them too
        const size_t chP = static_cast<size_t>(ch) * P;
        const T* zc = z + chP;
        const T* rc = r + chP;
        const T* wc = wv + chP;
        const T* pcp = pbuf + (static_cast<size_t>(s_par[ci.k]) * G.N + ch) * P;
        const int e0 = ci.eoff + ce;
#pragma unroll
        for (int h = 0; h < CPASS; ++h) {
            const int e = e0 + h * CROWS * W;
            du::cp_async_chunk<(0 * TH + 0) * TW * sizeof(T)>(s_chk + so + h * CROWS * TW * static_cast<unsigned int>(sizeof(T)), zc + e);
            du::cp_async_chunk<(1 * TH + 0) * TW * sizeof(T)>(s_chk + so + h * CROWS * TW * static_cast<unsigned int>(sizeof(T)), rc + e);
            du::cp_async_chunk<(2 * TH + 0) * TW * sizeof(T)>(s_chk + so + h * CROWS * TW * static_cast<unsigned int>(sizeof(T)), pcp + e);
            du::cp_async_chunk<(3 * TH + 0) * TW * sizeof(T)>(s_chk + so + h * CROWS * TW * static_cast<unsigned int>(sizeof(T)), wc + e);
        }
        advance(ci);
    };
#pragma unroll
    for (int j = 0; j < du::NST - 1; ++j) {
        if (j < nu) issue(j);
        cp_async_commit();
    }
    int kprev = 0, tprev = 0;
    int cur_k = -1, cur_scene = -1;
    T alpha = 0;
    size_t chP = 0;
    int stage = 0, stage_is = du::NST - 1;  // stage of unit j; stage the next issue goes to
    T kreg[DM][DM];
    for (int j = 0; j < nu; ++j) {
        cp_async_wait<du::NST - 2>();  // this thread's copies of unit j have landed
        __syncthreads();               // ... everyone's (the window); unit j - 1 is consumed by all
        if (j + du::NST - 1 < nu) issue(stage_is);
        cp_async_commit();
        if (++stage_is == du::NST) stage_is = 0;
        // per-tile partial of the previous unit (its warp sums are published by the barrier above)
        if (j > 0 && threadIdx.x == 0) {
            const double* wr = wred + ((j - 1) & 1) * (NT / 32) * 2;
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int wi = 0; wi < NT / 32; ++wi) {
                s0 += wr[2 * wi];
                s1 += wr[2 * wi + 1];
            }
            double* pd = part + (static_cast<size_t>(s_act[kprev]) * ntile + tprev) * 2;
            pd[0] = s0;
            pd[1] = s1;
        }
        if (cc.k != cur_k) {  // next channel: its scalars and, on a new scene, the phase sub-kernel
            cur_k = cc.k;
            const int ch = s_act[cur_k];
            alpha = s_alpha[cur_k];
            chP = static_cast<size_t>(ch) * P;
            const int scene = ch / G.cps;
            if (scene != cur_scene) {
                cur_scene = scene;
                const T* tp = taps + static_cast<size_t>(scene) * n * n;
#pragma unroll
                for (int a = 0; a < DM; ++a)
#pragma unroll
                    for (int b = 0; b < DM; ++b) {
                        const int tr = CF * (a + D::DLO) - pr + D::C, tcc = CF * (b + D::DLO) - pc + D::C;
                        kreg[a][b] = (tr >= 0 && tr < N_ && tcc >= 0 && tcc < N_) ? __ldg(tp + tr * N_ + tcc) : T(0);
                    }
            }
        }
        const T* sd = stg + stage * du::STG;
        // d of the thread's four outputs (K_D's gather: ascending (mm, b) per accumulator)
        const T* qa = sd + qoff;
        T acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int mm = 0; mm < DM + 3; ++mm) {
            T qv[DM];
#pragma unroll
            for (int b = 0; b < DM; ++b) qv[b] = qa[mm * QWC + b];
#pragma unroll
            for (int b = 0; b < DM; ++b)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int a = mm - k;
                    if (a >= 0 && a < DM) acc[k] = fma(kreg[a][b], qv[b], acc[k]);
                }
        }
        const T* sv = sd + du::WIN + (Ic0 * CF + pr) * TW + Jc * CF + pc;  // [array][tile row][tile column]
        T* zc = z + chP;
        T* rc = r + chP;
        const int e0 = cc.eoff + toff;
        double rr = 0.0, zz = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const T z0 = sv[(0 * TH + k * CF) * TW], r0v = sv[(1 * TH + k * CF) * TW], p0 = sv[(2 * TH + k * CF) * TW],
                    w0 = sv[(3 * TH + k * CF) * TW];
            const T ap = acc[k] + w0 * lam;      // pansharpen.cpp:222-223
            const T zn = z0 + p0 * alpha;        // :245
            const T rn = r0v - ap * alpha;       // :246
            const int e = e0 + k * rstep;
            __stcs(zc + e, zn);
            __stcs(rc + e, rn);
            rr += static_cast<double>(rn) * static_cast<double>(rn);
            zz += static_cast<double>(zn) * static_cast<double>(zn);
        }
        rr = warp_sum(rr);
        zz = warp_sum(zz);
        if (lane == 0) {
            double* wr = wred + (j & 1) * (NT / 32) * 2;
            wr[2 * warp] = rr;
            wr[2 * warp + 1] = zz;
        }
        kprev = cc.k;
        tprev = cc.by * ntx + cc.bx;
        advance(cc);
        if (++stage == du::NST) stage = 0;
    }
    __syncthreads();
    if (nu > 0 && threadIdx.x == 0) {  // the last unit's partial
        const double* wr = wred + ((nu - 1) & 1) * (NT / 32) * 2;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int wi = 0; wi < NT / 32; ++wi) {
            s0 += wr[2 * wi];
            s1 += wr[2 * wi + 1];
        }
        double* pd = part + (static_cast<size_t>(s_act[kprev]) * ntile + tprev) * 2;
        pd[0] = s0;
        pd[1] = s1;
        __threadfence();
    }
    if (nu == 0) return;
    // arrival on every channel this CTA has units of (thread i: i-th active channel); the last of a
    // channel's CTAs closes its iteration
    __shared__ unsigned char s_fin[du::MAXCH];
    __syncthreads();  // thread 0's partials are fenced
    for (int i = threadIdx.x; i < nact; i += NT) {
        const long long u0 = static_cast<long long>(i) * ntile;
        unsigned char fin = 0;
        if (u0 < a0 + nu && u0 + ntile > a0) {
            const unsigned int touch = static_cast<unsigned int>((u0 + ntile - 1) / per - u0 / per + 1);
            const unsigned int prev = atomicAdd(&st[s_act[i]].cnt_u, 1u);
            if (prev == touch - 1u) {
                __threadfence();
                fin = 1;
            }
        }
        s_fin[i] = fin;
    }
    __syncthreads();
    for (int i = 0; i < nact; ++i) {
        if (!s_fin[i]) continue;  // block-uniform
        const int ch = s_act[i];
        // row strips: the tiles of the owned rows only (rlo, rhi are multiples of the tile height)
        const int t_lo = G.dred ? (G.rlo / TH) * ntx : 0, t_hi = G.dred ? (G.rhi / TH) * ntx : ntile;
        const double2 tot = sum_partials2<NT>(part + (static_cast<size_t>(ch) * ntile + t_lo) * 2, t_hi - t_lo, red);
        if (threadIdx.x == 0 && G.dred) {  // distributed: publish the local sums only
            G.dred[G.N + 3 * ch + 1] = tot.x;
            G.dred[G.N + 3 * ch + 2] = tot.y;
            st[ch].cnt_u = 0;
        } else if (threadIdx.x == 0) {
            CgState& S = st[ch];
            const double rs_new = tot.x, zsq = tot.y;
            const int t = S.t;
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

// blockIdx.x = (scene, item = (band, strip), channel of the scene), channel fastest
template <bool CG>
__global__ void __launch_bounds__(kl::NTL, 16) k_llp(PsGeo G, const double* __restrict__ guide,
                                                    const double* __restrict__ wmu, const double* __restrict__ wg,
                                                    const double* __restrict__ pin, double* __restrict__ out,
                                                    CgState* st, double* __restrict__ part, int nbands, int kstrips,
                                                    int R) {
    using namespace kl;
    // channel-fastest CTA order within a scene: the channels of a (band, strip) item run
    // together, so the scene's guide maps are read from HBM once and hit in L2 for the others
    const int nblk = gridDim.x / G.N;
    int ch, item;
    if (G.N % G.cps == 0) {
        const int per_scene = nblk * G.cps, sc = blockIdx.x / per_scene, r = blockIdx.x - sc * per_scene;
        item = r / G.cps;
        ch = sc * G.cps + (r - item * G.cps);
    } else {
        ch = blockIdx.x % G.N;
        item = blockIdx.x / G.N;
    }
    const int scene = ch / G.cps;
    const int H = G.H, W = G.W;
    const size_t P = static_cast<size_t>(H) * W;
    const int lane = threadIdx.x;
    if (CG) {
        pdl_wait();
        pdl_trigger();
        if (__all_sync(0xffffffffu, st[ch].done != 0)) return;
    }
    const int nrb = (H + RB - 1) / RB;
    double dotp = 0.0;
    {
        const int band = item / kstrips, strip = item - band * kstrips;
        const int c0 = band * BAND, r0 = strip * R, r1 = min(H, r0 + R);
        const int X = wrap_once(c0 - HALO + lane, W);
        const double* pp = pin + ch * P;
        if (CG) pp = pin + (static_cast<size_t>(st[ch].t & 1) * G.N + ch) * P;
        const double* I = guide + scene * P + X;
        const double* MU = wmu + scene * P + X;
        const double* GK = wg + scene * P + X;
        const double* pc = pp + X;
        double* oc = out + ch * P + X;
        const bool writer = lane >= HALO && lane < HALO + BAND && c0 + lane - HALO < W;
        // interior-window count factor of column X (pansharpen.cpp:150-160)
        const int ncol = max(min(X + 1, W - 2) - max(X - 1, 1) + 1, 0);
        const double lam = G.lambda;
        // Rows: Y = the p row loaded by the step; S1 runs on row Y-1, S2 on Y-2, S3 on Y-3 and
        // S5 (the output) on Y-4. Row offsets (elements) shift down one slot per step; the loads
        // run two steps ahead (buffers A / B alternate, loop unrolled by two).
        const int yA = wrap_once(r0 - HALO, H);
        int ld_row = yA;                       // next row to load
        auto adv = [&](int r) { return r + 1 == H ? 0 : r + 1; };
        auto back = [&](int r, int k) { const int q = r - k; return q < 0 ? q + H : q; };
        struct Rowv {
            double p0, i1, m2, g2, d4, p4;
        };
        auto load = [&](Rowv& v, int y) {
            const int o0 = y * W, o1 = back(y, 1) * W, o2 = back(y, 2) * W, o4 = back(y, 4) * W;
            v.p0 = __ldg(pc + o0);
            v.i1 = __ldg(I + o1);
            v.m2 = __ldg(MU + o2);
            v.g2 = __ldg(GK + o2);
            v.d4 = oc[o4];
            v.p4 = __ldg(pc + o4);
        };
        double pm2 = 0.0, pm1 = 0.0, Im2 = 0.0, Im3 = 0.0, s2 = 0.0, s3 = 0.0;
        double hs_a = 0.0, hs_b = 0.0, his_a = 0.0, his_b = 0.0;
        double ha_a = 0.0, ha_b = 0.0, hc_a = 0.0, hc_b = 0.0, M_a = 0.0, M_b = 0.0;
        const int steps = (r1 - r0) + 2 * HALO;
        int r3 = back(yA, 3);                  // row of S3 (Y-3) for the current step
        int o4 = back(yA, 4) * W;              // output row offset (Y-4)
        int blk_left = RB - (r0 % RB);         // output rows left in the current partial block
        Rowv A, B;
        load(A, ld_row);
        ld_row = adv(ld_row);
        if (steps > 1) load(B, ld_row);
        ld_row = adv(ld_row);
        auto step = [&](Rowv& V, int st_i) {
            const double p0 = V.p0, Im1 = V.i1, mu2 = V.m2, g2 = V.g2, d4 = V.d4, p4 = V.p4;
            if (st_i + 2 < steps) load(V, ld_row);
            ld_row = adv(ld_row);
            // S1 at row Y-1: s = L p (ops.cpp:70-78 order), I s
            const double pl = __shfl_up_sync(0xffffffffu, pm1, 1), pr = __shfl_down_sync(0xffffffffu, pm1, 1);
            const double s1 = 4.0 * pm1 - pm2 - p0 - pl - pr;
            const double is1 = Im1 * s1;
            // S2 at row Y-2: window sums over rows Y-3..Y-1, coefficients a, c1
            const double hs1 = __shfl_up_sync(0xffffffffu, s1, 1) + s1 + __shfl_down_sync(0xffffffffu, s1, 1);
            const double his1 = __shfl_up_sync(0xffffffffu, is1, 1) + is1 + __shfl_down_sync(0xffffffffu, is1, 1);
            const double xb = (hs_a + hs_b + hs1) * (1.0 / 9.0);
            const double a2 = g2 * ((his_a + his_b + his1) * (1.0 / 9.0) - mu2 * xb);
            const double c2 = g2 != 0.0 ? xb - mu2 * a2 : 0.0;
            // S3 at row Y-3: M s = n s - box(c1) - I box(a)
            const double ha2 = __shfl_up_sync(0xffffffffu, a2, 1) + a2 + __shfl_down_sync(0xffffffffu, a2, 1);
            const double hc2 = __shfl_up_sync(0xffffffffu, c2, 1) + c2 + __shfl_down_sync(0xffffffffu, c2, 1);
            const int g3 = wrap_once(r3 + G.grow0, G.Hg);  // global row (strip decomposition)
            const int nrow = max(min(g3 + 1, G.Hg - 2) - max(g3 - 1, 1) + 1, 0);
            const double Mc = static_cast<double>(nrow * ncol) * s3 - (hc_a + hc_b + hc2) - Im3 * (ha_a + ha_b + ha2);
            // S5 at row Y-4: t = L (M s), out = d + lambda t
            const double Ml = __shfl_up_sync(0xffffffffu, M_b, 1), Mr = __shfl_down_sync(0xffffffffu, M_b, 1);
            const double t = 4.0 * M_b - M_a - Mc - Ml - Mr;
            const double val = d4 + t * lam;
            if (st_i >= 2 * HALO) {
                if (writer) {
                    oc[o4] = val;
                    const int yo = r0 + st_i - 2 * HALO;
                    if (yo >= G.rlo && yo < G.rhi) dotp += p4 * val;
                }
                if (CG && (--blk_left == 0 || st_i + 1 == steps)) {  // close the row block
                    const double ws = warp_sum(dotp);
                    const int yo = r0 + st_i - 2 * HALO;
                    if (lane == 0) part[(static_cast<size_t>(ch) * nbands + band) * nrb + yo / RB] = ws;
                    dotp = 0.0;
                    blk_left = RB;
                }
            }
            pm2 = pm1; pm1 = p0;
            Im3 = Im2; Im2 = Im1;
            s3 = s2; s2 = s1;
            hs_a = hs_b; hs_b = hs1; his_a = his_b; his_b = his1;
            ha_a = ha_b; ha_b = ha2; hc_a = hc_b; hc_b = hc2;
            M_a = M_b; M_b = Mc;
            r3 = adv(r3);
            o4 = o4 + W == static_cast<int>(P) ? 0 : o4 + W;
        };
        int st_i = 0;
        for (; st_i + 1 < steps; st_i += 2) {
            step(A, st_i);
            step(B, st_i + 1);
        }
        if (st_i < steps) step(A, st_i);
    }
    if (CG) {
        // arrival of this item (its row-block partials are written); the last item of the channel
        // sums all partials of the channel in a fixed order
        unsigned int prev = 0;
        if (lane == 0) {
            __threadfence();
            prev = atomicAdd(&st[ch].cnt_a, 1u);
        }
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == static_cast<unsigned int>(nblk) - 1u) {
            __threadfence();
            const double* pa = part + static_cast<size_t>(ch) * nbands * nrb;
            double sacc = 0.0;
#pragma unroll 8
            for (int i = lane; i < nbands * nrb; i += 32) sacc += __ldcg(pa + i);
            const double pAp = warp_sum(sacc);
            if (lane == 0 && G.dred) {  // distributed: publish the local sum only
                G.dred[ch] = pAp;
                st[ch].cnt_a = 0;
            } else if (lane == 0) {
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


// K_L on column PAIRS (W even): lane = columns (X, X+1), a warp spans 64 columns of which the
// inner 56 are output (BAND2). Loads are 16-byte, each stage exchanges one double with each
// neighbour lane (half the shuffles per pixel of k_llp), and the halo overhead is 64/56.
namespace kl {
constexpr int BAND2 = 56;
}
#ifndef FBMP_KL_NB
#define FBMP_KL_NB 4
#endif
#ifndef FBMP_KL_MINB
#define FBMP_KL_MINB 12  // K_L warps per SM the register budget is sized for
#endif
#ifndef FBMP_KL_UNROLL
#define FBMP_KL_UNROLL 3
#endif
constexpr int KL_UNROLL = FBMP_KL_UNROLL;
// LAP = false: the identity pansharpening prior (pansharpen.cpp:28-50): Ap = d + lambda M p (the
// S1 and S5 Laplacians become copies; everything else, including the row pipeline, is unchanged)
// DIN = false (fused path, CG only): d is not read; the kernel writes w = L M L p (unscaled) and
// sums p.w, and p.Ap = ||q||^2 + lambda p.w with ||q||^2 from K_Q3 (p . B^T U D B p = |D B p|^2);
// K_DU forms Ap = d + lambda w while it updates z and r.
template <bool CG, class T = double, bool LAP = true, bool DIN = true>
__global__ void __launch_bounds__(kl::NTL, FBMP_KL_MINB) k_llp2(PsGeo G, const T* __restrict__ guide,
                                                     const T* __restrict__ wmu, const T* __restrict__ wg,
                                                     const T* __restrict__ pin, T* __restrict__ out,
                                                     CgState* st, double* __restrict__ part, int nbands, int kstrips,
                                                     int R) {
    using V = v2<T>;
    using namespace kl;
    // channel-fastest CTA order within a scene: the channels of a (band, strip) item run
    // together, so the scene's guide maps are read from HBM once and hit in L2 for the others
    const int nblk = gridDim.x / G.N;
    int ch, item;
    if (G.N % G.cps == 0) {
        const int per_scene = nblk * G.cps, sc = blockIdx.x / per_scene, r = blockIdx.x - sc * per_scene;
        item = r / G.cps;
        ch = sc * G.cps + (r - item * G.cps);
    } else {
        ch = blockIdx.x % G.N;
        item = blockIdx.x / G.N;
    }
    const int scene = ch / G.cps;
    const int H = G.H, W = G.W;
    const size_t P = static_cast<size_t>(H) * W;
    const int lane = threadIdx.x;
    if (CG) {
        pdl_wait();
        pdl_trigger();
        if (__all_sync(0xffffffffu, st[ch].done != 0)) return;
    }
    const int nrb = (H + RB - 1) / RB;
    const unsigned FULL = 0xffffffffu;
    constexpr int NB = FBMP_KL_NB;           // ring depth: rows in flight = NB - 1
    __shared__ V ring[NB][5][32];            // p, I, mu, g, d rows of NB steps
    double dotp = 0.0;
    {
        const int band = item / kstrips, strip = item - band * kstrips;
        const int c0 = band * BAND2, r0 = strip * R, r1 = min(H, r0 + R);
        const int X = wrap_once(c0 - HALO + 2 * lane, W);  // even; X + 1 < W
        const T* pp = pin + ch * P;
        if (CG) pp = pin + (static_cast<size_t>(st[ch].t & 1) * G.N + ch) * P;
        const T* pc = pp + X;
        const T* I = guide + scene * P + X;
        const T* MU = wmu + scene * P + X;
        const T* GK = wg + scene * P + X;
        T* oc = out + ch * P + X;
        const int ox = c0 - HALO + 2 * lane;                 // unwrapped column of .x
        const bool writer = lane >= HALO / 2 && lane < (HALO + BAND2) / 2 && ox < W;
        const int nc0 = max(min(X + 1, W - 2) - max(X - 1, 1) + 1, 0);
        const int nc1 = max(min(X + 2, W - 2) - max(X, 1) + 1, 0);
        const T lam = static_cast<T>(G.lambda);
        auto back = [&](int r, int k) { const int q = r - k; return q < 0 ? q + H : q; };
        // row offsets (elements) of Y (p), Y-1 (I), Y-2 (mu, g) and Y-4 (d); they advance by W
        const int yA = wrap_once(r0 - HALO, H);
        int o0 = yA * W, o1 = back(yA, 1) * W, o2 = back(yA, 2) * W, o4 = back(yA, 4) * W;
        auto adv = [&](int o) { return o + W == static_cast<int>(P) ? 0 : o + W; };
        int r3 = back(yA, 3);
        V pm1 = {0, 0}, pm2 = {0, 0}, pm3 = {0, 0}, pm4 = {0, 0};
        V Im2 = {0, 0}, Im3 = {0, 0}, s2 = {0, 0}, s3 = {0, 0};
        V hs_a = {0, 0}, hs_b = {0, 0}, his_a = {0, 0}, his_b = {0, 0};
        V ha_a = {0, 0}, ha_b = {0, 0}, hc_a = {0, 0}, hc_b = {0, 0}, M_a = {0, 0}, M_b = {0, 0};
        const int steps = (r1 - r0) + 2 * HALO;
        int blk_left = RB;
        // the rows of step j stream into ring slot j % NB with cp.async, NB - 1 steps ahead of
        // their use (each lane copies and later reads its own 16 bytes: no warp barrier)
        // byte offsets of the next step to issue (32-bit: a plane is < 2^31 bytes), added to 64-bit
        // bases: one 64-bit add per address instead of a sign-extended scaled index
        const unsigned Wb = static_cast<unsigned>(W) * sizeof(T), Pb = static_cast<unsigned>(P) * sizeof(T);
        unsigned io0 = static_cast<unsigned>(o0) * sizeof(T), io1 = static_cast<unsigned>(o1) * sizeof(T),
                 io2 = static_cast<unsigned>(o2) * sizeof(T), io4 = static_cast<unsigned>(o4) * sizeof(T);
        const char* pcb = reinterpret_cast<const char*>(pc);
        const char* Ib = reinterpret_cast<const char*>(I);
        const char* MUb = reinterpret_cast<const char*>(MU);
        const char* GKb = reinterpret_cast<const char*>(GK);
        const char* ocb = reinterpret_cast<const char*>(oc);
        auto advb = [&](unsigned o) { const unsigned q = o + Wb; return q == Pb ? 0u : q; };
        auto issue = [&](int slot) {
            cp_async_pair(&ring[slot][0][lane], reinterpret_cast<const T*>(pcb + io0));
            cp_async_pair(&ring[slot][1][lane], reinterpret_cast<const T*>(Ib + io1));
            cp_async_pair(&ring[slot][2][lane], reinterpret_cast<const T*>(MUb + io2));
            cp_async_pair(&ring[slot][3][lane], reinterpret_cast<const T*>(GKb + io2));
            if constexpr (DIN) {
                cp_async_pair(&ring[slot][4][lane], reinterpret_cast<const T*>(ocb + io4));
                io4 = advb(io4);
            }
            io0 = advb(io0); io1 = advb(io1); io2 = advb(io2);
        };
#pragma unroll
        for (int j = 0; j < NB - 1; ++j) {
            if (j < steps) issue(j);
            cp_async_commit();
        }
#pragma unroll KL_UNROLL
        for (int st_i = 0; st_i < steps; ++st_i) {  // unrolled: the register windows rotate by renaming
            if (st_i + NB - 1 < steps) issue((st_i + NB - 1) % NB);
            cp_async_commit();
            cp_async_wait<NB - 1>();  // the group of step st_i has landed
            const int slot = st_i % NB;
            const V p0 = ring[slot][0][lane], Im1 = ring[slot][1][lane], mu2 = ring[slot][2][lane],
                    g2 = ring[slot][3][lane];
            V d4 = {0, 0};
            if constexpr (DIN) d4 = ring[slot][4][lane];
            const int o4c = o4;
            o4 = adv(o4);
            // S1 at row Y-1 (ops.cpp:70-78 order: 4 c - up - down - left - right)
            V s1, is1;
            if constexpr (LAP) {
                const T pL = __shfl_up_sync(FULL, pm1.y, 1), pR = __shfl_down_sync(FULL, pm1.x, 1);
                s1.x = T(4) * pm1.x - pm2.x - p0.x - pL - pm1.y;
                s1.y = T(4) * pm1.y - pm2.y - p0.y - pm1.x - pR;
            } else {
                s1 = pm1;
            }
            is1.x = Im1.x * s1.x;
            is1.y = Im1.y * s1.y;
            // S2 at row Y-2
            const T sL = __shfl_up_sync(FULL, s1.y, 1), sR = __shfl_down_sync(FULL, s1.x, 1);
            const T iL = __shfl_up_sync(FULL, is1.y, 1), iR = __shfl_down_sync(FULL, is1.x, 1);
            const V hs1 = mk2(sL + s1.x + s1.y, s1.x + s1.y + sR);
            const V his1 = mk2(iL + is1.x + is1.y, is1.x + is1.y + iR);
            constexpr T NINTH = T(1.0 / 9.0);
            V a2, c2;
            {
                const T xb = (hs_a.x + hs_b.x + hs1.x) * NINTH;
                a2.x = g2.x * ((his_a.x + his_b.x + his1.x) * NINTH - mu2.x * xb);
                c2.x = g2.x != T(0) ? xb - mu2.x * a2.x : T(0);
            }
            {
                const T xb = (hs_a.y + hs_b.y + hs1.y) * NINTH;
                a2.y = g2.y * ((his_a.y + his_b.y + his1.y) * NINTH - mu2.y * xb);
                c2.y = g2.y != T(0) ? xb - mu2.y * a2.y : T(0);
            }
            // S3 at row Y-3
            const T aL = __shfl_up_sync(FULL, a2.y, 1), aR = __shfl_down_sync(FULL, a2.x, 1);
            const T cL = __shfl_up_sync(FULL, c2.y, 1), cR = __shfl_down_sync(FULL, c2.x, 1);
            const V ha2 = mk2(aL + a2.x + a2.y, a2.x + a2.y + aR);
            const V hc2 = mk2(cL + c2.x + c2.y, c2.x + c2.y + cR);
            const int g3 = wrap_once(r3 + G.grow0, G.Hg);  // global row (strip decomposition)
            const int nrow = max(min(g3 + 1, G.Hg - 2) - max(g3 - 1, 1) + 1, 0);
            V Mc;
            Mc.x = static_cast<T>(nrow * nc0) * s3.x - (hc_a.x + hc_b.x + hc2.x) - Im3.x * (ha_a.x + ha_b.x + ha2.x);
            Mc.y = static_cast<T>(nrow * nc1) * s3.y - (hc_a.y + hc_b.y + hc2.y) - Im3.y * (ha_a.y + ha_b.y + ha2.y);
            // S5 at row Y-4
            T t0, t1;
            if constexpr (LAP) {
                const T ML = __shfl_up_sync(FULL, M_b.y, 1), MR = __shfl_down_sync(FULL, M_b.x, 1);
                t0 = T(4) * M_b.x - M_a.x - Mc.x - ML - M_b.y;
                t1 = T(4) * M_b.y - M_a.y - Mc.y - M_b.x - MR;
            } else {
                t0 = M_b.x;
                t1 = M_b.y;
            }
            const V val = DIN ? mk2(d4.x + t0 * lam, d4.y + t1 * lam) : mk2(t0, t1);
            if (st_i >= 2 * HALO) {
                if (writer) {
                    st2(oc + o4c, val);
                    const int yo = r0 + st_i - 2 * HALO;
                    if (yo >= G.rlo && yo < G.rhi)
                        dotp += static_cast<double>(pm4.x) * static_cast<double>(val.x) +
                                static_cast<double>(pm4.y) * static_cast<double>(val.y);
                }
                if (CG && (--blk_left == 0 || st_i + 1 == steps)) {  // close the row block
                    const double ws = warp_sum(dotp);
                    const int yo = r0 + st_i - 2 * HALO;
                    if (lane == 0) part[(static_cast<size_t>(ch) * nbands + band) * nrb + yo / RB] = ws;
                    dotp = 0.0;
                    blk_left = RB;
                }
            }
            pm4 = pm3; pm3 = pm2; pm2 = pm1; pm1 = p0;
            Im3 = Im2; Im2 = Im1;
            s3 = s2; s2 = s1;
            hs_a = hs_b; hs_b = hs1; his_a = his_b; his_b = his1;
            ha_a = ha_b; ha_b = ha2; hc_a = hc_b; hc_b = hc2;
            M_a = M_b; M_b = Mc;
            r3 = r3 + 1 == H ? 0 : r3 + 1;
        }
    }
    if (CG) {
        unsigned int prev = 0;
        if (lane == 0) {
            __threadfence();
            prev = atomicAdd(&st[ch].cnt_a, 1u);
        }
        prev = __shfl_sync(FULL, prev, 0);
        if (prev == static_cast<unsigned int>(nblk) - 1u) {
            __threadfence();
            const double* pa = part + static_cast<size_t>(ch) * nbands * nrb;
            double sacc = 0.0;
#pragma unroll 8
            for (int i = lane; i < nbands * nrb; i += 32) sacc += __ldcg(pa + i);
            double pAp = warp_sum(sacc);
            if (lane == 0 && G.dred) {  // distributed: publish the local sum only
                // fused chain: this strip's share of p.Ap = ||q||^2 + lambda p.w (linear in the strips)
                G.dred[ch] = DIN ? pAp : st[ch].qq + G.lambda * pAp;
                st[ch].cnt_a = 0;
            } else if (lane == 0) {
                CgState& S = st[ch];
                if constexpr (!DIN) pAp = S.qq + G.lambda * pAp;
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

// K_L of the fp32 mode (k_llp4f): the k_llp2 scheme with four columns per lane (16-byte float4
// rows, as the fp64 kernel moves 16-byte double2 rows), so a warp covers 120 output columns and
// every shuffle, cp.async and address computation serves four pixels instead of two. Per column
// the stage expressions are those of k_llp2 (same operand order); the p.Ap partials are fp64.
namespace kl {
constexpr int BAND4 = 120;  // output columns per warp of k_llp4f
}
template <bool CG, bool DIN = true>
__global__ void __launch_bounds__(kl::NTL, FBMP_KL_MINB) k_llp4f(PsGeo G, const float* __restrict__ guide,
                                                      const float* __restrict__ wmu, const float* __restrict__ wg,
                                                      const float* __restrict__ pin, float* __restrict__ out,
                                                      CgState* st, double* __restrict__ part, int nbands, int kstrips,
                                                      int R) {
    using namespace kl;
    const int nblk = gridDim.x / G.N;
    int ch, item;
    if (G.N % G.cps == 0) {
        const int per_scene = nblk * G.cps, sc = blockIdx.x / per_scene, r = blockIdx.x - sc * per_scene;
        item = r / G.cps;
        ch = sc * G.cps + (r - item * G.cps);
    } else {
        ch = blockIdx.x % G.N;
        item = blockIdx.x / G.N;
    }
    const int scene = ch / G.cps;
    const int H = G.H, W = G.W;
    const size_t P = static_cast<size_t>(H) * W;
    const int lane = threadIdx.x;
    if (CG) {
        pdl_wait();
        pdl_trigger();
        if (__all_sync(0xffffffffu, st[ch].done != 0)) return;
    }
    const int nrb = (H + RB - 1) / RB;
    const unsigned FULL = 0xffffffffu;
    constexpr int NB = FBMP_KL_NB;
    __shared__ float4 ring[NB][5][32];      // p, I, mu, g, d rows of NB steps
    double dotp = 0.0;
    {
        const int band = item / kstrips, strip = item - band * kstrips;
        const int c0 = band * BAND4, r0 = strip * R, r1 = min(H, r0 + R);
        const int X = wrap_once(c0 - HALO + 4 * lane, W);  // multiple of 4; X + 3 < W (W % 4 == 0)
        const float* pp = pin + ch * P;
        if (CG) pp = pin + (static_cast<size_t>(st[ch].t & 1) * G.N + ch) * P;
        const float* pc = pp + X;
        const float* I = guide + scene * P + X;
        const float* MU = wmu + scene * P + X;
        const float* GK = wg + scene * P + X;
        float* oc = out + ch * P + X;
        const int ox = c0 - HALO + 4 * lane;                 // unwrapped column of component 0
        const bool writer = lane >= HALO / 4 && lane < (HALO + BAND4) / 4 && ox < W;
        int ncol[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) ncol[j] = max(min(X + j + 1, W - 2) - max(X + j - 1, 1) + 1, 0);
        const float lam = static_cast<float>(G.lambda);
        auto back = [&](int r, int k) { const int q = r - k; return q < 0 ? q + H : q; };
        const int yA = wrap_once(r0 - HALO, H);
        int o4 = back(yA, 4) * W;
        auto adv = [&](int o) { return o + W == static_cast<int>(P) ? 0 : o + W; };
        int r3 = back(yA, 3);
        float pm1[4] = {}, pm2[4] = {}, pm3[4] = {}, pm4[4] = {}, Im2[4] = {}, Im3[4] = {}, s2[4] = {}, s3[4] = {};
        float hs_a[4] = {}, hs_b[4] = {}, his_a[4] = {}, his_b[4] = {};
        float ha_a[4] = {}, ha_b[4] = {}, hc_a[4] = {}, hc_b[4] = {}, M_a[4] = {}, M_b[4] = {};
        const int steps = (r1 - r0) + 2 * HALO;
        int blk_left = RB;
        int io0 = yA * W, io1 = back(yA, 1) * W, io2 = back(yA, 2) * W, io4 = o4;
        auto issue = [&](int slot) {
            cp_async16(&ring[slot][0][lane], pc + io0);
            cp_async16(&ring[slot][1][lane], I + io1);
            cp_async16(&ring[slot][2][lane], MU + io2);
            cp_async16(&ring[slot][3][lane], GK + io2);
            if constexpr (DIN) {
                cp_async16(&ring[slot][4][lane], oc + io4);
                io4 = adv(io4);
            }
            io0 = adv(io0); io1 = adv(io1); io2 = adv(io2);
        };
#pragma unroll
        for (int j = 0; j < NB - 1; ++j) {
            if (j < steps) issue(j);
            cp_async_commit();
        }
        auto unpack4 = [](const float4 v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; };
        // box sum of three horizontal neighbours: a[j-1] + a[j] + a[j+1] (k_llp2's operand order)
        auto hbox = [&](const float* a, float* o) {
            const float L = __shfl_up_sync(FULL, a[3], 1), Rr = __shfl_down_sync(FULL, a[0], 1);
            o[0] = L + a[0] + a[1];
            o[1] = a[0] + a[1] + a[2];
            o[2] = a[1] + a[2] + a[3];
            o[3] = a[2] + a[3] + Rr;
        };
        constexpr float NINTH = static_cast<float>(1.0 / 9.0);
#pragma unroll KL_UNROLL
        for (int st_i = 0; st_i < steps; ++st_i) {
            if (st_i + NB - 1 < steps) issue((st_i + NB - 1) % NB);
            cp_async_commit();
            cp_async_wait<NB - 1>();
            const int slot = st_i % NB;
            float p0[4], Im1[4], mu2[4], g2[4], d4[4];
            unpack4(ring[slot][0][lane], p0);
            unpack4(ring[slot][1][lane], Im1);
            unpack4(ring[slot][2][lane], mu2);
            unpack4(ring[slot][3][lane], g2);
            if constexpr (DIN) unpack4(ring[slot][4][lane], d4);
            const int o4c = o4;
            o4 = adv(o4);
            // S1 at row Y-1 (ops.cpp:70-78 order: 4 c - up - down - left - right)
            float s1[4], is1[4];
            {
                const float pL = __shfl_up_sync(FULL, pm1[3], 1), pR = __shfl_down_sync(FULL, pm1[0], 1);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float l = j == 0 ? pL : pm1[j - 1], r = j == 3 ? pR : pm1[j + 1];
                    s1[j] = 4.0f * pm1[j] - pm2[j] - p0[j] - l - r;
                    is1[j] = Im1[j] * s1[j];
                }
            }
            // S2 at row Y-2
            float hs1[4], his1[4], a2[4], c2[4];
            hbox(s1, hs1);
            hbox(is1, his1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float xb = (hs_a[j] + hs_b[j] + hs1[j]) * NINTH;
                a2[j] = g2[j] * ((his_a[j] + his_b[j] + his1[j]) * NINTH - mu2[j] * xb);
                c2[j] = g2[j] != 0.0f ? xb - mu2[j] * a2[j] : 0.0f;
            }
            // S3 at row Y-3
            float ha2[4], hc2[4], Mc[4];
            hbox(a2, ha2);
            hbox(c2, hc2);
            {
                const int g3 = wrap_once(r3 + G.grow0, G.Hg);
                const int nrow = max(min(g3 + 1, G.Hg - 2) - max(g3 - 1, 1) + 1, 0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    Mc[j] = static_cast<float>(nrow * ncol[j]) * s3[j] - (hc_a[j] + hc_b[j] + hc2[j]) -
                            Im3[j] * (ha_a[j] + ha_b[j] + ha2[j]);
            }
            // S5 at row Y-4
            {
                const float ML = __shfl_up_sync(FULL, M_b[3], 1), MR = __shfl_down_sync(FULL, M_b[0], 1);
                float val[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float l = j == 0 ? ML : M_b[j - 1], r = j == 3 ? MR : M_b[j + 1];
                    const float t = 4.0f * M_b[j] - M_a[j] - Mc[j] - l - r;
                    val[j] = DIN ? d4[j] + t * lam : t;
                }
                if (st_i >= 2 * HALO) {
                    if (writer) {
                        *reinterpret_cast<float4*>(oc + o4c) = make_float4(val[0], val[1], val[2], val[3]);
                        const int yo = r0 + st_i - 2 * HALO;
                        if (yo >= G.rlo && yo < G.rhi)
#pragma unroll
                            for (int j = 0; j < 4; ++j) dotp += static_cast<double>(pm4[j]) * static_cast<double>(val[j]);
                    }
                    if (CG && (--blk_left == 0 || st_i + 1 == steps)) {
                        const double ws = warp_sum(dotp);
                        const int yo = r0 + st_i - 2 * HALO;
                        if (lane == 0) part[(static_cast<size_t>(ch) * nbands + band) * nrb + yo / RB] = ws;
                        dotp = 0.0;
                        blk_left = RB;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                pm4[j] = pm3[j]; pm3[j] = pm2[j]; pm2[j] = pm1[j]; pm1[j] = p0[j];
                Im3[j] = Im2[j]; Im2[j] = Im1[j];
                s3[j] = s2[j]; s2[j] = s1[j];
                hs_a[j] = hs_b[j]; hs_b[j] = hs1[j]; his_a[j] = his_b[j]; his_b[j] = his1[j];
                ha_a[j] = ha_b[j]; ha_b[j] = ha2[j]; hc_a[j] = hc_b[j]; hc_b[j] = hc2[j];
                M_a[j] = M_b[j]; M_b[j] = Mc[j];
            }
            r3 = r3 + 1 == H ? 0 : r3 + 1;
        }
    }
    if (CG) {
        unsigned int prev = 0;
        if (lane == 0) {
            __threadfence();
            prev = atomicAdd(&st[ch].cnt_a, 1u);
        }
        prev = __shfl_sync(FULL, prev, 0);
        if (prev == static_cast<unsigned int>(nblk) - 1u) {
            __threadfence();
            const double* pa = part + static_cast<size_t>(ch) * nbands * nrb;
            double sacc = 0.0;
#pragma unroll 8
            for (int i = lane; i < nbands * nrb; i += 32) sacc += __ldcg(pa + i);
            double pAp = warp_sum(sacc);
            if (lane == 0 && G.dred) {
                G.dred[ch] = DIN ? pAp : st[ch].qq + G.lambda * pAp;
                st[ch].cnt_a = 0;
            } else if (lane == 0) {
                CgState& S = st[ch];
                if constexpr (!DIN) pAp = S.qq + G.lambda * pAp;
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

}  // namespace fast
}  // namespace fbmp_gpu
