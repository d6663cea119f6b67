// fsr_warpn.cuh -- FSR kernels for the supports without a dedicated kernel:
// the paper grid's N = 4, 8, 24 (S in {4, 8, 16, 24, 32}; the
// sweep of cli.py:41-50) and every other even N <= 32, one warp per target
// block, lane v < N owning spectral column v.
//
//   warpn_kernel   fp32 loop with the near-tie guard -- fsr_warp32.cuh's design
//                  (read that header first) with the row pairs (i, i + N/2):
//                  P = N/2 packed pairs per lane, FFMA2 update + objective, one
//                  LDS.128 of the row-pair table U[k][c] = (Wx[k+P], Wx[k],
//                  Wy[k+P], Wy[k]) per pair at row P + i - (pu mod P), column
//                  (v - pv) mod N; pair keys (any maximal lane wins, every
//                  near-tie is re-run in fp64), a brx pick of the winning pair.
//                  Lanes v >= N (N < 32) compute a copy of column v mod N and
//                  never win (key 0).
//   warpnd_kernel  the same support in fp64: validation precision and the
//                  guarded mode's re-runs (list mode).  R[u][v] for the N rows
//                  in registers (N complex doubles), W in a row-doubled table
//                  W2[r] = W[r mod N] (no wrap: row u - pu + N), fused update +
//                  objective + 64-bit key whose low 10 bits hold the reference's
//                  tie rank of the flat bin (_kernels.py:12-59: tree or linear),
//                  so the cross-lane u64 max is the reference's argmax exactly.
//   prologue       (both) gather of the N x N window (TMA boxes or plain loads,
//                  outside = unknown), mask-gated rho^d weights, packed z = f w +
//                  i w, fp64 2-D DFT on an N x (N+1) double2 tile (N = 24 as
//                  8 x 3 mixed radix; other even N as one radix-2 step over two
//                  direct N/2-point DFTs with compile-time twiddles), Hermitian
//                  split into R and W.
#pragma once

#include "fsr_pair64.cuh"
#include "fsr_warp32.cuh"

namespace fsr {

// ---------------------------------------------------------------- N-point DFT
// cos(2 pi m / 24), m = 0..6; the rest by quadrant symmetry
__host__ __device__ constexpr double cos24q(int m) {
    return m == 0 ? 1.0
         : m == 1 ? 0.96592582628906828674974319972890
         : m == 2 ? 0.86602540378443864676372317075294
         : m == 3 ? 0.70710678118654752440084436210485
         : m == 4 ? 0.5
         : m == 5 ? 0.25881904510252076234889883762405
                  : 0.0;
}
__host__ __device__ constexpr double cos24(int m) {  // m in [0, 24)
    return m <= 6 ? cos24q(m) : m <= 12 ? -cos24q(12 - m) : m <= 18 ? -cos24q(m - 12) : cos24q(24 - m);
}
__host__ __device__ constexpr double sin24(int m) { return cos24((m + 18) % 24); }  // sin x = cos(x - pi/2)

// cos / sin (2 pi m / n) as compile-time constants for any n: the angle is
// reduced to an octant by exact integer arithmetic (k = floor(8m / n)), then a
// Taylor series on [0, pi/4] (error below the double rounding).
__host__ __device__ constexpr double taylor_cos(double x) {
    double s = 1.0, t = 1.0;
    for (int k = 1; k < 12; ++k) {
        t *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
        s += t;
    }
    return s;
}
__host__ __device__ constexpr double taylor_sin(double x) {
    double s = x, t = x;
    for (int k = 1; k < 12; ++k) {
        t *= -x * x / ((2.0 * k) * (2.0 * k + 1.0));
        s += t;
    }
    return s;
}
__host__ __device__ constexpr double cos2pi(long long m, long long n) {
    m = ((m % n) + n) % n;
    const long long k = (8 * m) / n, r = 8 * m - k * n;  // octant, remainder in [0, n)
    const double qp = 0.78539816339744830961566084581988;  // pi / 4
    const double phi = qp * (double)r / (double)n, phc = qp * (double)(n - r) / (double)n;
    switch (k) {
        case 0: return taylor_cos(phi);
        case 1: return taylor_sin(phc);
        case 2: return -taylor_sin(phi);
        case 3: return -taylor_cos(phc);
        case 4: return -taylor_cos(phi);
        case 5: return -taylor_sin(phc);
        case 6: return taylor_sin(phi);
        default: return taylor_cos(phc);
    }
}
__host__ __device__ constexpr double sin2pi(long long m, long long n) { return cos2pi(4 * m - n, 4 * n); }

// Direct M-point DFT of the strided subsequence x[off + 2 j] (j < M) into y.
template <int M, int OFF, typename T, int NX>
__device__ __forceinline__ void dft_half(const cpx<T> (&x)[NX], cpx<T> (&y)[M]) {
#pragma unroll
    for (int k = 0; k < M; ++k) {
        T re = 0, im = 0;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const cpx<T> a = x[OFF + 2 * j];
            const int m = (k * j) % M;
            if (m == 0) {
                re += a.re;
                im += a.im;
            } else {
                const T c = (T)cos2pi(m, M), sn = (T)sin2pi(m, M);  // (a.re + i a.im)(c - i sn)
                re += a.re * c + a.im * sn;
                im += a.im * c - a.re * sn;
            }
        }
        y[k] = {re, im};
    }
}

// x[k] <- sum_n x[n] e^{-2 pi i k n / N} (unnormalised, numpy.fft convention)
template <int N, typename T>
__device__ __forceinline__ void fft_line(cpx<T> (&x)[N]) {
    if constexpr (N == 4) {
        fft_pow2<2>(x);
    } else if constexpr (N == 8) {
        fft_pow2<3>(x);
    } else if constexpr (N == 16) {
        fft_pow2<4>(x);
    } else if constexpr (N != 24) {
        // any other even N: one radix-2 step over two direct N/2-point DFTs
        // (even / odd samples), X[k] = E[k] + W^k O[k], X[k + N/2] = E[k] - W^k O[k]
        static_assert(N % 2 == 0 && N <= 32, "fft_line: even N <= 32");
        constexpr int M = N / 2;
        cpx<T> e[M], o[M];
        dft_half<M, 0>(x, e);
        dft_half<M, 1>(x, o);
#pragma unroll
        for (int k = 0; k < M; ++k) {
            cpx<T> t = o[k];
            if (k != 0) {
                const T c = (T)cos2pi(k, N), sn = (T)sin2pi(k, N);
                t = {o[k].re * c + o[k].im * sn, o[k].im * c - o[k].re * sn};
            }
            x[k] = {e[k].re + t.re, e[k].im + t.im};
            x[k + M] = {e[k].re - t.re, e[k].im - t.im};
        }
    } else {
        // decimation in time by 3: y_r = FFT8(x[3m + r]); X[k1 + 8 k2] =
        // sum_r W3^{r k2} (W24^{r k1} y_r[k1])
        cpx<T> y[3][8];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
#pragma unroll
            for (int m = 0; m < 8; ++m) y[r][m] = x[3 * m + r];
            fft_pow2<3>(y[r]);
        }
        constexpr double h3 = 0.86602540378443864676372317075294;  // sqrt(3) / 2
#pragma unroll
        for (int k1 = 0; k1 < 8; ++k1) {
            cpx<T> z[3];
            z[0] = y[0][k1];
#pragma unroll
            for (int r = 1; r < 3; ++r) {
                const int m = r * k1;  // < 24
                const cpx<T> a = y[r][k1];
                if (m == 0) {
                    z[r] = a;
                } else {
                    const T c = (T)cos24(m), s = (T)sin24(m);  // (a.re + i a.im)(c - i s)
                    z[r] = {a.re * c + a.im * s, a.im * c - a.re * s};
                }
            }
            const T sr = z[1].re + z[2].re, si = z[1].im + z[2].im;
            const T dr = z[1].re - z[2].re, di = z[1].im - z[2].im;
            const T mr = z[0].re - 0.5 * sr, mi = z[0].im - 0.5 * si;
            x[k1] = {z[0].re + sr, z[0].im + si};
            // X1 = m - i h3 d, X2 = m + i h3 d
            x[k1 + 8] = {mr + (T)h3 * di, mi - (T)h3 * dr};
            x[k1 + 16] = {mr - (T)h3 * di, mi + (T)h3 * dr};
        }
    }
}

// Gather + fp64 2-D DFT of one N x N window into tile t (N x (N+1) double2):
// afterwards t[u * (N+1) + v] = Z[u][v] = F{f w}[u][v] + i F{w}[u][v].
// Returns the early-stop energy sum f^2 w of this lane's column (lanes < N).
template <int N, typename IO>
__device__ __forceinline__ double wn_window_dft(const Warp32Args &a, const Warp32Maps &maps,
                                                double2 *t, uint32_t bar, uint32_t &phase,
                                                int64_t wr0, int64_t wc0, int lane) {
    using Box = TmaBox<IO, N, N>;
    constexpr int TS = N + 1;
    const int cl = lane % N;  // lanes >= N shadow a real column
    IO pf[N];
    uint32_t mbits = 0;
    if (a.use_tma) {
        const int x0 = (int)wc0;
        const int xp = x0 & ~(Box::ALIGN - 1), xm = x0 & ~15;
        const IO *spx = reinterpret_cast<const IO *>(t);
        const uint8_t *smk = reinterpret_cast<const uint8_t *>(t) + Box::STAGE_MK;
        tma_window(maps, bar, smem_u32(spx), smem_u32(smk), xp, xm, (int)wr0 - a.tma_y0,
                   Box::TX_BYTES);
        mbar_wait(bar, phase);
        phase ^= 1u;
        const IO *cpx_ = spx + (x0 - xp) + cl;
        const uint8_t *cmk = smk + (x0 - xm) + cl;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            pf[k] = cpx_[k * Box::PX];
            mbits |= (uint32_t)(cmk[k * Box::MK] != 0) << k;
        }
        __syncwarp();
    } else {
        const int64_t x = wc0 + cl;
        const bool xin = x >= 0 && x < a.W;
        const IO *px = static_cast<const IO *>(a.px);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const int64_t y = wr0 + k;
            const bool in = xin && y >= 0 && y < a.H;
            pf[k] = in ? __ldg(px + y * a.px_pitch + x) : (IO)0;
            mbits |= (uint32_t)(in && __ldg(a.mask + y * a.mask_pitch + x) != 0) << k;
        }
    }
    double energy = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double f = 0.0, w = 0.0;
        if ((mbits >> k) & 1u) {
            f = (double)pf[k];
            w = __ldg(a.decay64 + k * N + cl);
        }
        if (lane < N) t[k * TS + lane] = make_double2(f * w, w);
        energy = fma(f * f, w, energy);
    }
    __syncwarp();
    if (lane < N) {  // rows (lane = row)
        cpx<double> xv[N];
#pragma unroll
        for (int j = 0; j < N; ++j) { const double2 z = t[lane * TS + j]; xv[j] = {z.x, z.y}; }
        fft_line<N>(xv);
#pragma unroll
        for (int j = 0; j < N; ++j) t[lane * TS + j] = make_double2(xv[j].re, xv[j].im);
    }
    __syncwarp();
    if (lane < N) {  // columns (lane = column)
        cpx<double> xv[N];
#pragma unroll
        for (int j = 0; j < N; ++j) { const double2 z = t[j * TS + lane]; xv[j] = {z.x, z.y}; }
        fft_line<N>(xv);
#pragma unroll
        for (int j = 0; j < N; ++j) t[j * TS + lane] = make_double2(xv[j].re, xv[j].im);
    }
    __syncwarp();
    return lane < N ? energy : 0.0;
}

template <int N>
struct WnCfg {
    static constexpr int P = N / 2;                      // row pairs per lane
    static constexpr int TILE = N * (N + 1) * 16;        // fp64 DFT tile (bytes)
    static constexpr int UTAB = N * N * 16;              // U row-pair table (bytes)
    static constexpr int STAGE = TmaBox<double, N, N>::STAGE_BYTES;
    static constexpr int BYTES = (TILE > UTAB ? (TILE > STAGE ? TILE : STAGE) : (UTAB > STAGE ? UTAB : STAGE));
    static constexpr int F4 = (BYTES + 127) / 128 * 8;   // per-warp buffer in float4, 128 B
                                                         // multiple: every warp's TMA staging
                                                         // must start 128-byte aligned
};

template <int N, int WARPS>
struct WarpNSmem {
    float4 ubuf[WARPS][WnCfg<N>::F4];
    unsigned int red_key[WARPS][32];  // AM_SMEM scratch
    unsigned int red_rank[WARPS][32];
    unsigned long long bar[WARPS];
    float2 cs[N];                     // cos / sin (2 pi j / N)
};

// Row pair j of this lane: q = (Re lo, Re hi, Im lo, Im hi), wfp = (wf lo, wf hi);
// j warp-uniform (a switch the compiler lowers to one indirect branch).
template <int P>
__device__ __forceinline__ float4 pick_pairn(const float2 (&re)[P], const float2 (&im)[P],
                                             const float2 (&wf2)[P], int j, float2 &wfp) {
    float4 q = make_float4(re[0].x, re[0].y, im[0].x, im[0].y);
    wfp = wf2[0];
    switch (j) {
#define FSR_PICKN(k)                                                              \
    case k:                                                                       \
        if constexpr (k < P) {                                                    \
            q = make_float4(re[k].x, re[k].y, im[k].x, im[k].y);                  \
            wfp = wf2[k];                                                         \
        }                                                                         \
        break;
        FSR_PICKN(1) FSR_PICKN(2) FSR_PICKN(3) FSR_PICKN(4) FSR_PICKN(5) FSR_PICKN(6)
        FSR_PICKN(7) FSR_PICKN(8) FSR_PICKN(9) FSR_PICKN(10) FSR_PICKN(11) FSR_PICKN(12)
        FSR_PICKN(13) FSR_PICKN(14) FSR_PICKN(15)
#undef FSR_PICKN
        default: break;
    }
    return q;
}

// One objective/update pass over the lane's P row pairs (pair keys; see pass_x2).
template <int N, bool GUARD, bool HERM, bool UPDATE, bool SWAP>
__device__ __forceinline__ void passn(float2 (&re)[N / 2], float2 (&im)[N / 2], const float2 (&wf2)[N / 2],
                                      const float4 *up, float gr, float gi, uint32_t canon,
                                      uint32_t hmask, uint32_t &m1, uint32_t &m2) {
    constexpr int P = N / 2;
    m1 = 0;
    m2 = 0;
    uint32_t hpend = 0;
    const float2 ngr = make_float2(-gr, -gr), pgi = make_float2(gi, gi), ngi = make_float2(-gi, -gi);
#pragma unroll
    for (int i = 0; i < P; ++i) {
        float2 r = re[i], m = im[i];
        if (UPDATE) {
            const float4 w = up[i * N];  // U[P + i - pu % P][(v - pv) mod N]
            const float2 wx = SWAP ? make_float2(w.y, w.x) : make_float2(w.x, w.y);
            const float2 wy = SWAP ? make_float2(w.w, w.z) : make_float2(w.z, w.w);
            r = __ffma2_rn(wx, ngr, r);
            r = __ffma2_rn(wy, pgi, r);
            m = __ffma2_rn(wy, ngr, m);
            m = __ffma2_rn(wx, ngi, m);
            re[i] = r;
            im[i] = m;
        }
        const float2 mag = __ffma2_rn(r, r, __fmul2_rn(m, m));
        const float2 o = __fmul2_rn(mag, wf2[i]);
        float ox = o.x, oy = o.y;
        if (HERM) {
            ox = ((canon >> i) & 1u) ? ox : 0.f;
            oy = ((canon >> (i + P)) & 1u) ? oy : 0.f;
        }
        const uint32_t h = and_or(f2u(fmaxf(ox, oy)), hmask, (uint32_t)i);
        if (!GUARD) {
            m1 = max(m1, h);
        } else if ((i & 1) == 0) {
            hpend = h;
        } else {
            const uint32_t hmax = max(hpend, h), hmin = min(hpend, h);
            m2 = umax3(m2, hmin, min(m1, hmax));
            m1 = max(m1, hmax);
        }
    }
    if (GUARD && (P & 1)) {  // odd pair count (N = 2 mod 4): the last pair is still pending
        m2 = max(m2, min(m1, hpend));
        m1 = max(m1, hpend);
    }
}

// resident warps (blocks) per SM the register budget targets
#ifndef FSR_WN_WPS_24
#define FSR_WN_WPS_24 12  // 1080p: 12 -> 164 fps, 16 -> 158
#endif
#ifndef FSR_WN_WPS_SMALL
#define FSR_WN_WPS_SMALL 24  // N = 8 at 1080p: 24 -> 392 fps, 16 -> 365
#endif
template <int N>
constexpr int wn_warps_per_sm() { return N >= 24 ? FSR_WN_WPS_24 : FSR_WN_WPS_SMALL; }
template <typename IO, int N, int WARPS, int ARGMAX, bool GUARD, int OPTS>
__global__ void __launch_bounds__(WARPS * 32, wn_warps_per_sm<N>() / WARPS)
    warpn_kernel(Warp32Args a, const __grid_constant__ Warp32Maps maps) {
    constexpr int P = N / 2;
    constexpr bool TRACE = (OPTS & W32_TRACE) != 0, EARLY = (OPTS & W32_EARLY) != 0;
    constexpr bool KAPPA = (OPTS & W32_KAPPA) != 0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpNSmem<N, WARPS> &sm = *reinterpret_cast<WarpNSmem<N, WARPS> *>(smem_raw);
    constexpr bool REC = GUARD && (OPTS & W32_REPLAY) != 0;  // replay records (see warp32)
    uint16_t *seqw = REC ? reinterpret_cast<uint16_t *>(smem_raw + sizeof(WarpNSmem<N, WARPS>)) +
                               warp_id() * a.seq_stride
                         : nullptr;
    const int lane = lane_id(), wid = warp_id();
    if (threadIdx.x < N) {
        const double th = 6.283185307179586476925286766559 * threadIdx.x / N;
        sm.cs[threadIdx.x] = make_float2((float)cos(th), (float)sin(th));
    }
    const uint32_t bar = smem_u32(&sm.bar[wid]);
    if (lane == 0) mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t phase = 0;
    float4 *ub = sm.ubuf[wid];
    double2 *t = reinterpret_cast<double2 *>(ub);
    const int v = lane % N;  // spectral column (lanes >= N shadow column lane - N and never win)
    const bool live_lane = lane < N;
    // canonical half of each mirror pair (the lower tie rank of the reducer,
    // _kernels.py:12-59): bit u = row u of this lane's column
    uint32_t canon = 0;
#pragma unroll
    for (int u = 0; u < N; ++u) {
        const int tt = u * N + v, mt = ((N - u) % N) * N + ((N - v) % N);
        canon |= (uint32_t)(tie_rank(tt, a.tree != 0) <= tie_rank(mt, a.tree != 0)) << u;
    }
    float2 wf2[P];
#pragma unroll
    for (int i = 0; i < P; ++i) wf2[i] = make_float2(__ldg(a.wf + i * N + v), __ldg(a.wf + (i + P) * N + v));

    const int64_t total_warps = (int64_t)gridDim.x * WARPS;
    for (int64_t bi = (int64_t)blockIdx.x * WARPS + wid; bi < a.nblocks; bi += total_warps) {
        const int64_t bid = a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const float energy = (float)wn_window_dft<N, IO>(a, maps, t, bar, phase, r0 - a.L, c0 - a.L, lane);
        // split: R = (Z + conj Z(-u,-v)) / 2, W = (Z - conj Z(-u,-v)) / 2i, rounded to fp32 once
        float2 re[P], im[P];
        float2 Wf[N];
        {
            constexpr int TS = N + 1;
            const int mv = (N - v) % N;
#pragma unroll
            for (int u = 0; u < N; ++u) {
                const int nu = (N - u) % N;
                const double2 z = t[u * TS + v], zm = t[nu * TS + mv];
                const float rr = (float)((z.x + zm.x) * 0.5), ri = (float)((z.y - zm.y) * 0.5);
                if (u < P) {
                    re[u].x = rr;
                    im[u].x = ri;
                } else {
                    re[u - P].y = rr;
                    im[u - P].y = ri;
                }
                Wf[u] = make_float2((float)((z.y + zm.y) * 0.5), (float)((zm.x - z.x) * 0.5));
            }
        }
        __syncwarp();
        // U[k][c] = (Wx[k+P], Wx[k], Wy[k+P], Wy[k]) (rows mod N), row stride N float4
        if (live_lane) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const int k2 = (k + P) % N;
                ub[k * N + v] = make_float4(Wf[k2].x, Wf[k].x, Wf[k2].y, Wf[k].y);
            }
        }
        __syncwarp();
        const float w00 = ub[P * N].x;  // U[P][0].x = Wx[0][0] = sum of the weights
        int32_t *sel_b = (TRACE && a.sel) ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (!(w00 > 0.f)) {  // empty support (reconstruction.py:272-275)
            if (lane == 0) {
                unsigned slot = atomicAdd(a.empty_count, 1u);
                a.empty_list[slot] = (int32_t)bid;
                if (a.done) a.done[bid] = 0;
            }
            if (sel_b)
                for (int it = lane; it < a.iterations; it += 32) sel_b[it] = -1;
            __syncwarp();
            continue;
        }
        float thr = 0.f;
        if (EARLY && a.early_stop) {
            float e = energy;
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
            thr = 1e-12f * e;
        }
        const float ginv = a.gamma / w00;
        const int pm = a.L + lane / a.B, pn = a.L + lane % a.B;
        float acc = 0.f;
        bool herm = true, flagged = false;
        float gr = 0.f, gi = 0.f;
        int pu = 0, pv = 0;
        int it = 0;
        float fl = -1.f, ks = 0.f;
        int kf = -1;  // REC: the first flagged iteration
        auto step = [&](auto hconst) -> bool {
            constexpr bool H = decltype(hconst)::value;
            uint32_t m1, m2;
            int col = v - pv;
            col += col < 0 ? N : 0;
            const int pr = pu >= P ? pu - P : pu;
            const float4 *up = ub + (P - pr) * N + col;
            if (H && it == 0) {
                passn<N, GUARD, true, false, false>(re, im, wf2, up, gr, gi, canon, a.key_mask, m1, m2);
            } else if (pu >= P) {
                passn<N, GUARD, H, true, true>(re, im, wf2, up, gr, gi, canon, a.key_mask, m1, m2);
            } else {
                passn<N, GUARD, H, true, false>(re, im, wf2, up, gr, gi, canon, a.key_mask, m1, m2);
            }
            if (!live_lane) m1 = m2 = 0u;
            uint32_t kmax;
            int wl;
            cross_lane_best<ARGMAX, true>(m1, kmax, wl, sm.red_key[wid], sm.red_rank[wid]);
            const int j = (int)(kmax & 31u);  // the winning pair
            const float b1 = __uint_as_float(kmax & ~31u);
            if (EARLY && b1 < thr) {
                if (GUARD && b1 >= thr * a.omt) {
                    flagged = true;
                    if (REC && kf < 0) kf = it;
                }
                return false;
            }
            float2 wfp;
            const float4 q = pick_pairn<P>(re, im, wf2, j, wfp);
            // which half of the winning pair: both objectives recomputed as the pass did
            float olo = fmaf(q.x, q.x, q.z * q.z) * wfp.x, ohi = fmaf(q.y, q.y, q.w * q.w) * wfp.y;
            if (H) {
                olo = ((canon >> j) & 1u) ? olo : 0.f;
                ohi = ((canon >> (j + P)) & 1u) ? ohi : 0.f;
            }
            const bool hl = ohi > olo;
            const float po = hl ? olo : ohi;  // the pair partner
            float2 c = hl ? make_float2(q.y, q.w) : make_float2(q.x, q.z);
            const bool hi = __shfl_sync(0xffffffffu, (int)hl, wl) != 0;
            const int bu = j + (hi ? P : 0), bv = wl % N;
            if (TRACE && sel_b && lane == 0) sel_b[it] = bu * N + bv;
            if (REC) seqw[it] = (uint16_t)(bu * N + bv);  // uniform: every lane stores it (see warp32)
            c.x = __shfl_sync(0xffffffffu, c.x, wl);
            c.y = __shfl_sync(0xffffffffu, c.y, wl);
            const float2 cs = sm.cs[(bu * pm + bv * pn) % N];
            gr = c.x * ginv;
            gi = c.y * ginv;
            acc = fmaf(gr, cs.x, fmaf(-gi, cs.y, acc));
            pu = bu;
            pv = bv;
            if (GUARD) {
                const uint32_t kp = f2u(po) & a.key_mask;
                // per-lane test on the lane's own b2 candidate, warp OR after the loop
                // (no second reduction in the iteration chain; see warp32)
                const float b2 = __uint_as_float((lane == wl ? max(m2, kp) : m1) & ~31u);
                float gtest;
                if (KAPPA) {
                    const float sb1 = sqrt_approx(b1);
                    if (H && it == 0) ks = a.kappa * sb1;
                    gtest = b2 - fmaf(-ks, sb1, __fmul_rn(b1, a.omt));
                } else {
                    gtest = b2 - __fmul_rn(b1, a.omt);
                }
                fl = fmaxf(fl, gtest);
                if (REC && kf < 0 && gtest >= 0.f) kf = it;
                if (EARLY) {
                    const bool near_stop = b1 * a.omt < thr;
                    flagged |= near_stop;
                    if (REC && near_stop && kf < 0) kf = it;
                }
            }
            if (H) herm = (bu % (N / 2) == 0) && (bv % (N / 2) == 0);
            return true;
        };
        bool live = true;
        while (live && herm && it < a.iterations) {
            if (step(std::true_type{})) ++it; else live = false;
        }
        while (live && it < a.iterations) {
            if (step(std::false_type{})) ++it; else live = false;
            // replay build: a flagged block's remaining fp32 iterations are wasted
            // work (its fp64 re-run replays only the prefix), see warp32
            if (REC && (it & 3) == 0 && __any_sync(0xffffffffu, fl >= 0.f)) break;
        }
        flagged |= __any_sync(0xffffffffu, fl >= 0.f);  // per-lane guard tests (see warp32)
        if (REC) {  // the first flagged iteration over the lanes
            const uint32_t k = __reduce_min_sync(0xffffffffu, kf < 0 ? 0xffffffffu : (uint32_t)kf);
            kf = k == 0xffffffffu ? -1 : (int)k;
        }
        const int done = it;
        if (sel_b)
            for (int jj = done + lane; jj < a.iterations; jj += 32) sel_b[jj] = -1;
        if (lane == 0 && a.done) a.done[bid] = done;
        if (GUARD && flagged && a.rerun_list) {
            unsigned slot = 0;
            if (lane == 0) {
                slot = atomicAdd(a.rerun_count, 1u);
                a.rerun_list[slot] = (int32_t)bid;
            }
            if (REC) {
                slot = __shfl_sync(0xffffffffu, slot, 0);
                const int n = kf < 0 ? 0 : min(kf, a.seq_stride);
                if (lane == 0) a.rerun_kf[slot] = n;
                __syncwarp();
                uint16_t *dst = a.rerun_seq + (int64_t)slot * a.seq_stride;
                for (int jj = lane; jj < n; jj += 32) dst[jj] = seqw[jj];
            }
        }
        if (lane < a.B * a.B) {
            const int m = lane / a.B, n = lane % a.B;
            const int64_t y = r0 + m, xx = c0 + n;
            if (y < a.H && xx < a.W)
                static_cast<IO *>(a.out)[y * a.out_pitch + xx] =
                    a.mask[y * a.mask_pitch + xx] ? static_cast<const IO *>(a.px)[y * a.px_pitch + xx] : (IO)acc;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- fp64 kernel
template <int N, int WARPS>
struct WarpNdSmem {
    double2 buf[WARPS][(2 * N * N > N * (N + 1) ? 2 * N * N : N * (N + 1))];  // tile, then W2
    unsigned int red_hi[WARPS][32];
    unsigned int red_lo[WARPS][32];
    double2 cs[N];
};

// tie rank of flat bin t (_kernels.py:12-59) and its inverse (bitrev5 is an involution)
__host__ __device__ __forceinline__ int rank_to_bin(int r, bool tree) {
    return tree ? (int)((bitrev5((uint32_t)r >> 5) << 5) | bitrev5((uint32_t)r & 31u)) : r;
}

template <int N, int WARPS, int ARGMAX, typename IO>
__global__ void __launch_bounds__(WARPS * 32) warpnd_kernel(Pair64Args<IO> a) {
    const bool TREE = a.tree != 0;
    constexpr int TS = N + 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpNdSmem<N, WARPS> &sm = *reinterpret_cast<WarpNdSmem<N, WARPS> *>(smem_raw);
    if (threadIdx.x < N) {
        double sn, cn;
        sincospi(2.0 * threadIdx.x / N, &sn, &cn);
        sm.cs[threadIdx.x] = make_double2(cn, sn);
    }
    __syncthreads();
    const int lane = lane_id(), wid = warp_id();
    double2 *t = sm.buf[wid];
    const int v = lane % N;
    const bool live_lane = lane < N;
    // 1023 - rank(u N + v) for u = 0..N-1, three 10-bit fields per word
    uint32_t rk[(N + 2) / 3];
#pragma unroll
    for (int q = 0; q < (N + 2) / 3; ++q) rk[q] = 0;
#pragma unroll
    for (int u = 0; u < N; ++u) rk[u / 3] |= (uint32_t)(1023 - tie_rank(u * N + v, TREE)) << (10 * (u % 3));
    double wfr[N];
#pragma unroll
    for (int u = 0; u < N; ++u) wfr[u] = a.wf[u * N + v];

    const int64_t nblocks = a.list_count ? (int64_t)*a.list_count : a.nblocks;
    const int64_t stride = (int64_t)gridDim.x * WARPS;
    for (int64_t bi = (int64_t)blockIdx.x * WARPS + wid; bi < nblocks; bi += stride) {
        const int64_t bid = a.list ? (int64_t)a.list[bi] : a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const int64_t wr0 = r0 - a.L, x = c0 - a.L + v;
        const bool xin = x >= 0 && x < a.W;
        double energy = 0.0;
#pragma unroll 4
        for (int k = 0; k < N; ++k) {
            const int64_t y = wr0 + k;
            double f = 0.0, w = 0.0;
            if (xin && y >= 0 && y < a.H && a.mask[y * a.mask_pitch + x]) {
                f = load_px(a.px + y * a.px_pitch + x);
                w = a.decay[k * N + v];
            }
            if (live_lane) t[k * TS + lane] = make_double2(f * w, w);
            energy = fma(f * f, w, energy);
        }
        if (!live_lane) energy = 0.0;
        __syncwarp();
        cpx<double> R[N];
        if (live_lane) {  // rows
#pragma unroll
            for (int j = 0; j < N; ++j) { const double2 z = t[lane * TS + j]; R[j] = {z.x, z.y}; }
            fft_line<N>(R);
#pragma unroll
            for (int j = 0; j < N; ++j) t[lane * TS + j] = make_double2(R[j].re, R[j].im);
        }
        __syncwarp();
        if (live_lane) {  // columns
#pragma unroll
            for (int j = 0; j < N; ++j) { const double2 z = t[j * TS + lane]; R[j] = {z.x, z.y}; }
            fft_line<N>(R);
#pragma unroll
            for (int j = 0; j < N; ++j) t[j * TS + lane] = make_double2(R[j].re, R[j].im);
        }
        __syncwarp();
        // split: R in registers (column v), W to registers, then the row-doubled table W2
        double2 Wc[N];
        {
            const int mv = (N - v) % N;
#pragma unroll
            for (int u = 0; u < N; ++u) {
                const int nu = (N - u) % N;
                const double2 z = t[u * TS + v], zm = t[nu * TS + mv];
                R[u] = {(z.x + zm.x) * 0.5, (z.y - zm.y) * 0.5};
                Wc[u] = make_double2((z.y + zm.y) * 0.5, (zm.x - z.x) * 0.5);
            }
        }
        __syncwarp();
        if (live_lane) {
#pragma unroll
            for (int u = 0; u < N; ++u) {
                t[u * N + v] = Wc[u];
                t[(u + N) * N + v] = Wc[u];
            }
        }
        __syncwarp();
        const double w00 = t[0].x;
        int32_t *sel_b = a.sel ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (!(w00 > 0.0)) {
            if (lane == 0) {
                unsigned slot = atomicAdd(a.empty_count, 1u);
                if (a.empty_list) a.empty_list[slot] = (int32_t)bid;
                if (a.done) a.done[bid] = 0;
            }
            if (sel_b)
                for (int it = lane; it < a.iterations; it += 32) sel_b[it] = -1;
            __syncwarp();
            continue;
        }
        double thr = 0.0;
        if (a.early_stop) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, off);
            thr = 1e-12 * energy;
        }
        const double ginv = a.gamma / w00;
        const int B = a.B;
        const int pm = a.L + lane / B, pn = a.L + lane % B;
        const bool has_pix = lane < B * B;
        double acc = 0.0, gr = 0.0, gi = 0.0;
        int pu = 0, pv = 0;
        int done = 0;
        // replay (list mode): iterations < kf follow the fp32 kernel's recorded
        // selections with the update alone (see fsr_pair64.cuh)
        const int kf = a.list_kf ? a.list_kf[bi] : 0;
        const uint16_t *seq = a.list_kf ? a.list_seq + bi * (int64_t)a.seq_stride : nullptr;
        for (int it = 0; it < kf; ++it) {
            if (it > 0) {
                int col = v - pv;
                col += col < 0 ? N : 0;
                const double2 *wp = t + (N - pu) * N + col;
#pragma unroll
                for (int u = 0; u < N; ++u) {
                    const double2 w = wp[u * N];
                    double re = R[u].re, im = R[u].im;
                    re = fma(-gr, w.x, re);
                    re = fma(gi, w.y, re);
                    im = fma(-gr, w.y, im);
                    im = fma(-gi, w.x, im);
                    R[u].re = re;
                    R[u].im = im;
                }
            }
            const uint32_t s = seq[it];
            const int bu = (int)(s / N), bv = (int)(s - (s / N) * N);
            if (sel_b && lane == 0) sel_b[it] = bu * N + bv;
            double2 c = make_double2(R[0].re, R[0].im);
#pragma unroll
            for (int u = 1; u < N; ++u)
                if (u == bu) c = make_double2(R[u].re, R[u].im);
            c.x = __shfl_sync(0xffffffffu, c.x, bv);
            c.y = __shfl_sync(0xffffffffu, c.y, bv);
            gr = c.x * ginv;
            gi = c.y * ginv;
            pu = bu;
            pv = bv;
            if (has_pix) {
                const double2 e = sm.cs[(bu * pm + bv * pn) % N];
                acc = fma(gr, e.x, fma(-gi, e.y, acc));
            }
            done = it + 1;
        }
        for (int it = kf; it < a.iterations; ++it) {
            int col = v - pv;
            col += col < 0 ? N : 0;
            const double2 *wp = t + (N - pu) * N + col;  // row u - pu + N of W2
            unsigned long long best[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
            for (int u = 0; u < N; ++u) {
                double re = R[u].re, im = R[u].im;
                if (it > 0) {
                    const double2 w = wp[u * N];
                    re = fma(-gr, w.x, re);
                    re = fma(gi, w.y, re);
                    im = fma(-gr, w.y, im);
                    im = fma(-gi, w.x, im);
                    R[u].re = re;
                    R[u].im = im;
                }
                const double o = fma(re, re, im * im) * wfr[u];
                const uint32_t rkf = (rk[u / 3] >> (10 * (u % 3))) & 1023u;
                const uint32_t lo = ((uint32_t)__double2loint(o) & ~1023u) | rkf;
                const unsigned long long k =
                    ((unsigned long long)(uint32_t)__double2hiint(o) << 32) | (unsigned long long)lo;
                best[u & 3] = u64max(best[u & 3], k);
            }
            unsigned long long kb = u64max(u64max(best[0], best[1]), u64max(best[2], best[3]));
            if (!live_lane) kb = 0ull;
            const unsigned long long key = p64_warp_max<ARGMAX>(kb, sm.red_hi[wid], sm.red_lo[wid]);
            const int tb = rank_to_bin(1023 - (int)((uint32_t)key & 1023u), TREE);
            const int bu = tb / N, bv = tb - (tb / N) * N;
            if (sel_b && lane == 0) sel_b[it] = bu * N + bv;
            if (thr > 0.0 && __longlong_as_double((long long)key) < thr) break;
            double2 c = make_double2(R[0].re, R[0].im);
#pragma unroll
            for (int u = 1; u < N; ++u)
                if (u == bu) c = make_double2(R[u].re, R[u].im);
            c.x = __shfl_sync(0xffffffffu, c.x, bv);
            c.y = __shfl_sync(0xffffffffu, c.y, bv);
            gr = c.x * ginv;
            gi = c.y * ginv;
            pu = bu;
            pv = bv;
            if (has_pix) {
                const double2 e = sm.cs[(bu * pm + bv * pn) % N];
                acc = fma(gr, e.x, fma(-gi, e.y, acc));
            }
            done = it + 1;
        }
        if (sel_b)
            for (int it = done + lane; it < a.iterations; it += 32) sel_b[it] = -1;
        if (lane == 0 && a.done) a.done[bid] = done;
        if (has_pix) {
            const int m = lane / B, n = lane % B;
            const int64_t y = r0 + m, xx = c0 + n;
            if (y < a.H && xx < a.W)
                a.out[y * a.out_pitch + xx] =
                    a.mask[y * a.mask_pitch + xx] ? a.px[y * a.px_pitch + xx] : (IO)acc;
        }
        __syncwarp();
    }
}

}  // namespace fsr
