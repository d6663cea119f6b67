// fsr_warpseg.cuh -- fp32 loop kernel for the small supports N = 4, 8 and 16
// with 32 / N target blocks per warp ("segments" of N lanes, one block each).
//
// fsr_warpn.cuh gives a small support one warp per block, so at N = 8 three
// quarters of the lanes idle and the per-iteration argmax tail is paid per
// block.  Here every lane owns spectral column v = lane % N of block
// lane / N, so all 32 lanes work and one tail serves 32 / N blocks:
//   per lane   P = N/2 packed row pairs (i, i + P), FFMA2 update + objective,
//              one LDS.128 per pair from the segment's row-pair table.  warp32
//              swaps the float4 halves for pu >= P (warp-uniform there); here
//              pu differs between segments, so the table is extended by P rows
//              (U[N + k] = U[k]): since U[k + P] is U[k] with its halves
//              swapped, pair i reads row i + P - pu + (pu >= P ? N : 0), which
//              never wraps and never needs the swap
//   keys       the pair's larger objective with the pair index in the 5 low
//              bits; a log2(N)-step xor butterfly (never leaves the segment)
//              gives the segment's maximum and a ballot its lane; any maximal
//              bin may win (guarded: every near-tie is re-run in fp64; the
//              Hermitian phase keeps the canonical halves)
//   pick       the winning pair by a select chain (the pair differs between
//              segments, so no warp-uniform indirect branch)
//   guard      per-lane top-2 of the pair maxima, the winner's partner
//              recomputed, a second butterfly for b2 -- as warp32
//   prologue   plain loads (lane = window column of its block), fp64 2-D DFT
//              on the segment's N x (N+1) tile, Hermitian split
// Segments past the end of the work, empty-support windows and early-stopped
// blocks keep running in lock step with zero keys and no output.
#pragma once

#include "fsr_warpn.cuh"

namespace fsr {

template <int N>
struct SegCfg {
    static constexpr int P = N / 2;
    static constexpr int BPW = 32 / N;                 // blocks (segments) per warp
    static constexpr uint32_t KMASK = ~31u;            // 5 low key bits: the pair index
    static constexpr uint32_t SEGMASK = N == 32 ? 0xffffffffu : (1u << N) - 1u;
    static constexpr int TILE = N * (N + 1) * 16;
    static constexpr int UROWS = 3 * P;                // row-pair table rows, extended (below)
    static constexpr int UTAB = UROWS * N * 16;
    static constexpr int SEG = TILE > UTAB ? TILE : UTAB;  // bytes per segment
    static constexpr int SEG_F4 = SEG / 16;
    static constexpr int NPIX = (16 + N - 1) / N;      // target pixels per lane (B <= 4)
    static_assert(N == 4 || N == 8 || N == 16, "segmented kernel: N in {4, 8, 16}");
    static_assert(P <= 32, "the pair index fits the 5 key bits");
};

template <int N, int WARPS>
struct WarpSegSmem {
    float4 seg[WARPS][SegCfg<N>::BPW][SegCfg<N>::SEG_F4];
    float2 cs[N];
};

// max over the N lanes of this lane's segment (xor offsets < N stay inside it)
template <int N>
__device__ __forceinline__ uint32_t seg_max(uint32_t k) {
#pragma unroll
    for (int off = N / 2; off >= 1; off >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, off));
    return k;
}

template <int N, bool GUARD, bool HERM, bool UPDATE, uint32_t KMASK>
__device__ __forceinline__ void seg_pass(float2 (&re)[N / 2], float2 (&im)[N / 2], const float2 (&wf2)[N / 2],
                                         const float4 *up, float gr, float gi, uint32_t canon,
                                         uint32_t &m1, uint32_t &m2) {
    constexpr int P = N / 2;
    m1 = 0;
    m2 = 0;
    uint32_t hpend = 0;
    const float2 ngr = make_float2(-gr, -gr), pgi = make_float2(gi, gi), ngi = make_float2(-gi, -gi);
#pragma unroll
    for (int i = 0; i < P; ++i) {
        float2 r = re[i], m = im[i];
        if (UPDATE) {
            const float4 w = up[i * N];
            const float2 wx = make_float2(w.x, w.y), wy = make_float2(w.z, w.w);
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
        const uint32_t h = and_or(f2u(fmaxf(ox, oy)), KMASK, (uint32_t)i);  // the pair index
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
    if (GUARD && (P & 1)) {  // odd pair count: the last pair is still pending
        m2 = max(m2, min(m1, hpend));
        m1 = max(m1, hpend);
    }
}

#ifndef FSR_SEG_WARPS_PER_SM
#define FSR_SEG_WARPS_PER_SM 32     // N <= 8 (64 registers)
#endif
#ifndef FSR_SEG16_WARPS_PER_SM
#define FSR_SEG16_WARPS_PER_SM 16   // N = 16: 12 KiB of tables per warp
#endif
template <int N>
constexpr int seg_warps_per_sm() { return N == 16 ? FSR_SEG16_WARPS_PER_SM : FSR_SEG_WARPS_PER_SM; }
template <typename IO, int N, int WARPS, bool GUARD, int OPTS>
__global__ void __launch_bounds__(WARPS * 32, seg_warps_per_sm<N>() / WARPS)
    warpseg_kernel(Warp32Args a) {
    using C = SegCfg<N>;
    constexpr int P = C::P;
    constexpr bool TRACE = (OPTS & W32_TRACE) != 0, EARLY = (OPTS & W32_EARLY) != 0;
    constexpr bool KAPPA = (OPTS & W32_KAPPA) != 0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpSegSmem<N, WARPS> &sm = *reinterpret_cast<WarpSegSmem<N, WARPS> *>(smem_raw);
    const int lane = lane_id(), wid = warp_id();
    if (threadIdx.x < N) {
        const double th = 6.283185307179586476925286766559 * threadIdx.x / N;
        sm.cs[threadIdx.x] = make_float2((float)cos(th), (float)sin(th));
    }
    __syncthreads();
    const int sg = lane / N, v = lane % N, sbase = sg * N;
    float4 *segbuf = sm.seg[wid][sg];
    double2 *t = reinterpret_cast<double2 *>(segbuf);
    float4 *U = segbuf;  // row-pair table, 3P rows (rows N.. repeat rows 0..P-1)
    uint32_t canon = 0;
#pragma unroll
    for (int u = 0; u < N; ++u) {
        const int tt = u * N + v, mt = ((N - u) % N) * N + ((N - v) % N);
        canon |= (uint32_t)(tie_rank(tt, a.tree != 0) <= tie_rank(mt, a.tree != 0)) << u;
    }
    float2 wf2[P];
#pragma unroll
    for (int i = 0; i < P; ++i) wf2[i] = make_float2(__ldg(a.wf + i * N + v), __ldg(a.wf + (i + P) * N + v));
    const int64_t stride = (int64_t)gridDim.x * WARPS * C::BPW;
    for (int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * C::BPW; base < a.nblocks; base += stride) {
        const int64_t bi = base + sg;
        const bool real = bi < a.nblocks;
        const int64_t bid = a.first + (real ? bi : a.nblocks - 1);
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        // ---- gather (lane = window column of its block) + fp64 2-D DFT in the segment's tile
        constexpr int TS = N + 1;
        const int64_t wr0 = r0 - a.L, x = c0 - a.L + v;
        const bool xin = x >= 0 && x < a.W;
        double energy = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const int64_t y = wr0 + k;
            double f = 0.0, w = 0.0;
            if (xin && y >= 0 && y < a.H && __ldg(a.mask + y * a.mask_pitch + x)) {
                f = (double)__ldg(static_cast<const IO *>(a.px) + y * a.px_pitch + x);
                w = __ldg(a.decay64 + k * N + v);
            }
            t[k * TS + v] = make_double2(f * w, w);
            energy = fma(f * f, w, energy);
        }
        __syncwarp();
        {
            cpx<double> xv[N];
#pragma unroll
            for (int j = 0; j < N; ++j) { const double2 z = t[v * TS + j]; xv[j] = {z.x, z.y}; }
            fft_line<N>(xv);
#pragma unroll
            for (int j = 0; j < N; ++j) t[v * TS + j] = make_double2(xv[j].re, xv[j].im);
        }
        __syncwarp();
        {
            cpx<double> xv[N];
#pragma unroll
            for (int j = 0; j < N; ++j) { const double2 z = t[j * TS + v]; xv[j] = {z.x, z.y}; }
            fft_line<N>(xv);
#pragma unroll
            for (int j = 0; j < N; ++j) t[j * TS + v] = make_double2(xv[j].re, xv[j].im);
        }
        __syncwarp();
        float2 re[P], im[P], Wf[N];
        {
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
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const int k2 = (k + P) % N;
            U[k * N + v] = make_float4(Wf[k2].x, Wf[k].x, Wf[k2].y, Wf[k].y);
            if (k < P) U[(k + N) * N + v] = make_float4(Wf[k2].x, Wf[k].x, Wf[k2].y, Wf[k].y);
        }
        __syncwarp();
        const float w00 = U[P * N].x;  // Wx[0][0] = sum of the weights
        const bool empty = !(w00 > 0.f);
        int32_t *sel_b = (TRACE && a.sel && real) ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (empty && real && v == 0) {  // empty support (reconstruction.py:272-275)
            unsigned slot = atomicAdd(a.empty_count, 1u);
            a.empty_list[slot] = (int32_t)bid;
            if (a.done) a.done[bid] = 0;
        }
        // early stop threshold: 1e-12 * sum f^2 w over the segment
        float thr = 0.f;
        if (EARLY && a.early_stop) {
            float e = (float)energy;
#pragma unroll
            for (int off = N / 2; off >= 1; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
            thr = 1e-12f * e;
        }
        const float ginv = empty ? 0.f : a.gamma / w00;
        float acc[C::NPIX];
        int pmq[C::NPIX], pnq[C::NPIX];
#pragma unroll
        for (int q = 0; q < C::NPIX; ++q) {
            acc[q] = 0.f;
            const int p = v + q * N;
            pmq[q] = a.L + p / a.B;
            pnq[q] = a.L + p % a.B;
        }
        bool live = real && !empty;  // this segment still selects (uniform within it)
        bool herm = true, flagged = false;
        float gr = 0.f, gi = 0.f, fl = -1.f, ks = 0.f;
        int pu = 0, pv = 0, done = 0;
        auto step = [&](auto hconst, int it) {
            constexpr bool H = decltype(hconst)::value;
            int col = v - pv;
            col += col < 0 ? N : 0;
            const float4 *up = U + (P - pu + (pu >= P ? N : 0)) * N + col;
            const uint32_t cn = (H && herm) ? canon : 0xffffffffu;
            uint32_t m1, m2;
            if (H && it == 0)
                seg_pass<N, GUARD, true, false, C::KMASK>(re, im, wf2, up, gr, gi, cn, m1, m2);
            else
                seg_pass<N, GUARD, H, true, C::KMASK>(re, im, wf2, up, gr, gi, cn, m1, m2);
            if (!live) m1 = m2 = 0u;
            const uint32_t kmax = seg_max<N>(m1);
            const uint32_t bal = (__ballot_sync(0xffffffffu, m1 == kmax) >> sbase) & C::SEGMASK;
            const int wl = __ffs(bal) - 1, j = (int)(kmax & 31u);
            const float b1 = __uint_as_float(kmax & C::KMASK);
            bool go = live;
            if (EARLY && live && b1 < thr) {
                if (GUARD && b1 >= thr * a.omt) flagged = true;
                live = go = false;
            }
            // the winning pair of this segment (differs between segments: a select chain)
            float4 q = make_float4(re[0].x, re[0].y, im[0].x, im[0].y);
            float2 wfp = wf2[0];
#pragma unroll
            for (int i = 1; i < P; ++i)
                if (i == j) {
                    q = make_float4(re[i].x, re[i].y, im[i].x, im[i].y);
                    wfp = wf2[i];
                }
            float olo = fmaf(q.x, q.x, q.z * q.z) * wfp.x, ohi = fmaf(q.y, q.y, q.w * q.w) * wfp.y;
            if (H) {
                olo = ((cn >> j) & 1u) ? olo : 0.f;
                ohi = ((cn >> (j + P)) & 1u) ? ohi : 0.f;
            }
            const bool hl = ohi > olo;
            const float po = hl ? olo : ohi;
            const int src = sbase + wl;
            const bool hi = __shfl_sync(0xffffffffu, (int)hl, src) != 0;
            float cr = __shfl_sync(0xffffffffu, hl ? q.y : q.x, src);
            float ci = __shfl_sync(0xffffffffu, hl ? q.w : q.z, src);
            const int bu = j + (hi ? P : 0), bv = wl;
            if (TRACE && sel_b && v == 0 && go) sel_b[it] = bu * N + bv;
            if (!go) cr = ci = 0.f;  // a stopped or idle segment applies no update
            gr = cr * ginv;
            gi = ci * ginv;
#pragma unroll
            for (int qq = 0; qq < C::NPIX; ++qq) {
                const float2 cs = sm.cs[(bu * pmq[qq] + bv * pnq[qq]) % N];
                acc[qq] = fmaf(gr, cs.x, fmaf(-gi, cs.y, acc[qq]));
            }
            if (go) {
                pu = bu;
                pv = bv;
                done = it + 1;
            }
            if (GUARD) {
                const uint32_t kp = f2u(po) & C::KMASK;
                // per-lane test on the lane's own b2 candidate, OR over the segment
                // after the loop (no butterfly in the iteration chain; see warp32)
                const float b2 = __uint_as_float((v == wl ? max(m2, kp) : m1) & C::KMASK);
                const float omt = a.omt;
                float gap;
                if (KAPPA) {
                    const float sb1 = sqrt_approx(b1);
                    if (H && it == 0) ks = a.kappa * sb1;
                    gap = b2 - fmaf(-ks, sb1, __fmul_rn(b1, omt));
                } else {
                    gap = b2 - __fmul_rn(b1, omt);
                }
                if (go) fl = fmaxf(fl, gap);
                if (EARLY && go) flagged |= b1 * a.omt < thr;
            }
            if (H && go) herm = herm && (bu % (N / 2) == 0) && (bv % (N / 2) == 0);
        };
        int it = 0;
        while (it < a.iterations && __any_sync(0xffffffffu, herm && live)) {
            step(std::true_type{}, it);
            ++it;
            if (EARLY && !__any_sync(0xffffffffu, live)) break;
        }
        while (it < a.iterations) {
            if (EARLY && !__any_sync(0xffffffffu, live)) break;
            step(std::false_type{}, it);
            ++it;
        }
        flagged |= ((__ballot_sync(0xffffffffu, fl >= 0.f) >> sbase) & C::SEGMASK) != 0u;
        if (sel_b)
            for (int jj = done + v; jj < a.iterations; jj += N) sel_b[jj] = -1;
        if (real && !empty && v == 0) {
            if (a.done) a.done[bid] = done;
            if (GUARD && flagged && a.rerun_list) {
                unsigned slot = atomicAdd(a.rerun_count, 1u);
                a.rerun_list[slot] = (int32_t)bid;
            }
        }
        if (real && !empty) {
#pragma unroll
            for (int qq = 0; qq < C::NPIX; ++qq) {
                const int p = v + qq * N;
                if (p < a.B * a.B) {
                    const int m = p / a.B, n = p % a.B;
                    const int64_t y = r0 + m, xx = c0 + n;
                    if (y < a.H && xx < a.W)
                        static_cast<IO *>(a.out)[y * a.out_pitch + xx] =
                            a.mask[y * a.mask_pitch + xx] ? static_cast<const IO *>(a.px)[y * a.px_pitch + xx]
                                                          : (IO)acc[qq];
                }
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- fp64 variant
// warpsegd: the same segmented layout in fp64 (N = 4, 8) for the validation
// precision and the guarded re-runs (list mode): R[u][v] for the N rows in
// registers, the segment's row-doubled W table (row u - pu + N, no wrap), 64-bit
// keys whose low 10 bits hold the reference's tie rank of the flat bin (unique
// within a block, so the segment butterfly's u64 max is the reference's argmax).
template <int N>
struct SegdCfg {
    static constexpr int BPW = 32 / N;
    static constexpr int TILE = N * (N + 1);           // double2
    static constexpr int W2 = 2 * N * N;               // double2
    static constexpr int SEG = TILE > W2 ? TILE : W2;  // double2 per segment
    static constexpr int NPIX = 16 / N;
};

template <int N, int WARPS>
struct WarpSegdSmem {
    double2 seg[WARPS][SegdCfg<N>::BPW][SegdCfg<N>::SEG];
    double2 cs[N];
};

template <int N>
__device__ __forceinline__ unsigned long long seg_max64(unsigned long long k) {
#pragma unroll
    for (int off = N / 2; off >= 1; off >>= 1) {
        const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(k >> 32), off);
        const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)k, off);
        k = u64max(k, ((unsigned long long)hi << 32) | lo);
    }
    return k;
}

template <int N, int WARPS, typename IO>
__global__ void __launch_bounds__(WARPS * 32) warpsegd_kernel(Pair64Args<IO> a) {
    using C = SegdCfg<N>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpSegdSmem<N, WARPS> &sm = *reinterpret_cast<WarpSegdSmem<N, WARPS> *>(smem_raw);
    if (threadIdx.x < N) {
        double sn, cn;
        sincospi(2.0 * threadIdx.x / N, &sn, &cn);
        sm.cs[threadIdx.x] = make_double2(cn, sn);
    }
    __syncthreads();
    const bool TREE = a.tree != 0;
    const int lane = lane_id(), wid = warp_id();
    const int sg = lane / N, v = lane % N, sbase = sg * N;
    double2 *t = sm.seg[wid][sg];
    uint32_t rk[N];  // 1023 - rank(u N + v)
    double wfr[N];
#pragma unroll
    for (int u = 0; u < N; ++u) {
        rk[u] = (uint32_t)(1023 - tie_rank(u * N + v, TREE));
        wfr[u] = a.wf[u * N + v];
    }
    const int64_t nblocks = a.list_count ? (int64_t)*a.list_count : a.nblocks;
    const int64_t stride = (int64_t)gridDim.x * WARPS * C::BPW;
    for (int64_t base = ((int64_t)blockIdx.x * WARPS + wid) * C::BPW; base < nblocks; base += stride) {
        const int64_t bi = base + sg;
        const bool real = bi < nblocks;
        const int64_t bix = real ? bi : nblocks - 1;
        const int64_t bid = a.list ? (int64_t)a.list[bix] : a.first + bix;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        constexpr int TS = N + 1;
        const int64_t wr0 = r0 - a.L, x = c0 - a.L + v;
        const bool xin = x >= 0 && x < a.W;
        double energy = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const int64_t y = wr0 + k;
            double f = 0.0, w = 0.0;
            if (xin && y >= 0 && y < a.H && a.mask[y * a.mask_pitch + x]) {
                f = load_px(a.px + y * a.px_pitch + x);
                w = a.decay[k * N + v];
            }
            t[k * TS + v] = make_double2(f * w, w);
            energy = fma(f * f, w, energy);
        }
        __syncwarp();
        cpx<double> R[N];
#pragma unroll
        for (int j = 0; j < N; ++j) { const double2 z = t[v * TS + j]; R[j] = {z.x, z.y}; }
        fft_line<N>(R);
#pragma unroll
        for (int j = 0; j < N; ++j) t[v * TS + j] = make_double2(R[j].re, R[j].im);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < N; ++j) { const double2 z = t[j * TS + v]; R[j] = {z.x, z.y}; }
        fft_line<N>(R);
#pragma unroll
        for (int j = 0; j < N; ++j) t[j * TS + v] = make_double2(R[j].re, R[j].im);
        __syncwarp();
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
#pragma unroll
        for (int u = 0; u < N; ++u) {
            t[u * N + v] = Wc[u];
            t[(u + N) * N + v] = Wc[u];
        }
        __syncwarp();
        const double w00 = t[0].x;
        const bool empty = !(w00 > 0.0);
        int32_t *sel_b = (a.sel && real) ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (empty && real && v == 0) {
            unsigned slot = atomicAdd(a.empty_count, 1u);
            if (a.empty_list) a.empty_list[slot] = (int32_t)bid;
            if (a.done) a.done[bid] = 0;
        }
        double thr = 0.0;
        if (a.early_stop) {
#pragma unroll
            for (int off = N / 2; off >= 1; off >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, off);
            thr = 1e-12 * energy;
        }
        const double ginv = empty ? 0.0 : a.gamma / w00;
        double acc[C::NPIX];
        int pmq[C::NPIX], pnq[C::NPIX];
#pragma unroll
        for (int q = 0; q < C::NPIX; ++q) {
            acc[q] = 0.0;
            const int p = v + q * N;
            pmq[q] = a.L + p / a.B;
            pnq[q] = a.L + p % a.B;
        }
        bool live = real && !empty;
        double gr = 0.0, gi = 0.0;
        int pu = 0, pv = 0, done = 0;
        for (int it = 0; it < a.iterations; ++it) {
            if (a.early_stop && !__any_sync(0xffffffffu, live)) break;
            int col = v - pv;
            col += col < 0 ? N : 0;
            const double2 *wp = t + (N - pu) * N + col;  // row u - pu + N of W2
            unsigned long long best = 0ull;
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
                const uint32_t lo = ((uint32_t)__double2loint(o) & ~1023u) | rk[u];
                const unsigned long long k =
                    ((unsigned long long)(uint32_t)__double2hiint(o) << 32) | (unsigned long long)lo;
                best = u64max(best, k);
            }
            if (!live) best = 0ull;
            const unsigned long long key = seg_max64<N>(best);
            const int tb = rank_to_bin(1023 - (int)((uint32_t)key & 1023u), TREE);
            const int bu = tb / N, bv = tb - (tb / N) * N;
            bool go = live;
            if (live && thr > 0.0 && __longlong_as_double((long long)key) < thr) live = go = false;
            if (sel_b && v == 0 && go) sel_b[it] = bu * N + bv;
            double2 c = make_double2(R[0].re, R[0].im);
#pragma unroll
            for (int u = 1; u < N; ++u)
                if (u == bu) c = make_double2(R[u].re, R[u].im);
            c.x = __shfl_sync(0xffffffffu, c.x, sbase + bv);
            c.y = __shfl_sync(0xffffffffu, c.y, sbase + bv);
            gr = go ? c.x * ginv : 0.0;
            gi = go ? c.y * ginv : 0.0;
#pragma unroll
            for (int q = 0; q < C::NPIX; ++q) {
                const double2 e = sm.cs[(bu * pmq[q] + bv * pnq[q]) % N];
                acc[q] = fma(gr, e.x, fma(-gi, e.y, acc[q]));
            }
            if (go) {
                pu = bu;
                pv = bv;
                done = it + 1;
            }
        }
        if (sel_b)
            for (int it = done + v; it < a.iterations; it += N) sel_b[it] = -1;
        if (real && !empty && v == 0 && a.done) a.done[bid] = done;
        if (real && !empty) {
#pragma unroll
            for (int q = 0; q < C::NPIX; ++q) {
                const int p = v + q * N;
                if (p < a.B * a.B) {
                    const int m = p / a.B, n = p % a.B;
                    const int64_t y = r0 + m, xx = c0 + n;
                    if (y < a.H && xx < a.W)
                        a.out[y * a.out_pitch + xx] =
                            a.mask[y * a.mask_pitch + xx] ? a.px[y * a.px_pitch + xx] : (IO)acc[q];
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace fsr
