// fsr_cta64.cuh -- FSR kernel for support N = 64 (BASELINE configs[4]; beyond the
// reference's S^2 <= 1024 cap, so the linear reducer only: core.py:76-80,
// SURVEY §8c), fp32 loop with the near-tie guard, one 4-warp CTA per block.
//
// Per block (4096 bins):
//   threads    tid = h * 64 + v owns spectral column v and the 16 row pairs
//              (u, u + 32), u = 16h + i (i = 0..15): 32 bins, 64 registers, as
//              in fsr_warp32.cuh.  Threads with equal row u share h, so among
//              equal keys the lowest tid is the lowest column: the linear
//              reducer's tie order (_kernels.py:52-59) is "max key, then
//              lowest tid", and keys carry 63 - u in their 6 low bits.
//   W          row-pair table U64[k][c] = (W[k+32][c], W[k][c]) (x then y),
//              64 x 64 float4 = 64 KiB; pair i of thread (v, h) reads row
//              32 + 16h + i - (pu mod 32) (never wraps), halves swapped when
//              pu >= 32; lanes read consecutive columns (conflict-free).
//   argmax     per warp: redux + ballot (the warp's best key, its winning
//              lane's coefficient and its runner-up for the guard) into a
//              double-buffered slot; one __syncthreads; every thread then
//              reduces the 4 slots -- the paper's two-phase (in-warp, then
//              cross-warp) argmax with the coefficient carried along.
//   prologue   2-D TMA gather (68-column f32 and 80-column u8 boxes from
//              16-byte aligned starts), fp64 2-D FFT on a 64 x 65 double2
//              tile: each 64-point line as four 16-point register FFTs
//              (samples 4m + r) and a radix-4 combine with twiddles from a
//              shared table, frequency f landing at position
//              4 (f mod 16) + f div 16; Hermitian split, R and W rounded to
//              fp32 once.
//   re-runs    flagged blocks: the exact generic fp64 kernel in list mode.
#pragma once

#include "fsr_warp32.cuh"
#include "fsr_pair64.cuh"  // Pair64Args (the fp64 kernels' argument block)

namespace fsr {

constexpr int C64_THREADS = 128;
constexpr int C64_TS = 65;  // fp64 tile row stride (double2)
constexpr int C64_BOX_PX = TmaBox<float, 64, 64>::PX, C64_BOX_MK = TmaBox<float, 64, 64>::MK;
// staging 22528 B (f32 pixels) / 38912 B (f64 pixels), inside the 65 KiB region
constexpr int C64_REGION = 64 * C64_TS * 16;                      // 66560 >= 64 KiB U table

struct __align__(16) C64Slot {
    uint32_t k1, k2;  // warp best key, warp runner-up key
    float cre, cim;   // coefficient R[u*][v*] of the warp's best bin
    int32_t lane;
    int32_t pad[3];
};

struct C64Smem {
    unsigned char region[C64_REGION];  // TMA staging -> fp64 tile -> U64 table
    double2 tw[64];                    // e^{-2 pi i j / 64}
    float2 cs[64];                     // (cos, sin)(2 pi j / 64)
    C64Slot slot[2][4];
    unsigned int red_key[4][32], red_rank[4][32];
    double esum[4];
    unsigned long long bar;
    unsigned int rec_slot;  // replay records: the block's re-run slot
};

__device__ __forceinline__ int c64_pos(int f) { return ((f & 15) << 2) | (f >> 4); }
// Physical tile column of logical column c: the low two bits XOR-ed with bits
// 3-4.  Eight consecutive columns stay in eight distinct 16-byte bank groups
// (the window store, thread = column), and so do the columns c64_pos(v) of
// eight consecutive frequencies v (the split) -- both 4-way conflicts without it.
__device__ __forceinline__ int c64_col(int c) { return c ^ ((c >> 3) & 3); }

// One 64-point forward DFT line of the tile, shared by 2 threads per line
// (phase A: sub-FFTs r and r + 2; phase B: 8 combines each), all 64 lines.
// ROWS: line `ln` is tile row ln, element e at physical column c64_col(e);
// otherwise line `ln` is physical column ln, element e in row e.
template <bool ROWS>
__device__ __forceinline__ void c64_fft_lines(double2 *t, const double2 *tw, int tid) {
    const int ln = tid & 63, r0 = tid >> 6;  // r0 in {0, 1}
    double2 *line = ROWS ? t + ln * C64_TS : t + ln;
    auto el = [&](int e) -> double2 & { return ROWS ? line[c64_col(e)] : line[e * C64_TS]; };
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // phase A: 16-point FFTs of samples 4m + r, in place at 4k + r
        const int r = r0 + 2 * q;
        cpx<double> xv[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) { const double2 z = el(4 * m + r); xv[m] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int k = 0; k < 16; ++k) el(4 * k + r) = make_double2(xv[k].re, xv[k].im);
    }
    __syncthreads();
#pragma unroll 2
    for (int jj = 0; jj < 8; ++jj) {  // phase B: radix-4 combine of bin k
        const int k = r0 + 2 * jj;
        double2 a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double2 f = el(4 * k + r);
            if (r == 0) {
                a[0] = f;
            } else {
                const double2 w = tw[(r * k) & 63];
                a[r] = make_double2(f.x * w.x - f.y * w.y, f.x * w.y + f.y * w.x);
            }
        }
        const double2 s02 = make_double2(a[0].x + a[2].x, a[0].y + a[2].y);
        const double2 d02 = make_double2(a[0].x - a[2].x, a[0].y - a[2].y);
        const double2 s13 = make_double2(a[1].x + a[3].x, a[1].y + a[3].y);
        const double2 d13 = make_double2(a[1].x - a[3].x, a[1].y - a[3].y);
        // y_q = sum_r a_r (-i)^{rq}
        el(4 * k + 0) = make_double2(s02.x + s13.x, s02.y + s13.y);
        el(4 * k + 1) = make_double2(d02.x + d13.y, d02.y - d13.x);
        el(4 * k + 2) = make_double2(s02.x - s13.x, s02.y - s13.y);
        el(4 * k + 3) = make_double2(d02.x - d13.y, d02.y + d13.x);
    }
    __syncthreads();
}

template <bool GUARD, bool HERM, bool UPDATE, bool SWAP, bool PK = false>
__device__ __forceinline__ void pass64(float2 (&re)[16], float2 (&im)[16], const float2 (&wf2)[16],
                                       const float4 *up, float gr, float gi, uint32_t canon,
                                       int h, uint32_t hmask, uint32_t &m1, uint32_t &m2) {
    m1 = 0;
    m2 = 0;
    uint32_t hpend = 0;
    const float2 ngr = make_float2(-gr, -gr), pgi = make_float2(gi, gi), ngi = make_float2(-gi, -gi);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float2 r = re[i], m = im[i];
        if (UPDATE) {
            const float4 w = up[i * 64];
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
        const uint32_t u = (uint32_t)(16 * h + i);  // h is uniform per warp
        if (PK) {
            // pair key (as warp32): the pair's larger objective tagged with its
            // lower row; top-2 over pair keys, the half resolved after the argmax
            float ox = o.x, oy = o.y;
            if (HERM) {
                ox = ((canon >> i) & 1u) ? ox : 0.f;
                oy = ((canon >> (i + 16)) & 1u) ? oy : 0.f;
            }
            const uint32_t hk = and_or(f2u(fmaxf(ox, oy)), hmask, 63u - u);
            if ((i & 1) == 0) {
                hpend = hk;
            } else {
                const uint32_t hmax = max(hpend, hk), hmin = min(hpend, hk);
                m2 = umax3(m2, hmin, min(m1, hmax));
                m1 = max(m1, hmax);
            }
            continue;
        }
        uint32_t ka = and_or(f2u(o.x), hmask, 63u - u);
        uint32_t kb = and_or(f2u(o.y), hmask, 31u - u);  // row u + 32: 63 - (u + 32)
        if (HERM && GUARD) {
            ka = ((canon >> i) & 1u) ? ka : 0u;
            kb = ((canon >> (i + 16)) & 1u) ? kb : 0u;
        }
        if (GUARD) {
            const uint32_t hi = max(ka, kb), lo = min(ka, kb);
            m2 = umax3(m2, lo, min(m1, hi));
            m1 = max(m1, hi);
        } else {
            m1 = umax3(m1, ka, kb);
        }
    }
}

#ifndef FSR_C64_PAIRKEY
#define FSR_C64_PAIRKEY 1
#endif
template <typename IO, int ARGMAX, bool GUARD, int OPTS = 0>
__global__ void __launch_bounds__(C64_THREADS, 3)
    cta64_kernel(Warp32Args a, const __grid_constant__ Warp32Maps maps) {
    // pair keys in guarded mode (every near-tie is re-run in fp64, see warp32)
    constexpr bool PK = GUARD && FSR_C64_PAIRKEY;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    C64Smem &sm = *reinterpret_cast<C64Smem *>(smem_raw);
    // replay records (see warp32): the block's selections after the struct
    constexpr bool REC = GUARD && (OPTS & W32_REPLAY) != 0;
    uint16_t *seqw = REC ? reinterpret_cast<uint16_t *>(smem_raw + sizeof(C64Smem)) : nullptr;
    const int tid = threadIdx.x, lane = lane_id(), wid = warp_id();
    const int h = tid >> 6, v = tid & 63;
    if (tid < 64) {
        const double th = 6.283185307179586476925286766559 * tid / 64.0;
        sm.tw[tid] = make_double2(cos(th), -sin(th));
        sm.cs[tid] = make_float2((float)cos(th), (float)sin(th));
    }
    const uint32_t bar = smem_u32(&sm.bar);
    if (tid == 0) mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t phase = 0;
    double2 *t = reinterpret_cast<double2 *>(sm.region);
    float4 *ub = reinterpret_cast<float4 *>(sm.region);
    // canonical half of each mirror pair (linear rank = flat index): bit i row 16h+i, bit i+16 row +32
    uint32_t canon = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int u = 16 * h + i + 32 * hh;
            const int tt = u * 64 + v, mt = ((64 - u) & 63) * 64 + ((64 - v) & 63);
            canon |= (uint32_t)(tt <= mt) << (i + 16 * hh);
        }
    }
    const float one_minus_tau = 1.f - a.tau;

    for (int64_t bi = blockIdx.x; bi < a.nblocks; bi += gridDim.x) {
        const int64_t bid = a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const int64_t wr0 = r0 - a.L, wc0 = c0 - a.L;
        // ---- gather: thread owns window column v, rows 32h .. 32h + 31
        using Box = TmaBox<IO, 64, 64>;
        IO pf[32];
        uint32_t mbits = 0;
        if (a.use_tma) {
            const int x0 = (int)wc0, xp = x0 & ~(Box::ALIGN - 1), xm = x0 & ~15;
            const IO *spx = reinterpret_cast<const IO *>(sm.region);
            const uint8_t *smk = sm.region + Box::STAGE_MK;
            if (wid == 0)
                tma_window(maps, bar, smem_u32(spx), smem_u32(smk), xp, xm, (int)wr0 - a.tma_y0, Box::TX_BYTES);
            mbar_wait(bar, phase);
            phase ^= 1u;
            const IO *cpx = spx + 32 * h * Box::PX + (x0 - xp) + v;
            const uint8_t *cmk = smk + 32 * h * Box::MK + (x0 - xm) + v;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                pf[k] = cpx[k * Box::PX];
                mbits |= (uint32_t)(cmk[k * Box::MK] != 0) << k;
            }
        } else {
            const int64_t x = wc0 + v;
            const bool xin = x >= 0 && x < a.W;
            const IO *px = static_cast<const IO *>(a.px);
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int64_t y = wr0 + 32 * h + k;
                const bool in = xin && y >= 0 && y < a.H;
                pf[k] = in ? __ldg(px + y * a.px_pitch + x) : (IO)0;
                mbits |= (uint32_t)(in && __ldg(a.mask + y * a.mask_pitch + x) != 0) << k;
            }
        }
        __syncthreads();  // staging fully read before the tile overwrites it
        double energy = 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const int r = 32 * h + k;
            double f = 0.0, w = 0.0;
            if ((mbits >> k) & 1u) {
                f = (double)pf[k];
                w = __ldg(a.decay64 + r * 64 + v);
            }
            t[r * C64_TS + c64_col(v)] = make_double2(f * w, w);
            energy = fma(f * f, w, energy);
        }
        __syncthreads();
        c64_fft_lines<true>(t, sm.tw, tid);   // rows
        c64_fft_lines<false>(t, sm.tw, tid);  // columns
        // ---- split (thread (v, h): rows 16h + i and + 32 of column v)
        float2 re[16], im[16], Wl[16], Wh[16];
        {
            const int pv = c64_col(c64_pos(v)), pmv = c64_col(c64_pos((64 - v) & 63));
#pragma unroll
            for (int i = 0; i < 16; ++i) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int u = 16 * h + i + 32 * hh, nu = (64 - u) & 63;
                    const double2 z = t[c64_pos(u) * C64_TS + pv], zm = t[c64_pos(nu) * C64_TS + pmv];
                    const float rr = (float)((z.x + zm.x) * 0.5), ri = (float)((z.y - zm.y) * 0.5);
                    const float2 w = make_float2((float)((z.y + zm.y) * 0.5), (float)((zm.x - z.x) * 0.5));
                    if (hh == 0) {
                        re[i].x = rr;
                        im[i].x = ri;
                        Wl[i] = w;
                    } else {
                        re[i].y = rr;
                        im[i].y = ri;
                        Wh[i] = w;
                    }
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int u = 16 * h + i;
            ub[u * 64 + v] = make_float4(Wh[i].x, Wl[i].x, Wh[i].y, Wl[i].y);
            ub[(u + 32) * 64 + v] = make_float4(Wl[i].x, Wh[i].x, Wl[i].y, Wh[i].y);
        }
        // early-stop energy: CTA sum
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, off);
        if (lane == 0) sm.esum[wid] = energy;
        __syncthreads();
        const float w00 = ub[32 * 64].x;  // U64[32][0].x = Wx[0][0]
        int32_t *sel_b = a.sel ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (!(w00 > 0.f)) {
            if (tid == 0) {
                unsigned slot = atomicAdd(a.empty_count, 1u);
                a.empty_list[slot] = (int32_t)bid;
                if (a.done) a.done[bid] = 0;
            }
            if (sel_b)
                for (int it = tid; it < a.iterations; it += C64_THREADS) sel_b[it] = -1;
            __syncthreads();
            continue;
        }
        const float thr = a.early_stop ? 1e-12f * (float)(sm.esum[0] + sm.esum[1] + sm.esum[2] + sm.esum[3])
                                       : 0.f;
        float2 wf2[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            wf2[i] = make_float2(__ldg(a.wf + (16 * h + i) * 64 + v), __ldg(a.wf + (16 * h + i + 32) * 64 + v));
        const float ginv = a.gamma / w00;
        const int pm_ = a.L + tid / a.B, pn_ = a.L + tid % a.B;
        float acc = 0.f, gr = 0.f, gi = 0.f;
        bool herm = true, flagged = false;
        float ks = 0.f;  // kappa sqrt(B0) (see warp32)
        int kf = -1;     // REC: the first flagged iteration
        int pu = 0, pv = 0, it = 0;
        // one iteration; H: Hermitian phase, run as its own loop (see warp32)
        auto step = [&](auto hconst) -> bool {
            constexpr bool H = decltype(hconst)::value;
            uint32_t m1, m2;
            const float4 *up = ub + (32 + 16 * h - (pu & 31)) * 64 + ((v - pv) & 63);
            const bool swap = pu >= 32;
            if (H && it == 0)
                pass64<GUARD, true, false, false, PK>(re, im, wf2, up, gr, gi, canon, h, a.key_mask, m1, m2);
            else
                swap ? pass64<GUARD, H, true, true, PK>(re, im, wf2, up, gr, gi, canon, h, a.key_mask, m1, m2)
                     : pass64<GUARD, H, true, false, PK>(re, im, wf2, up, gr, gi, canon, h, a.key_mask, m1, m2);
            // phase 1: in-warp argmax, coefficient of the warp's best bin
            // (ARGMAX: the paper's __shfl_xor_sync butterfly, redux.sync + ballot,
            // or the shared-memory tree -- the same cross-lane step as warp32)
            uint32_t kw;
            int wl;
            cross_lane_best<ARGMAX, PK>(m1, kw, wl, sm.red_key[wid], sm.red_rank[wid]);
            uint32_t k1w = kw, cand2 = 0u;  // cand2: this thread's b2 candidate if its warp wins
            float cre, cim;
            if (PK) {
                // the warp's winning pair (row 16h + i and + 32): both halves'
                // objectives recomputed exactly as the pass did, the winner's half,
                // coefficient and pair partner read from lane wl
                const int ur0 = 63 - (int)(kw & 63u);
                float2 wfp;
                const float4 q = pick_pair(re, im, wf2, ur0, wfp);
                float olo = fmaf(q.x, q.x, q.z * q.z) * wfp.x, ohi = fmaf(q.y, q.y, q.w * q.w) * wfp.y;
                if (H) {
                    olo = ((canon >> (ur0 & 15)) & 1u) ? olo : 0.f;
                    ohi = ((canon >> ((ur0 & 15) + 16)) & 1u) ? ohi : 0.f;
                }
                const bool hl = ohi > olo;
                const float po = hl ? olo : ohi;
                cre = hl ? q.y : q.x;
                cim = hl ? q.w : q.z;
                const bool hi = __shfl_sync(0xffffffffu, (int)hl, wl) != 0;
                cre = __shfl_sync(0xffffffffu, cre, wl);
                cim = __shfl_sync(0xffffffffu, cim, wl);
                const int ur = ur0 + (hi ? 32 : 0);
                k1w = (kw & a.key_mask) | (uint32_t)(63 - ur);  // the bin's row for phase 2
                cand2 = lane == wl ? max(m2, f2u(po) & a.key_mask) : m1;
            } else {
                cand2 = GUARD ? (lane == wl ? m2 : m1) : 0u;
                const int ur = 63 - (int)(kw & 63u);
                float4 q;
                switch ((ur & 31) & 15) {
#define FSR_PK64(j) \
    case j: q = make_float4(re[j].x, re[j].y, im[j].x, im[j].y); break;
                    FSR_PK64(0) FSR_PK64(1) FSR_PK64(2) FSR_PK64(3) FSR_PK64(4) FSR_PK64(5) FSR_PK64(6)
                    FSR_PK64(7) FSR_PK64(8) FSR_PK64(9) FSR_PK64(10) FSR_PK64(11) FSR_PK64(12) FSR_PK64(13)
                    FSR_PK64(14)
                    default: q = make_float4(re[15].x, re[15].y, im[15].x, im[15].y); break;
#undef FSR_PK64
                }
                cre = ur < 32 ? q.x : q.y;
                cim = ur < 32 ? q.z : q.w;
                cre = __shfl_sync(0xffffffffu, cre, wl);
                cim = __shfl_sync(0xffffffffu, cim, wl);
            }
            C64Slot *sl = sm.slot[it & 1];
            if (lane == 0) {
                sl[wid].k1 = k1w;
                sl[wid].k2 = 0u;  // the guard tests per thread (below)
                sl[wid].cre = cre;
                sl[wid].cim = cim;
                sl[wid].lane = wl;
            }
            __syncthreads();
            // phase 2: across the 4 warps (max key, then lowest warp = lowest tid)
            uint32_t best = sl[0].k1, second = sl[0].k2;
            int bw = 0;
#pragma unroll
            for (int w = 1; w < 4; ++w) {
                const uint32_t k = sl[w].k1;
                if (k > best) {
                    second = max(best, max(second, sl[w].k2));
                    best = k;
                    bw = w;
                } else {
                    second = max(second, k);
                }
            }
            const int bu = 63 - (int)(best & 63u);
            const int bv = (bw * 32 + sl[bw].lane) & 63;
            const float b1 = __uint_as_float(best & ~63u);
            if (sel_b && tid == 0) sel_b[it] = bu * 64 + bv;
            if (REC) seqw[it] = (uint16_t)(bu * 64 + bv);  // CTA-uniform: every thread stores it (see warp32)
            if (b1 < thr) {
                if (GUARD && b1 >= thr * one_minus_tau) {
                    flagged = true;
                    if (REC && kf < 0) kf = it;
                }
                return false;
            }
            gr = sl[bw].cre * ginv;
            gi = sl[bw].cim * ginv;
            pu = bu;
            pv = bv;
            if (GUARD) {
                // b2 is the CTA maximum of the threads' candidates (the winning
                // thread's runner-up, everyone else's best); the test is made per
                // thread on its own candidate -- the largest per-thread result is the
                // test of b2, rounding being monotonic -- and OR-ed over the CTA after
                // the loop, so no reduction of b2 sits before the slot barrier
                (void)second;
                const uint32_t c2 = (wid == bw && lane == wl) ? cand2 : m1;
                const float b2 = __uint_as_float(c2 & ~63u);
                const float sb1 = sqrt_approx(b1);  // scale term (see warp32)
                if (H && it == 0) ks = a.kappa * sb1;
                const bool g = b2 >= fmaf(-ks, sb1, b1 * one_minus_tau) || b1 * one_minus_tau < thr;
                flagged |= g;
                if (REC && g && kf < 0) kf = it;
            }
            if (H) herm = ((bu & 31) == 0) && ((bv & 31) == 0);
            const float2 e = sm.cs[(bu * pm_ + bv * pn_) & 63];
            acc = fmaf(gr, e.x, fmaf(-gi, e.y, acc));
            return true;
        };
        bool live = true;  // false after an early stop (the iteration is not counted)
        while (live && herm && it < a.iterations) {
            if (step(std::true_type{})) ++it; else live = false;
        }
        while (live && it < a.iterations) {
            if (step(std::false_type{})) ++it; else live = false;
            // replay build: a flagged block's remaining fp32 iterations are wasted
            // work (its fp64 re-run replays only the prefix), see warp32.  Past 100
            // iterations only (W32_EXIT build): the check is a CTA barrier, which at
            // I = 100 (11 % flagged blocks) costs more than it saves (1080p 30.6 ->
            // 32.1 ms; 33.0 with a run-time I test)
            if (REC && (OPTS & W32_EXIT) && (it & 3) == 0 && __syncthreads_or(flagged)) break;
        }
        if (GUARD) flagged = __syncthreads_or(flagged) != 0;  // the per-thread guard tests
        if (REC && flagged) {  // the first flagged iteration over the CTA
            const uint32_t k = __reduce_min_sync(0xffffffffu, kf < 0 ? 0xffffffffu : (uint32_t)kf);
            if (lane == 0) sm.red_key[wid][0] = k;
            __syncthreads();
            const uint32_t km = min(min(sm.red_key[0][0], sm.red_key[1][0]), min(sm.red_key[2][0], sm.red_key[3][0]));
            kf = km == 0xffffffffu ? -1 : (int)km;
        }
        const int done = it;
        if (sel_b)
            for (int jj = done + tid; jj < a.iterations; jj += C64_THREADS) sel_b[jj] = -1;
        if (tid == 0 && a.done) a.done[bid] = done;
        if (GUARD && flagged && a.rerun_list) {
            if (tid == 0) {
                const unsigned slot = atomicAdd(a.rerun_count, 1u);
                a.rerun_list[slot] = (int32_t)bid;
                if (REC) sm.rec_slot = slot;
            }
            if (REC) {
                __syncthreads();  // the slot and the records
                const unsigned slot = sm.rec_slot;
                const int n = kf < 0 ? 0 : min(kf, a.seq_stride);
                if (tid == 0) a.rerun_kf[slot] = n;
                uint16_t *dst = a.rerun_seq + (int64_t)slot * a.seq_stride;
                for (int jj = tid; jj < n; jj += C64_THREADS) dst[jj] = seqw[jj];
            }
        }
        if (tid < a.B * a.B) {
            const int m = tid / a.B, n = tid % a.B;
            const int64_t y = r0 + m, xx = c0 + n;
            if (y < a.H && xx < a.W)
                static_cast<IO *>(a.out)[y * a.out_pitch + xx] =
                    a.mask[y * a.mask_pitch + xx] ? static_cast<const IO *>(a.px)[y * a.px_pitch + xx] : (IO)acc;
        }
        __syncthreads();  // the region is rewritten by the next block's gather
    }
}

// ---------------------------------------------------------------------------
// cta64d: the N = 64 loop in fp64 -- the fp64 (validation) precision for N = 64
// and the re-run of the guarded fp32 kernel's flagged blocks (list mode), in
// place of the CTA-per-block generic kernel.  Same thread map as cta64 (thread
// (v, h) owns column v, rows 16h + i and 16h + i + 32), R register-resident in
// fp64 (128 registers), the weight spectrum W as a plain 64 x 64 complex
// double table (64 KiB) NEXT TO the FFT tile, so the split writes W while the
// tile is still being read: W goes to a per-CTA global staging buffer (L2)
// and is copied into the tile's space once the tile is consumed, so a CTA
// needs 81 KiB of shared memory (W with rows 0..14 repeated after row 63)
// and two CTAs share an SM.
// Keys: the fp64 objective wf * fma(re, re, im*im) with its 6 low mantissa bits
// replaced by 63 - u (comparisons exact to 2^-46 relative, as pair64's 2^-47),
// warp max by a redux on the high word (the low word only breaks exact ties
// there), then the 4 warps through a double-buffered slot: max key, then the
// lowest warp = lowest column -- the linear reducer's order (_kernels.py:52-59).
// ---------------------------------------------------------------------------
struct __align__(16) C64dSlot {
    unsigned long long key;
    double cre, cim;  // R[u*][v*] of the warp's best bin
    int32_t lane;
    int32_t pad[3];
};

// W rows in shared memory: 64 plus copies of rows 0..14, so a thread's run of
// 16 rows (u - pu) & 63, u = 16h + i (+ 32), starts at one base row and never
// wraps: compile-time row offsets instead of a masked shift per row
constexpr int C64D_WROWS = 79;
constexpr int C64D_TILE = 64 * C64_TS > C64D_WROWS * 64 ? 64 * C64_TS : C64D_WROWS * 64;
struct C64dSmem {
    double2 tile[C64D_TILE];  // fp64 FFT tile (66 560 B), then W[u][v] (79 rows, 80 896 B)
    double2 tw[64];             // e^{-2 pi i j / 64}
    double2 cs[64];             // (cos, sin)(2 pi j / 64)
    C64dSlot slot[2][4];
    double esum[4];
};

__device__ __forceinline__ unsigned long long c64d_key(double o, int u) {
    return ((unsigned long long)__double_as_longlong(o) & ~63ull) | (unsigned long long)(63 - u);
}

template <bool UPDATE, bool OBJ = true>
__device__ __forceinline__ unsigned long long c64d_pass(double2 (&rl)[16], double2 (&rh)[16],
                                                        const double (&wl)[16], const double (&wh)[16],
                                                        const double2 *Wt, int h, int v, int pu, int pv,
                                                        double gr, double gi) {
    unsigned long long mk[2] = {0ull, 0ull};
    const int col = (v - pv) & 63;
    const double2 *wlo = Wt + ((16 * h - pu) & 63) * 64 + col;       // row (u - pu) & 63, i = 0
    const double2 *whi = Wt + ((16 * h + 32 - pu) & 63) * 64 + col;  // row (u + 32 - pu) & 63
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int u = 16 * h + i;
        double2 a = rl[i], b = rh[i];
        if (UPDATE) {
            const double2 wa = wlo[i * 64];
            const double2 wb = whi[i * 64];
            a.x = fma(-gr, wa.x, a.x);
            a.x = fma(gi, wa.y, a.x);
            a.y = fma(-gr, wa.y, a.y);
            a.y = fma(-gi, wa.x, a.y);
            b.x = fma(-gr, wb.x, b.x);
            b.x = fma(gi, wb.y, b.x);
            b.y = fma(-gr, wb.y, b.y);
            b.y = fma(-gi, wb.x, b.y);
            rl[i] = a;
            rh[i] = b;
        }
        if (OBJ) {
            const unsigned long long ka = c64d_key(fma(a.x, a.x, a.y * a.y) * wl[i], u);
            const unsigned long long kb = c64d_key(fma(b.x, b.x, b.y * b.y) * wh[i], u + 32);
            mk[i & 1] = max(mk[i & 1], max(ka, kb));  // two independent max chains
        }
    }
    return max(mk[0], mk[1]);
}

// Row pair i = u mod 16 of this thread in fp64, (rl[i], rh[i]), by one indirect branch
// (brx.idx over a 16-entry jump table); i must be warp-uniform.
__device__ __forceinline__ void c64d_pick(const double2 (&rl)[16], const double2 (&rh)[16], int i,
                                          double2 &lo, double2 &hi) {
    asm volatile(
        "{\n ts%=: .branchtargets L0_%=, L1_%=, L2_%=, L3_%=, L4_%=, L5_%=, L6_%=, L7_%=, L8_%=, L9_%=, L10_%=, L11_%=, L12_%=, L13_%=, L14_%=, L15_%=;\n"
        " brx.idx %4, ts%=;\n"
        " L0_%=: mov.f64 %0, %5; mov.f64 %1, %6; mov.f64 %2, %7; mov.f64 %3, %8; bra.uni Le_%=;\n"
        " L1_%=: mov.f64 %0, %9; mov.f64 %1, %10; mov.f64 %2, %11; mov.f64 %3, %12; bra.uni Le_%=;\n"
        " L2_%=: mov.f64 %0, %13; mov.f64 %1, %14; mov.f64 %2, %15; mov.f64 %3, %16; bra.uni Le_%=;\n"
        " L3_%=: mov.f64 %0, %17; mov.f64 %1, %18; mov.f64 %2, %19; mov.f64 %3, %20; bra.uni Le_%=;\n"
        " L4_%=: mov.f64 %0, %21; mov.f64 %1, %22; mov.f64 %2, %23; mov.f64 %3, %24; bra.uni Le_%=;\n"
        " L5_%=: mov.f64 %0, %25; mov.f64 %1, %26; mov.f64 %2, %27; mov.f64 %3, %28; bra.uni Le_%=;\n"
        " L6_%=: mov.f64 %0, %29; mov.f64 %1, %30; mov.f64 %2, %31; mov.f64 %3, %32; bra.uni Le_%=;\n"
        " L7_%=: mov.f64 %0, %33; mov.f64 %1, %34; mov.f64 %2, %35; mov.f64 %3, %36; bra.uni Le_%=;\n"
        " L8_%=: mov.f64 %0, %37; mov.f64 %1, %38; mov.f64 %2, %39; mov.f64 %3, %40; bra.uni Le_%=;\n"
        " L9_%=: mov.f64 %0, %41; mov.f64 %1, %42; mov.f64 %2, %43; mov.f64 %3, %44; bra.uni Le_%=;\n"
        " L10_%=: mov.f64 %0, %45; mov.f64 %1, %46; mov.f64 %2, %47; mov.f64 %3, %48; bra.uni Le_%=;\n"
        " L11_%=: mov.f64 %0, %49; mov.f64 %1, %50; mov.f64 %2, %51; mov.f64 %3, %52; bra.uni Le_%=;\n"
        " L12_%=: mov.f64 %0, %53; mov.f64 %1, %54; mov.f64 %2, %55; mov.f64 %3, %56; bra.uni Le_%=;\n"
        " L13_%=: mov.f64 %0, %57; mov.f64 %1, %58; mov.f64 %2, %59; mov.f64 %3, %60; bra.uni Le_%=;\n"
        " L14_%=: mov.f64 %0, %61; mov.f64 %1, %62; mov.f64 %2, %63; mov.f64 %3, %64; bra.uni Le_%=;\n"
        " L15_%=: mov.f64 %0, %65; mov.f64 %1, %66; mov.f64 %2, %67; mov.f64 %3, %68; bra.uni Le_%=;\n"
        " Le_%=:\n}"
        : "=d"(lo.x), "=d"(lo.y), "=d"(hi.x), "=d"(hi.y)
        : "r"(i & 15),
          "d"(rl[0].x), "d"(rl[0].y), "d"(rh[0].x), "d"(rh[0].y),
          "d"(rl[1].x), "d"(rl[1].y), "d"(rh[1].x), "d"(rh[1].y),
          "d"(rl[2].x), "d"(rl[2].y), "d"(rh[2].x), "d"(rh[2].y),
          "d"(rl[3].x), "d"(rl[3].y), "d"(rh[3].x), "d"(rh[3].y),
          "d"(rl[4].x), "d"(rl[4].y), "d"(rh[4].x), "d"(rh[4].y),
          "d"(rl[5].x), "d"(rl[5].y), "d"(rh[5].x), "d"(rh[5].y),
          "d"(rl[6].x), "d"(rl[6].y), "d"(rh[6].x), "d"(rh[6].y),
          "d"(rl[7].x), "d"(rl[7].y), "d"(rh[7].x), "d"(rh[7].y),
          "d"(rl[8].x), "d"(rl[8].y), "d"(rh[8].x), "d"(rh[8].y),
          "d"(rl[9].x), "d"(rl[9].y), "d"(rh[9].x), "d"(rh[9].y),
          "d"(rl[10].x), "d"(rl[10].y), "d"(rh[10].x), "d"(rh[10].y),
          "d"(rl[11].x), "d"(rl[11].y), "d"(rh[11].x), "d"(rh[11].y),
          "d"(rl[12].x), "d"(rl[12].y), "d"(rh[12].x), "d"(rh[12].y),
          "d"(rl[13].x), "d"(rl[13].y), "d"(rh[13].x), "d"(rh[13].y),
          "d"(rl[14].x), "d"(rl[14].y), "d"(rh[14].x), "d"(rh[14].y),
          "d"(rl[15].x), "d"(rl[15].y), "d"(rh[15].x), "d"(rh[15].y));
}

template <typename IO>
__global__ void __launch_bounds__(C64_THREADS, 2) cta64d_kernel(Pair64Args<IO> a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    C64dSmem &sm = *reinterpret_cast<C64dSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int h = tid >> 6, v = tid & 63;
    if (tid < 64) {
        double sn, cn;
        sincospi(tid / 32.0, &sn, &cn);
        sm.tw[tid] = make_double2(cn, -sn);
        sm.cs[tid] = make_double2(cn, sn);
    }
    // frequency prior of the thread's 32 bins (weights.py:40-56)
    double wl[16], wh[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        wl[i] = __ldg(a.wf + (16 * h + i) * 64 + v);
        wh[i] = __ldg(a.wf + (16 * h + i + 32) * 64 + v);
    }
    __syncthreads();
    const int64_t nblocks = a.list_count ? (int64_t)*a.list_count : a.nblocks;
    for (int64_t bi = blockIdx.x; bi < nblocks; bi += gridDim.x) {
        const int64_t bid = a.list ? (int64_t)a.list[bi] : a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const int64_t wr0 = r0 - a.L, wc0 = c0 - a.L;
        // ---- gather + spatial weight (sampling.py:93-107, weights.py:18-37)
        double energy = 0.0;
        {
            const int64_t x = wc0 + v;
            const bool xin = x >= 0 && x < a.W;
#pragma unroll 4
            for (int k = 0; k < 32; ++k) {
                const int r = 32 * h + k;
                const int64_t y = wr0 + r;
                double f = 0.0, w = 0.0;
                if (xin && y >= 0 && y < a.H && a.mask[y * a.mask_pitch + x]) {
                    f = (double)a.px[y * a.px_pitch + x];
                    w = __ldg(a.decay + r * 64 + v);
                }
                sm.tile[r * C64_TS + c64_col(v)] = make_double2(f * w, w);
                energy = fma(f * f, w, energy);
            }
        }
        __syncthreads();
        c64_fft_lines<true>(sm.tile, sm.tw, tid);   // rows
        c64_fft_lines<false>(sm.tile, sm.tw, tid);  // columns
        // ---- Hermitian split: R to registers, W staged through global memory
        double2 *gW = a.scratch + (int64_t)blockIdx.x * 4096;
        double2 rl[16], rh[16];
        {
            const int pv_ = c64_col(c64_pos(v)), pmv = c64_col(c64_pos((64 - v) & 63));
#pragma unroll
            for (int i = 0; i < 16; ++i) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int u = 16 * h + i + 32 * hh, nu = (64 - u) & 63;
                    const double2 z = sm.tile[c64_pos(u) * C64_TS + pv_];
                    const double2 zm = sm.tile[c64_pos(nu) * C64_TS + pmv];
                    const double2 r = make_double2((z.x + zm.x) * 0.5, (z.y - zm.y) * 0.5);
                    gW[u * 64 + v] = make_double2((z.y + zm.y) * 0.5, (zm.x - z.x) * 0.5);
                    if (hh == 0) rl[i] = r; else rh[i] = r;
                }
            }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, off);
        if (lane == 0) sm.esum[wid] = energy;
        __syncthreads();  // the tile is consumed: W moves into its space
        double2 *Wt = sm.tile;
#pragma unroll 4
        for (int e = tid; e < C64D_WROWS * 64; e += C64_THREADS) Wt[e] = gW[e & 4095];
        __syncthreads();
        const double w00 = Wt[0].x;  // W[0][0] = sum of the weights
        int32_t *sel_b = a.sel ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (!(w00 > 0.0)) {  // empty support (reconstruction.py:272-275)
            if (tid == 0) {
                unsigned slot = atomicAdd(a.empty_count, 1u);
                if (a.empty_list) a.empty_list[slot] = (int32_t)bid;
                if (a.done) a.done[bid] = 0;
            }
            if (sel_b)
                for (int it = tid; it < a.iterations; it += C64_THREADS) sel_b[it] = -1;
            __syncthreads();
            continue;
        }
        const double thr =
            a.early_stop ? 1e-12 * (sm.esum[0] + sm.esum[1] + sm.esum[2] + sm.esum[3]) : 0.0;
        const double ginv = a.gamma / w00;
        const int pm_ = a.L + tid / a.B, pn_ = a.L + tid % a.B;
        double acc = 0.0, gr = 0.0, gi = 0.0;
        int pu = 0, pv = 0, it = 0;
        // replay (list mode): iterations < kf follow the fp32 kernel's recorded
        // selections with the update alone (see fsr_pair64.cuh)
        const int kf = a.list_kf ? a.list_kf[bi] : 0;
        const uint16_t *seq = a.list_kf ? a.list_seq + bi * (int64_t)a.seq_stride : nullptr;
        for (; it < kf; ++it) {
            if (it > 0) c64d_pass<true, false>(rl, rh, wl, wh, Wt, h, v, pu, pv, gr, gi);
            const uint32_t s = seq[it];
            const int bu = (int)(s >> 6), bv = (int)(s & 63u);
            C64dSlot *sl = sm.slot[it & 1];
            double2 plo, phi;
            c64d_pick(rl, rh, bu & 15, plo, phi);  // bu uniform
            if (h == ((bu & 31) >> 4) && v == bv) {
                const double2 c = bu >= 32 ? phi : plo;
                sl[0].cre = c.x;
                sl[0].cim = c.y;
            }
            __syncthreads();
            if (sel_b && tid == 0) sel_b[it] = bu * 64 + bv;
            gr = sl[0].cre * ginv;
            gi = sl[0].cim * ginv;
            pu = bu;
            pv = bv;
            const double2 e = sm.cs[(bu * pm_ + bv * pn_) & 63];
            acc = fma(gr, e.x, fma(-gi, e.y, acc));
        }
        for (; it < a.iterations; ++it) {
            const unsigned long long kb =
                it == 0 ? c64d_pass<false>(rl, rh, wl, wh, Wt, h, v, pu, pv, gr, gi)
                        : c64d_pass<true>(rl, rh, wl, wh, Wt, h, v, pu, pv, gr, gi);
            // phase 1: warp max of the u64 keys (redux on the high word)
            const uint32_t hi = (uint32_t)(kb >> 32);
            const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
            uint32_t cand = __ballot_sync(0xffffffffu, hi == mh);
            if (__popc(cand) > 1) {
                const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? (uint32_t)kb : 0u);
                cand = __ballot_sync(0xffffffffu, hi == mh && (uint32_t)kb == ml);
            }
            const int wl_ = __ffs(cand) - 1;
            C64dSlot *sl = sm.slot[it & 1];
            // the warp's winning row pair, fetched on every lane (uniform branch)
            const int uw = 63 - (int)(__shfl_sync(0xffffffffu, (uint32_t)kb, wl_) & 63u);
            double2 plo, phi;
            c64d_pick(rl, rh, uw, plo, phi);
            if (lane == wl_) {
                const double2 c = uw >= 32 ? phi : plo;
                sl[wid].key = kb;
                sl[wid].cre = c.x;
                sl[wid].cim = c.y;
                sl[wid].lane = lane;
            }
            __syncthreads();
            // phase 2: the 4 warps (max key, then the lowest warp)
            unsigned long long best = sl[0].key;
            int bw = 0;
#pragma unroll
            for (int w = 1; w < 4; ++w)
                if (sl[w].key > best) {
                    best = sl[w].key;
                    bw = w;
                }
            const int bu = 63 - (int)(best & 63ull);
            const int bv = (bw * 32 + sl[bw].lane) & 63;
            const double b1 = __longlong_as_double((long long)(best & ~63ull));
            if (sel_b && tid == 0) sel_b[it] = bu * 64 + bv;
            if (b1 < thr) break;  // thr == 0 unless early stop is on
            gr = sl[bw].cre * ginv;
            gi = sl[bw].cim * ginv;
            pu = bu;
            pv = bv;
            const double2 e = sm.cs[(bu * pm_ + bv * pn_) & 63];
            acc = fma(gr, e.x, fma(-gi, e.y, acc));
        }
        const int done = it;
        if (sel_b)
            for (int jj = done + tid; jj < a.iterations; jj += C64_THREADS) sel_b[jj] = -1;
        if (tid == 0 && a.done) a.done[bid] = done;
        if (tid < a.B * a.B) {
            const int m = tid / a.B, n = tid % a.B;
            const int64_t y = r0 + m, xx = c0 + n;
            if (y < a.H && xx < a.W)
                a.out[y * a.out_pitch + xx] =
                    a.mask[y * a.mask_pitch + xx] ? a.px[y * a.px_pitch + xx] : (IO)acc;
        }
        __syncthreads();  // tile / W / slots are rewritten by the next block
    }
}

}  // namespace fsr
