// fsr_warp16.cuh -- FSR kernel for support N = 16 (the paper's S = 16, Fig. 5),
// fp32 loop with the near-tie guard, one warp per target block.
//
// Same structure as fsr_warp32.cuh (read that header first), scaled to 256
// bins per block:
//   lanes      lane l owns spectral column v(l) and row parity p = l & 1:
//              v = bitrev4(l >> 1) for the tree reducer, l >> 1 for linear.
//              Its 8 bins are rows u = p + 2j (j = 0..7), held as 4 packed
//              row pairs (u, u + 8) for j = i and j = i + 4.  With this map
//              "lowest lane" is exactly the reference's tie order between
//              lanes and the in-lane tie rank depends on j only: the tree
//              rank of flat bin t = 16u + v is (bitrev5(t >> 5), bitrev5(t & 31))
//              = (bitrev3(u >> 1), bitrev4(v), u & 1) (_kernels.py:12-49);
//              linear is (u, v).
//   W          row-pair table U16[k][c] = (W[k+8][c], W[k][c]) (x then y),
//              16 rows x 20 float4 (4-column pad: with the row-parity lanes the
//              8 lanes of an LDS.128 phase then hit 8 bank groups).  Pair i of
//              lane (v, p) reads row 8 + p + 2i - (pu mod 8), never wrapping;
//              pu >= 8 swaps halves (second pass variant).
//   prologue   TMA window gather (16 rows; 20-column f32 and 32-column u8
//              boxes from 16-byte aligned starts), fp64 2-D FFT on a 16 x 17
//              double2 tile (16 lanes, one line each), Hermitian split.
//   guard      per-lane top-2 keys; flagged blocks are re-run in fp64 by
//              warp16d (below) in list mode.
#pragma once

#include "fsr_warp32.cuh"

namespace fsr {

constexpr int W16_US = 20;  // U16 row stride (float4)
constexpr int W16_TS = 17;  // fp64 tile row stride (double2)
constexpr int W16_BOX_PX = TmaBox<float, 16, 16>::PX, W16_BOX_MK = TmaBox<float, 16, 16>::MK;
// staging: 1792 B (f32 pixels), 2816 B (f64 pixels) -- both inside the 5 KiB per warp

template <int WARPS>
struct Warp16Smem {
    float4 ubuf[WARPS][16 * W16_US];  // 5 KiB per warp: TMA staging, fp64 tile (4.25 KiB), U16
    float2 cs[16];
    unsigned int red_key[WARPS][32];
    unsigned int red_rank[WARPS][32];
    unsigned long long bar[WARPS];
};

__host__ __device__ __forceinline__ uint32_t bitrev4(uint32_t x) {
    return ((x & 1u) << 3) | ((x & 2u) << 1) | ((x & 4u) >> 1) | ((x & 8u) >> 3);
}
__host__ __device__ __forceinline__ uint32_t bitrev3(uint32_t x) {
    return ((x & 1u) << 2) | (x & 2u) | ((x & 4u) >> 2);
}

// Physical U16 column: tree-order lanes of one 8-lane phase read columns
// {x, x+4, x+8, x+12} (two rows each); a 4x4 transpose makes them contiguous.
template <bool TREE>
__device__ __forceinline__ int ucol16(int c) {
    return TREE ? (((c & 3) << 2) | (c >> 2)) : c;
}

template <bool TREE, bool GUARD, bool HERM, bool UPDATE, bool SWAP>
__device__ __forceinline__ void pass16(float2 (&re)[4], float2 (&im)[4], const float2 (&wf2)[4],
                                       const float4 *up, float gr, float gi, uint32_t canon,
                                       uint32_t hmask, uint32_t &m1, uint32_t &m2) {
    m1 = 0;
    m2 = 0;
    const float2 ngr = make_float2(-gr, -gr), pgi = make_float2(gi, gi), ngi = make_float2(-gi, -gi);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 r = re[i], m = im[i];
        if (UPDATE) {
            const float4 w = up[i * 2 * W16_US];
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
        const uint32_t rka = TREE ? bitrev3(i) : (uint32_t)i;          // j = i
        const uint32_t rkb = TREE ? bitrev3(i + 4) : (uint32_t)(i + 4); // j = i + 4
        uint32_t ka = and_or(f2u(o.x), hmask, 31u ^ rka);
        uint32_t kb = and_or(f2u(o.y), hmask, 31u ^ rkb);
        if (HERM && GUARD) {
            ka = ((canon >> i) & 1u) ? ka : 0u;
            kb = ((canon >> (i + 4)) & 1u) ? kb : 0u;
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

template <bool TREE, bool GUARD, bool HERM>
__device__ __forceinline__ void pass16_update(float2 (&re)[4], float2 (&im)[4], const float2 (&wf2)[4],
                                              const float4 *up, bool swap, float gr, float gi,
                                              uint32_t canon, uint32_t hmask, uint32_t &m1, uint32_t &m2) {
    if (swap)
        pass16<TREE, GUARD, HERM, true, true>(re, im, wf2, up, gr, gi, canon, hmask, m1, m2);
    else
        pass16<TREE, GUARD, HERM, true, false>(re, im, wf2, up, gr, gi, canon, hmask, m1, m2);
}

// Gather + fp64 2-D FFT + split for one N = 16 window.  Lane l gathers window
// column l & 15, rows (l >> 4) * 8 .. + 7; lanes 0..15 each transform one row,
// then one column; lane (v, p) then keeps rows p + 2j of spectral column v.
template <typename IO, bool TREE>
__device__ __forceinline__ double w16_prologue(const Warp32Args &a, const Warp32Maps &maps, float4 *ub,
                                               uint32_t bar, uint32_t &phase, float2 (&re)[4],
                                               float2 (&im)[4], int64_t wr0, int64_t wc0, int lane,
                                               int v, int p) {
    using Box = TmaBox<IO, 16, 16>;
    double2 *t = reinterpret_cast<double2 *>(ub);
    const int cl = lane & 15, rh = lane >> 4;
    IO pf[8];
    uint32_t pm[8];
    if (a.use_tma) {
        const int x0 = (int)wc0;
        const int xp = x0 & ~(Box::ALIGN - 1), xm = x0 & ~15;
        const IO *spx = reinterpret_cast<const IO *>(ub);
        const uint8_t *smk = reinterpret_cast<const uint8_t *>(ub) + Box::STAGE_MK;
        tma_window(maps, bar, smem_u32(spx), smem_u32(smk), xp, xm, (int)wr0 - a.tma_y0, Box::TX_BYTES);
        mbar_wait(bar, phase);
        phase ^= 1u;
        const IO *cpx = spx + rh * 8 * Box::PX + (x0 - xp) + cl;
        const uint8_t *cmk = smk + rh * 8 * Box::MK + (x0 - xm) + cl;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            pf[k] = cpx[k * Box::PX];
            pm[k] = cmk[k * Box::MK];
        }
        __syncwarp();
    } else {
        const int64_t x = wc0 + cl;
        const bool xin = x >= 0 && x < a.W;
        const IO *px = static_cast<const IO *>(a.px);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t y = wr0 + rh * 8 + k;
            const bool in = xin && y >= 0 && y < a.H;
            pf[k] = in ? __ldg(px + y * a.px_pitch + x) : (IO)0;
            pm[k] = in ? (uint32_t)__ldg(a.mask + y * a.mask_pitch + x) : 0u;
        }
    }
    double energy = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int r = rh * 8 + k;
        double f = 0.0, w = 0.0;
        if (pm[k]) {
            f = (double)pf[k];
            w = __ldg(a.decay64 + r * 16 + cl);
        }
        t[r * W16_TS + cl] = make_double2(f * w, w);
        energy = fma(f * f, w, energy);
    }
    __syncwarp();
    if (lane < 16) {  // rows
        cpx<double> xv[16];
        double2 *tr_ = t + lane * W16_TS;
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = tr_[j]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int j = 0; j < 16; ++j) tr_[j] = make_double2(xv[j].re, xv[j].im);
    }
    __syncwarp();
    if (lane < 16) {  // columns
        cpx<double> xv[16];
        double2 *tc = t + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = tc[j * W16_TS]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int j = 0; j < 16; ++j) tc[j * W16_TS] = make_double2(xv[j].re, xv[j].im);
    }
    __syncwarp();
    // split: R = (Z + conj Z(-u,-v)) / 2, W = (Z - conj Z(-u,-v)) / 2i, rounded to fp32 once
    const int mv = (16 - v) & 15;
    float2 Wl[4], Wh[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int u = p + 2 * i + 8 * hh, nu = (16 - u) & 15;
            const double2 z = t[u * W16_TS + v], zm = t[nu * W16_TS + mv];
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
    __syncwarp();
    // U16[k][c] = (Wx[k+8], Wx[k], Wy[k+8], Wy[k]); this lane owns rows k = p + 2i and k + 8
    float4 *ul = ub + ucol16<TREE>(v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = p + 2 * i;
        ul[k * W16_US] = make_float4(Wh[i].x, Wl[i].x, Wh[i].y, Wl[i].y);
        ul[(k + 8) * W16_US] = make_float4(Wl[i].x, Wh[i].x, Wl[i].y, Wh[i].y);
    }
    __syncwarp();
    return energy;
}

#ifndef FSR_W16_WARPS_PER_SM
#define FSR_W16_WARPS_PER_SM 24  // resident warps (blocks) per SM the register budget targets (measured at 1080p: 20 -> 24 is +3 %, 28 and 32 are slower)
#endif
template <typename IO, int WARPS, bool TREE, int ARGMAX, bool GUARD, int OPTS = W32_ALL>
__global__ void __launch_bounds__(WARPS * 32, FSR_W16_WARPS_PER_SM / WARPS)
    warp16_kernel(Warp32Args a, const __grid_constant__ Warp32Maps maps) {
    constexpr bool TRACE = (OPTS & W32_TRACE) != 0, EARLY = (OPTS & W32_EARLY) != 0;
    constexpr bool KAPPA = (OPTS & W32_KAPPA) != 0;
    // lane order as in warp32: tie-rank order only where the kernel breaks exact
    // ties itself; guarded, every near-tie is re-run in fp64, so natural order
    // (no bit reversals in the argmax tail) and any maximal lane may win
    constexpr bool LT = TREE && !GUARD;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Warp16Smem<WARPS> &sm = *reinterpret_cast<Warp16Smem<WARPS> *>(smem_raw);
    constexpr bool REC = GUARD && (OPTS & W32_REPLAY) != 0;  // replay records (see warp32)
    uint16_t *seqw = REC ? reinterpret_cast<uint16_t *>(smem_raw + sizeof(Warp16Smem<WARPS>)) +
                               warp_id() * a.seq_stride
                         : nullptr;
    const int lane = lane_id(), wid = warp_id();
    if (threadIdx.x < 16) {
        const double th = 6.283185307179586476925286766559 * threadIdx.x / 16.0;
        sm.cs[threadIdx.x] = make_float2((float)cos(th), (float)sin(th));
    }
    const uint32_t bar = smem_u32(&sm.bar[wid]);
    if (lane == 0) mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t phase = 0;
    float4 *ub = sm.ubuf[wid];
    const int p = lane & 1;
    const int v = LT ? (int)bitrev4((uint32_t)(lane >> 1)) : (lane >> 1);
    // canonical half of each mirror pair: bit i (row p+2i), bit i+4 (row p+2i+8)
    uint32_t canon = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int u = p + 2 * i + 8 * hh;
            const int t = u * 16 + v, mt = ((16 - u) & 15) * 16 + ((16 - v) & 15);
            canon |= (uint32_t)(tie_rank(t, TREE) <= tie_rank(mt, TREE)) << (i + 4 * hh);
        }
    }
    float2 wf2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        wf2[i] = make_float2(__ldg(a.wf + (p + 2 * i) * 16 + v), __ldg(a.wf + (p + 2 * i + 8) * 16 + v));

    const int64_t total_warps = (int64_t)gridDim.x * WARPS;
    for (int64_t bi = (int64_t)blockIdx.x * WARPS + wid; bi < a.nblocks; bi += total_warps) {
        const int64_t bid = a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        float2 re[4], im[4];
        const float energy =
            (float)w16_prologue<IO, LT>(a, maps, ub, bar, phase, re, im, r0 - a.L, c0 - a.L, lane, v, p);
        const float w00 = ub[8 * W16_US].x;  // U16[8][0].x = Wx[0][0] = sum of the weights
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
        float fl = -1.f;  // guard test as a float max (see warp32): flagged iff fl >= 0
        float ks = 0.f;   // kappa sqrt(B0) (see warp32)
        int kf = -1;      // REC: the first flagged iteration
        // one iteration; H: Hermitian phase (run as its own loop, see warp32)
        // synthesis deferred by one iteration (see warp32)
        int sidx = 0;
        bool has_pend = false;
        auto step = [&](auto hconst) -> bool {
            constexpr bool H = decltype(hconst)::value;
            uint32_t m1, m2;
            const bool pend = !H || has_pend;
            float2 e_pend = make_float2(0.f, 0.f);
            if (pend) e_pend = sm.cs[sidx];
            const float4 *up = ub + (8 + p - (pu & 7)) * W16_US + ucol16<LT>((v - pv) & 15);
            const bool swap = pu >= 8;
            if (H && it == 0) {
                pass16<LT, GUARD, true, false, false>(re, im, wf2, up, gr, gi, canon, a.key_mask, m1, m2);
            } else {
                pass16_update<LT, GUARD, H>(re, im, wf2, up, swap, gr, gi, canon, a.key_mask, m1, m2);
            }
            uint32_t kmax;
            int wl;
            cross_lane_best<ARGMAX, GUARD>(m1, kmax, wl, sm.red_key[wid], sm.red_rank[wid]);
            if (pend) acc = fmaf(gr, e_pend.x, fmaf(-gi, e_pend.y, acc));
            has_pend = false;
            const uint32_t rank = 31u - (kmax & 31u);
            const int j = LT ? (int)bitrev3(rank) : (int)rank;
            const int bu = (wl & 1) + 2 * j;
            const int bv = LT ? (int)bitrev4((uint32_t)(wl >> 1)) : (wl >> 1);
            const float b1 = __uint_as_float(kmax & ~31u);
            if (TRACE && sel_b && lane == 0) sel_b[it] = bu * 16 + bv;
            if (REC) seqw[it] = (uint16_t)(bu * 16 + bv);  // uniform: every lane stores it (see warp32)
            if (EARLY && b1 < thr) {
                if (GUARD && b1 >= thr * a.omt) {
                    flagged = true;
                    if (REC && kf < 0) kf = it;
                }
                return false;
            }
            float4 q;
            switch (j & 3) {
                case 0: q = make_float4(re[0].x, re[0].y, im[0].x, im[0].y); break;
                case 1: q = make_float4(re[1].x, re[1].y, im[1].x, im[1].y); break;
                case 2: q = make_float4(re[2].x, re[2].y, im[2].x, im[2].y); break;
                default: q = make_float4(re[3].x, re[3].y, im[3].x, im[3].y); break;
            }
            float2 c = j < 4 ? make_float2(q.x, q.z) : make_float2(q.y, q.w);
            c.x = __shfl_sync(0xffffffffu, c.x, wl);
            c.y = __shfl_sync(0xffffffffu, c.y, wl);
            gr = c.x * ginv;
            gi = c.y * ginv;
            pu = bu;
            pv = bv;
            if (GUARD) {
                // per-lane test on the lane's own b2 candidate, warp OR after the loop
                // (no second reduction in the iteration chain; see warp32)
                const float b2 = __uint_as_float(((lane == wl) ? m2 : m1) & ~31u);
                float gtest;
                if (KAPPA) {  // scale term (see warp32)
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
            if (H) herm = ((bu & 7) == 0) && ((bv & 7) == 0);
            sidx = (bu * pm + bv * pn) & 15;
            has_pend = true;
            return true;
        };
        bool live = true;  // false after an early stop (the iteration is not counted)
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
        if (has_pend) {
            const float2 e = sm.cs[sidx];
            acc = fmaf(gr, e.x, fmaf(-gi, e.y, acc));
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

}  // namespace fsr

// ---------------------------------------------------------------------------
// warp16d: the N = 16 kernel in fp64 -- the fp64 validation path for N = 16
// and the re-run kernel for blocks the fp32 guard flags (list mode).  Same
// lane map as warp16 (so "lowest lane" is the reference's tie order between
// lanes); R as 8 complex doubles per lane; W as two row-pair tables of
// double2, Ux[k][c] = (Wx[k+8][c], Wx[k][c]) and Uy likewise (row stride 20:
// conflict-free for the row-parity lanes); keys are the fp64 objective with
// the 3 low mantissa bits replaced by 7 - (in-lane tie rank), so a u64 max is
// exact to 2^-49 and ties resolve to the reference's rule (as in pair64).
#include "fsr_pair64.cuh"

namespace fsr {

template <int WARPS>
struct Warp16dSmem {
    double2 ux[WARPS][16 * W16_US];  // 5 KiB, also the 16 x 17 double2 FFT tile
    double2 uy[WARPS][16 * W16_US];  // 5 KiB
    double2 cs[16];
    unsigned int red_hi[WARPS][32];
    unsigned int red_lo[WARPS][32];
};

template <bool TREE, typename IO>
__device__ __forceinline__ double w16d_prologue(const Pair64Args<IO> &a, double2 *ux, double2 *uy,
                                                double (&rre)[8], double (&rim)[8], int64_t wr0,
                                                int64_t wc0, int lane, int v, int p) {
    double2 *t = ux;  // 16 x 17 double2
    const int cl = lane & 15, rh = lane >> 4;
    const int64_t x = wc0 + cl;
    const bool xin = x >= 0 && x < a.W;
    IO pf[8];
    uint32_t pm[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int64_t y = wr0 + rh * 8 + k;
        const bool in = xin && y >= 0 && y < a.H;
        pf[k] = in ? a.px[y * a.px_pitch + x] : (IO)0;
        pm[k] = in ? (uint32_t)a.mask[y * a.mask_pitch + x] : 0u;
    }
    double energy = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int r = rh * 8 + k;
        double f = 0.0, w = 0.0;
        if (pm[k]) {
            f = (double)pf[k];
            w = __ldg(a.decay + r * 16 + cl);
        }
        t[r * W16_TS + cl] = make_double2(f * w, w);
        energy = fma(f * f, w, energy);
    }
    __syncwarp();
    if (lane < 16) {
        cpx<double> xv[16];
        double2 *tr_ = t + lane * W16_TS;
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = tr_[j]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int j = 0; j < 16; ++j) tr_[j] = make_double2(xv[j].re, xv[j].im);
    }
    __syncwarp();
    if (lane < 16) {
        cpx<double> xv[16];
        double2 *tc = t + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = tc[j * W16_TS]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int j = 0; j < 16; ++j) tc[j * W16_TS] = make_double2(xv[j].re, xv[j].im);
    }
    __syncwarp();
    const int mv = (16 - v) & 15;
    double2 Wj[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int u = p + 2 * j, nu = (16 - u) & 15;
        const double2 z = t[u * W16_TS + v], zm = t[nu * W16_TS + mv];
        rre[j] = (z.x + zm.x) * 0.5;
        rim[j] = (z.y - zm.y) * 0.5;
        Wj[j] = make_double2((z.y + zm.y) * 0.5, (zm.x - z.x) * 0.5);
    }
    __syncwarp();
    const int pc = ucol16<TREE>(v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = p + 2 * i;  // rows k (j = i) and k + 8 (j = i + 4)
        ux[k * W16_US + pc] = make_double2(Wj[i + 4].x, Wj[i].x);
        uy[k * W16_US + pc] = make_double2(Wj[i + 4].y, Wj[i].y);
        ux[(k + 8) * W16_US + pc] = make_double2(Wj[i].x, Wj[i + 4].x);
        uy[(k + 8) * W16_US + pc] = make_double2(Wj[i].y, Wj[i + 4].y);
    }
    __syncwarp();
    return energy;
}

template <bool TREE, bool UPDATE, bool SWAP, bool OBJ = true>
__device__ __forceinline__ unsigned long long pass16d(double (&rre)[8], double (&rim)[8],
                                                      const double (&wf)[8], const double2 *pux,
                                                      const double2 *puy, double gr, double gi) {
    unsigned long long best[2] = {0ull, 0ull};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double2 wxp = make_double2(0.0, 0.0), wyp = make_double2(0.0, 0.0);
        if (UPDATE) {
            wxp = pux[i * 2 * W16_US];
            wyp = puy[i * 2 * W16_US];
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int j = i + 4 * hh;
            double re = rre[j], im = rim[j];
            if (UPDATE) {
                const bool first = (hh == 0) != SWAP;  // lo row reads the first half unless swapped
                const double wx = first ? wxp.x : wxp.y, wy = first ? wyp.x : wyp.y;
                re = fma(-gr, wx, re);
                re = fma(gi, wy, re);
                im = fma(-gr, wy, im);
                im = fma(-gi, wx, im);
                rre[j] = re;
                rim[j] = im;
            }
            if (OBJ) {
                const double o = fma(re, re, im * im) * wf[j];
                const uint32_t rk = TREE ? bitrev3((uint32_t)j) : (uint32_t)j;
                const uint32_t lo = ((uint32_t)__double2loint(o) & ~7u) | (7u - rk);
                const unsigned long long k =
                    ((unsigned long long)(uint32_t)__double2hiint(o) << 32) | (unsigned long long)lo;
                best[hh] = u64max(best[hh], k);
            }
        }
    }
    return u64max(best[0], best[1]);
}

#ifndef FSR_W16D_WARPS_PER_SM
#define FSR_W16D_WARPS_PER_SM 20  // fp64 N=16 1080p: 246 -> 258 fps over 16
#endif
template <int WARPS, bool TREE, int ARGMAX, typename IO>
__global__ void __launch_bounds__(WARPS * 32, FSR_W16D_WARPS_PER_SM / WARPS) warp16d_kernel(Pair64Args<IO> a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Warp16dSmem<WARPS> &sm = *reinterpret_cast<Warp16dSmem<WARPS> *>(smem_raw);
    const int lane = lane_id(), wid = warp_id();
    if (threadIdx.x < 16) {
        const double th = 6.283185307179586476925286766559 * threadIdx.x / 16.0;
        sm.cs[threadIdx.x] = make_double2(cos(th), sin(th));
    }
    __syncthreads();
    double2 *ux = sm.ux[wid], *uy = sm.uy[wid];
    const int p = lane & 1;
    const int v = TREE ? (int)bitrev4((uint32_t)(lane >> 1)) : (lane >> 1);
    double wf[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) wf[j] = __ldg(a.wf + (p + 2 * j) * 16 + v);

    const int64_t nblocks = a.list_count ? (int64_t)*a.list_count : a.nblocks;
    const int64_t total_warps = (int64_t)gridDim.x * WARPS;
    for (int64_t bi = (int64_t)blockIdx.x * WARPS + wid; bi < nblocks; bi += total_warps) {
        const int64_t bid = a.list ? (int64_t)a.list[bi] : a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        double rre[8], rim[8];
        const double energy = w16d_prologue<TREE, IO>(a, ux, uy, rre, rim, r0 - a.L, c0 - a.L, lane, v, p);
        const double w00 = ux[8 * W16_US].x;  // Ux[8][0].x = Wx[0][0]
        int32_t *sel_b = a.sel ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (!(w00 > 0.0)) {
            if (lane == 0) {
                if (a.empty_list) {
                    unsigned slot = atomicAdd(a.empty_count, 1u);
                    a.empty_list[slot] = (int32_t)bid;
                }
                if (a.done) a.done[bid] = 0;
            }
            if (sel_b)
                for (int it = lane; it < a.iterations; it += 32) sel_b[it] = -1;
            __syncwarp();
            continue;
        }
        double thr = 0.0;
        if (a.early_stop) {
            double e = energy;
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
            thr = 1e-12 * e;
        }
        const double ginv = a.gamma / w00;
        const int pm = a.L + lane / a.B, pn = a.L + lane % a.B;
        double acc = 0.0, gr = 0.0, gi = 0.0;
        int pu = 0, pv = 0, it = 0;
        // replay (list mode): iterations < kf follow the fp32 kernel's recorded
        // selections with the update alone (see fsr_pair64.cuh)
        const int kf = a.list_kf ? a.list_kf[bi] : 0;
        const uint16_t *seq = a.list_kf ? a.list_seq + bi * (int64_t)a.seq_stride : nullptr;
        for (; it < kf; ++it) {
            const int roff = (8 + p - (pu & 7)) * W16_US + ucol16<TREE>((v - pv) & 15);
            if (it > 0) {
                if (pu >= 8)
                    pass16d<TREE, true, true, false>(rre, rim, wf, ux + roff, uy + roff, gr, gi);
                else
                    pass16d<TREE, true, false, false>(rre, rim, wf, ux + roff, uy + roff, gr, gi);
            }
            const uint32_t s = seq[it];
            const int bu = (int)(s >> 4), bv = (int)(s & 15u);
            const int j = bu >> 1;
            const int wl = ((TREE ? (int)bitrev4((uint32_t)bv) : bv) << 1) | (bu & 1);
            if (sel_b && lane == 0) sel_b[it] = bu * 16 + bv;
            double cre, cim;
            switch (j) {
#define FSR_P16R(q) \
    case q: cre = rre[q]; cim = rim[q]; break;
                FSR_P16R(0) FSR_P16R(1) FSR_P16R(2) FSR_P16R(3) FSR_P16R(4) FSR_P16R(5) FSR_P16R(6)
                default: cre = rre[7]; cim = rim[7]; break;
#undef FSR_P16R
            }
            cre = __shfl_sync(0xffffffffu, cre, wl);
            cim = __shfl_sync(0xffffffffu, cim, wl);
            gr = cre * ginv;
            gi = cim * ginv;
            pu = bu;
            pv = bv;
            const double2 e = sm.cs[(bu * pm + bv * pn) & 15];
            acc = fma(gr, e.x, fma(-gi, e.y, acc));
        }
        for (; it < a.iterations; ++it) {
            const int roff = (8 + p - (pu & 7)) * W16_US + ucol16<TREE>((v - pv) & 15);
            unsigned long long kb;
            if (it == 0)
                kb = pass16d<TREE, false, false>(rre, rim, wf, ux + roff, uy + roff, gr, gi);
            else if (pu >= 8)
                kb = pass16d<TREE, true, true>(rre, rim, wf, ux + roff, uy + roff, gr, gi);
            else
                kb = pass16d<TREE, true, false>(rre, rim, wf, ux + roff, uy + roff, gr, gi);
            const unsigned long long key = p64_warp_max<ARGMAX>(kb, sm.red_hi[wid], sm.red_lo[wid]);
            const int wl = __ffs(__ballot_sync(0xffffffffu, kb == key)) - 1;
            const uint32_t rank = 7u - ((uint32_t)key & 7u);
            const int j = TREE ? (int)bitrev3(rank) : (int)rank;
            const int bu = (wl & 1) + 2 * j;
            const int bv = TREE ? (int)bitrev4((uint32_t)(wl >> 1)) : (wl >> 1);
            if (sel_b && lane == 0) sel_b[it] = bu * 16 + bv;
            if (thr > 0.0 && __longlong_as_double((long long)key) < thr) break;
            double cre, cim;
            switch (j) {
#define FSR_P16D(q) \
    case q: cre = rre[q]; cim = rim[q]; break;
                FSR_P16D(0) FSR_P16D(1) FSR_P16D(2) FSR_P16D(3) FSR_P16D(4) FSR_P16D(5) FSR_P16D(6)
                default: cre = rre[7]; cim = rim[7]; break;
#undef FSR_P16D
            }
            cre = __shfl_sync(0xffffffffu, cre, wl);
            cim = __shfl_sync(0xffffffffu, cim, wl);
            gr = cre * ginv;
            gi = cim * ginv;
            pu = bu;
            pv = bv;
            const double2 e = sm.cs[(bu * pm + bv * pn) & 15];
            acc = fma(gr, e.x, fma(-gi, e.y, acc));
        }
        const int done = it;
        if (sel_b)
            for (int jj = done + lane; jj < a.iterations; jj += 32) sel_b[jj] = -1;
        if (lane == 0 && a.done) a.done[bid] = done;
        if (lane < a.B * a.B) {
            const int m = lane / a.B, n = lane % a.B;
            const int64_t y = r0 + m, xx = c0 + n;
            if (y < a.H && xx < a.W)
                a.out[y * a.out_pitch + xx] = a.mask[y * a.mask_pitch + xx] ? a.px[y * a.px_pitch + xx] : (IO)acc;
        }
        __syncwarp();
    }
}

}  // namespace fsr
