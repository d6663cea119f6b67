// fsr_warp32.cuh -- production FSR kernel for support N = 32, fp32, one warp
// per target block, everything register/shared-memory resident.
//
// Per block (reference path reconstruction.py:246-280 + _kernels.py:62-126):
//   gather     lane l loads window column l (coalesced 128 B rows), mask-gated
//              rho^d weights, packed z = f*w + i*w           (sampling.py:93-107,
//                                                              weights.py:18-37)
//   FFT        32-point in-register FFT along rows, smem transpose, FFT along
//              columns; split Z into R = F{f w} and W = F{w}, exactly Hermitian
//   loop       lane v owns spectral column v (R[u][v], u = 0..31, 64 regs);
//              W lives in shared memory with duplicated rows so the circular
//              shift W[(u-pu) mod 32][(v-pv) mod 32] is a per-lane base plus an
//              immediate offset; the residual update of iteration it-1 is fused
//              with the objective pass of iteration it, so R never leaves
//              registers and W is read once per bin per iteration.
//   argmax     per-lane running max over packed keys (objective bits with the
//              5 low mantissa bits replaced by the row's tie rank), then a
//              cross-lane step: __shfl_xor_sync butterfly on (key, lane rank)
//              (the paper's register argmax), or redux.sync, or a shared-memory
//              tree (the paper's comparison point) -- template ARGMAX.
//   synthesis  lanes p < B*B accumulate g(m,n) += Re(gp e^{2 pi i(u m + v n)/32})
//              directly (no inverse FFT, only the B x B target pixels), then
//              merge (known pixels copied) and stitch.
//   guard      fp32 near-tie guard: per-lane top-2 keys give the best and the
//              second-best objective of every iteration (excluding the exact
//              conjugate mirror while the state is exactly Hermitian); a block
//              whose relative gap ever drops below tau is queued for an fp64
//              re-run, which is what makes fp32 production match the fp64
//              reference within tolerance.
#pragma once

#include "fsr_common.cuh"
#include "fsr_fft.cuh"

namespace fsr {

enum ArgmaxImpl { AM_SHFL = 0, AM_SMEM = 1, AM_REDUX = 2 };

constexpr int W32_N = 32;
constexpr int W32_WROW = 32;                         // complex per W row
constexpr int W32_WBYTES = 2 * 32 * W32_WROW * 8;    // duplicated rows: 16 KiB
constexpr int W32_TILE_STRIDE = 33;                  // padded transpose tile row

struct Warp32Args {
    const float *px;
    int64_t px_pitch;
    const uint8_t *mask;
    int64_t mask_pitch;
    float *out;
    int64_t out_pitch;
    int64_t H, W;
    int B, L, iterations, early_stop;
    int64_t bcols, first, nblocks;
    float gamma;
    float tau;             // guard: relative gap threshold
    const float *decay;    // [32*32]
    const double *decay64; // [32*32] (fp64 prologue)
    const float *wf;       // [32*32]
    int32_t *sel;          // [total blocks, iterations] or null
    int32_t *done;         // [total blocks] or null
    unsigned int *empty_count;
    int32_t *empty_list;
    unsigned int *rerun_count;
    int32_t *rerun_list;
    float *gap_out;        // debug: per-block [2] min top-2 gaps (relative, scaled) or null
    int guard_mode;        // 0: relative gap (b1-b2)/b1; 1: cancellation-scaled (b1-b2)/sqrt(b1*B0)
};

template <int WARPS>
struct Warp32Smem {
    float2 wbuf[WARPS][2 * 32 * W32_WROW];  // duplicated-row W, also the transpose tile
    float2 cs[32];                          // cos/sin(2 pi j / 32)
    unsigned int red_key[WARPS][32];        // AM_SMEM scratch
    unsigned int red_rank[WARPS][32];
    float4 hist[WARPS][32];                 // deferred synthesis: (gr, gi, u, v) per selection
};

__device__ __forceinline__ uint32_t f2u(float x) { return __float_as_uint(x); }

// Extract R[u] for a warp-uniform dynamic u (jump table, no divergence).
__device__ __forceinline__ float2 pick32(const cpx<float> (&R)[32], int u) {
    float2 c;
    switch (u) {
#define FSR_PICK(i) \
    case i: c = make_float2(R[i].re, R[i].im); break;
        FSR_PICK(0) FSR_PICK(1) FSR_PICK(2) FSR_PICK(3) FSR_PICK(4) FSR_PICK(5) FSR_PICK(6)
        FSR_PICK(7) FSR_PICK(8) FSR_PICK(9) FSR_PICK(10) FSR_PICK(11) FSR_PICK(12)
        FSR_PICK(13) FSR_PICK(14) FSR_PICK(15) FSR_PICK(16) FSR_PICK(17) FSR_PICK(18)
        FSR_PICK(19) FSR_PICK(20) FSR_PICK(21) FSR_PICK(22) FSR_PICK(23) FSR_PICK(24)
        FSR_PICK(25) FSR_PICK(26) FSR_PICK(27) FSR_PICK(28) FSR_PICK(29) FSR_PICK(30)
        default: c = make_float2(R[31].re, R[31].im); break;
#undef FSR_PICK
    }
    return c;
}

// Cross-lane argmax on (key desc, rank asc); every lane gets the winner.
template <int ARGMAX>
__device__ __forceinline__ void cross_lane_best(uint32_t &key, uint32_t &rank,
                                                unsigned int *skey, unsigned int *srank) {
    const int lane = lane_id();
    if (ARGMAX == AM_SHFL) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            uint32_t ok = __shfl_xor_sync(0xffffffffu, key, off);
            uint32_t orank = __shfl_xor_sync(0xffffffffu, rank, off);
            bool take = ok > key || (ok == key && orank < rank);
            key = take ? ok : key;
            rank = take ? orank : rank;
        }
    } else if (ARGMAX == AM_REDUX) {
        const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
        const uint32_t tied = __ballot_sync(0xffffffffu, key == kmax);
        if (__popc(tied) == 1) {
            rank = __shfl_sync(0xffffffffu, rank, __ffs(tied) - 1);
        } else {  // exact tie on (objective, row rank): lowest lane rank wins
            rank = __reduce_min_sync(0xffffffffu, key == kmax ? rank : 0xffffffffu);
        }
        key = kmax;
    } else {  // AM_SMEM: classic shared-memory tree reduction
        skey[lane] = key;
        srank[lane] = rank;
        __syncwarp();
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
            if (lane < s) {
                uint32_t ok = skey[lane + s], orank = srank[lane + s];
                uint32_t mk = skey[lane], mr = srank[lane];
                if (ok > mk || (ok == mk && orank < mr)) {
                    skey[lane] = ok;
                    srank[lane] = orank;
                }
            }
            __syncwarp();
        }
        key = skey[0];
        rank = srank[0];
        __syncwarp();
    }
}

__device__ __forceinline__ uint32_t warp_max_u32(uint32_t x) {
    return __reduce_max_sync(0xffffffffu, x);
}

// One objective/update pass over the 32 rows a lane owns.
// HERM: the state is exactly Hermitian, keys of non-canonical bins are zeroed.
template <bool TREE, bool GUARD, bool HERM, bool UPDATE>
__device__ __forceinline__ void pass32(cpx<float> (&R)[32], const float (&wfr)[17],
                                       const float2 *wrow, float gr, float gi,
                                       uint32_t canon, uint32_t &m1, uint32_t &m2) {
    m1 = 0;
    m2 = 0;
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        float re = R[u].re, im = R[u].im;
        if (UPDATE) {
            const float2 w = wrow[u * W32_WROW];  // W[(u - pu) mod 32][(v - pv) mod 32]
            re = fmaf(-gr, w.x, re);
            re = fmaf(gi, w.y, re);
            im = fmaf(-gr, w.y, im);
            im = fmaf(-gi, w.x, im);
            R[u].re = re;
            R[u].im = im;
        }
        const float mag = fmaf(re, re, im * im);
        const float o = mag * wfr[u <= 16 ? u : 32 - u];
        const uint32_t rk = TREE ? ((u & 1) << 4 | (u & 2) << 2 | (u & 4) | (u & 8) >> 2 | (u & 16) >> 4)
                                     : (uint32_t)u;
        uint32_t key = (f2u(o) | 31u) ^ rk;  // low 5 bits = 31 - rank(u)
        if (HERM && GUARD) key = ((canon >> u) & 1u) ? key : 0u;
        if (GUARD) {
            uint32_t t = min(m1, key);
            m2 = max(m2, t);
        }
        m1 = max(m1, key);
    }
}

__device__ __forceinline__ int w32_tidx(int r, int c) { return r * 32 + (c ^ r); }

// fp64 prologue: gather, weights, 2-D FFT and Hermitian split in double
// precision, then R (registers) and W (duplicated-row shared layout) rounded
// to fp32 once.  Halves the initial spectral error of the fp32 loop (whose late
// iterations compare objectives of a residual 10^2-10^3 below R0), which cuts
// the guard's fp64 re-runs.  Returns the early-stop energy sum f^2 w.
__device__ __forceinline__ double w32_prologue_f64(const Warp32Args &a, float2 *wb, cpx<float> (&R)[32],
                                                   int64_t wr0, int64_t x, bool xin, int lane) {
    double2 *t = reinterpret_cast<double2 *>(wb);  // 16 KiB: XOR-swizzled 32x32 double2 tile
    double energy = 0.0;
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
        const int64_t y = wr0 + k;
        double f = 0.0, w = 0.0;
        if (xin && y >= 0 && y < a.H && a.mask[y * a.mask_pitch + x]) {
            f = (double)a.px[y * a.px_pitch + x];
            w = a.decay64[k * 32 + lane];
        }
        t[w32_tidx(k, lane)] = make_double2(f * w, w);
        energy = fma(f * f, w, energy);
    }
    __syncwarp();
    // Each 32-point line is done as two 16-point halves (even / odd samples) with
    // the radix-2 combine written back in place: line position 2m holds
    // frequency m, position 2m+1 frequency m+16 (permutation s below).  Peak
    // live data: 16 complex doubles.
    {
        cpx<double> xv[16];
        // rows (lane = window row)
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = t[w32_tidx(lane, 2 * j)]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int j = 0; j < 16; ++j) t[w32_tidx(lane, 2 * j)] = make_double2(xv[j].re, xv[j].im);
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = t[w32_tidx(lane, 2 * j + 1)]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const double2 e = t[w32_tidx(lane, 2 * m)];
            const double c = tw_cos(m), sn = tw_sin(m);
            const double tr = xv[m].re * c + xv[m].im * sn, ti = xv[m].im * c - xv[m].re * sn;
            t[w32_tidx(lane, 2 * m)] = make_double2(e.x + tr, e.y + ti);
            t[w32_tidx(lane, 2 * m + 1)] = make_double2(e.x - tr, e.y - ti);
        }
        __syncwarp();
        // columns (lane = frequency v, stored at line position cv)
        const int cv = lane < 16 ? 2 * lane : 2 * (lane - 16) + 1;
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = t[w32_tidx(2 * j, cv)]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int j = 0; j < 16; ++j) t[w32_tidx(2 * j, cv)] = make_double2(xv[j].re, xv[j].im);
#pragma unroll
        for (int j = 0; j < 16; ++j) { const double2 z = t[w32_tidx(2 * j + 1, cv)]; xv[j] = {z.x, z.y}; }
        fft_pow2<4>(xv);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const double2 e = t[w32_tidx(2 * m, cv)];
            const double c = tw_cos(m), sn = tw_sin(m);
            const double tr = xv[m].re * c + xv[m].im * sn, ti = xv[m].im * c - xv[m].re * sn;
            t[w32_tidx(2 * m, cv)] = make_double2(e.x + tr, e.y + ti);
            t[w32_tidx(2 * m + 1, cv)] = make_double2(e.x - tr, e.y - ti);
        }
        __syncwarp();
    }
    // split: Z[u][v] sits at (s(u), s(v)), s(f) = f < 16 ? 2f : 2(f-16)+1.
    // R and W are rounded to fp32 once, W kept in registers until every read is done.
    const int mv = (32 - lane) & 31;
    const int cv = lane < 16 ? 2 * lane : 2 * (lane - 16) + 1;
    const int cm = mv < 16 ? 2 * mv : 2 * (mv - 16) + 1;
    float2 Wf[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        const int nu = (32 - u) & 31;
        const int su = u < 16 ? 2 * u : 2 * (u - 16) + 1;
        const int sn = nu < 16 ? 2 * nu : 2 * (nu - 16) + 1;
        const double2 z = t[w32_tidx(su, cv)], zm = t[w32_tidx(sn, cm)];
        R[u] = {(float)((z.x + zm.x) * 0.5), (float)((z.y - zm.y) * 0.5)};
        Wf[u] = make_float2((float)((z.y + zm.y) * 0.5), (float)((zm.x - z.x) * 0.5));
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        wb[u * W32_WROW + lane] = Wf[u];
        wb[(u + 32) * W32_WROW + lane] = Wf[u];
    }
    __syncwarp();
    return energy;
}

#ifndef FSR_W32_FFT64
#define FSR_W32_FFT64 1
#endif
template <int WARPS, bool TREE, int ARGMAX, bool GUARD, bool FFT64 = (FSR_W32_FFT64 != 0)>
__global__ void __launch_bounds__(WARPS * 32, 12 / WARPS) warp32_kernel(Warp32Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Warp32Smem<WARPS> &sm = *reinterpret_cast<Warp32Smem<WARPS> *>(smem_raw);
    const int lane = lane_id(), wid = warp_id();
    if (threadIdx.x < 32) {
        const double th = 6.283185307179586476925286766559 * threadIdx.x / 32.0;
        sm.cs[threadIdx.x] = make_float2((float)cos(th), (float)sin(th));
    }
    __syncthreads();
    float2 *wb = sm.wbuf[wid];
    const int v = lane;
    const uint32_t lrank = TREE ? bitrev5(lane) : lane;
    // canonical half of each mirror pair (lower tie rank), bit u of this lane's column
    uint32_t canon = 0;
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        int t = u * 32 + v, mt = ((32 - u) & 31) * 32 + ((32 - v) & 31);
        canon |= (uint32_t)(tie_rank(t, TREE) <= tie_rank(mt, TREE)) << u;
    }
    // folded frequency prior of this column: wf[u][v] == wf[32-u][v] (weights.py:40-56)
    float wfr[17];
#pragma unroll
    for (int u = 0; u <= 16; ++u) wfr[u] = a.wf[u * 32 + v];

    const int64_t total_warps = (int64_t)gridDim.x * WARPS;
    for (int64_t i = (int64_t)blockIdx.x * WARPS + wid; i < a.nblocks; i += total_warps) {
        const int64_t bid = a.first + i;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const int64_t wr0 = r0 - a.L, x = c0 - a.L + lane;
        const bool xin = x >= 0 && x < a.W;
        cpx<float> R[32];
        float energy = 0.f;
        if (FFT64) {
            energy = (float)w32_prologue_f64(a, wb, R, wr0, x, xin, lane);
        } else {
            // ---- gather: lane = window column; row k coalesced across lanes
    #pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int64_t y = wr0 + k;
                float f = 0.f, w = 0.f;
                if (xin && y >= 0 && y < a.H) {
                    if (a.mask[y * a.mask_pitch + x]) {
                        f = a.px[y * a.px_pitch + x];
                        w = a.decay[k * 32 + lane];
                    }
                }
                // w scaled by 2^7 (exact) so both halves of the packed transform have
                // comparable magnitude and W is not swamped by the rounding of F{f w}
                R[k] = {f * w, w * 128.f};
                energy = fmaf(f * f, w, energy);
            }
            // ---- 2-D FFT of z: transpose (lane = row k), FFT over l, transpose, FFT over k
            float2 *tile = wb;  // padded [32][33]
    #pragma unroll
            for (int k = 0; k < 32; ++k) tile[k * W32_TILE_STRIDE + lane] = make_float2(R[k].re, R[k].im);
            __syncwarp();
    #pragma unroll
            for (int l = 0; l < 32; ++l) {
                float2 z = tile[lane * W32_TILE_STRIDE + l];
                R[l] = {z.x, z.y};
            }
            __syncwarp();
            fft32(R);  // lane k: Y[k][v], register v
    #pragma unroll
            for (int q = 0; q < 32; ++q) tile[lane * W32_TILE_STRIDE + q] = make_float2(R[q].re, R[q].im);
            __syncwarp();
    #pragma unroll
            for (int k = 0; k < 32; ++k) {
                float2 z = tile[k * W32_TILE_STRIDE + lane];
                R[k] = {z.x, z.y};
            }
            __syncwarp();
            fft32(R);  // lane v: Z[u][v], register u
            // ---- split Z into R and W via the conjugate mirror Z[-u][-v]:
            // Z -> upper half of wb (stride 32), W -> lower half, then duplicate rows.
            float2 *zt = wb + 32 * W32_WROW;
    #pragma unroll
            for (int u = 0; u < 32; ++u) zt[u * W32_WROW + lane] = make_float2(R[u].re, R[u].im);
            __syncwarp();
            const int mv = (32 - lane) & 31;
    #pragma unroll
            for (int u = 0; u < 32; ++u) {
                const float2 zm = zt[((32 - u) & 31) * W32_WROW + mv];
                const float zr = R[u].re, zi = R[u].im;
                R[u] = {(zr + zm.x) * 0.5f, (zi - zm.y) * 0.5f};
                wb[u * W32_WROW + lane] = make_float2((zi + zm.y) * (0.5f / 128.f), (zm.x - zr) * (0.5f / 128.f));
            }
            __syncwarp();
    #pragma unroll
            for (int u = 0; u < 32; ++u) zt[u * W32_WROW + lane] = wb[u * W32_WROW + lane];
            __syncwarp();
        }
        const float w00 = wb[0].x;
        int32_t *sel_b = a.sel ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
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
        // early stop threshold: 1e-12 * sum f^2 w (reconstruction.py:262-266)
        float thr = 0.f;
        if (a.early_stop) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, off);
            thr = 1e-12f * energy;
        }
        const float ginv = a.gamma / w00;
        // target pixel of this lane (p < B*B): window coordinates (L + m, L + n)
        const int B = a.B;
        const int pm = a.L + lane / B, pn = a.L + lane % B;
        const bool has_pix = lane < B * B;
        float acc = 0.f;
        bool herm = true;
        bool flagged = false;
        float min_gap = 1.f, min_gap2 = 1.f, B0 = 0.f;
        const float one_minus_tau = 1.f - a.tau;
        float gr = 0.f, gi = 0.f;
        int pu = 0, pv = 0;
        int done = 0;
        float4 *hist = sm.hist[wid];
        for (int it = 0; it < a.iterations; ++it) {
            uint32_t m1, m2;
            const float2 *wrow = wb + (32 - pu) * W32_WROW + ((v - pv) & 31);
            if (it == 0) {
                pass32<TREE, GUARD, true, false>(R, wfr, wrow, gr, gi, canon, m1, m2);
            } else if (herm) {
                pass32<TREE, GUARD, true, true>(R, wfr, wrow, gr, gi, canon, m1, m2);
            } else {
                pass32<TREE, GUARD, false, true>(R, wfr, wrow, gr, gi, canon, m1, m2);
            }
            uint32_t key = m1, rank = lrank;
            cross_lane_best<ARGMAX>(key, rank, sm.red_key[wid], sm.red_rank[wid]);
            const uint32_t urank = 31u - (key & 31u);
            const int bu = TREE ? (int)bitrev5(urank) : (int)urank;
            const int bv = TREE ? (int)bitrev5(rank) : (int)rank;
            const float b1 = __uint_as_float(key & ~31u);
            if (GUARD) {
                // second-best objective: the winner lane's runner-up or any other lane's best
                const uint32_t k2 = warp_max_u32((lane == bv) ? m2 : m1);
                const float b2 = __uint_as_float(k2 & ~31u);
                flagged |= b1 > 0.f && b2 >= b1 * one_minus_tau;
                // a stop decision within tau of the threshold is also ambiguous
                flagged |= thr > 0.f && fabsf(b1 - thr) <= a.tau * thr;
                if (a.gap_out) {  // guard-study instrumentation (tools/guard_study.py)
                    if (it == 0) B0 = b1;
                    min_gap = fminf(min_gap, b1 > 0.f ? (b1 - b2) / b1 : 1.f);
                    min_gap2 = fminf(min_gap2, b1 > 0.f ? (b1 - b2) * rsqrtf(b1 * B0) : 1.f);
                }
            }
            if (sel_b && lane == 0) sel_b[it] = bu * 32 + bv;
            if (thr > 0.f && b1 < thr) break;
            float2 c = pick32(R, bu);
            c.x = __shfl_sync(0xffffffffu, c.x, bv);
            c.y = __shfl_sync(0xffffffffu, c.y, bv);
            gr = c.x * ginv;
            gi = c.y * ginv;
            pu = bu;
            pv = bv;
            // a non-self-mirror selection breaks the exact Hermitian symmetry
            herm = herm && (((32 - bu) & 31) == bu) && (((32 - bv) & 31) == bv);
            // deferred synthesis of the target pixels: record, flush every 32
            if (lane == 0) hist[it & 31] = make_float4(gr, gi, __int_as_float(bu), __int_as_float(bv));
            if ((it & 31) == 31) {
                __syncwarp();
#pragma unroll 4
                for (int j = 0; j < 32; ++j) {
                    const float4 h = hist[j];
                    const float2 e = sm.cs[(__float_as_int(h.z) * pm + __float_as_int(h.w) * pn) & 31];
                    acc = fmaf(h.x, e.x, fmaf(-h.y, e.y, acc));
                }
                __syncwarp();
            }
            done = it + 1;
        }
        {
            __syncwarp();
            const int rem = done & 31;
            for (int j = 0; j < rem; ++j) {
                const float4 h = hist[j];
                const float2 e = sm.cs[(__float_as_int(h.z) * pm + __float_as_int(h.w) * pn) & 31];
                acc = fmaf(h.x, e.x, fmaf(-h.y, e.y, acc));
            }
            __syncwarp();
        }
        if (sel_b)
            for (int it = done + lane; it < a.iterations; it += 32) sel_b[it] = -1;
        if (lane == 0) {
            if (a.done) a.done[bid] = done;
            if (GUARD && a.gap_out) {
                a.gap_out[2 * bid] = min_gap;
                a.gap_out[2 * bid + 1] = min_gap2;
            }
            if (GUARD && flagged && a.rerun_list) {
                unsigned slot = atomicAdd(a.rerun_count, 1u);
                a.rerun_list[slot] = (int32_t)bid;
            }
        }
        // merge + stitch
        if (has_pix) {
            const int m = lane / B, n = lane % B;
            const int64_t y = r0 + m, xx = c0 + n;
            if (y < a.H && xx < a.W)
                a.out[y * a.out_pitch + xx] =
                    a.mask[y * a.mask_pitch + xx] ? a.px[y * a.px_pitch + xx] : acc;
        }
        __syncwarp();
    }
}

}  // namespace fsr
