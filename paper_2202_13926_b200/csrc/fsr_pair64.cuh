// fsr_pair64.cuh -- production FSR kernel for support N = 32 in fp64: one warp
// PAIR per target block, the residual spectrum register-resident.
//
// Why fp64: the greedy decisions of the late iterations compare objectives of
// a residual that has shrunk by 10^2..10^3 against R0; an fp32 loop carries an
// absolute error of ~eps32*|R0| and so flips 20-50 % of the blocks' selection
// paths against the fp64 reference (tools/guard_study.py), far
// outside the 1e-3 pixel tolerance.  B200 runs DFMA at half the FFMA rate, and
// the loop below is bounded by shared-memory bandwidth for W (16 B/bin) and the
// DP pipe (7 DP ops/bin) about equally.
//
// Layout per block (warps 2p and 2p+1 of the CTA, "halves" H = 0, 1):
//   * lane v owns spectral column v; half H owns a set of 16 rows closed under
//     u -> -u mod 32:  H=0: {0..7, 16, 25..31},  H=1: {8..15, 17..24}, so the
//     folded frequency prior needs 9 / 8 doubles and the conjugate split never
//     crosses halves.  R[u][v] for the 16 rows: 64 registers.
//   * one 24 KiB shared buffer per block: XOR-swizzled transpose tile during the
//     2-D FFT, then W[u][v] row-major for the loop, rows 0..15 repeated as rows
//     32..47 (rows read across lanes: conflict-free; the circular row shift is
//     one base address per iteration plus compile-time row offsets).
//   * FFT: each 32-point line is split radix-2 between the halves (16-point
//     in-register FFT of the even / odd samples, exchanged through the tile).
//   * per iteration: fused residual update + objective + running max over
//     packed keys (fp64 objective with the 5 low mantissa bits replaced by the
//     row's tie rank: comparisons exact to 2^-47), cross-lane argmax (template:
//     shfl butterfly / redux / shared-memory tree), one named barrier to combine
//     the two halves through double-buffered slots that also carry the winning
//     coefficient R[u*][v*], so no second round trip is needed.
#pragma once

#include "fsr_common.cuh"
#include "fsr_fft.cuh"
#include "fsr_warp32.cuh"

namespace fsr {

#ifndef FSR_P64_BRX
#define FSR_P64_BRX 1
#endif
// W table rows per block: 48 = rows 0..31 plus copies of rows 0..15, so each
// half's rows (one circular run of 15 or 17 rows, plus row 16 for H=0) are read
// at compile-time offsets from one per-iteration base (no wrap); 32 = the
// 16 KiB-aligned table with a masked row shift (two ALU ops per row)
#ifndef FSR_P64_ROWS
#define FSR_P64_ROWS 48
#endif
constexpr int kP64Rows = FSR_P64_ROWS;
static_assert(kP64Rows == 32 || kP64Rows == 48, "FSR_P64_ROWS must be 32 or 48");

template <typename IO>
struct Pair64Args {
    const IO *px;
    int64_t px_pitch;
    const uint8_t *mask;
    int64_t mask_pitch;
    IO *out;
    int64_t out_pitch;
    int64_t H, W;
    int B, L, iterations, early_stop;
    int64_t bcols, first, nblocks;
    const int32_t *list;            // optional block-id list (length *list_count)
    const unsigned int *list_count;
    double gamma;
    const double *decay;            // [32*32]
    const double *wf;               // [32*32]
    int32_t *sel;                   // [total blocks, iterations] or null
    int32_t *done;
    unsigned int *empty_count;
    int32_t *empty_list;
    double2 *scratch;               // cta64d: per-CTA 64 KiB staging of W (null elsewhere)
    int tree;                       // reducer for kernels that take it at run time (warpnd)
    // replay (pair64 list mode): list entry b re-runs iterations [0, list_kf[b]) as
    // argmax-free updates along the fp32 kernel's selections list_seq[b * seq_stride + j]
    // (u * 32 + v), whose decisions the guard found unambiguous, then searches in fp64
    const int32_t *list_kf;
    const uint16_t *list_seq;
    int seq_stride;
};

struct __align__(16) PairSlot {
    double key;
    uint32_t lrank;
    uint32_t pad;
    double cre, cim;
    double energy;
    double pad2;
};

// One greedy selection, kept for the deferred synthesis of the target pixels.
struct __align__(16) SelEntry {
    double gr, gi;  // gamma * c / W00
    int u, v;       // selected bin
    int pad[2];
};

template <int BPC>
struct Pair64Smem {
    double2 buf[BPC][kP64Rows * 32];  // FFT tile (rows 0..31), then the W table
    double2 align_pad[kP64Rows == 32 ? 1024 : 1];  // 32 rows: room to align &buf to 16 KiB
    PairSlot slot[BPC][2][2];     // [block][parity][half]
    unsigned int red_hi[BPC][2][32];
    unsigned int red_lo[BPC][2][32];
    SelEntry hist[BPC][2][16];    // per half: every other selection, flushed every 32
    double acc_x[BPC][32];        // half 1's partial pixel sums
    double2 cs[32];               // (cos, sin)(2 pi j / 32)
};

// Deferred synthesis: acc += sum_j Re(gp_j e^{2 pi i (u_j m + v_j n)/32}) over n entries.
template <int BPC>
__device__ __forceinline__ double p64_flush(const Pair64Smem<BPC> &sm, const SelEntry *h, int n,
                                            int pm, int pn, double acc) {
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
        const SelEntry e = h[j];
        const double2 cs = sm.cs[(e.u * pm + e.v * pn) & 31];
        acc = fma(e.gr, cs.x, fma(-e.gi, cs.y, acc));
    }
    return acc;
}

// rows owned by half H, slot i = 0..15 (closed under u -> -u mod 32)
__host__ __device__ constexpr int p64_row(int H, int i) {
    return H == 0 ? (i < 8 ? i : (i == 8 ? 16 : 16 + i)) : (i < 8 ? 8 + i : 9 + i);
}
__host__ __device__ constexpr int p64_fold(int u) { return u <= 16 ? u : 32 - u; }
__host__ __device__ constexpr uint32_t brev5c(int x) {
    return (uint32_t)(((x & 1) << 4) | ((x & 2) << 2) | (x & 4) | ((x & 8) >> 2) | ((x & 16) >> 4));
}
// slot of row u in half H (or -1)
__host__ __device__ constexpr int p64_slot(int H, int u) {
    return H == 0 ? (u < 8 ? u : (u == 16 ? 8 : (u >= 25 ? u - 16 : -1)))
                  : (u >= 8 && u < 16 ? u - 8 : (u >= 17 && u <= 24 ? u - 9 : -1));
}

__device__ __forceinline__ int tidx(int r, int c) { return r * 32 + (c ^ r); }  // swizzled tile

__device__ __forceinline__ void bar_pair(int id) {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

__device__ __forceinline__ double2 ldd2(const double2 *p) { return *p; }

template <typename IO>
__device__ __forceinline__ double load_px(const IO *p) { return (double)__ldg(p); }

// Extract R[i] for a warp-uniform dynamic slot i in [0, 16).
__device__ __forceinline__ double2 pick16(const cpx<double> (&R)[16], int i) {
    double2 c;
    switch (i) {
#define FSR_PICK(k) \
    case k: c = make_double2(R[k].re, R[k].im); break;
        FSR_PICK(0) FSR_PICK(1) FSR_PICK(2) FSR_PICK(3) FSR_PICK(4) FSR_PICK(5) FSR_PICK(6)
        FSR_PICK(7) FSR_PICK(8) FSR_PICK(9) FSR_PICK(10) FSR_PICK(11) FSR_PICK(12) FSR_PICK(13)
        FSR_PICK(14)
        default: c = make_double2(R[15].re, R[15].im); break;
#undef FSR_PICK
    }
    return c;
}

// R[i] of this lane by one indirect branch (brx.idx jump table); i warp-uniform.
__device__ __forceinline__ double2 pick16_brx(const cpx<double> (&R)[16], int i) {
    double2 c;
    asm volatile(
        "{\n ts%=: .branchtargets L0_%=, L1_%=, L2_%=, L3_%=, L4_%=, L5_%=, L6_%=, L7_%=, L8_%=, L9_%=, L10_%=, L11_%=, L12_%=, L13_%=, L14_%=, L15_%=;\n"
        " brx.idx %2, ts%=;\n"
        " L0_%=: mov.f64 %0, %3; mov.f64 %1, %4; bra.uni Le_%=;\n"
        " L1_%=: mov.f64 %0, %5; mov.f64 %1, %6; bra.uni Le_%=;\n"
        " L2_%=: mov.f64 %0, %7; mov.f64 %1, %8; bra.uni Le_%=;\n"
        " L3_%=: mov.f64 %0, %9; mov.f64 %1, %10; bra.uni Le_%=;\n"
        " L4_%=: mov.f64 %0, %11; mov.f64 %1, %12; bra.uni Le_%=;\n"
        " L5_%=: mov.f64 %0, %13; mov.f64 %1, %14; bra.uni Le_%=;\n"
        " L6_%=: mov.f64 %0, %15; mov.f64 %1, %16; bra.uni Le_%=;\n"
        " L7_%=: mov.f64 %0, %17; mov.f64 %1, %18; bra.uni Le_%=;\n"
        " L8_%=: mov.f64 %0, %19; mov.f64 %1, %20; bra.uni Le_%=;\n"
        " L9_%=: mov.f64 %0, %21; mov.f64 %1, %22; bra.uni Le_%=;\n"
        " L10_%=: mov.f64 %0, %23; mov.f64 %1, %24; bra.uni Le_%=;\n"
        " L11_%=: mov.f64 %0, %25; mov.f64 %1, %26; bra.uni Le_%=;\n"
        " L12_%=: mov.f64 %0, %27; mov.f64 %1, %28; bra.uni Le_%=;\n"
        " L13_%=: mov.f64 %0, %29; mov.f64 %1, %30; bra.uni Le_%=;\n"
        " L14_%=: mov.f64 %0, %31; mov.f64 %1, %32; bra.uni Le_%=;\n"
        " L15_%=: mov.f64 %0, %33; mov.f64 %1, %34; bra.uni Le_%=;\n"
        " Le_%=:\n}"
        : "=d"(c.x), "=d"(c.y)
        : "r"(i & 15),
          "d"(R[0].re), "d"(R[0].im),
          "d"(R[1].re), "d"(R[1].im),
          "d"(R[2].re), "d"(R[2].im),
          "d"(R[3].re), "d"(R[3].im),
          "d"(R[4].re), "d"(R[4].im),
          "d"(R[5].re), "d"(R[5].im),
          "d"(R[6].re), "d"(R[6].im),
          "d"(R[7].re), "d"(R[7].im),
          "d"(R[8].re), "d"(R[8].im),
          "d"(R[9].re), "d"(R[9].im),
          "d"(R[10].re), "d"(R[10].im),
          "d"(R[11].re), "d"(R[11].im),
          "d"(R[12].re), "d"(R[12].im),
          "d"(R[13].re), "d"(R[13].im),
          "d"(R[14].re), "d"(R[14].im),
          "d"(R[15].re), "d"(R[15].im));
    return c;
}

// Packed 64-bit keys: the fp64 objective with its 10 low mantissa bits replaced
// by (31 - row rank) << 5 | (31 - lane rank).  Objectives are >= 0, so keys
// order like the objectives (exact to 2^-42 relative) and ties resolve to the
// reference's rule (tree: lexicographic (bitrev5(u), bitrev5(v)); linear:
// flat index); every bin's key is unique, so a plain u64 max is the argmax.
__device__ __forceinline__ unsigned long long u64max(unsigned long long a, unsigned long long b) {
    return a > b ? a : b;
}

// Shared address of W[(u - pu) & 31][(v - pv) & 31] for slot i of half H.
//   48 rows: P = address of row (S_H - pu) & 31 (S_0 = 25, S_1 = 8) plus the
//            column, ycv = address of row (16 - pu) & 31 plus the column (H=0);
//   32 rows: P = ((32 - pu) & 31) << 9, ycv = table | ((v - pv) & 31) << 4.
template <int H>
__device__ __forceinline__ uint32_t p64_waddr(int i, uint32_t P, uint32_t ycv) {
    const int u = p64_row(H, i);
    if (kP64Rows == 32) return ((P + ((uint32_t)u << 9)) & 0x3E00u) | ycv;
    if (H == 0 && u == 16) return ycv;
    const int k = H == 0 ? (u - 25) & 31 : u - 8;  // position in the half's circular run
    return P + ((uint32_t)k << 9);
}
// The per-iteration (P, ycv) of p64_waddr for selection (pu, pv).
template <int H>
__device__ __forceinline__ void p64_wbase(uint32_t wb, int lane, int pu, int pv, uint32_t &P,
                                          uint32_t &ycv) {
    const uint32_t col = (uint32_t)((lane - pv) & 31) << 4;
    if (kP64Rows == 32) {
        P = (uint32_t)((32 - pu) & 31) << 9;
        ycv = wb | col;
    } else {
        P = wb + ((uint32_t)(((H == 0 ? 25 : 8) - pu) & 31) << 9) + col;
        ycv = wb + ((uint32_t)((16 - pu) & 31) << 9) + col;
    }
}

// The residual update alone (replayed iterations): R -= gp W(. - pu, . - pv).
template <int H>
__device__ __forceinline__ void p64_update(cpx<double> (&R)[16], uint32_t P, uint32_t ycv, double gr,
                                           double gi) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const uint32_t addr = p64_waddr<H>(i, P, ycv);
        double2 w;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y) : "r"(addr));
        double re = R[i].re, im = R[i].im;
        re = fma(-gr, w.x, re);
        re = fma(gi, w.y, re);
        im = fma(-gr, w.y, im);
        im = fma(-gi, w.x, im);
        R[i].re = re;
        R[i].im = im;
    }
}

// One residual-update + objective pass over the 16 rows of half H.
// P = ((32 - pu) & 31) << 9, ycv = shared address of W | ((v - pv) & 31) << 4.
// Returns the lane's best key with the lane-rank bits still all ones.
template <int H, bool TREE, bool UPDATE>
__device__ __forceinline__ unsigned long long p64_pass(cpx<double> (&R)[16], const double (&wfr)[17],
                                                       uint32_t P, uint32_t ycv, double gr,
                                                       double gi, uint32_t cmask) {
    unsigned long long best[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int u = p64_row(H, i);
        double re = R[i].re, im = R[i].im;
        if (UPDATE) {
            // W[(u - pu) & 31][(v - pv) & 31]
            const uint32_t addr = p64_waddr<H>(i, P, ycv);
            double2 w;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y) : "r"(addr));
            re = fma(-gr, w.x, re);
            re = fma(gi, w.y, re);
            im = fma(-gr, w.y, im);
            im = fma(-gi, w.x, im);
            R[i].re = re;
            R[i].im = im;
        }
        const double mag = fma(re, re, im * im);
        const double o = mag * wfr[p64_fold(u)];
        const uint32_t rk = TREE ? brev5c(u) : (uint32_t)u;
        // low 10 bits <- (31 - rk) << 5 | 31: bitwise mux with the 0x3FF mask, one LOP3
        uint32_t lo;
        asm("lop3.b32 %0, %1, %2, %3, 0xD8;"
            : "=r"(lo) : "r"((uint32_t)__double2loint(o)), "r"(((31u - rk) << 5) | 31u), "r"(cmask));
        const unsigned long long k =
            ((unsigned long long)(uint32_t)__double2hiint(o) << 32) | (unsigned long long)lo;
        best[i & 3] = u64max(best[i & 3], k);
    }
    return u64max(u64max(best[0], best[1]), u64max(best[2], best[3]));
}

// Warp max of unique u64 keys; every lane receives it.
template <int ARGMAX>
__device__ __forceinline__ unsigned long long p64_warp_max(unsigned long long k, unsigned int *shi,
                                                           unsigned int *slo) {
    uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
    if (ARGMAX == AM_REDUX) {
        const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
        const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        return ((unsigned long long)mh << 32) | ml;
    } else if (ARGMAX == AM_SHFL) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const uint32_t oh = __shfl_xor_sync(0xffffffffu, hi, off);
            const uint32_t ol = __shfl_xor_sync(0xffffffffu, lo, off);
            const unsigned long long o = ((unsigned long long)oh << 32) | ol;
            const unsigned long long m = u64max(o, ((unsigned long long)hi << 32) | lo);
            hi = (uint32_t)(m >> 32);
            lo = (uint32_t)m;
        }
        return ((unsigned long long)hi << 32) | lo;
    } else {  // shared-memory tree (the paper's comparison point)
        const int lane = lane_id();
        shi[lane] = hi;
        slo[lane] = lo;
        __syncwarp();
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
            if (lane < s) {
                const unsigned long long o = ((unsigned long long)shi[lane + s] << 32) | slo[lane + s];
                const unsigned long long m = ((unsigned long long)shi[lane] << 32) | slo[lane];
                if (o > m) {
                    shi[lane] = (uint32_t)(o >> 32);
                    slo[lane] = (uint32_t)o;
                }
            }
            __syncwarp();
        }
        const unsigned long long r = ((unsigned long long)shi[0] << 32) | slo[0];
        __syncwarp();
        return r;
    }
}

template <int BPC, int H, bool TREE, int ARGMAX, typename IO>
__device__ __forceinline__ void p64_half(const Pair64Args<IO> &a, Pair64Smem<BPC> &sm,
                                         double2 *bufs, int pair) {
    const int lane = lane_id();
    const int bar_id = 1 + pair;
    double2 *buf = bufs + pair * (kP64Rows * 32);
    const uint32_t wb = (uint32_t)__cvta_generic_to_shared(buf);  // 16 KiB aligned when kP64Rows == 32
    const uint32_t lrank = TREE ? bitrev5(lane) : (uint32_t)lane;
    double wfr[17];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int f = p64_fold(p64_row(H, i));
        wfr[f] = a.wf[f * 32 + lane];
    }
    const int64_t nblocks = a.list_count ? (int64_t)*a.list_count : a.nblocks;
    const int64_t stride = (int64_t)gridDim.x * BPC;
    int parity = 0;
    for (int64_t bi = (int64_t)blockIdx.x * BPC + pair; bi < nblocks; bi += stride) {
        const int64_t bid = a.list ? (int64_t)a.list[bi] : a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const int64_t wr0 = r0 - a.L, x = c0 - a.L + lane;
        const bool xin = x >= 0 && x < a.W;
        // ---- gather: lane = window column, half H takes rows 16H..16H+15
        double energy = 0.0;
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
            const int k = 16 * H + j;
            const int64_t y = wr0 + k;
            double f = 0.0, w = 0.0;
            if (xin && y >= 0 && y < a.H && a.mask[y * a.mask_pitch + x]) {
                f = load_px(a.px + y * a.px_pitch + x);
                w = a.decay[k * 32 + lane];
            }
            buf[tidx(k, lane)] = make_double2(f * w, w);  // packed z = f w + i w
            energy = fma(f * f, w, energy);
        }
        if (a.early_stop) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, off);
            if (lane == 0) sm.slot[pair][parity][H].energy = energy;
        }
        bar_pair(bar_id);
        // ---- row FFTs (lane = window row k): half H transforms samples l = 2j + H
        {
            cpx<double> x16[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const double2 z = buf[tidx(lane, 2 * j + H)];
                x16[j] = {z.x, z.y};
            }
            fft_pow2<4>(x16);
            bar_pair(bar_id);
#pragma unroll
            for (int m = 0; m < 16; ++m) buf[tidx(lane, 16 * H + m)] = make_double2(x16[m].re, x16[m].im);
            bar_pair(bar_id);
            // combine: Y[m] = E[m] + W32^m O[m] (H=0), Y[m+16] = E[m] - W32^m O[m] (H=1)
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const double2 o = buf[tidx(lane, 16 * (1 - H) + m)];
                const double c = tw_cos(m), s = tw_sin(m);
                double er, ei, orr, oi;
                if (H == 0) { er = x16[m].re; ei = x16[m].im; orr = o.x; oi = o.y; }
                else { er = o.x; ei = o.y; orr = x16[m].re; oi = x16[m].im; }
                const double tr = orr * c + oi * s, ti = oi * c - orr * s;  // W32^m O = O (c - i s)
                x16[m] = H == 0 ? cpx<double>{er + tr, ei + ti} : cpx<double>{er - tr, ei - ti};
            }
            bar_pair(bar_id);
#pragma unroll
            for (int m = 0; m < 16; ++m) buf[tidx(lane, 16 * H + m)] = make_double2(x16[m].re, x16[m].im);
            bar_pair(bar_id);
            // ---- column FFTs (lane = column v): half H transforms rows k = 2j + H
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const double2 z = buf[tidx(2 * j + H, lane)];
                x16[j] = {z.x, z.y};
            }
            fft_pow2<4>(x16);
            bar_pair(bar_id);
#pragma unroll
            for (int u = 0; u < 16; ++u) buf[tidx(16 * H + u, lane)] = make_double2(x16[u].re, x16[u].im);
            bar_pair(bar_id);
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const double2 o = buf[tidx(16 * (1 - H) + u, lane)];
                const double c = tw_cos(u), s = tw_sin(u);
                double er, ei, orr, oi;
                if (H == 0) { er = x16[u].re; ei = x16[u].im; orr = o.x; oi = o.y; }
                else { er = o.x; ei = o.y; orr = x16[u].re; oi = x16[u].im; }
                const double tr = orr * c + oi * s, ti = oi * c - orr * s;
                x16[u] = H == 0 ? cpx<double>{er + tr, ei + ti} : cpx<double>{er - tr, ei - ti};
            }
            bar_pair(bar_id);
#pragma unroll
            for (int u = 0; u < 16; ++u) buf[tidx(16 * H + u, lane)] = make_double2(x16[u].re, x16[u].im);
            bar_pair(bar_id);
        }
        // ---- split Z into R (registers) and W (row-major in buf), pairs (u, -u) of this half
        cpx<double> R[16];
        const int mv = (32 - lane) & 31;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int u = p64_row(H, i);
            const int nu = (32 - u) & 31;
            if (u > 16 && u != 0) continue;  // handled as the partner of 32 - u
            const int j = p64_slot(H, nu);
            const double2 zp = buf[tidx(u, lane)], zpm = buf[tidx(nu, mv)];
            const double2 zn = buf[tidx(nu, lane)], znm = buf[tidx(u, mv)];
            R[i] = {(zp.x + zpm.x) * 0.5, (zp.y - zpm.y) * 0.5};
            const double2 wp = make_double2((zp.y + zpm.y) * 0.5, (zpm.x - zp.x) * 0.5);
            double2 wn = wp;
            if (nu != u) {
                R[j] = {(zn.x + znm.x) * 0.5, (zn.y - znm.y) * 0.5};
                wn = make_double2((zn.y + znm.y) * 0.5, (znm.x - zn.x) * 0.5);
            }
            __syncwarp();
            buf[u * 32 + lane] = wp;
            if (nu != u) buf[nu * 32 + lane] = wn;
            if (kP64Rows == 48) {  // rows 32..47 repeat rows 0..15 (outside the FFT tile)
                if (u < 16) buf[(u + 32) * 32 + lane] = wp;
                if (nu != u && nu < 16) buf[(nu + 32) * 32 + lane] = wn;
            }
            __syncwarp();
        }
        bar_pair(bar_id);
        const double w00 = buf[0].x;
        int32_t *sel_b = a.sel ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (!(w00 > 0.0)) {
            if (H == 0 && lane == 0) {
                unsigned slot = atomicAdd(a.empty_count, 1u);
                if (a.empty_list) a.empty_list[slot] = (int32_t)bid;
                if (a.done) a.done[bid] = 0;
            }
            if (H == 0 && sel_b)
                for (int it = lane; it < a.iterations; it += 32) sel_b[it] = -1;
            bar_pair(bar_id);
            continue;
        }
        double thr = 0.0;
        if (a.early_stop)
            thr = 1e-12 * (sm.slot[pair][parity][0].energy + sm.slot[pair][parity][1].energy);
        const double ginv = a.gamma / w00;
        const int B = a.B;
        const int pm = a.L + lane / B, pn = a.L + lane % B;
        const bool has_pix = lane < B * B;
        double acc = 0.0;
        double gr = 0.0, gi = 0.0;
        uint32_t P = 0, ycv = wb;
        const uint32_t cmask = 0x3FFu;
        SelEntry *hist = sm.hist[pair][H];
        int done = 0;
        const int kf = a.list_kf ? a.list_kf[bi] : 0;
        const uint16_t *seq = a.list_kf ? a.list_seq + bi * (int64_t)a.seq_stride : nullptr;
        for (int it = 0; it < a.iterations; ++it) {
            if (it < kf) {
                // replayed iteration: the selection is known, only the update runs;
                // the half holding row wu publishes R[wu][wv] (one pair barrier)
                const uint32_t s = seq[it];
                const int wu = (int)(s >> 5), wv = (int)(s & 31u);
                if (it > 0) p64_update<H>(R, P, ycv, gr, gi);
                const int hold = p64_slot(0, wu) >= 0 ? 0 : 1;
                PairSlot *ps = &sm.slot[pair][parity][0];
                if (H == hold) {
                    const double2 cw = pick16_brx(R, p64_slot(H, wu) & 15);
                    if (lane == wv) {
                        ps[H].cre = cw.x;
                        ps[H].cim = cw.y;
                    }
                }
                bar_pair(bar_id);
                const double2 c = make_double2(ps[hold].cre, ps[hold].cim);
                parity ^= 1;
                if (H == 0 && sel_b && lane == 0) sel_b[it] = wu * 32 + wv;
                gr = c.x * ginv;
                gi = c.y * ginv;
                p64_wbase<H>(wb, lane, wu, wv, P, ycv);
                if ((it & 1) == H && lane == 0) hist[(it >> 1) & 15] = SelEntry{gr, gi, wu, wv, {0, 0}};
                if ((it & 31) == 31) {
                    __syncwarp();
                    acc = p64_flush(sm, hist, 16, pm, pn, acc);
                    __syncwarp();
                }
                done = it + 1;
                continue;
            }
            unsigned long long kb = it == 0
                ? p64_pass<H, TREE, false>(R, wfr, P, ycv, gr, gi, cmask)
                : p64_pass<H, TREE, true>(R, wfr, P, ycv, gr, gi, cmask);
            kb ^= lrank;  // lane-rank bits: 31 - lrank; every key is unique
            // warp argmax -> the winning lane of this half (warp-uniform)
            int wl;
            if (ARGMAX == AM_REDUX) {
                // one redux on the high words; the low words only break exact ties there
                const uint32_t hi = (uint32_t)(kb >> 32);
                const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
                uint32_t cand = __ballot_sync(0xffffffffu, hi == mh);
                if (__popc(cand) > 1) {
                    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? (uint32_t)kb : 0u);
                    cand = __ballot_sync(0xffffffffu, hi == mh && (uint32_t)kb == ml);
                }
                wl = __ffs(cand) - 1;
            } else {
                const unsigned long long key = p64_warp_max<ARGMAX>(kb, sm.red_hi[pair][H],
                                                                    sm.red_lo[pair][H]);
                wl = __ffs(__ballot_sync(0xffffffffu, kb == key)) - 1;
            }
            PairSlot *ps = &sm.slot[pair][parity][0];
#if FSR_P64_BRX
            // the winning row, made warp-uniform, then one indirect-branch pick on
            // every lane; the winning lane publishes its coefficient R[u*][v]
            const uint32_t klo = __shfl_sync(0xffffffffu, (uint32_t)kb, wl);
            const uint32_t rrw = 31u - ((klo >> 5) & 31u);
            const double2 cw = pick16_brx(R, p64_slot(H, TREE ? (int)bitrev5(rrw) : (int)rrw) & 15);
#endif
            if (lane == wl) {
                // only the winning lane extracts its coefficient R[u*][v] and publishes it
#if FSR_P64_BRX
                const double2 c = cw;
#else
                const uint32_t rr = 31u - (((uint32_t)kb >> 5) & 31u);
                const int bu = TREE ? (int)bitrev5(rr) : (int)rr;
                const double2 c = pick16(R, p64_slot(H, bu) & 15);
#endif
                ps[H].key = __longlong_as_double((long long)kb);
                ps[H].cre = c.x;
                ps[H].cim = c.y;
            }
            bar_pair(bar_id);
            // combine the halves: the larger key wins (keys are unique)
            const unsigned long long k0 = (unsigned long long)__double_as_longlong(ps[0].key);
            const unsigned long long k1 = (unsigned long long)__double_as_longlong(ps[1].key);
            const double c0r = ps[0].cre, c0i = ps[0].cim, c1r = ps[1].cre, c1i = ps[1].cim;
            const bool other = k1 > k0;
            const unsigned long long wkey = other ? k1 : k0;
            double2 c = make_double2(other ? c1r : c0r, other ? c1i : c0i);
            parity ^= 1;
            const uint32_t wlo = (uint32_t)wkey;
            const uint32_t wrr = 31u - ((wlo >> 5) & 31u), wlr = 31u - (wlo & 31u);
            const int wu = TREE ? (int)bitrev5(wrr) : (int)wrr;
            const int wv = TREE ? (int)bitrev5(wlr) : (int)wlr;
            if (H == 0 && sel_b && lane == 0) sel_b[it] = wu * 32 + wv;
            if (thr > 0.0 && __longlong_as_double((long long)wkey) < thr) break;
            gr = c.x * ginv;
            gi = c.y * ginv;
            p64_wbase<H>(wb, lane, wu, wv, P, ycv);
            // record every other selection per half; both halves flush together every 32
            if ((it & 1) == H && lane == 0) hist[(it >> 1) & 15] = SelEntry{gr, gi, wu, wv, {0, 0}};
            if ((it & 31) == 31) {
                __syncwarp();
                acc = p64_flush(sm, hist, 16, pm, pn, acc);
                __syncwarp();
            }
            done = it + 1;
        }
        {
            // flush the selections recorded since the last full flush
            const int rem = done & 31;
            const int mine = (rem + 1 - H) >> 1;  // entries of this half among the last rem
            __syncwarp();
            acc = p64_flush(sm, hist, mine, pm, pn, acc);
        }
        if (H == 1 && has_pix) sm.acc_x[pair][lane] = acc;
        bar_pair(bar_id);
        if (H == 0) {
            if (sel_b)
                for (int it = done + lane; it < a.iterations; it += 32) sel_b[it] = -1;
            if (lane == 0 && a.done) a.done[bid] = done;
            if (has_pix) {
                acc += sm.acc_x[pair][lane];
                const int m = lane / B, n = lane % B;
                const int64_t y = r0 + m, xx = c0 + n;
                if (y < a.H && xx < a.W)
                    a.out[y * a.out_pitch + xx] =
                        a.mask[y * a.mask_pitch + xx] ? a.px[y * a.px_pitch + xx] : (IO)acc;
            }
        }
        bar_pair(bar_id);  // buf is rewritten by the next block
    }
}

#ifndef FSR_P64_MAXREG
#define FSR_P64_MAXREG 128
#endif
template <int BPC, bool TREE, int ARGMAX, typename IO>
__global__ void __maxnreg__(FSR_P64_MAXREG) pair64_kernel(Pair64Args<IO> a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Pair64Smem<BPC> &sm = *reinterpret_cast<Pair64Smem<BPC> *>(smem_raw);
    if (threadIdx.x < 32) {
        double s, c;
        sincospi(2.0 * threadIdx.x / 32.0, &s, &c);
        sm.cs[threadIdx.x] = make_double2(c, s);
    }
    __syncthreads();
    // 32-row tables: align the block buffers to 16 KiB in the shared window (row
    // shift by masking); 48-row tables need no alignment
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&sm.buf[0][0]);
    const uint32_t pad = kP64Rows == 32 ? (0x4000u - (b0 & 0x3FFFu)) & 0x3FFFu : 0u;
    double2 *bufs = reinterpret_cast<double2 *>(reinterpret_cast<char *>(&sm.buf[0][0]) + pad);
    // warps p and p + BPC form block p's pair: same SMSP (warp % 4) when BPC % 4 == 0,
    // so the per-iteration pair barrier never waits on another scheduler's queue
    const int w = warp_id();
    const int pair = w % BPC;
    if (w >= BPC)
        p64_half<BPC, 1, TREE, ARGMAX, IO>(a, sm, bufs, pair);
    else
        p64_half<BPC, 0, TREE, ARGMAX, IO>(a, sm, bufs, pair);
}

}  // namespace fsr
