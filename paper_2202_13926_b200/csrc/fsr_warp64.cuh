// fsr_warp64.cuh -- production FSR kernel for support N = 32 in fp64, ONE warp
// per target block (no per-iteration barrier), the residual spectrum
// register-resident (lane v owns spectral column v, R[u][v] for all 32 rows:
// 128 registers).
//
// Compared with the warp-pair kernel (fsr_pair64.cuh) this trades occupancy
// (about 10 warps/SM at ~190 registers) for the absence of the per-iteration
// pair barrier and half the per-iteration argmax/extract overhead per bin.
// Per block:
//   gather     lane = window column, coalesced rows, mask-gated rho^d weights,
//              packed z = f w + i w written to an XOR-swizzled 16 KiB tile
//   2-D FFT    32-point in-register FFT along rows (lane = row), then along
//              columns (lane = column), both in place in the tile
//   split      conjugate pairs (u, -u): R (registers) and W (row-major in the
//              same tile), exactly Hermitian
//   loop       per iteration one fused pass over 32 rows: W[(u-pu)][(v-pv)]
//              (LDS.128, row shift by a 2-op mask), residual update (4 DFMA),
//              objective (3 DP), packed 64-bit key, 4 running maxima; then the
//              lane-rank bits, one warp u64 argmax (shfl butterfly / redux /
//              shared-memory tree), extraction of R[u*] from the winning lane
//              and the coefficient for the next pass.
//   synthesis  lanes p < B*B accumulate the target pixels directly.
#pragma once

#include "fsr_common.cuh"
#include "fsr_fft.cuh"
#include "fsr_pair64.cuh"

namespace fsr {

#ifndef FSR_W64_MAXREG
#define FSR_W64_MAXREG 200
#endif

template <int WARPS>
struct Warp64Smem {
    double2 buf[WARPS][32 * 32];  // 16 KiB per block; aligned to 16 KiB at run time
    double2 align_pad[1024];
    unsigned int red_hi[WARPS][32];
    unsigned int red_lo[WARPS][32];
    double2 cs[32];
};

// R[u] for a warp-uniform dynamic u in [0, 32).
__device__ __forceinline__ double2 pick32d(const cpx<double> (&R)[32], int u) {
    double2 c;
    switch (u) {
#define FSR_PICK(k) \
    case k: c = make_double2(R[k].re, R[k].im); break;
        FSR_PICK(0) FSR_PICK(1) FSR_PICK(2) FSR_PICK(3) FSR_PICK(4) FSR_PICK(5) FSR_PICK(6)
        FSR_PICK(7) FSR_PICK(8) FSR_PICK(9) FSR_PICK(10) FSR_PICK(11) FSR_PICK(12) FSR_PICK(13)
        FSR_PICK(14) FSR_PICK(15) FSR_PICK(16) FSR_PICK(17) FSR_PICK(18) FSR_PICK(19)
        FSR_PICK(20) FSR_PICK(21) FSR_PICK(22) FSR_PICK(23) FSR_PICK(24) FSR_PICK(25)
        FSR_PICK(26) FSR_PICK(27) FSR_PICK(28) FSR_PICK(29) FSR_PICK(30)
        default: c = make_double2(R[31].re, R[31].im); break;
#undef FSR_PICK
    }
    return c;
}

// Fused residual update + objective + packed-key max over the 32 rows.
template <bool TREE, bool UPDATE>
__device__ __forceinline__ unsigned long long w64_pass(cpx<double> (&R)[32], const double (&wfr)[17],
                                                       uint32_t P, uint32_t ycv, double gr,
                                                       double gi, uint32_t cmask) {
    unsigned long long best[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        double re = R[u].re, im = R[u].im;
        if (UPDATE) {
            const uint32_t addr = ((P + ((uint32_t)u << 9)) & 0x3E00u) | ycv;
            double2 w;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y) : "r"(addr));
            re = fma(-gr, w.x, re);
            re = fma(gi, w.y, re);
            im = fma(-gr, w.y, im);
            im = fma(-gi, w.x, im);
            R[u].re = re;
            R[u].im = im;
        }
        const double mag = fma(re, re, im * im);
        const double o = mag * wfr[p64_fold(u)];
        const uint32_t rk = TREE ? brev5c(u) : (uint32_t)u;
        uint32_t lo;
        asm("lop3.b32 %0, %1, %2, %3, 0xD8;"
            : "=r"(lo) : "r"((uint32_t)__double2loint(o)), "r"(((31u - rk) << 5) | 31u), "r"(cmask));
        const unsigned long long k =
            ((unsigned long long)(uint32_t)__double2hiint(o) << 32) | (unsigned long long)lo;
        best[u & 3] = u64max(best[u & 3], k);
    }
    return u64max(u64max(best[0], best[1]), u64max(best[2], best[3]));
}

template <int WARPS, bool TREE, int ARGMAX, typename IO>
__global__ void __maxnreg__(FSR_W64_MAXREG) warp64_kernel(Pair64Args<IO> a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Warp64Smem<WARPS> &sm = *reinterpret_cast<Warp64Smem<WARPS> *>(smem_raw);
    if (threadIdx.x < 32) {
        double s, c;
        sincospi(2.0 * threadIdx.x / 32.0, &s, &c);
        sm.cs[threadIdx.x] = make_double2(c, s);
    }
    __syncthreads();
    const int lane = lane_id(), wid = warp_id();
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&sm.buf[0][0]);
    const uint32_t pad = (0x4000u - (b0 & 0x3FFFu)) & 0x3FFFu;
    double2 *buf = reinterpret_cast<double2 *>(reinterpret_cast<char *>(&sm.buf[0][0]) + pad) +
                   wid * 1024;
    const uint32_t wb = (uint32_t)__cvta_generic_to_shared(buf);  // 16 KiB aligned
    const uint32_t lrank = TREE ? bitrev5(lane) : (uint32_t)lane;
    double wfr[17];
#pragma unroll
    for (int f = 0; f <= 16; ++f) wfr[f] = a.wf[f * 32 + lane];

    const int64_t nblocks = a.list_count ? (int64_t)*a.list_count : a.nblocks;
    const int64_t stride = (int64_t)gridDim.x * WARPS;
    for (int64_t bi = (int64_t)blockIdx.x * WARPS + wid; bi < nblocks; bi += stride) {
        const int64_t bid = a.list ? (int64_t)a.list[bi] : a.first + bi;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const int64_t wr0 = r0 - a.L, x = c0 - a.L + lane;
        const bool xin = x >= 0 && x < a.W;
        double energy = 0.0;
        // ---- gather (lane = window column)
#pragma unroll 4
        for (int k = 0; k < 32; ++k) {
            const int64_t y = wr0 + k;
            double f = 0.0, w = 0.0;
            if (xin && y >= 0 && y < a.H && a.mask[y * a.mask_pitch + x]) {
                f = load_px(a.px + y * a.px_pitch + x);
                w = a.decay[k * 32 + lane];
            }
            buf[tidx(k, lane)] = make_double2(f * w, w);
            energy = fma(f * f, w, energy);
        }
        __syncwarp();
        cpx<double> R[32];
        // ---- row FFTs (lane = row), in place
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            const double2 z = buf[tidx(lane, l)];
            R[l] = {z.x, z.y};
        }
        fft32(R);
#pragma unroll
        for (int l = 0; l < 32; ++l) buf[tidx(lane, l)] = make_double2(R[l].re, R[l].im);
        __syncwarp();
        // ---- column FFTs (lane = column), in place
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double2 z = buf[tidx(k, lane)];
            R[k] = {z.x, z.y};
        }
        fft32(R);
#pragma unroll
        for (int u = 0; u < 32; ++u) buf[tidx(u, lane)] = make_double2(R[u].re, R[u].im);
        __syncwarp();
        // ---- split conjugate pairs (u, -u): R in registers, W row-major in buf
        const int mv = (32 - lane) & 31;
#pragma unroll
        for (int u = 0; u <= 16; ++u) {
            const int nu = (32 - u) & 31;
            const double2 zp = buf[tidx(u, lane)], zpm = buf[tidx(nu, mv)];
            const double2 zn = buf[tidx(nu, lane)], znm = buf[tidx(u, mv)];
            R[u] = {(zp.x + zpm.x) * 0.5, (zp.y - zpm.y) * 0.5};
            const double2 wp = make_double2((zp.y + zpm.y) * 0.5, (zpm.x - zp.x) * 0.5);
            double2 wn = wp;
            if (nu != u) {
                R[nu] = {(zn.x + znm.x) * 0.5, (zn.y - znm.y) * 0.5};
                wn = make_double2((zn.y + znm.y) * 0.5, (znm.x - zn.x) * 0.5);
            }
            __syncwarp();
            buf[u * 32 + lane] = wp;
            if (nu != u) buf[nu * 32 + lane] = wn;
            __syncwarp();
        }
        const double w00 = __shfl_sync(0xffffffffu, lane == 0 ? buf[0].x : 0.0, 0);
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
        uint32_t P = 0, ycv = wb;
        const uint32_t cmask = 0x3FFu;
        int done = 0;
        for (int it = 0; it < a.iterations; ++it) {
            unsigned long long kb = it == 0 ? w64_pass<TREE, false>(R, wfr, P, ycv, gr, gi, cmask)
                                            : w64_pass<TREE, true>(R, wfr, P, ycv, gr, gi, cmask);
            kb ^= lrank;
            const unsigned long long key = p64_warp_max<ARGMAX>(kb, sm.red_hi[wid], sm.red_lo[wid]);
            const uint32_t klo = (uint32_t)key;
            const uint32_t rr = 31u - ((klo >> 5) & 31u), lr = 31u - (klo & 31u);
            const int bu = TREE ? (int)bitrev5(rr) : (int)rr;
            const int bv = TREE ? (int)bitrev5(lr) : (int)lr;
            if (sel_b && lane == 0) sel_b[it] = bu * 32 + bv;
            if (thr > 0.0 && __longlong_as_double((long long)key) < thr) break;
            double2 c = pick32d(R, bu);
            c.x = __shfl_sync(0xffffffffu, c.x, bv);
            c.y = __shfl_sync(0xffffffffu, c.y, bv);
            gr = c.x * ginv;
            gi = c.y * ginv;
            P = (uint32_t)((32 - bu) & 31) << 9;
            ycv = wb | ((uint32_t)((lane - bv) & 31) << 4);
            if (has_pix) {
                const double2 e = sm.cs[(bu * pm + bv * pn) & 31];
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
