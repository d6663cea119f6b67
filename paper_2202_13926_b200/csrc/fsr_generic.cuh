// fsr_generic.cuh -- CTA-per-block FSR kernels for any support N <= 64.
//
// These are the exact-semantics kernels: residual and weight spectra live in
// shared memory, every thread owns a strided set of the N*N bins, and all
// loop arithmetic is strict IEEE (no FMA) so the fp64 instantiation
// reproduces the reference loop bit for bit (_kernels.py:62-126).  They
// serve (1) the array-level operator fsr_iterate_spectra, (2) the fp64
// validation image path for every N, (3) the fp64 re-run of blocks flagged by
// the fp32 near-tie guard, and (4) fp32 image reconstruction for supports
// without a register-resident specialisation.
#pragma once

#include "fsr_common.cuh"

namespace fsr {

constexpr int GEN_THREADS = 256;
constexpr int GEN_MAX_PIX = 16;  // ceil(B*B / GEN_THREADS) for B <= 64

struct Best {
    double obj;  // objective (exact copy, fp64 or widened fp32)
    int rank;
    int t;
};

__device__ __forceinline__ bool better(const Best &a, const Best &b) {
    return a.obj > b.obj || (a.obj == b.obj && a.rank < b.rank);
}

__device__ __forceinline__ Best warp_best(Best b) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        Best o;
        o.obj = __shfl_xor_sync(0xffffffffu, b.obj, off);
        o.rank = __shfl_xor_sync(0xffffffffu, b.rank, off);
        o.t = __shfl_xor_sync(0xffffffffu, b.t, off);
        if (better(o, b)) b = o;
    }
    return b;
}

// Block-wide argmax (all threads receive the result).  scratch: >= 32 Best.
__device__ __forceinline__ Best block_best(Best b, Best *scratch) {
    b = warp_best(b);
    const int nw = blockDim.x >> 5;
    if (lane_id() == 0) scratch[warp_id()] = b;
    __syncthreads();
    if (warp_id() == 0) {
        Best c = lane_id() < nw ? scratch[lane_id()] : Best{-HUGE_VAL, 0x7fffffff, 0};
        c = warp_best(c);
        if (lane_id() == 0) scratch[32] = c;
    }
    __syncthreads();
    Best r = scratch[32];
    return r;
}

__device__ __forceinline__ int block_sum(int v, int *scratch) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int nw = blockDim.x >> 5;
    if (lane_id() == 0) scratch[warp_id()] = v;
    __syncthreads();
    int s = 0;
    for (int i = 0; i < nw; ++i) s += scratch[i];
    __syncthreads();
    return s;
}

template <typename Real>
struct LoopShared {
    Best red[33];
    int isum[32];
    cpx<Real> gp;
    int u, v, t, stop;
    double energy;
};

// One block's greedy loop on spectra already in shared memory.
// on_select(it, u, v, gp) is called by every thread after each selection.
// Returns the number of model updates applied; *pending is set when the last
// update has not yet been applied to sR (the caller applies it if needed).
template <typename Real, typename OnSelect>
__device__ int generic_loop(cpx<Real> *sR, const cpx<Real> *sW, const Real *wf, int N,
                            int iterations, Real gamma, bool tree, Real thr, bool want_ties,
                            LoopShared<Real> &sh, int32_t *sel_out, double *obj_out,
                            uint8_t *ties_out, OnSelect on_select) {
    const int n = N * N;
    const Real w00 = sW[0].re;
    bool have_prev = false;
    cpx<Real> gp = {0, 0};
    int pu = 0, pv = 0;
    int done = 0;
    for (int it = 0; it < iterations; ++it) {
        Best mine = {-HUGE_VAL, 0x7fffffff, 0};
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            cpx<Real> r = sR[t];
            if (have_prev) {
                int k = t / N, l = t - k * N;
                int i = k - pu; i += (i < 0) ? N : 0;
                int j = l - pv; j += (j < 0) ? N : 0;
                cpx<Real> tt = scmul(gp, sW[i * N + j]);
                r.re = ssub(r.re, tt.re);
                r.im = ssub(r.im, tt.im);
                sR[t] = r;
            }
            Real o = smul(wf[t], sadd(smul(r.re, r.re), smul(r.im, r.im)));
            Best cand = {(double)o, tie_rank(t, tree), t};
            if (better(cand, mine)) mine = cand;
        }
        Best best = block_best(mine, sh.red);  // contains __syncthreads (sR updates visible)
        int ties = 0;
        if (want_ties) {
            int cnt = 0;
            for (int t = threadIdx.x; t < n; t += blockDim.x) {
                cpx<Real> r = sR[t];
                Real o = smul(wf[t], sadd(smul(r.re, r.re), smul(r.im, r.im)));
                cnt += ((double)o == best.obj);
            }
            ties = block_sum(cnt, sh.isum);
        }
        if (threadIdx.x == 0) {
            if (sel_out) sel_out[it] = best.t;
            if (obj_out) obj_out[it] = best.obj;
            if (ties_out) ties_out[it] = ties > 1 ? 1 : 0;
            int stop = (thr > Real(0) && (Real)best.obj < thr);
            sh.stop = stop;
            if (!stop) {
                int u = best.t / N, v = best.t - (best.t / N) * N;
                cpx<Real> c = sR[best.t];
                // gp = gamma * complex(c.re / w00, c.im / w00)  (real promoted to complex)
                cpx<Real> q = {c.re / w00, c.im / w00};
                cpx<Real> g = {gamma, Real(0)};
                sh.gp = scmul(g, q);
                sh.u = u;
                sh.v = v;
                sh.t = best.t;
            }
        }
        __syncthreads();
        if (sh.stop) break;
        gp = sh.gp;
        pu = sh.u;
        pv = sh.v;
        have_prev = true;
        on_select(it, pu, pv, gp);
        done = it + 1;
        __syncthreads();  // sh reused next iteration
    }
    if (have_prev && sh.stop == 0 && done == iterations) {
        // apply the last selection's residual update (needed by the operator)
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            int k = t / N, l = t - k * N;
            int i = k - pu; i += (i < 0) ? N : 0;
            int j = l - pv; j += (j < 0) ? N : 0;
            cpx<Real> r = sR[t];
            cpx<Real> tt = scmul(gp, sW[i * N + j]);
            r.re = ssub(r.re, tt.re);
            r.im = ssub(r.im, tt.im);
            sR[t] = r;
        }
    }
    __syncthreads();
    return done;
}

// ---------------------------------------------------------------------------
// Array-level operator: reconstruct_batch (_kernels.py:129-149), fp64 strict.
struct IterateArgs {
    int64_t count;
    int N, iterations, tree;
    double gamma;
    cpx<double> *R;        // [count, N*N] in/out
    cpx<double> *G;        // [count, N*N] in/out (accumulated)
    const cpx<double> *W;  // [count, N*N]
    const double *wf;      // [N*N]
    const double *thr;     // [count] or null
    int32_t *sel;          // [count, iterations] or null
    double *obj;
    uint8_t *ties;
    int32_t *done;         // [count] or null
};

#ifdef FSR_ABI_TU  // non-template kernel: defined in fsr_abi.cu's translation unit only
__global__ void __launch_bounds__(GEN_THREADS) iterate_spectra_kernel(IterateArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.N * a.N;
    cpx<double> *sR = reinterpret_cast<cpx<double> *>(smem_raw);
    cpx<double> *sW = sR + n;
    __shared__ LoopShared<double> sh;
    for (int64_t b = blockIdx.x; b < a.count; b += gridDim.x) {
        const cpx<double> *Wb = a.W + b * n;
        if (!(Wb[0].re > 0.0)) {  // _kernels.py:144-145: spectra[b,0,0].real <= 0 -> skip
            if (threadIdx.x == 0 && a.done) a.done[b] = 0;
            continue;
        }
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            sR[t] = a.R[b * n + t];
            sW[t] = Wb[t];
        }
        __syncthreads();
        cpx<double> *Gb = a.G + b * n;
        const int64_t it_stride = a.iterations > 0 ? a.iterations : 1;
        const double nn = (double)n;
        int done = generic_loop<double>(
            sR, sW, a.wf, a.N, a.iterations, a.gamma, a.tree != 0, a.thr ? a.thr[b] : 0.0,
            a.ties != nullptr, sh, a.sel ? a.sel + b * it_stride : nullptr,
            a.obj ? a.obj + b * it_stride : nullptr, a.ties ? a.ties + b * it_stride : nullptr,
            [&](int, int u, int v, cpx<double> gp) {
                if (threadIdx.x == 0) {
                    // model[u, v] += gp * n  (int promoted to complex)
                    cpx<double> add = scmul(gp, cpx<double>{nn, 0.0});
                    cpx<double> m = Gb[u * a.N + v];
                    m.re = sadd(m.re, add.re);
                    m.im = sadd(m.im, add.im);
                    Gb[u * a.N + v] = m;
                }
            });
        for (int t = threadIdx.x; t < n; t += blockDim.x) a.R[b * n + t] = sR[t];
        if (threadIdx.x == 0 && a.done) a.done[b] = done;
        __syncthreads();
    }
}
#endif

// ---------------------------------------------------------------------------
// Image path, CTA per block: gather -> w = decay*mask -> packed 2-D DFT ->
// loop -> direct synthesis of the B x B target pixels -> merge -> stitch.
template <typename Real, typename IO>
struct ImageArgs {
    const IO *px;
    int64_t px_pitch;
    const uint8_t *mask;
    int64_t mask_pitch;
    IO *out;
    int64_t out_pitch;
    int64_t H, W;
    int B, L, N, iterations;
    int64_t bcols;       // ceil(W / B)
    int64_t first;       // first block id (row0 * bcols)
    int64_t nblocks;     // blocks in this launch
    const int32_t *list; // optional explicit block-id list (length nblocks)
    const unsigned int *list_count;  // if set, the list length is read on the device
    Real gamma;
    int tree, early_stop;
    Tables<Real> tab;
    int32_t *sel;        // [total blocks, iterations] or null (indexed by block id)
    int32_t *done;       // [total blocks] or null
    unsigned int *empty_count;
    int32_t *empty_list;  // block ids of empty-support blocks (capacity nblocks) or null
};

template <typename Real, typename IO>
__global__ void __launch_bounds__(GEN_THREADS) image_generic_kernel(ImageArgs<Real, IO> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.N, n = N * N;
    cpx<Real> *sR = reinterpret_cast<cpx<Real> *>(smem_raw);
    cpx<Real> *sW = sR + n;
    __shared__ LoopShared<Real> sh;
    const int64_t nblocks = a.list_count ? (int64_t)*a.list_count : a.nblocks;
    for (int64_t i = blockIdx.x; i < nblocks; i += gridDim.x) {
        const int64_t bid = a.list ? a.list[i] : a.first + i;
        const int64_t brow = bid / a.bcols, bcol = bid - brow * a.bcols;
        const int64_t r0 = brow * a.B, c0 = bcol * a.B;
        const int64_t wr0 = r0 - a.L, wc0 = c0 - a.L;
        const int h = (int)min((int64_t)a.B, a.H - r0), w = (int)min((int64_t)a.B, a.W - c0);
        // gather (sampling.py:93-107: outside the image = unknown) + weights
        double e_local = 0.0;
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            int k = t / N, l = t - k * N;
            int64_t y = wr0 + k, x = wc0 + l;
            Real f = 0, wt = 0;
            if (y >= 0 && y < a.H && x >= 0 && x < a.W && a.mask[y * a.mask_pitch + x]) {
                f = (Real)a.px[y * a.px_pitch + x];
                wt = a.tab.decay[t];
            }
            sR[t] = {f * wt, wt};  // packed z = f*w + i*w
            e_local += (double)(f * f * wt);
        }
        if (a.early_stop) {
            // thresholds = EARLY_STOP_RELATIVE * sum(signal^2 * w) (reconstruction.py:262-266)
            double e = e_local;
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
            if (lane_id() == 0) sh.red[warp_id()].obj = e;
            __syncthreads();
            if (threadIdx.x == 0) {
                double s = 0;
                for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += sh.red[q].obj;
                sh.energy = s;
            }
        }
        __syncthreads();
        // row DFT: T[k][v] = sum_l z[k][l] e^{-2 pi i l v / N}  -> sW
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            int k = t / N, v = t - k * N;
            Real ar = 0, ai = 0;
            int idx = 0;
            for (int l = 0; l < N; ++l) {
                cpx<Real> z = sR[k * N + l];
                Real c = a.tab.cs[2 * idx], s = a.tab.cs[2 * idx + 1];
                ar += z.re * c + z.im * s;
                ai += z.im * c - z.re * s;
                idx += v; idx -= (idx >= N) ? N : 0;
            }
            sW[t] = {ar, ai};
        }
        __syncthreads();
        // column DFT: Z[u][v] = sum_k T[k][v] e^{-2 pi i k u / N}  -> sR
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            int u = t / N, v = t - u * N;
            Real ar = 0, ai = 0;
            int idx = 0;
            for (int k = 0; k < N; ++k) {
                cpx<Real> z = sW[k * N + v];
                Real c = a.tab.cs[2 * idx], s = a.tab.cs[2 * idx + 1];
                ar += z.re * c + z.im * s;
                ai += z.im * c - z.re * s;
                idx += u; idx -= (idx >= N) ? N : 0;
            }
            sR[t] = {ar, ai};
        }
        __syncthreads();
        // split the packed transform: R = (Z[t] + conj Z[-t]) / 2, W = (Z[t] - conj Z[-t]) / 2i.
        // Both come out exactly Hermitian (R[-t] == conj R[t] bitwise).
        {
            cpx<Real> rr[(64 * 64 + GEN_THREADS - 1) / GEN_THREADS], ww[(64 * 64 + GEN_THREADS - 1) / GEN_THREADS];
            int q = 0;
            for (int t = threadIdx.x; t < n; t += blockDim.x, ++q) {
                int u = t / N, v = t - u * N;
                int mt = ((N - u) % N) * N + (N - v) % N;
                cpx<Real> z = sR[t], zm = sR[mt];
                rr[q] = {(z.re + zm.re) * Real(0.5), (z.im - zm.im) * Real(0.5)};
                ww[q] = {(z.im + zm.im) * Real(0.5), (zm.re - z.re) * Real(0.5)};
            }
            __syncthreads();
            q = 0;
            for (int t = threadIdx.x; t < n; t += blockDim.x, ++q) {
                sR[t] = rr[q];
                sW[t] = ww[q];
            }
        }
        __syncthreads();
        const bool empty = !(sW[0].re > Real(0));
        int32_t *sel_b = a.sel ? a.sel + bid * (int64_t)max(a.iterations, 1) : nullptr;
        if (empty) {
            if (threadIdx.x == 0) {
                unsigned slot = atomicAdd(a.empty_count, 1u);
                if (a.empty_list) a.empty_list[slot] = (int32_t)bid;
                if (a.done) a.done[bid] = 0;
            }
            if (sel_b)
                for (int it = threadIdx.x; it < a.iterations; it += blockDim.x) sel_b[it] = -1;
            __syncthreads();
            continue;
        }
        // pixel accumulators for direct synthesis: g = sum Re(gp e^{+2 pi i (u m + v n)/N})
        Real acc[GEN_MAX_PIX];
#pragma unroll
        for (int q = 0; q < GEN_MAX_PIX; ++q) acc[q] = 0;
        const int npix = h * w;
        const Real thr = a.early_stop ? (Real)(1e-12 * sh.energy) : Real(0);
        const Real *cs = a.tab.cs;
        const int L = a.L;
        int done = generic_loop<Real>(
            sR, sW, a.tab.wf, N, a.iterations, a.gamma, a.tree != 0, thr, false, sh, sel_b,
            nullptr, nullptr, [&](int, int u, int v, cpx<Real> gp) {
#pragma unroll
                for (int q = 0; q < GEN_MAX_PIX; ++q) {
                    int p = threadIdx.x + q * blockDim.x;
                    if (p < npix) {
                        int m = L + p / w, nn = L + p % w;
                        int idx = (u * m + v * nn) % N;
                        acc[q] += gp.re * cs[2 * idx] - gp.im * cs[2 * idx + 1];
                    }
                }
            });
        if (sel_b)
            for (int it = done + threadIdx.x; it < a.iterations; it += blockDim.x) sel_b[it] = -1;
        if (threadIdx.x == 0 && a.done) a.done[bid] = done;
        // merge + stitch: known pixels copied, unknown from the model (reconstruction.py:270-280)
#pragma unroll
        for (int q = 0; q < GEN_MAX_PIX; ++q) {
            int p = threadIdx.x + q * blockDim.x;
            if (p < npix) {
                int m = p / w, nn = p % w;
                int64_t y = r0 + m, x = c0 + nn;
                a.out[y * a.out_pitch + x] =
                    a.mask[y * a.mask_pitch + x] ? a.px[y * a.px_pitch + x] : (IO)acc[q];
            }
        }
        __syncthreads();
    }
}

// Empty-support fallback (reconstruction.py:236-237, 272-275).
//
// mean_partial_kernel: per-CTA (sum of known pixels, count of known pixels)
// over rows [0, H), each thread striding over the pixels in a fixed order and
// the CTA combining its threads by a fixed tree -- so, for a fixed grid, the
// partials (and the mean fill_empty_kernel forms from them) are bitwise
// reproducible.  A no-op unless some block of the call was empty.
template <typename IO>
__global__ void __launch_bounds__(256) mean_partial_kernel(const IO *px, int64_t px_pitch,
                                                           const uint8_t *mask, int64_t mask_pitch,
                                                           int64_t H, int64_t W,
                                                           const unsigned int *empty_count,
                                                           double2 *partials) {
    if (*empty_count == 0) return;
    __shared__ double2 ws[8];
    double s = 0.0, c = 0.0;
    const int64_t total = H * W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = i / W, x = i - y * W;
        if (mask[y * mask_pitch + x]) {
            s += (double)px[y * px_pitch + x];
            c += 1.0;
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        s += __shfl_down_sync(0xffffffffu, s, off);
        c += __shfl_down_sync(0xffffffffu, c, off);
    }
    if (lane_id() == 0) ws[warp_id()] = make_double2(s, c);
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 t = ws[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            t.x += ws[w].x;
            t.y += ws[w].y;
        }
        partials[blockIdx.x] = t;
    }
}

// fill_empty_kernel: the listed blocks get `fill_value`, or (partials != null)
// sum/count of the nparts partials, summed by one warp in a fixed order (every
// CTA forms the same value).  status = 2 if a block was empty but the image
// holds no known sample ("no known samples", reconstruction.py:273-274).
template <typename IO>
__global__ void fill_empty_kernel(IO *out, int64_t out_pitch, int64_t H, int64_t W, int B,
                                  int64_t bcols, const int32_t *list, const unsigned int *count,
                                  const double2 *partials, int nparts, double fill_value,
                                  int *status) {
    const int n = (int)*count;
    if (n == 0) return;
    __shared__ double fill_s;
    if (threadIdx.x < 32) {
        double fill = fill_value;
        if (partials) {
            double S = 0.0, C = 0.0;
            for (int i = threadIdx.x; i < nparts; i += 32) {
                S += partials[i].x;
                C += partials[i].y;
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                S += __shfl_xor_sync(0xffffffffu, S, off);
                C += __shfl_xor_sync(0xffffffffu, C, off);
            }
            if (C == 0.0 && blockIdx.x == 0 && threadIdx.x == 0) *status = 2;
            fill = C > 0.0 ? S / C : 0.0;
        }
        if (threadIdx.x == 0) fill_s = fill;
    }
    __syncthreads();
    const double fill = fill_s;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int64_t bid = list[i];
        const int64_t r0 = (bid / bcols) * B, c0 = (bid % bcols) * B;
        const int h = (int)min((int64_t)B, H - r0), w = (int)min((int64_t)B, W - c0);
        for (int q = threadIdx.x; q < h * w; q += blockDim.x)
            out[(r0 + q / w) * out_pitch + c0 + q % w] = (IO)fill;
    }
}

}  // namespace fsr
