// fsr_spatial.cuh -- the FFT-free spatial-domain oracle on the GPU (SURVEY §8f
// row 4), an independent cross-check of the frequency-domain engine.
//
// Restates the reference's direct-summation oracle (pkg/src/fsrkit/oracle.py:
// 25-132) for supports S <= 16: every iteration projects the weighted
// residual onto all S^2 complex exponential basis images by explicit
// summation (no FFT, no residual spectrum, no shifted weight spectrum),
// selects the first maximum of wf * |proj|^2 in flat index order
// (oracle.py:81-82, np.argmax), counts the objectives within 1e-9 of it as a
// tie (oracle.py:83, TIE_RELATIVE), adds gamma * proj[t] / W00 times the basis
// image to the spatial model and recomputes the residual, its weighted copy
// and its weighted energy from scratch (oracle.py:89-98).  fp64 throughout.
//
// One CTA of 256 threads per block; thread t owns basis image / frequency t
// for the projection and pixel t for the model update.  The basis phase of
// (t, pixel) is exp(2 pi i ((k m + l n) mod S) / S) from a twiddle table --
// the reference evaluates exp of the unreduced angle, a difference in the last
// bits that the reference's own acceptance test absorbs (objectives to 1e-9
// relative, test_acceptance.py:32-91).
#pragma once

#include "fsr_common.cuh"

namespace fsr {

struct SpatialArgs {
    const double *signal;   // [count][S*S]
    const uint8_t *mask;    // [count][S*S]
    const double *spatial;  // [count][S*S] spatial weights w (decay * mask)
    const double *wf;       // [S*S] frequency prior
    double *out;            // [count][S*S] merged output (mask ? signal : Re model)
    double *obj;            // [count][I]
    int32_t *sel;           // [count][I] flat frequency index u*S + v
    uint8_t *ties;          // [count][I]
    double *energy;         // [count][I + 1] weighted residual energy
    int64_t count;
    int S, iterations;
    double gamma;
};

constexpr int SP_THREADS = 256;

// block-wide sum of one double per thread (fixed tree order)
__device__ __forceinline__ double sp_block_sum(double v, double *scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < SP_THREADS / 32; ++w) s += scratch[w];
    return s;
}

__global__ void __launch_bounds__(SP_THREADS) spatial_oracle_kernel(SpatialArgs a) {
    __shared__ double2 rw[256];     // weighted residual (signal - model) * w
    __shared__ double2 model[256];
    __shared__ double2 tw[16];      // exp(2 pi i j / S)
    __shared__ double scratch[SP_THREADS / 32];
    __shared__ double best_v[SP_THREADS / 32];
    __shared__ int best_i[SP_THREADS / 32];
    __shared__ double2 pick;        // proj[t*]
    __shared__ int pick_t;
    const int S = a.S, n = S * S, t = threadIdx.x;
    const int lane = t & 31, wid = t >> 5;
    const int64_t b = blockIdx.x;
    const double *sig = a.signal + b * n;
    const double *w = a.spatial + b * n;
    if (t < S) {
        double sn, cs;
        sincospi(2.0 * t / S, &sn, &cs);
        tw[t] = make_double2(cs, sn);
    }
    const double sg = t < n ? sig[t] : 0.0, wt = t < n ? w[t] : 0.0;
    if (t < n) {
        model[t] = make_double2(0.0, 0.0);
        rw[t] = make_double2(sg * wt, 0.0);
    }
    const double w00 = sp_block_sum(wt, scratch);
    double e0 = sp_block_sum(t < n ? sg * sg * wt : 0.0, scratch);
    if (t == 0) a.energy[b * (a.iterations + 1)] = e0;
    const int k = t / S, l = t - (t / S) * S;  // frequency (k, l) of thread t
    const double wft = t < n ? a.wf[t] : 0.0;
    for (int it = 0; it < a.iterations; ++it) {
        __syncthreads();
        // projection onto basis image t by direct summation: sum conj(phi_t) rw
        double pr = 0.0, pi = 0.0;
        if (t < n) {
            for (int m = 0; m < S; ++m)
                for (int q = 0; q < S; ++q) {
                    const double2 e = tw[(k * m + l * q) % S];
                    const double2 r = rw[m * S + q];
                    pr += e.x * r.x + e.y * r.y;  // (cos - i sin)(re + i im)
                    pi += e.x * r.y - e.y * r.x;
                }
        }
        // objective (oracle.py:81) and the first maximum in flat order
        const double o = t < n ? __dmul_rn(wft, __dadd_rn(__dmul_rn(pr, pr), __dmul_rn(pi, pi))) : -1.0;
        double bv = o;
        int bi = t;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            best_v[wid] = bv;
            best_i[wid] = bi;
        }
        __syncthreads();
        double best = best_v[0];
        int tb = best_i[0];
        for (int w2 = 1; w2 < SP_THREADS / 32; ++w2)
            if (best_v[w2] > best || (best_v[w2] == best && best_i[w2] < tb)) {
                best = best_v[w2];
                tb = best_i[w2];
            }
        if (t == tb) {
            pick = make_double2(pr, pi);
            pick_t = t;
        }
        // tie: more than one objective within 1e-9 of the maximum (oracle.py:83)
        const double near = (t < n && o >= best * (1.0 - 1e-9)) ? 1.0 : 0.0;
        const double cnt = sp_block_sum(near, scratch);  // also orders pick/pick_t
        const int ts = pick_t;
        const double2 pj = pick;
        if (t == 0) {
            a.obj[b * a.iterations + it] = best;
            a.sel[b * a.iterations + it] = ts;
            a.ties[b * a.iterations + it] = best > 0.0 ? (uint8_t)(cnt > 1.0) : (uint8_t)1;
        }
        // model += (gamma p) phi_t ; residual, weighted residual, energy recomputed
        const double gpr = a.gamma * (pj.x / w00), gpi = a.gamma * (pj.y / w00);
        const int ku = ts / S, lv = ts - (ts / S) * S;
        double en = 0.0;
        if (t < n) {
            const int m = t / S, q = t - (t / S) * S;
            const double2 e = tw[(ku * m + lv * q) % S];  // phi_ts(m, q)
            double2 md = model[t];
            md.x += gpr * e.x - gpi * e.y;
            md.y += gpr * e.y + gpi * e.x;
            model[t] = md;
            const double rr = sg - md.x, ri = -md.y;
            rw[t] = make_double2(rr * wt, ri * wt);
            en = (rr * rr + ri * ri) * wt;
        }
        en = sp_block_sum(en, scratch);
        if (t == 0) a.energy[b * (a.iterations + 1) + it + 1] = en;
    }
    if (t < n) {
        const uint8_t mk = a.mask[b * n + t];
        a.out[b * n + t] = mk ? sg : model[t].x;
    }
}

}  // namespace fsr
