// fsr_common.cuh -- shared device types and helpers for the FSR kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fsr {

template <typename Real>
struct cpx {
    Real re, im;
};

// Strict IEEE scalar ops: no FMA contraction, round-to-nearest.  The fp64
// validation path uses these so that its loop reproduces numba's bits
// (reference _kernels.py:62-126 is compiled without fast-math or contraction).
__device__ __forceinline__ double smul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ssub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float smul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float sadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float ssub(float a, float b) { return __fsub_rn(a, b); }

// numba's complex128 multiply: (a+bi)(c+di) = (ac-bd) + (ad+bc)i, strict.
template <typename Real>
__device__ __forceinline__ cpx<Real> scmul(cpx<Real> x, cpx<Real> y) {
    Real ac = smul(x.re, y.re), bd = smul(x.im, y.im);
    Real ad = smul(x.re, y.im), bc = smul(x.im, y.re);
    return {ssub(ac, bd), sadd(ad, bc)};
}

// Tie rank of flat bin t (smaller wins among equal objectives).
//  linear (_kernels.py:52-59): the first maximum, rank = t.
//  tree   (_kernels.py:12-49): groups of 32 consecutive records, strict '>'
//         lock-step passes with offsets 16..1; the winner among maxima is the
//         lexicographic minimum of (bitrev5(t >> 5), bitrev5(t & 31)).
__host__ __device__ __forceinline__ uint32_t bitrev5(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __brev(x) >> 27;  // BREV + SHF
#else
    return ((x & 1u) << 4) | ((x & 2u) << 2) | (x & 4u) | ((x & 8u) >> 2) | ((x & 16u) >> 4);
#endif
}
__host__ __device__ __forceinline__ int tie_rank(int t, bool tree) {
    return tree ? (int)((bitrev5((uint32_t)t >> 5) << 5) | bitrev5((uint32_t)t & 31u)) : t;
}

// Device-side constant tables for one (N, rho): decay grid rho^dist
// (weights.py:18-27), frequency prior w_f (weights.py:40-56) and the DFT
// twiddles cos/sin(2*pi*j/N).
template <typename Real>
struct Tables {
    const Real *decay;  // [N*N]
    const Real *wf;     // [N*N]
    const Real *cs;     // [2*N] interleaved cos, sin of 2*pi*j/N
};

// sqrt for the guard's scale term (one MUFU; ~2 ulp is immaterial there).
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace fsr
