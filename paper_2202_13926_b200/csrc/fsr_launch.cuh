// fsr_launch.cuh -- launchers of the image kernels, one translation unit per
// (kernel family, pixel type, argmax variant) so the library builds in
// parallel (see Makefile: k_*.cu are compiled once per variant with -D).
//
// Every launcher sizes a persistent grid from the occupancy API (a multiple of
// the SM count, one wave), launches on `st` and returns the launch status, or
// kNotBuilt for a variant that has no instantiation (the caller reports it).
// The host logic that chooses among them lives in fsr_abi.cu.
#pragma once

#include <cuda_runtime.h>

#include "fsr_generic.cuh"
#include "fsr_pair64.cuh"
#include "fsr_warp32.cuh"

namespace fsr {

constexpr cudaError_t kNotBuilt = cudaErrorNotYetImplemented;

// OPTS bits for the fp32 kernels (trace / early-stop code compiled in)
constexpr int LOPT_TRACE = 1, LOPT_EARLY = 2, LOPT_KAPPA = 4, LOPT_REPLAY = 8;  // = W32_*

// N = 32 fp32 loop (fsr_warp32.cuh).  study: guard-study instrumentation
// (tools/guard_study.py; redux, f32 pixels only).
template <typename IO, int AM>
cudaError_t warp32_launch(const Warp32Args &a, const Warp32Maps &maps, bool tree, bool guard,
                          bool study, int opts, int sms, cudaStream_t st);
// N = 16 fp32 loop (fsr_warp16.cuh)
template <typename IO, int AM>
cudaError_t warp16_launch(const Warp32Args &a, const Warp32Maps &maps, bool tree, bool guard,
                          int opts, int sms, cudaStream_t st);
// N = 64 fp32 loop (fsr_cta64.cuh), linear reducer
template <typename IO, int AM>
cudaError_t cta64_launch(const Warp32Args &a, const Warp32Maps &maps, bool guard, int opts, int sms,
                         cudaStream_t st);

// fp64 kernels: validation precision and the guarded re-runs (list mode)
template <typename IO>
cudaError_t pair64_launch(const Pair64Args<IO> &a, bool tree, int am, int64_t want_blocks, int sms,
                          cudaStream_t st);
template <typename IO>
cudaError_t warp64_launch(const Pair64Args<IO> &a, bool tree, int am, int64_t want_blocks, int sms,
                          cudaStream_t st);
template <typename IO>
cudaError_t warp16d_launch(const Pair64Args<IO> &a, bool tree, int am, int64_t want_blocks, int sms,
                           cudaStream_t st);
// cta64d stages W through a per-CTA global buffer of 64 KiB: cta64d_grid gives
// the grid (the caller sizes a.scratch to grid * 4096 double2), then launch
template <typename IO>
cudaError_t cta64d_grid(int64_t want_blocks, int sms, int *grid);
template <typename IO>
cudaError_t cta64d_launch(const Pair64Args<IO> &a, int grid, cudaStream_t st);
// N in {4, 8, 24} (fsr_warpn.cuh): fp32 loop (reducer in a.tree) and fp64
template <typename IO, int N>
cudaError_t warpn_launch(const Warp32Args &a, const Warp32Maps &maps, int am, bool guard, int opts,
                         int sms, cudaStream_t st);
template <typename IO, int N>
cudaError_t warpnd_launch_n(const Pair64Args<IO> &a, int am, int64_t want_blocks, int sms, cudaStream_t st);
// the even supports up to 20 other than 16, and 24 (fsr_warpn.cuh), one object per
// (IO, N); N = 22, 26, 28, 30 stay on the generic kernel (their fully unrolled
// direct half-DFTs stall ptxas for tens of minutes)
#define FSR_WN_SUPPORTS(X) X(4) X(6) X(8) X(10) X(12) X(14) X(18) X(20) X(24)
template <typename IO>
inline cudaError_t warpnd_launch(const Pair64Args<IO> &a, int N, int am, int64_t want_blocks, int sms,
                                 cudaStream_t st) {
#define FSR_WND_CASE(n) \
    if (N == n) return warpnd_launch_n<IO, n>(a, am, want_blocks, sms, st);
    FSR_WN_SUPPORTS(FSR_WND_CASE)
#undef FSR_WND_CASE
    return kNotBuilt;
}
// N in {4, 8}, B <= 4: 32 / N blocks per warp (fsr_warpseg.cuh; own segmented argmax)
template <typename IO, int N>
cudaError_t warpseg_launch(const Warp32Args &a, bool guard, int opts, int sms, cudaStream_t st);
template <typename IO>
inline cudaError_t warpseg_any(const Warp32Args &a, int N, bool guard, int opts, int sms, cudaStream_t st) {
    if (N == 4) return warpseg_launch<IO, 4>(a, guard, opts, sms, st);
    if (N == 8) return warpseg_launch<IO, 8>(a, guard, opts, sms, st);
    return kNotBuilt;
}
// N in {4, 8}, B <= 4, fp64: the segmented layout (fsr_warpseg.cuh)
template <typename IO>
cudaError_t warpsegd_launch(const Pair64Args<IO> &a, int N, int64_t want_blocks, int sms, cudaStream_t st);
template <typename IO>
inline cudaError_t warpn_any(const Warp32Args &a, const Warp32Maps &m, int N, int am, bool guard,
                             int opts, int sms, cudaStream_t st) {
#define FSR_WN_CASE(n) \
    if (N == n) return warpn_launch<IO, n>(a, m, am, guard, opts, sms, st);
    FSR_WN_SUPPORTS(FSR_WN_CASE)
#undef FSR_WN_CASE
    return kNotBuilt;
}
// any support <= 64, strict IEEE (fsr_generic.cuh)
template <typename Real, typename IO>
cudaError_t generic_launch(const ImageArgs<Real, IO> &a, int grid, cudaStream_t st);

// runtime argmax variant -> the per-variant instantiation
template <typename IO>
inline cudaError_t warp32_any(const Warp32Args &a, const Warp32Maps &m, bool tree, int am, bool guard,
                              bool study, int opts, int sms, cudaStream_t st) {
    if (am == AM_SHFL) return warp32_launch<IO, AM_SHFL>(a, m, tree, guard, study, opts, sms, st);
    if (am == AM_SMEM) return warp32_launch<IO, AM_SMEM>(a, m, tree, guard, study, opts, sms, st);
    if (am == AM_REDUX) return warp32_launch<IO, AM_REDUX>(a, m, tree, guard, study, opts, sms, st);
    return kNotBuilt;
}
template <typename IO>
inline cudaError_t warp16_any(const Warp32Args &a, const Warp32Maps &m, bool tree, int am, bool guard,
                              int opts, int sms, cudaStream_t st) {
    if (am == AM_SHFL) return warp16_launch<IO, AM_SHFL>(a, m, tree, guard, opts, sms, st);
    if (am == AM_SMEM) return warp16_launch<IO, AM_SMEM>(a, m, tree, guard, opts, sms, st);
    if (am == AM_REDUX) return warp16_launch<IO, AM_REDUX>(a, m, tree, guard, opts, sms, st);
    return kNotBuilt;
}
template <typename IO>
inline cudaError_t cta64_any(const Warp32Args &a, const Warp32Maps &m, int am, bool guard, int opts,
                             int sms, cudaStream_t st) {
    if (am == AM_SHFL) return cta64_launch<IO, AM_SHFL>(a, m, guard, opts, sms, st);
    if (am == AM_SMEM) return cta64_launch<IO, AM_SMEM>(a, m, guard, opts, sms, st);
    if (am == AM_REDUX) return cta64_launch<IO, AM_REDUX>(a, m, guard, opts, sms, st);
    return kNotBuilt;
}

// Persistent grid of `per_block_threads`-thread CTAs for kernel k: the SM count
// times the resident CTAs per SM, capped by the work.
template <typename K>
cudaError_t persistent_grid(K k, int threads, size_t smem, int64_t want_ctas, int sms, int *grid) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    int64_t g = want_ctas < 1 ? 1 : want_ctas;
    if (g > (int64_t)sms * per_sm) g = (int64_t)sms * per_sm;
    *grid = (int)g;
    return cudaSuccess;
}

}  // namespace fsr
