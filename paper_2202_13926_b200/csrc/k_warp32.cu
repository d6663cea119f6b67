// k_warp32.cu -- instantiations of the N = 32 fp32 loop kernel (fsr_warp32.cuh)
// for one pixel type FSR_IO and one argmax variant FSR_AM (set by the Makefile;
// one object per pair, built in parallel).
//
// Every argmax variant gets the same option set: the production build without
// trace or early-stop code (OPTS = 0) and the full one (OPTS = 3); redux also
// has trace-only / early-stop-only builds.  So the C5 argmax ablation compares
// kernels that differ only in the cross-lane argmax.
#include "fsr_launch.cuh"

#ifndef FSR_IO
#define FSR_IO float
#endif
#ifndef FSR_AM
#define FSR_AM 2
#endif
#ifndef FSR_W32_CTA_WARPS
#define FSR_W32_CTA_WARPS 4
#endif

namespace fsr {

namespace {
template <typename IO, int AM, bool TREE, bool GUARD, bool STUDY, int OPTS>
cudaError_t go(const Warp32Args &a, const Warp32Maps &maps, int sms, cudaStream_t st) {
    constexpr int WARPS = FSR_W32_CTA_WARPS;
    auto k = warp32_kernel<IO, WARPS, TREE, AM, GUARD, STUDY, OPTS>;
    // W32_REPLAY: the warps' selection records after the struct
    const size_t smem = sizeof(Warp32Smem<WARPS>) +
                        ((OPTS & W32_REPLAY) ? ((size_t)WARPS * a.seq_stride * 2 + 15) / 16 * 16 : 0);
    int grid = 1;
    cudaError_t e = persistent_grid(k, WARPS * 32, smem, (a.nblocks + WARPS - 1) / WARPS, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, WARPS * 32, smem, st>>>(a, maps);
    return cudaGetLastError();
}

template <typename IO, int AM, bool TREE, bool GUARD>
cudaError_t by_opts(const Warp32Args &a, const Warp32Maps &maps, int opts, int sms, cudaStream_t st) {
    if (opts == 0) return go<IO, AM, TREE, GUARD, false, 0>(a, maps, sms, st);
    if constexpr (GUARD) {
        if (opts == LOPT_KAPPA) return go<IO, AM, TREE, GUARD, false, LOPT_KAPPA>(a, maps, sms, st);
        if constexpr (AM == AM_REDUX) {
            if (opts == LOPT_REPLAY) return go<IO, AM, TREE, GUARD, false, LOPT_REPLAY>(a, maps, sms, st);
            if (opts == (LOPT_KAPPA | LOPT_REPLAY))
                return go<IO, AM, TREE, GUARD, false, LOPT_KAPPA | LOPT_REPLAY>(a, maps, sms, st);
        }
    }
    if constexpr (AM == AM_REDUX) {
        if (opts == LOPT_TRACE) return go<IO, AM, TREE, GUARD, false, LOPT_TRACE>(a, maps, sms, st);
        if (opts == LOPT_EARLY) return go<IO, AM, TREE, GUARD, false, LOPT_EARLY>(a, maps, sms, st);
    }
    if constexpr (GUARD && AM == AM_REDUX)
        if (opts & LOPT_REPLAY) return go<IO, AM, TREE, GUARD, false, W32_ALL | W32_REPLAY>(a, maps, sms, st);
    return go<IO, AM, TREE, GUARD, false, W32_ALL>(a, maps, sms, st);
}
}  // namespace

template <typename IO, int AM>
cudaError_t warp32_launch(const Warp32Args &a, const Warp32Maps &maps, bool tree, bool guard,
                          bool study, int opts, int sms, cudaStream_t st) {
    if (study) {
        if constexpr (AM == AM_REDUX && std::is_same<IO, float>::value)
            return tree ? go<IO, AM, true, true, true, W32_ALL>(a, maps, sms, st)
                        : go<IO, AM, false, true, true, W32_ALL>(a, maps, sms, st);
        return kNotBuilt;
    }
    if (tree) return guard ? by_opts<IO, AM, true, true>(a, maps, opts, sms, st)
                           : by_opts<IO, AM, true, false>(a, maps, opts, sms, st);
    return guard ? by_opts<IO, AM, false, true>(a, maps, opts, sms, st)
                 : by_opts<IO, AM, false, false>(a, maps, opts, sms, st);
}

template cudaError_t warp32_launch<FSR_IO, FSR_AM>(const Warp32Args &, const Warp32Maps &, bool, bool,
                                                   bool, int, int, cudaStream_t);

}  // namespace fsr
