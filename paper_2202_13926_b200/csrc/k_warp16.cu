// k_warp16.cu -- instantiations of the N = 16 fp32 loop kernel (fsr_warp16.cuh)
// for pixel type FSR_IO and argmax variant FSR_AM (one object per pair).
// Options as in k_warp32.cu: OPTS = 0 (production) and 3 (trace + early stop)
// for every argmax variant.
#include "fsr_launch.cuh"
#include "fsr_warp16.cuh"

#ifndef FSR_IO
#define FSR_IO float
#endif
#ifndef FSR_AM
#define FSR_AM 2
#endif

namespace fsr {

namespace {
template <typename IO, int AM, bool TREE, bool GUARD, int OPTS>
cudaError_t go(const Warp32Args &a, const Warp32Maps &maps, int sms, cudaStream_t st) {
    constexpr int WARPS = 4;
    auto k = warp16_kernel<IO, WARPS, TREE, AM, GUARD, OPTS>;
    const size_t smem = sizeof(Warp16Smem<WARPS>) +
                        ((OPTS & W32_REPLAY) ? ((size_t)WARPS * a.seq_stride * 2 + 15) / 16 * 16 : 0);
    int grid = 1;
    cudaError_t e = persistent_grid(k, WARPS * 32, smem, (a.nblocks + WARPS - 1) / WARPS, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, WARPS * 32, smem, st>>>(a, maps);
    return cudaGetLastError();
}
}  // namespace

template <typename IO, int AM>
cudaError_t warp16_launch(const Warp32Args &a, const Warp32Maps &maps, bool tree, bool guard,
                          int opts, int sms, cudaStream_t st) {
    if (opts == 0) {
        if (tree) return guard ? go<IO, AM, true, true, 0>(a, maps, sms, st) : go<IO, AM, true, false, 0>(a, maps, sms, st);
        return guard ? go<IO, AM, false, true, 0>(a, maps, sms, st) : go<IO, AM, false, false, 0>(a, maps, sms, st);
    }
    if (opts == LOPT_KAPPA && guard)
        return tree ? go<IO, AM, true, true, W32_KAPPA>(a, maps, sms, st) : go<IO, AM, false, true, W32_KAPPA>(a, maps, sms, st);
    if constexpr (AM == AM_REDUX) {
        if (guard && opts == LOPT_REPLAY)
            return tree ? go<IO, AM, true, true, W32_REPLAY>(a, maps, sms, st)
                        : go<IO, AM, false, true, W32_REPLAY>(a, maps, sms, st);
        if (guard && opts == (LOPT_KAPPA | LOPT_REPLAY))
            return tree ? go<IO, AM, true, true, W32_KAPPA | W32_REPLAY>(a, maps, sms, st)
                        : go<IO, AM, false, true, W32_KAPPA | W32_REPLAY>(a, maps, sms, st);
        if (guard && (opts & LOPT_REPLAY))
            return tree ? go<IO, AM, true, true, W32_ALL | W32_REPLAY>(a, maps, sms, st)
                        : go<IO, AM, false, true, W32_ALL | W32_REPLAY>(a, maps, sms, st);
    }
    if (tree) return guard ? go<IO, AM, true, true, W32_ALL>(a, maps, sms, st) : go<IO, AM, true, false, W32_ALL>(a, maps, sms, st);
    return guard ? go<IO, AM, false, true, W32_ALL>(a, maps, sms, st) : go<IO, AM, false, false, W32_ALL>(a, maps, sms, st);
}

template cudaError_t warp16_launch<FSR_IO, FSR_AM>(const Warp32Args &, const Warp32Maps &, bool, bool,
                                                   int, int, cudaStream_t);

}  // namespace fsr
