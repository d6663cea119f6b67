// k_cta64.cu -- instantiations of the N = 64 fp32 loop kernel (fsr_cta64.cuh)
// for pixel type FSR_IO and in-warp argmax variant FSR_AM (one object per pair;
// the cross-warp phase is the same for all).
#include "fsr_launch.cuh"
#include "fsr_cta64.cuh"

#ifndef FSR_IO
#define FSR_IO float
#endif
#ifndef FSR_AM
#define FSR_AM 2
#endif

namespace fsr {

namespace {
template <typename IO, int AM, bool GUARD, int OPTS = 0>
cudaError_t go(const Warp32Args &a, const Warp32Maps &maps, int sms, cudaStream_t st) {
    auto k = cta64_kernel<IO, AM, GUARD, OPTS>;
    const size_t smem = sizeof(C64Smem) + ((OPTS & W32_REPLAY) ? ((size_t)a.seq_stride * 2 + 15) / 16 * 16 : 0);
    int grid = 1;
    cudaError_t e = persistent_grid(k, C64_THREADS, smem, a.nblocks, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, C64_THREADS, smem, st>>>(a, maps);
    return cudaGetLastError();
}
}  // namespace

template <typename IO, int AM>
cudaError_t cta64_launch(const Warp32Args &a, const Warp32Maps &maps, bool guard, int opts, int sms,
                         cudaStream_t st) {
    if constexpr (AM == AM_REDUX)
        if (guard && (opts & LOPT_REPLAY))
            return a.iterations > 100 ? go<IO, AM, true, W32_REPLAY | W32_EXIT>(a, maps, sms, st)
                                      : go<IO, AM, true, W32_REPLAY>(a, maps, sms, st);
    return guard ? go<IO, AM, true>(a, maps, sms, st) : go<IO, AM, false>(a, maps, sms, st);
}

template cudaError_t cta64_launch<FSR_IO, FSR_AM>(const Warp32Args &, const Warp32Maps &, bool, int,
                                                  int, cudaStream_t);

}  // namespace fsr
