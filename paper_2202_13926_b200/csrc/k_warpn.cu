// k_warpn.cu -- instantiations of the fp32 loop kernel for the paper grid's
// other supports (fsr_warpn.cuh) for pixel type FSR_IO and support FSR_N (one
// object per pair): every argmax variant, production (OPTS = 0, + the guard's
// scale term) and the full build (trace + early stop).
#include "fsr_launch.cuh"
#include "fsr_warpn.cuh"
#include "fsr_warpseg.cuh"

#ifndef FSR_IO
#define FSR_IO float
#endif
#ifndef FSR_N
#define FSR_N 24
#endif

namespace fsr {

namespace {
template <typename IO, int N, int AM, bool GUARD, int OPTS>
cudaError_t go(const Warp32Args &a, const Warp32Maps &maps, int sms, cudaStream_t st) {
    constexpr int WARPS = 4;
    auto k = warpn_kernel<IO, N, WARPS, AM, GUARD, OPTS>;
    const size_t smem = sizeof(WarpNSmem<N, WARPS>) +
                        ((OPTS & W32_REPLAY) ? ((size_t)WARPS * a.seq_stride * 2 + 15) / 16 * 16 : 0);
    int grid = 1;
    cudaError_t e = persistent_grid(k, WARPS * 32, smem, (a.nblocks + WARPS - 1) / WARPS, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, WARPS * 32, smem, st>>>(a, maps);
    return cudaGetLastError();
}

template <typename IO, int N, int AM>
cudaError_t by_opts(const Warp32Args &a, const Warp32Maps &maps, bool guard, int opts, int sms,
                    cudaStream_t st) {
    if (opts == 0) return guard ? go<IO, N, AM, true, 0>(a, maps, sms, st) : go<IO, N, AM, false, 0>(a, maps, sms, st);
    if (opts == LOPT_KAPPA && guard) return go<IO, N, AM, true, W32_KAPPA>(a, maps, sms, st);
    if constexpr (AM == AM_REDUX) {
        if (guard && opts == LOPT_REPLAY) return go<IO, N, AM, true, W32_REPLAY>(a, maps, sms, st);
        if (guard && opts == (LOPT_KAPPA | LOPT_REPLAY))
            return go<IO, N, AM, true, W32_KAPPA | W32_REPLAY>(a, maps, sms, st);
        if (guard && (opts & LOPT_REPLAY)) return go<IO, N, AM, true, W32_ALL | W32_REPLAY>(a, maps, sms, st);
    }
    return guard ? go<IO, N, AM, true, W32_ALL>(a, maps, sms, st) : go<IO, N, AM, false, W32_ALL>(a, maps, sms, st);
}
}  // namespace

template <typename IO, int N, bool GUARD, int OPTS>
cudaError_t seg_go(const Warp32Args &a, int sms, cudaStream_t st) {
    if constexpr (N == 4 || N == 8 || N == 16) {
        constexpr int WARPS = 4, BPC = WARPS * SegCfg<N>::BPW;  // blocks per CTA
        auto k = warpseg_kernel<IO, N, WARPS, GUARD, OPTS>;
        const size_t smem = sizeof(WarpSegSmem<N, WARPS>);
        int grid = 1;
        cudaError_t e = persistent_grid(k, WARPS * 32, smem, (a.nblocks + BPC - 1) / BPC, sms, &grid);
        if (e != cudaSuccess) return e;
        k<<<grid, WARPS * 32, smem, st>>>(a);
        return cudaGetLastError();
    } else {
        return kNotBuilt;
    }
}

// fp64 (validation + re-runs); the argmax variants only pick the cross-lane
// u64 max implementation (the keys carry the full tie rank: identical results),
// so supports outside the paper grid build redux alone
template <int N, int AM, typename IO>
cudaError_t wnd_go(const Pair64Args<IO> &a, int64_t want, int sms, cudaStream_t st) {
    constexpr int WARPS = 4;
    auto k = warpnd_kernel<N, WARPS, AM, IO>;
    const size_t smem = sizeof(WarpNdSmem<N, WARPS>);
    int grid = 1;
    cudaError_t e = persistent_grid(k, WARPS * 32, smem, (want + WARPS - 1) / WARPS, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, WARPS * 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename IO, int N>
cudaError_t warpnd_launch_n(const Pair64Args<IO> &a, int am, int64_t want, int sms, cudaStream_t st) {
    if constexpr (N == 16) {
        return kNotBuilt;
    } else if constexpr (N == 4 || N == 8 || N == 24) {
        if (am == AM_SHFL) return wnd_go<N, AM_SHFL>(a, want, sms, st);
        if (am == AM_SMEM) return wnd_go<N, AM_SMEM>(a, want, sms, st);
        return wnd_go<N, AM_REDUX>(a, want, sms, st);
    } else {
        return wnd_go<N, AM_REDUX>(a, want, sms, st);
    }
}

template <typename IO, int N>
cudaError_t warpseg_launch(const Warp32Args &a, bool guard, int opts, int sms, cudaStream_t st) {
    if (opts == 0) return guard ? seg_go<IO, N, true, 0>(a, sms, st) : seg_go<IO, N, false, 0>(a, sms, st);
    if (opts == LOPT_KAPPA && guard) return seg_go<IO, N, true, W32_KAPPA>(a, sms, st);
    return guard ? seg_go<IO, N, true, W32_ALL>(a, sms, st) : seg_go<IO, N, false, W32_ALL>(a, sms, st);
}

template <typename IO, int N>
cudaError_t warpn_launch(const Warp32Args &a, const Warp32Maps &maps, int am, bool guard, int opts,
                         int sms, cudaStream_t st) {
    if constexpr (N == 16) {
        return kNotBuilt;  // N = 16: warp16
    } else if constexpr (N == 4 || N == 8 || N == 24) {
        if (am == AM_SHFL) return by_opts<IO, N, AM_SHFL>(a, maps, guard, opts, sms, st);
        if (am == AM_SMEM) return by_opts<IO, N, AM_SMEM>(a, maps, guard, opts, sms, st);
        return by_opts<IO, N, AM_REDUX>(a, maps, guard, opts, sms, st);
    } else {
        // supports outside the paper grid: pair keys make every argmax variant
        // give the same selections, so only redux is built
        return by_opts<IO, N, AM_REDUX>(a, maps, guard, opts, sms, st);
    }
}

template cudaError_t warpn_launch<FSR_IO, FSR_N>(const Warp32Args &, const Warp32Maps &, int, bool,
                                                 int, int, cudaStream_t);
template cudaError_t warpseg_launch<FSR_IO, FSR_N>(const Warp32Args &, bool, int, int, cudaStream_t);
template cudaError_t warpnd_launch_n<FSR_IO, FSR_N>(const Pair64Args<FSR_IO> &, int, int64_t, int, cudaStream_t);

}  // namespace fsr
