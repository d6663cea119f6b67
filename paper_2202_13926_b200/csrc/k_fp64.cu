// k_fp64.cu -- instantiations of the fp64 image kernels for pixel type FSR_IO:
// pair64 / warp64 (N = 32), warp16d (N = 16), cta64d (N = 64) and the generic
// CTA-per-block kernel (any N <= 64, fp64 and fp32 loops).  These serve the
// fp64 validation precision and the guarded fp32 mode's re-runs (list mode).
#include "fsr_launch.cuh"
#include "fsr_cta64.cuh"
#include "fsr_warp16.cuh"
#include "fsr_warp64.cuh"
#include "fsr_warpn.cuh"
#include "fsr_warpseg.cuh"

#ifndef FSR_IO
#define FSR_IO float
#endif
#ifndef FSR_P64_BPC
#define FSR_P64_BPC 4
#endif

namespace fsr {

namespace {
constexpr int kPairBPC = FSR_P64_BPC;
constexpr int kWarp64Warps = 5;
constexpr int kW16dWarps = 4;

template <typename IO, bool TREE, int AM>
cudaError_t pair_go(const Pair64Args<IO> &a, int64_t want, int sms, cudaStream_t st) {
    auto k = pair64_kernel<kPairBPC, TREE, AM, IO>;
    const size_t smem = sizeof(Pair64Smem<kPairBPC>);
    int grid = 1;
    cudaError_t e = persistent_grid(k, kPairBPC * 64, smem, (want + kPairBPC - 1) / kPairBPC, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, kPairBPC * 64, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename IO, bool TREE, int AM>
cudaError_t warp64_go(const Pair64Args<IO> &a, int64_t want, int sms, cudaStream_t st) {
    auto k = warp64_kernel<kWarp64Warps, TREE, AM, IO>;
    const size_t smem = sizeof(Warp64Smem<kWarp64Warps>);
    int grid = 1;
    cudaError_t e = persistent_grid(k, kWarp64Warps * 32, smem, (want + kWarp64Warps - 1) / kWarp64Warps, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, kWarp64Warps * 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename IO, bool TREE, int AM>
cudaError_t w16d_go(const Pair64Args<IO> &a, int64_t want, int sms, cudaStream_t st) {
    auto k = warp16d_kernel<kW16dWarps, TREE, AM, IO>;
    const size_t smem = sizeof(Warp16dSmem<kW16dWarps>);
    int grid = 1;
    cudaError_t e = persistent_grid(k, kW16dWarps * 32, smem, (want + kW16dWarps - 1) / kW16dWarps, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, kW16dWarps * 32, smem, st>>>(a);
    return cudaGetLastError();
}

#define FSR_BY_TREE_AM(GO)                                                       \
    if (tree && am == AM_SHFL) return GO<IO, true, AM_SHFL>(a, want, sms, st);   \
    if (!tree && am == AM_SHFL) return GO<IO, false, AM_SHFL>(a, want, sms, st); \
    if (tree && am == AM_REDUX) return GO<IO, true, AM_REDUX>(a, want, sms, st); \
    if (!tree && am == AM_REDUX) return GO<IO, false, AM_REDUX>(a, want, sms, st); \
    if (tree && am == AM_SMEM) return GO<IO, true, AM_SMEM>(a, want, sms, st);   \
    if (!tree && am == AM_SMEM) return GO<IO, false, AM_SMEM>(a, want, sms, st); \
    return kNotBuilt;
}  // namespace

template <typename IO>
cudaError_t pair64_launch(const Pair64Args<IO> &a, bool tree, int am, int64_t want, int sms, cudaStream_t st) {
    FSR_BY_TREE_AM(pair_go)
}
template <typename IO>
cudaError_t warp64_launch(const Pair64Args<IO> &a, bool tree, int am, int64_t want, int sms, cudaStream_t st) {
    FSR_BY_TREE_AM(warp64_go)
}
template <typename IO>
cudaError_t warp16d_launch(const Pair64Args<IO> &a, bool tree, int am, int64_t want, int sms, cudaStream_t st) {
    FSR_BY_TREE_AM(w16d_go)
}
#undef FSR_BY_TREE_AM

template <int N, typename IO>
cudaError_t wsd_go(const Pair64Args<IO> &a, int64_t want, int sms, cudaStream_t st) {
    constexpr int WARPS = 4, BPC = WARPS * SegdCfg<N>::BPW;
    auto k = warpsegd_kernel<N, WARPS, IO>;
    const size_t smem = sizeof(WarpSegdSmem<N, WARPS>);
    int grid = 1;
    cudaError_t e = persistent_grid(k, WARPS * 32, smem, (want + BPC - 1) / BPC, sms, &grid);
    if (e != cudaSuccess) return e;
    k<<<grid, WARPS * 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename IO>
cudaError_t warpsegd_launch(const Pair64Args<IO> &a, int N, int64_t want, int sms, cudaStream_t st) {
    if (N == 4) return wsd_go<4>(a, want, sms, st);
    if (N == 8) return wsd_go<8>(a, want, sms, st);
    return kNotBuilt;
}

template <typename IO>
cudaError_t cta64d_grid(int64_t want, int sms, int *grid) {
    return persistent_grid(cta64d_kernel<IO>, C64_THREADS, sizeof(C64dSmem), want, sms, grid);
}
template <typename IO>
cudaError_t cta64d_launch(const Pair64Args<IO> &a, int grid, cudaStream_t st) {
    cta64d_kernel<IO><<<grid, C64_THREADS, sizeof(C64dSmem), st>>>(a);
    return cudaGetLastError();
}

template <typename Real, typename IO>
cudaError_t generic_launch(const ImageArgs<Real, IO> &a, int grid, cudaStream_t st) {
    const size_t smem = (size_t)2 * a.N * a.N * 2 * sizeof(Real);
    auto k = image_generic_kernel<Real, IO>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    // small supports (N*N <= 256: the paper grid's S = 8, 12) get a CTA sized to
    // their bin count instead of 256 mostly idle threads, and proportionally
    // more CTAs; the kernel's per-thread arrays cover 16 strides of the CTA
    const int n = a.N * a.N;
    int threads = GEN_THREADS;
    if (n <= GEN_THREADS && a.B * a.B <= 16 * 64) threads = n < 64 ? 64 : (n + 31) / 32 * 32;
    int64_t g = (int64_t)grid * (GEN_THREADS / threads);
    if (!a.list_count && g > (a.nblocks > 1 ? a.nblocks : 1)) g = a.nblocks > 1 ? a.nblocks : 1;
    k<<<(int)g, threads, smem, st>>>(a);
    return cudaGetLastError();
}

template cudaError_t pair64_launch<FSR_IO>(const Pair64Args<FSR_IO> &, bool, int, int64_t, int, cudaStream_t);
template cudaError_t warp64_launch<FSR_IO>(const Pair64Args<FSR_IO> &, bool, int, int64_t, int, cudaStream_t);
template cudaError_t warp16d_launch<FSR_IO>(const Pair64Args<FSR_IO> &, bool, int, int64_t, int, cudaStream_t);
template cudaError_t cta64d_grid<FSR_IO>(int64_t, int, int *);
template cudaError_t warpsegd_launch<FSR_IO>(const Pair64Args<FSR_IO> &, int, int64_t, int, cudaStream_t);
template cudaError_t cta64d_launch<FSR_IO>(const Pair64Args<FSR_IO> &, int, cudaStream_t);
template cudaError_t generic_launch<double, FSR_IO>(const ImageArgs<double, FSR_IO> &, int, cudaStream_t);
template cudaError_t generic_launch<float, FSR_IO>(const ImageArgs<float, FSR_IO> &, int, cudaStream_t);

}  // namespace fsr
