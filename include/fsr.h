/*
 * fsr.h -- C ABI of the B200 Frequency Selective Reconstruction engine (libfsr.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as void*, a cudaStream_t).  Every entry point returns an
 * fsr_status; fsr_last_error() gives the message, whose text for the
 * FSR_EINVAL/FSR_ENOSAMPLES cases is the reference's ValueError text so that
 * the Python shim can raise the same exception.
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   fsr_reconstruct_f64/_f32      <- fsrkit.reconstruction.reconstruct_image
 *                                    pkg/src/fsrkit/reconstruction.py:216-290
 *   fsr_iterate_spectra           <- fsrkit._kernels.reconstruct_batch /
 *                                    reconstruct_iterations
 *                                    pkg/src/fsrkit/_kernels.py:62-149
 *   fsr_params_init / validation  <- fsrkit.core.FsrParams
 *                                    pkg/src/fsrkit/core.py:45-85
 *   fsr_spatial_oracle            <- fsrkit.oracle.oracle_reconstruct_traced
 *                                    pkg/src/fsrkit/oracle.py:25-132
 * The reference has no compiled FFI; INTEGRATION.md shows the ctypes binding
 * (the package's own shim, paper_2202_13926_b200/_lib.py) a maintainer of
 * the reference would add.
 */
#ifndef FSR_H_
#define FSR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSR_ABI_VERSION 4  /* 2: f64 pixels on every path, explicit empty-support fill for strips;
                              3: guard_kappa; 4: fsr_pin_host / fsr_unpin_host, direct DMA for
                              page-locked host buffers */

typedef enum {
    FSR_OK = 0,
    FSR_EINVAL = 1,      /* invalid argument -> ValueError (reference messages) */
    FSR_ENOSAMPLES = 2,  /* "no known samples" (reconstruction.py:273-274) -> ValueError */
    FSR_ECUDA = 3,       /* CUDA runtime failure -> RuntimeError */
    FSR_EUNSUPPORTED = 4 /* valid in the reference but not built here -> ValueError */
} fsr_status;

typedef enum { FSR_REDUCER_TREE = 0, FSR_REDUCER_LINEAR = 1 } fsr_reducer;

typedef enum {
    FSR_PREC_FP64 = 0,         /* validation mode: fp64 loop and transforms */
    FSR_PREC_FP32 = 1,         /* production: fp32 loop, near-tie blocks re-run in fp64 */
    FSR_PREC_FP32_UNGUARDED = 2 /* ablation: pure fp32, no re-run */
} fsr_precision;

typedef enum {
    FSR_ARGMAX_SHFL = 0,  /* register argmax: __shfl_xor_sync butterflies (the paper's) */
    FSR_ARGMAX_SMEM = 1,  /* shared-memory tree argmax (the paper's comparison point) */
    FSR_ARGMAX_REDUX = 2  /* redux.sync.max on packed keys + ballot */
} fsr_argmax_impl;

/* Mirrors FsrParams (core.py:45-85) plus the engine knobs. */
typedef struct {
    int32_t block;       /* B, target block side (>= 1) */
    int32_t border;      /* L, support = B + 2L (the "N" of BASELINE.json) */
    int32_t iterations;  /* I (>= 0) */
    int32_t reducer;     /* fsr_reducer: tie-break rule of the reference reducers */
    int32_t early_stop;  /* reconstruction.py:27, 262-266 */
    int32_t precision;   /* fsr_precision */
    int32_t argmax_impl; /* fsr_argmax_impl */
    int32_t kernel;      /* N=32 fp64 kernel: 0 auto (= warp pair), 1 one warp per block, 2 warp pair */
    double rho;          /* (0, 1) */
    double gamma;        /* (0, 1] */
    double guard_tau;    /* fp32 near-tie guard, relative term: a block is re-run in fp64 when
                            some iteration's top-2 objectives satisfy
                            b1 - b2 <= guard_tau * b1 + guard_kappa * sqrt(b1 * B0)
                            (B0 = the block's first maximum); 0 (default) = auto */
    double guard_kappa;  /* fp32 near-tie guard, scale term (the fp32 residual's absolute error
                            follows B0, not b1); 0 (default) = auto, < 0 = off */
} fsr_params;

typedef struct fsr_engine fsr_engine;

/* Defaults of the BASELINE configs: B=4, L=14 (N=32), I=100, rho=0.7, gamma=0.5, tree;
 * fp64 precision, redux argmax, guard_tau 0 (auto). */
void fsr_params_init(fsr_params *p);

/* Validate like FsrParams.__post_init__ (core.py:63-80); the S^2<=1024 cap is
 * lifted except for the tree reducer, whose two-phase lane groups cover at
 * most 1024 records (reduce.py:112-117). */
int fsr_params_validate(const fsr_params *p, char *msg, int msg_len);

/* Create an engine over the listed CUDA devices (NULL/0 -> device 0).  Image
 * calls split the block rows into contiguous strips, one per device. */
int fsr_engine_create(const int32_t *devices, int32_t n_devices, fsr_engine **out);
void fsr_engine_destroy(fsr_engine *eng);
const char *fsr_last_error(const fsr_engine *eng);
const char *fsr_status_string(int status);
int32_t fsr_abi_version(void);

/* Page-lock (cudaHostRegister, portable) / release a host range, so host-buffer
 * calls DMA to and from it directly instead of staging through the engine's
 * pinned buffers.  Python's result arrays live in such a recycled pool.  The
 * range must stay allocated until fsr_unpin_host. */
int fsr_pin_host(void *p, size_t bytes);
int fsr_unpin_host(void *p);

/*
 * Whole-path call with HOST buffers (reconstruct_image).  px: H*W pixels on the
 * 0..255 scale, row-major; unknown pixels are ignored (the reference requires
 * them to be zero).  mask: H*W bytes, nonzero = known.  out: H*W, must not
 * overlap px or mask (FSR_EINVAL "output buffer overlaps an input buffer").  sel (nullable): [n_blocks, iterations] selected flat bins
 * (u*N+v) per block in partition order, -1 after an early stop; done
 * (nullable): [n_blocks] iterations run.  Synchronous.
 *
 * Every precision takes either pixel type: _f64 is the reference's own input
 * contract (core.py:24, f64 pixels), and the fp32-loop kernels read f64 pixels
 * directly (their gather / weighting / FFT prologue runs in fp64), so FP32 on
 * _f64 buffers is the production mode on the reference's exact inputs.
 * The caller's buffers may be pageable: each device's chunks are staged
 * through engine-owned pinned buffers by a small host thread pool, and the
 * engine's devices run their strips concurrently (one host thread each).
 * Page-locked buffers (cudaHostAlloc'd, or registered with fsr_pin_host) skip
 * the staging: px/mask are copied to the device and results to `out` directly.
 */
int fsr_reconstruct_f64(fsr_engine *eng, const fsr_params *p, const double *px,
                        const uint8_t *mask, int64_t height, int64_t width, double *out,
                        int32_t *sel, int32_t *done);
int fsr_reconstruct_f32(fsr_engine *eng, const fsr_params *p, const float *px,
                        const uint8_t *mask, int64_t height, int64_t width, float *out,
                        int32_t *sel, int32_t *done);

/*
 * Strip variant for sharded callers (one process per GPU): only target-block
 * rows [row0, row1) are reconstructed; only the image rows their windows touch
 * (the strip plus L = border rows above and below) are read and only the
 * strip's output rows of `out` (a full H*W host buffer) are written.
 * fill: the value of empty-support blocks -- the mean of the known samples of
 * the WHOLE frame (reconstruction.py:236-237), which a strip holder computes
 * once (or gets by an all-reduce of sum and count); pass NaN to have it
 * computed here from px/mask, which then must hold every row of the frame.
 */
int fsr_reconstruct_rows_f32(fsr_engine *eng, const fsr_params *p, const float *px,
                             const uint8_t *mask, int64_t height, int64_t width, int64_t row0,
                             int64_t row1, double fill, float *out);
int fsr_reconstruct_rows_f64(fsr_engine *eng, const fsr_params *p, const double *px,
                             const uint8_t *mask, int64_t height, int64_t width, int64_t row0,
                             int64_t row1, double fill, double *out);

/*
 * Device-resident call on the engine's first device, asynchronous on `stream`
 * (a cudaStream_t; NULL = legacy default stream).  d_px/d_mask/d_out are
 * device pointers with row pitches in ELEMENTS.  row0/row1 restrict the work
 * to target-block rows [row0, row1) of the full image (strip partitioning);
 * pass 0 and ceil(H/B) for the whole frame.  Only the image rows the strip's
 * windows touch (L rows above and below) are read, unless fill is NaN: then
 * the empty-support fill is the mean of the known samples of all H rows,
 * summed on the device in a fixed order (deterministic), and all H rows must
 * be valid.  With no known sample anywhere the call's fsr_last_stats returns
 * FSR_ENOSAMPLES ("no known samples").  Calls on one engine are serialised in
 * issue order even across different streams (each waits for the previous
 * call's end), because they share the engine's per-call scratch.  Pitches
 * below the width and a d_out range overlapping d_px or d_mask are refused
 * (FSR_EINVAL): later chunks still read rows that earlier chunks write.
 */
int fsr_reconstruct_device_f32(fsr_engine *eng, const fsr_params *p, const float *d_px,
                               int64_t px_pitch, const uint8_t *d_mask, int64_t mask_pitch,
                               int64_t height, int64_t width, int64_t row0, int64_t row1,
                               float *d_out, int64_t out_pitch, double fill, void *stream);
int fsr_reconstruct_device_f64(fsr_engine *eng, const fsr_params *p, const double *d_px,
                               int64_t px_pitch, const uint8_t *d_mask, int64_t mask_pitch,
                               int64_t height, int64_t width, int64_t row0, int64_t row1,
                               double *d_out, int64_t out_pitch, double fill, void *stream);

/*
 * Array-level loop operator (_kernels.reconstruct_batch plus the traces of
 * reconstruct_iterations).  Host arrays, complex128 interleaved (re, im):
 * R [count, N, N] in/out residual spectra, G [count, N, N] in/out model
 * spectra (accumulated into, as the reference does), W [count, N, N] weight
 * spectra, wf [N, N], thr [count] early-stop thresholds (nullable = 0).
 * Traces (nullable) are [count, iterations]: sel, obj, ties; done [count].
 * Blocks with W[0,0].re <= 0 are skipped (done = 0).  fp64 strict IEEE, no
 * FMA: bitwise equal to the reference.  p->block/border/rho are ignored.
 */
int fsr_iterate_spectra(fsr_engine *eng, const fsr_params *p, int64_t count, int32_t N,
                        double *R, double *G, const double *W, const double *wf,
                        const double *thr, int32_t *sel, double *obj, uint8_t *ties,
                        int32_t *done);

/*
 * FFT-free spatial-domain oracle (oracle.oracle_reconstruct_traced), an
 * independent cross-check of the frequency-domain path, supports S <= 16.
 * Host arrays: signal/spatial [count, S, S] f64 (spatial = decay * mask, the
 * WeightSet's w), mask [count, S, S] u8, wf [S, S] f64; outputs out
 * [count, S, S] (mask ? signal : Re model), objectives/selections/ties
 * [count, iterations], energies [count, iterations + 1].  fp64; the first
 * maximum in flat order; a tie is > 1 objective within 1e-9 of the maximum.
 */
int fsr_spatial_oracle(fsr_engine *eng, int32_t support, int32_t iterations, double gamma,
                       int64_t count, const double *signal, const uint8_t *mask,
                       const double *spatial, const double *wf, double *out, double *objectives,
                       int32_t *selections, uint8_t *ties, double *energies);

/*
 * The callers either side of the loop, on the engine's first device,
 * asynchronous on `stream` (device pointers, pitches in elements):
 *
 * fsr_quarter_sample_device: quarter sampling of a frame exactly as
 * fsrkit.sampling.quarter_sample (pkg/src/fsrkit/sampling.py:18-29 SplitMix64,
 * 53-80): one known pixel per 2x2 cell (edge cells of odd frames shrink);
 * writes the mask (1 = known) and the sampled frame (unknown pixels 0).
 *
 * fsr_sq_error_device: *d_sse = sum over pixels of (clamp(test,0,255) - ref)^2
 * in fp64 (fsrkit.metrics.psnr, metrics.py:35-48: PSNR = 10 log10(255^2 /
 * (sse / (height*width)))); deterministic summation order.
 */
int fsr_quarter_sample_device(fsr_engine *eng, const float *d_img, int64_t img_pitch,
                              int64_t height, int64_t width, uint64_t seed, float *d_sampled,
                              int64_t sampled_pitch, uint8_t *d_mask, int64_t mask_pitch,
                              void *stream);
int fsr_sq_error_device(fsr_engine *eng, const float *d_ref, int64_t ref_pitch, const float *d_test,
                        int64_t test_pitch, int64_t height, int64_t width, double *d_sse,
                        void *stream);

/* Statistics of the last image call (kernel times of the first device).  For
 * an asynchronous device call this waits for it, and returns FSR_ENOSAMPLES if
 * the call found an empty-support block but no known sample. */
typedef struct {
    int64_t blocks;          /* target blocks processed */
    int64_t rerun_blocks;    /* blocks re-run in fp64 by the near-tie guard */
    int64_t empty_blocks;    /* blocks with no known sample in the window */
    int32_t kernel_launches; /* kernels launched by the call (all devices) */
    int32_t flags;           /* FSR_STATS_* bits of the first device's launch */
    double kernel_ms;        /* device time of the last call's kernels (first device) */
    double main_ms;          /* device time of the dominant kernel (first device; summed over chunks) */
} fsr_stats;
/* fsr_stats.flags: the N=32 fp32 kernel gathered its windows with TMA (2-D
 * tensor maps, zero fill outside the image).  Set FSR_NO_TMA=1 in the
 * environment before fsr_engine_create to force the plain-load gather.
 * Calls over at least 24 block rows run in 3..12 row chunks alternating
 * over up to eight internal streams (forked from / joined into the caller's stream
 * for the device API); results are identical to one launch.  FSR_NO_CHUNK=1
 * at fsr_engine_create makes every call a single launch (kernel timing). */
#define FSR_STATS_TMA_GATHER 1
/* fsr_stats.flags: a guarded FP32 request was served by the fp64 kernels (more
 * than 300 iterations, N = 4 (whose fp64 kernel is faster than fp32 plus its
 * ~45 % re-runs), or a support without an fp32 register kernel -- the fp32 ones
 * cover every even N from 6 to 20, 24, 32 and N = 64 with the linear reducer). */
#define FSR_STATS_SERVED_FP64 2
int fsr_last_stats(const fsr_engine *eng, fsr_stats *out);

#ifdef __cplusplus
}
#endif

#endif /* FSR_H_ */
