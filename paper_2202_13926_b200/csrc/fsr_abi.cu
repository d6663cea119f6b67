// fsr_abi.cu -- the C ABI of libfsr.so (include/fsr.h) and the engine behind it.
//
// Host side: parameter validation with the reference's messages
// (core.py:63-80, reconstruction.py:58-61, 273-274), per-(N, rho) constant
// tables (weights.py:18-27, 40-56), per-device buffers and streams, strip
// partitioning of the block rows over the engine's devices, and
// kernel dispatch:
//   precision FP64            -> image_generic_kernel<double>  (validation)
//   precision FP32, N=32,B<=5 -> warp32_kernel (+ fp64 re-run of guarded blocks)
//   precision FP32, N=16,B<=5 -> warp16_kernel (+ warp16d fp64 re-run of guarded blocks)
//   precision FP32, N=64       -> cta64_kernel (+ generic fp64 re-run of guarded blocks)
//   precision FP32, other N   -> image_generic_kernel<float>  (+ fp64 re-run)
// No CPU fallback: without a CUDA device every entry point returns FSR_ECUDA.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#define FSR_ABI_TU
#include "../../include/fsr.h"
#include "fsr_common.cuh"
#include "fsr_generic.cuh"
#include "fsr_warp32.cuh"
#include "fsr_warp16.cuh"
#include "fsr_cta64.cuh"
#include "fsr_pair64.cuh"
#include "fsr_aux.cuh"
#include "fsr_spatial.cuh"
#include "fsr_warp64.cuh"
#include "fsr_launch.cuh"

using namespace fsr;

namespace {

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    int dev = -1;
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, need);
        if (e == cudaSuccess) bytes = need;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

struct TableSet {
    DevBuf f64, f32;  // decay[N*N] | wf[N*N] | cs[2N]
};

// Pinned host staging of the host-buffer calls (SURVEY §8b "Ownership": the
// engine owns device buffers and pinned staging, reused across calls).
struct HostBuf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaHostAlloc(&p, need, cudaHostAllocPortable);
        if (e == cudaSuccess) bytes = need;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

struct ChunkCtr {              // device-side, per row chunk, zeroed on the chunk's stream
    unsigned int rerun_count;  // blocks queued for the fp64 re-run (guarded fp32)
    unsigned int skip_empty;   // the re-run kernels' empty counter (already counted)
};
struct CallCtr {               // device-side, per call and device, zeroed once per call
    unsigned int empty_count;  // empty-support blocks over all chunks (list: Device::empty_list)
    int status;                // 2: an empty block but no known sample anywhere
};

// A small persistent worker pool for the host-side staging copies (parallel
// memcpy between the caller's pageable buffers and the pinned staging).  All
// state is under one mutex; tasks are few (a chunk's rows in T pieces) and
// each is a large memcpy, so the lock is never contended in practice.
class Pool {
  public:
    explicit Pool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    int size() const { return (int)workers_.size() + 1; }
    // fn(i) for i in [0, n) on the workers and the calling thread; returns when all are done
    void run(int n, const std::function<void(int)> &fn) {
        std::unique_lock<std::mutex> lk(m_);
        job_ = &fn;
        next_ = 0;
        total_ = n;
        pending_ = n;
        cv_.notify_all();
        while (next_ < total_) {
            const int i = next_++;
            lk.unlock();
            fn(i);
            lk.lock();
            --pending_;
        }
        done_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
        total_ = 0;
    }

  private:
    void loop() {
        std::unique_lock<std::mutex> lk(m_);
        for (;;) {
            cv_.wait(lk, [&] { return stop_ || (job_ && next_ < total_); });
            if (stop_) return;
            const int i = next_++;
            const std::function<void(int)> *f = job_;
            lk.unlock();
            (*f)(i);
            lk.lock();
            if (--pending_ == 0) done_.notify_all();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)> *job_ = nullptr;
    int next_ = 0, total_ = 0, pending_ = 0;
    bool stop_ = false;
};

// rows [0, rows) of `bytes_per_row` from src to dst, split over the pool
void pool_copy(Pool *pool, void *dst, const void *src, int64_t rows, size_t bytes_per_row) {
    const size_t total = (size_t)rows * bytes_per_row;
    const int parts = (pool && total >= ((size_t)1 << 20)) ? pool->size() : 1;
    auto piece = [&](int i) {
        const int64_t r0 = rows * i / parts, r1 = rows * (i + 1) / parts;
        if (r1 > r0)
            std::memcpy((char *)dst + r0 * bytes_per_row, (const char *)src + r0 * bytes_per_row,
                        (size_t)(r1 - r0) * bytes_per_row);
    };
    if (parts == 1) piece(0);
    else pool->run(parts, piece);
}

struct Device {
    int id = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_done = nullptr;  // end of the engine's last call on this device (calls are serialised)
    DevBuf px, mask, out, sel, done, empty_list, rerun_list, call_ctr, chunk_ctrs, fill_partials;
    DevBuf rerun_kf, rerun_seq;  // replay records of the guarded N = 32 / 16 kernels (per re-run slot)
    int replay_min_iters = 101;  // replay the fp64 re-runs' unambiguous prefix from this I on
                                 // (FSR_REPLAY_MIN; 0 = never)
    DevBuf R, G, W, wf, thr, obj, ties, partials, c64scratch;
    HostBuf hin, hout;  // pinned staging of a lane's chunk (host-buffer calls)
    std::map<std::pair<int, double>, std::unique_ptr<TableSet>> tables;
    int launches = 0;
    float *gap_debug = nullptr;  // device buffer for fsr_debug_guard_gaps (null = off)
    bool tma_enabled = true;     // window gather by TMA when the rows allow it
    bool chunking = true;        // large calls in row chunks over kLanes streams (FSR_NO_CHUNK=1: off)
    int used_tma = 0;            // last fp32-loop launch gathered by TMA
    int served_fp64 = 0;         // last launch: a guarded fp32 request served by the fp64 kernels
    bool segmented = true;       // N <= 8: 32/N blocks per warp (FSR_NO_SEG=1: one warp per block)
    // Calls run as K row chunks over kLanes "lanes" (same GPU, own stream, staging
    // buffers and re-run scratch): one chunk's copies, fp64 re-run and launch
    // tail overlap the other chunks' main kernels.
    std::vector<std::unique_ptr<Device>> lanes;
    std::unique_ptr<Pool> pool;  // host staging copies (host-buffer calls)
    int last_chunks = 0;         // chunks of the last call (for its statistics)
    cudaEvent_t ck0[16] = {}, ck1[16] = {};  // per-chunk main-kernel brackets (K <= 16)
    cudaEvent_t ck2[16] = {};  // FSR_CHUNK_TRACE: end of each chunk's work (main kernel + re-run)
    // host pipeline: the chunk whose output is still in this lane's pinned staging
    bool pending = false;
    int64_t pend_oa = 0, pend_ob = 0;
};

}  // namespace

struct fsr_engine {
    std::vector<std::unique_ptr<Device>> devs;
    std::string err;
    std::mutex err_mu;  // err is written by the per-device worker threads of a host call
    std::mutex mu;
    fsr_stats stats{};
    bool device_stats_pending = false;
};

namespace {

thread_local std::string g_err;

int fail(fsr_engine *eng, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (eng) {
        std::lock_guard<std::mutex> lk(eng->err_mu);
        eng->err = buf;
    }
    g_err = buf;
    return code;
}

#define CUDA_TRY(eng, expr)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(eng, FSR_ECUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__, #expr);                                           \
    } while (0)

// ----------------------------------------------------------------- tables
// Host restatement of the reference tables in fp64 (the product computes its
// own; bitwise identity with numpy is not required past the FFT boundary).
void host_tables(int N, double rho, std::vector<double> &decay, std::vector<double> &wf,
                 std::vector<double> &cs) {
    decay.resize((size_t)N * N);
    wf.resize((size_t)N * N);
    cs.resize(2 * (size_t)N);
    const double center = (N - 1) / 2.0;  // weights.py:21
    for (int k = 0; k < N; ++k)
        for (int l = 0; l < N; ++l) {
            double dk = (k - center) * (k - center), dl = (l - center) * (l - center);
            decay[(size_t)k * N + l] = std::pow(rho, std::sqrt(dk + dl));
        }
    // weights.py:50-56: folded = N/2 - |idx - N/2|; wf = (1 - sqrt2*sqrt(nk + nl))^2, >= 0
    std::vector<double> norm(N);
    for (int k = 0; k < N; ++k) {
        double folded = N / 2.0 - std::fabs(k - N / 2.0);
        norm[k] = folded * folded / (double)(N * N);
    }
    for (int k = 0; k < N; ++k)
        for (int l = 0; l < N; ++l) {
            double inner = 1.0 - std::sqrt(2.0) * std::sqrt(norm[k] + norm[l]);
            double v = inner * inner;
            wf[(size_t)k * N + l] = v > 0.0 ? v : 0.0;
        }
    // twiddles with exact quadrant symmetry
    for (int j = 0; j < N; ++j) {
        long double th = 2.0L * 3.14159265358979323846264338327950288L * (long double)j / N;
        cs[2 * j] = (double)cosl(th);
        cs[2 * j + 1] = (double)sinl(th);
    }
    for (int j = 0; j < N; ++j) {
        int m = (N - j) % N;  // cos(-x) = cos(x), sin(-x) = -sin(x): exact mirror
        if (m < j) {
            cs[2 * j] = cs[2 * m];
            cs[2 * j + 1] = -cs[2 * m + 1];
        }
        if (4 * j == N || 4 * j == 3 * N) cs[2 * j] = 0.0;
        if (2 * j == N) cs[2 * j + 1] = 0.0;
        if (j == 0) cs[1] = 0.0;
    }
}

template <typename Real>
int get_tables(fsr_engine *eng, Device &d, int N, double rho, Tables<Real> &out) {
    auto key = std::make_pair(N, rho);
    auto it = d.tables.find(key);
    if (it == d.tables.end()) {
        std::vector<double> decay, wf, cs;
        host_tables(N, rho, decay, wf, cs);
        auto ts = std::make_unique<TableSet>();
        size_t n = (size_t)N * N, tot = 2 * n + 2 * (size_t)N;
        std::vector<double> all;
        all.insert(all.end(), decay.begin(), decay.end());
        all.insert(all.end(), wf.begin(), wf.end());
        all.insert(all.end(), cs.begin(), cs.end());
        std::vector<float> allf(all.begin(), all.end());
        CUDA_TRY(eng, ts->f64.ensure(tot * sizeof(double)));
        CUDA_TRY(eng, ts->f32.ensure(tot * sizeof(float)));
        CUDA_TRY(eng, cudaMemcpy(ts->f64.p, all.data(), tot * sizeof(double), cudaMemcpyHostToDevice));
        CUDA_TRY(eng, cudaMemcpy(ts->f32.p, allf.data(), tot * sizeof(float), cudaMemcpyHostToDevice));
        it = d.tables.emplace(key, std::move(ts)).first;
    }
    const size_t n = (size_t)N * N;
    const Real *base = sizeof(Real) == 8 ? (const Real *)it->second->f64.p : (const Real *)it->second->f32.p;
    out.decay = base;
    out.wf = base + n;
    out.cs = base + 2 * n;
    return FSR_OK;
}

// ------------------------------------------------------------ validation
int validate(const fsr_params *p, char *msg, int len) {
    auto set = [&](const char *m) {
        if (msg && len > 0) snprintf(msg, len, "%s", m);
        return FSR_EINVAL;
    };
    if (!p) return set("null parameters");
    if (p->block < 1) return set("target block size must be at least 1");
    if (p->border < 0) return set("border must be non-negative");
    if (!(p->rho > 0.0 && p->rho < 1.0)) return set("decay factor rho must lie in (0, 1)");
    if (!(p->gamma > 0.0 && p->gamma <= 1.0))
        return set("compensation factor gamma must lie in (0, 1]");
    if (p->iterations < 0) return set("iteration count must be non-negative");
    if (p->reducer != FSR_REDUCER_TREE && p->reducer != FSR_REDUCER_LINEAR)
        return set("unknown argmax strategy, expected one of ('tree', 'linear')");
    if (p->precision < FSR_PREC_FP64 || p->precision > FSR_PREC_FP32_UNGUARDED)
        return set("unknown precision");
    if (p->argmax_impl < FSR_ARGMAX_SHFL || p->argmax_impl > FSR_ARGMAX_REDUX)
        return set("unknown argmax implementation");
    const int64_t s = (int64_t)p->block + 2 * (int64_t)p->border;
    if (s < 2) return set("support must be at least 2");
    if (s > 64) {
        if (msg && len > 0)
            snprintf(msg, len, "support block %lldx%lld exceeds the 64x64 engine limit",
                     (long long)s, (long long)s);
        return FSR_EUNSUPPORTED;
    }
    if (p->reducer == FSR_REDUCER_TREE && s * s > 1024) {
        if (msg && len > 0)
            snprintf(msg, len,
                     "support block %lldx%lld exceeds the 1024-lane reduction capacity",
                     (long long)s, (long long)s);
        return FSR_EINVAL;
    }
    if (!(p->guard_tau >= 0.0 && p->guard_tau < 1.0)) return set("guard_tau must lie in [0, 1)");
    if (!(p->guard_kappa < 1.0)) return set("guard_kappa must be below 1");
    if (p->kernel < 0 || p->kernel > 2) return set("unknown kernel variant");
    return FSR_OK;
}

int check_params(fsr_engine *eng, const fsr_params *p) {
    char msg[256] = {0};
    int rc = validate(p, msg, sizeof msg);
    if (rc != FSR_OK) return fail(eng, rc, "%s", msg);
    return FSR_OK;
}

// One kernel launch through a launcher of fsr_launch.cuh: count it, map errors.
#define LAUNCH_TRY(eng, d, expr)                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ == kNotBuilt) return fail(eng, FSR_EINVAL, "kernel variant not built: %s", #expr); \
        if (e_ != cudaSuccess)                                                                   \
            return fail(eng, FSR_ECUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_),   \
                        __FILE__, __LINE__, #expr);                                              \
        (d).launches++;                                                                          \
    } while (0)

template <typename Real, typename IO>
int launch_generic(fsr_engine *eng, Device &d, const ImageArgs<Real, IO> &a, int grid, cudaStream_t st) {
    LAUNCH_TRY(eng, d, (generic_launch<Real, IO>(a, grid, st)));
    return FSR_OK;
}

// N=32 fp64 kernel: auto/pair = two warps per block (pair64), warp = one (warp64)
template <typename IO>
int launch_fp64_n32(fsr_engine *eng, Device &d, const Pair64Args<IO> &a, const fsr_params *p,
                    int64_t want_blocks, cudaStream_t st) {
    const bool tree = p->reducer == FSR_REDUCER_TREE;
    if (p->kernel != 1)
        LAUNCH_TRY(eng, d, (pair64_launch<IO>(a, tree, p->argmax_impl, want_blocks, d.sms, st)));
    else
        LAUNCH_TRY(eng, d, (warp64_launch<IO>(a, tree, p->argmax_impl, want_blocks, d.sms, st)));
    return FSR_OK;
}

template <typename IO>
int launch_warp16d(fsr_engine *eng, Device &d, const Pair64Args<IO> &a, bool tree, int am,
                   int64_t want_blocks, cudaStream_t st) {
    LAUNCH_TRY(eng, d, (warp16d_launch<IO>(a, tree, am, want_blocks, d.sms, st)));
    return FSR_OK;
}

template <typename IO>
int launch_warpnd(fsr_engine *eng, Device &d, const Pair64Args<IO> &a, int N, int am,
                  int64_t want_blocks, cudaStream_t st) {
    if ((N == 4 || N == 8) && a.B <= 4 && d.segmented)  // 32/N blocks per warp (fsr_warpseg.cuh)
        LAUNCH_TRY(eng, d, (warpsegd_launch<IO>(a, N, want_blocks, d.sms, st)));
    else
        LAUNCH_TRY(eng, d, (warpnd_launch<IO>(a, N, am, want_blocks, d.sms, st)));
    return FSR_OK;
}

template <typename IO>
int launch_cta64d(fsr_engine *eng, Device &d, const Pair64Args<IO> &a, int64_t want_blocks,
                  cudaStream_t st) {
    int grid = 1;
    CUDA_TRY(eng, cta64d_grid<IO>(want_blocks, d.sms, &grid));
    CUDA_TRY(eng, d.c64scratch.ensure((size_t)grid * 4096 * sizeof(double2)));
    Pair64Args<IO> b = a;
    b.scratch = d.c64scratch.as<double2>();
    LAUNCH_TRY(eng, d, (cta64d_launch<IO>(b, grid, st)));
    return FSR_OK;
}

template <typename IO>
Pair64Args<IO> pair64_args(const fsr_params *p, const IO *px, int64_t px_pitch, const uint8_t *mask,
                           int64_t mask_pitch, IO *out, int64_t out_pitch, int64_t H, int64_t W,
                           int64_t bcols, int64_t first, int64_t nblocks, const Tables<double> &tab,
                           int32_t *sel, int32_t *done, unsigned int *empty_count,
                           int32_t *empty_list) {
    Pair64Args<IO> a{};
    a.px = px; a.px_pitch = px_pitch; a.mask = mask; a.mask_pitch = mask_pitch;
    a.out = out; a.out_pitch = out_pitch; a.H = H; a.W = W;
    a.B = p->block; a.L = p->border; a.iterations = p->iterations; a.early_stop = p->early_stop;
    a.bcols = bcols; a.first = first; a.nblocks = nblocks; a.list = nullptr; a.list_count = nullptr;
    a.gamma = p->gamma; a.decay = tab.decay; a.wf = tab.wf; a.sel = sel; a.done = done;
    a.empty_count = empty_count; a.empty_list = empty_list;
    a.tree = p->reducer == FSR_REDUCER_TREE;
    return a;
}

bool pair64_eligible(const fsr_params *p) {
    return p->block + 2 * p->border == 32 && p->block * p->block <= 32;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
// (declared early: warpn launchers below)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// Tensor maps for the fp32-loop kernels' window gather: box_rows-row boxes
// widened to 16-byte aligned starts (TmaBox<IO, ROWS, N> columns), zero fill
// outside the image, for f32 or f64 pixels.  Returns false when TMA cannot
// address the buffers (rows not 16-byte aligned); the kernel then gathers
// with plain loads.
template <typename IO>
bool window_maps(const IO *px, int64_t px_pitch, const uint8_t *mask, int64_t mask_pitch,
                 int64_t H, int64_t W, Warp32Maps *m, int N) {
    const int box_px = N + 16 / (int)sizeof(IO), box_mk = (N + 30) / 16 * 16, box_rows = N;
    if ((reinterpret_cast<uintptr_t>(px) & 15) || ((px_pitch * (int64_t)sizeof(IO)) & 15) ||
        (reinterpret_cast<uintptr_t>(mask) & 15) || (mask_pitch & 15) || H < 1 || W < 1 ||
        H > (int64_t)INT32_MAX || W > (int64_t)INT32_MAX)
        return false;
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    const cuuint32_t bpx[2] = {(cuuint32_t)box_px, (cuuint32_t)box_rows},
                     bmk[2] = {(cuuint32_t)box_mk, (cuuint32_t)box_rows}, estr[2] = {1, 1};
    const cuuint64_t spx[1] = {(cuuint64_t)px_pitch * sizeof(IO)}, smk[1] = {(cuuint64_t)mask_pitch};
    const CUtensorMapDataType dt =
        sizeof(IO) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    if (enc(&m->px, dt, 2, const_cast<IO *>(px), dims, spx, bpx, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(&m->mask, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t *>(mask), dims, smk, bmk, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    return true;
}

bool cta64_eligible(const fsr_params *p) {
    return p->block + 2 * p->border == 64 && p->block * p->block <= C64_THREADS &&
           p->reducer == FSR_REDUCER_LINEAR && p->precision != FSR_PREC_FP64;
}

bool cta64d_eligible(const fsr_params *p) {
    return p->block + 2 * p->border == 64 && p->block * p->block <= C64_THREADS &&
           p->reducer == FSR_REDUCER_LINEAR;
}

// the supports without a dedicated kernel (fsr_warpn.cuh): one warp per block,
// the paper grid's 4, 8, 24 and every other even N up to 20 (not 16)
bool warpn_support(int N) { return N == 24 || (N >= 4 && N <= 20 && N % 2 == 0 && N != 16); }
bool warpnd_eligible(const fsr_params *p) {
    return warpn_support(p->block + 2 * p->border) && p->block * p->block <= 32;
}
bool warpn_eligible(const fsr_params *p) { return warpnd_eligible(p) && p->precision != FSR_PREC_FP64; }

bool warp16d_eligible(const fsr_params *p) {
    return p->block + 2 * p->border == 16 && p->block * p->block <= 32;
}

bool warp16_eligible(const fsr_params *p) {
    const int N = p->block + 2 * p->border;
    return N == 16 && p->block * p->block <= 32 && p->precision != FSR_PREC_FP64;
}

bool warp32_eligible(const fsr_params *p) {
    const int N = p->block + 2 * p->border;
    return N == 32 && p->block * p->block <= 32 && p->precision != FSR_PREC_FP64;
}

// The near-tie guard: a block is re-run in fp64 when some iteration has
//     b1 - b2 <= tau b1 + kappa sqrt(b1 B0)
// (top-2 objectives b1 >= b2, B0 = the block's first maximum).  The fp32
// residual's absolute error follows the largest values it has held (~eps32
// sqrt(B0)), so late iterations, whose b1 lies 1e-7..1e-8 below B0, need the
// scale term: a relative tau alone misses their near-ties (the reference's
// 512^2 KAT at N = 16, I = 200 had a block whose iteration-163 gap was 1.1e-5
// relative but 3e-9 of sqrt(b1 B0)).  Defaults, measured over 17 natural and
// noise frames with tools/flip_errors.py:
//     tau   = 5e-5 * k_N,                 k_N = 2 for N = 64, else 1
//     kappa = 1e-7 * max(0, I / 100 - 1)  (none up to the default 100 iterations)
// and for the small supports N <= 14 (196 bins or fewer: after a few dozen
// iterations every objective lies far below B0, so the scale term would flag
// nearly every block -- 95 % at N = 8, I = 200 -- while tau = 5e-5 misses flips
// at N = 10..14: 0.24-0.42 gray levels):
//     tau   = 2e-4, kappa = 0             (1080p N = 8, I = 100: max 0.09 gray
//                                          levels at 15 % re-runs; I = 200: 0.17;
//                                          N = 10..14: <= 0.15 at 16-18 %)
// An explicit guard_tau > 0 / guard_kappa > 0 is used as given; guard_kappa < 0
// turns the scale term off.
double guard_tau_for(const fsr_params *p) {
    if (p->guard_tau > 0.0) return p->guard_tau;
    const int N = p->block + 2 * p->border;
    return N >= 64 ? 1e-4 : N <= 14 ? 2e-4 : 5e-5;
}

double guard_kappa_for(const fsr_params *p) {
    if (p->guard_kappa > 0.0) return p->guard_kappa;
    if (p->guard_kappa < 0.0) return 0.0;
    if (p->block + 2 * p->border <= 14) return 0.0;
    return 1e-7 * std::max(0.0, p->iterations / 100.0 - 1.0);
}

// Enqueue the image path for target-block rows [row0, row1) on lane d, stream st:
// the main kernel, then (guarded fp32) the fp64 re-run of the flagged blocks.
// px/mask/out are "virtual" row-0 pointers (absolute row y at ptr + y*pitch).
// Empty-support blocks are appended to the call's list (call->empty_count,
// empty_list); the caller fills them once all chunks are done (enqueue_fill or
// on the host).  ev_main0/1 bracket the main kernel.
template <typename IO>
int enqueue_image(fsr_engine *eng, Device &d, const fsr_params *p, const IO *px, int64_t px_pitch,
                  const uint8_t *mask, int64_t mask_pitch, IO *out, int64_t out_pitch, int64_t H,
                  int64_t W, int64_t row0, int64_t row1, int32_t *sel, int32_t *done, cudaStream_t st,
                  ChunkCtr *cc, CallCtr *call, int32_t *empty_list, cudaEvent_t ev_main0,
                  cudaEvent_t ev_main1) {
    const cudaEvent_t ev_end = ev_main1;
    const int N = p->block + 2 * p->border;
    const int64_t bcols = (W + p->block - 1) / p->block;
    const int64_t first = row0 * bcols, nblocks = (row1 - row0) * bcols;
    if (nblocks <= 0) return FSR_OK;
    // Beyond ~300 iterations the guard re-runs most blocks (tau grows with I,
    // tools/guard_check.py: 90-99 % at I = 500), so the guarded fp32 request is
    // served by the fp64 kernels directly -- faster, and exact.
    const fsr_params *p_req = p;
    fsr_params pl = *p;
    // (FSR_FP64_ABOVE: A/B knob.  Re-measured with the replay builds' early exit,
    // 1080p: at I = 400 fp32 + replayed re-runs and fp64 tie within 5 % either way
    // -- N=32 15.1 / 15.1, N=64 3.2 / 3.1, N=16 60 / 69, N=24 21 / 23 fps)
    static const int fp64_above = [] { const char *e = std::getenv("FSR_FP64_ABOVE"); return e ? atoi(e) : 300; }();
    if (pl.precision == FSR_PREC_FP32 && pl.iterations > fp64_above) pl.precision = FSR_PREC_FP64;
    // N = 4 (L = 0 at B = 4: the window is the block) re-runs ~45 % of the blocks,
    // and its segmented fp64 kernel is faster than fp32 + re-runs (1080p: 2226 vs
    // 1702 fps) -- and exact
    if (pl.precision == FSR_PREC_FP32 && N == 4) pl.precision = FSR_PREC_FP64;
    p = &pl;
    CUDA_TRY(eng, cudaMemsetAsync(cc, 0, sizeof(ChunkCtr), st));
    CUDA_TRY(eng, cudaEventRecord(ev_main0, st));
    const bool guarded = p->precision == FSR_PREC_FP32;
    if (guarded) CUDA_TRY(eng, d.rerun_list.ensure((size_t)nblocks * sizeof(int32_t)));
    // replay (N = 16, 32, 64; redux argmax): the fp32 kernel records each flagged block's
    // selections up to its first ambiguous iteration; warp16d / pair64 / cta64d replay them without
    // the objective / argmax, then searches in fp64 from there
    // (the segmented N <= 8 kernel does not record: its re-runs are cheap)
    // From I = 101 on (recording costs the N <= 32 main kernels ~3.6 %, more
    // than the replay saves at I = 100), at any I for N = 64 (recording is free
    // next to its 4096-bin pass; 1080p I=100: 24.4 -> 25.5 fps).
    const bool replay = guarded && (warp32_eligible(p) || warp16_eligible(p) || cta64_eligible(p) ||
                                    (warpn_eligible(p) && N == 24)) &&
                        p->argmax_impl == FSR_ARGMAX_REDUX && d.replay_min_iters > 0 &&
                        (p->iterations >= d.replay_min_iters || (cta64_eligible(p) && d.replay_min_iters <= 101));
    if (replay) {
        CUDA_TRY(eng, d.rerun_kf.ensure((size_t)nblocks * sizeof(int32_t)));
        CUDA_TRY(eng, d.rerun_seq.ensure((size_t)nblocks * p->iterations * sizeof(uint16_t)));
    }
    const int gen_grid = d.sms * 8;
    int rc = FSR_OK;
    // the fp32-loop kernels take f32 or f64 pixels (the reference's own input
    // type); their prologue (gather, weights, FFT, split) runs in fp64 either way
    const bool fast32 = warp32_eligible(p);
    const bool fast16 = warp16_eligible(p);
    const bool fast64 = cta64_eligible(p);
    const bool fastn = warpn_eligible(p);
    d.served_fp64 = p_req->precision == FSR_PREC_FP32 &&
                    (p->precision == FSR_PREC_FP64 || !(fast32 || fast16 || fast64 || fastn));
    if (p->precision == FSR_PREC_FP64 || !(fast32 || fast16 || fast64 || fastn)) {
        if (p->precision == FSR_PREC_FP64 && pair64_eligible(p)) {
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> a = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, first, nblocks, tab, sel, done,
                                               &call->empty_count, empty_list);
            if ((rc = launch_fp64_n32<IO>(eng, d, a, p, nblocks, st))) return rc;
            CUDA_TRY(eng, cudaEventRecord(ev_end, st));
        } else if (p->precision == FSR_PREC_FP64 && warp16d_eligible(p)) {
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> a = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, first, nblocks, tab, sel, done,
                                               &call->empty_count, empty_list);
            if ((rc = launch_warp16d<IO>(eng, d, a, p->reducer == FSR_REDUCER_TREE, p->argmax_impl,
                                         nblocks, st)))
                return rc;
            CUDA_TRY(eng, cudaEventRecord(ev_end, st));
        } else if (p->precision == FSR_PREC_FP64 && cta64d_eligible(p)) {
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> a = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, first, nblocks, tab, sel, done,
                                               &call->empty_count, empty_list);
            if ((rc = launch_cta64d<IO>(eng, d, a, nblocks, st))) return rc;
            CUDA_TRY(eng, cudaEventRecord(ev_end, st));
        } else if (p->precision == FSR_PREC_FP64 && warpnd_eligible(p)) {
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> a = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, first, nblocks, tab, sel, done,
                                               &call->empty_count, empty_list);
            if ((rc = launch_warpnd<IO>(eng, d, a, N, p->argmax_impl, nblocks, st))) return rc;
            CUDA_TRY(eng, cudaEventRecord(ev_end, st));
        } else if (p->precision == FSR_PREC_FP64) {
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            ImageArgs<double, IO> a{px, px_pitch, mask, mask_pitch, out, out_pitch, H, W,
                                    p->block, p->border, N, p->iterations, bcols, first, nblocks,
                                    nullptr, nullptr, p->gamma, p->reducer == FSR_REDUCER_TREE,
                                    p->early_stop, tab, sel, done, &call->empty_count,
                                    empty_list};
            if ((rc = launch_generic(eng, d, a, (int)std::min<int64_t>(nblocks, gen_grid), st))) return rc;
            CUDA_TRY(eng, cudaEventRecord(ev_end, st));
        } else {
            // fp32 on the generic kernel: no near-tie guard there, so a guarded
            // request is served in fp64 (exact) for these supports
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            if (p->precision == FSR_PREC_FP32_UNGUARDED) {
                Tables<float> tf;
                if ((rc = get_tables<float>(eng, d, N, p->rho, tf))) return rc;
                ImageArgs<float, IO> a{px, px_pitch, mask, mask_pitch, out, out_pitch, H, W,
                                       p->block, p->border, N, p->iterations, bcols, first,
                                       nblocks, nullptr, nullptr, (float)p->gamma,
                                       p->reducer == FSR_REDUCER_TREE, p->early_stop, tf, sel,
                                       done, &call->empty_count, empty_list};
                if ((rc = launch_generic(eng, d, a, (int)std::min<int64_t>(nblocks, gen_grid), st))) return rc;
                CUDA_TRY(eng, cudaEventRecord(ev_end, st));
            } else {
                ImageArgs<double, IO> a{px, px_pitch, mask, mask_pitch, out, out_pitch, H, W,
                                        p->block, p->border, N, p->iterations, bcols, first,
                                        nblocks, nullptr, nullptr, p->gamma,
                                        p->reducer == FSR_REDUCER_TREE, p->early_stop, tab, sel,
                                        done, &call->empty_count, empty_list};
                if ((rc = launch_generic(eng, d, a, (int)std::min<int64_t>(nblocks, gen_grid), st))) return rc;
                CUDA_TRY(eng, cudaEventRecord(ev_end, st));
            }
        }
    } else {
        Tables<float> tf;
        if ((rc = get_tables<float>(eng, d, N, p->rho, tf))) return rc;
        Tables<double> td;
        if ((rc = get_tables<double>(eng, d, N, p->rho, td))) return rc;
        Warp32Args a{};
        a.decay64 = td.decay;
        a.px = px;
        a.px_pitch = px_pitch;
        a.mask = mask;
        a.mask_pitch = mask_pitch;
        a.out = out;
        a.out_pitch = out_pitch;
        a.H = H;
        a.W = W;
        a.B = p->block;
        a.L = p->border;
        a.iterations = p->iterations;
        a.early_stop = p->early_stop;
        a.bcols = bcols;
        a.first = first;
        a.nblocks = nblocks;
        a.gamma = (float)p->gamma;
        a.tau = (float)guard_tau_for(p);
        a.omt = 1.f - a.tau;
        a.kappa = (float)guard_kappa_for(p);
        a.tree = p->reducer == FSR_REDUCER_TREE;
        if (replay) {
            a.rerun_kf = d.rerun_kf.as<int32_t>();
            a.rerun_seq = d.rerun_seq.as<uint16_t>();
            a.seq_stride = p->iterations;
        }
        a.wf = tf.wf;
        a.sel = sel;
        a.done = done;
        a.empty_count = &call->empty_count;
        a.empty_list = empty_list;
        a.rerun_count = &cc->rerun_count;
        a.rerun_list = guarded ? d.rerun_list.as<int32_t>() : nullptr;
        a.gap_out = d.gap_debug ? d.gap_debug - 2 * first : nullptr;
        a.key_mask = 0xffffffe0u;
        Warp32Maps maps;
        std::memset(&maps, 0, sizeof(maps));
        // the maps start at the first row this call reads, not at the virtual
        // row-0 pointer: a tensor map's base must be a real address of the
        // buffer (a base below the allocation faults), and zero fill at the
        // map's edges is still exactly the image's edges, because the strip's
        // rows only end early where the image does
        const int64_t ty0 = std::max<int64_t>(0, row0 * p->block - p->border);
        const int64_t ty1 = std::min<int64_t>(H, row1 * p->block + p->border);
        a.tma_y0 = (int)ty0;
        const IO *tpx = px + ty0 * px_pitch;
        const uint8_t *tmk = mask + ty0 * mask_pitch;
        const bool tree = p->reducer == FSR_REDUCER_TREE;
        // trace / early-stop code only in the launches that need it
        const int opts = (sel ? LOPT_TRACE : 0) | (p->early_stop ? LOPT_EARLY : 0) |
                         (guarded && a.kappa > 0.f ? LOPT_KAPPA : 0) | (replay ? LOPT_REPLAY : 0);
        const int nsup = fast64 ? 64 : fast16 ? 16 : fastn ? N : 32;
        a.use_tma = (d.tma_enabled &&
                     window_maps<IO>(tpx, px_pitch, tmk, mask_pitch, ty1 - ty0, W, &maps, nsup)) ? 1 : 0;
        d.used_tma = a.use_tma;
        if (fast64) {
            a.key_mask = 0xffffffc0u;  // 6 rank bits (row u of 64)
            LAUNCH_TRY(eng, d, (cta64_any<IO>(a, maps, p->argmax_impl, guarded, opts, d.sms, st)));
        } else if (fast16) {
            // (warpseg with two blocks per warp measured 8 % slower at N = 16, 1080p:
            // 2.39 vs 2.21 ms; warp16's two lanes per column already issue 70 %)
            LAUNCH_TRY(eng, d, (warp16_any<IO>(a, maps, tree, p->argmax_impl, guarded, opts, d.sms, st)));
        } else if (fastn && (N == 4 || N == 8) && p->block <= 4 && d.segmented) {
            LAUNCH_TRY(eng, d, (warpseg_any<IO>(a, N, guarded, opts, d.sms, st)));
        } else if (fastn) {
            LAUNCH_TRY(eng, d, (warpn_any<IO>(a, maps, N, p->argmax_impl, guarded, opts, d.sms, st)));
        } else {
            const bool study = d.gap_debug != nullptr;
            if (study && p->argmax_impl != FSR_ARGMAX_REDUX)
                return fail(eng, FSR_EINVAL, "guard study needs argmax=redux");
            LAUNCH_TRY(eng, d, (warp32_any<IO>(a, maps, tree, p->argmax_impl, guarded || study, study,
                                               opts, d.sms, st)));
        }
        CUDA_TRY(eng, cudaEventRecord(ev_end, st));
        if (guarded && fast64) {
            // fp64 re-run of ambiguous blocks on the N=64 fp64 kernel (list mode)
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> r = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, 0, 0, tab, sel, done,
                                               &cc->skip_empty /* empties already counted */, nullptr);
            r.list = d.rerun_list.as<int32_t>();
            r.list_count = &cc->rerun_count;
            if (replay) {
                r.list_kf = d.rerun_kf.as<int32_t>();
                r.list_seq = d.rerun_seq.as<uint16_t>();
                r.seq_stride = p->iterations;
            }
            if ((rc = launch_cta64d<IO>(eng, d, r, (int64_t)d.sms, st))) return rc;
        } else if (guarded && fastn) {
            // fp64 re-run of ambiguous blocks on the fp64 one-warp kernel (list mode)
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> r = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, 0, 0, tab, sel, done,
                                               &cc->skip_empty /* empties already counted */, nullptr);
            r.list = d.rerun_list.as<int32_t>();
            r.list_count = &cc->rerun_count;
            if (replay) {
                r.list_kf = d.rerun_kf.as<int32_t>();
                r.list_seq = d.rerun_seq.as<uint16_t>();
                r.seq_stride = p->iterations;
            }
            if ((rc = launch_warpnd<IO>(eng, d, r, N, p->argmax_impl, (int64_t)d.sms * 16, st))) return rc;
        } else if (guarded && fast16) {
            // fp64 re-run of ambiguous blocks on the N=16 fp64 register kernel (list mode)
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> r = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, 0, 0, tab, sel, done,
                                               &cc->skip_empty /* empties already counted */, nullptr);
            r.list = d.rerun_list.as<int32_t>();
            r.list_count = &cc->rerun_count;
            if (replay) {
                r.list_kf = d.rerun_kf.as<int32_t>();
                r.list_seq = d.rerun_seq.as<uint16_t>();
                r.seq_stride = p->iterations;
            }
            if ((rc = launch_warp16d<IO>(eng, d, r, p->reducer == FSR_REDUCER_TREE, p->argmax_impl,
                                         (int64_t)d.sms * 16, st)))
                return rc;
        } else if (guarded) {
            // fp64 re-run of the blocks whose fp32 greedy decisions were ambiguous
            Tables<double> tab;
            if ((rc = get_tables<double>(eng, d, N, p->rho, tab))) return rc;
            Pair64Args<IO> r = pair64_args<IO>(p, px, px_pitch, mask, mask_pitch, out, out_pitch, H,
                                               W, bcols, 0, 0, tab, sel, done,
                                               &cc->skip_empty /* empties already counted */, nullptr);
            r.list = d.rerun_list.as<int32_t>();
            r.list_count = &cc->rerun_count;
            if (replay) {
                r.list_kf = d.rerun_kf.as<int32_t>();
                r.list_seq = d.rerun_seq.as<uint16_t>();
                r.seq_stride = p->iterations;
            }
            if ((rc = launch_fp64_n32<IO>(eng, d, r, p, (int64_t)d.sms * 16, st))) return rc;
        }
    }
    return FSR_OK;
}

// Empty-support fallback for a whole call (reconstruction.py:236-237, 272-275),
// enqueued after every chunk: the listed blocks get `fill`, or (fill = NaN) the
// mean of the known samples of rows [0, H) of px/mask, summed on the device in
// a fixed order (deterministic).  Both kernels return at once when no block was
// empty; an empty block without any known sample sets call->status = 2.
template <typename IO>
int enqueue_fill(fsr_engine *eng, Device &d, const IO *px, int64_t px_pitch, const uint8_t *mask,
                 int64_t mask_pitch, IO *out, int64_t out_pitch, int64_t H, int64_t W, int B,
                 CallCtr *call, const int32_t *list, double fill, cudaStream_t st) {
    const int64_t bcols = (W + B - 1) / B;
    const double2 *parts = nullptr;
    int nparts = 0;
    if (fill != fill) {
        nparts = d.sms * 2;
        CUDA_TRY(eng, d.fill_partials.ensure((size_t)nparts * sizeof(double2)));
        mean_partial_kernel<IO><<<nparts, 256, 0, st>>>(px, px_pitch, mask, mask_pitch, H, W,
                                                         &call->empty_count,
                                                         d.fill_partials.as<double2>());
        CUDA_TRY(eng, cudaGetLastError());
        d.launches++;
        parts = d.fill_partials.as<double2>();
    }
    fill_empty_kernel<IO><<<d.sms, 128, 0, st>>>(out, out_pitch, H, W, B, bcols, list,
                                                 &call->empty_count, parts, nparts, fill,
                                                 &call->status);
    CUDA_TRY(eng, cudaGetLastError());
    d.launches++;
    return FSR_OK;
}

int select_device(fsr_engine *eng, Device &d) {
    CUDA_TRY(eng, cudaSetDevice(d.id));
    return FSR_OK;
}

// Calls run in K row chunks alternating over kLanes lanes (same GPU, own
// stream, staging and scratch): one chunk's copies, fp64 re-run and launch tail
// overlap the other chunks' main kernels.  K = block_rows / 40, at least 3 for
// any call of 24 block rows or more (so a 4K strip at 8 GPUs, 67 rows, still
// overlaps its re-run) and at most 12.
int chunk_count(const Device &d, int64_t block_rows) {
#ifndef FSR_CHUNK_ROWS
#define FSR_CHUNK_ROWS 40  // block rows per chunk (at least); 1080p: 40 rows is +0.5-1 % over 64
#endif
#ifndef FSR_MAX_CHUNKS
#define FSR_MAX_CHUNKS 12  // 4K (540 block rows): 12 chunks (e2e: 4 -> 8 +0.4 %, 8 -> 12 +0.2 %)
#endif
#ifndef FSR_MIN_CHUNKS
#define FSR_MIN_CHUNKS 3
#endif
    if (d.gap_debug || !d.chunking || block_rows < 8 * FSR_MIN_CHUNKS) return 1;
    static const int max_chunks = [] {  // FSR_MAX_CHUNKS_RT: run-time A/B knob (<= 16)
        const char *e = std::getenv("FSR_MAX_CHUNKS_RT");
        const int n = e ? atoi(e) : FSR_MAX_CHUNKS;
        return n < 1 ? 1 : n > 16 ? 16 : n;
    }();
    return (int)std::min<int64_t>(max_chunks,
                                  std::max<int64_t>(FSR_MIN_CHUNKS, block_rows / FSR_CHUNK_ROWS));
}

#ifndef FSR_LANES
#define FSR_LANES 8  // one stream per chunk at 4K (2 lanes: e2e 37.6, 4: 38.2, 8: 38.4 fps; device 38.8)
#endif
// streams a chunked call alternates over (FSR_LANES_RT: run-time A/B knob, 1..16)
static const int kLanes = [] {
    const char *e = std::getenv("FSR_LANES_RT");
    const int n = e ? atoi(e) : FSR_LANES;
    return n < 1 ? 1 : n > 16 ? 16 : n;
}();

#ifndef FSR_STAGE_THREADS
#define FSR_STAGE_THREADS 4  // host threads per device for the staging copies (incl. the caller)
#endif

int ensure_lanes(fsr_engine *eng, Device &d) {
    while ((int)d.lanes.size() < kLanes) {
        auto ln = std::make_unique<Device>();
        ln->id = d.id;
        ln->sms = d.sms;
        ln->tma_enabled = d.tma_enabled;
        ln->segmented = d.segmented;
        ln->replay_min_iters = d.replay_min_iters;
        CUDA_TRY(eng, cudaStreamCreateWithFlags(&ln->stream, cudaStreamNonBlocking));
        CUDA_TRY(eng, cudaEventCreateWithFlags(&ln->ev0, cudaEventDisableTiming));
        CUDA_TRY(eng, cudaEventCreate(&ln->ev1));
        d.lanes.push_back(std::move(ln));
    }
    for (int c = 0; c < 16; ++c)
        if (!d.ck0[c]) {
            CUDA_TRY(eng, cudaEventCreate(&d.ck0[c]));
            CUDA_TRY(eng, cudaEventCreate(&d.ck1[c]));
            CUDA_TRY(eng, cudaEventCreate(&d.ck2[c]));
        }
    return FSR_OK;
}

// FSR_CHUNK_TRACE: print each chunk's main-kernel bracket and end of work (stderr)
static bool chunk_trace() {
    static const bool t = std::getenv("FSR_CHUNK_TRACE") != nullptr;
    return t;
}

// Chunk c of K over block rows [row0, row1)
inline void chunk_rows(int64_t row0, int64_t row1, int c, int K, int64_t &r0, int64_t &r1) {
    r0 = row0 + (row1 - row0) * c / K;
    r1 = row0 + (row1 - row0) * (c + 1) / K;
}

// Per-call scratch of device d: the call counter, K chunk counters and the empty
// list (capacity nb blocks), zeroed on d.stream after the engine's previous call.
int begin_call(fsr_engine *eng, Device &d, int K, int64_t nb, cudaStream_t st) {
    CUDA_TRY(eng, d.call_ctr.ensure(sizeof(CallCtr)));
    CUDA_TRY(eng, d.chunk_ctrs.ensure((size_t)std::max(K, 1) * sizeof(ChunkCtr)));
    CUDA_TRY(eng, d.empty_list.ensure((size_t)std::max<int64_t>(nb, 1) * sizeof(int32_t)));
    // calls on one engine are serialised: the scratch above is reused by the next call
    CUDA_TRY(eng, cudaStreamWaitEvent(st, d.ev_done, 0));
    CUDA_TRY(eng, cudaMemsetAsync(d.call_ctr.p, 0, sizeof(CallCtr), st));
    CUDA_TRY(eng, cudaEventRecord(d.ev0, st));
    d.launches = 0;
    d.last_chunks = K;
    return FSR_OK;
}

// Kernel-side statistics of the last call on device d (waits for it).
int read_call_stats(fsr_engine *eng, Device &d, CallCtr &call, int64_t &reruns, float &ms, float &main_ms) {
    CUDA_TRY(eng, cudaEventSynchronize(d.ev1));
    ms = 0.f;
    main_ms = 0.f;
    if (cudaEventElapsedTime(&ms, d.ev0, d.ev1) != cudaSuccess) ms = 0.f;
    const bool trace = chunk_trace();  // pipeline timeline (stderr)
    for (int c = 0; c < d.last_chunks; ++c) {  // the chunks' main-kernel brackets
        float t = 0.f;
        if (cudaEventElapsedTime(&t, d.ck0[c], d.ck1[c]) == cudaSuccess) main_ms += t;
        if (trace) {
            float t0 = 0.f, t1 = 0.f, t2 = 0.f;
            cudaEventElapsedTime(&t0, d.ev0, d.ck0[c]);
            cudaEventElapsedTime(&t1, d.ev0, d.ck1[c]);
            cudaEventElapsedTime(&t2, d.ev0, d.ck2[c]);
            fprintf(stderr, "chunk %2d: main kernel %7.3f .. %7.3f ms, work done %7.3f ms\n", c, t0, t1, t2);
        }
    }
    if (trace) fprintf(stderr, "call: %.3f ms\n", ms);
    (void)cudaGetLastError();
    CUDA_TRY(eng, cudaMemcpy(&call, d.call_ctr.p, sizeof(CallCtr), cudaMemcpyDeviceToHost));
    std::vector<ChunkCtr> cc(std::max(d.last_chunks, 1));
    CUDA_TRY(eng, cudaMemcpy(cc.data(), d.chunk_ctrs.p, cc.size() * sizeof(ChunkCtr),
                             cudaMemcpyDeviceToHost));
    reruns = 0;
    for (const ChunkCtr &c : cc) reruns += c.rerun_count;
    return FSR_OK;
}

// Device-resident call on device d, asynchronous on st: K chunks forked onto the
// lanes from st and joined back into it, then the empty-support fill.
template <typename IO>
int device_call(fsr_engine *eng, Device &d, const fsr_params *p, const IO *d_px, int64_t px_pitch,
                const uint8_t *d_mask, int64_t mask_pitch, int64_t H, int64_t W, int64_t row0,
                int64_t row1, IO *d_out, int64_t out_pitch, double fill, cudaStream_t st) {
    const int64_t bcols = (W + p->block - 1) / p->block;
    const int K = chunk_count(d, row1 - row0);
    int rc = ensure_lanes(eng, d);
    if (rc) return rc;
    if ((rc = begin_call(eng, d, K, (row1 - row0) * bcols, st))) return rc;
    CallCtr *call = d.call_ctr.as<CallCtr>();
    const int nl = std::min(K, kLanes);
    for (int l = 0; l < nl; ++l) {
        d.lanes[l]->launches = 0;
        d.lanes[l]->gap_debug = d.gap_debug;
        CUDA_TRY(eng, cudaStreamWaitEvent(d.lanes[l]->stream, d.ev0, 0));
    }
    for (int c = 0; c < K; ++c) {
        Device &ld = *d.lanes[c % kLanes];
        int64_t r0, r1;
        chunk_rows(row0, row1, c, K, r0, r1);
        rc = enqueue_image<IO>(eng, ld, p, d_px, px_pitch, d_mask, mask_pitch, d_out, out_pitch, H, W,
                               r0, r1, nullptr, nullptr, ld.stream, d.chunk_ctrs.as<ChunkCtr>() + c,
                               call, d.empty_list.as<int32_t>(), d.ck0[c], d.ck1[c]);
        if (rc) return rc;
        if (chunk_trace()) CUDA_TRY(eng, cudaEventRecord(d.ck2[c], ld.stream));
        d.used_tma = ld.used_tma;
        d.served_fp64 = ld.served_fp64;
    }
    for (int l = 0; l < nl; ++l) {
        Device &ld = *d.lanes[l];
        d.launches += ld.launches;
        CUDA_TRY(eng, cudaEventRecord(ld.ev1, ld.stream));
        CUDA_TRY(eng, cudaStreamWaitEvent(st, ld.ev1, 0));
    }
    if ((rc = enqueue_fill<IO>(eng, d, d_px, px_pitch, d_mask, mask_pitch, d_out, out_pitch, H, W,
                               p->block, call, d.empty_list.as<int32_t>(), fill, st)))
        return rc;
    CUDA_TRY(eng, cudaEventRecord(d.ev1, st));
    CUDA_TRY(eng, cudaEventRecord(d.ev_done, st));
    return FSR_OK;
}

// Result of one device's share of a host-buffer call.
struct HostPart {
    int64_t row0 = 0, row1 = 0;
    int rc = FSR_OK;
    CallCtr call{};
    int64_t reruns = 0;
    float ms = 0.f, main_ms = 0.f;
    std::vector<int32_t> empty;  // empty-support block ids (host fill)
};

// One device's strip of a host-buffer call, run by its own host thread when the
// engine has several devices.  Chunk c goes to lane c % kLanes: its pixel and
// mask rows (strip + halo) are copied by the staging pool into the lane's pinned
// buffer, sent H2D, reconstructed, and its output rows come back D2H into pinned
// staging, copied to the caller's buffer once the lane is reused or the call
// drains -- so the caller's pageable buffers never block the pipeline.
template <typename IO>
int host_strip(fsr_engine *eng, Device &d, const fsr_params *p, const IO *px, const uint8_t *mask,
               int64_t H, int64_t W, IO *out, int32_t *sel, int32_t *done, HostPart &hp) {
    const int B = p->block, L = p->border;
    const int64_t bcols = (W + B - 1) / B, rows = hp.row1 - hp.row0;
    const int64_t it_stride = std::max(p->iterations, 1);
    int rc = select_device(eng, d);
    if (rc) return rc;
    if (!d.pool) {
        const char *st_env = std::getenv("FSR_STAGE_THREADS");  // A/B knob
        const int nt = st_env ? std::max(1, atoi(st_env)) : FSR_STAGE_THREADS;
        d.pool = std::make_unique<Pool>(nt - 1);
    }
    const int K = chunk_count(d, rows);
    if ((rc = ensure_lanes(eng, d))) return rc;
    if ((rc = begin_call(eng, d, K, rows * bcols, d.stream))) return rc;
    CallCtr *call = d.call_ctr.as<CallCtr>();
    const int nl = std::min(K, kLanes);
    for (int l = 0; l < nl; ++l) {
        Device &ld = *d.lanes[l];
        ld.launches = 0;
        ld.pending = false;
        ld.gap_debug = d.gap_debug;
        CUDA_TRY(eng, cudaStreamWaitEvent(ld.stream, d.ev0, 0));
    }
    // Finished chunks are copied to the caller's buffer in chunk (= completion)
    // order: the persistent grids of the lanes' kernels run nearly one after the
    // other, so chunk c's copy-out overlaps chunks c+1.. on the GPU and only the
    // last chunk's is exposed.
    // page-locked caller buffers (cudaHostAlloc / fsr_pin_host) are DMA'd directly:
    // no staging copy of the input, no copy-out of the result
    auto locked = [](const void *p, size_t bytes) {
        auto one = [](const void *q) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
                (void)cudaGetLastError();
                return false;
            }
            return at.type == cudaMemoryTypeHost;
        };
        return bytes > 0 && one(p) && one(static_cast<const char *>(p) + bytes - 1);
    };
    const int64_t ya_all = std::max<int64_t>(0, hp.row0 * B - L), yb_all = std::min<int64_t>(H, hp.row1 * B + L);
    const int64_t oa_all = std::min<int64_t>(H, hp.row0 * B), ob_all = std::min<int64_t>(H, hp.row1 * B);
    const bool direct_in = locked(px + ya_all * W, (size_t)(yb_all - ya_all) * W * sizeof(IO)) &&
                           locked(mask + ya_all * W, (size_t)(yb_all - ya_all) * W);
    const bool direct_out = locked(out + oa_all * W, (size_t)(ob_all - oa_all) * W * sizeof(IO));
    std::deque<Device *> fifo;  // lanes with a pending chunk, oldest first
    // FSR_HOST_TRACE: host-side timeline of the call (stderr, ms since entry)
    static const bool htrace = std::getenv("FSR_HOST_TRACE") != nullptr;
    const auto t_entry = std::chrono::steady_clock::now();
    auto ms_now = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry).count();
    };
    auto drain_one = [&]() -> int {  // the oldest pending chunk -> caller's buffer
        Device &ld = *fifo.front();
        fifo.pop_front();
        const double t0 = htrace ? ms_now() : 0.0;
        CUDA_TRY(eng, cudaEventSynchronize(ld.ev1));
        const double t1 = htrace ? ms_now() : 0.0;
        if (!direct_out)
            pool_copy(d.pool.get(), out + ld.pend_oa * W, ld.hout.p, ld.pend_ob - ld.pend_oa,
                      (size_t)W * sizeof(IO));
        if (htrace)
            fprintf(stderr, "host: drain rows %lld..%lld wait %.3f..%.3f copy-out ..%.3f ms\n",
                    (long long)ld.pend_oa, (long long)ld.pend_ob, t0, t1, ms_now());
        ld.pending = false;
        return FSR_OK;
    };
    for (int c = 0; c < K; ++c) {
        Device &ld = *d.lanes[c % kLanes];
        while (ld.pending)
            if ((rc = drain_one())) return rc;
        int64_t r0, r1;
        chunk_rows(hp.row0, hp.row1, c, K, r0, r1);  // (half-size first/last chunks: measured no gain)
        const int64_t ya = std::max<int64_t>(0, r0 * B - L), yb = std::min<int64_t>(H, r1 * B + L);
        const int64_t oa = std::min<int64_t>(H, r0 * B), ob = std::min<int64_t>(H, r1 * B);
        const int64_t rows_in = yb - ya, rows_out = ob - oa, nb = (r1 - r0) * bcols;
        const size_t px_bytes = (size_t)rows_in * W * sizeof(IO), mk_bytes = (size_t)rows_in * W;
        CUDA_TRY(eng, ld.px.ensure(px_bytes));
        CUDA_TRY(eng, ld.mask.ensure(mk_bytes));
        CUDA_TRY(eng, ld.out.ensure((size_t)rows_out * W * sizeof(IO)));
        if (!direct_in) CUDA_TRY(eng, ld.hin.ensure(px_bytes + mk_bytes));
        if (!direct_out) CUDA_TRY(eng, ld.hout.ensure((size_t)rows_out * W * sizeof(IO)));
        if (sel) CUDA_TRY(eng, ld.sel.ensure((size_t)nb * it_stride * sizeof(int32_t)));
        if (done) CUDA_TRY(eng, ld.done.ensure((size_t)nb * sizeof(int32_t)));
        const double ts0 = htrace ? ms_now() : 0.0;
        const void *src_px = px + ya * W, *src_mk = mask + ya * W;
        if (!direct_in) {
            pool_copy(d.pool.get(), ld.hin.p, px + ya * W, rows_in, (size_t)W * sizeof(IO));
            pool_copy(d.pool.get(), ld.hin.as<char>() + px_bytes, mask + ya * W, rows_in, (size_t)W);
            src_px = ld.hin.p;
            src_mk = ld.hin.as<char>() + px_bytes;
        }
        if (htrace) fprintf(stderr, "host: chunk %d staged %.3f..%.3f ms\n", c, ts0, ms_now());
        CUDA_TRY(eng, cudaMemcpyAsync(ld.px.p, src_px, px_bytes, cudaMemcpyHostToDevice, ld.stream));
        CUDA_TRY(eng, cudaMemcpyAsync(ld.mask.p, src_mk, mk_bytes, cudaMemcpyHostToDevice, ld.stream));
        const IO *vpx = ld.px.as<IO>() - ya * W;
        const uint8_t *vmask = ld.mask.as<uint8_t>() - ya * W;
        IO *vout = ld.out.as<IO>() - oa * W;
        int32_t *vsel = sel ? ld.sel.as<int32_t>() - r0 * bcols * it_stride : nullptr;
        int32_t *vdone = done ? ld.done.as<int32_t>() - r0 * bcols : nullptr;
        rc = enqueue_image<IO>(eng, ld, p, vpx, W, vmask, W, vout, W, H, W, r0, r1, vsel, vdone,
                               ld.stream, d.chunk_ctrs.as<ChunkCtr>() + c, call,
                               d.empty_list.as<int32_t>(), d.ck0[c], d.ck1[c]);
        if (rc) return rc;
        if (chunk_trace()) CUDA_TRY(eng, cudaEventRecord(d.ck2[c], ld.stream));
        CUDA_TRY(eng, cudaMemcpyAsync(direct_out ? (void *)(out + oa * W) : ld.hout.p, ld.out.p,
                                      (size_t)rows_out * W * sizeof(IO), cudaMemcpyDeviceToHost,
                                      ld.stream));
        // traces (validation only) go straight to the caller's buffers
        if (sel)
            CUDA_TRY(eng, cudaMemcpyAsync(sel + r0 * bcols * it_stride, ld.sel.p,
                                          (size_t)nb * it_stride * sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, ld.stream));
        if (done)
            CUDA_TRY(eng, cudaMemcpyAsync(done + r0 * bcols, ld.done.p, (size_t)nb * sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, ld.stream));
        CUDA_TRY(eng, cudaEventRecord(ld.ev1, ld.stream));
        ld.pending = true;
        ld.pend_oa = oa;
        ld.pend_ob = ob;
        fifo.push_back(&ld);
        d.used_tma = ld.used_tma;
        d.served_fp64 = ld.served_fp64;
    }
    if (htrace) fprintf(stderr, "host: all chunks enqueued %.3f ms\n", ms_now());
    while (!fifo.empty())
        if ((rc = drain_one())) return rc;
    if (htrace) fprintf(stderr, "host: drained %.3f ms\n", ms_now());
    for (int l = 0; l < nl; ++l) {
        Device &ld = *d.lanes[l];
        d.launches += ld.launches;
        CUDA_TRY(eng, cudaStreamWaitEvent(d.stream, ld.ev1, 0));
    }
    CUDA_TRY(eng, cudaEventRecord(d.ev1, d.stream));
    CUDA_TRY(eng, cudaEventRecord(d.ev_done, d.stream));
    if ((rc = read_call_stats(eng, d, hp.call, hp.reruns, hp.ms, hp.main_ms))) return rc;
    if (hp.call.empty_count > 0) {
        hp.empty.resize(hp.call.empty_count);
        CUDA_TRY(eng, cudaMemcpy(hp.empty.data(), d.empty_list.p, hp.empty.size() * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost));
    }
    return FSR_OK;
}

// Host-buffer whole-image call: block rows [rbeg, rend) split into contiguous
// strips over the engine's first max_devs devices, each run by host_strip
// (concurrently, one host thread per device).  Empty-support blocks get
// `fill`, or (fill = NaN) the mean of the known samples of the caller's full
// image (reconstruction.py:236-237; "no known samples" if there is none).
// [a, a + an) and [b, b + bn) share a byte (the output must never alias an input:
// chunks write rows that later chunks' halos still read)
bool overlaps(const void *a, size_t an, const void *b, size_t bn) {
    const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return an > 0 && bn > 0 && x < y + bn && y < x + an;
}

template <typename IO>
int reconstruct_host(fsr_engine *eng, const fsr_params *p, const IO *px, const uint8_t *mask,
                     int64_t H, int64_t W, IO *out, int32_t *sel, int32_t *done,
                     int64_t rbeg = 0, int64_t rend = -1, double fill = NAN, int max_devs = 0) {
    if (!eng) return fail(nullptr, FSR_EINVAL, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    int rc = check_params(eng, p);
    if (rc) return rc;
    if (H < 1 || W < 1) return fail(eng, FSR_EINVAL, "image must have at least one pixel");
    if (!px || !mask || !out) return fail(eng, FSR_EINVAL, "null image buffer");
    {
        const size_t n = (size_t)H * (size_t)W;
        if (overlaps(out, n * sizeof(IO), px, n * sizeof(IO)) || overlaps(out, n * sizeof(IO), mask, n))
            return fail(eng, FSR_EINVAL, "output buffer overlaps an input buffer");
    }
    const int B = p->block;
    const int64_t brows_all = (H + B - 1) / B, bcols = (W + B - 1) / B;
    if (rend < 0) rend = brows_all;
    if (rbeg < 0 || rend > brows_all || rbeg > rend)
        return fail(eng, FSR_EINVAL, "block-row range out of bounds");
    const int64_t brows = rend - rbeg;
    const int nd = max_devs > 0 ? std::min<int>(max_devs, (int)eng->devs.size()) : (int)eng->devs.size();
    eng->stats = fsr_stats{};
    eng->device_stats_pending = false;
    eng->stats.blocks = brows * bcols;
    std::vector<HostPart> parts(nd);
    for (int g = 0; g < nd; ++g) {
        parts[g].row0 = rbeg + brows * g / nd;
        parts[g].row1 = rbeg + brows * (g + 1) / nd;
    }
    auto run = [&](int g) {
        if (parts[g].row1 > parts[g].row0)
            parts[g].rc = host_strip<IO>(eng, *eng->devs[g], p, px, mask, H, W, out, sel, done, parts[g]);
    };
    int busy = 0;
    for (int g = 0; g < nd; ++g) busy += parts[g].row1 > parts[g].row0;
    if (busy <= 1) {
        for (int g = 0; g < nd; ++g) run(g);
    } else {
        std::vector<std::thread> th;
        for (int g = 0; g < nd; ++g) th.emplace_back(run, g);
        for (auto &t : th) t.join();
    }
    for (int g = 0; g < nd; ++g)
        if (parts[g].rc) return parts[g].rc;  // eng->err holds the message
    int64_t empty_total = 0;
    for (int g = 0; g < nd; ++g) {
        const HostPart &hp = parts[g];
        empty_total += hp.call.empty_count;
        eng->stats.rerun_blocks += hp.reruns;
        eng->stats.kernel_launches += eng->devs[g]->launches;
        if (g == 0) {
            eng->stats.flags = (eng->devs[0]->used_tma ? FSR_STATS_TMA_GATHER : 0) |
                               (eng->devs[0]->served_fp64 ? FSR_STATS_SERVED_FP64 : 0);
            eng->stats.kernel_ms = hp.ms;
            eng->stats.main_ms = hp.main_ms;
        }
    }
    eng->stats.empty_blocks = empty_total;
    if (empty_total > 0) {
        // reconstruction.py:236-237, 272-275
        if (fill != fill) {
            double s = 0.0;
            int64_t known = 0;
            for (int64_t i = 0; i < H * W; ++i)
                if (mask[i]) {
                    s += (double)px[i];
                    ++known;
                }
            if (known == 0) return fail(eng, FSR_ENOSAMPLES, "no known samples");
            fill = s / (double)known;
        }
        for (const HostPart &hp : parts)
            for (int32_t bid : hp.empty) {
                const int64_t r0 = (bid / bcols) * B, c0 = (bid % bcols) * B;
                for (int64_t y = r0; y < std::min<int64_t>(H, r0 + B); ++y)
                    for (int64_t x = c0; x < std::min<int64_t>(W, c0 + B); ++x) out[y * W + x] = (IO)fill;
            }
    }
    return FSR_OK;
}

template <typename IO>
int reconstruct_device(fsr_engine *eng, const fsr_params *p, const IO *d_px, int64_t px_pitch,
                       const uint8_t *d_mask, int64_t mask_pitch, int64_t height, int64_t width,
                       int64_t row0, int64_t row1, IO *d_out, int64_t out_pitch, double fill,
                       void *stream) {
    if (!eng) return fail(nullptr, FSR_EINVAL, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    int rc = check_params(eng, p);
    if (rc) return rc;
    if (height < 1 || width < 1) return fail(eng, FSR_EINVAL, "image must have at least one pixel");
    if (!d_px || !d_mask || !d_out) return fail(eng, FSR_EINVAL, "null image buffer");
    if (px_pitch < width || mask_pitch < width || out_pitch < width)
        return fail(eng, FSR_EINVAL, "row pitch smaller than the width");
    {
        const size_t npx = (size_t)((height - 1) * px_pitch + width) * sizeof(IO);
        const size_t nmk = (size_t)((height - 1) * mask_pitch + width);
        const size_t nout = (size_t)((height - 1) * out_pitch + width) * sizeof(IO);
        if (overlaps(d_out, nout, d_px, npx) || overlaps(d_out, nout, d_mask, nmk))
            return fail(eng, FSR_EINVAL, "output buffer overlaps an input buffer");
    }
    const int64_t brows = (height + p->block - 1) / p->block;
    if (row0 < 0 || row1 > brows || row0 > row1) return fail(eng, FSR_EINVAL, "block-row range out of bounds");
    Device &d = *eng->devs[0];
    if ((rc = select_device(eng, d))) return rc;
    rc = device_call<IO>(eng, d, p, d_px, px_pitch, d_mask, mask_pitch, height, width, row0, row1,
                         d_out, out_pitch, fill, (cudaStream_t)stream);
    eng->stats = fsr_stats{};
    eng->stats.blocks = (row1 - row0) * ((width + p->block - 1) / p->block);
    eng->stats.kernel_launches = d.launches;
    eng->stats.flags = (d.used_tma ? FSR_STATS_TMA_GATHER : 0) | (d.served_fp64 ? FSR_STATS_SERVED_FP64 : 0);
    eng->device_stats_pending = rc == FSR_OK;
    return rc;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

void fsr_params_init(fsr_params *p) {
    if (!p) return;
    std::memset(p, 0, sizeof *p);
    p->block = 4;
    p->border = 14;
    p->iterations = 100;
    p->reducer = FSR_REDUCER_TREE;
    p->early_stop = 0;
    p->precision = FSR_PREC_FP64;
    p->argmax_impl = FSR_ARGMAX_REDUX;  // bitwise-identical to shfl/smem, fastest on B200
    p->rho = 0.7;
    p->gamma = 0.5;
    p->guard_tau = 0.0;    // auto: guard_tau_for(p)
    p->guard_kappa = 0.0;  // auto: guard_kappa_for(p)
}

int fsr_params_validate(const fsr_params *p, char *msg, int msg_len) {
    return validate(p, msg, msg_len);
}

int32_t fsr_abi_version(void) { return FSR_ABI_VERSION; }

int fsr_pin_host(void *p, size_t bytes) {
    if (!p || bytes == 0) return FSR_EINVAL;
    if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) != cudaSuccess) {
        (void)cudaGetLastError();
        return FSR_ECUDA;
    }
    return FSR_OK;
}

int fsr_unpin_host(void *p) {
    if (!p) return FSR_EINVAL;
    if (cudaHostUnregister(p) != cudaSuccess) {
        (void)cudaGetLastError();
        return FSR_ECUDA;
    }
    return FSR_OK;
}

const char *fsr_status_string(int status) {
    switch (status) {
        case FSR_OK: return "ok";
        case FSR_EINVAL: return "invalid argument";
        case FSR_ENOSAMPLES: return "no known samples";
        case FSR_ECUDA: return "CUDA error";
        case FSR_EUNSUPPORTED: return "unsupported";
        default: return "unknown status";
    }
}

const char *fsr_last_error(const fsr_engine *eng) {
    return eng ? eng->err.c_str() : g_err.c_str();
}

int fsr_engine_create(const int32_t *devices, int32_t n_devices, fsr_engine **out) {
    if (!out) return fail(nullptr, FSR_EINVAL, "null output pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count < 1)
        return fail(nullptr, FSR_ECUDA, "no CUDA device available (%s); libfsr has no CPU fallback",
                    cudaGetErrorString(e));
    auto eng = std::make_unique<fsr_engine>();
    std::vector<int> ids;
    if (!devices || n_devices <= 0) ids.push_back(0);
    else ids.assign(devices, devices + n_devices);
    for (int id : ids) {
        if (id < 0 || id >= count) return fail(nullptr, FSR_EINVAL, "invalid device id %d", id);
        auto d = std::make_unique<Device>();
        d->id = id;
        CUDA_TRY(nullptr, cudaSetDevice(id));
        cudaDeviceProp prop;
        CUDA_TRY(nullptr, cudaGetDeviceProperties(&prop, id));
        if (prop.major < 10)
            return fail(nullptr, FSR_ECUDA, "device %d is sm_%d%d; libfsr is built for sm_100a",
                        id, prop.major, prop.minor);
        d->sms = prop.multiProcessorCount;
        const char *no_tma = std::getenv("FSR_NO_TMA");  // A/B switch for the TMA window gather
        d->tma_enabled = !(no_tma && *no_tma && *no_tma != '0');
        const char *no_chunk = std::getenv("FSR_NO_CHUNK");  // one launch per call (kernel timing)
        d->chunking = !(no_chunk && *no_chunk && *no_chunk != '0');
        const char *no_seg = std::getenv("FSR_NO_SEG");  // A/B switch for the segmented small-N kernel
        d->segmented = !(no_seg && *no_seg && *no_seg != '0');
        const char *rmin = std::getenv("FSR_REPLAY_MIN");  // A/B: smallest I that replays (0 = never)
        if (rmin && *rmin) d->replay_min_iters = atoi(rmin);
        CUDA_TRY(nullptr, cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
        CUDA_TRY(nullptr, cudaEventCreate(&d->ev0));
        CUDA_TRY(nullptr, cudaEventCreate(&d->ev1));
        CUDA_TRY(nullptr, cudaEventCreateWithFlags(&d->ev_done, cudaEventDisableTiming));
        CUDA_TRY(nullptr, cudaEventRecord(d->ev_done, d->stream));
        eng->devs.push_back(std::move(d));
    }
    *out = eng.release();
    return FSR_OK;
}

void fsr_engine_destroy(fsr_engine *eng) {
    if (!eng) return;
    for (auto &dp : eng->devs) {
        Device &d = *dp;
        cudaSetDevice(d.id);
        cudaStreamSynchronize(d.stream);
        d.pool.reset();
        for (auto &ln : d.lanes) {
            cudaStreamSynchronize(ln->stream);
            for (DevBuf *b : {&ln->px, &ln->mask, &ln->out, &ln->sel, &ln->done, &ln->rerun_list, &ln->rerun_kf, &ln->rerun_seq,
                              &ln->c64scratch})
                b->release();
            ln->hin.release();
            ln->hout.release();
            for (auto &kv : ln->tables) {
                kv.second->f64.release();
                kv.second->f32.release();
            }
            cudaEventDestroy(ln->ev0);
            cudaEventDestroy(ln->ev1);
            cudaStreamDestroy(ln->stream);
        }
        for (DevBuf *b : {&d.px, &d.mask, &d.out, &d.sel, &d.done, &d.empty_list, &d.rerun_list, &d.rerun_kf, &d.rerun_seq,
                          &d.call_ctr, &d.chunk_ctrs, &d.fill_partials, &d.R, &d.G, &d.W, &d.wf,
                          &d.thr, &d.obj, &d.ties, &d.partials, &d.c64scratch})
            b->release();
        for (auto &kv : d.tables) {
            kv.second->f64.release();
            kv.second->f32.release();
        }
        for (int c = 0; c < 16; ++c)
            if (d.ck0[c]) {
                cudaEventDestroy(d.ck0[c]);
                cudaEventDestroy(d.ck1[c]);
                cudaEventDestroy(d.ck2[c]);
            }
        cudaEventDestroy(d.ev0);
        cudaEventDestroy(d.ev1);
        cudaEventDestroy(d.ev_done);
        cudaStreamDestroy(d.stream);
    }
    delete eng;
}

int fsr_reconstruct_f64(fsr_engine *eng, const fsr_params *p, const double *px,
                        const uint8_t *mask, int64_t height, int64_t width, double *out,
                        int32_t *sel, int32_t *done) {
    return reconstruct_host<double>(eng, p, px, mask, height, width, out, sel, done);
}

int fsr_reconstruct_f32(fsr_engine *eng, const fsr_params *p, const float *px,
                        const uint8_t *mask, int64_t height, int64_t width, float *out,
                        int32_t *sel, int32_t *done) {
    return reconstruct_host<float>(eng, p, px, mask, height, width, out, sel, done);
}

int fsr_reconstruct_rows_f32(fsr_engine *eng, const fsr_params *p, const float *px,
                             const uint8_t *mask, int64_t height, int64_t width, int64_t row0,
                             int64_t row1, double fill, float *out) {
    return reconstruct_host<float>(eng, p, px, mask, height, width, out, nullptr, nullptr, row0,
                                   row1, fill);
}

int fsr_reconstruct_rows_f64(fsr_engine *eng, const fsr_params *p, const double *px,
                             const uint8_t *mask, int64_t height, int64_t width, int64_t row0,
                             int64_t row1, double fill, double *out) {
    return reconstruct_host<double>(eng, p, px, mask, height, width, out, nullptr, nullptr, row0,
                                    row1, fill);
}

int fsr_reconstruct_device_f32(fsr_engine *eng, const fsr_params *p, const float *d_px,
                               int64_t px_pitch, const uint8_t *d_mask, int64_t mask_pitch,
                               int64_t height, int64_t width, int64_t row0, int64_t row1,
                               float *d_out, int64_t out_pitch, double fill, void *stream) {
    return reconstruct_device<float>(eng, p, d_px, px_pitch, d_mask, mask_pitch, height, width, row0,
                                     row1, d_out, out_pitch, fill, stream);
}

int fsr_reconstruct_device_f64(fsr_engine *eng, const fsr_params *p, const double *d_px,
                               int64_t px_pitch, const uint8_t *d_mask, int64_t mask_pitch,
                               int64_t height, int64_t width, int64_t row0, int64_t row1,
                               double *d_out, int64_t out_pitch, double fill, void *stream) {
    return reconstruct_device<double>(eng, p, d_px, px_pitch, d_mask, mask_pitch, height, width, row0,
                                      row1, d_out, out_pitch, fill, stream);
}

// Not part of include/fsr.h: development hook for the guard study
// (tools/guard_study.py).  Runs the N=32 fp32 kernel on the first device with
// the top-2 tracking on but no re-run, returning each block's minimum relative
// top-2 gap over its iterations and the first iteration whose gap is below
// guard_tau, plus the selection trace.
int fsr_debug_guard_gaps(fsr_engine *eng, const fsr_params *p_in, const float *px,
                         const uint8_t *mask, int64_t H, int64_t W, float *out, float *gaps,
                         int32_t *sel) {
    if (!eng) return fail(nullptr, FSR_EINVAL, "null engine");
    fsr_params p = *p_in;
    p.precision = FSR_PREC_FP32_UNGUARDED;
    if (!warp32_eligible(&p)) return fail(eng, FSR_EINVAL, "guard study needs N=32, B*B<=32");
    const int64_t nb = ((H + p.block - 1) / p.block) * ((W + p.block - 1) / p.block);
    Device &d = *eng->devs[0];
    int rc = select_device(eng, d);
    if (rc) return rc;
    DevBuf g;
    CUDA_TRY(eng, g.ensure((size_t)nb * 2 * sizeof(float)));
    {
        std::lock_guard<std::mutex> lock(eng->mu);
        d.gap_debug = g.as<float>();
    }
    // first device only (max_devs = 1) and one launch (chunk_count is 1 with
    // gap_debug set), so the gap buffer indexes every block
    rc = reconstruct_host<float>(eng, &p, px, mask, H, W, out, sel, nullptr, 0, -1, NAN, 1);
    {
        std::lock_guard<std::mutex> lock(eng->mu);
        d.gap_debug = nullptr;
    }
    if (rc == FSR_OK)
        CUDA_TRY(eng, cudaMemcpy(gaps, g.p, (size_t)nb * 2 * sizeof(float), cudaMemcpyDeviceToHost));
    g.release();
    return rc;
}

int fsr_last_stats(const fsr_engine *eng_c, fsr_stats *out) {
    if (!eng_c || !out) return FSR_EINVAL;
    fsr_engine *eng = const_cast<fsr_engine *>(eng_c);
    std::lock_guard<std::mutex> lock(eng->mu);
    if (eng->device_stats_pending) {
        // the device-API call was asynchronous: wait for it, then read the counters
        Device &d = *eng->devs[0];
        int rc = select_device(eng, d);
        if (rc) return rc;
        CallCtr call{};
        int64_t reruns = 0;
        float ms = 0.f, mm = 0.f;
        if ((rc = read_call_stats(eng, d, call, reruns, ms, mm))) return rc;
        eng->stats.kernel_ms = ms;
        eng->stats.main_ms = mm;
        eng->stats.rerun_blocks = reruns;
        eng->stats.empty_blocks = call.empty_count;
        eng->device_stats_pending = false;
        *out = eng->stats;
        // the device API's "no known samples" (reconstruction.py:273-274)
        if (call.status == 2) return fail(eng, FSR_ENOSAMPLES, "no known samples");
        return FSR_OK;
    }
    *out = eng->stats;
    return FSR_OK;
}

int fsr_spatial_oracle(fsr_engine *eng, int32_t support, int32_t iterations, double gamma,
                       int64_t count, const double *signal, const uint8_t *mask,
                       const double *spatial, const double *wf, double *out, double *objectives,
                       int32_t *selections, uint8_t *ties, double *energies) {
    if (!eng) return fail(nullptr, FSR_EINVAL, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    if (support < 1 || support > 16)
        return fail(eng, FSR_EUNSUPPORTED, "spatial oracle supports S <= 16 (got %d)", support);
    if (iterations < 0) return fail(eng, FSR_EINVAL, "iteration count must be non-negative");
    if (!(gamma > 0.0 && gamma <= 1.0)) return fail(eng, FSR_EINVAL, "gamma must lie in (0, 1]");
    if (count < 0 || !signal || !mask || !spatial || !wf || !out || !objectives || !selections ||
        !ties || !energies)
        return fail(eng, FSR_EINVAL, "null or empty arrays");
    if (count == 0) return FSR_OK;
    if (count > (int64_t)INT32_MAX) return fail(eng, FSR_EINVAL, "too many blocks");
    Device &d = *eng->devs[0];
    int rc = select_device(eng, d);
    if (rc) return rc;
    const size_t n = (size_t)support * support, it = (size_t)std::max(iterations, 1);
    DevBuf b_sig, b_mask, b_w, b_wf, b_out, b_obj, b_sel, b_ties, b_en;
    auto cleanup = [&]() {
        for (DevBuf *b : {&b_sig, &b_mask, &b_w, &b_wf, &b_out, &b_obj, &b_sel, &b_ties, &b_en})
            b->release();
    };
    auto run = [&]() -> int {
        CUDA_TRY(eng, b_sig.ensure(count * n * sizeof(double)));
        CUDA_TRY(eng, b_mask.ensure(count * n));
        CUDA_TRY(eng, b_w.ensure(count * n * sizeof(double)));
        CUDA_TRY(eng, b_wf.ensure(n * sizeof(double)));
        CUDA_TRY(eng, b_out.ensure(count * n * sizeof(double)));
        CUDA_TRY(eng, b_obj.ensure(count * it * sizeof(double)));
        CUDA_TRY(eng, b_sel.ensure(count * it * sizeof(int32_t)));
        CUDA_TRY(eng, b_ties.ensure(count * it));
        CUDA_TRY(eng, b_en.ensure(count * (it + 1) * sizeof(double)));
        CUDA_TRY(eng, cudaMemcpyAsync(b_sig.p, signal, count * n * sizeof(double), cudaMemcpyHostToDevice, d.stream));
        CUDA_TRY(eng, cudaMemcpyAsync(b_mask.p, mask, count * n, cudaMemcpyHostToDevice, d.stream));
        CUDA_TRY(eng, cudaMemcpyAsync(b_w.p, spatial, count * n * sizeof(double), cudaMemcpyHostToDevice, d.stream));
        CUDA_TRY(eng, cudaMemcpyAsync(b_wf.p, wf, n * sizeof(double), cudaMemcpyHostToDevice, d.stream));
        SpatialArgs a{b_sig.as<double>(), b_mask.as<uint8_t>(), b_w.as<double>(), b_wf.as<double>(),
                      b_out.as<double>(), b_obj.as<double>(), b_sel.as<int32_t>(), b_ties.as<uint8_t>(),
                      b_en.as<double>(), count, support, iterations, gamma};
        spatial_oracle_kernel<<<(unsigned)count, SP_THREADS, 0, d.stream>>>(a);
        CUDA_TRY(eng, cudaGetLastError());
        CUDA_TRY(eng, cudaMemcpyAsync(out, b_out.p, count * n * sizeof(double), cudaMemcpyDeviceToHost, d.stream));
        if (iterations > 0) {
            CUDA_TRY(eng, cudaMemcpyAsync(objectives, b_obj.p, count * iterations * sizeof(double),
                                          cudaMemcpyDeviceToHost, d.stream));
            CUDA_TRY(eng, cudaMemcpyAsync(selections, b_sel.p, count * iterations * sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, d.stream));
            CUDA_TRY(eng, cudaMemcpyAsync(ties, b_ties.p, count * iterations, cudaMemcpyDeviceToHost, d.stream));
        }
        CUDA_TRY(eng, cudaMemcpyAsync(energies, b_en.p, count * (iterations + 1) * sizeof(double),
                                      cudaMemcpyDeviceToHost, d.stream));
        CUDA_TRY(eng, cudaStreamSynchronize(d.stream));
        return FSR_OK;
    };
    rc = run();
    cleanup();
    return rc;
}

int fsr_iterate_spectra(fsr_engine *eng, const fsr_params *p, int64_t count, int32_t N,
                        double *R, double *G, const double *W, const double *wf,
                        const double *thr, int32_t *sel, double *obj, uint8_t *ties,
                        int32_t *done) {
    if (!eng) return fail(nullptr, FSR_EINVAL, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    if (!p) return fail(eng, FSR_EINVAL, "null parameters");
    if (N < 1 || N > 64) return fail(eng, FSR_EUNSUPPORTED, "support %d outside [1, 64]", N);
    if (p->iterations < 0) return fail(eng, FSR_EINVAL, "iteration count must be non-negative");
    if (p->reducer != FSR_REDUCER_TREE && p->reducer != FSR_REDUCER_LINEAR)
        return fail(eng, FSR_EINVAL, "unknown argmax strategy, expected one of ('tree', 'linear')");
    if (p->reducer == FSR_REDUCER_TREE && N * N > 1024)
        return fail(eng, FSR_EINVAL, "record count exceeds two-phase capacity");
    if (count < 0 || !R || !G || !W || !wf) return fail(eng, FSR_EINVAL, "null or empty arrays");
    if (count == 0) return FSR_OK;
    Device &d = *eng->devs[0];
    int rc = select_device(eng, d);
    if (rc) return rc;
    const size_t n = (size_t)N * N, cbytes = (size_t)count * n * 16;
    const int64_t its = std::max(p->iterations, 1);
    CUDA_TRY(eng, d.R.ensure(cbytes));
    CUDA_TRY(eng, d.G.ensure(cbytes));
    CUDA_TRY(eng, d.W.ensure(cbytes));
    CUDA_TRY(eng, d.wf.ensure(n * 8));
    if (thr) CUDA_TRY(eng, d.thr.ensure((size_t)count * 8));
    if (sel) CUDA_TRY(eng, d.sel.ensure((size_t)count * its * 4));
    if (obj) CUDA_TRY(eng, d.obj.ensure((size_t)count * its * 8));
    if (ties) CUDA_TRY(eng, d.ties.ensure((size_t)count * its));
    if (done) CUDA_TRY(eng, d.done.ensure((size_t)count * 4));
    cudaStream_t st = d.stream;
    CUDA_TRY(eng, cudaMemcpyAsync(d.R.p, R, cbytes, cudaMemcpyHostToDevice, st));
    CUDA_TRY(eng, cudaMemcpyAsync(d.G.p, G, cbytes, cudaMemcpyHostToDevice, st));
    CUDA_TRY(eng, cudaMemcpyAsync(d.W.p, W, cbytes, cudaMemcpyHostToDevice, st));
    CUDA_TRY(eng, cudaMemcpyAsync(d.wf.p, wf, n * 8, cudaMemcpyHostToDevice, st));
    if (thr) CUDA_TRY(eng, cudaMemcpyAsync(d.thr.p, thr, (size_t)count * 8, cudaMemcpyHostToDevice, st));
    IterateArgs a{count, N, p->iterations, p->reducer == FSR_REDUCER_TREE, p->gamma,
                  d.R.as<cpx<double>>(), d.G.as<cpx<double>>(), d.W.as<const cpx<double>>(),
                  d.wf.as<const double>(), thr ? d.thr.as<const double>() : nullptr,
                  sel ? d.sel.as<int32_t>() : nullptr, obj ? d.obj.as<double>() : nullptr,
                  ties ? d.ties.as<uint8_t>() : nullptr, done ? d.done.as<int32_t>() : nullptr};
    const size_t smem = 2 * n * 16;
    if (smem > 48 * 1024)
        CUDA_TRY(eng, cudaFuncSetAttribute(iterate_spectra_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::min<int64_t>(count, (int64_t)d.sms * 8);
    CUDA_TRY(eng, cudaEventRecord(d.ev0, st));
    iterate_spectra_kernel<<<grid, GEN_THREADS, smem, st>>>(a);
    CUDA_TRY(eng, cudaGetLastError());
    CUDA_TRY(eng, cudaEventRecord(d.ev1, st));
    CUDA_TRY(eng, cudaMemcpyAsync(R, d.R.p, cbytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(eng, cudaMemcpyAsync(G, d.G.p, cbytes, cudaMemcpyDeviceToHost, st));
    if (sel) CUDA_TRY(eng, cudaMemcpyAsync(sel, d.sel.p, (size_t)count * its * 4, cudaMemcpyDeviceToHost, st));
    if (obj) CUDA_TRY(eng, cudaMemcpyAsync(obj, d.obj.p, (size_t)count * its * 8, cudaMemcpyDeviceToHost, st));
    if (ties) CUDA_TRY(eng, cudaMemcpyAsync(ties, d.ties.p, (size_t)count * its, cudaMemcpyDeviceToHost, st));
    if (done) CUDA_TRY(eng, cudaMemcpyAsync(done, d.done.p, (size_t)count * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(eng, cudaStreamSynchronize(st));
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, d.ev0, d.ev1) != cudaSuccess) ms = 0.f;
    (void)cudaGetLastError();
    eng->stats = fsr_stats{};
    eng->device_stats_pending = false;
    eng->stats.blocks = count;
    eng->stats.kernel_launches = 1;
    eng->stats.kernel_ms = ms;
    return FSR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Callers either side of the loop, on the device.

int fsr_quarter_sample_device(fsr_engine *eng, const float *d_img, int64_t img_pitch,
                              int64_t height, int64_t width, uint64_t seed, float *d_sampled,
                              int64_t sampled_pitch, uint8_t *d_mask, int64_t mask_pitch,
                              void *stream) {
    if (!eng) return fail(nullptr, FSR_EINVAL, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    if (height < 1 || width < 1) return fail(eng, FSR_EINVAL, "image must have at least one pixel");
    Device &d = *eng->devs[0];
    int rc = select_device(eng, d);
    if (rc) return rc;
    const int64_t cells = ((height + 1) / 2) * ((width + 1) / 2);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cells + 255) / 256, (int64_t)d.sms * 16));
    quarter_sample_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_img, img_pitch, height, width, seed,
                                                                  d_sampled, sampled_pitch, d_mask,
                                                                  mask_pitch);
    CUDA_TRY(eng, cudaGetLastError());
    return FSR_OK;
}

int fsr_sq_error_device(fsr_engine *eng, const float *d_ref, int64_t ref_pitch, const float *d_test,
                        int64_t test_pitch, int64_t height, int64_t width, double *d_sse,
                        void *stream) {
    if (!eng) return fail(nullptr, FSR_EINVAL, "null engine");
    std::lock_guard<std::mutex> lock(eng->mu);
    if (height < 1 || width < 1) return fail(eng, FSR_EINVAL, "image must have at least one pixel");
    Device &d = *eng->devs[0];
    int rc = select_device(eng, d);
    if (rc) return rc;
    const int grid = d.sms * 4;  // fixed grid: the fixed-order final sum is deterministic
    CUDA_TRY(eng, d.partials.ensure((size_t)grid * sizeof(double)));
    cudaStream_t st = (cudaStream_t)stream;
    sq_err_partial_kernel<<<grid, 256, 0, st>>>(d_ref, ref_pitch, d_test, test_pitch, height, width,
                                                d.partials.as<double>());
    CUDA_TRY(eng, cudaGetLastError());
    sq_err_final_kernel<<<1, 32, 0, st>>>(d.partials.as<double>(), grid, d_sse);
    CUDA_TRY(eng, cudaGetLastError());
    return FSR_OK;
}
