// fsr_aux.cuh -- the callers either side of the loop, on the device
// (SURVEY §8f row 1): quarter sampling of a frame and the PSNR/MSE of a
// reconstruction against its original, so a frame stream needs no host
// pre- or post-processing.
//
//   quarter_sample_kernel  reference sampling.py:18-29 (SplitMix64) and
//                          53-80 (quarter_sample): one known pixel per 2x2
//                          cell, cell i (row-major over the cells) picks
//                          z_i mod (cell_h * cell_w) with
//                          z_i = mix(seed + (i + 1) * 0x9E3779B97F4A7C15);
//                          edge cells of odd frames shrink to 1 row/column.
//                          Writes the mask (u8) and the sampled frame (unknown
//                          pixels zero, as SampledImage requires).
//                          HBM-bound: 4 B read + 5 B written per pixel.
//   sq_err_partial_kernel  metrics.py:35-48: sum of (clamp(test, 0, 255) - ref)^2
//   sq_err_final_kernel    in fp64, per-CTA partials then one fixed-order sum
//                          (deterministic for a given grid).
#pragma once

#include "fsr_common.cuh"

namespace fsr {

__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// One thread per 2x2 cell; consecutive threads take consecutive cells of a
// cell row, so each of the two pixel rows is written as coalesced float2 /
// uchar2 pairs.
__global__ void quarter_sample_kernel(const float *img, int64_t img_pitch, int64_t H, int64_t W,
                                      uint64_t seed, float *sampled, int64_t s_pitch,
                                      uint8_t *mask, int64_t m_pitch) {
    const int64_t rows = (H + 1) / 2, cols = (W + 1) / 2, n = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cr = i / cols, cc = i - cr * cols;
        const uint64_t ch = (2 * cr + 1 < H) ? 2 : 1, cw = (2 * cc + 1 < W) ? 2 : 1;
        const uint64_t sel = splitmix64_at(seed, (uint64_t)i) % (ch * cw);
        const int dr = (int)(sel / cw), dc = (int)(sel % cw);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int64_t y = 2 * cr + r;
            if (y >= H) break;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int64_t x = 2 * cc + c;
                if (x >= W) break;
                const bool known = r == dr && c == dc;
                mask[y * m_pitch + x] = known ? 1 : 0;
                sampled[y * s_pitch + x] = known ? img[y * img_pitch + x] : 0.f;
            }
        }
    }
}

__global__ void sq_err_partial_kernel(const float *ref, int64_t ref_pitch, const float *test,
                                      int64_t test_pitch, int64_t H, int64_t W, double *partial) {
    double acc = 0.0;
    const int64_t n = H * W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = i / W, x = i - y * W;
        const double t = fmin(fmax((double)test[y * test_pitch + x], 0.0), 255.0);
        const double d = t - (double)ref[y * ref_pitch + x];
        acc = fma(d, d, acc);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    __shared__ double sw[32];
    if (lane_id() == 0) sw[warp_id()] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sw[w];
        partial[blockIdx.x] = s;
    }
}

__global__ void sq_err_final_kernel(const double *partial, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += partial[i];
        *out = s;
    }
}

}  // namespace fsr
