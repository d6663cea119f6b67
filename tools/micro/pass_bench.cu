// Throughput microbenchmarks for the warp32 production pass on B200.
//   pipe tests: FFMA / FFMA2 / FMUL2 / integer (LOP3+VIMNMX) issue rates with
//               many independent chains and 12 warps per SM
//   pass tests: the real pass_x2 (fsr_warp32.cuh) in a loop with a cheap
//               synthetic selection sequence (no cross-lane argmax), 12 warps
//               per SM, to separate the pass's own bound from the serial part
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2202_13926_b200/csrc pass_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "fsr_warp32.cuh"

using namespace fsr;

constexpr int REPS = 4096;

__global__ void __launch_bounds__(128, 3) ffma_tput(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = a + j + threadIdx.x;
    float y = b + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < REPS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], y, a);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(128, 3) ffma2_tput(float *out, float a, float b) {
    float2 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = make_float2(a + j + threadIdx.x, a - j);
    float2 y = make_float2(b + threadIdx.x, b * 0.5f), c = make_float2(a, b);
#pragma unroll 1
    for (int i = 0; i < REPS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __ffma2_rn(x[j], y, c);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j].x + x[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(128, 3) ffma2s_tput(float *out, float a, float b) {
    // scalar-broadcast operand form, as in the pass
    float2 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = make_float2(a + j + threadIdx.x, a - j);
    float2 y = make_float2(b + threadIdx.x, b * 0.5f);
    const float g = a * 0.25f;
#pragma unroll 1
    for (int i = 0; i < REPS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __ffma2_rn(y, make_float2(g, g), x[j]);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j].x + x[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(128, 3) int_tput(unsigned *out, unsigned a, unsigned mask) {
    unsigned x[8], m1 = 0, m2 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = a * (j + 1) + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < REPS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            const unsigned ka = (x[j] & mask) | (j + 3), kb = (x[j + 1] & mask) | (j + 5);
            const unsigned hi = max(ka, kb), lo = min(ka, kb);
            m2 = max(max(m2, lo), min(m1, hi));
            m1 = max(m1, hi);
            x[j] += m1;
            x[j + 1] ^= m2;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = m1 + m2 + x[0];
}

template <bool GUARD, int MINB = 3>
__global__ void __launch_bounds__(128, MINB) pass_tput(float *out, uint32_t hmask, int iters) {
    extern __shared__ float4 ubraw[];
    // 16 KiB per warp; with more than 3 CTAs per SM the warps of a CTA share
    // one table (timing is what matters here, not the values)
    float4 (*ub)[32 * 32] = reinterpret_cast<float4 (*)[32 * 32]>(ubraw);
    const int lane = threadIdx.x & 31, wid = MINB == 4 ? 0 : threadIdx.x >> 5;
    for (int i = lane; i < 32 * 32; i += 32)
        ub[wid][i] = make_float4(1e-3f * (i & 31), 1e-3f * (i >> 5), 2e-3f, -1e-3f);
    __syncwarp();
    float2 re[16], im[16], wf2[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        re[i] = make_float2(1.f + i + lane, 2.f - i);
        im[i] = make_float2(0.5f * i, lane * 0.25f);
        wf2[i] = make_float2(0.9f - 0.01f * i, 0.5f + 0.01f * i);
    }
    int pu = 3, pv = 7;
    float gr = 1e-6f, gi = -2e-6f;
    uint32_t acc = 0;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        uint32_t m1, m2;
        const float4 *up = ub[wid] + (16 - (pu & 15)) * 32 + ((lane - pv) & 31);
        pass_update<true, GUARD, false>(re, im, wf2, up, pu >= 16, gr, gi, 0u, hmask, m1, m2);
        acc += m1 ^ m2;
        gr = __uint_as_float((m1 & 0x007fffffu) | 0x2f000000u);  // data-dependent, tiny
        gi = -gr;
        pu = (pu + 7 + (int)(m1 & 1)) & 31;
        pv = (pv + 5) & 31;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += re[i].x + re[i].y + im[i].x + im[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
}


template <int MODE>
__device__ __forceinline__ void pass_part(float2 (&re)[16], float2 (&im)[16], const float2 (&wf2)[16],
                                          const float4 *up, float gr, float gi, uint32_t hmask,
                                          uint32_t &m1, uint32_t &m2) {
    m1 = 0;
    m2 = 0;
    const float2 ngr = make_float2(-gr, -gr), pgi = make_float2(gi, gi), ngi = make_float2(-gi, -gi);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float2 r = re[i], m = im[i];
        if (MODE == 0 || MODE == 3) {
            const float4 w = up[i * 32];
            if (MODE == 0) {
                r = __ffma2_rn(make_float2(w.x, w.y), ngr, r);
                r = __ffma2_rn(make_float2(w.z, w.w), pgi, r);
                m = __ffma2_rn(make_float2(w.z, w.w), ngr, m);
                m = __ffma2_rn(make_float2(w.x, w.y), ngi, m);
            } else {
                r.x += w.x; r.y += w.y; m.x += w.z; m.y += w.w;
            }
            re[i] = r;
            im[i] = m;
        } else {
            const float2 mag = __ffma2_rn(r, r, __fmul2_rn(m, m));
            const float2 o = __fmul2_rn(mag, wf2[i]);
            uint32_t ka = (__float_as_uint(o.x) & hmask) | (31u ^ i);
            uint32_t kb = (__float_as_uint(o.y) & hmask) | (15u ^ i);
            if (MODE == 1) {
                const uint32_t hi = max(ka, kb), lo = min(ka, kb);
                m2 = umax3(m2, lo, min(m1, hi));
                m1 = max(m1, hi);
            } else {
                m1 = umax3(m1, ka, kb);
            }
            re[i].x += 1e-30f * m1;  // keep the values live and changing
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(128, 3) part_tput(float *out, uint32_t hmask, int iters) {
    extern __shared__ float4 ubraw[];
    float4 (*ub)[32 * 32] = reinterpret_cast<float4 (*)[32 * 32]>(ubraw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = lane; i < 32 * 32; i += 32)
        ub[wid][i] = make_float4(1e-3f * (i & 31), 1e-3f * (i >> 5), 2e-3f, -1e-3f);
    __syncwarp();
    float2 re[16], im[16], wf2[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        re[i] = make_float2(1.f + i + lane, 2.f - i);
        im[i] = make_float2(0.5f * i, lane * 0.25f);
        wf2[i] = make_float2(0.9f - 0.01f * i, 0.5f + 0.01f * i);
    }
    int pu = 3, pv = 7;
    float gr = 1e-6f, gi = -2e-6f;
    uint32_t acc = 0;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        uint32_t m1, m2;
        const float4 *up = ub[wid] + (16 - (pu & 15)) * 32 + ((lane - pv) & 31);
        pass_part<MODE>(re, im, wf2, up, gr, gi, hmask, m1, m2);
        acc += m1 ^ m2;
        gr = __uint_as_float((__float_as_uint(re[3].x) & 0x007fffffu) | 0x2f000000u);
        gi = -gr;
        pu = (pu + 7 + (int)(acc & 1)) & 31;
        pv = (pv + 5) & 31;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += re[i].x + re[i].y + im[i].x + im[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int grid = sms * 3, block = 128;
    float *out;
    cudaMalloc(&out, grid * block * sizeof(float) * 2);
    cudaFuncSetAttribute(pass_tput<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(pass_tput<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(pass_tput<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(part_tput<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(part_tput<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(part_tput<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(part_tput<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double smsp = sms * 4.0;
    auto report = [&](const char *name, double warp_instr_per_smsp, float ms) {
        // cycles at the max clock (the bench runs unthrottled at 1965 MHz)
        const double cyc = ms * 1e-3 * clk_khz * 1e3;
        printf("%-34s %8.3f ms  %.3f warp-instr/clk/SMSP\n", name, ms, warp_instr_per_smsp / cyc);
    };
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0);
        ffma_tput<<<grid, block>>>(out, 1.0f, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        report("FFMA (3-reg, 8 chains)", (double)grid * 4 * REPS * 8 / smsp, ms);
        cudaEventRecord(e0);
        ffma2_tput<<<grid, block>>>(out, 1.0f, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        report("FFMA2 (3-reg pairs, 8 chains)", (double)grid * 4 * REPS * 8 / smsp, ms);
        cudaEventRecord(e0);
        ffma2s_tput<<<grid, block>>>(out, 1.0f, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        report("FFMA2 (scalar-broadcast, 8 ch)", (double)grid * 4 * REPS * 8 / smsp, ms);
        cudaEventRecord(e0);
        int_tput<<<grid, block>>>((unsigned *)out, 12345u, 0xffffffe0u);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        report("int key+top2 (approx instr)", (double)grid * 4 * REPS * 4 * 9 / smsp, ms);
        const int iters = 2000;
        cudaEventRecord(e0);
        pass_tput<true><<<grid, block, 65536>>>(out, 0xffffffe0u, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        {
            const double cyc = ms * 1e-3 * clk_khz * 1e3;
            printf("%-34s %8.3f ms  %.1f clk per pass per SMSP (3 warps/SMSP)\n", "pass guarded", ms,
                   cyc / ((double)grid * 4 * iters / smsp));
        }
        for (int cps : {1, 2, 4}) {
            const int g2 = sms * cps;
            const int sm_bytes = cps == 4 ? 16384 : 65536;
            cudaEventRecord(e0);
            if (cps == 4) pass_tput<true, 4><<<g2, block, sm_bytes>>>(out, 0xffffffe0u, iters);
            else pass_tput<true, 3><<<g2, block, sm_bytes>>>(out, 0xffffffe0u, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double cyc = ms * 1e-3 * clk_khz * 1e3;
            printf("pass guarded, %d warps/SMSP            %8.3f ms  %.1f clk per pass per SMSP\n", cps, ms,
                   cyc / ((double)g2 * 4 * iters / smsp));
        }
        {
            const char *nm[4] = {"part: LDS + update (4 FFMA2/pair)", "part: objective+keys+top2", "part: objective+keys+max3", "part: LDS only"};
            for (int md = 0; md < 4; ++md) {
                cudaEventRecord(e0);
                if (md == 0) part_tput<0><<<grid, block, 65536>>>(out, 0xffffffe0u, iters);
                if (md == 1) part_tput<1><<<grid, block, 65536>>>(out, 0xffffffe0u, iters);
                if (md == 2) part_tput<2><<<grid, block, 65536>>>(out, 0xffffffe0u, iters);
                if (md == 3) part_tput<3><<<grid, block, 65536>>>(out, 0xffffffe0u, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                const double cyc = ms * 1e-3 * clk_khz * 1e3;
                printf("%-38s %8.3f ms  %.1f clk per pass per SMSP\n", nm[md], ms, cyc / ((double)grid * 4 * iters / smsp));
            }
        }
        cudaEventRecord(e0);
        pass_tput<false><<<grid, block, 65536>>>(out, 0xffffffe0u, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        {
            const double cyc = ms * 1e-3 * clk_khz * 1e3;
            printf("%-34s %8.3f ms  %.1f clk per pass per SMSP (3 warps/SMSP)\n", "pass unguarded", ms,
                   cyc / ((double)grid * 4 * iters / smsp));
        }
    }
    printf("clock %d kHz, %d SMs, %s\n", clk_khz, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
