// Saturating non-tensor FP32 / FP64 throughput on B200 (sm_100a): the
// denominators of the FSR loop kernels' roofline fractions.
//
// Every SM is filled to its thread limit (2048 threads = 64 warps = 16 warps
// per SMSP; 148 x 2 CTAs of 1024 threads, one wave) and every thread runs 8
// independent dependency chains of FFMA, FFMA2 (sm_100 paired fp32,
// fma.rn.f32x2) or DFMA for seconds, so neither latency nor launch overhead
// can hide in the number.  The same kernels are also run at 3 warps per SMSP
// (the FSR kernels' occupancy) to show how much of the round-1 microbenchmark's
// 0.54-0.59 FFMA warp-instructions/clk/SMSP was latency, not pipe rate.
//
// Output: one line per (form, occupancy): time, clock from %globaltimer /
// clock64, TFLOP/s (an FMA = 2 flops; FFMA2 = 4 per lane) and warp
// instructions per clock per SMSP.  The tools/micro/peak_flops.py driver
// samples nvidia-smi clocks around it and writes the JSON under profiles/.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peak_flops peak_flops.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ unsigned long long g_t[4];

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int CHAINS>
__global__ void __launch_bounds__(1024, 2) k_ffma(float *out, float a, float b, int reps) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_t[0] = clock64(); g_t[2] = gtimer(); }
    float x[CHAINS];
    const float y = b * 0.5f + threadIdx.x * 1e-7f, z = a * 0.25f;
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) x[j] = a + j + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < reps; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < CHAINS; ++j) x[j] = fmaf(x[j], y, z);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_t[1] = clock64(); g_t[3] = gtimer(); }
}

template <int CHAINS>
__global__ void __launch_bounds__(1024, 2) k_ffma2(float *out, float a, float b, int reps) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_t[0] = clock64(); g_t[2] = gtimer(); }
    float2 x[CHAINS];
    const float2 y = make_float2(b * 0.5f + threadIdx.x * 1e-7f, b), z = make_float2(a * 0.25f, a);
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) x[j] = make_float2(a + j + threadIdx.x, b - j);
#pragma unroll 1
    for (int i = 0; i < reps; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < CHAINS; ++j) x[j] = __ffma2_rn(x[j], y, z);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) s += x[j].x + x[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_t[1] = clock64(); g_t[3] = gtimer(); }
}

template <int CHAINS>
__global__ void __launch_bounds__(1024, 2) k_dfma(double *out, double a, double b, int reps) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_t[0] = clock64(); g_t[2] = gtimer(); }
    double x[CHAINS];
    const double y = b * 0.5 + threadIdx.x * 1e-9, z = a * 0.25;
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) x[j] = a + j + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < reps; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < CHAINS; ++j) x[j] = fma(x[j], y, z);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_t[1] = clock64(); g_t[3] = gtimer(); }
}

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

template <typename K, typename T>
void run(const char *name, K kern, T *buf, int sms, int threads, int ctas_per_sm, int reps,
         double flop_per_fma_lane, int chains) {
    const int grid = sms * ctas_per_sm;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    kern<<<grid, threads>>>(buf, (T)1.0001, (T)0.9999, reps / 16 + 1);  // warm-up
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    unsigned long long t[4] = {0, 0, 0, 0};
    for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0));
        kern<<<grid, threads>>>(buf, (T)1.0001, (T)0.9999, reps);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) {
            best = ms;
            CK(cudaMemcpyFromSymbol(t, g_t, sizeof t));
        }
    }
    const double fmas = (double)grid * threads * reps * 16.0 * chains;  // per lane
    const double tflops = fmas * flop_per_fma_lane / (best * 1e-3) / 1e12;
    const double mhz = (double)(t[1] - t[0]) / ((double)(t[3] - t[2]) * 1e-3);
    const double warp_instr = fmas / 32.0;
    const double per_clk_smsp = warp_instr / (sms * 4.0) / ((double)best * 1e-3 * mhz * 1e6);
    printf("%-6s warps/SMSP=%2d chains=%d  %9.3f ms  %7.1f MHz  %8.2f TFLOP/s  %.3f warp-instr/clk/SMSP\n",
           name, threads * ctas_per_sm / 128, chains, best, mhz, tflops, per_clk_smsp);
    fflush(stdout);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

int main(int argc, char **argv) {
    int reps = argc > 1 ? atoi(argv[1]) : 40000;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    printf("device %s, %d SMs, clockRate %d kHz\n", prop.name, sms, prop.clockRate);
    float *fb;
    double *db;
    CK(cudaMalloc(&fb, (size_t)sms * 2048 * sizeof(float)));
    CK(cudaMalloc(&db, (size_t)sms * 2048 * sizeof(double)));
    // full occupancy: 2 x 1024 threads per SM = 16 warps per SMSP
    run("FFMA", k_ffma<8>, fb, sms, 1024, 2, reps, 2.0, 8);
    run("FFMA2", k_ffma2<8>, fb, sms, 1024, 2, reps, 4.0, 8);
    run("DFMA", k_dfma<8>, db, sms, 1024, 2, reps / 4, 2.0, 8);
    // the FSR kernels' occupancy: 12 warps per SM = 3 per SMSP (384 threads, 1 CTA)
    run("FFMA", k_ffma<8>, fb, sms, 384, 1, reps, 2.0, 8);
    run("FFMA2", k_ffma2<8>, fb, sms, 384, 1, reps, 4.0, 8);
    run("DFMA", k_dfma<8>, db, sms, 384, 1, reps / 4, 2.0, 8);
    CK(cudaFree(fb));
    CK(cudaFree(db));
    return 0;
}
