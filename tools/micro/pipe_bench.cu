// Issue/pipe throughput of the FP32 forms the FSR pass uses, on B200 (sm_100a).
// Each kernel runs 12 warps per SM (3 per SMSP), 8 independent chains per
// thread, long loops; reports warp-instructions per clock per SMSP.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipe_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int REPS = 1 << 15;

__device__ unsigned long long g_clk[2], g_ns[2];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define KERNEL_BEGIN(name, T)                                                   \
    __global__ void __launch_bounds__(128, 3) name(float *out, float a, float b) { \
        if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = clock64(); g_ns[0] = gtimer(); } \
        T x[8];                                                                 \
        _Pragma("unroll") for (int j = 0; j < 8; ++j) init(x[j], a + j + threadIdx.x, b - j);
#define KERNEL_LOOP _Pragma("unroll 1") for (int i = 0; i < REPS; ++i) { _Pragma("unroll") for (int j = 0; j < 8; ++j) {
#define KERNEL_END                                                              \
    } }                                                                         \
    float s = 0;                                                                \
    _Pragma("unroll") for (int j = 0; j < 8; ++j) s += sum(x[j]);               \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[1] = clock64(); g_ns[1] = gtimer(); } \
    }

__device__ __forceinline__ void init(float &x, float a, float b) { x = a * b; }
__device__ __forceinline__ void init(float2 &x, float a, float b) { x = make_float2(a, b); }
__device__ __forceinline__ void init(unsigned &x, float a, float b) { x = __float_as_uint(a * b); }
__device__ __forceinline__ float sum(float x) { return x; }
__device__ __forceinline__ float sum(float2 x) { return x.x + x.y; }
__device__ __forceinline__ float sum(unsigned x) { return (float)x; }

// FFMA, two loop-invariant register operands
KERNEL_BEGIN(k_ffma_rr, float)
float y = b * 0.5f + threadIdx.x, z = a * 0.25f;
KERNEL_LOOP x[j] = fmaf(x[j], y, z);
KERNEL_END
// FFMA, immediate addend
KERNEL_BEGIN(k_ffma_ri, float)
float y = b * 0.5f + threadIdx.x;
KERNEL_LOOP x[j] = fmaf(x[j], y, 1.5f);
KERNEL_END
// FFMA, three distinct per-chain registers (no reuse possible for two operands)
KERNEL_BEGIN(k_ffma_3r, float)
float y[8], z[8];
_Pragma("unroll") for (int j = 0; j < 8; ++j) { y[j] = b + j * threadIdx.x; z[j] = a - j; }
KERNEL_LOOP x[j] = fmaf(y[j], x[j], z[j]); y[j] = fmaf(z[j], y[j], x[j]);
KERNEL_END
// FFMA2 with pair operands
KERNEL_BEGIN(k_ffma2_rr, float2)
float2 y = make_float2(b * 0.5f + threadIdx.x, b), z = make_float2(a, a * 0.5f);
KERNEL_LOOP x[j] = __ffma2_rn(x[j], y, z);
KERNEL_END
// FFMA2 with a scalar-broadcast operand (the pass's update form)
KERNEL_BEGIN(k_ffma2_bc, float2)
float2 w[8];
_Pragma("unroll") for (int j = 0; j < 8; ++j) w[j] = make_float2(b + j, a - j * threadIdx.x);
const float g = a * 0.125f;
KERNEL_LOOP x[j] = __ffma2_rn(w[j], make_float2(g, g), x[j]);
KERNEL_END
// FMUL2
KERNEL_BEGIN(k_fmul2, float2)
float2 y = make_float2(0.999f, 1.001f);
KERNEL_LOOP x[j] = __fmul2_rn(x[j], y);
KERNEL_END
// FMUL
KERNEL_BEGIN(k_fmul, float)
float y = 0.999f + threadIdx.x * 1e-9f;
KERNEL_LOOP x[j] = x[j] * y;
KERNEL_END
// FADD
KERNEL_BEGIN(k_fadd, float)
float y = 0.999f + threadIdx.x * 1e-9f;
KERNEL_LOOP x[j] = x[j] + y;
KERNEL_END
// LOP3
KERNEL_BEGIN(k_lop3, unsigned)
unsigned m = 0xffffffe0u + (threadIdx.x >> 10);
KERNEL_LOOP x[j] = (x[j] & m) | (unsigned)(j + 1 + i);
KERNEL_END
// IMNMX
KERNEL_BEGIN(k_imnmx, unsigned)
unsigned m = 12345u + threadIdx.x;
KERNEL_LOOP x[j] = max(x[j] + 0, m + j) ;
KERNEL_END
// FFMA2 + VIMNMX interleaved (fma pipe + alu pipe); both results live
#define KERNEL_END_K                                                            \
    } }                                                                         \
    float s = 0;                                                                \
    _Pragma("unroll") for (int j = 0; j < 8; ++j) s += sum(x[j]) + (float)k[j]; \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[1] = clock64(); g_ns[1] = gtimer(); } \
    }
KERNEL_BEGIN(k_mix, float2)
unsigned k[8];
_Pragma("unroll") for (int j = 0; j < 8; ++j) k[j] = threadIdx.x + j;
float2 y = make_float2(b * 0.5f + threadIdx.x, b), z = make_float2(a, a * 0.5f);
unsigned m = 12345u + threadIdx.x;
KERNEL_LOOP x[j] = __ffma2_rn(x[j], y, z); k[j] = max(k[j], m + j);
KERNEL_END_K
// FFMA + VIMNMX interleaved
KERNEL_BEGIN(k_mix1, float)
unsigned k[8];
_Pragma("unroll") for (int j = 0; j < 8; ++j) k[j] = threadIdx.x + j;
float y = b * 0.5f + threadIdx.x, z = a;
unsigned m = 12345u + threadIdx.x;
KERNEL_LOOP x[j] = fmaf(x[j], y, z); k[j] = max(k[j], m + j);
KERNEL_END_K
// VIMNMX two chains per element (alu only, 16 per iteration)
KERNEL_BEGIN(k_alu2, float)
unsigned k[8], q[8];
_Pragma("unroll") for (int j = 0; j < 8; ++j) { k[j] = threadIdx.x + j; q[j] = threadIdx.x * 3 + j; }
unsigned m = 12345u + threadIdx.x;
KERNEL_LOOP k[j] = max(k[j], m + j); q[j] = min(q[j], m - j);
_Pragma("unroll") for (int j = 0; j < 8; ++j) x[j] = (float)(k[j] ^ q[j]);
KERNEL_END

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int grid = sms * 3, block = 128;
    float *out;
    cudaMalloc(&out, grid * block * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct K { const char *name; void (*f)(float *, float, float); double per_iter; };
    K ks[] = {{"FFMA  x=fma(x,y,z) (2 inv regs)", k_ffma_rr, 8},
              {"FFMA  x=fma(x,y,imm)", k_ffma_ri, 8},
              {"FFMA  3 distinct regs", k_ffma_3r, 16},
              {"FFMA2 pair operands", k_ffma2_rr, 8},
              {"FFMA2 scalar broadcast", k_ffma2_bc, 8},
              {"FMUL2", k_fmul2, 8},
              {"FMUL", k_fmul, 8},
              {"FADD", k_fadd, 8},
              {"LOP3", k_lop3, 8},
              {"IMNMX", k_imnmx, 8},
              {"FFMA2+VIMNMX (count both)", k_mix, 16},
              {"FFMA+VIMNMX (count both)", k_mix1, 16},
              {"VIMNMX+VIMNMX (count both)", k_alu2, 16}};
    for (int w = 0; w < 200; ++w) k_ffma_rr<<<grid, block>>>(out, 1.0f, 0.999f);  // clock ramp
    cudaDeviceSynchronize();
    for (int rep = 0; rep < 2; ++rep)
        for (auto &k : ks) {
            k.f<<<grid, block>>>(out, 1.0f, 0.999f);  // warm
            cudaEventRecord(e0);
            k.f<<<grid, block>>>(out, 1.0f, 0.999f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long c[2], n[2];
            cudaMemcpyFromSymbol(c, g_clk, sizeof(c));
            cudaMemcpyFromSymbol(n, g_ns, sizeof(n));
            const double mhz = (double)(c[1] - c[0]) / (double)(n[1] - n[0]) * 1e3;
            const double cyc = ms * 1e-3 * mhz * 1e6;
            const double instr = (double)grid * 4 * REPS * k.per_iter / (sms * 4.0);
            if (rep) printf("%-34s %8.3f ms  %6.0f MHz  %.3f warp-instr/clk/SMSP\n", k.name, ms, mhz, instr / cyc);
        }
    printf("clock %d kHz, %d SMs, %s\n", clk_khz, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
