// Microbenchmarks (B200): latency of dependent DFMA / FFMA / LDS.128 / REDUX / SHFL
// and DFMA throughput per SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_lat(double* out, double a, double b, long long* cyc) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
__global__ void ffma_lat(float* out, float a, float b, long long* cyc) {
  float x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = fmaf(x, b, a); x = fmaf(x, b, a); x = fmaf(x, b, a); x = fmaf(x, b, a); }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
__global__ void lds_lat(double* out, long long* cyc) {
  __shared__ double2 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_double2((i * 7 + 1) & 1023, 0.0);
  __syncthreads();
  int idx = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { double2 v = s[idx]; idx = (int)v.x; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = idx; }
}
__global__ void redux_lat(unsigned* out, long long* cyc) {
  unsigned x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = __reduce_max_sync(0xffffffffu, x) + threadIdx.x; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
__global__ void shfl_lat(unsigned* out, long long* cyc) {
  unsigned x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = __shfl_xor_sync(0xffffffffu, x, 1) + 1; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
// throughput: many independent DFMA chains per thread, many warps
__global__ void dfma_tput(double* out, double a, double b, long long* cyc) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* d; long long* c; unsigned* u; float* f;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 64); cudaMalloc(&u, 64); cudaMalloc(&f, 64);
  long long h;
  dfma_lat<<<1, 32>>>(d, 1.0, 0.999, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h / 4096.0);
  ffma_lat<<<1, 32>>>(f, 1.0f, 0.999f, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", h / 4096.0);
  lds_lat<<<1, 32>>>(d, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS.128 pointer-chase latency: %.2f cycles\n", h / 1024.0);
  redux_lat<<<1, 32>>>(u, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("REDUX.MAX + IADD latency: %.2f cycles\n", h / 1024.0);
  shfl_lat<<<1, 32>>>(u, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("SHFL + IADD latency: %.2f cycles\n", h / 1024.0);
  for (int warps = 1; warps <= 16; warps *= 2) {
    dfma_tput<<<148, 32 * warps>>>(d, 1.0, 0.999, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    // per SM: warps * 32 threads * 8192 DFMA in h cycles
    printf("DFMA throughput, %2d warps/SM, 8 chains: %.1f DFMA lanes/clk/SM\n", warps,
           warps * 32.0 * 8192 / h);
  }
  return 0;
}
