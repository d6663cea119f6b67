// TMA probe 2: 1-D bulk copy, and 2-D tensor copy with the descriptor in global memory.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void wait0(uint32_t bar) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                     : "=r"(done) : "r"(bar) : "memory");
}

template <int MODE>
__global__ void k(const CUtensorMap *gtm, const float *src, float *out, int x0, int y0) {
    __shared__ __align__(1024) unsigned char buf[8192];
    __shared__ __align__(8) unsigned long long barm;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&barm);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf);
    if (MODE == 2) {
        if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;");
        __syncwarp();
        asm volatile(
            "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
            "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], 4096;\n"
            "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n}"
            ::"r"(dst), "l"(reinterpret_cast<uint64_t>(gtm)), "r"(x0), "r"(y0), "r"(bar) : "memory");
        wait0(bar);
    } else if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4096));
        if (MODE == 0) {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst), "l"(src), "r"(4096), "r"(bar) : "memory");
        } else {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(dst), "l"(reinterpret_cast<uint64_t>(gtm)), "r"(x0), "r"(y0), "r"(bar) : "memory");
        }
        wait0(bar);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = reinterpret_cast<float *>(buf)[i];
}

int main(int argc, char **argv) {
    const int sw = argc > 1 ? atoi(argv[1]) : 0;
    const int H = 64, W = 96;
    float *d;
    cudaMalloc(&d, H * W * 4);
    cudaMemset(d, 0, H * W * 4);
    float *out;
    cudaMalloc(&out, 8192);
    alignas(64) CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    const cuuint64_t str[1] = {(cuuint64_t)W * 4};
    const cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)sw,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap *gtm;
    cudaMalloc(&gtm, sizeof(tm));
    cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    printf("encode %d\n", (int)r);
    k<0><<<1, 32>>>(gtm, d, out, 10, 5);
    printf("bulk 1-D: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    const int xs[4] = {0, 4, 10, -14}, ys[4] = {0, 5, 5, -14};
    for (int c = 0; c < 4; ++c) {
        k<2><<<1, 32>>>(gtm, d, out, xs[c], ys[c]);
        printf("tensor 2-D elect.sync (%d,%d): %s\n", xs[c], ys[c], cudaGetErrorString(cudaDeviceSynchronize()));
    }
    k<1><<<1, 32>>>(gtm, d, out, 10, 5);
    printf("tensor 2-D (global desc): %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
