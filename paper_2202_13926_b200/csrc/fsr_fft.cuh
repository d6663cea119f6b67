// fsr_fft.cuh -- in-register 32-point complex FFT (one lane, 32 values).
//
// Radix-2 decimation in frequency, fully unrolled: every twiddle index is a
// compile-time constant, so twiddles become immediates and the bit-reversed
// output order is a static register renaming.  Forward sign (e^{-2 pi i kn/N},
// the unnormalised numpy.fft convention the reference uses).
#pragma once

#include "fsr_common.cuh"

namespace fsr {

// cos(2 pi m / 32), m = 0..8; the others follow by exact quadrant symmetry.
__host__ __device__ constexpr double cos32(int m) {
    return m == 0 ? 1.0
         : m == 1 ? 0.98078528040323044912618223613424
         : m == 2 ? 0.92387953251128675612818318939679
         : m == 3 ? 0.83146961230254523707878837761791
         : m == 4 ? 0.70710678118654752440084436210485
         : m == 5 ? 0.55557023301960222474283081394853
         : m == 6 ? 0.38268343236508977172845998403040
         : m == 7 ? 0.19509032201612826784828486847702
                  : 0.0;
}

// cos / sin of 2 pi m / 32 for m in [0, 16)
__host__ __device__ constexpr double tw_cos(int m) { return m <= 8 ? cos32(m) : -cos32(16 - m); }
__host__ __device__ constexpr double tw_sin(int m) { return m <= 8 ? cos32(8 - m) : cos32(m - 8); }

// x[k] <- sum_n x[n] e^{-2 pi i k n / M}, M = 2^LOGM <= 32, output in NATURAL order.
template <int LOGM, typename T>
__device__ __forceinline__ void fft_pow2(cpx<T> (&x)[1 << LOGM]) {
    constexpr int M = 1 << LOGM;
#pragma unroll
    for (int h = M / 2; h >= 1; h >>= 1) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
            if ((j & h) == 0) {
                cpx<T> a = x[j], b = x[j + h];
                x[j] = {a.re + b.re, a.im + b.im};
                T dr = a.re - b.re, di = a.im - b.im;
                const int m = (j & (h - 1)) * (16 / h);  // stage twiddle W_{2h}^{j mod h} = W_32^m
                if (m == 0) {
                    x[j + h] = {dr, di};
                } else if (m == 8) {  // * (-i)
                    x[j + h] = {di, -dr};
                } else {
                    const T c = (T)tw_cos(m), s = (T)tw_sin(m);
                    // (dr + i di)(c - i s)
                    x[j + h] = {dr * c + di * s, di * c - dr * s};
                }
            }
        }
    }
    // undo the bit reversal (static renaming)
    cpx<T> y[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
        int r = 0;
#pragma unroll
        for (int b = 0; b < LOGM; ++b) r |= ((k >> b) & 1) << (LOGM - 1 - b);
        y[k] = x[r];
    }
#pragma unroll
    for (int k = 0; k < M; ++k) x[k] = y[k];
}

template <typename T>
__device__ __forceinline__ void fft32(cpx<T> (&x)[32]) { fft_pow2<5, T>(x); }

}  // namespace fsr
