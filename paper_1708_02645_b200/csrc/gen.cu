// gen.cu -- synthetic-input generator (test/bench harness; NOT the method).
// Device twin of qmcgen.positions(): the same counter-based integer recipe,
// implemented independently (no code shared with qmcgen/ or oracle/).
// Holds none of the method's arithmetic: it only draws numbers.
#include "qmcj2.h"

#include <cstdio>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

unsigned long long mix64_host(unsigned long long z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

template <typename T> __device__ __forceinline__ T draw(unsigned long long h, T L);

template <> __device__ __forceinline__ float draw<float>(unsigned long long h, float L) {
    const float u = (float)(unsigned)(h >> 40) * 5.9604644775390625e-08f;   // 2^-24
    float x = __fmul_rn(L, u);
    if (x >= L) x = __uint_as_float(__float_as_uint(L) - 1u);
    return x;
}
template <> __device__ __forceinline__ double draw<double>(unsigned long long h, double L) {
    const double u = (double)(h >> 11) * 1.1102230246251565e-16;              // 2^-53
    double x = __dmul_rn(L, u);
    if (x >= L) x = __longlong_as_double(__double_as_longlong(L) - 1ll);
    return x;
}

template <typename T>
__global__ void gen_kernel(unsigned long long key, int64_t W, int64_t w_offset, int64_t i_offset,
                           int64_t N_local, int64_t Np, T L, T *__restrict__ R) {
    const int64_t total = W * 3 * Np;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int64_t row = e / Np, i = e - row * Np;
        const int64_t w = row / 3, d = row - w * 3;
        T x = T(0);
        if (i < N_local) {
            const unsigned long long ctr =
                ((unsigned long long)((w_offset + w) * 3 + d) << 32) | (unsigned long long)(i_offset + i);
            x = draw<T>(mix64(key ^ ctr), L);
        }
        R[e] = x;
    }
}

}  // namespace

extern "C" qj2_status qj2gen_positions(qj2_dtype dtype, uint64_t seed, int64_t W, int64_t w_offset,
                                       int64_t i_offset, int64_t N_local, int64_t Np,
                                       double L, void *R, void *stream) {
    if (W < 0 || w_offset < 0 || i_offset < 0 || N_local < 0 || Np < N_local || !(L > 0))
        return QJ2_EINVAL;
    if (i_offset + N_local > (1ll << 32)) return QJ2_ERANGE;
    if (W == 0 || Np == 0) return QJ2_OK;
    if (!R) return QJ2_EINVAL;
    const unsigned long long key = mix64_host(seed * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int blocks = 148 * 16;
    if (dtype == QJ2_FP32)
        gen_kernel<float><<<blocks, 256, 0, s>>>(key, W, w_offset, i_offset, N_local, Np, (float)L, static_cast<float *>(R));
    else if (dtype == QJ2_FP64)
        gen_kernel<double><<<blocks, 256, 0, s>>>(key, W, w_offset, i_offset, N_local, Np, L, static_cast<double *>(R));
    else
        return QJ2_EINVAL;
    return cudaGetLastError() == cudaSuccess ? QJ2_OK : QJ2_ECUDA;
}

namespace {
__global__ void gen_spo_kernel(unsigned long long key, int64_t total, int64_t ld, int64_t n_orb,
                               float *__restrict__ coef) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int64_t o = e % ld;
        float x = 0.f;
        if (o < n_orb) {
            const unsigned long long h = mix64(key ^ (unsigned long long)e);
            x = (float)(unsigned)(h >> 40) * 1.1920928955078125e-07f - 1.0f;   // 2^-23: 2u - 1, exact
        }
        coef[e] = x;
    }
}
}  // namespace

extern "C" qj2_status qj2gen_spo_table(uint64_t seed, int64_t nx, int64_t ny, int64_t nz, int64_t n_orb,
                                       int64_t ld, float *coef, void *stream) {
    if (nx < 1 || ny < 1 || nz < 1 || n_orb < 1 || ld < n_orb) return QJ2_EINVAL;
    if (!coef) return QJ2_EINVAL;
    const unsigned long long k0 = mix64_host(seed * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull);
    const unsigned long long key = mix64_host(k0 ^ 0x5A0C0EFF1C1E17A5ull);
    gen_spo_kernel<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(key, nx * ny * nz * ld, ld, n_orb, coef);
    return cudaGetLastError() == cudaSuccess ? QJ2_OK : QJ2_ECUDA;
}
