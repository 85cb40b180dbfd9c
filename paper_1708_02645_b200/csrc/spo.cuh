// spo.cuh -- NEXT-4: tricubic B-spline SPO evaluation ("Bspline-v",
// "Bspline-vgh") over the read-only 3D table
// shared by all walkers, fused with the determinant ratio
// of Eq. 6 ("a dot product of the k-th row of A^{-1} and
// v(phi_1(r'_k), ..., phi_{N/2}(r'_k))") and its gradient / Laplacian ratios.
// Written for sm_100a; shares nothing with oracle/.
//
// Mapping: TPW threads per walker (NV = 4 (v) or 2 (vgh) orbitals per
// thread and pass), WPC walkers per CTA.  Per walker the 64 coefficient rows
// (ix_a, iy_b, iz_c) are gathered as 16 (a, b) columns of 4 z-rows (4 x 16 B
// per thread, a contiguous 4 * ld * 4 B chunk unless the z index wraps); the
// z-sums s0 = sum B_c P, s1 = sum B'_c P, s2 = sum B''_c P are combined with
// the 6 (a, b) weights into the 10 outputs (v, g, h): 88 FMAs per 4 rows of
// a float4.  HBM/L2-bound random gathers: 64 * ld * 4 bytes per walker.
#pragma once

#include "qmcj2.h"
#include <cstdint>

namespace qj2 {

struct SpoParams {
    int64_t W, nx, ny, nz, n_orb, ld, nvec;    // nvec = ld / NV (NV = 4 for v, 2 for vgh)
    const float *coef;                          // [nx][ny][nz][ld]
    double L[3];
    int32_t pos_f64;                            // position dtype
    const void *pos;                            // row w at pos + w * pos_stride (elements)
    int64_t pos_stride;
    const float *Ainv;                          // row of walker w at Ainv + w*ainv_stride + krow[w]*ainv_ld
    int64_t ainv_stride, ainv_ld;
    const int32_t *krow;                        // or NULL (Ainv rows pre-gathered)
    double *out;                                // [W][5] (rho, Gx, Gy, Gz, L) or NULL
    float *spo_out;                             // [W][NQ][ld] or NULL
    int32_t tpw, wpc;                           // threads per walker, walkers per CTA
};

// NV consecutive orbitals per thread: 4 for Bspline-v, 2 for Bspline-vgh
// (10 accumulators x NV must stay in registers).
template <int NV> struct alignas(4 * NV) FV { float v[NV]; };

__device__ __forceinline__ FV<4> ld_row(const FV<4> *p) {
    FV<4> r;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]) : "l"(p));
    return r;
}
__device__ __forceinline__ FV<2> ld_row(const FV<2> *p) {
    FV<2> r;
    asm("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.v[0]), "=f"(r.v[1]) : "l"(p));
    return r;
}

// One axis: wrapped control indices (times the row stride) and the basis
// weights B, B' * n/L, B'' * (n/L)^2 at the fractional coordinate.  The
// coordinate is reduced in fp64 (u up to n ~ 100: an fp32 u would carry
// ~5e-6 absolute error into t), then the weights are rounded to fp32.
struct AxisW {
    int32_t off[4];         // element offsets in vectors (the host checks the table has < 2^31 vectors)
    float B[4], D[4], S[4];
};

__device__ __forceinline__ void axis_weights(double x, double L, int64_t n, int32_t stride, AxisW &a) {
    double xw = fmod(x, L);
    if (xw < 0) xw += L;
    const double u = xw / L * (double)n;
    double fi = floor(u);
    const double t = u - fi;
    int64_t i = (int64_t)fi;
    if (i >= n) i -= n;
    for (int c = 0; c < 4; ++c) {
        int64_t j = i - 1 + c;
        j = j < 0 ? j + n : (j >= n ? j - n : j);
        a.off[c] = (int32_t)j * stride;
    }
    const double g = 1.0 - t, s = (double)n / L;
    a.B[0] = (float)(g * g * g / 6.0);
    a.B[1] = (float)((3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0);
    a.B[2] = (float)((-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0);
    a.B[3] = (float)(t * t * t / 6.0);
    a.D[0] = (float)(-0.5 * g * g * s);
    a.D[1] = (float)(0.5 * (3.0 * t * t - 4.0 * t) * s);
    a.D[2] = (float)(0.5 * (-3.0 * t * t + 2.0 * t + 1.0) * s);
    a.D[3] = (float)(0.5 * t * t * s);
    a.S[0] = (float)((1.0 - t) * s * s);
    a.S[1] = (float)((3.0 * t - 2.0) * s * s);
    a.S[2] = (float)((1.0 - 3.0 * t) * s * s);
    a.S[3] = (float)(t * s * s);
}

template <int NV>
__device__ __forceinline__ void fma4(FV<NV> &acc, float w, const FV<NV> &x) {
#pragma unroll
    for (int e = 0; e < NV; ++e) acc.v[e] = fmaf(w, x.v[e], acc.v[e]);
}
template <int NV> __device__ __forceinline__ FV<NV> zero4() {
    FV<NV> z;
#pragma unroll
    for (int e = 0; e < NV; ++e) z.v[e] = 0.f;
    return z;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// VGH = false: Bspline-v (values only; ratio rho only).
template <bool VGH>
__global__ void __launch_bounds__(256, 2) spo_kernel(const __grid_constant__ SpoParams p) {
    constexpr int NV = VGH ? 2 : 4;
    using Vt = FV<NV>;
    constexpr int NQ = VGH ? 10 : 1;
    constexpr int NR = VGH ? 5 : 1;           // ratio partials: rho, ∇ (3), ∇²
    __shared__ double red[8][NR];             // per warp partials (<= 8 warps per CTA)
    const int wl = threadIdx.x / p.tpw;       // walker slot in the CTA
    const int lane = threadIdx.x - wl * p.tpw;
    const int64_t w = (int64_t)blockIdx.x * p.wpc + wl;
    const bool active = wl < p.wpc && w < p.W;

    double part[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) part[r] = 0.0;

    if (active) {
        double x[3];
        if (p.pos_f64) {
            const double *ps = static_cast<const double *>(p.pos) + w * p.pos_stride;
            x[0] = ps[0]; x[1] = ps[1]; x[2] = ps[2];
        } else {
            const float *ps = static_cast<const float *>(p.pos) + w * p.pos_stride;
            x[0] = ps[0]; x[1] = ps[1]; x[2] = ps[2];
        }
        AxisW ax, ay, az;
        axis_weights(x[0], p.L[0], p.nx, (int32_t)(p.ny * p.nz * p.nvec), ax);
        axis_weights(x[1], p.L[1], p.ny, (int32_t)(p.nz * p.nvec), ay);
        axis_weights(x[2], p.L[2], p.nz, (int32_t)p.nvec, az);
        const Vt *coef = reinterpret_cast<const Vt *>(p.coef);
        const float *arow = nullptr;
        if (p.Ainv) arow = p.Ainv + w * p.ainv_stride + (p.krow ? (int64_t)p.krow[w] * p.ainv_ld : 0);

        for (int64_t j = lane; j < p.nvec; j += p.tpw) {
            Vt acc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] = zero4<NV>();
#pragma unroll 1
            for (int a = 0; a < 4; ++a) {
                // x weights of control plane a (selects keep the arrays in registers)
                const int32_t xo = a == 0 ? ax.off[0] : a == 1 ? ax.off[1] : a == 2 ? ax.off[2] : ax.off[3];
                const float bx = a == 0 ? ax.B[0] : a == 1 ? ax.B[1] : a == 2 ? ax.B[2] : ax.B[3];
                const float dx = a == 0 ? ax.D[0] : a == 1 ? ax.D[1] : a == 2 ? ax.D[2] : ax.D[3];
                const float sx = a == 0 ? ax.S[0] : a == 1 ? ax.S[1] : a == 2 ? ax.S[2] : ax.S[3];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const Vt *col = coef + (uint32_t)(xo + ay.off[b] + (int32_t)j);
                    Vt r[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) r[c] = ld_row(col + az.off[c]);
                    Vt s0 = zero4<NV>();
#pragma unroll
                    for (int c = 0; c < 4; ++c) fma4(s0, az.B[c], r[c]);
                    const float wv = bx * ay.B[b];
                    fma4(acc[0], wv, s0);
                    if constexpr (VGH) {
                        Vt s1 = zero4<NV>(), s2 = zero4<NV>();
#pragma unroll
                        for (int c = 0; c < 4; ++c) { fma4(s1, az.D[c], r[c]); fma4(s2, az.S[c], r[c]); }
                        const float wgx = dx * ay.B[b], wgy = bx * ay.D[b];
                        const float whxx = sx * ay.B[b], whxy = dx * ay.D[b], whyy = bx * ay.S[b];
                        fma4(acc[1], wgx, s0);      // gx
                        fma4(acc[2], wgy, s0);      // gy
                        fma4(acc[3], wv, s1);       // gz
                        fma4(acc[4], whxx, s0);     // hxx
                        fma4(acc[5], whxy, s0);     // hxy
                        fma4(acc[6], wgx, s1);      // hxz
                        fma4(acc[7], whyy, s0);     // hyy
                        fma4(acc[8], wgy, s1);      // hyz
                        fma4(acc[9], wv, s2);       // hzz
                    }
                }
            }
            if (p.spo_out) {
                Vt *o = reinterpret_cast<Vt *>(p.spo_out + w * NQ * p.ld) + j;
#pragma unroll
                for (int q = 0; q < NQ; ++q) o[q * p.nvec] = acc[q];
            }
            if (arow) {
                // lanes [n_orb, ld) do not enter the ratio
                const int64_t o0 = j * NV;
                float av[NV];
#pragma unroll
                for (int e = 0; e < NV; ++e) av[e] = o0 + e < p.n_orb ? arow[o0 + e] : 0.f;
                auto dot = [&](const Vt &v) {
                    double d = 0.0;
#pragma unroll
                    for (int e = 0; e < NV; ++e) d += (double)av[e] * v.v[e];
                    return d;
                };
                part[0] += dot(acc[0]);
                if constexpr (VGH) {
                    part[1] += dot(acc[1]);
                    part[2] += dot(acc[2]);
                    part[3] += dot(acc[3]);
                    part[4] += dot(acc[4]) + dot(acc[7]) + dot(acc[9]);
                }
            }
        }
    }
    if (!p.out || !p.Ainv) return;
    // walker reduction: warps are walker-aligned (tpw is a multiple of 32)
#pragma unroll
    for (int r = 0; r < NR; ++r) part[r] = warp_sum_d(part[r]);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int r = 0; r < NR; ++r) red[warp][r] = part[r];
    }
    __syncthreads();
    if (active && lane == 0) {
        const int wpw = p.tpw >> 5, w0 = wl * wpw;
        double s[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            s[r] = 0.0;
            for (int k = 0; k < wpw; ++k) s[r] += red[w0 + k][r];
        }
        double *o = p.out + w * 5;
        o[0] = s[0];
        if constexpr (VGH) {
            const double inv = 1.0 / s[0];
            o[1] = s[1] * inv; o[2] = s[2] * inv; o[3] = s[3] * inv; o[4] = s[4] * inv;
        } else {
            o[1] = o[2] = o[3] = o[4] = 0.0;
        }
    }
}

cudaError_t launch_spo(const SpoParams &p, bool vgh, cudaStream_t s);

}  // namespace qj2
