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
#include "j2_device.cuh"
#include "bulk.cuh"
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
    int64_t ppw;                                // evaluations per walker (A^{-1} row of walker w / ppw)
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
    // a non-finite coordinate gathers row 0 with NaN weights (NaN outputs, no stray address)
    const bool fin = isfinite(x);
    double xw = fin ? fmod(x, L) : 0.0;
    if (xw < 0) xw += L;
    const double u = xw / L * (double)n;
    double fi = floor(u);
    const double t = fin ? u - fi : __longlong_as_double(0x7ff8000000000000ll);
    int64_t i = (int64_t)fi;
    if (i >= n) i -= n;
    i = (i < 0 || i >= n) ? 0 : i;
    for (int c = 0; c < 4; ++c) {
        int64_t j = i - 1 + c;
        j = j < 0 ? j + n : (j >= n ? j - n : j);
        QJ2_DCHECK(j >= 0 && j < n);
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
        if (p.Ainv) {
            const int64_t wa = w / p.ppw;
            arow = p.Ainv + wa * p.ainv_stride + (p.krow ? (int64_t)p.krow[wa] * p.ainv_ld : 0);
        }

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

// ===========================================================================
// TMA-pipelined variant (the default when a walker's orbitals fit one pass of
// the consumer warps): persistent CTAs, one producer warp gathers each
// walker's coefficient block plane by plane (x plane a = 0..3: 16 rows of
// ld floats; the 4 z rows of an (a, b) column are one contiguous bulk copy
// unless z wraps) into a ring of NST shared-memory stages with
// cp.async.bulk + mbarrier complete_tx; NC consumer warps (one vector of NV
// orbitals per thread) read the rows from shared memory.  The producer also
// computes the walker's basis weights (fp64 -> fp32) into the stage header,
// loading 32 walkers' positions per warp-wide load.  Per SM up to NST stages
// (~190 KB) of gathers are in flight instead of ~50 KB of LDGs.
// ===========================================================================
constexpr int SPO_HDR = 48;                   // floats per stage header (36 weights, padded to 192 B)
constexpr int SPO_MAXC = 16;                  // consumer warps per CTA, at most
// Orbitals per consumer thread (2: one orbital per thread measured 1.4x slower
// for vgh -- per-row overhead no longer amortised).
template <bool VGH> __host__ __device__ constexpr int spo_tma_nv() { return 2; }

template <bool VGH, int NR>
__device__ __forceinline__ void spo_finalize(const SpoParams &p, const double *red, uint32_t rbar, int NC,
                                             int64_t i, int64_t w) {
    const uint32_t slot = (uint32_t)(i & 1), use = (uint32_t)(i >> 1);
    mbar_wait(rbar + 8 * slot, use & 1);
    const double *rb = red + slot * SPO_MAXC * NR;
    double s[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        s[r] = 0.0;
        for (int k = 0; k < NC; ++k) s[r] += rb[k * NR + r];
    }
    mbar_arrive(rbar + 8 * (2 + slot));
    double *o = p.out + w * 5;
    o[0] = s[0];
    if constexpr (VGH) {
        const double inv = 1.0 / s[0];
        o[1] = s[1] * inv; o[2] = s[2] * inv; o[3] = s[3] * inv; o[4] = s[4] * inv;
    } else {
        o[1] = o[2] = o[3] = o[4] = 0.0;
    }
}

template <bool VGH>
__global__ void spo_tma_kernel(const __grid_constant__ SpoParams p, int nst) {
    constexpr int NV = spo_tma_nv<VGH>();    // orbitals per consumer thread
    using Vt = FV<NV>;
    constexpr int NQ = VGH ? 10 : 1;
    constexpr int NR = VGH ? 5 : 1;
    const int NC = blockDim.x / 32 - 1;       // consumer warps (<= SPO_MAXC)
    const int64_t ld = p.ld;
    const uint32_t stage_bytes = (uint32_t)(16 * ld * 4);

    extern __shared__ __align__(128) unsigned char smem[];
    float *ring = reinterpret_cast<float *>(smem);                                        // [nst][16][ld]
    float *hdr = reinterpret_cast<float *>(smem + (size_t)nst * stage_bytes);             // [nst][SPO_HDR]
    uint64_t *bars = reinterpret_cast<uint64_t *>(hdr + (size_t)nst * SPO_HDR);          // full[nst], empty[nst]
    double *red = reinterpret_cast<double *>(bars + 2 * nst);                             // [2][SPO_MAXC][NR]
    const uint32_t rbar = (uint32_t)__cvta_generic_to_shared(red + 2 * SPO_MAXC * NR);    // full[2], empty[2]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
    const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(ring);
    if (threadIdx.x == 0) {
        for (int st = 0; st < nst; ++st) {
            mbar_init(bar0 + 8 * st, 1);                  // full: the producer's expect_tx arrival
            mbar_init(bar0 + 8 * (nst + st), NC);         // empty: one arrival per consumer warp
        }
        for (int sl = 0; sl < 2; ++sl) {
            mbar_init(rbar + 8 * sl, NC);                 // ratio partials published by every consumer warp
            mbar_init(rbar + 8 * (2 + sl), 1);            // ... and read by the finalizer
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t G = gridDim.x;

    // =====================  producer warp  =====================
    if (warp == NC) {
        uint32_t n = 0;
        const int32_t sx = (int32_t)(p.ny * p.nz * ld), sy = (int32_t)(p.nz * ld);
        for (int64_t base = blockIdx.x; base < p.W; base += 32 * G) {
            // lane l prepares walker base + l*G (one warp-wide position load per 32 walkers)
            const int64_t wl = base + lane * G;
            float wts[36];
            int32_t i0[3] = {0, 0, 0};
            if (wl < p.W) {
                double x[3];
                if (p.pos_f64) {
                    const double *ps = static_cast<const double *>(p.pos) + wl * p.pos_stride;
                    x[0] = ps[0]; x[1] = ps[1]; x[2] = ps[2];
                } else {
                    const float *ps = static_cast<const float *>(p.pos) + wl * p.pos_stride;
                    x[0] = ps[0]; x[1] = ps[1]; x[2] = ps[2];
                }
                const int64_t nn[3] = {p.nx, p.ny, p.nz};
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    AxisW a;
                    axis_weights(x[d], p.L[d], nn[d], 1, a);
                    i0[d] = a.off[1];                      // control point of a = 1 is the cell index i
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        wts[d * 12 + c] = a.B[c];
                        wts[d * 12 + 4 + c] = a.D[c];
                        wts[d * 12 + 8 + c] = a.S[c];
                    }
                }
            }
            for (int qw = 0; qw < 32; ++qw) {
                const int64_t w = base + qw * G;
                if (w >= p.W) break;
                const int32_t ix = __shfl_sync(0xffffffffu, i0[0], qw);
                const int32_t iy = __shfl_sync(0xffffffffu, i0[1], qw);
                const int32_t iz = __shfl_sync(0xffffffffu, i0[2], qw);
                const bool zc = iz >= 1 && iz + 2 < p.nz;        // the 4 z rows are contiguous
                for (int a = 0; a < 4; ++a, ++n) {
                    const uint32_t slot = n % (uint32_t)nst, round = n / (uint32_t)nst;
                    mbar_wait(bar0 + 8 * (nst + slot), (round & 1) ^ 1);
                    if (lane == qw) {
                        // header of plane a: per column b the 6 (x, y) weights (wv, wgx, wgy,
                        // whxx, whxy, whyy), then the 12 z weights (B, B', B'')
                        float *h = hdr + slot * SPO_HDR;
                        const float bx = a == 0 ? wts[0] : a == 1 ? wts[1] : a == 2 ? wts[2] : wts[3];
                        const float dx = a == 0 ? wts[4] : a == 1 ? wts[5] : a == 2 ? wts[6] : wts[7];
                        const float sx = a == 0 ? wts[8] : a == 1 ? wts[9] : a == 2 ? wts[10] : wts[11];
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            h[b * 6 + 0] = bx * wts[12 + b];
                            h[b * 6 + 1] = dx * wts[12 + b];
                            h[b * 6 + 2] = bx * wts[16 + b];
                            h[b * 6 + 3] = sx * wts[12 + b];
                            h[b * 6 + 4] = dx * wts[16 + b];
                            h[b * 6 + 5] = bx * wts[20 + b];
                        }
#pragma unroll
                        for (int e = 0; e < 12; ++e) h[24 + e] = wts[24 + e];
                    }
                    __syncwarp();
                    const uint32_t full = bar0 + 8 * slot;
                    if (lane == 0) mbar_expect_tx(full, stage_bytes);   // also the producer's arrival
                    __syncwarp();
                    int32_t xa = ix - 1 + a;
                    xa = xa < 0 ? xa + (int32_t)p.nx : (xa >= p.nx ? xa - (int32_t)p.nx : xa);
                    if (lane < 16) {                          // lane = b*4 + c: row (b, c) of plane a
                        const int b = lane >> 2, c = lane & 3;
                        int32_t yb = iy - 1 + b;
                        yb = yb < 0 ? yb + (int32_t)p.ny : (yb >= p.ny ? yb - (int32_t)p.ny : yb);
                        int32_t zc0 = iz - 1 + c;
                        zc0 = zc0 < 0 ? zc0 + (int32_t)p.nz : (zc0 >= p.nz ? zc0 - (int32_t)p.nz : zc0);
                        const uint32_t dst = ring0 + slot * stage_bytes + (uint32_t)(lane * ld * 4);
                        if (zc) {
                            if (c == 0)
                                bulk_g2s(dst, p.coef + ((int64_t)xa * sx + (int64_t)yb * sy + (int64_t)zc0 * ld),
                                         (uint32_t)(4 * ld * 4), full);
                        } else {
                            bulk_g2s(dst, p.coef + ((int64_t)xa * sx + (int64_t)yb * sy + (int64_t)zc0 * ld),
                                     (uint32_t)(ld * 4), full);
                        }
                    }
                }
            }
        }
        return;
    }

    // =====================  consumer warps  =====================
    const int t = threadIdx.x;                  // consumer thread: orbital vector j = t
    const int64_t nvec = ld / NV;
    const bool has = t < nvec;
    uint32_t n = 0;
    int64_t it = 0, w_prev = -1;
    for (int64_t w = blockIdx.x; w < p.W; w += G, ++it) {
        // A^{-1} row entries of this thread's orbitals (used after the gather)
        float av[NV];
        const int64_t wa = w / p.ppw;
        const float *arow = p.Ainv ? p.Ainv + wa * p.ainv_stride + (p.krow ? (int64_t)p.krow[wa] * p.ainv_ld : 0)
                                   : nullptr;
#pragma unroll
        for (int e = 0; e < NV; ++e) {
            const int64_t o = (int64_t)t * NV + e;
            av[e] = (arow && has && o < p.n_orb) ? __ldg(arow + o) : 0.f;
        }
        Vt acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = zero4<NV>();
        for (int a = 0; a < 4; ++a, ++n) {
            const uint32_t slot = n % (uint32_t)nst, round = n / (uint32_t)nst;
            mbar_wait(bar0 + 8 * slot, round & 1);
            const float4 *h4 = reinterpret_cast<const float4 *>(hdr + slot * SPO_HDR);
            float hw[36];
#pragma unroll
            for (int e = 0; e < 9; ++e) {
                const float4 v = h4[e];
                hw[4 * e] = v.x; hw[4 * e + 1] = v.y; hw[4 * e + 2] = v.z; hw[4 * e + 3] = v.w;
            }
            if (has) {
                const Vt *st = reinterpret_cast<const Vt *>(ring + (size_t)slot * 16 * ld) + t;
                const int64_t rs = ld / NV;           // row stride in vectors
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    Vt r[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) r[c] = st[(b * 4 + c) * rs];
                    Vt s0 = zero4<NV>();
#pragma unroll
                    for (int c = 0; c < 4; ++c) fma4(s0, hw[24 + c], r[c]);
                    const float wv = hw[b * 6 + 0];
                    fma4(acc[0], wv, s0);
                    if constexpr (VGH) {
                        Vt s1 = zero4<NV>(), s2 = zero4<NV>();
#pragma unroll
                        for (int c = 0; c < 4; ++c) { fma4(s1, hw[28 + c], r[c]); fma4(s2, hw[32 + c], r[c]); }
                        const float wgx = hw[b * 6 + 1], wgy = hw[b * 6 + 2];
                        fma4(acc[1], wgx, s0);
                        fma4(acc[2], wgy, s0);
                        fma4(acc[3], wv, s1);
                        fma4(acc[4], hw[b * 6 + 3], s0);
                        fma4(acc[5], hw[b * 6 + 4], s0);
                        fma4(acc[6], wgx, s1);
                        fma4(acc[7], hw[b * 6 + 5], s0);
                        fma4(acc[8], wgy, s1);
                        fma4(acc[9], wv, s2);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bar0 + 8 * (nst + slot));
        }
        if (has && p.spo_out) {
            Vt *o = reinterpret_cast<Vt *>(p.spo_out + w * NQ * ld) + t;
#pragma unroll
            for (int q = 0; q < NQ; ++q) o[q * nvec] = acc[q];
        }
        if (!p.out || !p.Ainv) continue;
        double part[NR];
        auto dot = [&](const Vt &v) {
            double d = 0.0;
#pragma unroll
            for (int e = 0; e < NV; ++e) d += (double)av[e] * v.v[e];
            return d;
        };
        part[0] = dot(acc[0]);
        if constexpr (VGH) {
            part[1] = dot(acc[1]); part[2] = dot(acc[2]); part[3] = dot(acc[3]);
            part[4] = dot(acc[4]) + dot(acc[7]) + dot(acc[9]);
        }
        // partials -> 2-slot ring in shared memory (full: NC warp arrivals,
        // empty: the finalizer's arrival); thread 0 finalizes walker i - 1
        // after publishing walker i, so no warp waits for the others here.
        const uint32_t slot = (uint32_t)(it & 1), use = (uint32_t)(it >> 1);
        double *rb = red + slot * SPO_MAXC * NR;
        if (lane == 0) mbar_wait(rbar + 8 * (2 + slot), (use & 1) ^ 1);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const double v = warp_sum_d(part[r]);
            if (lane == 0) rb[warp * NR + r] = v;
        }
        if (lane == 0) mbar_arrive(rbar + 8 * slot);
        if (t == 0 && it > 0) spo_finalize<VGH, NR>(p, red, rbar, NC, it - 1, w_prev);
        w_prev = w;
    }
    if (t == 0 && it > 0 && p.out && p.Ainv) spo_finalize<VGH, NR>(p, red, rbar, NC, it - 1, w_prev);
}

cudaError_t launch_spo(const SpoParams &p, bool vgh, bool force_ldg, cudaStream_t s);

}  // namespace qj2
