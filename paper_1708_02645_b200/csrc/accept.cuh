// accept.cuh -- NEXT-2: the accept-side update of the per-electron J2 state
// (SURVEY.md section 8(f) NEXT-2), written for sm_100a.
//
// On acceptance of electron k's move r_k -> r'_k (Alg. 1 L9):
//   * every partner i != k: state_i += T_i(r'_k) - T_i(r_k), where
//     T_i(r) = (U, U' d/|d|, U'' + 2U'/|d|) with d = minimg(r_i - r)
//     (the 5N J2 state; the Ref updated "the column and row
//     ... for each accepted move", here on 5N accumulators);
//   * electron k: state_k = qj2_eval's (V, G, L) at r'_k (passed in: the ratio
//     step already computed it, "reuse the computed values");
//   * R[:, k] = r'_k ("both R and Rsoa (6 floats), are updated").
// Rejected walkers are untouched (their CTAs exit at once).
//
// Mapping: one CTA per (walker, tile of ATILE sources).  Every thread owns
// AVPT source vectors per iteration: it loads their x|y|z and the 5 state
// lanes (16-byte loads, L1 no-allocate), evaluates the functor twice (old and
// new partner position; same spin channel), adds the difference in T, and
// stores the 5 state lanes back (16-byte streaming stores).  HBM-bound: 12 B
// of R + 20 B read + 20 B written per source (fp32).
#pragma once

#include "qmcj2.h"
#include "j2_device.cuh"

namespace qj2 {

constexpr int ATPB = 256;     // threads per CTA
constexpr int ACCEPT_FAST_MAX_M = 16;   // fp32 geometry up to m = 16 intervals (see accept_terms_fast)
constexpr int AITER = 4;      // iterations per tile
// vectors per thread per iteration: fp32 2 (each 8 x 16-byte loads in
// flight), fp64 1 (fits 128 registers without spilling)
template <typename T> __host__ __device__ constexpr int avpt() { return sizeof(T) == 4 ? 2 : 1; }

struct AcceptParams {
    int64_t W, N_total, N_up, i_offset, N_local, Np;
    int64_t tiles_per_walker;
    int32_t m;
    double inv_delta;
    void *R;                      // [W][3][Np] in/out
    void *state;                  // [W][5][Np] in/out
    const int32_t *k;             // [W] global
    const void *r_new;            // row w at r_new + w * r_stride
    int64_t r_stride;
    const void *r_old;            // row w at r_old + w * r_old_stride (caller's, or gathered into the workspace)
    int64_t r_old_stride;
    const int32_t *accept;        // [W]
    const double *out_new;        // row w at out_new + w * out_stride: (V, Gx, Gy, Gz, L) at r'_k
    int64_t out_stride;
    // fused Metropolis (qj2_metropolis_accept): u != NULL -> accept iff u[w] < exp(2 (V_new - V_ref)),
    // V_ref = v_ref[w * v_ref_stride]; the decision is written to acc_out
    const double *u;
    const double *v_ref;
    int64_t v_ref_stride;
    int32_t *acc_out;
    double L[3];
    double pcoef[2 * (QJ2_MAX_M + 1)][4];   // power basis: [0, m] same spin, [m+1, 2m+1] opposite
};

template <typename T> struct AVec;
template <> struct AVec<float> {
    static __device__ __forceinline__ float4 ld(const float4 *p) {
        float4 v;
        asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
        return v;
    }
};
// 32-byte load / streaming store of two adjacent fp32 vectors (sm_100: LDG/STG.E.ENL2.256)
__device__ __forceinline__ void ld8(const float4 *p, float4 &a, float4 &b) {
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(p));
}
__device__ __forceinline__ void st8cs(float4 *p, const float4 &a, const float4 &b) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w) : "memory");
}
template <> struct AVec<double> {
    static __device__ __forceinline__ double2 ld(const double2 *p) {
        double2 v;
        asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
        return v;
    }
};

// r_old[w] = R[w][:, k - i_offset] for accepted walkers (unsharded callers
// that do not pass r_old).  A separate launch so that the update kernel's
// write of R[:, k] cannot race with other CTAs reading r_k.
template <typename T>
__global__ void gather_rk_kernel(const __grid_constant__ AcceptParams p, T *__restrict__ r_old) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= p.W || !p.accept[w]) return;
    const int64_t kl = (int64_t)p.k[w] - p.i_offset;
    if (kl < 0 || kl >= p.N_local) return;
    const T *Rw = static_cast<const T *>(p.R) + w * 3 * p.Np;
    for (int d = 0; d < 3; ++d) r_old[w * 3 + d] = Rw[d * p.Np + kl];
}

// fp64 geometry (AxisD, min_image_d, functor_from_r2_d): j2_device.cuh.

// Old/new functor terms of one partner; returns the (dV, dGx, dGy, dGz, dL)
// update in physical units (dead partners: exactly zero).
template <typename T>
__device__ __forceinline__ void accept_terms(T x, T y, T z, bool dead, const AxisD (&ao)[3],
                                             const AxisD (&an)[3], uint32_t base, int m, double invd64,
                                             T invd, T (&dl)[5]) {
    T t[2][5];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const AxisD(&a)[3] = s ? an : ao;
        const double ddx = min_image_d((double)x, a[0]);
        const double ddy = min_image_d((double)y, a[1]);
        const double ddz = min_image_d((double)z, a[2]);
        double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
        r2 = dead ? 1e30 : r2;                 // lands on the all-zero interval: every term 0
        T ir;
        const FunctorEval<T> e = functor_from_r2_d<T>(r2, invd64, base, m, ir);
        const T g = e.du * ir;                 // U' delta / r
        t[s][0] = e.u;
        t[s][1] = g * T(ddx);
        t[s][2] = g * T(ddy);
        t[s][3] = g * T(ddz);
        t[s][4] = fma(e.h, invd, g);           // (U'' delta^2/2)/delta + U' delta/r  -> x 2/delta = U'' + 2U'/r
    }
    dl[0] = t[1][0] - t[0][0];
    dl[1] = (t[1][1] - t[0][1]) * invd;
    dl[2] = (t[1][2] - t[0][2]) * invd;
    dl[3] = (t[1][3] - t[0][3]) * invd;
    dl[4] = (t[1][4] - t[0][4]) * (T(2) * invd);
}

// Fast path (fp32 geometry, the same arithmetic as the eval kernel): per
// pair-term error ~ (m + 4) * 2^-23 of the functor scale -- within the 1e-5
// per-entry bar for m <= 16 (measured 4e-6 at m = 8 and 16, 3e-5 at m = 64);
// finer functor grids take accept_terms above (the host picks by m).
template <typename T>
__device__ __forceinline__ void accept_terms_fast(T x, T y, T z, bool dead, const Axis<T> (&ao)[3],
                                                  const Axis<T> (&an)[3], uint32_t base,
                                                  typename Traits<T>::U clamp, T invd, T (&dl)[5]) {
    using Tr = Traits<T>;
    T t[2][5];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const Axis<T>(&a)[3] = s ? an : ao;
        const T dx = min_image(x, a[0]);
        const T dy = min_image(y, a[1]);
        const T dz = min_image(z, a[2]);
        T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        r2 = dead ? T(1e30) : r2;              // lands on the all-zero interval: every term 0
        const T ir = Tr::rsqrt(r2);
        const FunctorEval<T> e = functor_from_t<T>(r2 * ir * invd, base, clamp);
        const T g = e.du * ir;                 // U' delta / r
        t[s][0] = e.u;
        t[s][1] = g * dx;
        t[s][2] = g * dy;
        t[s][3] = g * dz;
        t[s][4] = fma(e.h, invd, g);
    }
    dl[0] = t[1][0] - t[0][0];
    dl[1] = (t[1][1] - t[0][1]) * invd;
    dl[2] = (t[1][2] - t[0][2]) * invd;
    dl[3] = (t[1][3] - t[0][3]) * invd;
    dl[4] = (t[1][4] - t[0][4]) * (T(2) * invd);
}

// PREC: fp64 geometry (accept_terms) instead of the fp32 fast path.  V8 (fp32, rows 32-byte
// aligned): a thread's two vectors per iteration are adjacent and move with 256-bit loads and
// stores.
template <typename T, bool PREC, bool V8 = false>
__global__ void __launch_bounds__(ATPB, sizeof(T) == 4 ? 2 : 1)
j2_accept_kernel(const __grid_constant__ AcceptParams p) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    constexpr int AVPT = avpt<T>();
    constexpr int TILE = ATPB * AVPT * AITER * VW;
    const int64_t w = (int64_t)blockIdx.x / p.tiles_per_walker;
    const int64_t tile = (int64_t)blockIdx.x - w * p.tiles_per_walker;
    QJ2_DCHECK(w < p.W && p.N_local <= p.Np && 2 * (p.m + 1) <= 2 * (QJ2_MAX_M + 1));
    if (p.u) {                                 // fused Metropolis (the same decision in every CTA of w)
        const double rho = exp(p.out_new[w * p.out_stride] - p.v_ref[w * p.v_ref_stride]);
        const bool acc = p.u[w] < rho * rho;
        if (tile == 0 && threadIdx.x == 0) p.acc_out[w] = acc ? 1 : 0;
        if (!acc) return;
    } else if (!p.accept[w]) {
        return;                                // rejected: nothing to do (Alg. 1 L9 "or reject")
    }

    __shared__ Coef4<T> tab[2 * (QJ2_MAX_M + 1)];
    for (int e = threadIdx.x; e < 2 * (p.m + 1); e += blockDim.x) {
        Coef4<T> c;
        c.a0 = T(p.pcoef[e][0]); c.a1 = T(p.pcoef[e][1]); c.a2 = T(p.pcoef[e][2]); c.a3 = T(p.pcoef[e][3]);
        tab[e] = c;
    }
    const int64_t kg = p.k[w];
    const T *rn = static_cast<const T *>(p.r_new) + w * p.r_stride;
    const T *ro = static_cast<const T *>(p.r_old) + w * p.r_old_stride;
    AxisD an[3], ao[3];
    Axis<T> fan[3], fao[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        // the cell as the kernel's type sees it (fp32 L for fp32 positions)
        const double Ld = (double)T(p.L[d]);
        an[d].c = (double)rn[d]; an[d].L = Ld; an[d].half = 0.5 * Ld;
        ao[d].c = (double)ro[d]; ao[d].L = Ld; ao[d].half = 0.5 * Ld;
        fan[d] = make_axis<T>(rn[d], T(p.L[d]));
        fao[d] = make_axis<T>(ro[d], T(p.L[d]));
    }
    const typename Tr::U clamp = (typename Tr::U)p.m;
    const bool k_up = kg < p.N_up;
    const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(tab);
    const uint32_t base_same = tab0, base_opp = tab0 + (uint32_t)((p.m + 1) * (int)sizeof(Coef4<T>));
    const uint32_t base_up = k_up ? base_same : base_opp;      // partners i < N_up
    const uint32_t base_dn = k_up ? base_opp : base_same;      // partners i >= N_up
    const T invd = T(p.inv_delta);
    const int64_t t0 = tile * TILE;                            // local index of the tile's first source
    const int64_t kl = kg - p.i_offset;                        // k's local index (may be outside the slice)
    const int64_t nl = p.N_local;
    const int64_t g_off = p.i_offset;
    __syncthreads();

    T *Rw = static_cast<T *>(p.R) + w * 3 * p.Np;
    T *Sw = static_cast<T *>(p.state) + w * 5 * p.Np;
    V *vx = reinterpret_cast<V *>(Rw), *vy = reinterpret_cast<V *>(Rw + p.Np), *vz = reinterpret_cast<V *>(Rw + 2 * p.Np);
    V *vs[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) vs[c] = reinterpret_cast<V *>(Sw + c * p.Np);

#pragma unroll 1
    for (int it = 0; it < AITER; ++it) {
        int64_t vi[AVPT];
        bool live[AVPT];
        V bx[AVPT], by[AVPT], bz[AVPT], bs[AVPT][5];
#pragma unroll
        for (int u = 0; u < AVPT; ++u) {
            const int64_t li = V8 ? t0 + (((int64_t)it * ATPB + threadIdx.x) * AVPT + u) * VW
                                  : t0 + ((int64_t)(it * AVPT + u) * ATPB + threadIdx.x) * VW;
            live[u] = li < nl;
            vi[u] = li / VW;
            QJ2_DCHECK(!live[u] || (vi[u] + 1) * VW <= p.Np);
        }
        if constexpr (V8) {
            static_assert(sizeof(T) == 4 && AVPT == 2, "V8: two fp32 vectors per thread");
            if (live[1]) {                                 // both vectors: one 32-byte access per lane
                ld8(vx + vi[0], bx[0], bx[1]);
                ld8(vy + vi[0], by[0], by[1]);
                ld8(vz + vi[0], bz[0], bz[1]);
#pragma unroll
                for (int c = 0; c < 5; ++c) ld8(vs[c] + vi[0], bs[0][c], bs[1][c]);
            } else if (live[0]) {
                bx[0] = AVec<T>::ld(vx + vi[0]);
                by[0] = AVec<T>::ld(vy + vi[0]);
                bz[0] = AVec<T>::ld(vz + vi[0]);
#pragma unroll
                for (int c = 0; c < 5; ++c) bs[0][c] = AVec<T>::ld(vs[c] + vi[0]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < AVPT; ++u) {
                if (live[u]) {
                    bx[u] = AVec<T>::ld(vx + vi[u]);
                    by[u] = AVec<T>::ld(vy + vi[u]);
                    bz[u] = AVec<T>::ld(vz + vi[u]);
#pragma unroll
                    for (int c = 0; c < 5; ++c) bs[u][c] = AVec<T>::ld(vs[c] + vi[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < AVPT; ++u) {
            if (!live[u]) continue;
            const int64_t li0 = vi[u] * VW;
            bool has_k = false;
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const int64_t li = li0 + e;
                const bool is_k = li == kl;
                has_k |= is_k;
                const bool dead = is_k || li >= nl;
                const uint32_t base = (li + g_off < p.N_up) ? base_up : base_dn;
                T dl[5];
                if constexpr (PREC)
                    accept_terms<T>(Tr::comp(bx[u], e), Tr::comp(by[u], e), Tr::comp(bz[u], e), dead, ao, an, base,
                                    p.m, p.inv_delta, invd, dl);
                else
                    accept_terms_fast<T>(Tr::comp(bx[u], e), Tr::comp(by[u], e), Tr::comp(bz[u], e), dead, fao, fan,
                                         base, clamp, invd, dl);
#pragma unroll
                for (int c = 0; c < 5; ++c) {
                    T s = Tr::comp(bs[u][c], e) + dl[c];
                    if (is_k) s = T(p.out_new[w * p.out_stride + c]);     // electron k: values at R'
                    Tr::set(bs[u][c], e, s);
                }
            }
            if (!V8) {
#pragma unroll
                for (int c = 0; c < 5; ++c) __stcs(vs[c] + vi[u], bs[u][c]);
            }
            if (has_k) {                                   // commit r'_k into Rsoa
                const int e = (int)(kl - li0);
                QJ2_DCHECK(e >= 0 && e < VW);
                V nx = bx[u], ny = by[u], nz = bz[u];
                Tr::set(nx, e, rn[0]); Tr::set(ny, e, rn[1]); Tr::set(nz, e, rn[2]);
                vx[vi[u]] = nx; vy[vi[u]] = ny; vz[vi[u]] = nz;
            }
        }
        if constexpr (V8) {
            if (live[1]) {
#pragma unroll
                for (int c = 0; c < 5; ++c) st8cs(vs[c] + vi[0], bs[0][c], bs[1][c]);
            } else if (live[0]) {
#pragma unroll
                for (int c = 0; c < 5; ++c) __stcs(vs[c] + vi[0], bs[0][c]);
            }
        }
    }
}

cudaError_t launch_accept_f32(const AcceptParams &p, void *r_old_ws, cudaStream_t s);
cudaError_t launch_accept_f64(const AcceptParams &p, void *r_old_ws, cudaStream_t s);

template <typename T>
inline int64_t accept_tile() { return (int64_t)ATPB * avpt<T>() * AITER * Traits<T>::VW; }

}  // namespace qj2
