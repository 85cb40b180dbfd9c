// sweep.cu -- the resident-walker sweep kernel (qj2_sweep) and its launch.
// The design, in order of the per-move steps, is in sweep.cuh and DESIGN.md section 7.
#include <cstdlib>

#include "sweep.cuh"

namespace qj2 {

// Template parameters:
//   TPB  threads per walker (one CTA per walker): 128 for 384 < N <= 768, else 256;
//   SPT  partners per thread, ceil(N / TPB); only the five differences
//        T_i(r'_k) - T_i(r_k) are kept per partner;
//   J1   the one-body Jastrow over the (<= 256) ions joins each move's ratio;
//   FULL N == TPB * SPT (NiO-64's 768 = 128 x 6, 1024 = 256 x 4): the shared-memory
//        layout and the partner bounds are compile-time constants.
// CTAs per SM at 128 threads: 7 without J1 (72 registers, no spills; 148 x 7 = 1036
// walkers in one wave), 8 with J1 (64 registers) -- measured: N64S 3.28 ms at 7 vs 3.52
// at 8, N64SJ 3.82 at 8 vs 3.87 at 7 (profiles/r01_s4/ab_minb.log).  QJ2_SWEEP_MINB_J1:
// A/B builds only.
#ifndef QJ2_SWEEP_MINB_J1
#define QJ2_SWEEP_MINB_J1 8
#endif
template <int TPB, int SPT, bool J1>
constexpr int sweep_minb() {
    return TPB == 128 ? (SPT <= 6 ? (J1 ? QJ2_SWEEP_MINB_J1 : 7) : 4) : (SPT <= 3 ? (J1 ? 3 : 4) : 2);
}

template <int TPB, int SPT, bool J1, bool FULL>
__global__ void __launch_bounds__(TPB, sweep_minb<TPB, SPT, J1>()) j2_sweep_kernel(const __grid_constant__ SweepParams p) {
    constexpr int NV = J1 ? 12 : 6;           // reduced values per move: dJ and the terms at r'_k (J2, J1)
    constexpr int NW = TPB / 32;
    extern __shared__ __align__(16) float sw_smem[];
    const int64_t w = blockIdx.x;
    const int N = FULL ? TPB * SPT : (int)p.N;
    // dynamic shared memory, sized by the call (every byte counts at 7-8 CTAs/SM):
    // R (SoA) [3][N] | state [5][N] | J2 table [2(m+1)] | J1 table [n_rows1] | ions [n_ions] (2 arrays)
    float *rx = sw_smem, *ry = rx + N, *rz = ry + N;
    float *st = rz + N;
    Coef4<float> *tab = reinterpret_cast<Coef4<float> *>(sw_smem + 8 * N);
    Coef4<float> *tab1 = tab + 2 * (p.m + 1);
    // per ion, resolved once: (x, y, z, 1/delta_s) and (table row base, m_s) of its species
    float4 *ion_p = reinterpret_cast<float4 *>(tab1 + (J1 ? p.n_rows1 : 0));
    uint2 *ion_c = reinterpret_cast<uint2 *>(ion_p + (J1 ? p.n_ions : 0));
    __shared__ double red2[2][NW][NV];               // double-buffered by move parity
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < 2 * (p.m + 1); e += TPB) {
        Coef4<float> c;
        c.a0 = (float)p.pcoef[e][0]; c.a1 = (float)p.pcoef[e][1];
        c.a2 = (float)p.pcoef[e][2]; c.a3 = (float)p.pcoef[e][3];
        tab[e] = c;
    }
    if constexpr (J1) {
        for (int e = tid; e < p.n_rows1; e += TPB) {
            Coef4<float> c;
            c.a0 = (float)p.pcoef1[e][0]; c.a1 = (float)p.pcoef1[e][1];
            c.a2 = (float)p.pcoef1[e][2]; c.a3 = (float)p.pcoef1[e][3];
            tab1[e] = c;
        }
        for (int j = tid; j < p.n_ions; j += TPB) {
            int sp = 0;
#pragma unroll
            for (int b = 1; b < QJ2_MAX_SPECIES; ++b) sp += (b < p.n_species && j >= p.sp_start[b]) ? 1 : 0;
            ion_p[j] = make_float4(p.ions[j], p.ions[p.Np_ion + j], p.ions[2 * p.Np_ion + j], p.sp_invd[sp]);
            ion_c[j] = make_uint2((uint32_t)__cvta_generic_to_shared(tab1) +
                                      (uint32_t)(p.sp_tab[sp] * (int)sizeof(Coef4<float>)),
                                  (uint32_t)p.sp_m[sp]);
        }
    }
    const float *Rg = p.R + w * 3 * p.Np;
    const float *Sg = p.state + w * 5 * p.Np;
    for (int i = tid; i < N; i += TPB) {
        rx[i] = Rg[i]; ry[i] = Rg[p.Np + i]; rz[i] = Rg[2 * p.Np + i];
#pragma unroll
        for (int c = 0; c < 5; ++c) st[c * N + i] = Sg[c * p.Np + i];
    }
    __syncthreads();
    const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(tab);
    const uint32_t tab_opp = tab0 + (uint32_t)((p.m + 1) * (int)sizeof(Coef4<float>));
    const unsigned clamp = (unsigned)p.m;
    const float invd = p.invd;

    for (int64_t s = 0; s < p.S; ++s) {
        // k outside [0, N) (a precondition): no partner is excluded, the move is never
        // accepted (nothing is written) and its accept entry is -1
        const int k = p.ks[s * p.W + w];
        const float *tr = p.trials + (s * p.W + w) * 6;
        Axis<float> a0[3], a1[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            a0[d] = make_axis<float>(tr[d], p.L[d]);
            a1[d] = make_axis<float>(tr[3 + d], p.L[d]);
        }
        const bool k_up = k < p.N_up;
        // 1. pair terms at r_k (q = 0) and r'_k (q = 1): their differences are kept per
        //    partner (the update), summed over partners only where a move needs the sum:
        //    dv = sum_i U(r'_k) - U(r_k) (dJ2) and acc = the terms at r'_k (state_k)
        // position-outer: only one position's axes are live (64 registers, no spills)
        float d[SPT][5];
        float dv = 0.f, acc[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) acc[c] = 0.f;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const Axis<float>(&a)[3] = q ? a1 : a0;
#pragma unroll
            for (int j = 0; j < SPT; ++j) {
                const int i = tid + j * TPB;
                const bool live = (FULL || i < N) && i != k;
                const int ii = (FULL || i < N) ? i : 0;
                const float x = rx[ii], y = ry[ii], z = rz[ii];
                const uint32_t base = ((ii < p.N_up) == k_up) ? tab0 : tab_opp;
                const float dx = min_image(x, a[0]), dy = min_image(y, a[1]), dz = min_image(z, a[2]);
                float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                r2 = live ? r2 : 1e30f;            // the zero row: every term exactly 0
                const float ir = Traits<float>::rsqrt(r2);
                const FunctorEval<float> e = functor_from_t<float>(r2 * ir * invd, base, clamp);
                const float g = e.du * ir;         // U' delta / r
                float t[5];
                t[0] = e.u;
                t[1] = g * dx;
                t[2] = g * dy;
                t[3] = g * dz;
                t[4] = fmaf(e.h, invd, g);      // (U'' + 2U'/r) * delta / 2
                if (q == 0) {
#pragma unroll
                    for (int c = 0; c < 5; ++c) d[j][c] = t[c];
                } else {
#pragma unroll
                    for (int c = 0; c < 5; ++c) {
                        d[j][c] = t[c] - d[j][c];
                        acc[c] += t[c];
                    }
                    dv += d[j][0];
                }
            }
        }
        // 1b. J1: thread tid takes ions tid, tid + TPB at both positions, in physical units
        //     (species differ in delta): dv1 = sum U(r'_k) - U(r_k); at r'_k V, G = -U' d/r,
        //     L = U'' + 2U'/r (electron k's J1 state on acceptance)
        float dv1 = 0.f, a1c[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) a1c[c] = 0.f;
        if constexpr (J1) {
#pragma unroll
            for (int ion = tid; ion < SW_MAX_IONS; ion += TPB) {
                if (ion >= p.n_ions) break;
                const float4 ip = ion_p[ion];
                const uint2 ic = ion_c[ion];
                const uint32_t base1 = ic.x;
                const float iv = ip.w;
                const float x = ip.x, y = ip.y, z = ip.z;
                float u0 = 0.f;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const Axis<float>(&a)[3] = q ? a1 : a0;
                    const float dx = min_image(x, a[0]), dy = min_image(y, a[1]), dz = min_image(z, a[2]);
                    const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                    const float ir = Traits<float>::rsqrt(r2);
                    const FunctorEval<float> e = functor_from_t<float>(r2 * ir * iv, base1, ic.y);
                    if (q == 0) {
                        u0 = e.u;
                    } else {
                        const float g = e.du * ir * iv;           // U'/r
                        dv1 += e.u - u0;
                        a1c[0] += e.u;
                        a1c[1] += -g * dx;
                        a1c[2] += -g * dy;
                        a1c[3] += -g * dz;
                        a1c[4] += 2.f * (e.h * iv * iv + g);    // U'' + 2U'/r
                    }
                }
            }
        }
        // 2. block reduction, fixed order: a reduce-scatter across the warp (8 or 16
        //    slots for 6 or 12 values: one shuffle per slot and level instead of five
        //    per value), one partial per value and warp in shared memory. Levels 1-2
        //    (lanes 16 and 8 apart) add in fp32 -- partials of <= 4 lanes x 6 terms, the
        //    eval kernel's fp32 partials of <= 32 terms -- the rest in fp64.
        {
            constexpr int NS = J1 ? 16 : 8;
            constexpr int OREM = J1 ? 1 : 2;        // lanes below this distance hold copies of one slot
            float vf[NS];
            vf[0] = dv;
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                vf[1 + c] = acc[c];
                if (J1) vf[7 + c] = a1c[c];
            }
            if (J1) vf[6] = dv1;
#pragma unroll
            for (int c = NV; c < NS; ++c) vf[c] = 0.f;
            int slot = 0;
#pragma unroll
            for (int h = NS / 2, o = 16; o >= 8; h >>= 1, o >>= 1) {
                const bool up = lane & o;           // this lane keeps the upper half of the slots
#pragma unroll
                for (int j = 0; j < h; ++j) {
                    const float send = up ? vf[j] : vf[j + h];
                    const float keep = up ? vf[j + h] : vf[j];
                    vf[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
                slot += up ? h : 0;
            }
            double v[NS / 4];
#pragma unroll
            for (int j = 0; j < NS / 4; ++j) v[j] = (double)vf[j];
#pragma unroll
            for (int h = NS / 8, o = 4; h >= 1; h >>= 1, o >>= 1) {
                const bool up = lane & o;
#pragma unroll
                for (int j = 0; j < h; ++j) {
                    const double send = up ? v[j] : v[j + h];
                    const double keep = up ? v[j + h] : v[j];
                    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
                slot += up ? h : 0;
            }
#pragma unroll
            for (int o = OREM; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
            if ((lane & (2 * OREM - 1)) == 0 && slot < NV) red2[s & 1][warp][slot] = v[0];
        }
        __syncthreads();
        // 3. Metropolis: every thread sums dJ and takes the same decision (no second
        //    barrier); thread 0 records it
        double (*red)[NV] = red2[s & 1];
        double djs = 0.0;
#pragma unroll
        for (int wi = 0; wi < NW; ++wi) {
            djs += red[wi][0];
            if (J1) djs += red[wi][6];              // dJ = dJ2 + dJ1 (Eq. 4-5)
        }
        // u < exp(2 dJ2): an fp32 exp settles it unless u is within 1e-4 of the threshold (its
        // relative error is < 2e-5 for |dJ2| < 100) or the fp32 value over/underflows; then fp64.
        // Either way the decision equals the fp64 test.
        const double uu = p.u[s * p.W + w];
        const float e32 = __expf(2.f * (float)djs);
        bool accepted;
        if (isfinite(e32) && e32 > 1e-30f && fabs((float)uu - e32) > 1e-4f * e32 && fabs(djs) < 100.0) {
            accepted = (float)uu < e32;
        } else {
            const double rho = exp(djs);
            accepted = uu < rho * rho;
        }
        const bool k_ok = (unsigned)k < (unsigned)N;
        accepted = accepted && k_ok;
        if (tid == 0) {
            p.acc[s * p.W + w] = k_ok ? (accepted ? 1 : 0) : -1;
            if (p.dj) p.dj[s * p.W + w] = djs;
        }
        // 4. accept: partners from the kept terms, then electron k and its position
        if (accepted) {
            const float sg = invd, sl = 2.f * invd;
#pragma unroll
            for (int j = 0; j < SPT; ++j) {
                const int i = tid + j * TPB;
                if ((FULL || i < N) && i != k) {
                    st[0 * N + i] += d[j][0];
                    st[1 * N + i] += d[j][1] * sg;
                    st[2 * N + i] += d[j][2] * sg;
                    st[3 * N + i] += d[j][3] * sg;
                    st[4 * N + i] += d[j][4] * sl;
                }
            }
            if (tid == k % TPB) {     // the thread that owns slot k (no cross-thread writes)
                // state_k = (V, G, L) at r'_k: G = -invd * sum g d, L = 2 invd * sum (h invd + g)
                double f[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int wi = 0; wi < NW; ++wi)
#pragma unroll
                    for (int c = 0; c < 5; ++c) f[c] += red[wi][1 + c];
                st[0 * N + k] = (float)f[0];
                st[1 * N + k] = (float)(-p.inv_delta * f[1]);
                st[2 * N + k] = (float)(-p.inv_delta * f[2]);
                st[3 * N + k] = (float)(-p.inv_delta * f[3]);
                st[4 * N + k] = (float)(2.0 * p.inv_delta * f[4]);
                rx[k] = tr[3]; ry[k] = tr[4]; rz[k] = tr[5];
                if constexpr (J1) {                  // electron k's J1 state: U^1_k and derivatives at r'_k
                    double f1[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int wi = 0; wi < NW; ++wi)
#pragma unroll
                        for (int c = 0; c < 5; ++c) f1[c] += red[wi][7 + c];
                    float *S1 = p.state_j1 + w * 5 * p.Np;
#pragma unroll
                    for (int c = 0; c < 5; ++c) S1[c * p.Np + k] = (float)f1[c];
                }
            }
        }
        // no barrier: every thread only touches its own slots of R and the state,
        // and the partials are double-buffered (a warp writes red2[s & 1] again at
        // move s + 2, after every thread has passed the barrier of move s + 1)
    }
    float *Rw = p.R + w * 3 * p.Np;
    float *Sw = p.state + w * 5 * p.Np;
    for (int i = tid; i < N; i += TPB) {
        Rw[i] = rx[i]; Rw[p.Np + i] = ry[i]; Rw[2 * p.Np + i] = rz[i];
#pragma unroll
        for (int c = 0; c < 5; ++c) Sw[c * p.Np + i] = st[c * N + i];
    }
}

cudaError_t launch_sweep(const SweepParams &p, cudaStream_t s) {
    const bool j1 = p.n_ions > 0;
    const size_t smem = (size_t)8 * p.N * sizeof(float)                       // R (3) + state (5) per electron
                      + (size_t)(2 * (p.m + 1) + (j1 ? p.n_rows1 : 0)) * sizeof(Coef4<float>)
                      + (j1 ? (size_t)p.n_ions * (sizeof(float4) + sizeof(uint2)) : 0);
    // 128 threads per walker for 384 < N <= 768 (7-8 CTAs/SM), else 256 (64 and 96
    // threads per walker were measured too: profiles/r01_s4/ab_tpb.log)
    int tpb = (p.N > 384 && p.N <= 768) ? 128 : SW_TPB;
    if (const char *e = getenv("QJ2_SWEEP_TPB")) tpb = atoi(e) == 128 && p.N <= 768 ? 128 : SW_TPB;   // A/B
    const int spt = (int)((p.N + tpb - 1) / tpb);
    // compile-time layout where N fills the threads exactly (N64SJ 4.39 -> 3.98 ms, N64S at 7
    // CTAs/SM 3.40 -> 3.28 ms)
    const bool full = p.N == (int64_t)tpb * spt && !getenv("QJ2_SWEEP_NOFULL");
#define QJ2_SWEEP_LAUNCH(T_, S_)                                                            \
    (j1 ? (j2_sweep_kernel<T_, S_, true, false><<<(unsigned)p.W, T_, smem, s>>>(p), 0)       \
        : (j2_sweep_kernel<T_, S_, false, false><<<(unsigned)p.W, T_, smem, s>>>(p), 0))
#define QJ2_SWEEP_LAUNCH_FULL(T_, S_)                                                       \
    (j1 ? (j2_sweep_kernel<T_, S_, true, true><<<(unsigned)p.W, T_, smem, s>>>(p), 0)        \
        : (j2_sweep_kernel<T_, S_, false, true><<<(unsigned)p.W, T_, smem, s>>>(p), 0))
    if (tpb == 128) {
        switch (spt) {
            case 1: case 2: case 3: case 4: QJ2_SWEEP_LAUNCH(128, 4); break;
            case 5: QJ2_SWEEP_LAUNCH(128, 5); break;
            default:
                if (full) QJ2_SWEEP_LAUNCH_FULL(128, 6);
                else QJ2_SWEEP_LAUNCH(128, 6);
                break;
        }
    } else {
        switch (spt) {
            case 1: QJ2_SWEEP_LAUNCH(256, 1); break;
            case 2: QJ2_SWEEP_LAUNCH(256, 2); break;
            case 3: QJ2_SWEEP_LAUNCH(256, 3); break;
            default:
                if (full) QJ2_SWEEP_LAUNCH_FULL(256, 4);
                else QJ2_SWEEP_LAUNCH(256, 4);
                break;
        }
    }
#undef QJ2_SWEEP_LAUNCH
#undef QJ2_SWEEP_LAUNCH_FULL
    return cudaGetLastError();
}

}  // namespace qj2
