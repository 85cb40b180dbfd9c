// sweep.cu -- the resident-walker sweep kernel (qj2_sweep), the from-scratch
// state kernel (qj2_state_init) and their launches.  The design, in order of
// the per-move steps, is in sweep.cuh and DESIGN.md section 7.
#include "sweep.cuh"

namespace qj2 {

// Template parameters of the sweep kernel:
//   TPB  threads per walker (one CTA per walker): 64 for N <= 768, else 128;
//   SPT  partners per thread (a tier >= ceil(N / TPB)); the five pair terms at r'_k are
//        kept per partner between the ratio and the update;
//   J1   the one-body Jastrow over the (<= 256) ions joins each move's ratio;
//   FULL N == TPB * SPT with N_up = N / 2 and SPT even (NiO-64's 768 = 64 x 12, 1024 =
//        128 x 8): the shared-memory layout, the partner bounds and every partner's spin
//        half (j < SPT/2: up) are compile-time constants.
// NiO-64: 64 threads x 12 partners at <= 128 registers, 7 CTAs per SM, 148 x 7 = 1036
// walkers in one wave.
// Threads x partners per walker: 64 x 4 / 6 / 8 / 10 / 12 for N <= 768 (two warps per walker:
// the per-move work -- proposal, axes, reduction, decision -- is shared by 4-12 partners per
// thread), 128 x 8 for 768 < N <= 1024.  Resident CTAs per SM so that the register file holds
// the SPT x 5 pair terms kept between the ratio and the update.
template <int TPB, int SPT, bool J1>
constexpr int sweep_minb() {
    if (TPB == 64) return SPT <= 4 ? 12 : SPT <= 8 ? 10 : SPT <= 10 ? 8 : (J1 ? 8 : 7);
    return 5;   // 128 x 8
}

// The proposal of Alg. 1 L5 without drift (reading R24): r + delta in fp32, wrapped
// into [0, L) (|delta| < L): the oracle's orc_propose_f32, operation for operation.
__device__ __forceinline__ float propose(float r, float d, float L) {
    float x = __fadd_rn(r, d);
    if (x < 0.0f) x = __fadd_rn(x, L);
    if (x >= L) x = __fadd_rn(x, -L);
    return x;
}

// Pair terms of one partner at (x, y, z) against a position's axes, with the eval
// kernel's fp32 arithmetic, in raw units: t = (U, g dx, g dy, g dz, h invd + g),
// g = U' delta / r, h = U'' delta^2 / 2, d = partner - position.  A dead partner
// (r^2 forced to 1e30, i.e. onto the all-zero interval) gives exactly 0.
__device__ __forceinline__ void pair_raw(float x, float y, float z, const Axis<float> (&a)[3], bool live,
                                         uint32_t base, unsigned clamp, float invd, float (&t)[5]) {
    const float dx = min_image(x, a[0]), dy = min_image(y, a[1]), dz = min_image(z, a[2]);
    float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    r2 = live ? r2 : 1e30f;
    const float ir = Traits<float>::rsqrt(r2);
    const FunctorEval<float> e = functor_from_t<float>(r2 * ir * invd, base, clamp);
    const float g = e.du * ir;
    t[0] = e.u;
    t[1] = g * dx;
    t[2] = g * dy;
    t[3] = g * dz;
    t[4] = fmaf(e.h, invd, g);
}

// Shared-memory staging common to both kernels: the J2 power-basis table (same-spin
// rows [0, m], opposite-spin rows [m+1, 2m+1]) and, with J1, the species tables and
// per ion (x, y, z, 1/delta_s) and (table row address, m_s) of its species.
template <bool J1>
__device__ __forceinline__ void stage_tables(const SweepParams &p, Coef4<float> *tab, Coef4<float> *tab1,
                                             float4 *ion_p, uint2 *ion_c, int tid, int nthr) {
    for (int e = tid; e < 2 * (p.m + 1); e += nthr) {
        Coef4<float> c;
        c.a0 = (float)p.pcoef[e][0]; c.a1 = (float)p.pcoef[e][1];
        c.a2 = (float)p.pcoef[e][2]; c.a3 = (float)p.pcoef[e][3];
        tab[e] = c;
    }
    if constexpr (J1) {
        for (int e = tid; e < p.n_rows1; e += nthr) {
            Coef4<float> c;
            c.a0 = (float)p.pcoef1[e][0]; c.a1 = (float)p.pcoef1[e][1];
            c.a2 = (float)p.pcoef1[e][2]; c.a3 = (float)p.pcoef1[e][3];
            tab1[e] = c;
        }
        for (int j = tid; j < p.n_ions; j += nthr) {
            int sp = 0;
#pragma unroll
            for (int b = 1; b < QJ2_MAX_SPECIES; ++b) sp += (b < p.n_species && j >= p.sp_start[b]) ? 1 : 0;
            ion_p[j] = make_float4(p.ions[j], p.ions[p.Np_ion + j], p.ions[2 * p.Np_ion + j], p.sp_invd[sp]);
            ion_c[j] = make_uint2((uint32_t)__cvta_generic_to_shared(tab1) +
                                      (uint32_t)(p.sp_tab[sp] * (int)sizeof(Coef4<float>)),
                                  (uint32_t)p.sp_m[sp]);
        }
    }
}

// Moves s0 .. s0 + SW_MCH - 1 (those < S) of walker w into shared memory: k, delta, u.
constexpr int SW_MCH = 32;
__device__ __forceinline__ void stage_moves(const SweepParams &p, int w, int64_t s0, int *mk, float (*md)[3],
                                            double *mu, int tid, int nthr) {
    for (int e = tid; e < 5 * SW_MCH; e += nthr) {
        const int j = e < SW_MCH ? e : (e < 4 * SW_MCH ? (e - SW_MCH) / 3 : e - 4 * SW_MCH);
        const int64_t s = s0 + j;
        if (s >= p.S) continue;
        const int64_t sw = s * p.W + w;
        if (e < SW_MCH) mk[j] = p.ks[sw];
        else if (e < 4 * SW_MCH) { const int c = (e - SW_MCH) % 3; md[j][c] = p.delta[sw * 3 + c]; }
        else mu[j] = p.u[sw];
    }
}

template <int TPB, int SPT, bool J1, bool FULL>
__global__ void __launch_bounds__(TPB, sweep_minb<TPB, SPT, J1>()) j2_sweep_kernel(const __grid_constant__ SweepParams p) {
    constexpr int NV = J1 ? 11 : 5;           // reduced values: sums at r'_k (J2: V, Gx, Gy, Gz, L); J1: dJ1 + 5
    constexpr int NW = TPB / 32;
    extern __shared__ __align__(16) float sw_smem[];
    const int w = blockIdx.x;
    const int N = FULL ? TPB * SPT : p.N;
    // dynamic shared memory, sized by the call (every byte counts at 7 CTAs/SM), one 16-byte
    // vector per electron and array, so a partner is one LDS.128 (and its state one more):
    // P4 [N] = (x, y, z, L) | S4 [N] = (V, Gx, Gy, Gz) (state in physical units) |
    // J2 table [2(m+1)] | J1 table | ions (2 arrays)
    float4 *P4 = reinterpret_cast<float4 *>(sw_smem);
    float4 *S4 = P4 + N;
    Coef4<float> *tab = reinterpret_cast<Coef4<float> *>(sw_smem + 8 * N);
    Coef4<float> *tab1 = tab + 2 * (p.m + 1);
    float4 *ion_p = reinterpret_cast<float4 *>(tab1 + (J1 ? p.n_rows1 : 0));
    uint2 *ion_c = reinterpret_cast<uint2 *>(ion_p + (J1 ? p.n_ions : 0));
    __shared__ double red2[2][NW][NV];               // double-buffered by move parity
    __shared__ float vk2[2];                         // U^2_k(R) published by the owner of slot k
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    QJ2_DCHECK(w < p.W && N <= p.Np && N == p.N && p.n_ions <= SW_MAX_IONS && p.S <= 0x7fffffff &&
               (uint32_t)((8 * N) * sizeof(float) + (2 * (p.m + 1) + (J1 ? p.n_rows1 : 0)) * sizeof(Coef4<float>) +
                          (J1 ? p.n_ions * (sizeof(float4) + sizeof(uint2)) : 0)) <= dyn_smem_bytes());
    stage_tables<J1>(p, tab, tab1, ion_p, ion_c, tid, TPB);
    const float *Rg = p.R + (int64_t)w * 3 * p.Np;
    const float *Sg = p.state + (int64_t)w * 5 * p.Np;
    for (int i = tid; i < N; i += TPB) {
        P4[i] = make_float4(Rg[i], Rg[p.Np + i], Rg[2 * p.Np + i], Sg[4 * p.Np + i]);
        S4[i] = make_float4(Sg[i], Sg[p.Np + i], Sg[2 * p.Np + i], Sg[3 * p.Np + i]);
    }
    __shared__ int mv_k[2][SW_MCH];
    __shared__ float mv_d[2][SW_MCH][3];
    __shared__ double mv_u[2][SW_MCH];
    stage_moves(p, w, 0, mv_k[0], mv_d[0], mv_u[0], tid, TPB);
    __syncthreads();
    const uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab);
    const uint32_t tab_o = tab_s + (uint32_t)((p.m + 1) * (int)sizeof(Coef4<float>));
    const unsigned clamp = (unsigned)p.m;
    const float invd = p.invd, sl = 2.f * p.invd;
    const int n_up = p.N_up;
    const float L0 = p.L[0], L1 = p.L[1], L2 = p.L[2];

    int prev_k = -1;
    bool prev_acc = false;
    const int S = (int)p.S;
    for (int s = 0; s < S; ++s) {
        const int b = (s / SW_MCH) & 1, jm = s % SW_MCH;
        // the moves are staged SW_MCH at a time: chunk c + 1 is loaded during the second
        // move of chunk c, into the buffer of chunk c - 1 (whose last reads, u after the
        // barrier of move SW_MCH*c - 1, precede the barrier of move SW_MCH*c); it is
        // visible after that move's barrier
        if (jm == 1 && s - 1 + SW_MCH < S)
            stage_moves(p, w, s - 1 + SW_MCH, mv_k[b ^ 1], mv_d[b ^ 1], mv_u[b ^ 1], tid, TPB);
        const int k = mv_k[b][jm];
        const float dlx = mv_d[b][jm][0], dly = mv_d[b][jm][1], dlz = mv_d[b][jm][2];
        // k outside [0, N) (a precondition): the move is never accepted and flagged -1
        const bool k_ok = (unsigned)k < (unsigned)N;
        const int kk = k_ok ? k : 0;
        QJ2_DCHECK(kk >= 0 && kk < N && jm < SW_MCH);
        // r_k was written by its owner in the previous move (the same electron moved
        // twice in a row): make the write visible before everyone reads it
        if (kk == prev_k && prev_acc) __syncthreads();
        const float4 pk = P4[kk];
        const float xk = pk.x, yk = pk.y, zk = pk.z;
        const float xn = propose(xk, dlx, L0), yn = propose(yk, dly, L1), zn = propose(zk, dlz, L2);
        const bool k_up = kk < n_up;
        const uint32_t bu = k_up ? tab_s : tab_o, bd = k_up ? tab_o : tab_s;   // partner spin up / down
        if (tid == (kk & (TPB - 1))) vk2[s & 1] = S4[kk].x;                   // U^2_k(R), the stored state
        // 1. pair terms at r'_k, kept per partner; their sums are electron k's values at R'
        float t1[SPT][5];
        float acc[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
        {
            Axis<float> a1[3];
            a1[0] = make_axis<float>(xn, L0);
            a1[1] = make_axis<float>(yn, L1);
            a1[2] = make_axis<float>(zn, L2);
#pragma unroll
            for (int j = 0; j < SPT; ++j) {
                const int i = tid + j * TPB;
                const bool inb = FULL || i < N;
                const int ii = inb ? i : 0;
                const float4 pi = P4[ii];
                const bool dn = FULL ? (j >= SPT / 2) : (ii >= n_up);        // partner's spin half
                pair_raw(pi.x, pi.y, pi.z, a1, inb && i != kk, dn ? bd : bu, clamp, invd, t1[j]);
#pragma unroll
                for (int c = 0; c < 5; ++c) acc[c] += t1[j][c];
            }
        }
        // 1b. J1: thread tid takes ions tid, tid + TPB at both positions, in physical units
        //     (species differ in delta): dv1 = sum U(r'_k) - U(r_k); at r'_k V, G = -U' d/r,
        //     L = U'' + 2U'/r (electron k's J1 row on acceptance)
        float dv1 = 0.f, a1c[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
        if constexpr (J1) {
            Axis<float> a0[3], a1[3];
            a0[0] = make_axis<float>(xk, L0); a0[1] = make_axis<float>(yk, L1); a0[2] = make_axis<float>(zk, L2);
            a1[0] = make_axis<float>(xn, L0); a1[1] = make_axis<float>(yn, L1); a1[2] = make_axis<float>(zn, L2);
#pragma unroll
            for (int ion = tid; ion < SW_MAX_IONS; ion += TPB) {
                if (ion >= p.n_ions) break;
                const float4 ip = ion_p[ion];
                const uint2 ic = ion_c[ion];
                const float iv = ip.w;
                float u0 = 0.f;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const Axis<float>(&a)[3] = q ? a1 : a0;
                    const float dx = min_image(ip.x, a[0]), dy = min_image(ip.y, a[1]), dz = min_image(ip.z, a[2]);
                    const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                    const float ir = Traits<float>::rsqrt(r2);
                    const FunctorEval<float> e = functor_from_t<float>(r2 * ir * iv, ic.x, ic.y);
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
        //    slots for 5 or 11 values: one shuffle per slot and level instead of one
        //    per value), one partial per value and warp in shared memory.  The first FL
        //    levels add in fp32 -- partials of <= 2^FL lanes x SPT <= 32 terms, the eval
        //    kernel's fp32 partial rule -- the rest in fp64.
        {
            constexpr int NS = J1 ? 16 : 8;
            constexpr int OREM = J1 ? 1 : 2;        // lanes below this distance hold copies of one slot
            constexpr int FL = 4 * SPT <= 32 ? 2 : 1;
            static_assert((1 << FL) * SPT <= 32, "fp32 partials of at most 32 terms");
            float vf[NS];
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                vf[c] = acc[c];
                if (J1) vf[6 + c] = a1c[c];
            }
            if (J1) vf[5] = dv1;
#pragma unroll
            for (int c = NV; c < NS; ++c) vf[c] = 0.f;
            int slot = 0;
#pragma unroll
            for (int l = 0, h = NS / 2, o = 16; l < FL; ++l, h >>= 1, o >>= 1) {
                const bool up = lane & o;           // this lane keeps the upper half of the slots
#pragma unroll
                for (int j = 0; j < h; ++j) {
                    const float send = up ? vf[j] : vf[j + h];
                    const float keep = up ? vf[j + h] : vf[j];
                    vf[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
                slot += up ? h : 0;
            }
            constexpr int NF = NS >> FL;            // slots left for the fp64 levels
            double v[NF];
#pragma unroll
            for (int j = 0; j < NF; ++j) v[j] = (double)vf[j];
#pragma unroll
            for (int h = NF / 2, o = 16 >> FL; h >= 1; h >>= 1, o >>= 1) {
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
        // 3. ratio and Metropolis: every thread sums the partials and takes the same
        //    decision (no second barrier); thread 0 records it
        const double (*red)[NV] = red2[s & 1];
        double vnew = 0.0, dj1 = 0.0;
#pragma unroll
        for (int wi = 0; wi < NW; ++wi) {
            vnew += red[wi][0];
            if (J1) dj1 += red[wi][5];
        }
        const double djs = (vnew - (double)vk2[s & 1]) + dj1;      // dJ2 + dJ1 (Eq. 4-5)
        const double uu = mv_u[b][jm];
        // u < exp(2 dJ): an fp32 exp settles it unless u is within 1e-4 of the threshold (its
        // relative error is < 2e-5 for |dJ| < 100) or the fp32 value over/underflows; then fp64.
        // Either way the decision equals the fp64 test.
        const float e32 = __expf(2.f * (float)djs);
        bool accepted;
        if (isfinite(e32) && e32 > 1e-30f && fabs((float)uu - e32) > 1e-4f * e32 && fabs(djs) < 100.0) {
            accepted = (float)uu < e32;
        } else {
            const double rho = exp(djs);
            accepted = uu < rho * rho;
        }
        accepted = accepted && k_ok;
        if (tid == 0) {
            const int64_t sw = (int64_t)s * p.W + w;
            p.acc[sw] = k_ok ? (accepted ? 1 : 0) : -1;
            if (p.dj) p.dj[sw] = k_ok ? djs : 0.0;
        }
        // 4. accept: pair terms at r_k, partners += T(r'_k) - T(r_k); the owner of slot k
        //    writes state_k = the sums at r'_k and r_k <- r'_k
        if (accepted) {
            Axis<float> a0[3];
            a0[0] = make_axis<float>(xk, L0);
            a0[1] = make_axis<float>(yk, L1);
            a0[2] = make_axis<float>(zk, L2);
#pragma unroll
            for (int j = 0; j < SPT; ++j) {
                const int i = tid + j * TPB;
                const bool inb = FULL || i < N;
                const int ii = inb ? i : 0;
                float t0[5];
                const float4 pi = P4[ii];
                const bool dn = FULL ? (j >= SPT / 2) : (ii >= n_up);
                pair_raw(pi.x, pi.y, pi.z, a0, inb && i != kk, dn ? bd : bu, clamp, invd, t0);
                // the self slot adds T - T = 0 (both terms masked) and is then overwritten by its owner
                if (inb) {
                    QJ2_DCHECK(i < N);
                    float4 si = S4[i];
                    si.x += t1[j][0] - t0[0];
                    si.y = fmaf(t1[j][1] - t0[1], invd, si.y);
                    si.z = fmaf(t1[j][2] - t0[2], invd, si.z);
                    si.w = fmaf(t1[j][3] - t0[3], invd, si.w);
                    S4[i] = si;
                    reinterpret_cast<float *>(P4 + i)[3] = fmaf(t1[j][4] - t0[4], sl, pi.w);
                }
            }
            if (tid == (kk & (TPB - 1))) {     // the thread that owns slot k (no cross-thread writes)
                // state_k = (V, G, L) at r'_k: G = -invd * sum g d, L = 2 invd * sum (h invd + g)
                double f[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int wi = 0; wi < NW; ++wi)
#pragma unroll
                    for (int c = 0; c < 4; ++c) f[c] += red[wi][1 + c];
                S4[kk] = make_float4((float)vnew, (float)(-p.inv_delta * f[0]), (float)(-p.inv_delta * f[1]),
                                     (float)(-p.inv_delta * f[2]));
                P4[kk] = make_float4(propose(xk, mv_d[b][jm][0], L0), propose(yk, mv_d[b][jm][1], L1),
                                     propose(zk, mv_d[b][jm][2], L2), (float)(2.0 * p.inv_delta * f[3]));
                if constexpr (J1) {                  // electron k's J1 row: U^1_k and derivatives at r'_k
                    double f1[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int wi = 0; wi < NW; ++wi)
#pragma unroll
                        for (int c = 0; c < 5; ++c) f1[c] += red[wi][6 + c];
                    float *S1 = p.state_j1 + (int64_t)w * 5 * p.Np;
#pragma unroll
                    for (int c = 0; c < 5; ++c) S1[c * p.Np + kk] = (float)f1[c];
                }
            }
        }
        prev_k = kk;
        prev_acc = accepted;
        // no barrier: every thread only touches its own slots of R and the state, the
        // partials and U^2_k are double-buffered (a warp writes red2[s & 1] again at move
        // s + 2, after every thread has passed the barrier of move s + 1), and r_k of the
        // next move is re-synchronised above when its owner has just written it
    }
    float *Rw = p.R + (int64_t)w * 3 * p.Np;
    float *Sw = p.state + (int64_t)w * 5 * p.Np;
    for (int i = tid; i < N; i += TPB) {         // own slots only: no barrier needed
        const float4 pi = P4[i], si = S4[i];
        Rw[i] = pi.x; Rw[p.Np + i] = pi.y; Rw[2 * p.Np + i] = pi.z;
        Sw[i] = si.x; Sw[p.Np + i] = si.y; Sw[2 * p.Np + i] = si.z; Sw[3 * p.Np + i] = si.w; Sw[4 * p.Np + i] = pi.w;
    }
}

// ---------------------------------------------------------------------------
// qj2_state_init: the state of every electron from scratch (the "new states
// periodically computed from scratch" of PAPER:764-765), one CTA per walker,
// positions in shared memory, one electron per thread at a time, its partners
// walked in a uniform loop (every partner read is a shared-memory broadcast);
// fp32 partials of <= 32 terms flushed to fp64, as in the eval kernel.
// ---------------------------------------------------------------------------
constexpr int SI_TPB = 256;

template <bool J1>
__global__ void __launch_bounds__(SI_TPB) state_init_kernel(const __grid_constant__ SweepParams p) {
    extern __shared__ __align__(16) float si_smem[];
    const int w = blockIdx.x, N = p.N, tid = threadIdx.x;
    QJ2_DCHECK(w < p.W && N <= p.Np && p.n_ions <= SW_MAX_IONS &&
               (uint32_t)(((3 * N + 3) & ~3) * sizeof(float) + (2 * (p.m + 1) + (J1 ? p.n_rows1 : 0)) *
                          sizeof(Coef4<float>) + (J1 ? p.n_ions * (sizeof(float4) + sizeof(uint2)) : 0)) <= dyn_smem_bytes());
    float *rx = si_smem, *ry = rx + N, *rz = ry + N;
    const int N4 = (3 * N + 3) & ~3;
    Coef4<float> *tab = reinterpret_cast<Coef4<float> *>(si_smem + N4);
    Coef4<float> *tab1 = tab + 2 * (p.m + 1);
    float4 *ion_p = reinterpret_cast<float4 *>(tab1 + (J1 ? p.n_rows1 : 0));
    uint2 *ion_c = reinterpret_cast<uint2 *>(ion_p + (J1 ? p.n_ions : 0));
    stage_tables<J1>(p, tab, tab1, ion_p, ion_c, tid, SI_TPB);
    const float *Rg = p.R + (int64_t)w * 3 * p.Np;
    for (int i = tid; i < N; i += SI_TPB) { rx[i] = Rg[i]; ry[i] = Rg[p.Np + i]; rz[i] = Rg[2 * p.Np + i]; }
    __syncthreads();
    const uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab);
    const uint32_t tab_o = tab_s + (uint32_t)((p.m + 1) * (int)sizeof(Coef4<float>));
    const float invd = p.invd;
    float *Sw = p.state + (int64_t)w * 5 * p.Np;
    for (int e = tid; e < ((N + SI_TPB - 1) / SI_TPB) * SI_TPB; e += SI_TPB) {
        const bool ok = e < N;
        const int ee = ok ? e : 0;
        Axis<float> a[3];
        a[0] = make_axis<float>(rx[ee], p.L[0]);
        a[1] = make_axis<float>(ry[ee], p.L[1]);
        a[2] = make_axis<float>(rz[ee], p.L[2]);
        const bool e_up = ee < p.N_up;
        const uint32_t bu = e_up ? tab_s : tab_o, bd = e_up ? tab_o : tab_s;
        double d[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int i0 = 0; i0 < N; i0 += 32) {
            float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            const int i1 = min(i0 + 32, N);
            for (int i = i0; i < i1; ++i) {
                float t[5];
                pair_raw(rx[i], ry[i], rz[i], a, i != ee, i >= p.N_up ? bd : bu, (unsigned)p.m, invd, t);
                acc[0] += t[0]; acc[1] += t[1]; acc[2] += t[2]; acc[3] += t[3]; acc[4] += t[4];
            }
#pragma unroll
            for (int c = 0; c < 5; ++c) d[c] += (double)acc[c];
        }
        if (ok) {
            // partner-minus-electron displacements: G_e = -invd * sum g d, L_e = 2 invd * sum (h invd + g)
            Sw[ee] = (float)d[0];
            Sw[p.Np + ee] = (float)(-p.inv_delta * d[1]);
            Sw[2 * p.Np + ee] = (float)(-p.inv_delta * d[2]);
            Sw[3 * p.Np + ee] = (float)(-p.inv_delta * d[3]);
            Sw[4 * p.Np + ee] = (float)(2.0 * p.inv_delta * d[4]);
        }
        if constexpr (J1) {                     // electron e's J1 row over the ions, physical units
            double f[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            for (int i0 = 0; i0 < p.n_ions; i0 += 32) {
                float acc[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
                const int i1 = min(i0 + 32, p.n_ions);
                for (int ion = i0; ion < i1; ++ion) {
                    const float4 ip = ion_p[ion];
                    const uint2 ic = ion_c[ion];
                    const float dx = min_image(ip.x, a[0]), dy = min_image(ip.y, a[1]), dz = min_image(ip.z, a[2]);
                    const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                    const float ir = Traits<float>::rsqrt(r2);
                    const FunctorEval<float> fe = functor_from_t<float>(r2 * ir * ip.w, ic.x, ic.y);
                    const float g = fe.du * ir * ip.w;                  // U'/r
                    acc[0] += fe.u;
                    acc[1] += -g * dx;
                    acc[2] += -g * dy;
                    acc[3] += -g * dz;
                    acc[4] += 2.f * (fe.h * ip.w * ip.w + g);        // U'' + 2U'/r
                }
#pragma unroll
                for (int c = 0; c < 5; ++c) f[c] += (double)acc[c];
            }
            if (ok) {
                float *S1 = p.state_j1 + (int64_t)w * 5 * p.Np;
#pragma unroll
                for (int c = 0; c < 5; ++c) S1[c * p.Np + ee] = (float)f[c];
            }
        }
    }
}

static size_t table_smem(const SweepParams &p, bool j1) {
    return (size_t)(2 * (p.m + 1) + (j1 ? p.n_rows1 : 0)) * sizeof(Coef4<float>) +
           (j1 ? (size_t)p.n_ions * (sizeof(float4) + sizeof(uint2)) : 0);
}

cudaError_t launch_sweep(const SweepParams &p, cudaStream_t s) {
    const bool j1 = p.n_ions > 0;
    const size_t smem = (size_t)8 * p.N * sizeof(float) + table_smem(p, j1);   // R (3) + state (5) per electron
#define QJ2_SWEEP_LAUNCH(T_, S_, F_)                                                         \
    (j1 ? (j2_sweep_kernel<T_, S_, true, F_><<<(unsigned)p.W, T_, smem, s>>>(p), 0)           \
        : (j2_sweep_kernel<T_, S_, false, F_><<<(unsigned)p.W, T_, smem, s>>>(p), 0))
    // the same-spin halves as compile-time partner ranges when N fills the threads exactly
    // (NiO-64's 768 = 64 x 12, 1024 = 128 x 8, ...); a tier's unused partner slots are masked
    // (tiers every 128 electrons: at most 1/6 of the slots idle above N = 256; the tiers against
    // the round-1 ones (128 x 4-6, 256 x 1-4): profiles/r02/ab_results.txt)
    auto is_full = [&](int tpb, int spt) { return p.N == tpb * spt && 2 * p.N_up == p.N && spt % 2 == 0; };
#define QJ2_SWEEP_TIER(T_, S_) \
    if (is_full(T_, S_)) QJ2_SWEEP_LAUNCH(T_, S_, true); else QJ2_SWEEP_LAUNCH(T_, S_, false)
    if (p.N <= 256) { QJ2_SWEEP_TIER(64, 4); }
    else if (p.N <= 384) { QJ2_SWEEP_TIER(64, 6); }
    else if (p.N <= 512) { QJ2_SWEEP_TIER(64, 8); }
    else if (p.N <= 640) { QJ2_SWEEP_TIER(64, 10); }
    else if (p.N <= 768) { QJ2_SWEEP_TIER(64, 12); }
    else { QJ2_SWEEP_TIER(128, 8); }
#undef QJ2_SWEEP_TIER
#undef QJ2_SWEEP_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_state_init(const SweepParams &p, cudaStream_t s) {
    const bool j1 = p.n_ions > 0;
    const size_t smem = (size_t)((3 * p.N + 3) & ~3) * sizeof(float) + table_smem(p, j1);
    if (j1) state_init_kernel<true><<<(unsigned)p.W, SI_TPB, smem, s>>>(p);
    else state_init_kernel<false><<<(unsigned)p.W, SI_TPB, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace qj2
