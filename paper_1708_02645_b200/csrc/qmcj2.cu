// qmcj2.cu -- sm_100a kernels and C-ABI entry points of the J2 / distance-row
// hot path of arXiv 1708.02645 (declared and documented in include/qmcj2.h).
//
// Kernel map:
//   j2_eval_kernel<T, PB>   the hot path: one CTA per (walker, trial group,
//                           source tile); SoA lanes streamed with coalesced
//                           128-bit loads, per-term math in T, fp32 partials of
//                           32 terms flushed to fp64, warp-shuffle + smem CTA
//                           reduction, deterministic cross-CTA reduction by the
//                           last CTA of each (walker, group).
//   ratio_kernel            dJ2 and exp(dJ2) after a sharded reduction.
//   vgl_kernel / minimg_kernel   batched building blocks.
//   check_kernel            optional precondition scan.
#include "qmcj2.h"
#include "j2_device.cuh"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <cstdlib>
#include <algorithm>

namespace qj2 {

constexpr int TPB = 256;          // threads per CTA
constexpr int ITERS = 8;          // vector iterations per sub-tile: 32 fp32 terms per thread per trial
constexpr int SUB = 4;            // sub-tiles per CTA tile
constexpr int NACC = 6;           // V, Gx, Gy, Gz, sum h, sum du/r  (per trial)
constexpr int MAXPB = 4;

// ---------------------------------------------------------------------------
// Kernel parameters (by value, __grid_constant__).
// ---------------------------------------------------------------------------
struct EvalParams {
    int64_t W, N_total, N_up, i_offset, N_local, Np;
    int64_t tiles_per_walker;     // ceil(N_local / CH)
    int64_t n_groups;             // ceil(P / PB)
    int32_t P, m;
    const void *R;
    const int32_t *k;
    const void *r_trial;
    double *out;
    void *row_out;
    const double *V_cur;
    double *ratio_out;
    double *partials;             // [W][n_groups][tiles][PB][NACC]
    unsigned int *counters;       // [W][n_groups]
    double L[3];
    double inv_delta;
    float inv_delta_f;
    double pcoef[2][QJ2_MAX_M + 1][4];   // power basis per interval; row m = 0
};

// ---------------------------------------------------------------------------
// Helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ void load_table(const EvalParams &p, Coef4<T> *tab) {
    const int n = 2 * (p.m + 1);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int s = e / (p.m + 1), j = e % (p.m + 1);
        Coef4<T> c;
        c.a0 = T(p.pcoef[s][j][0]);
        c.a1 = T(p.pcoef[s][j][1]);
        c.a2 = T(p.pcoef[s][j][2]);
        c.a3 = T(p.pcoef[s][j][3]);
        tab[e] = c;
    }
}

// Per-trial constants: the three axes' minimum-image constants.
template <typename T> struct Trial { Axis<T> ax, ay, az; };

// Functor + accumulation for one source at squared distance r2 (and
// displacement d).  acc: V, Gx, Gy, Gz (sum du/r * d), H (sum h), S (sum du/r).
// Final scaling to U', U'' happens once, in fp64, per tile.
template <typename T>
__device__ __forceinline__ T accumulate(T dx, T dy, T dz, T r2, T inv_delta, uint32_t tab_base,
                                        typename Traits<T>::U clamp_bits, T *acc) {
    using Tr = Traits<T>;
    const T ir = Tr::rsqrt(r2);
    const T r = r2 * ir;
    const FunctorEval<T> e = functor_from_t<T>(r * inv_delta, tab_base, clamp_bits);
    const T g = e.du * ir;
    acc[0] += e.u;
    acc[1] = fma(g, dx, acc[1]);
    acc[2] = fma(g, dy, acc[2]);
    acc[3] = fma(g, dz, acc[3]);
    acc[4] += e.h;
    acc[5] += g;
    return r;
}

// Minimum image for one axis, optionally specialised on the trial
// coordinate's case (SPEC = 1: case A, c < L/2; 0: case B; -1: unified,
// see make_axis).  Specialised forms take 3 instructions instead of 4, but the
// 8 per-walker bodies measured slower on B200 (instruction-cache pressure,
// DESIGN.md section 9); the kernel uses the unified form.
template <typename T, int SPEC>
__device__ __forceinline__ T min_image_k(T x, const Axis<T> &a) {
    if constexpr (SPEC < 0) {
        return min_image(x, a);
    } else if constexpr (SPEC == 1) {           // case A: wrap shifts the source (x - L exact)
        const T xs = x > a.thr ? x - a.a1 : x;
        return xs - a.b0;
    } else {                                    // case B: wrap shifts the trial (c - L exact)
        return x - (x > a.thr ? a.b1 : a.b0);
    }
}

// Masks of a sub-tile that is not "clean" (ragged length, holds the self
// source k, or straddles the spin boundary N_up).  All offsets are relative to
// the sub-tile start.
struct SubMask {
    int len;          // valid sources in the sub-tile
    int k_rel;        // self source, or -1
    int up_rel;       // first spin-down source (clamped to [0, SCH])
    bool k_up;        // spin of k
};

// One sub-tile.  Every thread walks ITERS vectors at a constant stride of TPB
// vectors, so every load address is base + immediate; PF vector groups are in
// flight ahead of the one being consumed (software pipelining).
// GEN = false: full sub-tile, no self source, one spin channel (`base`).
// GEN = true: loads predicated on the sub-tile length; per source, dead
// sources (self, padding) get r^2 = BIG, which lands on the all-zero interval
// (every accumulated quantity exactly 0), and the channel is chosen per source.
template <typename T, int PB, bool ROW, int PF, bool GEN, int NT = TPB, int SX = -1, int SY = -1, int SZ = -1>
__device__ __forceinline__ void tile_run(int tid,const typename Traits<T>::V *__restrict__ px,
                                         const typename Traits<T>::V *__restrict__ py,
                                         const typename Traits<T>::V *__restrict__ pz,
                                         const Trial<T> (&tr)[PB], int np, T inv_delta, uint32_t base,
                                         uint32_t base_opp, const SubMask &mk,
                                         typename Traits<T>::U clamp_bits, T (&acc)[PB][NACC],
                                         typename Traits<T>::V *const (&rowp)[PB], int64_t row_stride) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    // GEN: vector index clamped into the sub-tile (vectors past the end reload
    // the last valid vector; their sources are all dead), so loads need no
    // predicate and the pipeline has the same shape as the fast path.
    const int vmax = GEN ? (mk.len - 1) / VW : 0;
    auto voff = [&](int j) -> int {
        return GEN ? min(j * NT + tid, vmax) - tid : j * NT;   // relative to this thread's vector
    };
    V bx[ITERS], by[ITERS], bz[ITERS];      // fully unrolled: only PF+1 groups are live
#pragma unroll
    for (int j = 0; j < PF && j < ITERS; ++j) {
        bx[j] = Tr::ld_stream(px + voff(j));
        by[j] = Tr::ld_stream(py + voff(j));
        bz[j] = Tr::ld_stream(pz + voff(j));
    }
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
        if (it + PF < ITERS) {
            bx[it + PF] = Tr::ld_stream(px + voff(it + PF));
            by[it + PF] = Tr::ld_stream(py + voff(it + PF));
            bz[it + PF] = Tr::ld_stream(pz + voff(it + PF));
        }
        const int rel = (it * NT + tid) * VW;
        if (!GEN || rel < mk.len) {
        V ro[PB][4];
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            bool dead = false;
            uint32_t b = base;
            if (GEN) {
                const int li = rel + e;
                dead = (li >= mk.len) || (li == mk.k_rel);
                b = ((li < mk.up_rel) == mk.k_up) ? base : base_opp;
            }
            const T x = Tr::comp(bx[it], e), y = Tr::comp(by[it], e), z = Tr::comp(bz[it], e);
#pragma unroll
            for (int q = 0; q < PB; ++q) {
                if (PB == 1 || q < np) {
                    const T dx = min_image_k<T, SX>(x, tr[q].ax);
                    const T dy = min_image_k<T, SY>(y, tr[q].ay);
                    const T dz = min_image_k<T, SZ>(z, tr[q].az);
                    T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                    if (GEN) r2 = dead ? T(1e30) : r2;
                    const T r = accumulate<T>(dx, dy, dz, r2, inv_delta, b, clamp_bits, acc[q]);
                    if (ROW) { Tr::set(ro[q][0], e, r); Tr::set(ro[q][1], e, dx); Tr::set(ro[q][2], e, dy); Tr::set(ro[q][3], e, dz); }
                }
            }
        }
        if (ROW) {
#pragma unroll
            for (int q = 0; q < PB; ++q)
                if (PB == 1 || q < np)
#pragma unroll
                    for (int c = 0; c < 4; ++c) __stcs(rowp[q] + c * row_stride + it * NT, ro[q][c]);
        }
        }
    }
}

// PF: prefetch distance (vector groups in flight), MINB: resident CTAs per SM
// (register budget).
template <typename T, int PB, bool ROW, int PF = 1, int MINB = ((sizeof(T) == 4 && PB == 1) ? 4 : 2)>
__global__ void __launch_bounds__(TPB, MINB)
j2_eval_kernel(const __grid_constant__ EvalParams p) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    constexpr int SCH = TPB * VW * ITERS;         // sub-tile: 32 terms per thread
    constexpr int CH = SCH * SUB;                 // tile handled by one CTA
    __shared__ Coef4<T> tab[2 * (QJ2_MAX_M + 1)];
    __shared__ double red[TPB / 32][PB * NACC];
    __shared__ int last_flag;

    // tile decode: chunk fastest so consecutive CTAs stream consecutive memory
    // (32-bit arithmetic: the host guarantees W * n_groups * tiles < 2^31)
    const uint32_t b = blockIdx.x;
    const uint32_t tpw32 = (uint32_t)p.tiles_per_walker;
    const uint32_t per_w = tpw32 * (uint32_t)p.n_groups;
    const uint32_t w32 = b / per_w;
    const uint32_t rem = b - w32 * per_w;
    const uint32_t g32 = rem / tpw32;
    const int64_t tpw = p.tiles_per_walker;
    const int64_t w = w32, g = g32, c = rem - g32 * tpw32;
    const int32_t p0 = (int32_t)g * PB;
    const int np = min(PB, p.P - p0);

    load_table<T>(p, tab);

    const int64_t kw = p.k[w];
    const bool k_up = kw < p.N_up;
    const T L0 = T(p.L[0]), L1 = T(p.L[1]), L2 = T(p.L[2]);
    Trial<T> tr[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) {
        const int qq = q < np ? q : 0;
        const T *rt = static_cast<const T *>(p.r_trial) + ((w * p.P + p0 + qq) * 3);
        tr[q].ax = make_axis<T>(rt[0], L0);
        tr[q].ay = make_axis<T>(rt[1], L1);
        tr[q].az = make_axis<T>(rt[2], L2);
    }
    const T inv_delta = sizeof(T) == 4 ? T(p.inv_delta_f) : T(p.inv_delta);
    const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tab);
    const uint32_t magic_off = (uint32_t)(Tr::MAGIC_BITS * (typename Tr::U)sizeof(Coef4<T>));
    const uint32_t base_same = tab_addr - magic_off;
    const uint32_t base_opp = tab_addr + (uint32_t)((p.m + 1) * sizeof(Coef4<T>)) - magic_off;
    const typename Tr::U clamp_bits = Tr::MAGIC_BITS + (typename Tr::U)p.m;

    const int64_t start = c * CH;
    const int64_t end = min(start + (int64_t)CH, p.N_local);
    const int64_t k_local = kw - p.i_offset;
    const int64_t nup_local = p.N_up - p.i_offset;   // first local index of the spin-down half

    const T *Rw = static_cast<const T *>(p.R) + w * 3 * p.Np;
    const int64_t voff = (start >> (VW == 4 ? 2 : 1)) + threadIdx.x;   // this thread's first vector
    const V *px = reinterpret_cast<const V *>(Rw) + voff;
    const V *py = reinterpret_cast<const V *>(Rw + p.Np) + voff;
    const V *pz = reinterpret_cast<const V *>(Rw + 2 * p.Np) + voff;
    V *rowp[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q)
        rowp[q] = ROW ? reinterpret_cast<V *>(static_cast<T *>(p.row_out) + ((w * p.P + p0 + (q < np ? q : 0)) * 4) * p.Np) + voff
                      : nullptr;
    const int64_t row_stride = p.Np / VW;
    __syncthreads();

    // The tile is SUB sub-tiles of SCH sources.  Per sub-tile, each thread
    // accumulates <= ITERS*VW = 32 terms in T, then flushes to fp64
    // ("quantities per walker ... in double precision").
    double dacc[PB][NACC];
#pragma unroll
    for (int q = 0; q < PB; ++q)
#pragma unroll
        for (int a = 0; a < NACC; ++a) dacc[q][a] = 0.0;

#pragma unroll 1
    for (int sidx = 0; sidx < SUB; ++sidx) {
        const int64_t sstart = start + (int64_t)sidx * SCH;
        if (sstart >= end) break;
        const int64_t send = min(sstart + (int64_t)SCH, end);
        const int64_t vs = (int64_t)sidx * (SCH / VW);
        T acc[PB][NACC];
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) acc[q][a] = T(0);
        const bool k_in = k_local >= sstart && k_local < send;
        const bool masked = (send - sstart != SCH) || k_in || (nup_local > sstart && nup_local < send);
        V *rp[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) rp[q] = ROW ? rowp[q] + vs : nullptr;
        if (masked) {
            SubMask mk;
            mk.len = (int)(send - sstart);
            mk.k_rel = k_in ? (int)(k_local - sstart) : -1;
            mk.up_rel = (int)max((int64_t)0, min(nup_local - sstart, (int64_t)SCH));
            mk.k_up = true;   // base_same is "channel of sources below up_rel" iff k is up
            const uint32_t b_lo = k_up ? base_same : base_opp;   // channel of sources i < N_up
            const uint32_t b_hi = k_up ? base_opp : base_same;   // channel of sources i >= N_up
            tile_run<T, PB, ROW, PF, true>(threadIdx.x, px + vs, py + vs, pz + vs, tr, np, inv_delta, b_lo, b_hi, mk,
                                           clamp_bits, acc, rp, row_stride);
        } else {
            const bool tile_up = sstart < nup_local;
            const uint32_t base = (tile_up == k_up) ? base_same : base_opp;
            SubMask mk{SCH, -1, 0, true};
            tile_run<T, PB, ROW, PF, false>(threadIdx.x, px + vs, py + vs, pz + vs, tr, np, inv_delta, base, base, mk,
                                            clamp_bits, acc, rp, row_stride);
        }
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) dacc[q][a] += (double)acc[q][a];
    }

    // ---- CTA reduction in fp64 (fixed order: deterministic) ----
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < PB; ++q)
#pragma unroll
        for (int a = 0; a < NACC; ++a) {
            const double v = warp_sum(dacc[q][a]);
            if (lane == 0) red[warp][q * NACC + a] = v;
        }
    __syncthreads();

    double tot = 0.0;   // thread t < PB*NACC holds value t of this tile
    if (threadIdx.x < PB * NACC) {
#pragma unroll
        for (int wi = 0; wi < TPB / 32; ++wi) tot += red[wi][threadIdx.x];
    }

    const int64_t wg = w * p.n_groups + g;
    if (tpw > 1) {
        // publish this tile's partials; the last CTA of (w, g) reduces them
        double *part = p.partials + (wg * tpw + c) * (PB * NACC);
        if (threadIdx.x < PB * NACC) part[threadIdx.x] = tot;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned prev = atomicAdd(p.counters + wg, 1u);
            last_flag = (prev == (unsigned)(tpw - 1));
        }
        __syncthreads();
        if (!last_flag) return;
        __threadfence();
        // warp 0: value v summed over tiles, lane-strided then shuffle tree
        if (warp == 0) {
            const double *base = p.partials + wg * tpw * (PB * NACC);
            for (int v = 0; v < PB * NACC; ++v) {
                double s = 0.0;
                for (int64_t t = lane; t < tpw; t += 32) s += __ldcg(base + t * (PB * NACC) + v);
                s = warp_sum(s);
                if (lane == v) tot = s;      // lane v keeps value v (PB*NACC <= 24 < 32)
            }
        }
    }

    // ---- finalize: lane t < PB*NACC of warp 0 holds value (q = t / NACC, a = t % NACC) ----
    if (warp == 0) {
        const double id = p.inv_delta;
        const double V0 = __shfl_sync(0xffffffffu, tot, 0);   // V of this group's first trial
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            double s[NACC];
#pragma unroll
            for (int a = 0; a < NACC; ++a) s[a] = __shfl_sync(0xffffffffu, tot, q * NACC + a);
            if (lane == 0 && q < np) {
                const int64_t o = w * p.P + p0 + q;
                const double V = s[0];
                p.out[o * 5 + 0] = V;
                p.out[o * 5 + 1] = -id * s[1];
                p.out[o * 5 + 2] = -id * s[2];
                p.out[o * 5 + 3] = -id * s[3];
                p.out[o * 5 + 4] = 2.0 * id * id * s[4] + 2.0 * id * s[5];
                if (p.ratio_out) {   // e^{dJ2} factor of Eq. 4 (host guarantees a valid reference)
                    const double dj = V - (p.V_cur ? p.V_cur[w] : V0);
                    p.ratio_out[o * 2 + 0] = dj;
                    p.ratio_out[o * 2 + 1] = exp(dj);
                }
            }
        }
    }
}

// Small-N mapping (one tile per walker and many walkers, e.g. C1, C2, C4):
// one warp per (walker, trial group) walks all of the walker's sources in
// per-warp sub-tiles of 32*VW*ITERS sources (<= 32 fp32 terms per lane, then
// an fp64 flush), so there is no shared-memory reduction, no cross-CTA
// partials and no counters; the warp's fp64 shuffle tree is the whole
// (deterministic) reduction.
template <typename T, int PB, bool ROW, int PF, int MINB = (sizeof(T) == 4 && PB == 1 && !ROW) ? 3 : 2>
__global__ void __launch_bounds__(TPB, MINB)
j2_eval_warp_kernel(const __grid_constant__ EvalParams p, int64_t n_units) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    constexpr int SCH = 32 * VW * ITERS;
    __shared__ Coef4<T> tab[2 * (QJ2_MAX_M + 1)];
    load_table<T>(p, tab);
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t unit = (int64_t)blockIdx.x * (TPB / 32) + warp;
    if (unit >= n_units) return;
    const int64_t w = unit / p.n_groups, g = unit - w * p.n_groups;
    const int32_t p0 = (int32_t)g * PB;
    const int np = min(PB, p.P - p0);
    const int64_t kw = p.k[w];
    const bool k_up = kw < p.N_up;
    const T L0 = T(p.L[0]), L1 = T(p.L[1]), L2 = T(p.L[2]);
    Trial<T> tr[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) {
        const int qq = q < np ? q : 0;
        const T *rt = static_cast<const T *>(p.r_trial) + ((w * p.P + p0 + qq) * 3);
        tr[q].ax = make_axis<T>(rt[0], L0);
        tr[q].ay = make_axis<T>(rt[1], L1);
        tr[q].az = make_axis<T>(rt[2], L2);
    }
    const T inv_delta = sizeof(T) == 4 ? T(p.inv_delta_f) : T(p.inv_delta);
    const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tab);
    const uint32_t magic_off = (uint32_t)(Tr::MAGIC_BITS * (typename Tr::U)sizeof(Coef4<T>));
    const uint32_t base_same = tab_addr - magic_off;
    const uint32_t base_opp = tab_addr + (uint32_t)((p.m + 1) * sizeof(Coef4<T>)) - magic_off;
    const typename Tr::U clamp_bits = Tr::MAGIC_BITS + (typename Tr::U)p.m;
    const int64_t k_local = kw - p.i_offset;
    const int64_t nup_local = p.N_up - p.i_offset;
    const T *Rw = static_cast<const T *>(p.R) + w * 3 * p.Np;
    const int64_t row_stride = p.Np / VW;

    double dacc[PB][NACC];
#pragma unroll
    for (int q = 0; q < PB; ++q)
#pragma unroll
        for (int a = 0; a < NACC; ++a) dacc[q][a] = 0.0;

    for (int64_t sstart = 0; sstart < p.N_local; sstart += SCH) {
        const int64_t send = min(sstart + (int64_t)SCH, p.N_local);
        const int64_t voff = (sstart / VW) + lane;
        const V *px = reinterpret_cast<const V *>(Rw) + voff;
        const V *py = reinterpret_cast<const V *>(Rw + p.Np) + voff;
        const V *pz = reinterpret_cast<const V *>(Rw + 2 * p.Np) + voff;
        V *rp[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q)
            rp[q] = ROW ? reinterpret_cast<V *>(static_cast<T *>(p.row_out) + ((w * p.P + p0 + (q < np ? q : 0)) * 4) * p.Np) + voff
                        : nullptr;
        T acc[PB][NACC];
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) acc[q][a] = T(0);
        const bool k_in = k_local >= sstart && k_local < send;
        const bool masked = (send - sstart != SCH) || k_in || (nup_local > sstart && nup_local < send);
        if (masked) {
            SubMask mk;
            mk.len = (int)(send - sstart);
            mk.k_rel = k_in ? (int)(k_local - sstart) : -1;
            mk.up_rel = (int)max((int64_t)0, min(nup_local - sstart, (int64_t)SCH));
            mk.k_up = true;
            const uint32_t b_lo = k_up ? base_same : base_opp;
            const uint32_t b_hi = k_up ? base_opp : base_same;
            tile_run<T, PB, ROW, PF, true, 32>(lane, px, py, pz, tr, np, inv_delta, b_lo, b_hi, mk, clamp_bits,
                                               acc, rp, row_stride);
        } else {
            const uint32_t base = ((sstart < nup_local) == k_up) ? base_same : base_opp;
            SubMask mk{SCH, -1, 0, true};
            tile_run<T, PB, ROW, PF, false, 32>(lane, px, py, pz, tr, np, inv_delta, base, base, mk, clamp_bits,
                                                acc, rp, row_stride);
        }
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) dacc[q][a] += (double)acc[q][a];
    }

    const double id = p.inv_delta;
    double V0 = 0.0;
#pragma unroll
    for (int q = 0; q < PB; ++q) {
        double s[NACC];
#pragma unroll
        for (int a = 0; a < NACC; ++a) s[a] = warp_sum(dacc[q][a]);
        if (q == 0) V0 = s[0];
        if (lane == 0 && q < np) {
            const int64_t o = w * p.P + p0 + q;
            p.out[o * 5 + 0] = s[0];
            p.out[o * 5 + 1] = -id * s[1];
            p.out[o * 5 + 2] = -id * s[2];
            p.out[o * 5 + 3] = -id * s[3];
            p.out[o * 5 + 4] = 2.0 * id * id * s[4] + 2.0 * id * s[5];
            if (p.ratio_out) {
                const double dj = s[0] - (p.V_cur ? p.V_cur[w] : V0);
                p.ratio_out[o * 2 + 0] = dj;
                p.ratio_out[o * 2 + 1] = exp(dj);
            }
        }
    }
}

}  // namespace qj2

#include "j2_tma.cuh"

// ===========================================================================
// Small kernels
// ===========================================================================
namespace qj2 {

__global__ void ratio_kernel(int64_t W, int32_t P, const double *__restrict__ out,
                             const double *__restrict__ V_cur, double *__restrict__ ratio_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= W * P) return;
    const int64_t w = i / P;
    const double ref = V_cur ? V_cur[w] : out[(w * P) * 5];
    const double dj = out[i * 5] - ref;
    ratio_out[i * 2 + 0] = dj;
    ratio_out[i * 2 + 1] = exp(dj);
}

struct VglParams {
    int64_t n;
    int32_t m;
    double inv_delta;
    double pcoef[QJ2_MAX_M + 1][4];
};

template <typename T>
__global__ void vgl_kernel(const __grid_constant__ VglParams p, const T *__restrict__ r, double *__restrict__ out) {
    using Tr = Traits<T>;
    __shared__ Coef4<T> tab[QJ2_MAX_M + 1];
    for (int e = threadIdx.x; e <= p.m; e += blockDim.x) {
        Coef4<T> c;
        c.a0 = T(p.pcoef[e][0]); c.a1 = T(p.pcoef[e][1]); c.a2 = T(p.pcoef[e][2]); c.a3 = T(p.pcoef[e][3]);
        tab[e] = c;
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) -
                          (uint32_t)(Tr::MAGIC_BITS * (typename Tr::U)sizeof(Coef4<T>));
    const T id = T(p.inv_delta);
    const FunctorEval<T> e = functor_from_t<T>(r[i] * id, base, Tr::MAGIC_BITS + (typename Tr::U)p.m);
    out[i * 3 + 0] = (double)e.u;
    out[i * 3 + 1] = (double)e.du * p.inv_delta;
    out[i * 3 + 2] = 2.0 * (double)e.h * p.inv_delta * p.inv_delta;
}

template <typename T>
__global__ void minimg_kernel(int64_t n, T L0, T L1, T L2, const T *__restrict__ a,
                              const T *__restrict__ b, T *__restrict__ out) {
    using Tr = Traits<T>;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const T dx = min_image(b[i * 3 + 0], make_axis<T>(a[i * 3 + 0], L0));
    const T dy = min_image(b[i * 3 + 1], make_axis<T>(a[i * 3 + 1], L1));
    const T dz = min_image(b[i * 3 + 2], make_axis<T>(a[i * 3 + 2], L2));
    const T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    out[i * 4 + 0] = r2 == T(0) ? T(0) : r2 * Tr::rsqrt(r2);
    out[i * 4 + 1] = dx;
    out[i * 4 + 2] = dy;
    out[i * 4 + 3] = dz;
}

template <typename T>
__global__ void check_kernel(int64_t W, int64_t N_total, int64_t N_local, int64_t Np, T L0, T L1, T L2,
                             const T *__restrict__ R, const int32_t *__restrict__ k, int32_t P,
                             const T *__restrict__ rt, int32_t *flag) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int f = 0;
    const T Ls[3] = {L0, L1, L2};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < W * 3 * N_local; i += stride) {
        const int64_t w = i / (3 * N_local), rem = i - w * 3 * N_local, d = rem / N_local, j = rem - d * N_local;
        const T x = R[(w * 3 + d) * Np + j];
        if (!(x >= T(0) && x < Ls[d])) f |= 1;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < W; i += stride)
        if (k[i] < 0 || k[i] >= N_total) f |= 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < W * P * 3; i += stride) {
        const T x = rt[i];
        if (!(x >= T(0) && x < Ls[i % 3])) f |= 4;
    }
    if (f) atomicOr(flag, f);
}

}  // namespace qj2

// ===========================================================================
// Host side: validation, functor preparation, launches (C ABI)
// ===========================================================================
using namespace qj2;

namespace {

thread_local char g_err[512] = "";

qj2_status fail(qj2_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

qj2_status cuda_fail(cudaError_t e, const char *what) {
    return fail(QJ2_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

qj2_status check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int major = 0, minor = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(QJ2_ENOTSUP, "device %d is sm_%d%d; this library is built for sm_100a (B200)", dev, major, minor);
    return QJ2_OK;
}

qj2_status validate_functor(const qj2_functor *fn) {
    if (!fn) return fail(QJ2_EINVAL, "fn is NULL");
    if (fn->reserved != 0) return fail(QJ2_EINVAL, "fn->reserved must be 0");
    for (int d = 0; d < 3; ++d)
        if (!(fn->L[d] > 0) || !std::isfinite(fn->L[d])) return fail(QJ2_EINVAL, "L[%d] must be finite and > 0", d);
    const double Lmin = std::fmin(fn->L[0], std::fmin(fn->L[1], fn->L[2]));
    if (!(fn->r_cut > 0) || !(fn->r_cut <= 0.5 * Lmin))
        return fail(QJ2_EINVAL, "r_cut must satisfy 0 < r_cut <= min(L)/2 (got %g, min L %g)", fn->r_cut, Lmin);
    if (fn->m < 4 || fn->m > QJ2_MAX_M) return fail(QJ2_EINVAL, "m must be in [4, %d] (got %d)", QJ2_MAX_M, fn->m);
    for (int s = 0; s < 2; ++s) {
        for (int j = 0; j < fn->m + 3; ++j)
            if (!std::isfinite(fn->coef[s][j])) return fail(QJ2_EINVAL, "coef[%d][%d] not finite", s, j);
        for (int j = fn->m; j < fn->m + 3; ++j)
            if (fn->coef[s][j] != 0.0) return fail(QJ2_EINVAL, "coef[%d][%d] must be 0 (C2 cutoff)", s, j);
    }
    return QJ2_OK;
}

// B-spline coefficients -> per-interval power basis in f.
void power_basis(const double *c, int m, double (*pc)[4]) {
    for (int j = 0; j < m; ++j) {
        const double c0 = c[j], c1 = c[j + 1], c2 = c[j + 2], c3 = c[j + 3];
        pc[j][0] = (c0 + 4.0 * c1 + c2) / 6.0;
        pc[j][1] = (c2 - c0) / 2.0;
        pc[j][2] = (c0 - 2.0 * c1 + c2) / 2.0;
        pc[j][3] = (-c0 + 3.0 * c1 - 3.0 * c2 + c3) / 6.0;
    }
    pc[m][0] = pc[m][1] = pc[m][2] = pc[m][3] = 0.0;
}

inline int vw_of(qj2_dtype d) { return d == QJ2_FP32 ? 4 : 2; }
inline int64_t ch_of(qj2_dtype d) { return (int64_t)TPB * vw_of(d) * ITERS * SUB; }
inline int pb_of(int32_t P) { return P == 1 ? 1 : P == 2 ? 2 : MAXPB; }
inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

void ws_layout(int64_t W, int32_t P, int64_t N_local, qj2_dtype dtype,
               size_t *part_bytes, size_t *cnt_bytes) {
    const int64_t tpw = (N_local + ch_of(dtype) - 1) / ch_of(dtype);
    const int pb = pb_of(P);
    const int64_t ng = (P + pb - 1) / pb;
    *part_bytes = tpw > 1 ? align256((size_t)W * ng * tpw * pb * NACC * sizeof(double)) : 0;
    *cnt_bytes = tpw > 1 ? align256((size_t)W * ng * sizeof(unsigned)) : 0;
}

// Kernel choice (A/B measurements only): QJ2_KERNEL=ldg1 (prefetch distance
// 1, 4 CTAs/SM) or tma323 (TMA-pipelined persistent kernel, 3 CTAs/SM, 2
// vectors per lane per stage, 3 stages); default: LDG kernel, prefetch 2.
struct TmaCfg { int minb, vpt, nst; };
constexpr TmaCfg kTmaCfgs[] = {{3, 2, 3}};
int kernel_choice() {   // -1 = LDG kernel, else index into kTmaCfgs
    const char *e = getenv("QJ2_KERNEL");
    if (!e) return -1;
    if (strcmp(e, "ldg") == 0) return -1;
    if (strncmp(e, "tma", 3) == 0 && strlen(e) == 6) {
        for (int i = 0; i < (int)(sizeof(kTmaCfgs) / sizeof(kTmaCfgs[0])); ++i)
            if (e[3] - '0' == kTmaCfgs[i].minb && e[4] - '0' == kTmaCfgs[i].vpt && e[5] - '0' == kTmaCfgs[i].nst)
                return i;
    }
    return -1;
}

template <typename T, int PB, int MINB, int VPT, int NST>
cudaError_t launch_tma(const EvalParams &p, int64_t nblocks, cudaStream_t s) {
    auto kern = j2_eval_tma_kernel<T, PB, MINB, VPT, NST>;
    const size_t smem = tma_smem_bytes<T>(PB, VPT, NST);
    static int configured = 0;          // benign race: idempotent attribute set
    static int blocks_per_sm = 0, sms = 0;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, TMA_THREADS, smem);
        if (e != cudaSuccess) return e;
        configured = 1;
    }
    const int64_t grid = std::min<int64_t>(nblocks, (int64_t)sms * std::max(blocks_per_sm, 1));
    kern<<<(unsigned)grid, TMA_THREADS, smem, s>>>(p, (uint32_t)nblocks);
    return cudaGetLastError();
}

// Warp-per-walker mapping when a walker's slice is one CTA tile and there
// are enough (walker, group) units to fill the GPU (or the slice is tiny).
bool use_warp_mapping(const EvalParams &p) {
    return p.tiles_per_walker == 1 && (p.W * p.n_groups >= 4096 || p.N_local <= 2048);
}

template <typename T, int PB>
cudaError_t launch_eval(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s) {
    if (use_warp_mapping(p)) {
        const int64_t units = p.W * p.n_groups;
        const unsigned nbw = (unsigned)((units + TPB / 32 - 1) / (TPB / 32));
        if (row) j2_eval_warp_kernel<T, PB, true, 1><<<nbw, TPB, 0, s>>>(p, units);
        else     j2_eval_warp_kernel<T, PB, false, 2><<<nbw, TPB, 0, s>>>(p, units);
        return cudaGetLastError();
    }
    const int kc = row ? -1 : kernel_choice();
    switch (kc) {
        case 0: return launch_tma<T, PB, 3, 2, 3>(p, nblocks, s);
        default: break;
    }
    const char *e = getenv("QJ2_KERNEL");
    const unsigned nb = (unsigned)nblocks;
    if (row) {
        j2_eval_kernel<T, PB, true><<<nb, TPB, 0, s>>>(p);
    } else if constexpr (PB == 1 && sizeof(T) == 4) {
        if (e && strcmp(e, "ldg1") == 0)       // A/B: prefetch distance 1, 4 CTAs/SM
            j2_eval_kernel<T, PB, false, 1, 4><<<nb, TPB, 0, s>>>(p);
        else    // default: two vector groups in flight per thread, 3 CTAs/SM (80 registers);
                // measured best on B200
            j2_eval_kernel<T, PB, false, 2, 3><<<nb, TPB, 0, s>>>(p);
    } else if constexpr (PB == 1) {             // fp64: two groups in flight, 2 CTAs/SM
        j2_eval_kernel<T, PB, false, 2, 2><<<nb, TPB, 0, s>>>(p);
    } else {
        j2_eval_kernel<T, PB, false><<<nb, TPB, 0, s>>>(p);
    }
    return cudaGetLastError();
}

qj2_status eval_impl(const qj2_functor *fn, qj2_dtype dtype,
                     int64_t W, int64_t N_total, int64_t N_up,
                     int64_t i_offset, int64_t N_local, int64_t Np,
                     const void *R, const int32_t *k, int32_t P, const void *r_trial,
                     double *out, void *row_out, const double *V_cur, double *ratio_out,
                     void *workspace, size_t workspace_bytes, cudaStream_t stream, bool check_dev) {
    qj2_status st = validate_functor(fn);
    if (st) return st;
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype %d", (int)dtype);
    if (W < 0) return fail(QJ2_EINVAL, "W < 0");
    if (N_total < 2) return fail(QJ2_EINVAL, "N_total must be >= 2");
    if (N_up < 0 || N_up > N_total) return fail(QJ2_ERANGE, "N_up out of [0, N_total]");
    if (i_offset < 0 || N_local < 1) return fail(QJ2_EINVAL, "need i_offset >= 0 and N_local >= 1");
    if (i_offset + N_local > N_total) return fail(QJ2_ERANGE, "i_offset + N_local > N_total");
    if (Np < N_local || Np % vw_of(dtype) != 0)
        return fail(QJ2_EINVAL, "Np must be >= N_local and a multiple of %d", vw_of(dtype));
    if (P < 1 || P > QJ2_MAX_P) return fail(QJ2_EINVAL, "P must be in [1, %d]", QJ2_MAX_P);
    const int pb = pb_of(P);
    const int64_t ng = (P + pb - 1) / pb;
    if (ratio_out) {
        if (i_offset != 0 || N_local != N_total)
            return fail(QJ2_EINVAL, "ratio_out needs an unsharded call; use qj2_ratio after reducing");
        if (!V_cur && ng != 1) return fail(QJ2_EINVAL, "ratio_out with V_cur == NULL needs P <= %d", MAXPB);
    }
    if (W == 0) return QJ2_OK;
    if (!R || !k || !r_trial || !out) return fail(QJ2_EINVAL, "R, k, r_trial and out must be non-NULL");
    if (((uintptr_t)R & 15) || (row_out && ((uintptr_t)row_out & 15)))
        return fail(QJ2_EINVAL, "R and row_out must be 16-byte aligned");
    size_t part_b, cnt_b;
    ws_layout(W, P, N_local, dtype, &part_b, &cnt_b);
    if (part_b + cnt_b > 0 && (!workspace || workspace_bytes < part_b + cnt_b))
        return fail(QJ2_EINVAL, "workspace too small: need %zu bytes", part_b + cnt_b);
    const int64_t tpw = (N_local + ch_of(dtype) - 1) / ch_of(dtype);
    const int64_t nblocks = W * ng * tpw;
    if (nblocks > 0x7fffffffLL) return fail(QJ2_EINVAL, "problem too large for one launch (%lld CTAs)", (long long)nblocks);
    if (check_dev) { st = check_device(); if (st) return st; }

    EvalParams p;
    memset(&p, 0, sizeof p);
    p.W = W; p.N_total = N_total; p.N_up = N_up; p.i_offset = i_offset; p.N_local = N_local; p.Np = Np;
    p.tiles_per_walker = tpw; p.n_groups = ng; p.P = P; p.m = fn->m;
    p.R = R; p.k = k; p.r_trial = r_trial; p.out = out; p.row_out = row_out;
    p.V_cur = V_cur; p.ratio_out = ratio_out;
    p.partials = part_b ? static_cast<double *>(workspace) : nullptr;
    p.counters = cnt_b ? reinterpret_cast<unsigned *>(static_cast<char *>(workspace) + part_b) : nullptr;
    for (int d = 0; d < 3; ++d) p.L[d] = fn->L[d];
    p.inv_delta = (double)fn->m / fn->r_cut;
    p.inv_delta_f = (float)p.inv_delta;
    power_basis(fn->coef[0], fn->m, p.pcoef[0]);
    power_basis(fn->coef[1], fn->m, p.pcoef[1]);

    const bool row = row_out != nullptr;
    cudaError_t e;
    if (cnt_b) {   // completion counters start at zero every call (no caller-side init needed)
        e = cudaMemsetAsync(p.counters, 0, (size_t)W * ng * sizeof(unsigned), stream);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counters)");
    }
    if (dtype == QJ2_FP32) {
        e = pb == 1 ? launch_eval<float, 1>(p, nblocks, row, stream)
          : pb == 2 ? launch_eval<float, 2>(p, nblocks, row, stream)
                    : launch_eval<float, MAXPB>(p, nblocks, row, stream);
    } else {
        e = pb == 1 ? launch_eval<double, 1>(p, nblocks, row, stream)
          : pb == 2 ? launch_eval<double, 2>(p, nblocks, row, stream)
                    : launch_eval<double, MAXPB>(p, nblocks, row, stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "j2_eval_kernel launch");
    return QJ2_OK;
}

}  // namespace

extern "C" {

int32_t qj2_version(void) { return QJ2_VERSION; }

const char *qj2_status_string(qj2_status s) {
    switch (s) {
        case QJ2_OK: return "ok";
        case QJ2_EINVAL: return "invalid-argument";
        case QJ2_ERANGE: return "out-of-range";
        case QJ2_ENOTSUP: return "not-supported (device is not sm_100)";
        case QJ2_ECUDA: return "cuda-error";
    }
    return "unknown-status";
}

const char *qj2_last_error(void) { return g_err; }

qj2_status qj2_device_check(void) { return check_device(); }

qj2_status qj2_padded_size(int64_t n, int64_t block, int64_t *out) {
    if (!out) return fail(QJ2_EINVAL, "out is NULL");
    if (n < 0) return fail(QJ2_EINVAL, "n < 0");
    if (block < 1) return fail(QJ2_EINVAL, "block < 1");
    const int64_t nn = n < 1 ? 1 : n;
    *out = ((nn + block - 1) / block) * block;
    return QJ2_OK;
}

qj2_status qj2_eval_workspace_size(int64_t W, int32_t P, int64_t N_local, qj2_dtype dtype, size_t *bytes) {
    if (!bytes) return fail(QJ2_EINVAL, "bytes is NULL");
    if (W < 0 || P < 1 || P > QJ2_MAX_P || N_local < 1) return fail(QJ2_EINVAL, "bad W/P/N_local");
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype");
    size_t a, b;
    ws_layout(W, P, N_local, dtype, &a, &b);
    *bytes = a + b;
    return QJ2_OK;
}

qj2_status qj2_eval(const qj2_functor *fn, qj2_dtype dtype,
                    int64_t W, int64_t N_total, int64_t N_up,
                    int64_t i_offset, int64_t N_local, int64_t Np,
                    const void *R, const int32_t *k, int32_t P, const void *r_trial,
                    double *out, void *row_out, const double *V_cur, double *ratio_out,
                    void *workspace, size_t workspace_bytes, void *stream) {
    return eval_impl(fn, dtype, W, N_total, N_up, i_offset, N_local, Np, R, k, P, r_trial, out, row_out,
                     V_cur, ratio_out, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), true);
}

qj2_status qj2_ratio(int64_t W, int32_t P, const double *out, const double *V_cur, double *ratio_out, void *stream) {
    if (W < 0 || P < 1 || P > QJ2_MAX_P) return fail(QJ2_EINVAL, "bad W/P");
    if (W == 0) return QJ2_OK;
    if (!out || !ratio_out) return fail(QJ2_EINVAL, "out and ratio_out must be non-NULL");
    qj2_status st = check_device();
    if (st) return st;
    const int64_t n = W * P;
    ratio_kernel<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(W, P, out, V_cur, ratio_out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "ratio_kernel launch");
}

qj2_status qj2_functor_eval_vgl(const qj2_functor *fn, qj2_dtype dtype, int32_t channel,
                                int64_t n, const void *r, double *out, void *stream) {
    qj2_status st = validate_functor(fn);
    if (st) return st;
    if (channel != 0 && channel != 1) return fail(QJ2_EINVAL, "channel must be 0 or 1");
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype");
    if (n < 0) return fail(QJ2_EINVAL, "n < 0");
    if (n == 0) return QJ2_OK;
    if (!r || !out) return fail(QJ2_EINVAL, "r and out must be non-NULL");
    st = check_device();
    if (st) return st;
    VglParams p;
    memset(&p, 0, sizeof p);
    p.n = n; p.m = fn->m; p.inv_delta = (double)fn->m / fn->r_cut;
    power_basis(fn->coef[channel], fn->m, p.pcoef);
    const unsigned nb = (unsigned)((n + 255) / 256);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == QJ2_FP32) vgl_kernel<float><<<nb, 256, 0, s>>>(p, static_cast<const float *>(r), out);
    else                   vgl_kernel<double><<<nb, 256, 0, s>>>(p, static_cast<const double *>(r), out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "vgl_kernel launch");
}

qj2_status qj2_min_image_disp(const double L[3], qj2_dtype dtype, int64_t n,
                              const void *a, const void *b, void *out, void *stream) {
    if (!L) return fail(QJ2_EINVAL, "L is NULL");
    for (int d = 0; d < 3; ++d) if (!(L[d] > 0)) return fail(QJ2_EINVAL, "L[%d] must be > 0", d);
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype");
    if (n < 0) return fail(QJ2_EINVAL, "n < 0");
    if (n == 0) return QJ2_OK;
    if (!a || !b || !out) return fail(QJ2_EINVAL, "a, b and out must be non-NULL");
    qj2_status st = check_device();
    if (st) return st;
    const unsigned nb = (unsigned)((n + 255) / 256);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == QJ2_FP32)
        minimg_kernel<float><<<nb, 256, 0, s>>>(n, (float)L[0], (float)L[1], (float)L[2], static_cast<const float *>(a),
                                                static_cast<const float *>(b), static_cast<float *>(out));
    else
        minimg_kernel<double><<<nb, 256, 0, s>>>(n, L[0], L[1], L[2], static_cast<const double *>(a),
                                                 static_cast<const double *>(b), static_cast<double *>(out));
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "minimg_kernel launch");
}

qj2_status qj2_check_inputs(const qj2_functor *fn, qj2_dtype dtype,
                            int64_t W, int64_t N_total, int64_t N_local, int64_t Np,
                            const void *R, const int32_t *k, int32_t P, const void *r_trial,
                            int32_t *d_flag, void *stream) {
    qj2_status st = validate_functor(fn);
    if (st) return st;
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype");
    if (W < 0 || N_total < 2 || N_local < 1 || Np < N_local || P < 1 || P > QJ2_MAX_P)
        return fail(QJ2_EINVAL, "bad sizes");
    if (W == 0) return QJ2_OK;
    if (!R || !k || !r_trial || !d_flag) return fail(QJ2_EINVAL, "NULL pointer");
    st = check_device();
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == QJ2_FP32)
        check_kernel<float><<<1184, 256, 0, s>>>(W, N_total, N_local, Np, (float)fn->L[0], (float)fn->L[1], (float)fn->L[2],
                                                 static_cast<const float *>(R), k, P, static_cast<const float *>(r_trial), d_flag);
    else
        check_kernel<double><<<1184, 256, 0, s>>>(W, N_total, N_local, Np, fn->L[0], fn->L[1], fn->L[2],
                                                  static_cast<const double *>(R), k, P, static_cast<const double *>(r_trial), d_flag);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "check_kernel launch");
}

// ---------------------------------------------------------------------------
// Host-buffer path: two staging buffers, H2D of chunk c+1 overlaps kernel c.
// ---------------------------------------------------------------------------
static void host_layout(int64_t W, int32_t P, int64_t Np, qj2_dtype dtype, int64_t cw, size_t off[8]) {
    const size_t sz = dtype == QJ2_FP32 ? 4 : 8;
    size_t evalws, a, b;
    ws_layout(cw, P, Np, dtype, &a, &b);
    evalws = a + b;
    off[0] = 0;                                                   // eval workspace (per chunk)
    off[1] = off[0] + align256(evalws);                           // R staging x2
    off[2] = off[1] + 2 * align256((size_t)cw * 3 * Np * sz);     // k staging x2
    off[3] = off[2] + 2 * align256((size_t)cw * 4);               // r_trial staging x2
    off[4] = off[3] + 2 * align256((size_t)cw * P * 3 * sz);      // out [W][P][5]
    off[5] = off[4] + align256((size_t)W * P * 5 * 8);            // ratio [W][P][2]
    off[6] = off[5] + align256((size_t)W * P * 2 * 8);            // V_cur [W]
    off[7] = off[6] + align256((size_t)W * 8);                    // total
}

qj2_status qj2_eval_host_workspace_size(int64_t W, int32_t P, int64_t Np, qj2_dtype dtype,
                                        int64_t chunk_walkers, size_t *bytes) {
    if (!bytes) return fail(QJ2_EINVAL, "bytes is NULL");
    if (W < 0 || P < 1 || P > QJ2_MAX_P || Np < 1 || chunk_walkers < 1) return fail(QJ2_EINVAL, "bad sizes");
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype");
    size_t off[8];
    host_layout(W, P, Np, dtype, chunk_walkers < W ? chunk_walkers : (W > 0 ? W : 1), off);
    *bytes = off[7];
    return QJ2_OK;
}

qj2_status qj2_eval_host(const qj2_functor *fn, qj2_dtype dtype,
                         int64_t W, int64_t N_total, int64_t N_up,
                         int64_t i_offset, int64_t N_local, int64_t Np,
                         const void *R_host, const int32_t *k_host, int32_t P, const void *r_trial_host,
                         double *out_host, const double *V_cur_host, double *ratio_out_host,
                         int64_t chunk_walkers, void *workspace, size_t workspace_bytes, void *stream) {
    if (chunk_walkers < 1) return fail(QJ2_EINVAL, "chunk_walkers < 1");
    if (W < 0) return fail(QJ2_EINVAL, "W < 0");
    if (W == 0) return validate_functor(fn);
    if (!R_host || !k_host || !r_trial_host || !out_host) return fail(QJ2_EINVAL, "NULL host pointer");
    const int64_t cw = chunk_walkers < W ? chunk_walkers : W;
    size_t off[8];
    if (P < 1 || P > QJ2_MAX_P) return fail(QJ2_EINVAL, "P must be in [1, %d]", QJ2_MAX_P);
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype");
    host_layout(W, P, Np, dtype, cw, off);
    if (!workspace || workspace_bytes < off[7]) return fail(QJ2_EINVAL, "workspace too small: need %zu bytes", off[7]);
    qj2_status st = check_device();
    if (st) return st;
    char *ws = static_cast<char *>(workspace);
    const size_t sz = dtype == QJ2_FP32 ? 4 : 8;
    const size_t rbytes = (size_t)cw * 3 * Np * sz, kbytes = (size_t)cw * 4, tbytes = (size_t)cw * P * 3 * sz;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaStream_t cs = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
    }
    double *out_d = reinterpret_cast<double *>(ws + off[4]);
    double *ratio_d = ratio_out_host ? reinterpret_cast<double *>(ws + off[5]) : nullptr;
    double *vcur_d = V_cur_host ? reinterpret_cast<double *>(ws + off[6]) : nullptr;
    // the copy stream must not start before prior work on the caller's stream
    cudaEvent_t start_ev = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&start_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(start_ev, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, start_ev, 0);
    if (e == cudaSuccess && vcur_d) e = cudaMemcpyAsync(vcur_d, V_cur_host, (size_t)W * 8, cudaMemcpyHostToDevice, cs);
    for (int64_t c0 = 0, ci = 0; e == cudaSuccess && c0 < W; c0 += cw, ++ci) {
        const int b = (int)(ci & 1);
        const int64_t n = (W - c0) < cw ? (W - c0) : cw;
        char *Rd = ws + off[1] + b * align256(rbytes);
        int32_t *kd = reinterpret_cast<int32_t *>(ws + off[2] + b * align256(kbytes));
        char *td = ws + off[3] + b * align256(tbytes);
        if (ci >= 2) e = cudaStreamWaitEvent(cs, freed[b], 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(Rd, static_cast<const char *>(R_host) + (size_t)c0 * 3 * Np * sz,
                                                  (size_t)n * 3 * Np * sz, cudaMemcpyHostToDevice, cs);
        if (e == cudaSuccess) e = cudaMemcpyAsync(kd, k_host + c0, (size_t)n * 4, cudaMemcpyHostToDevice, cs);
        if (e == cudaSuccess) e = cudaMemcpyAsync(td, static_cast<const char *>(r_trial_host) + (size_t)c0 * P * 3 * sz,
                                                  (size_t)n * P * 3 * sz, cudaMemcpyHostToDevice, cs);
        if (e == cudaSuccess) e = cudaEventRecord(copied[b], cs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, copied[b], 0);
        if (e != cudaSuccess) break;
        st = eval_impl(fn, dtype, n, N_total, N_up, i_offset, N_local, Np, Rd, kd, P, td,
                       out_d + c0 * P * 5, nullptr, vcur_d ? vcur_d + c0 : nullptr,
                       ratio_d ? ratio_d + c0 * P * 2 : nullptr, ws + off[0], off[1] - off[0], s, false);
        if (st) break;
        e = cudaEventRecord(freed[b], s);
    }
    if (e == cudaSuccess && !st) e = cudaMemcpyAsync(out_host, out_d, (size_t)W * P * 5 * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && !st && ratio_d)
        e = cudaMemcpyAsync(ratio_out_host, ratio_d, (size_t)W * P * 2 * 8, cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = e2;
    cudaStreamSynchronize(cs);
    for (int i = 0; i < 2; ++i) {
        if (copied[i]) cudaEventDestroy(copied[i]);
        if (freed[i]) cudaEventDestroy(freed[i]);
    }
    if (start_ev) cudaEventDestroy(start_ev);
    if (cs) cudaStreamDestroy(cs);
    if (st) return st;
    if (e != cudaSuccess) return cuda_fail(e, "qj2_eval_host");
    return QJ2_OK;
}

}  // extern "C"
