// j2_kernels.cuh -- the hot-path kernels (included by qmcj2.cu).
//
// One kernel core serves two rows of SURVEY.md section 8:
//   * J2 (section 8(a), the hot path): sources = the walker's own electrons,
//     self-exclusion i != k, two source groups (spin halves);
//     a group's functor is the same-spin or opposite-spin channel relative to
//     k's spin.
//   * J1 (NEXT-1): sources = the ions, shared by all walkers (walker stride 0,
//     PAPER:1306-1308), no self term, one source group per species, each with
//     its own functor, cutoff and interval count.
// Sources are contiguous groups [grp_start[g], grp_start[g+1]); a sub-tile
// inside one group is "clean" and runs with uniform functor constants.
//
// Accumulation: per sub-tile each thread sums <= 32 terms in T (raw Horner
// outputs), then flushes to fp64 with the sub-tile's group scale factors, so
// the fp64 accumulators hold physical (V, Gx, Gy, Gz, L)
// ("quantities per walker ... in double precision").
#pragma once

namespace qj2 {

constexpr int TPB = 256;          // threads per CTA
#ifndef QJ2_ITERS
#define QJ2_ITERS 8
#endif
constexpr int ITERS = QJ2_ITERS;  // vector iterations per sub-tile: 32 fp32 terms per thread per trial (A/B: -DQJ2_ITERS=n)
#ifndef QJ2_SUB
#define QJ2_SUB 25
#endif
constexpr int SUB = QJ2_SUB;      // sub-tiles per CTA tile: 25 x 8192 fp32 sources (A/B builds: -DQJ2_SUB=n)

constexpr int NACC = 6;           // fp32 accumulators per trial: V, Gx, Gy, Gz, sum h, sum du/r
constexpr int NOUT = 5;           // fp64 physical outputs per trial: V, Gx, Gy, Gz, L
constexpr int MAXG = 4;           // source groups (J2: 2 spin halves; J1: up to 4 species)
constexpr int MAXTAB = MAXG * (QJ2_MAX_M + 1);

enum { MODE_J2 = 0, MODE_J1 = 1 };

// fp64 accumulators per trial: J2 keeps the 6 raw sums (one delta for every
// group: scaled once at the end); J1 keeps 5 physical values (species differ
// in delta: scaled at every sub-tile flush).
template <int MODE> __host__ __device__ constexpr int ndacc() { return MODE == MODE_J2 ? NACC : NOUT; }

// ---------------------------------------------------------------------------
// Kernel parameters (by value, __grid_constant__).
// ---------------------------------------------------------------------------
struct EvalParams {
    int64_t W, N_total, N_up, i_offset, N_local, Np;
    int64_t tiles_per_walker;     // ceil(N_local / CH)
    int32_t P, m;                 // m: J2 interval count
    int32_t mode;                 // MODE_J2 | MODE_J1 (the kernels are also templated on it)
    int32_t n_src_groups;         // J2: 2; J1: species
    int32_t n_tab;                // table rows to stage in shared memory
    int64_t src_stride;           // elements between walkers' source blocks (J2 3*Np, J1 0)
    int64_t grp_start[MAXG + 1];  // global source index boundaries of the groups
    int32_t grp_tab[MAXG];        // J1: first table row of species g
    int32_t grp_m[MAXG];          // J1: interval count of species g
    double grp_invd[MAXG];        // J1: 1/delta of species g
    const void *R;
    const int32_t *k;             // J2 only
    const void *r_trial;
    double *out;
    void *row_out;
    const double *V_cur;
    double *ratio_out;
    double *partials;             // [W][P][tiles][ndacc]
    unsigned int *counters;       // [W][P]
    double L[3];
    double inv_delta;             // J2: 1/delta
    float inv_delta_f;            // J2: 1/delta rounded to fp32
    double pcoef[MAXTAB][4];      // power basis per interval (J2: [0,m] same spin, [m+1,2m+1] opposite)
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
    QJ2_DCHECK(p.n_tab <= MAXTAB);
    for (int e = threadIdx.x; e < p.n_tab; e += blockDim.x) {
        Coef4<T> c;
        c.a0 = T(p.pcoef[e][0]);
        c.a1 = T(p.pcoef[e][1]);
        c.a2 = T(p.pcoef[e][2]);
        c.a3 = T(p.pcoef[e][3]);
        tab[e] = c;
    }
}

// Functor constants of one source group for the current walker.
template <typename T>
struct GroupC {
    uint32_t base;                    // shared address of the group's row 0
    T invd;                           // 1/delta
    typename Traits<T>::U clamp;      // m (the group's zero row)
    double sg, sh, ss;                // fp64 flush scales: G = sg*acc, L = sh*acc_h + ss*acc_s
};

__device__ __forceinline__ int src_group(const EvalParams &p, int64_t gi) {
    int g = 0;
    for (int b = 1; b < p.n_src_groups; ++b) g += (gi >= p.grp_start[b]) ? 1 : 0;
    return g;
}

// kg: group (spin half) of the walker's active electron (J2).  MODE is a
// template parameter so that, for J2, 1/delta and m are kernel-parameter
// constants and the base a select between two precomputed values: all
// warp-uniform, so they live in uniform registers and the hot loop keeps its
// regular registers for data.
template <typename T, int MODE>
__device__ __forceinline__ GroupC<T> group_consts(const EvalParams &p, int g, int kg, uint32_t tab_addr) {
    using Tr = Traits<T>;
    GroupC<T> c;
    double invd;
    if constexpr (MODE == MODE_J2) {
        c.base = tab_addr + ((g == kg) ? 0u : (uint32_t)((p.m + 1) * (int)sizeof(Coef4<T>)));
        c.invd = sizeof(T) == 4 ? T(p.inv_delta_f) : T(p.inv_delta);
        c.clamp = (typename Tr::U)p.m;
        invd = p.inv_delta;
    } else {
        c.base = tab_addr + (uint32_t)(p.grp_tab[g] * (int)sizeof(Coef4<T>));
        c.invd = T(p.grp_invd[g]);
        c.clamp = (typename Tr::U)p.grp_m[g];
        invd = p.grp_invd[g];
    }
    c.sg = -invd;
    c.sh = 2.0 * invd * invd;
    c.ss = 2.0 * invd;
    return c;
}

// Per-trial constants: the three axes' minimum-image constants.
template <typename T> struct Trial {
    Axis<T> ax, ay, az;
    AxisD d[3];       // PREC: the same trial coordinates for the fp64 geometry
};

// One source term with the fp64 geometry (PREC: fp32 functors finer than m = 16, whose
// fp32 t = r/delta would carry ~m 2^-23 of absolute error into the interval fraction):
// the displacement exactly in fp64, r and t in fp64, f rounded to T for the Horner
// (functor_from_r2_d, as the accept path); the gradient factors from the once-rounded
// displacement and 1/r.  Returns r; d* receive the rounded displacement.
template <typename T, bool GEN>
__device__ __forceinline__ T term_prec(T x, T y, T z, bool dead, const Trial<T> &tr, const GroupC<T> &gc,
                                       uint32_t base, T *acc, T &dx, T &dy, T &dz) {
    const double ddx = min_image_d((double)x, tr.d[0]);
    const double ddy = min_image_d((double)y, tr.d[1]);
    const double ddz = min_image_d((double)z, tr.d[2]);
    double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
    if (GEN) r2 = dead ? 1e30 : r2;
    T ir;
    const FunctorEval<T> e = functor_from_r2_d<T>(r2, -gc.sg, base, (int)gc.clamp, ir);
    dx = T(ddx);
    dy = T(ddy);
    dz = T(ddz);
    const T g = e.du * ir;
    acc[0] += e.u;
    acc[1] = fma(g, dx, acc[1]);
    acc[2] = fma(g, dy, acc[2]);
    acc[3] = fma(g, dz, acc[3]);
    acc[4] += e.h;
    acc[5] += g;
    return T(r2) * ir;
}

// Functor + accumulation for one source at squared distance r2 (and
// displacement d).  acc: V, Gx, Gy, Gz (sum du/r * d), H (sum h), S (sum du/r)
// in raw units (scaled at the flush), or, with PHYS, already scaled by this
// source's 1/delta (per-source groups in a masked J1 sub-tile).
template <typename T, bool PHYS = false>
__device__ __forceinline__ T accumulate(T dx, T dy, T dz, T r2, T inv_delta, uint32_t tab_base,
                                        typename Traits<T>::U clamp_bits, T *acc) {
    using Tr = Traits<T>;
    const T ir = Tr::rsqrt(r2);
    const T r = r2 * ir;
    const FunctorEval<T> e = functor_from_t<T>(r * inv_delta, tab_base, clamp_bits);
    T g = e.du * ir;
    T h = e.h;
    if (PHYS) {
        g *= inv_delta;                        // U'/r
        h *= T(2) * inv_delta * inv_delta;     // U''
    }
    acc[0] += e.u;
    acc[1] = fma(g, dx, acc[1]);
    acc[2] = fma(g, dy, acc[2]);
    acc[3] = fma(g, dz, acc[3]);
    acc[4] += h;
    acc[5] += g;
    return r;
}

// A sub-tile that is not "clean": ragged length, holds the self source k, or
// straddles a group boundary.  Offsets relative to the sub-tile start.
struct SubMask {
    int len;          // valid sources in the sub-tile
    int k_rel;        // self source, or -1
    int64_t g0;       // global index of the sub-tile's first source
    int up_rel;       // J2: first spin-down source of the sub-tile (len if none)
    uint32_t base_hi; // J2: table base of the spin-down sources
};

// One sub-tile.  Every thread walks ITERS vectors at a constant stride of NT
// vectors, so every load address is base + immediate; PF vector groups are in
// flight ahead of the one being consumed (software pipelining).
// GEN = false: full sub-tile, no self source, one group (constants gc).
// GEN = true: vector indices clamped into the sub-tile (vectors past the end
// reload the last valid vector; their sources are dead) so loads stay
// unpredicated; per source, dead sources (self, padding) get r^2 = BIG, which
// lands on the all-zero interval (every accumulated quantity exactly 0), and
// the source's group picks the functor.  J2 groups share delta, so only the
// table row changes (raw accumulation); J1 groups differ in delta, so GEN
// sub-tiles accumulate physical units (PHYS).
template <typename T, bool ROW, int PF, bool GEN, int NT, int MODE, bool PREC = false>
__device__ __forceinline__ void tile_run(int tid, const EvalParams &p, int kg, uint32_t tab_addr,
                                         const typename Traits<T>::V *__restrict__ px,
                                         const typename Traits<T>::V *__restrict__ py,
                                         const typename Traits<T>::V *__restrict__ pz,
                                         const Trial<T> &tr, const GroupC<T> &gc,
                                         const SubMask &mk, T (&acc)[NACC],
                                         typename Traits<T>::V *rowp, int64_t row_stride) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
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
            V ro[4];
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                bool dead = false;
                uint32_t base = gc.base;
                if (GEN) {
                    const int li = rel + e;
                    dead = (li >= mk.len) || (li == mk.k_rel);
                    if (MODE == MODE_J2) base = li < mk.up_rel ? gc.base : mk.base_hi;   // spin halves
                }
                const T x = Tr::comp(bx[it], e), y = Tr::comp(by[it], e), z = Tr::comp(bz[it], e);
                T dx, dy, dz, r;
                if constexpr (PREC) {
                    r = term_prec<T, GEN>(x, y, z, dead, tr, gc, base, acc, dx, dy, dz);
                } else {
                    dx = min_image(x, tr.ax);
                    dy = min_image(y, tr.ay);
                    dz = min_image(z, tr.az);
                    T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                    if (GEN) r2 = dead ? T(1e30) : r2;
                    r = accumulate<T>(dx, dy, dz, r2, gc.invd, base, gc.clamp, acc);
                }
                if (ROW) { Tr::set(ro[0], e, r); Tr::set(ro[1], e, dx); Tr::set(ro[2], e, dy); Tr::set(ro[3], e, dz); }
            }
            if (ROW) {
#pragma unroll
                for (int c = 0; c < 4; ++c) __stcs(rowp + c * row_stride + it * NT, ro[c]);
            }
        }
    }
}

// A clean sub-tile with 256-bit loads (sm_100 `ld.v8.f32` / `ld.v4.f64`, SASS LDG.E.ENL2.256):
// thread tid takes the vector pairs (2 tid, 2 tid + 1) + 2 NT j, j < ITERS / 2 -- the same
// 32 terms per thread, half the load instructions, and a streaming read that reaches 7.40
// instead of 7.28 TB/s on this pattern (tools/probe/read_probe.cu).  px: the sub-tile's
// vector tid (the v4 mapping's base), so px + tid is this thread's first pair; rows must be
// 32-byte aligned (the host checks).  PFP pairs in flight ahead of the one consumed.
template <typename T> struct Pair8 { typename Traits<T>::V a, b; };   // 32 bytes: two vectors
__device__ __forceinline__ Pair8<float> ld_stream8(const float4 *p) {
    Pair8<float> v;
    asm("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y), "=f"(v.b.z), "=f"(v.b.w)
        : "l"(p));
    return v;
}
__device__ __forceinline__ Pair8<double> ld_stream8(const double2 *p) {
    Pair8<double> v;
    asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.a.x), "=d"(v.a.y), "=d"(v.b.x), "=d"(v.b.y) : "l"(p));
    return v;
}

template <typename T, int PFP, int NT>
__device__ __forceinline__ void tile_run_v8(int tid, const typename Traits<T>::V *__restrict__ px,
                                            const typename Traits<T>::V *__restrict__ py,
                                            const typename Traits<T>::V *__restrict__ pz, const Trial<T> &tr,
                                            const GroupC<T> &gc, T (&acc)[NACC]) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int NP = ITERS / 2;                  // vector pairs per thread
    const V *qx = px + tid, *qy = py + tid, *qz = pz + tid;
    Pair8<T> bx[NP], by[NP], bz[NP];
#pragma unroll
    for (int j = 0; j < PFP && j < NP; ++j) {
        bx[j] = ld_stream8(qx + j * 2 * NT);
        by[j] = ld_stream8(qy + j * 2 * NT);
        bz[j] = ld_stream8(qz + j * 2 * NT);
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        if (j + PFP < NP) {
            bx[j + PFP] = ld_stream8(qx + (j + PFP) * 2 * NT);
            by[j + PFP] = ld_stream8(qy + (j + PFP) * 2 * NT);
            bz[j + PFP] = ld_stream8(qz + (j + PFP) * 2 * NT);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const V vx = h ? bx[j].b : bx[j].a, vy = h ? by[j].b : by[j].a, vz = h ? bz[j].b : bz[j].a;
#pragma unroll
            for (int e = 0; e < Tr::VW; ++e) {
                const T dx = min_image(Tr::comp(vx, e), tr.ax);
                const T dy = min_image(Tr::comp(vy, e), tr.ay);
                const T dz = min_image(Tr::comp(vz, e), tr.az);
                const T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                accumulate<T>(dx, dy, dz, r2, gc.invd, gc.base, gc.clamp, acc);
            }
        }
    }
}

// A J1 sub-tile straddling a species boundary: rare, so a compact rolled
// loop (one vector per iteration, no prefetch) keeps the instruction
// footprint small.  The species is looked up per source and the terms are
// accumulated in physical units because species differ in delta.  (J2's spin
// straddle stays in the pipelined loop: both halves share delta.)
template <typename T, bool ROW, int NT, int MODE>
__device__ __forceinline__ void tile_multi(int tid, const EvalParams &p, int kg, uint32_t tab_addr,
                                           const typename Traits<T>::V *__restrict__ px,
                                           const typename Traits<T>::V *__restrict__ py,
                                           const typename Traits<T>::V *__restrict__ pz,
                                           const Trial<T> &tr, const SubMask &mk, T (&acc)[NACC],
                                           typename Traits<T>::V *rowp, int64_t row_stride) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
        const int rel = (it * NT + tid) * VW;
        if (rel >= mk.len) break;
        const V vx = Tr::ld_stream(px + it * NT), vy = Tr::ld_stream(py + it * NT), vz = Tr::ld_stream(pz + it * NT);
        V ro[4];
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            const int li = rel + e;
            const bool dead = (li >= mk.len) || (li == mk.k_rel);
            const int gsrc = MODE == MODE_J2 ? (mk.g0 + li >= p.N_up ? 1 : 0) : src_group(p, mk.g0 + li);
            const GroupC<T> ge = group_consts<T, MODE>(p, gsrc, kg, tab_addr);
            const T x = Tr::comp(vx, e), y = Tr::comp(vy, e), z = Tr::comp(vz, e);
            const T dx = min_image(x, tr.ax);
            const T dy = min_image(y, tr.ay);
            const T dz = min_image(z, tr.az);
            T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
            r2 = dead ? T(1e30) : r2;
            const T r = accumulate<T, MODE == MODE_J1>(dx, dy, dz, r2, ge.invd, ge.base, ge.clamp, acc);
            if (ROW) { Tr::set(ro[0], e, r); Tr::set(ro[1], e, dx); Tr::set(ro[2], e, dy); Tr::set(ro[3], e, dz); }
        }
        if (ROW) {
#pragma unroll
            for (int c = 0; c < 4; ++c) __stcs(rowp + c * row_stride + it * NT, ro[c]);
        }
    }
}

// A J2 sub-tile that is not clean (holds k, straddles N_up, or is ragged), as a compact
// rolled loop: one vector group per iteration, the next one loaded ahead.  Small code
// (one copy of the term instead of ITERS x VW) for kernels whose warps run clean and
// masked sub-tiles at the same time (the warp kernel: one masked sub-tile of six at C4).
template <typename T, bool ROW, int NT, bool PREC = false>
__device__ __forceinline__ void tile_gen_compact(int tid, const typename Traits<T>::V *__restrict__ px,
                                                 const typename Traits<T>::V *__restrict__ py,
                                                 const typename Traits<T>::V *__restrict__ pz, const Trial<T> &tr,
                                                 const GroupC<T> &gc, const SubMask &mk, T (&acc)[NACC],
                                                 typename Traits<T>::V *rowp, int64_t row_stride) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    const int vmax = (mk.len - 1) / VW;
    auto ld = [&](int it, V &x, V &y, V &z) {
        const int o = min(it * NT + tid, vmax) - tid;
        x = Tr::ld_stream(px + o); y = Tr::ld_stream(py + o); z = Tr::ld_stream(pz + o);
    };
    V nx, ny, nz;
    ld(0, nx, ny, nz);
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
        const int rel = (it * NT + tid) * VW;
        const V bx = nx, by = ny, bz = nz;
        if (it + 1 < ITERS) ld(it + 1, nx, ny, nz);
        if (rel < mk.len) {
            V ro[4];
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const int li = rel + e;
                const bool dead = (li >= mk.len) || (li == mk.k_rel);
                const uint32_t base = li < mk.up_rel ? gc.base : mk.base_hi;
                T dx, dy, dz, r;
                if constexpr (PREC) {
                    r = term_prec<T, true>(Tr::comp(bx, e), Tr::comp(by, e), Tr::comp(bz, e), dead, tr, gc, base, acc,
                                           dx, dy, dz);
                } else {
                    dx = min_image(Tr::comp(bx, e), tr.ax);
                    dy = min_image(Tr::comp(by, e), tr.ay);
                    dz = min_image(Tr::comp(bz, e), tr.az);
                    T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                    r2 = dead ? T(1e30) : r2;
                    r = accumulate<T>(dx, dy, dz, r2, gc.invd, base, gc.clamp, acc);
                }
                if (ROW) { Tr::set(ro[0], e, r); Tr::set(ro[1], e, dx); Tr::set(ro[2], e, dy); Tr::set(ro[3], e, dz); }
            }
            if (ROW) {
#pragma unroll
                for (int c = 0; c < 4; ++c) __stcs(rowp + c * row_stride + it * NT, ro[c]);
            }
        }
    }
}

// Flush a sub-tile's T partials into the fp64 accumulators: raw for J2,
// physical (scaled by the sub-tile group's delta factors) for J1.
template <typename T, int MODE>
__device__ __forceinline__ void flush(T (&acc)[NACC], double (&dacc)[ndacc<MODE>()], double sg, double sh, double ss) {
    if constexpr (MODE == MODE_J2) {
#pragma unroll
        for (int a = 0; a < NACC; ++a) dacc[a] += (double)acc[a];
    } else {
        dacc[0] += (double)acc[0];
        dacc[1] += sg * (double)acc[1];
        dacc[2] += sg * (double)acc[2];
        dacc[3] += sg * (double)acc[3];
        dacc[4] += sh * (double)acc[4] + ss * (double)acc[5];
    }
}

// Physical (V, G, L) of one trial from the reduced fp64 accumulators.
template <int MODE>
__device__ __forceinline__ void to_physical(const EvalParams &p, const double *s, double (&o)[NOUT]) {
    if constexpr (MODE == MODE_J2) {
        const double id = p.inv_delta;
        o[0] = s[0];
        o[1] = -id * s[1];
        o[2] = -id * s[2];
        o[3] = -id * s[3];
        o[4] = 2.0 * id * id * s[4] + 2.0 * id * s[5];
    } else {
#pragma unroll
        for (int a = 0; a < NOUT; ++a) o[a] = s[a];
    }
}

// Process the sub-tile [sstart, send) (local indices) of one walker for a team
// of NT threads: classify, run the clean or the masked loop, flush to fp64.
template <typename T, bool ROW, int PF, int NT, int MODE>
__device__ __forceinline__ void sub_tile(int tid, const EvalParams &p, int kg, uint32_t tab_addr,
                                         int64_t sstart, int64_t send, int64_t k_local,
                                         const typename Traits<T>::V *px, const typename Traits<T>::V *py,
                                         const typename Traits<T>::V *pz, const Trial<T> &tr,
                                         double (&dacc)[ndacc<MODE>()], typename Traits<T>::V *rp,
                                         int64_t row_stride) {
    constexpr int SCH = NT * Traits<T>::VW * ITERS;
    T acc[NACC];
#pragma unroll
    for (int a = 0; a < NACC; ++a) acc[a] = T(0);
    const int64_t g0 = sstart + p.i_offset;                 // global index of the first source
    int grp;
    bool one_group;
    if constexpr (MODE == MODE_J2) {                        // two spin halves: one compare each
        grp = g0 >= p.N_up ? 1 : 0;
        one_group = (send - 1 + p.i_offset >= p.N_up ? 1 : 0) == grp;
    } else {
        grp = src_group(p, g0);
        one_group = src_group(p, send - 1 + p.i_offset) == grp;
    }
    const bool k_in = k_local >= sstart && k_local < send;
    SubMask mk;
    mk.len = (int)(send - sstart);
    mk.k_rel = k_in ? (int)(k_local - sstart) : -1;
    mk.g0 = g0;
    mk.up_rel = mk.len;
    const GroupC<T> gc = group_consts<T, MODE>(p, grp, kg, tab_addr);
    mk.base_hi = gc.base;
    if constexpr (MODE == MODE_J2) {
        if (!one_group) {           // straddles N_up: both halves share delta, select the table per source
            mk.up_rel = (int)(p.N_up - g0);
            mk.base_hi = group_consts<T, MODE>(p, 1, kg, tab_addr).base;
        }
    }
    if (mk.len == SCH && !k_in && one_group) {                 // clean
        tile_run<T, ROW, PF, false, NT, MODE>(tid, p, kg, tab_addr, px, py, pz, tr, gc, mk, acc, rp, row_stride);
        flush<T, MODE>(acc, dacc, gc.sg, gc.sh, gc.ss);
    } else if (one_group || MODE == MODE_J2) {                // ragged, holds k, or straddles N_up (J2)
        tile_run<T, ROW, PF, true, NT, MODE>(tid, p, kg, tab_addr, px, py, pz, tr, gc, mk, acc, rp, row_stride);
        flush<T, MODE>(acc, dacc, gc.sg, gc.sh, gc.ss);
    } else {                                                   // J1: straddles a species boundary
        tile_multi<T, ROW, NT, MODE>(tid, p, kg, tab_addr, px, py, pz, tr, mk, acc, rp, row_stride);
        if constexpr (MODE == MODE_J2) flush<T, MODE>(acc, dacc, gc.sg, gc.sh, gc.ss);   // shared delta: raw
        else flush<T, MODE>(acc, dacc, -1.0, 1.0, 2.0);                                  // already physical
    }
}

// J2 sub-tile with 32-bit classification relative to the walker's tile
// (tile length tlen, k at k_t or -1, sources [0, up_t) of the tile spin-up)
// and the two per-walker functor constant sets.  s0: the sub-tile's offset.
template <typename T, bool ROW, int PF, int NT, bool COMPACT_GEN = false, bool PREC = false, bool V8 = false>
__device__ __forceinline__ void j2_sub_tile32(int tid, const EvalParams &p, int kg, uint32_t tab_addr, int32_t s0,
                                              int32_t tlen, int32_t k_t, int32_t up_t, const GroupC<T> &g_up,
                                              const GroupC<T> &g_dn, const typename Traits<T>::V *px,
                                              const typename Traits<T>::V *py, const typename Traits<T>::V *pz,
                                              const Trial<T> &tr, double (&dacc)[NACC], typename Traits<T>::V *rp,
                                              int64_t row_stride) {
    constexpr int SCH = NT * Traits<T>::VW * ITERS;
    const int32_t len = min(SCH, tlen - s0);
    const int32_t k_rel = k_t - s0;
    const bool k_in = k_t >= 0 && (uint32_t)k_rel < (uint32_t)len;
    const int32_t up_rel = up_t - s0;                 // sources [0, up_rel) of the sub-tile are spin-up
    const bool straddle = up_rel > 0 && up_rel < len;
    const GroupC<T> &gc = up_rel > 0 ? g_up : g_dn;   // the group of the sub-tile's first source
    T acc[NACC];
#pragma unroll
    for (int a = 0; a < NACC; ++a) acc[a] = T(0);
    SubMask mk;
    mk.len = len;
    mk.k_rel = k_in ? k_rel : -1;
    mk.g0 = 0;                                         // (J1 only)
    mk.up_rel = straddle ? up_rel : len;
    mk.base_hi = straddle ? g_dn.base : gc.base;
    if (len == SCH && !k_in && !straddle) {
        if constexpr (V8 && !ROW && !PREC)
            tile_run_v8<T, (PF + 1) / 2, NT>(tid, px, py, pz, tr, gc, acc);
        else
            tile_run<T, ROW, PF, false, NT, MODE_J2, PREC>(tid, p, kg, tab_addr, px, py, pz, tr, gc, mk, acc, rp,
                                                           row_stride);
    } else if constexpr (COMPACT_GEN)
        tile_gen_compact<T, ROW, NT, PREC>(tid, px, py, pz, tr, gc, mk, acc, rp, row_stride);
    else
        tile_run<T, ROW, PF, true, NT, MODE_J2, PREC>(tid, p, kg, tab_addr, px, py, pz, tr, gc, mk, acc, rp, row_stride);
    flush<T, MODE_J2>(acc, dacc, gc.sg, gc.sh, gc.ss);      // J2: raw sums (one delta for both groups)
}

// L2 prefetch of a contiguous byte range by the TMA engine (no registers, no
// completion to wait for): the loads of a later sub-tile then hit L2.
__device__ __forceinline__ void l2_prefetch(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// CTA kernel, J2: how many sub-tiles ahead the TMA engine prefetches into L2 (0: none).
// fp64: one (C3f64 2.78 -> 2.51 ms per step: the register pipeline holds only two
// vector groups per thread at 2 CTAs/SM, the prefetch turns its loads into L2 hits);
// fp32: none (its 3 CTAs/SM already keep the HBM busy; the prefetch costs 10-20%:
// profiles/r02/ab_results.txt).  A/B builds: -DQJ2_L2PF64=n / -DQJ2_L2PF32=n.
#ifndef QJ2_L2PF64
#define QJ2_L2PF64 1
#endif
#ifndef QJ2_L2PF32
#define QJ2_L2PF32 0
#endif

// Per-walker setup shared by the CTA and warp kernels.
template <typename T, int MODE, bool PREC = false>
__device__ __forceinline__ void walker_setup(const EvalParams &p, int64_t w, int32_t g, Trial<T> &tr, int &kg,
                                             int64_t &k_local) {
    const int64_t kw = MODE == MODE_J2 ? (int64_t)p.k[w] : -1;
    kg = (MODE == MODE_J2 && kw >= p.N_up) ? 1 : 0;
    k_local = MODE == MODE_J2 ? kw - p.i_offset : -1;
    const T *rt = static_cast<const T *>(p.r_trial) + ((w * p.P + g) * 3);
    tr.ax = make_axis<T>(rt[0], T(p.L[0]));
    tr.ay = make_axis<T>(rt[1], T(p.L[1]));
    tr.az = make_axis<T>(rt[2], T(p.L[2]));
    if constexpr (PREC) {     // the cell as the kernel's type sees it (fp32 L for fp32 positions)
#pragma unroll
        for (int d = 0; d < 3; ++d) tr.d[d] = make_axis_d((double)rt[d], (double)T(p.L[d]));
    }
}

// Write the physical totals of trial g of walker w and the fused ratio (against V_cur,
// or, for P = 1 without V_cur, against this trial itself: the host launches a separate
// ratio kernel when P > 1 and V_cur == NULL).
template <int MODE>
__device__ __forceinline__ void write_out(const EvalParams &p, int64_t w, int32_t g, const double *sraw) {
    double s[NOUT];
    to_physical<MODE>(p, sraw, s);
    const int64_t o = w * p.P + g;
#pragma unroll
    for (int a = 0; a < NOUT; ++a) p.out[o * 5 + a] = s[a];
    if (p.ratio_out) {   // e^{dJ} factor of Eq. 4 (host guarantees a valid reference)
        const double dj = s[0] - (p.V_cur ? p.V_cur[w] : s[0]);
        p.ratio_out[o * 2 + 0] = dj;
        p.ratio_out[o * 2 + 1] = exp(dj);
    }
}

// CTA reduction in fp64 (fixed order: deterministic), cross-tile partials
// (the last CTA of (w, g) reduces them) and the physical write-out.  red:
// [TPB/32][ND] shared doubles.
template <int MODE>
__device__ __forceinline__ void cta_reduce_write(const EvalParams &p, const double (&dacc)[ndacc<MODE>()], int64_t w,
                                                 int32_t g, int64_t c, double *red, int *last_flag) {
    constexpr int ND = ndacc<MODE>();
    const int64_t tpw = p.tiles_per_walker;
    QJ2_DCHECK(tpw == 1 || (p.partials != nullptr && p.counters != nullptr));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < ND; ++a) {
        const double v = warp_sum(dacc[a]);
        if (lane == 0) red[warp * ND + a] = v;
    }
    __syncthreads();

    double tot = 0.0;   // thread t < ND holds value t of this tile
    if (threadIdx.x < ND) {
#pragma unroll
        for (int wi = 0; wi < TPB / 32; ++wi) tot += red[wi * ND + threadIdx.x];
    }

    const int64_t wg = w * p.P + g;
    if (tpw > 1) {
        // publish this tile's partials; the last CTA of (w, g) reduces them
        double *part = p.partials + (wg * tpw + c) * ND;
        if (threadIdx.x < ND) part[threadIdx.x] = tot;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned prev = atomicAdd(p.counters + wg, 1u);
            *last_flag = (prev == (unsigned)(tpw - 1));
        }
        __syncthreads();
        if (!*last_flag) return;
        __threadfence();
        // warp 0: value v summed over tiles, lane-strided then shuffle tree
        if (warp == 0) {
            const double *base = p.partials + wg * tpw * ND;
            for (int v = 0; v < ND; ++v) {
                double s = 0.0;
                for (int64_t t = lane; t < tpw; t += 32) s += __ldcg(base + t * ND + v);
                s = warp_sum(s);
                if (lane == v) tot = s;      // lane v keeps value v (ND <= 6 < 32)
            }
        }
    }

    // ---- finalize: lane a < ND of warp 0 holds value a ----
    if (warp == 0) {
        double s[ND];
#pragma unroll
        for (int a = 0; a < ND; ++a) s[a] = __shfl_sync(0xffffffffu, tot, a);
        if (lane == 0) write_out<MODE>(p, w, g, s);
    }
}

// ===========================================================================
// Long rows: one CTA per (walker, trial, tile of SUB sub-tiles).
// PF: prefetch distance (vector groups in flight), MINB: resident CTAs per SM.
// ===========================================================================
template <typename T, bool ROW, int PF, int MINB, int MODE = MODE_J2, bool PREC = false, bool V8 = false>
__global__ void __launch_bounds__(TPB, MINB)
j2_eval_kernel(const __grid_constant__ EvalParams p) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    constexpr int SCH = TPB * VW * ITERS;         // sub-tile: 32 terms per thread
    constexpr int CH = SCH * SUB;                 // tile handled by one CTA
    constexpr int ND = ndacc<MODE>();
    __shared__ Coef4<T> tab[MAXTAB];
    __shared__ double red[TPB / 32 * ND];
    __shared__ int last_flag;

    // tile decode: trial fastest, then tile, then walker, so the CTAs of one tile's
    // trials run together (one HBM read, L2 hits for the others) and consecutive
    // tiles stream consecutive memory (32-bit arithmetic: the host guarantees
    // W * P * tiles < 2^31)
    const uint32_t b = blockIdx.x;
    const uint32_t P32 = (uint32_t)p.P;
    const uint32_t per_w = (uint32_t)p.tiles_per_walker * P32;
    const uint32_t w32 = b / per_w;
    const uint32_t rem = b - w32 * per_w;
    const uint32_t c32 = rem / P32;
        const int64_t w = w32, c = c32;
    const int32_t g = (int32_t)(rem - c32 * P32);

    load_table<T>(p, tab);
    Trial<T> tr;
    int kg;
    int64_t k_local;
    walker_setup<T, MODE, PREC>(p, w, g, tr, kg, k_local);
    const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tab);

    const int64_t start = c * CH;
    const int64_t end = min(start + (int64_t)CH, p.N_local);
    // every vector this CTA loads (and row vector it stores) lies in [start, end) of lanes of Np
    QJ2_DCHECK(w < p.W && g < p.P && c < p.tiles_per_walker && start < end && end <= p.Np && p.N_local <= p.Np);
    const T *Rw = static_cast<const T *>(p.R) + w * p.src_stride;
    const int64_t voff = (start >> (VW == 4 ? 2 : 1)) + threadIdx.x;   // this thread's first vector
    const V *px = reinterpret_cast<const V *>(Rw) + voff;
    const V *py = reinterpret_cast<const V *>(Rw + p.Np) + voff;
    const V *pz = reinterpret_cast<const V *>(Rw + 2 * p.Np) + voff;
    V *rowp = ROW ? reinterpret_cast<V *>(static_cast<T *>(p.row_out) + ((w * p.P + g) * 4) * p.Np) + voff : nullptr;
    const int64_t row_stride = p.Np / VW;
    __syncthreads();

    double dacc[ND];
#pragma unroll
    for (int a = 0; a < ND; ++a) dacc[a] = 0.0;

    if constexpr (MODE == MODE_J2) {
        // J2: classify sub-tiles with 32-bit offsets relative to the tile, from
        // three per-CTA values (length, k, first spin-down source), and the two
        // per-CTA functor constant sets (same / opposite spin as k)
        const int32_t tlen = (int32_t)(end - start);
        const int32_t k_t = (k_local >= start && k_local < end) ? (int32_t)(k_local - start) : -1;
        const int64_t up64 = p.N_up - p.i_offset - start;
        const int32_t up_t = up64 <= 0 ? 0 : (up64 >= tlen ? tlen : (int32_t)up64);
        const GroupC<T> g_up = group_consts<T, MODE>(p, 0, kg, tab_addr);
        const GroupC<T> g_dn = group_consts<T, MODE>(p, 1, kg, tab_addr);
        constexpr int L2PF = sizeof(T) == 8 ? QJ2_L2PF64 : QJ2_L2PF32;
        // one thread asks the TMA engine for sub-tile s + L2PF of the three streams while
        // sub-tile s is loaded (sizes rounded up to 16 B stay inside the Np-padded rows)
        auto prefetch_sub = [&](int sp) {
            const int32_t a = sp * SCH;
            if (threadIdx.x == 0 && sp < SUB && a < tlen) {
                const uint32_t bytes = (uint32_t)((min(SCH, tlen - a) * (int)sizeof(T) + 15) & ~15);
#pragma unroll
                for (int d = 0; d < 3; ++d) l2_prefetch(Rw + d * p.Np + start + a, bytes);
            }
        };
#pragma unroll
        for (int sp = 1; sp < L2PF; ++sp) prefetch_sub(sp);
#pragma unroll 1
        for (int sidx = 0; sidx < SUB; ++sidx) {
            const int32_t s0 = sidx * SCH;
            if (s0 >= tlen) break;
            if constexpr (L2PF > 0) prefetch_sub(sidx + L2PF);
            const int64_t vs = (int64_t)sidx * (SCH / VW);
            j2_sub_tile32<T, ROW, PF, TPB, false, PREC, V8>(threadIdx.x, p, kg, tab_addr, s0, tlen, k_t, up_t, g_up, g_dn, px + vs,
                                           py + vs, pz + vs, tr, dacc, ROW ? rowp + vs : nullptr, row_stride);
        }
    } else {
#pragma unroll 1
        for (int sidx = 0; sidx < SUB; ++sidx) {
            const int64_t sstart = start + (int64_t)sidx * SCH;
            if (sstart >= end) break;
            const int64_t send = min(sstart + (int64_t)SCH, end);
            const int64_t vs = (int64_t)sidx * (SCH / VW);
            sub_tile<T, ROW, PF, TPB, MODE>(threadIdx.x, p, kg, tab_addr, sstart, send, k_local, px + vs, py + vs,
                                            pz + vs, tr, dacc, ROW ? rowp + vs : nullptr, row_stride);
        }
    }

    cta_reduce_write<MODE>(p, dacc, w, g, c, red, &last_flag);
}

// ===========================================================================
// Short rows with many walkers (C1, C2, C4 waves): one warp per (walker,
// trial) walks all of the walker's sources in per-warp sub-tiles of
// 32*VW*ITERS sources; the warp's fp64 shuffle tree is the whole
// (deterministic) reduction: no shared-memory reduction, no cross-CTA
// partials, no counters.  COMPACT_GEN (rows of >= 4 sub-tiles): the masked
// sub-tile (the one holding k, a straddle, the ragged end) runs the compact
// rolled loop, so the resident warps -- each at its own walker's clean or
// masked sub-tile -- share a 31 KB instead of a 52 KB instruction footprint
// (C4 wave: instruction-fetch stalls 25% of samples; 0.833 -> 0.886 of the
// HBM peak); short rows, where most sub-tiles are masked, keep the pipelined
// masked loop.
// ===========================================================================
template <typename T, bool ROW, int PF, int MINB, int MODE = MODE_J2, bool COMPACT_GEN = false, bool PREC = false,
          bool V8 = false>
__global__ void __launch_bounds__(TPB, MINB)
j2_eval_warp_kernel(const __grid_constant__ EvalParams p, int64_t n_units) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    constexpr int SCH = 32 * VW * ITERS;
    __shared__ Coef4<T> tab[MAXTAB];
    load_table<T>(p, tab);
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t unit = (int64_t)blockIdx.x * (TPB / 32) + warp;
    if (unit >= n_units) return;
    const int64_t w = unit / p.P;
    const int32_t g = (int32_t)(unit - w * p.P);
    QJ2_DCHECK(w < p.W && p.N_local <= p.Np && p.tiles_per_walker == 1);
    Trial<T> tr;
    int kg;
    int64_t k_local;
    walker_setup<T, MODE, PREC>(p, w, g, tr, kg, k_local);
    const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tab);
    const T *Rw = static_cast<const T *>(p.R) + w * p.src_stride;
    const int64_t row_stride = p.Np / VW;

    constexpr int ND = ndacc<MODE>();
    double dacc[ND];
#pragma unroll
    for (int a = 0; a < ND; ++a) dacc[a] = 0.0;

    // J2: per-walker 32-bit classification state (the slice is one tile)
    const int32_t tlen = (int32_t)p.N_local;
    const int32_t k_t = (MODE == MODE_J2 && k_local >= 0 && k_local < p.N_local) ? (int32_t)k_local : -1;
    const int64_t up64 = p.N_up - p.i_offset;
    const int32_t up_t = up64 <= 0 ? 0 : (up64 >= tlen ? tlen : (int32_t)up64);
    GroupC<T> g_up, g_dn;
    if constexpr (MODE == MODE_J2) {
        g_up = group_consts<T, MODE>(p, 0, kg, tab_addr);
        g_dn = group_consts<T, MODE>(p, 1, kg, tab_addr);
    }
    for (int64_t sstart = 0; sstart < p.N_local; sstart += SCH) {
        const int64_t send = min(sstart + (int64_t)SCH, p.N_local);
        const int64_t voff = (sstart / VW) + lane;
        const V *px = reinterpret_cast<const V *>(Rw) + voff;
        const V *py = reinterpret_cast<const V *>(Rw + p.Np) + voff;
        const V *pz = reinterpret_cast<const V *>(Rw + 2 * p.Np) + voff;
        V *rp = ROW ? reinterpret_cast<V *>(static_cast<T *>(p.row_out) + ((w * p.P + g) * 4) * p.Np) + voff : nullptr;
        if constexpr (MODE == MODE_J2)
            j2_sub_tile32<T, ROW, PF, 32, COMPACT_GEN, PREC, V8>(lane, p, kg, tab_addr, (int32_t)sstart, tlen, k_t, up_t, g_up,
                                                        g_dn, px, py, pz, tr, dacc, rp, row_stride);
        else
            sub_tile<T, ROW, PF, 32, MODE>(lane, p, kg, tab_addr, sstart, send, k_local, px, py, pz, tr, dacc, rp,
                                           row_stride);
    }

    double s[ND];
#pragma unroll
    for (int a = 0; a < ND; ++a) s[a] = warp_sum(dacc[a]);
    if (lane == 0) write_out<MODE>(p, w, g, s);
}


// ===========================================================================
// J1 with a small ion set (NEXT-1; NiO-64 has 64 ions): one thread per
// (walker, trial).  The ions (x|y|z, padded to 16 B per ion) and the
// species' functor rows are staged in shared memory once per CTA; every
// thread walks all ions species by species (a uniform loop: all lanes read
// the same ion, a shared-memory broadcast) with the species' constants, fp32
// partials of <= 32 terms flushed to fp64 in physical units.  No cross-thread
// reduction at all.  The ions are fixed and shared by every walker
// (PAPER:1306-1308).
// ===========================================================================
constexpr int J1_MAX_IONS = 4096;

template <typename T, bool PREC = false>
__global__ void __launch_bounds__(TPB) j1_thread_kernel(const __grid_constant__ EvalParams p, int64_t n_units) {
    using Tr = Traits<T>;
    __shared__ Coef4<T> tab[MAXTAB];
    extern __shared__ __align__(16) unsigned char j1_smem[];
    T *ion = reinterpret_cast<T *>(j1_smem);          // [n][4]: x, y, z, 0
    QJ2_DCHECK(p.N_local * 4 * (int64_t)sizeof(T) <= dyn_smem_bytes() && p.N_local <= p.Np && p.n_tab <= MAXTAB);
    load_table<T>(p, tab);
    const T *src = static_cast<const T *>(p.R);
    for (int64_t i = threadIdx.x; i < p.N_local; i += blockDim.x) {
        ion[i * 4 + 0] = src[i];
        ion[i * 4 + 1] = src[p.Np + i];
        ion[i * 4 + 2] = src[2 * p.Np + i];
        ion[i * 4 + 3] = T(0);
    }
    __syncthreads();
    const int64_t unit = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (unit >= n_units) return;
    const int64_t w = unit / p.P;
    const int32_t pp = (int32_t)(unit - w * p.P);
    const T *rt = static_cast<const T *>(p.r_trial) + unit * 3;
    const Axis<T> ax = make_axis<T>(rt[0], T(p.L[0])), ay = make_axis<T>(rt[1], T(p.L[1])),
                  az = make_axis<T>(rt[2], T(p.L[2]));
    Trial<T> trp;         // PREC (an fp32 species functor finer than m = 16): the fp64 geometry
    if constexpr (PREC) {
#pragma unroll
        for (int d = 0; d < 3; ++d) trp.d[d] = make_axis_d((double)rt[d], (double)T(p.L[d]));
    }
    const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tab);
    double dacc[NOUT] = {0.0, 0.0, 0.0, 0.0, 0.0};
    auto term = [&](int32_t i, const GroupC<T> &gc, T (&acc)[NACC]) {
        T x, y, z;
        if constexpr (sizeof(T) == 4) {
            const float4 v = reinterpret_cast<const float4 *>(ion)[i];    // one LDS.128 (broadcast)
            x = v.x; y = v.y; z = v.z;
        } else {
            const double2 v = reinterpret_cast<const double2 *>(ion)[2 * i];
            x = v.x; y = v.y; z = ion[i * 4 + 2];
        }
        if constexpr (PREC) {
            T dx, dy, dz;
            term_prec<T, false>(x, y, z, false, trp, gc, gc.base, acc, dx, dy, dz);
        } else {
            const T dx = min_image(x, ax), dy = min_image(y, ay), dz = min_image(z, az);
            const T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
            accumulate<T>(dx, dy, dz, r2, gc.invd, gc.base, gc.clamp, acc);
        }
    };
    for (int g = 0; g < p.n_src_groups; ++g) {
        GroupC<T> gc = group_consts<T, MODE_J1>(p, g, 0, tab_addr);
        // keep the species' row base as one value: otherwise the compiler re-associates
        // row offset and table base into every term's address (one more add per term)
        asm volatile("" : "+r"(gc.base));
        const int32_t i1 = (int32_t)p.grp_start[g + 1];
        for (int32_t i0 = (int32_t)p.grp_start[g]; i0 < i1; i0 += 32) {
            T acc[NACC] = {T(0), T(0), T(0), T(0), T(0), T(0)};
            if (i1 - i0 >= 32) {                 // full chunk: fixed trip count, fully pipelined
#pragma unroll 8
                for (int32_t i = 0; i < 32; ++i) term(i0 + i, gc, acc);
            } else {
#pragma unroll 1
                for (int32_t i = i0; i < i1; ++i) term(i, gc, acc);
            }
            dacc[0] += (double)acc[0];
            dacc[1] += gc.sg * (double)acc[1];
            dacc[2] += gc.sg * (double)acc[2];
            dacc[3] += gc.sg * (double)acc[3];
            dacc[4] += gc.sh * (double)acc[4] + gc.ss * (double)acc[5];
        }
    }
    double *o = p.out + unit * 5;
#pragma unroll
    for (int a = 0; a < NOUT; ++a) o[a] = dacc[a];
    if (p.ratio_out) {     // V_cur, or (P == 1) the fused reference is this unit itself
        const double dj = dacc[0] - (p.V_cur ? p.V_cur[w] : dacc[0]);
        p.ratio_out[unit * 2 + 0] = dj;
        p.ratio_out[unit * 2 + 1] = exp(dj);
    }
    (void)pp;
}

}  // namespace qj2
