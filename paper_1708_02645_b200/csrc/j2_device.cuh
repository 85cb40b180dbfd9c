// j2_device.cuh -- device building blocks of the J2 / distance-row hot path
// (arXiv 1708.02645), written for sm_100a.  Product code: shares nothing with
// oracle/.
//
// Layout/precision decisions are in DESIGN.md ("Kernels").  In short:
//  * minimum image with a single rounding (case split on the trial coordinate,
//    exact shifts by Sterbenz's lemma) -- PAPER:1298-1304, SPEC:113-121, 138;
//  * functor as a per-interval power basis in shared memory, evaluated by
//    Horner with branch-free cutoff (index clamped onto an all-zero interval)
//    -- PAPER:817-819, 1473-1475 ("branch conditions originated from the
//    finite cutoff");
//  * 1/r from MUFU rsqrt (fp32) / accurate rsqrt (fp64).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Debug build (-DQJ2_CHECK; tools/ab/build_check.sh): device-side checks of every
// index computed from the arguments before it addresses global or shared memory
// (the substitute for compute-sanitizer, which this pool does not offer).  A failed
// check prints its location and traps, so the launch fails with a sticky error.
#ifdef QJ2_CHECK
#define QJ2_DCHECK(cond)                                                                        \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("QJ2_CHECK failed at %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__,  \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                                   \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define QJ2_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace qj2 {

// Dynamic shared memory of the launch, in bytes (for QJ2_DCHECK of layouts).
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t x;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(x));
    return x;
}

// ---------------------------------------------------------------------------
// Type traits
// ---------------------------------------------------------------------------
template <typename T> struct Traits;

template <> struct Traits<float> {
    using V = float4;                       // 16-byte vector of sources
    static constexpr int VW = 4;
    using U = unsigned int;
    static constexpr float MAGIC = 12582912.0f;          // 1.5 * 2^23
    static constexpr unsigned MAGIC_BITS = 0x4B400000u;  // bits of MAGIC
    static __device__ __forceinline__ float add_rd(float a, float b) { return __fadd_rd(a, b); }
    static __device__ __forceinline__ unsigned bits(float a) { return __float_as_uint(a); }
    static __device__ __forceinline__ float rsqrt(float x) {
        float y;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    static __device__ __forceinline__ float4 ld_stream(const float4 *p) {
        float4 v;
        asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
            : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
        return v;
    }
    static __device__ __forceinline__ float comp(const float4 &v, int e) {
        return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
    }
    static __device__ __forceinline__ void set(float4 &v, int e, float x) {
        if (e == 0) v.x = x; else if (e == 1) v.y = x; else if (e == 2) v.z = x; else v.w = x;
    }
    static __device__ __forceinline__ float below(float L) {   // largest float < L (L > 0)
        return __uint_as_float(__float_as_uint(L) - 1u);
    }
};

template <> struct Traits<double> {
    using V = double2;
    static constexpr int VW = 2;
    using U = unsigned long long;
    static constexpr double MAGIC = 6755399441055744.0;                  // 1.5 * 2^52
    static constexpr unsigned long long MAGIC_BITS = 0x4338000000000000ull;
    static __device__ __forceinline__ double add_rd(double a, double b) { return __dadd_rd(a, b); }
    static __device__ __forceinline__ unsigned long long bits(double a) {
        return (unsigned long long)__double_as_longlong(a);
    }
    static __device__ __forceinline__ double rsqrt(double x) { return ::rsqrt(x); }
    static __device__ __forceinline__ double2 ld_stream(const double2 *p) {
        double2 v;
        asm("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];"
            : "=d"(v.x), "=d"(v.y) : "l"(p));
        return v;
    }
    static __device__ __forceinline__ double comp(const double2 &v, int e) { return e == 0 ? v.x : v.y; }
    static __device__ __forceinline__ void set(double2 &v, int e, double x) {
        if (e == 0) v.x = x; else v.y = x;
    }
    static __device__ __forceinline__ double below(double L) {
        return __longlong_as_double(__double_as_longlong(L) - 1ll);
    }
};

// One interval of the functor in power basis: U(f) = a0 + a1 f + a2 f^2 + a3 f^3,
// f in [0,1) the fractional position inside the interval.  Interval m (and
// every clamped index beyond) is all zeros: U = U' = U'' = 0 at r >= r_cut.
template <typename T> struct alignas(4 * sizeof(T)) Coef4 { T a0, a1, a2, a3; };

// ---------------------------------------------------------------------------
// Minimum image with one rounding.
// For a trial coordinate c in [0, L) only one wrap direction is possible:
//   case A (c <  L/2): wrap iff x > c + L/2, then d = (x - L) - c, where x - L
//                      is exact (x in [L/2, L): Sterbenz);
//   case B (c >= L/2): wrap iff x <= c - L/2, then d = x - (c - L), where
//                      c - L is exact.
// Unified per trial coordinate with 4 constants so the inner loop has no
// data-dependent branch:  hit = x > thr;  xs = hit ? x - a1 : x;
//                         d = xs - (hit ? b1 : b0).
// ---------------------------------------------------------------------------
template <typename T> struct Axis { T thr, a1, b1, b0; };

template <typename T>
__device__ __forceinline__ Axis<T> make_axis(T c, T L) {
    Axis<T> a;
    const T half = L * T(0.5);
    if (c < half) {               // case A
        a.thr = c + half;         // rounding here only matters at |d| = L/2 (+-1 ulp)
        a.a1 = L;
        a.b1 = c;
        a.b0 = c;
    } else {                      // case B: "hit" means no wrap
        a.thr = c - half;         // exact (Sterbenz)
        a.a1 = T(0);
        a.b1 = c;
        a.b0 = c - L;             // exact (Sterbenz)
    }
    return a;
}

template <typename T>
__device__ __forceinline__ T min_image(T x, const Axis<T> &a) {
    const bool hit = x > a.thr;
    const T xs = hit ? x - a.a1 : x;
    return xs - (hit ? a.b1 : a.b0);
}

// ---------------------------------------------------------------------------
// Functor evaluation from t = r/delta (power basis, Horner).
//   returns u = U, du = U' * delta, h = U'' * delta^2 / 2.
// The interval index j = floor(t) is obtained with the round-down magic-number
// add (no F2I), clamped to m (the zero interval).
// tab_base: shared-memory byte address of table row 0, minus
// MAGIC_BITS * sizeof(Coef4) (so bits * sizeof(Coef4) + tab_base addresses j).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ld_shared_c4(uint32_t addr, float &a0, float &a1, float &a2, float &a3) {
    asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3) : "r"(addr));
}
__device__ __forceinline__ void ld_shared_c4(uint32_t addr, double &a0, double &a1, double &a2, double &a3) {
    asm("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(a0), "=d"(a1) : "r"(addr));
    asm("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(a2), "=d"(a3) : "r"(addr + 16));
}

template <typename T>
struct FunctorEval {
    T u, du, h;
};

// tab_base: shared-memory byte address of the functor's row 0; m_clamp = m
// (the functor's all-zero row).  j = min(bits(MAGIC + floor(t)) - MAGIC_BITS, m)
// is one VIADDMNMX (immediate -MAGIC_BITS) and the address one LEA; keeping the
// magic bias out of the base stops ptxas from re-adding it per term.
template <typename T>
__device__ __forceinline__ FunctorEval<T> functor_from_t(T t, uint32_t tab_base,
                                                         typename Traits<T>::U m_clamp) {
    using Tr = Traits<T>;
    const T tf = Tr::add_rd(t, Tr::MAGIC);                // MAGIC + floor(t), t >= 0
    typename Tr::U jb = Tr::bits(tf) - Tr::MAGIC_BITS;    // floor(t) (huge for t = BIG or NaN)
    jb = jb < m_clamp ? jb : m_clamp;                    // min(floor(t), m)
    const T f = t - (tf - Tr::MAGIC);
    T a0, a1, a2, a3;
    ld_shared_c4(tab_base + (uint32_t)jb * (uint32_t)sizeof(Coef4<T>), a0, a1, a2, a3);
    FunctorEval<T> e;
    const T p = fma(a3, f, a2);       // a2 + a3 f
    const T q = fma(p, f, a1);        // a1 + a2 f + a3 f^2
    e.u = fma(q, f, a0);              // U
    const T r1 = fma(a3, f, p);       // a2 + 2 a3 f
    e.du = fma(r1, f, q);             // a1 + 2 a2 f + 3 a3 f^2   = U' delta
    e.h = fma(a3, f, r1);             // a2 + 3 a3 f              = U'' delta^2 / 2
    return e;
}

// Functor argument in fp64 (the accept path compares single pair terms, not
// N-term sums; the fp32 eval path takes it for functors finer than m = 16).  With t = r/delta up to m, any relative error in r becomes
// an absolute error ~ m * eps in the interval fraction f and from there in
// U' and U'' -- the fp32 displacement's own rounding (2^-24) alone gives
// ~1e-5 of the functor scale at m = 64.  So the displacement is formed
// exactly in fp64 (the difference of two fp32 values and the +-L shift are
// exact), r and t follow in fp64, and only f is rounded to T for the fp32
// Horner; the fp32 displacement (one rounding) and 1/r feed the gradient
// factors, whose errors are relative and not amplified by t.
struct AxisD { double c, half, L; };

__device__ __forceinline__ AxisD make_axis_d(double c, double L) {
    AxisD a;
    a.c = c;
    a.half = 0.5 * L;
    a.L = L;
    return a;
}

__device__ __forceinline__ double min_image_d(double x, const AxisD &a) {
    double d = x - a.c;                        // exact for fp32 (or fp64 in range) inputs
    if (d > a.half) d -= a.L;
    else if (d <= -a.half) d += a.L;
    return d;
}

template <typename T>
__device__ __forceinline__ FunctorEval<T> functor_from_r2_d(double r2, double invd64, uint32_t base, int m, T &ir) {
    const double ird = rsqrt(r2);
    const double t = r2 * ird * invd64;
    const double fl = floor(t);
    const int j = fl < (double)m ? (int)fl : m;    // r >= r_cut (and dead partners) -> the zero row
    const T f = T(t - fl);
    ir = T(ird);
    T a0, a1, a2, a3;
    ld_shared_c4(base + (uint32_t)j * (uint32_t)sizeof(Coef4<T>), a0, a1, a2, a3);
    FunctorEval<T> e;
    const T pp = fma(a3, f, a2);
    const T q = fma(pp, f, a1);
    e.u = fma(q, f, a0);
    const T r1 = fma(a3, f, pp);
    e.du = fma(r1, f, q);
    e.h = fma(a3, f, r1);
    return e;
}

}  // namespace qj2
