// qmcj2.cu -- C-ABI entry points (declared and documented in include/qmcj2.h)
// and the small kernels of the J2 / distance-row hot path of arXiv 1708.02645
// and its NEXT rows, for sm_100a.
//
// Kernel map (one translation unit each where noted):
//   j2_eval_kernel           the hot path (j2_kernels.cuh, launch_*.cu): one CTA
//                            per (walker, trial, tile of 25 sub-tiles); SoA lanes
//                            streamed with 128-bit loads, per-term math in T,
//                            fp32 partials of 32 terms flushed to fp64, warp
//                            shuffle + smem CTA reduction, deterministic
//                            cross-CTA reduction by the last CTA of (walker, trial)
//   j2_eval_warp_kernel      short rows, many walkers: one warp per (walker, trial)
//   j1_thread_kernel         J1 over small ion sets: one thread per (walker, trial)
//   j2_accept_kernel         NEXT-2 accept-side update (accept.cuh, launch_accept.cu),
//                            optionally with the Metropolis test fused
//   j2_sweep_kernel          NEXT-2 whole sweeps (optionally with J1), walkers resident
//                            in smem, one barrier per move (sweep.cu)
//   spo_tma_kernel / spo_kernel   NEXT-4 Bspline-v/vgh + determinant ratio (spo.cu)
//   ratio_kernel, metropolis_kernel, vgl_kernel, minimg_kernel, check_kernel  (here)
//   gen_kernel, gen_spo_table kernels  synthetic inputs (gen.cu; harness)
#include "qmcj2.h"
#include "j2_device.cuh"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <cstdlib>
#include <algorithm>

#include "launch.cuh"
#include "accept.cuh"
#include "spo.cuh"
#include "sweep.cuh"

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

// Metropolis decision (Alg. 1 L9) for a J2-only trial function, symmetric
// proposal: accept iff u < rho^2.
__global__ void metropolis_kernel(int64_t W, const double *__restrict__ ratio, int64_t stride,
                                  const double *__restrict__ u, int32_t *__restrict__ accept) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= W) return;
    const double rho = ratio[w * stride + 1];
    accept[w] = u[w] < rho * rho ? 1 : 0;
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
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
    const T id = T(p.inv_delta);
    const FunctorEval<T> e = functor_from_t<T>(r[i] * id, base, (typename Tr::U)p.m);
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
inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// One trial per CTA (or warp): the P trials of a walker's tile run on P consecutive
// CTAs, so the tile is read from HBM once and from L2 by the other P - 1 (measured on
// B200 against 2 and 4 trials per thread, which need 124-127 registers and run at 2
// CTAs/SM: P = 2 1.84 vs 2.79 ms, P = 12 10.3 vs 20.8 ms on C3).
void ws_layout(int64_t W, int32_t P, int64_t N_local, qj2_dtype dtype,
               size_t *part_bytes, size_t *cnt_bytes) {
    const int64_t tpw = (N_local + ch_of(dtype) - 1) / ch_of(dtype);
    *part_bytes = tpw > 1 ? align256((size_t)W * P * tpw * NACC * sizeof(double)) : 0;
    *cnt_bytes = tpw > 1 ? align256((size_t)W * P * sizeof(unsigned)) : 0;
}

// Kernel launches live in launch_*.cu (one translation unit per dtype / trial
// batch, compiled in parallel); see launch.cuh.
// Shared tail of qj2_eval / qj2_eval_j1: workspace, counters, dispatch.
qj2_status launch_common(EvalParams &p, qj2_dtype dtype, void *workspace, size_t workspace_bytes,
                         cudaStream_t stream, bool check_dev) {
    if (((uintptr_t)p.R & 15) || (p.row_out && ((uintptr_t)p.row_out & 15)))
        return fail(QJ2_EINVAL, "source positions and row_out must be 16-byte aligned");
    size_t part_b, cnt_b;
    ws_layout(p.W, p.P, p.N_local, dtype, &part_b, &cnt_b);
    if (part_b + cnt_b > 0 && (!workspace || workspace_bytes < part_b + cnt_b))
        return fail(QJ2_EINVAL, "workspace too small: need %zu bytes", part_b + cnt_b);
    const int64_t tpw = (p.N_local + ch_of(dtype) - 1) / ch_of(dtype);
    const int64_t nblocks = p.W * p.P * tpw;
    if (nblocks > 0x7fffffffLL) return fail(QJ2_EINVAL, "problem too large for one launch (%lld CTAs)", (long long)nblocks);
    if (check_dev) { qj2_status st = check_device(); if (st) return st; }
    p.tiles_per_walker = tpw;
    p.partials = part_b ? static_cast<double *>(workspace) : nullptr;
    p.counters = cnt_b ? reinterpret_cast<unsigned *>(static_cast<char *>(workspace) + part_b) : nullptr;
    const bool row = p.row_out != nullptr;
    cudaError_t e;
    if (cnt_b) {   // completion counters start at zero every call (no caller-side init needed)
        e = cudaMemsetAsync(p.counters, 0, (size_t)p.W * p.P * sizeof(unsigned), stream);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counters)");
    }
    const bool j1 = p.mode == MODE_J1;
    if (dtype == QJ2_FP32) {
        e = j1 ? launch_f32_j1(p, nblocks, row, stream) : launch_f32_j2(p, nblocks, row, stream);
    } else {
        e = j1 ? launch_f64_j1(p, nblocks, row, stream) : launch_f64_j2(p, nblocks, row, stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "j2_eval_kernel launch");
    return QJ2_OK;
}

// The fused ratio relative to trial 0 (V_cur == NULL) needs trial 0 in the same
// CTA; for P > 1 it is a second (tiny) launch after the reduction.
qj2_status launch_with_ratio(EvalParams &p, qj2_dtype dtype, void *workspace, size_t workspace_bytes,
                             cudaStream_t stream, bool check_dev) {
    double *ratio_out = p.ratio_out;
    const bool after = ratio_out && !p.V_cur && p.P > 1;
    if (after) p.ratio_out = nullptr;
    qj2_status st = launch_common(p, dtype, workspace, workspace_bytes, stream, check_dev);
    if (st || !after) return st;
    const int64_t n = p.W * p.P;
    ratio_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(p.W, p.P, p.out, nullptr, ratio_out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "ratio_kernel launch");
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
    if (ratio_out) {
        if (i_offset != 0 || N_local != N_total)
            return fail(QJ2_EINVAL, "ratio_out needs an unsharded call; use qj2_ratio after reducing");
    }
    if (W == 0) return QJ2_OK;
    if (!R || !k || !r_trial || !out) return fail(QJ2_EINVAL, "R, k, r_trial and out must be non-NULL");

    EvalParams p;
    memset(&p, 0, sizeof p);
    p.W = W; p.N_total = N_total; p.N_up = N_up; p.i_offset = i_offset; p.N_local = N_local; p.Np = Np;
    p.P = P; p.m = fn->m;
    p.mode = MODE_J2;
    p.src_stride = 3 * Np;
    p.n_src_groups = 2;                       // spin halves [0, N_up), [N_up, N_total)
    p.grp_start[0] = 0; p.grp_start[1] = N_up; p.grp_start[2] = N_total;
    for (int g = 3; g <= MAXG; ++g) p.grp_start[g] = N_total;
    p.R = R; p.k = k; p.r_trial = r_trial; p.out = out; p.row_out = row_out;
    p.V_cur = V_cur; p.ratio_out = ratio_out;
    for (int d = 0; d < 3; ++d) p.L[d] = fn->L[d];
    p.inv_delta = (double)fn->m / fn->r_cut;
    p.inv_delta_f = (float)p.inv_delta;
    power_basis(fn->coef[0], fn->m, p.pcoef);                  // rows [0, m]: same spin
    power_basis(fn->coef[1], fn->m, p.pcoef + (fn->m + 1));    // rows [m+1, 2m+1]: opposite spin
    p.n_tab = 2 * (fn->m + 1);
    return launch_with_ratio(p, dtype, workspace, workspace_bytes, stream, check_dev);
}

qj2_status validate_j1_functor(const qj2_j1_functor *fn) {
    if (!fn) return fail(QJ2_EINVAL, "fn is NULL");
    if (fn->reserved != 0) return fail(QJ2_EINVAL, "fn->reserved must be 0");
    if (fn->n_species < 1 || fn->n_species > QJ2_MAX_SPECIES)
        return fail(QJ2_EINVAL, "n_species must be in [1, %d]", QJ2_MAX_SPECIES);
    for (int d = 0; d < 3; ++d)
        if (!(fn->L[d] > 0) || !std::isfinite(fn->L[d])) return fail(QJ2_EINVAL, "L[%d] must be finite and > 0", d);
    const double Lmin = std::fmin(fn->L[0], std::fmin(fn->L[1], fn->L[2]));
    for (int s = 0; s < fn->n_species; ++s) {
        if (!(fn->r_cut[s] > 0) || !(fn->r_cut[s] <= 0.5 * Lmin))
            return fail(QJ2_EINVAL, "r_cut[%d] must satisfy 0 < r_cut <= min(L)/2", s);
        if (fn->m[s] < 4 || fn->m[s] > QJ2_MAX_M) return fail(QJ2_EINVAL, "m[%d] must be in [4, %d]", s, QJ2_MAX_M);
        for (int j = 0; j < fn->m[s] + 3; ++j)
            if (!std::isfinite(fn->coef[s][j])) return fail(QJ2_EINVAL, "coef[%d][%d] not finite", s, j);
        for (int j = fn->m[s]; j < fn->m[s] + 3; ++j)
            if (fn->coef[s][j] != 0.0) return fail(QJ2_EINVAL, "coef[%d][%d] must be 0 (C2 cutoff)", s, j);
    }
    return QJ2_OK;
}

qj2_status eval_j1_impl(const qj2_j1_functor *fn, qj2_dtype dtype, int64_t W, const int64_t *species_start,
                        int64_t Np, const void *ions, int32_t P, const void *r_trial, double *out, void *row_out,
                        const double *V_cur, double *ratio_out, void *workspace, size_t workspace_bytes,
                        cudaStream_t stream) {
    qj2_status st = validate_j1_functor(fn);
    if (st) return st;
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype %d", (int)dtype);
    if (W < 0) return fail(QJ2_EINVAL, "W < 0");
    if (!species_start) return fail(QJ2_EINVAL, "species_start is NULL");
    if (species_start[0] != 0) return fail(QJ2_EINVAL, "species_start[0] must be 0");
    for (int s = 0; s < fn->n_species; ++s)
        if (species_start[s + 1] < species_start[s]) return fail(QJ2_EINVAL, "species_start must be nondecreasing");
    const int64_t n_ions = species_start[fn->n_species];
    if (n_ions < 1) return fail(QJ2_EINVAL, "need at least one ion");
    if (Np < n_ions || Np % vw_of(dtype) != 0)
        return fail(QJ2_EINVAL, "Np must be >= n_ions and a multiple of %d", vw_of(dtype));
    if (P < 1 || P > QJ2_MAX_P) return fail(QJ2_EINVAL, "P must be in [1, %d]", QJ2_MAX_P);
    if (W == 0) return QJ2_OK;
    if (!ions || !r_trial || !out) return fail(QJ2_EINVAL, "ions, r_trial and out must be non-NULL");

    EvalParams p;
    memset(&p, 0, sizeof p);
    p.W = W; p.N_total = n_ions; p.N_up = 0; p.i_offset = 0; p.N_local = n_ions; p.Np = Np;
    p.P = P; p.m = 0;
    p.mode = MODE_J1;
    p.src_stride = 0;                          // one ion set shared by all walkers
    p.n_src_groups = fn->n_species;
    int row = 0;
    for (int g = 0; g <= MAXG; ++g) p.grp_start[g] = g <= fn->n_species ? species_start[g] : n_ions;
    for (int s = 0; s < fn->n_species; ++s) {
        p.grp_tab[s] = row;
        p.grp_m[s] = fn->m[s];
        p.grp_invd[s] = (double)fn->m[s] / fn->r_cut[s];
        power_basis(fn->coef[s], fn->m[s], p.pcoef + row);
        row += fn->m[s] + 1;
    }
    p.n_tab = row;
    p.R = ions; p.k = nullptr; p.r_trial = r_trial; p.out = out; p.row_out = row_out;
    p.V_cur = V_cur; p.ratio_out = ratio_out;
    for (int d = 0; d < 3; ++d) p.L[d] = fn->L[d];
    return launch_with_ratio(p, dtype, workspace, workspace_bytes, stream, true);
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

qj2_status qj2_eval_j1(const qj2_j1_functor *fn, qj2_dtype dtype, int64_t W, const int64_t *species_start,
                       int64_t Np, const void *ions, int32_t P, const void *r_trial, double *out, void *row_out,
                       const double *V_cur, double *ratio_out, void *workspace, size_t workspace_bytes,
                       void *stream) {
    return eval_j1_impl(fn, dtype, W, species_start, Np, ions, P, r_trial, out, row_out, V_cur, ratio_out,
                        workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
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
// NEXT-2: accept-side update (include/qmcj2.h).
// ---------------------------------------------------------------------------
qj2_status qj2_accept_workspace_size(int64_t W, qj2_dtype dtype, size_t *bytes) {
    if (!bytes) return fail(QJ2_EINVAL, "bytes is NULL");
    if (W < 0) return fail(QJ2_EINVAL, "W < 0");
    if (dtype != QJ2_FP32 && dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad dtype");
    *bytes = align256((size_t)W * 3 * (dtype == QJ2_FP32 ? 4 : 8));
    return QJ2_OK;
}

qj2_status qj2_accept(const qj2_functor *fn, qj2_dtype dtype,
                      int64_t W, int64_t N_total, int64_t N_up,
                      int64_t i_offset, int64_t N_local, int64_t Np,
                      void *R, void *state, const int32_t *k,
                      const void *r_new, int64_t r_stride, const void *r_old,
                      const int32_t *accept, const double *out_new, int64_t out_stride,
                      void *workspace, size_t workspace_bytes, void *stream) {
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
    if (out_stride < 5) return fail(QJ2_EINVAL, "out_stride must be >= 5");
    if (r_stride < 3) return fail(QJ2_EINVAL, "r_stride must be >= 3");
    if (W == 0) return QJ2_OK;
    if (!R || !state || !k || !r_new || !accept || !out_new)
        return fail(QJ2_EINVAL, "R, state, k, r_new, accept and out_new must be non-NULL");
    if (((uintptr_t)R & 15) || ((uintptr_t)state & 15)) return fail(QJ2_EINVAL, "R and state must be 16-byte aligned");
    size_t need = 0;
    qj2_accept_workspace_size(W, dtype, &need);
    if (!r_old && (!workspace || workspace_bytes < need))
        return fail(QJ2_EINVAL, "workspace too small: need %zu bytes (or pass r_old)", need);
    const int64_t tile = dtype == QJ2_FP32 ? accept_tile<float>() : accept_tile<double>();
    const int64_t tpw = (N_local + tile - 1) / tile;
    if (W * tpw > 0x7fffffffLL) return fail(QJ2_EINVAL, "problem too large for one launch");
    st = check_device();
    if (st) return st;
    AcceptParams p;
    memset(&p, 0, sizeof p);
    p.W = W; p.N_total = N_total; p.N_up = N_up; p.i_offset = i_offset; p.N_local = N_local; p.Np = Np;
    p.tiles_per_walker = tpw;
    p.m = fn->m;
    p.inv_delta = (double)fn->m / fn->r_cut;
    p.R = R; p.state = state; p.k = k; p.r_new = r_new; p.r_stride = r_stride; p.r_old = r_old; p.r_old_stride = 3;
    p.accept = accept;
    p.out_new = out_new; p.out_stride = out_stride;
    for (int d = 0; d < 3; ++d) p.L[d] = fn->L[d];
    power_basis(fn->coef[0], fn->m, p.pcoef);
    power_basis(fn->coef[1], fn->m, p.pcoef + (fn->m + 1));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = dtype == QJ2_FP32 ? launch_accept_f32(p, workspace, s) : launch_accept_f64(p, workspace, s);
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "j2_accept_kernel launch");
}

qj2_status qj2_metropolis_accept(const qj2_functor *fn, qj2_dtype dtype,
                                 int64_t W, int64_t N_total, int64_t N_up,
                                 int64_t i_offset, int64_t N_local, int64_t Np,
                                 void *R, void *state, const int32_t *k,
                                 const void *r_new, const void *r_old, int64_t r_stride,
                                 const double *out_new, const double *v_ref, int64_t out_stride,
                                 int64_t v_ref_stride, const double *u, int32_t *accept, void *stream) {
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
    if (r_stride < 3 || out_stride < 5 || v_ref_stride < 1)
        return fail(QJ2_EINVAL, "need r_stride >= 3, out_stride >= 5, v_ref_stride >= 1");
    if (W == 0) return QJ2_OK;
    if (!R || !state || !k || !r_new || !r_old || !out_new || !v_ref || !u || !accept)
        return fail(QJ2_EINVAL, "R, state, k, r_new, r_old, out_new, v_ref, u and accept must be non-NULL");
    if (((uintptr_t)R & 15) || ((uintptr_t)state & 15)) return fail(QJ2_EINVAL, "R and state must be 16-byte aligned");
    const int64_t tile = dtype == QJ2_FP32 ? accept_tile<float>() : accept_tile<double>();
    const int64_t tpw = (N_local + tile - 1) / tile;
    if (W * tpw > 0x7fffffffLL) return fail(QJ2_EINVAL, "problem too large for one launch");
    st = check_device();
    if (st) return st;
    AcceptParams p;
    memset(&p, 0, sizeof p);
    p.W = W; p.N_total = N_total; p.N_up = N_up; p.i_offset = i_offset; p.N_local = N_local; p.Np = Np;
    p.tiles_per_walker = tpw;
    p.m = fn->m;
    p.inv_delta = (double)fn->m / fn->r_cut;
    p.R = R; p.state = state; p.k = k; p.r_new = r_new; p.r_stride = r_stride; p.r_old = r_old;
    p.r_old_stride = r_stride; p.accept = accept;
    p.out_new = out_new; p.out_stride = out_stride;
    p.u = u; p.v_ref = v_ref; p.v_ref_stride = v_ref_stride; p.acc_out = accept;
    for (int d = 0; d < 3; ++d) p.L[d] = fn->L[d];
    power_basis(fn->coef[0], fn->m, p.pcoef);
    power_basis(fn->coef[1], fn->m, p.pcoef + (fn->m + 1));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = dtype == QJ2_FP32 ? launch_accept_f32(p, nullptr, s) : launch_accept_f64(p, nullptr, s);
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "j2_accept_kernel launch");
}

// Shared validation and parameter set-up of qj2_sweep / qj2_state_init.
static qj2_status sweep_params(const qj2_functor *fn, int64_t W, int64_t N, int64_t N_up, int64_t Np,
                               const qj2_sweep_j1 *j1, SweepParams &p) {
    qj2_status st = validate_functor(fn);
    if (st) return st;
    if (fn->m > ACCEPT_FAST_MAX_M)
        return fail(QJ2_EINVAL, "the resident-walker kernels keep fp32 pair terms: m must be <= %d (use qj2_eval + "
                    "qj2_metropolis_accept per move for finer functors)", ACCEPT_FAST_MAX_M);
    if (W < 0) return fail(QJ2_EINVAL, "W must be >= 0");
    if (N < 2 || N > SW_MAXN) return fail(QJ2_EINVAL, "need 2 <= N <= %d (walker resident in shared memory)", SW_MAXN);
    if (N_up < 0 || N_up > N) return fail(QJ2_ERANGE, "N_up out of [0, N]");
    if (Np < N) return fail(QJ2_EINVAL, "Np must be >= N");
    if (W > 0x7fffffffLL) return fail(QJ2_EINVAL, "W too large for one launch");
    int64_t n_ions = 0;
    if (j1) {
        st = validate_j1_functor(j1->fn);
        if (st) return st;
        for (int d = 0; d < 3; ++d)
            if (j1->fn->L[d] != fn->L[d]) return fail(QJ2_EINVAL, "the J1 and J2 functors must share the cell");
        for (int sp = 0; sp < j1->fn->n_species; ++sp)
            if (j1->fn->m[sp] > ACCEPT_FAST_MAX_M)
                return fail(QJ2_EINVAL, "the resident-walker kernels keep fp32 J1 terms: m[%d] must be <= %d", sp,
                            ACCEPT_FAST_MAX_M);
        if (!j1->species_start || j1->species_start[0] != 0)
            return fail(QJ2_EINVAL, "j1->species_start must be non-NULL with species_start[0] == 0");
        for (int sp = 0; sp < j1->fn->n_species; ++sp)
            if (j1->species_start[sp + 1] < j1->species_start[sp])
                return fail(QJ2_EINVAL, "j1->species_start must be nondecreasing");
        n_ions = j1->species_start[j1->fn->n_species];
        if (n_ions < 1 || n_ions > SW_MAX_IONS) return fail(QJ2_EINVAL, "the resident-walker kernels take 1..%d ions",
                                                            SW_MAX_IONS);
        if (j1->Np_ion < n_ions) return fail(QJ2_EINVAL, "j1->Np_ion must be >= the number of ions");
    }
    memset(&p, 0, sizeof p);
    p.W = (int32_t)W; p.N = (int32_t)N; p.N_up = (int32_t)N_up; p.Np = Np;
    p.m = fn->m;
    p.inv_delta = (double)fn->m / fn->r_cut;
    p.invd = (float)p.inv_delta;
    for (int d = 0; d < 3; ++d) p.L[d] = (float)fn->L[d];
    power_basis(fn->coef[0], fn->m, p.pcoef);
    power_basis(fn->coef[1], fn->m, p.pcoef + (fn->m + 1));
    if (j1) {
        p.n_ions = (int32_t)n_ions;
        p.n_species = j1->fn->n_species;
        int row = 0;
        for (int sp = 0; sp <= QJ2_MAX_SPECIES; ++sp)
            p.sp_start[sp] = (int32_t)(sp <= p.n_species ? j1->species_start[sp] : n_ions);
        for (int sp = 0; sp < p.n_species; ++sp) {
            p.sp_tab[sp] = row;
            p.sp_m[sp] = j1->fn->m[sp];
            p.sp_invd[sp] = (float)((double)j1->fn->m[sp] / j1->fn->r_cut[sp]);
            power_basis(j1->fn->coef[sp], j1->fn->m[sp], p.pcoef1 + row);
            row += j1->fn->m[sp] + 1;
        }
        p.n_rows1 = row;
        p.ions = j1->ions; p.Np_ion = j1->Np_ion; p.state_j1 = j1->state;
    }
    return QJ2_OK;
}

qj2_status qj2_sweep(const qj2_functor *fn, int64_t W, int64_t N, int64_t N_up, int64_t Np,
                     float *R, float *state, int64_t S, const int32_t *ks, const float *delta,
                     const double *u, int32_t *accept, double *dj, const qj2_sweep_j1 *j1,
                     void *stream) {
    SweepParams p;
    qj2_status st = sweep_params(fn, W, N, N_up, Np, j1, p);
    if (st) return st;
    if (S < 0 || S > 0x7fffffffLL) return fail(QJ2_EINVAL, "S must be in [0, 2^31)");
    if (W == 0 || S == 0) return QJ2_OK;
    if (!R || !state || !ks || !delta || !u || !accept)
        return fail(QJ2_EINVAL, "R, state, ks, delta, u and accept must be non-NULL");
    if (j1 && (!j1->ions || !j1->state)) return fail(QJ2_EINVAL, "j1->ions and j1->state must be non-NULL");
    st = check_device();
    if (st) return st;
    p.S = S;
    p.R = R; p.state = state; p.ks = ks; p.delta = delta; p.u = u; p.acc = accept; p.dj = dj;
    cudaError_t e = launch_sweep(p, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "j2_sweep_kernel launch");
}

qj2_status qj2_state_init(const qj2_functor *fn, int64_t W, int64_t N, int64_t N_up, int64_t Np,
                          const float *R, float *state, const qj2_sweep_j1 *j1, void *stream) {
    SweepParams p;
    qj2_status st = sweep_params(fn, W, N, N_up, Np, j1, p);
    if (st) return st;
    if (W == 0) return QJ2_OK;
    if (!R || !state) return fail(QJ2_EINVAL, "R and state must be non-NULL");
    if (j1 && (!j1->ions || !j1->state)) return fail(QJ2_EINVAL, "j1->ions and j1->state must be non-NULL");
    st = check_device();
    if (st) return st;
    p.R = const_cast<float *>(R); p.state = state;
    cudaError_t e = launch_state_init(p, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "state_init_kernel launch");
}

qj2_status qj2_metropolis(int64_t W, const double *ratio, int64_t ratio_stride,
                          const double *u, int32_t *accept, void *stream) {
    if (W < 0) return fail(QJ2_EINVAL, "W < 0");
    if (ratio_stride < 2) return fail(QJ2_EINVAL, "ratio_stride must be >= 2");
    if (W == 0) return QJ2_OK;
    if (!ratio || !u || !accept) return fail(QJ2_EINVAL, "ratio, u and accept must be non-NULL");
    qj2_status st = check_device();
    if (st) return st;
    metropolis_kernel<<<(unsigned)((W + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        W, ratio, ratio_stride, u, accept);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "metropolis_kernel launch");
}

// ---------------------------------------------------------------------------
// NEXT-4: tricubic B-spline SPOs + determinant ratio (include/qmcj2.h).
// ---------------------------------------------------------------------------
qj2_status qj2_spo_eval(const qj2_spo_table *tab, int32_t what, qj2_dtype pos_dtype, int64_t W,
                        const void *pos, int64_t pos_stride,
                        const float *Ainv, int64_t ainv_stride, int64_t ainv_ld, const int32_t *krow,
                        int64_t points_per_walker, double *out, float *spo_out, void *stream) {
    if (!tab) return fail(QJ2_EINVAL, "tab is NULL");
    if (points_per_walker < 1) return fail(QJ2_EINVAL, "points_per_walker must be >= 1");
    const bool force_gather = (what & QJ2_SPO_GATHER) != 0;
    what &= ~QJ2_SPO_GATHER;
    if (what != QJ2_SPO_V && what != QJ2_SPO_VGH)
        return fail(QJ2_EINVAL, "what must be QJ2_SPO_V or QJ2_SPO_VGH (optionally | QJ2_SPO_GATHER)");
    if (pos_dtype != QJ2_FP32 && pos_dtype != QJ2_FP64) return fail(QJ2_EINVAL, "bad pos_dtype");
    for (int d = 0; d < 3; ++d)
        if (!(tab->L[d] > 0) || !std::isfinite(tab->L[d])) return fail(QJ2_EINVAL, "L[%d] must be finite and > 0", d);
    if (tab->nx < 4 || tab->ny < 4 || tab->nz < 4) return fail(QJ2_EINVAL, "grid dimensions must be >= 4");
    if (tab->n_orb < 1 || tab->ld < tab->n_orb || tab->ld % 4 != 0)
        return fail(QJ2_EINVAL, "need 1 <= n_orb <= ld and ld %% 4 == 0");
    if (tab->nx * tab->ny * tab->nz * tab->ld >= (1ll << 31)) return fail(QJ2_EINVAL, "table too large (>= 2^31 floats)");
    if (W < 0 || pos_stride < 3) return fail(QJ2_EINVAL, "need W >= 0 and pos_stride >= 3");
    if (Ainv && (ainv_stride < 0 || (krow && ainv_ld < tab->n_orb)))
        return fail(QJ2_EINVAL, "bad Ainv strides");
    if (W == 0) return QJ2_OK;
    if (!tab->coef || !pos) return fail(QJ2_EINVAL, "coef and pos must be non-NULL");
    if (((uintptr_t)tab->coef & 15) || (spo_out && ((uintptr_t)spo_out & 15)))
        return fail(QJ2_EINVAL, "coef and spo_out must be 16-byte aligned");
    qj2_status st = check_device();
    if (st) return st;
    const bool vgh = what == QJ2_SPO_VGH;
    const int nv = vgh ? 2 : 4;                   // orbitals per thread (spo.cuh)
    SpoParams p;
    memset(&p, 0, sizeof p);
    p.W = W; p.nx = tab->nx; p.ny = tab->ny; p.nz = tab->nz; p.n_orb = tab->n_orb; p.ld = tab->ld;
    p.nvec = tab->ld / nv;
    p.coef = tab->coef;
    for (int d = 0; d < 3; ++d) p.L[d] = tab->L[d];
    p.pos_f64 = pos_dtype == QJ2_FP64; p.pos = pos; p.pos_stride = pos_stride;
    p.Ainv = Ainv; p.ainv_stride = ainv_stride; p.ainv_ld = ainv_ld; p.krow = krow; p.ppw = points_per_walker;
    p.out = out; p.spo_out = spo_out;
    const int64_t lanes = ((p.nvec + 31) / 32) * 32;
    p.tpw = (int32_t)(lanes < 256 ? lanes : 256);
    p.wpc = 256 / p.tpw;
    cudaError_t e = launch_spo(p, vgh, force_gather, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QJ2_OK : cuda_fail(e, "spo_kernel launch");
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
