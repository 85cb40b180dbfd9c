/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the hot path of
 * Mathuriya et al., "Embracing a new era of highly efficient and productive
 * quantum Monte Carlo simulations" (SC'17, arXiv 1708.02645): the on-the-fly
 * electron-electron distance row and the two-body Jastrow (J2) value,
 * gradient and Laplacian of a particle-by-particle move; and, for the NEXT
 * rows, the one-body Jastrow over the electron-ion row, the per-electron 5N
 * J2 state with its accept-side update, and the tricubic B-spline orbitals
 * with the determinant ratio.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_1708_02645_b200/) shares no code with it and never calls it.
 *
 * Citations: PAPER:n is a line of /root/reference/PAPER.md, SPEC:n a line of
 * /root/reference/SPEC.md (a spec written from the paper; used for
 * interfaces and test ideas only).  Readings of the paper where it is silent
 * are numbered R1..R23 as in DESIGN.md.
 *
 * Everything is scalar fp64, IEEE round-to-nearest, no SIMD pragmas, sums are
 * Neumaier-compensated.  Positions given in fp32 are promoted to fp64 exactly
 * by the caller.
 *
 * Parity status: every function here is pinned -- tests/test_oracle_pins.py
 * (J2/J1 eval, functor, minimum image: closed forms, brute force, finite
 * differences, library B-spline, worked examples), tests/test_oracle_accept.py
 * (5N state and accept: pair-sum brute force, finite differences, state from
 * scratch after many accepted moves), tests/test_oracle_spo.py (tricubic SPOs
 * and determinant ratio: scipy separable splines, Marsden, LU determinants),
 * tests/test_inputs.py (the generator twins, bitwise); and
 * tests/test_oracle_mutations.py shows 18 plausible one-line mistakes each
 * fail a pin.  Nothing is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------------ */
/* Compensated (Neumaier) summation.                                         */
/* ------------------------------------------------------------------------ */
typedef struct { double s, c; } nsum;

static void nsum_add(nsum *a, double x)
{
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else                       a->c += (x - t) + a->s;
    a->s = t;
}
static double nsum_get(const nsum *a) { return a->s + a->c; }

/* ------------------------------------------------------------------------ */
/* Minimum-image displacement b - a on an orthorhombic, fully periodic cell.  */
/* SPEC:113-121 (min_image_disp: "displacement = b - a wrapped to nearest     */
/* image"), SPEC:138 ("disp_d in (-L_d/2, L_d/2]").  Reading R7.              */
/* The paper's row is d(k,i) = |r_i - r_k|, dr(k,i) = r_i - r_k (PAPER:1300-  */
/* 1301), so the oracle is called with a = trial position, b = source i.      */
/* ------------------------------------------------------------------------ */
void orc_min_image(const double L[3], const double a[3], const double b[3],
                   double d[3], double *dist)
{
    double s = 0.0;
    for (int c = 0; c < 3; ++c) {
        double t = b[c] - a[c];
        if (t > 0.5 * L[c])        t -= L[c];
        else if (t <= -0.5 * L[c]) t += L[c];
        d[c] = t;
        s += t * t;
    }
    *dist = sqrt(s);
}

/* ------------------------------------------------------------------------ */
/* Uniform cubic B-spline radial functor U(r), U'(r), U''(r).                 */
/* PAPER:817-819 ("The one-dimensional cubic B-spline is extensively used"),  */
/* SPEC:256-258 (CubicBspline1D: r_cut, m intervals, delta = r_cut/m, m+3     */
/* coefficients, zero for r >= r_cut), SPEC:279-287 (functor_eval_vgl).       */
/* Readings R3 (index/basis convention) and R5 (contribute iff r < r_cut).    */
/*   t = r/delta, j = min(floor(t), m-1), f = t - j,                          */
/*   U = sum_a c[j+a] B_a(f),  U' = sum c[j+a] B_a'(f)/delta,                 */
/*   U'' = sum c[j+a] B_a''(f)/delta^2.                                       */
/* The tail c[m..m+2] is NOT forced to zero here (closed-form pins use        */
/* polynomial coefficient sequences); the cutoff test is explicit.            */
/* ------------------------------------------------------------------------ */
void orc_bspline(const double *c, int m, double r_cut, double r, double out[3])
{
    if (!(r < r_cut)) { out[0] = out[1] = out[2] = 0.0; return; }
    double delta = r_cut / (double)m;
    double t = r / delta;
    int j = (int)floor(t);
    if (j > m - 1) j = m - 1;
    if (j < 0) j = 0;
    double f = t - (double)j;
    double g = 1.0 - f;

    double B0 = g * g * g / 6.0;
    double B1 = (3.0 * f * f * f - 6.0 * f * f + 4.0) / 6.0;
    double B2 = (-3.0 * f * f * f + 3.0 * f * f + 3.0 * f + 1.0) / 6.0;
    double B3 = f * f * f / 6.0;

    double D0 = -0.5 * g * g;
    double D1 = 0.5 * (3.0 * f * f - 4.0 * f);
    double D2 = 0.5 * (-3.0 * f * f + 2.0 * f + 1.0);
    double D3 = 0.5 * f * f;

    double S0 = 1.0 - f;
    double S1 = 3.0 * f - 2.0;
    double S2 = 1.0 - 3.0 * f;
    double S3 = f;

    out[0] = c[j] * B0 + c[j + 1] * B1 + c[j + 2] * B2 + c[j + 3] * B3;
    out[1] = (c[j] * D0 + c[j + 1] * D1 + c[j + 2] * D2 + c[j + 3] * D3) / delta;
    out[2] = (c[j] * S0 + c[j + 1] * S1 + c[j + 2] * S2 + c[j + 3] * S3) / (delta * delta);
}

/* Spin channel of the pair (i, k): 0 = same spin, 1 = opposite spin.
 * PAPER:800-801 (N^u = N^d = N/2), SPEC:431 (indices [0,N/2) up, like/unlike
 * channels).  Reading R6. */
static int spin_channel(int64_t i, int64_t k, int64_t n_up)
{
    return ((i < n_up) == (k < n_up)) ? 0 : 1;
}

/* ------------------------------------------------------------------------ */
/* The hot path: for each walker w and trial p, with r = r_trial[w][p],       */
/*   V  = sum_{i != k, i in slice}  U_s(|d_i|)                                */
/*   G  = -sum U_s'(|d_i|) d_i / |d_i|                                        */
/*   L  = sum [U_s''(|d_i|) + 2 U_s'(|d_i|)/|d_i|]                            */
/* with d_i = minimg(r_i - r).  This is U^2_k of PAPER:1382 ("Two-body        */
/* Jastrow takes the similar form as Delta J2 = U^2_k(R') - U^2_k(R)"),       */
/* i.e. one term of Eq. (5), and its gradient and Laplacian   */
/* with respect to the moved electron (Alg. 1 L8).  Readings R1,   */
/* R2, R8, R11, R12.  abs_out receives the absolute-term sums                 */
/* (sum|U|, sum|U' d_c/r|, sum|U''| + 2|U'|/r) used by the parity tolerance.  */
/*                                                                            */
/* Sharding: the slice holds global sources [i_offset, i_offset + N_local);   */
/* R is [W][3][Np] over the slice.  Spin and self-exclusion use global        */
/* indices.                                                                   */
/*                                                                            */
/* row_out (optional) is Fig. 6's temporary row v:          */
/* [W][P][4][Np] = (r, dx, dy, dz); slot k and padding are left untouched.    */
/*                                                                            */
/* Returns 0, or 1 + (flat index w*P+p) of the first coincident pair          */
/* (r == 0 inside the cutoff: reading R9, undefined, the oracle refuses).     */
/* ------------------------------------------------------------------------ */
typedef struct {
    const double *L; double r_cut; int m; const double *coef; /* [2][m+3] */
    int64_t W, N_total, N_up, i_offset, N_local, Np;
    const double *R; const int32_t *k; int32_t P; const double *r_trial;
    const float *Rf; const float *r_trial_f;   /* fp32 inputs, promoted exactly (or NULL) */
    double *out; double *abs_out; double *row_out;
    int64_t w_begin, w_end;
    int64_t status;
} orc_job;

static int64_t eval_walkers(orc_job *J)
{
    const int mc = J->m + 3;
    for (int64_t w = J->w_begin; w < J->w_end; ++w) {
        const double *Rw = J->R ? J->R + w * 3 * J->Np : NULL;
        int64_t kw = J->k[w];
        for (int32_t p = 0; p < J->P; ++p) {
            double rt[3];
            for (int c = 0; c < 3; ++c)
                rt[c] = J->r_trial_f ? (double)J->r_trial_f[(w * J->P + p) * 3 + c]
                                     : J->r_trial[(w * J->P + p) * 3 + c];
            nsum V = {0, 0}, G[3] = {{0, 0}, {0, 0}, {0, 0}}, Lp = {0, 0};
            nsum AV = {0, 0}, AG[3] = {{0, 0}, {0, 0}, {0, 0}}, AL = {0, 0};
            double *row = J->row_out ? J->row_out + ((w * J->P + p) * 4) * J->Np : NULL;
            for (int64_t il = 0; il < J->N_local; ++il) {
                int64_t i = J->i_offset + il;          /* global index */
                if (i == kw) continue;                 /* i != k, Eq. (5) */
                double src[3];
                for (int c = 0; c < 3; ++c)
                    src[c] = J->Rf ? (double)J->Rf[(w * 3 + c) * J->Np + il] : Rw[c * J->Np + il];
                double d[3], rho;
                orc_min_image(J->L, rt, src, d, &rho);
                if (row) {
                    row[il] = rho;
                    row[J->Np + il] = d[0];
                    row[2 * J->Np + il] = d[1];
                    row[3 * J->Np + il] = d[2];
                }
                if (!(rho < J->r_cut)) continue;       /* finite cutoff */
                if (rho == 0.0) return 1 + w * J->P + p;
                int s = spin_channel(i, kw, J->N_up);
                double u[3];
                orc_bspline(J->coef + s * mc, J->m, J->r_cut, rho, u);
                nsum_add(&V, u[0]);
                nsum_add(&AV, fabs(u[0]));
                for (int c = 0; c < 3; ++c) {
                    double g = u[1] * d[c] / rho;
                    nsum_add(&G[c], -g);
                    nsum_add(&AG[c], fabs(g));
                }
                nsum_add(&Lp, u[2] + 2.0 * u[1] / rho);
                nsum_add(&AL, fabs(u[2]) + 2.0 * fabs(u[1]) / rho);
            }
            double *o = J->out + (w * J->P + p) * 5;
            o[0] = nsum_get(&V);
            o[1] = nsum_get(&G[0]); o[2] = nsum_get(&G[1]); o[3] = nsum_get(&G[2]);
            o[4] = nsum_get(&Lp);
            if (J->abs_out) {
                double *a = J->abs_out + (w * J->P + p) * 5;
                a[0] = nsum_get(&AV);
                a[1] = nsum_get(&AG[0]); a[2] = nsum_get(&AG[1]); a[3] = nsum_get(&AG[2]);
                a[4] = nsum_get(&AL);
            }
        }
    }
    return 0;
}

static void *eval_thread(void *arg)
{
    orc_job *J = (orc_job *)arg;
    J->status = eval_walkers(J);
    return NULL;
}

static int64_t run_eval(orc_job proto, int nthreads)
{
    int64_t W = proto.W;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > W) nthreads = (int)(W > 0 ? W : 1);
    orc_job *jobs = (orc_job *)calloc((size_t)nthreads, sizeof(orc_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t per = (W + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        orc_job J = proto;
        J.w_begin = t * per < W ? t * per : W;
        J.w_end = (t + 1) * per < W ? (t + 1) * per : W;
        J.status = 0;
        jobs[t] = J;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, eval_thread, &jobs[t]);
    eval_thread(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    int64_t st = 0;
    for (int t = 0; t < nthreads && !st; ++t) st = jobs[t].status;
    free(jobs); free(th);
    return st;
}

int64_t orc_eval(const double L[3], double r_cut, int m, const double *coef,
                 int64_t W, int64_t N_total, int64_t N_up,
                 int64_t i_offset, int64_t N_local, int64_t Np,
                 const double *R, const int32_t *k, int32_t P, const double *r_trial,
                 double *out, double *abs_out, double *row_out, int nthreads)
{
    orc_job J = { L, r_cut, m, coef, W, N_total, N_up, i_offset, N_local, Np,
                  R, k, P, r_trial, NULL, NULL, out, abs_out, row_out, 0, 0, 0 };
    return run_eval(J, nthreads);
}

/* Same computation on fp32 inputs (each coordinate promoted exactly to fp64). */
int64_t orc_eval_f32(const double L[3], double r_cut, int m, const double *coef,
                     int64_t W, int64_t N_total, int64_t N_up,
                     int64_t i_offset, int64_t N_local, int64_t Np,
                     const float *R, const int32_t *k, int32_t P, const float *r_trial,
                     double *out, double *abs_out, double *row_out, int nthreads)
{
    orc_job J = { L, r_cut, m, coef, W, N_total, N_up, i_offset, N_local, Np,
                  NULL, k, P, NULL, R, r_trial, out, abs_out, row_out, 0, 0, 0 };
    return run_eval(J, nthreads);
}

/* ------------------------------------------------------------------------ */
/* Brute-force two-body Jastrow of one configuration, Eq. (3) second term     */
/* under reading R1: J2 = sum_{i<j} U_s(|r_i - r_j|) over     */
/* unordered pairs, so that Delta J2 = J2(R') - J2(R) reproduces Eq. (5).     */
/* O(N^2); used only by the pins on tiny N.                                   */
/* ------------------------------------------------------------------------ */
double orc_j2_total(const double L[3], double r_cut, int m, const double *coef,
                    int64_t N, int64_t N_up, int64_t Np, const double *R)
{
    const int mc = m + 3;
    nsum J = {0, 0};
    for (int64_t i = 0; i < N; ++i)
        for (int64_t j = i + 1; j < N; ++j) {
            double a[3] = { R[i], R[Np + i], R[2 * Np + i] };
            double b[3] = { R[j], R[Np + j], R[2 * Np + j] };
            double d[3], rho, u[3];
            orc_min_image(L, a, b, d, &rho);
            orc_bspline(coef + spin_channel(i, j, N_up) * mc, m, r_cut, rho, u);
            nsum_add(&J, u[0]);
        }
    return nsum_get(&J);
}

/* Batched functor evaluation (SPEC:279 functor_eval_vgl) for the pins. */
void orc_bspline_batch(const double *c, int m, double r_cut, int64_t n,
                       const double *r, double *out /* [n][3] */)
{
    for (int64_t i = 0; i < n; ++i) orc_bspline(c, m, r_cut, r[i], out + 3 * i);
}

/* Batched minimum image for the pins: out[n][4] = (dist, d). */
void orc_min_image_batch(const double L[3], int64_t n, const double *a,
                         const double *b, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        double d[3], rho;
        orc_min_image(L, a + 3 * i, b + 3 * i, d, &rho);
        out[4 * i] = rho; out[4 * i + 1] = d[0]; out[4 * i + 2] = d[1]; out[4 * i + 3] = d[2];
    }
}

/* ------------------------------------------------------------------------ */
/* Host twin of the seeded input generator (qmcgen.positions), written       */
/* independently in plain C so the oracle side can draw large samples        */
/* quickly.  Not part of the method.  Pinned bitwise against qmcgen by       */
/* tests/test_inputs.py.                                                      */
/* ------------------------------------------------------------------------ */
static uint64_t orc_mix64(uint64_t z)
{
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

typedef struct { uint64_t key; int64_t w0, w1, N, Np; double L; int f32; void *R; int64_t wbase; } gen_job;

static void *gen_thread(void *arg)
{
    gen_job *J = (gen_job *)arg;
    for (int64_t a = J->w0; a < J->w1; ++a)
        for (int d = 0; d < 3; ++d)
            for (int64_t i = 0; i < J->Np; ++i) {
                size_t o = ((size_t)a * 3 + (size_t)d) * (size_t)J->Np + (size_t)i;
                if (i >= J->N) {
                    if (J->f32) ((float *)J->R)[o] = 0.0f; else ((double *)J->R)[o] = 0.0;
                    continue;
                }
                uint64_t ctr = ((uint64_t)((J->wbase + a) * 3 + d) << 32) | (uint64_t)i;
                uint64_t h = orc_mix64(J->key ^ ctr);
                if (J->f32) {
                    float Lf = (float)J->L;
                    float u = (float)(uint32_t)(h >> 40) * 5.9604644775390625e-08f;
                    float x = Lf * u;
                    if (x >= Lf) x = nextafterf(Lf, 0.0f);
                    ((float *)J->R)[o] = x;
                } else {
                    double u = (double)(h >> 11) * 1.1102230246251565e-16;
                    double x = J->L * u;
                    if (x >= J->L) x = nextafter(J->L, 0.0);
                    ((double *)J->R)[o] = x;
                }
            }
    return NULL;
}

/* R[n_walkers][3][Np] for global walker ids wbase .. wbase+n_walkers-1. */
void orc_gen_positions(uint64_t seed, int64_t wbase, int64_t n_walkers, int64_t N, int64_t Np,
                       double L, int f32, void *R, int nthreads)
{
    uint64_t key = orc_mix64(seed * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n_walkers) nthreads = (int)(n_walkers > 0 ? n_walkers : 1);
    gen_job *jobs = (gen_job *)calloc((size_t)nthreads, sizeof(gen_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t per = (n_walkers + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        int64_t a = t * per, b = (t + 1) * per;
        if (a > n_walkers) a = n_walkers;
        if (b > n_walkers) b = n_walkers;
        gen_job J = { key, a, b, N, Np, L, f32, R, wbase };
        jobs[t] = J;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, gen_thread, &jobs[t]);
    gen_thread(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs); free(th);
}

/* ------------------------------------------------------------------------ */
/* NEXT-1: one-body Jastrow over the electron-ion (AB) row.                   */
/* "Delta J1 = U^1_k(R') - U^1_k(R), U^1_k = sum_I^{N_ion}   */
/* U_I(|r_I - r_k|)"; Eq. (3) first term; ions fixed and      */
/* shared by all walkers; per-species functors U_I          */
/* (Fig. 3 caption).  Ions are given sorted by   */
/* species: species s owns ions [sp_start[s], sp_start[s+1]).  Species s has  */
/* its own cutoff r_cut[s], m[s] intervals and m[s]+3 coefficients at         */
/* coef + s*coef_stride.  For each walker w and trial p, r = r_trial[w][p]:   */
/*   V = sum_I U_s(I)(|d_I|), G = -sum U' d/|d|, L = sum U'' + 2U'/|d|,       */
/*   d_I = minimg(r_I - r)  (no self term: electrons and ions differ).        */
/* Returns 0 or 1 + (w*P+p) if an ion coincides with the trial position      */
/* inside its cutoff (undefined, refused).                                   */
/* ------------------------------------------------------------------------ */
int64_t orc_eval_j1(const double L[3], int n_species, const int64_t *sp_start,
                    const double *r_cut, const int *m, const double *coef, int coef_stride,
                    int64_t W, int64_t n_ions, int64_t Np, const double *ions /* [3][Np] */,
                    int32_t P, const double *r_trial, double *out, double *abs_out)
{
    (void)n_ions;
    for (int64_t w = 0; w < W; ++w)
        for (int32_t p = 0; p < P; ++p) {
            const double *rt = r_trial + (w * P + p) * 3;
            nsum V = {0, 0}, G[3] = {{0, 0}, {0, 0}, {0, 0}}, Lp = {0, 0};
            nsum AV = {0, 0}, AG[3] = {{0, 0}, {0, 0}, {0, 0}}, AL = {0, 0};
            for (int s = 0; s < n_species; ++s)
                for (int64_t I = sp_start[s]; I < sp_start[s + 1]; ++I) {
                    double src[3] = { ions[I], ions[Np + I], ions[2 * Np + I] };
                    double d[3], rho, u[3];
                    orc_min_image(L, rt, src, d, &rho);
                    if (!(rho < r_cut[s])) continue;
                    if (rho == 0.0) return 1 + w * P + p;
                    orc_bspline(coef + s * coef_stride, m[s], r_cut[s], rho, u);
                    nsum_add(&V, u[0]);
                    nsum_add(&AV, fabs(u[0]));
                    for (int c = 0; c < 3; ++c) {
                        double g = u[1] * d[c] / rho;
                        nsum_add(&G[c], -g);
                        nsum_add(&AG[c], fabs(g));
                    }
                    nsum_add(&Lp, u[2] + 2.0 * u[1] / rho);
                    nsum_add(&AL, fabs(u[2]) + 2.0 * fabs(u[1]) / rho);
                }
            double *o = out + (w * P + p) * 5;
            o[0] = nsum_get(&V);
            o[1] = nsum_get(&G[0]); o[2] = nsum_get(&G[1]); o[3] = nsum_get(&G[2]);
            o[4] = nsum_get(&Lp);
            if (abs_out) {
                double *a = abs_out + (w * P + p) * 5;
                a[0] = nsum_get(&AV);
                a[1] = nsum_get(&AG[0]); a[2] = nsum_get(&AG[1]); a[3] = nsum_get(&AG[2]);
                a[4] = nsum_get(&AL);
            }
        }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT-2: the per-electron J2 state ("5N") and the accept-side update.       */
/*                                                                            */
/* State of electron e ("we can afford to eliminate the      */
/* intermediate data all together and keep the memory use of J2 at 5N"; the   */
/* values, gradients (D=3) and Laplacians of PAPER:1384-1386 summed over the  */
/* partner index):                                                            */
/*   V_e = sum_{j != e} U_s(r_ej)                                             */
/*   G_e = grad_e J2 = sum_{j != e} U_s'(r_ej) (r_e - r_j)/r_ej               */
/*   L_e = lap_e J2  = sum_{j != e} U_s''(r_ej) + 2 U_s'(r_ej)/r_ej           */
/* with r_e - r_j the minimum-image displacement (reading R7) and s the spin  */
/* channel of the pair (R6).  Stored SoA as state[5][Np] per walker (the      */
/* Rsoa layout).  Since U_s(r) depends on the pair only,     */
/* J2 = (1/2) sum_e V_e (reading R1) and G_e, L_e are the exact gradient and  */
/* Laplacian of J2 with respect to r_e.                                       */
/*                                                                            */
/* orc_j2_state: the state of one configuration from scratch, a direct        */
/* O(N^2) loop (the state "periodically computed from scratch"). */
/* abs_state (optional) receives the absolute-term sums.                      */
/* Returns 0, or 1 + e for the first electron with a coincident partner.      */
/* ------------------------------------------------------------------------ */
static int pair_terms(const double L[3], double r_cut, int m, const double *cs,
                      const double re[3], const double rj[3], double t[5], double a[5])
{
    /* t = (U, U' dx/r, U' dy/r, U' dz/r, U'' + 2U'/r) with d = re - rj,
     * a = their absolute values (|U''| + 2|U'|/r for the last). */
    double d[3], rho, u[3];
    orc_min_image(L, rj, re, d, &rho);          /* d = minimg(re - rj) */
    for (int c = 0; c < 5; ++c) t[c] = a[c] = 0.0;
    if (!(rho < r_cut)) return 0;
    if (rho == 0.0) return 1;
    orc_bspline(cs, m, r_cut, rho, u);
    t[0] = u[0];
    for (int c = 0; c < 3; ++c) t[1 + c] = u[1] * d[c] / rho;
    t[4] = u[2] + 2.0 * u[1] / rho;
    a[0] = fabs(u[0]);
    for (int c = 0; c < 3; ++c) a[1 + c] = fabs(t[1 + c]);
    a[4] = fabs(u[2]) + 2.0 * fabs(u[1]) / rho;
    return 0;
}

int64_t orc_j2_state(const double L[3], double r_cut, int m, const double *coef,
                     int64_t N, int64_t N_up, int64_t Np, const double *R1,
                     double *state, double *abs_state)
{
    const int mc = m + 3;
    for (int64_t e = 0; e < N; ++e) {
        nsum S[5], A[5];
        for (int c = 0; c < 5; ++c) { S[c].s = S[c].c = 0.0; A[c].s = A[c].c = 0.0; }
        double re[3] = { R1[e], R1[Np + e], R1[2 * Np + e] };
        for (int64_t j = 0; j < N; ++j) {
            if (j == e) continue;
            double rj[3] = { R1[j], R1[Np + j], R1[2 * Np + j] };
            double t[5], a[5];
            if (pair_terms(L, r_cut, m, coef + spin_channel(e, j, N_up) * mc, re, rj, t, a))
                return 1 + e;
            for (int c = 0; c < 5; ++c) { nsum_add(&S[c], t[c]); nsum_add(&A[c], a[c]); }
        }
        for (int c = 0; c < 5; ++c) {
            state[c * Np + e] = nsum_get(&S[c]);
            if (abs_state) abs_state[c * Np + e] = nsum_get(&A[c]);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* orc_accept: Alg. 1 L9 "Accept r_k <- r'_k" for the J2 share of the state   */
/* (PAPER:850), batched over walkers.  For every walker w with accept[w] != 0 */
/* (rejected walkers are left untouched, "or reject"), with k = k[w],         */
/* r_k = R[w][:, k] (before the update) and r'_k = r_new[w]:                  */
/*   for i != k:  state_i += T_i(r'_k) - T_i(r_k),   T_i(r) = the pair terms  */
/*                of pair_terms(r_i, r) -- electron i's partner k moved       */
/*                (Delta J2 = U^2_k(R') - U^2_k(R); the Ref's     */
/*                "column and row are updated for each accepted move",        */
/*                PAPER:1386-1387, here on the 5N accumulators);              */
/*   state_k = sum_{i != k} T_k(r'_k) with d = r'_k - r_i (the from-scratch   */
/*                values at R', equal to qj2_eval's output at r'_k: V, and    */
/*                G = -sum U' (r_i - r'_k)/r);                                */
/*   R[w][:, k] = r'_k  ("both R and Rsoa (6 floats) are updated with the new */
/*                position").                                */
/* Everything fp64 (inputs promoted exactly by the caller).  abs_state        */
/* (optional, [W][5][Np]) receives |state_old| + |T(r')| + |T(r)| per entry   */
/* (sum of |T(r')| for k; untouched for rejected walkers) for the tolerance.  */
/* Returns 0, or 1 + w for the first walker with a coincident pair.          */
/* ------------------------------------------------------------------------ */
int64_t orc_accept(const double L[3], double r_cut, int m, const double *coef,
                   int64_t W, int64_t N, int64_t N_up, int64_t Np,
                   double *R, double *state, const int32_t *k, const double *r_new,
                   const int32_t *accept, double *abs_state)
{
    const int mc = m + 3;
    for (int64_t w = 0; w < W; ++w) {
        if (!accept[w]) continue;
        double *Rw = R + w * 3 * Np;
        double *Sw = state + w * 5 * Np;
        double *Aw = abs_state ? abs_state + w * 5 * Np : NULL;
        const int64_t kw = k[w];
        const double rk[3] = { Rw[kw], Rw[Np + kw], Rw[2 * Np + kw] };
        const double rn[3] = { r_new[3 * w], r_new[3 * w + 1], r_new[3 * w + 2] };
        nsum Sk[5], Ak[5];
        for (int c = 0; c < 5; ++c) { Sk[c].s = Sk[c].c = 0.0; Ak[c].s = Ak[c].c = 0.0; }
        for (int64_t i = 0; i < N; ++i) {
            if (i == kw) continue;
            const double *cs = coef + spin_channel(i, kw, N_up) * mc;
            double ri[3] = { Rw[i], Rw[Np + i], Rw[2 * Np + i] };
            double tn[5], an[5], to[5], ao[5], tk[5], ak[5];
            if (pair_terms(L, r_cut, m, cs, ri, rn, tn, an)) return 1 + w;   /* d = r_i - r'_k */
            if (pair_terms(L, r_cut, m, cs, ri, rk, to, ao)) return 1 + w;   /* d = r_i - r_k  */
            if (pair_terms(L, r_cut, m, cs, rn, ri, tk, ak)) return 1 + w;   /* d = r'_k - r_i */
            for (int c = 0; c < 5; ++c) {
                double old = Sw[c * Np + i];
                Sw[c * Np + i] = old + (tn[c] - to[c]);
                if (Aw) Aw[c * Np + i] = fabs(old) + an[c] + ao[c];
                nsum_add(&Sk[c], tk[c]);
                nsum_add(&Ak[c], ak[c]);
            }
        }
        for (int c = 0; c < 5; ++c) {
            Sw[c * Np + kw] = nsum_get(&Sk[c]);
            if (Aw) Aw[c * Np + kw] = nsum_get(&Ak[c]);
        }
        for (int c = 0; c < 3; ++c) Rw[c * Np + kw] = rn[c];
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: tricubic B-spline single-particle orbitals and the determinant     */
/* ratio.                                                                     */
/*                                                                            */
/* SPOs phi_o(r), o < n_orb, from a read-only 3D B-spline table shared by all */
/* walkers ("the read-only 3D B-spline table which is shared  */
/* by all the threads"; Table 1 "FFT grid", "# of unique SPOs", PAPER:936-    */
/* 958; kernels "Bspline-v" and "Bspline-vgh").   */
/* Reading R22: uniform periodic tricubic B-spline on an          */
/* nx x ny x nz grid over the cell, coefficients P[ix][iy][iz][o] (orbital    */
/* fastest, stride ld >= n_orb), for coordinate u = x/L_x * nx (x wrapped     */
/* into [0, L_x)): i = floor(u), t = u - i, basis B_a(t) as in orc_bspline,   */
/* control points (i - 1 + a) mod nx, a = 0..3; likewise y, z:                */
/*   phi_o = sum_{a,b,c} B_a(tx) B_b(ty) B_c(tz) P[(ix-1+a)%nx][..][..][o],   */
/* gradient and Hessian from the analytic basis derivatives scaled by nx/L_x  */
/* etc.  Outputs v[o], g[3][o], h[6][o] (xx, xy, xz, yy, yz, zz), fp64.       */
/* abs_out (optional, [10][n_orb]) receives the same sums over |weights*P|.   */
/* ------------------------------------------------------------------------ */
static void basis3(double t, double B[4], double D[4], double S[4])
{
    double g = 1.0 - t;
    B[0] = g * g * g / 6.0;
    B[1] = (3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0;
    B[2] = (-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0;
    B[3] = t * t * t / 6.0;
    D[0] = -0.5 * g * g;
    D[1] = 0.5 * (3.0 * t * t - 4.0 * t);
    D[2] = 0.5 * (-3.0 * t * t + 2.0 * t + 1.0);
    D[3] = 0.5 * t * t;
    S[0] = 1.0 - t;
    S[1] = 3.0 * t - 2.0;
    S[2] = 1.0 - 3.0 * t;
    S[3] = t;
}

static void axis_setup(double x, double L, int64_t n, int64_t idx[4], double B[4], double D[4],
                       double S[4], double *scale)
{
    double xw = fmod(x, L);
    if (xw < 0) xw += L;
    double u = xw / L * (double)n;
    double fi = floor(u);
    double t = u - fi;
    int64_t i = (int64_t)fi;
    if (i >= n) { i -= n; }          /* u == n after rounding */
    for (int a = 0; a < 4; ++a) idx[a] = ((i - 1 + a) % n + n) % n;
    basis3(t, B, D, S);
    *scale = (double)n / L;
}

void orc_spo_vgh(int64_t nx, int64_t ny, int64_t nz, int64_t n_orb, int64_t ld,
                 const float *P, const double L[3], const double pos[3],
                 double *v, double *g, double *h, double *abs_out)
{
    int64_t ix[4], iy[4], iz[4];
    double Bx[4], Dx[4], Sx[4], By[4], Dy[4], Sy[4], Bz[4], Dz[4], Sz[4], sx, sy, sz;
    axis_setup(pos[0], L[0], nx, ix, Bx, Dx, Sx, &sx);
    axis_setup(pos[1], L[1], ny, iy, By, Dy, Sy, &sy);
    axis_setup(pos[2], L[2], nz, iz, Bz, Dz, Sz, &sz);
    for (int64_t o = 0; o < n_orb; ++o) {
        nsum acc[10], aab[10];
        for (int c = 0; c < 10; ++c) { acc[c].s = acc[c].c = 0.0; aab[c].s = aab[c].c = 0.0; }
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                for (int c = 0; c < 4; ++c) {
                    double p = (double)P[((ix[a] * ny + iy[b]) * nz + iz[c]) * ld + o];
                    double w[10] = {
                        Bx[a] * By[b] * Bz[c],                       /* v   */
                        Dx[a] * By[b] * Bz[c] * sx,                  /* gx  */
                        Bx[a] * Dy[b] * Bz[c] * sy,                  /* gy  */
                        Bx[a] * By[b] * Dz[c] * sz,                  /* gz  */
                        Sx[a] * By[b] * Bz[c] * sx * sx,             /* hxx */
                        Dx[a] * Dy[b] * Bz[c] * sx * sy,             /* hxy */
                        Dx[a] * By[b] * Dz[c] * sx * sz,             /* hxz */
                        Bx[a] * Sy[b] * Bz[c] * sy * sy,             /* hyy */
                        Bx[a] * Dy[b] * Dz[c] * sy * sz,             /* hyz */
                        Bx[a] * By[b] * Sz[c] * sz * sz };           /* hzz */
                    for (int q = 0; q < 10; ++q) {
                        nsum_add(&acc[q], w[q] * p);
                        nsum_add(&aab[q], fabs(w[q] * p));
                    }
                }
        v[o] = nsum_get(&acc[0]);
        for (int d = 0; d < 3; ++d) g[d * n_orb + o] = nsum_get(&acc[1 + d]);
        for (int q = 0; q < 6; ++q) h[q * n_orb + o] = nsum_get(&acc[4 + q]);
        if (abs_out)
            for (int q = 0; q < 10; ++q) abs_out[q * n_orb + o] = nsum_get(&aab[q]);
    }
}

/* ------------------------------------------------------------------------ */
/* Determinant ratio of a move of electron k (Eq. 6: "a dot    */
/* product of the k-th row of A^{-1} and v(phi_1(r'_k), ..., phi_{N/2}(r'_k))"*/
/* via det(A + u e_k') = (1 + e_k' A^{-1} u) det(A)), with A(i,j) = phi_i(r_j)*/
/* (PAPER:821-823), and the same lemma for the derivatives:   */
/*   rho = sum_i Ainv[k][i] phi_i(r'),                                        */
/*   G   = sum_i Ainv[k][i] grad phi_i(r') / rho     (= grad_k ln D at R'),   */
/*   L   = sum_i Ainv[k][i] lap phi_i(r') / rho      (= lap_k D / D at R').   */
/* Here "row k of A^{-1}" is A^{-1}[k][:] with A^{-1} A = I, so that          */
/* sum_i Ainv[k][i] A(i,j) = delta_kj (reading R23).  out = (rho, Gx, Gy, Gz, */
/* L); abs_out = the sums of |terms| (for rho) used by the tolerance.         */
/* ------------------------------------------------------------------------ */
void orc_det_ratio(int64_t n, const double *Ainv_row, const double *v, const double *g,
                   const double *h, double out[5], double abs_out[5])
{
    nsum r = {0, 0}, G[3] = {{0, 0}, {0, 0}, {0, 0}}, Lp = {0, 0};
    nsum ar = {0, 0}, aG[3] = {{0, 0}, {0, 0}, {0, 0}}, aL = {0, 0};
    for (int64_t i = 0; i < n; ++i) {
        double a = Ainv_row[i];
        nsum_add(&r, a * v[i]);
        nsum_add(&ar, fabs(a * v[i]));
        for (int d = 0; d < 3; ++d) {
            nsum_add(&G[d], a * g[d * n + i]);
            nsum_add(&aG[d], fabs(a * g[d * n + i]));
        }
        double lap = h[0 * n + i] + h[3 * n + i] + h[5 * n + i];
        nsum_add(&Lp, a * lap);
        nsum_add(&aL, fabs(a * h[0 * n + i]) + fabs(a * h[3 * n + i]) + fabs(a * h[5 * n + i]));
    }
    double rho = nsum_get(&r);
    out[0] = rho;
    for (int d = 0; d < 3; ++d) out[1 + d] = nsum_get(&G[d]) / rho;
    out[4] = nsum_get(&Lp) / rho;
    if (abs_out) {
        abs_out[0] = nsum_get(&ar);
        for (int d = 0; d < 3; ++d) abs_out[1 + d] = nsum_get(&aG[d]);
        abs_out[4] = nsum_get(&aL);
    }
}

/* Host twin of the synthetic SPO table generator (qmcgen.spo_table), in     */
/* plain C for large tables.  Not part of the method.  Pinned bitwise        */
/* against qmcgen by tests/test_inputs.py.                                   */
typedef struct { uint64_t key; int64_t e0, e1, ld, n_orb; float *coef; } spo_gen_job;

static void *spo_gen_thread(void *arg)
{
    spo_gen_job *J = (spo_gen_job *)arg;
    for (int64_t e = J->e0; e < J->e1; ++e) {
        int64_t o = e % J->ld;
        float x = 0.0f;
        if (o < J->n_orb) {
            uint64_t h = orc_mix64(J->key ^ (uint64_t)e);
            x = (float)(uint32_t)(h >> 40) * 1.1920928955078125e-07f - 1.0f;
        }
        J->coef[e] = x;
    }
    return NULL;
}

void orc_gen_spo_table(uint64_t seed, int64_t nx, int64_t ny, int64_t nz, int64_t n_orb, int64_t ld,
                       float *coef, int nthreads)
{
    uint64_t k0 = orc_mix64(seed * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull);
    uint64_t key = orc_mix64(k0 ^ 0x5A0C0EFF1C1E17A5ull);
    int64_t total = nx * ny * nz * ld;
    if (nthreads < 1) nthreads = 1;
    spo_gen_job *jobs = (spo_gen_job *)calloc((size_t)nthreads, sizeof(spo_gen_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t per = (total + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        int64_t a = t * per, b = (t + 1) * per;
        if (a > total) a = total;
        if (b > total) b = total;
        spo_gen_job J = { key, a, b, ld, n_orb, coef };
        jobs[t] = J;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, spo_gen_thread, &jobs[t]);
    spo_gen_thread(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs); free(th);
}

/* ------------------------------------------------------------------------ */
/* NEXT-2 at the paper's system sizes: whole particle-by-particle sweeps      */
/* (Alg. 1 L4-L9) of the Jastrow-only trial function.          */
/*                                                                            */
/* orc_propose_f32: Alg. 1 L5 "r'_k <- r_k + ... + delta" without the drift   */
/* term (reading R24: the drift needs grad ln Psi_T including the           */
/* determinant, out of scope), in fp32 -- the sweep's position type -- and    */
/* wrapped into the periodic cell [0, L_d) (SPEC:138 cell convention):        */
/*   x = r + delta (one fp32 rounding); if x < 0: x += L; if x >= L: x -= L.  */
/* Precondition |delta| < L_d.  The second test also catches x + L rounding   */
/* up to L exactly (the result is then 0, the same point of the torus).       */
/* ------------------------------------------------------------------------ */
void orc_propose_f32(const double L[3], int64_t n, const float *r, const float *delta, float *out)
{
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) {
            const float Lf = (float)L[c];
            float x = r[3 * i + c] + delta[3 * i + c];
            if (x < 0.0f) x = x + Lf;
            if (x >= Lf) x = x - Lf;
            out[3 * i + c] = x;
        }
}

/* One-body row of electron position r over the ions (the J1 values of        */
/* orc_eval_j1 for one position, no absolute sums): o = (V, G, L).            */
static int j1_row(const double L[3], int n_species, const int64_t *sp_start, const double *r_cut,
                  const int *m, const double *coef, int coef_stride, int64_t Np, const double *ions,
                  const double r[3], double o[5])
{
    nsum S[5];
    for (int c = 0; c < 5; ++c) S[c].s = S[c].c = 0.0;
    for (int s = 0; s < n_species; ++s)
        for (int64_t I = sp_start[s]; I < sp_start[s + 1]; ++I) {
            double src[3] = { ions[I], ions[Np + I], ions[2 * Np + I] };
            double d[3], rho, u[3];
            orc_min_image(L, r, src, d, &rho);
            if (!(rho < r_cut[s])) continue;
            if (rho == 0.0) return 1;
            orc_bspline(coef + s * coef_stride, m[s], r_cut[s], rho, u);
            nsum_add(&S[0], u[0]);
            for (int c = 0; c < 3; ++c) nsum_add(&S[1 + c], -u[1] * d[c] / rho);
            nsum_add(&S[4], u[2] + 2.0 * u[1] / rho);
        }
    for (int c = 0; c < 5; ++c) o[c] = nsum_get(&S[c]);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* orc_sweep: S particle-by-particle moves of every walker, in order, as the  */
/* paper's compute-on-the-fly J2 does them (the 5N state     */
/* holds U^2_e(R) of every electron so the ratio reuses it; only the row of   */
/* the moved electron at R' is computed):                                     */
/*   for s = 0..S-1, walker w, k = ks[s][w]:                                  */
/*     r_k = R[w][:, k] (the walker's CURRENT position of k), r'_k =          */
/*       orc_propose_f32(r_k, delta[s][w]);                                   */
/*     T' = sum_{i != k} T_k(r'_k) (pair_terms with d = r'_k - r_i: V, G, L   */
/*       of electron k at R');                                                */
/*     dJ2 = T'_V - state[w][V][k]     (Eq. 5, with            */
/*       U^2_k(R) = the stored state);                            */
/*     with ions (n_species > 0): dJ1 = U^1_k(r'_k) - U^1_k(r_k) over the     */
/*       ions, dJ = dJ1 + dJ2 (Eq. 4);                      */
/*     own decision (Alg. 1 L9, reading R19): accept iff u[s][w] < rho^2,    */
/*       rho = exp(dJ);                                                       */
/*     the decision applied is forced[s][w] when forced != NULL (to replay a  */
/*       trajectory whose decisions were taken elsewhere), else the own one;  */
/*     on acceptance: the update of orc_accept (partners += T_i(r'_k) -       */
/*       T_i(r_k), state_k = T', R[:, k] = r'_k) and, with ions, electron k's */
/*       J1 row state_j1[w][:, k] = (V, G, L) of U^1 at r'_k.                 */
/*   A move whose k is outside [0, N) changes nothing: acc_out = -1, dj = 0.  */
/* R is fp32 (positions stay fp32 numbers: the proposal is fp32), states fp64.*/
/* Outputs acc_out[s][w] (own decision 0/1, or -1), dj_out[s][w] (dJ).       */
/* Walkers are independent (threads over walkers).  Returns 0, or 1 + w of    */
/* the first walker with a coincident pair.                                   */
/* ------------------------------------------------------------------------ */
typedef struct {
    const double *L; double r_cut; int m; const double *coef;
    int64_t W, N, N_up, Np;
    float *R; double *state;
    int64_t S; const int32_t *ks; const float *delta; const double *u; const int32_t *forced;
    int32_t *acc_out; double *dj_out;
    int n_species; const int64_t *sp_start; const double *r_cut1; const int *m1; const double *coef1;
    int coef1_stride; int64_t Np_ion; const double *ions; double *state_j1;
    int64_t w0, w1, status;
} sweep_job;

static int64_t sweep_walker(sweep_job *J, int64_t w)
{
    const int mc = J->m + 3;
    const int64_t Np = J->Np;
    float *Rw = J->R + w * 3 * Np;
    double *Sw = J->state + w * 5 * Np;
    for (int64_t s = 0; s < J->S; ++s) {
        const int64_t sw = s * J->W + w;
        const int64_t k = J->ks[sw];
        if (k < 0 || k >= J->N) { J->acc_out[sw] = -1; J->dj_out[sw] = 0.0; continue; }
        float rkf[3] = { Rw[k], Rw[Np + k], Rw[2 * Np + k] }, rnf[3];
        orc_propose_f32(J->L, 1, rkf, J->delta + 3 * sw, rnf);
        const double rk[3] = { rkf[0], rkf[1], rkf[2] }, rn[3] = { rnf[0], rnf[1], rnf[2] };
        nsum Tk[5];
        for (int c = 0; c < 5; ++c) Tk[c].s = Tk[c].c = 0.0;
        for (int64_t i = 0; i < J->N; ++i) {
            if (i == k) continue;
            const double ri[3] = { Rw[i], Rw[Np + i], Rw[2 * Np + i] };
            double t[5], a[5];
            if (pair_terms(J->L, J->r_cut, J->m, J->coef + spin_channel(i, k, J->N_up) * mc, rn, ri, t, a))
                return 1;
            for (int c = 0; c < 5; ++c) nsum_add(&Tk[c], t[c]);
        }
        double dj = nsum_get(&Tk[0]) - Sw[k];
        double o1n[5] = {0, 0, 0, 0, 0};
        if (J->n_species > 0) {
            double o1o[5];
            if (j1_row(J->L, J->n_species, J->sp_start, J->r_cut1, J->m1, J->coef1, J->coef1_stride, J->Np_ion,
                       J->ions, rn, o1n) ||
                j1_row(J->L, J->n_species, J->sp_start, J->r_cut1, J->m1, J->coef1, J->coef1_stride, J->Np_ion,
                       J->ions, rk, o1o))
                return 1;
            dj += o1n[0] - o1o[0];
        }
        const double rho = exp(dj);
        const int own = J->u[sw] < rho * rho ? 1 : 0;
        J->acc_out[sw] = own;
        J->dj_out[sw] = dj;
        const int a = J->forced ? (J->forced[sw] > 0) : own;
        if (!a) continue;
        for (int64_t i = 0; i < J->N; ++i) {
            if (i == k) continue;
            const double *cs = J->coef + spin_channel(i, k, J->N_up) * mc;
            const double ri[3] = { Rw[i], Rw[Np + i], Rw[2 * Np + i] };
            double tn[5], to[5], an[5], ao[5];
            if (pair_terms(J->L, J->r_cut, J->m, cs, ri, rn, tn, an)) return 1;   /* d = r_i - r'_k */
            if (pair_terms(J->L, J->r_cut, J->m, cs, ri, rk, to, ao)) return 1;   /* d = r_i - r_k  */
            for (int c = 0; c < 5; ++c) Sw[c * Np + i] += tn[c] - to[c];
        }
        for (int c = 0; c < 5; ++c) Sw[c * Np + k] = nsum_get(&Tk[c]);
        for (int c = 0; c < 3; ++c) Rw[c * Np + k] = rnf[c];
        if (J->n_species > 0)
            for (int c = 0; c < 5; ++c) J->state_j1[(w * 5 + c) * Np + k] = o1n[c];
    }
    return 0;
}

static void *sweep_thread(void *arg)
{
    sweep_job *J = (sweep_job *)arg;
    J->status = 0;
    for (int64_t w = J->w0; w < J->w1 && !J->status; ++w)
        if (sweep_walker(J, w)) J->status = 1 + w;
    return NULL;
}

int64_t orc_sweep(const double L[3], double r_cut, int m, const double *coef,
                  int64_t W, int64_t N, int64_t N_up, int64_t Np, float *R, double *state,
                  int64_t S, const int32_t *ks, const float *delta, const double *u, const int32_t *forced,
                  int32_t *acc_out, double *dj_out,
                  int n_species, const int64_t *sp_start, const double *r_cut1, const int *m1,
                  const double *coef1, int coef1_stride, int64_t Np_ion, const double *ions,
                  double *state_j1, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > W) nthreads = (int)(W > 0 ? W : 1);
    sweep_job *jobs = (sweep_job *)calloc((size_t)nthreads, sizeof(sweep_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t per = (W + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        sweep_job J = { L, r_cut, m, coef, W, N, N_up, Np, R, state, S, ks, delta, u, forced, acc_out, dj_out,
                        n_species, sp_start, r_cut1, m1, coef1, coef1_stride, Np_ion, ions, state_j1, 0, 0, 0 };
        J.w0 = t * per < W ? t * per : W;
        J.w1 = (t + 1) * per < W ? (t + 1) * per : W;
        jobs[t] = J;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, sweep_thread, &jobs[t]);
    sweep_thread(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    int64_t st = 0;
    for (int t = 0; t < nthreads && !st; ++t) st = jobs[t].status;
    free(jobs); free(th);
    return st;
}
