/*
 * qmcj2.h -- C ABI of the B200 (sm_100a) hot path of arXiv 1708.02645
 * (Mathuriya et al., SC'17): the batched on-the-fly electron-electron distance
 * row and two-body Jastrow (J2) value, gradient and Laplacian of a
 * particle-by-particle move.
 *
 * Citations: PAPER:n = line n of the paper's LaTeX,
 * SPEC:n = line n of the CPU-miniapp spec written from it (interfaces only).
 *
 * Conventions common to every entry point
 * ---------------------------------------
 * - Plain pointers and sizes only.  "device" pointers are CUDA device
 *   (or managed) memory owned by the caller; "host" pointers are host memory
 *   owned by the caller.  The library never frees caller memory and
 *   allocates no device memory (scratch comes from the caller's workspace).
 * - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   Device-pointer entry points are asynchronous on that stream; asynchronous
 *   device faults surface at the caller's next synchronisation.
 * - Every entry point validates its arguments on the host before any launch
 *   and returns a qj2_status; no exception crosses the ABI.  On failure,
 *   qj2_last_error() returns a thread-local detail string.
 * - The library holds no global mutable state: calls on different streams with
 *   different workspaces are independent and may run concurrently.
 * - Device entry points require an sm_100 device (else QJ2_ENOTSUP).
 * - All sizes are int64; all flat offsets inside kernels are 64-bit.
 * - Kernel variants are chosen from the arguments alone (one variant per
 *   argument shape; no environment variable is read).  The alternatives
 *   measured against them are compile-time builds (tools/ab).
 */
#ifndef QMCJ2_H
#define QMCJ2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QJ2_VERSION 20000 /* major*10000 + minor*100 + patch */

typedef enum {
    QJ2_OK = 0,
    QJ2_EINVAL = 1,   /* invalid argument ("invalid-argument") */
    QJ2_ERANGE = 2,   /* out-of-range index/slice ("out-of-range") */
    QJ2_ENOTSUP = 3,  /* current device is not sm_100 (B200) */
    QJ2_ECUDA = 4     /* CUDA launch / runtime failure */
} qj2_status;

typedef enum { QJ2_FP32 = 0, QJ2_FP64 = 1 } qj2_dtype;

enum { QJ2_MAX_M = 64, QJ2_MAX_P = 64, QJ2_MAX_SPECIES = 4 };

/*
 * Two-body Jastrow functor U_s(r) and the simulation cell.
 * PAPER:812-819 (Eq. 3, "one-dimensional cubic B-spline")
 * ("finite cutoff"), SPEC:256-258 (uniform B-spline: delta = r_cut/m, m+3
 * coefficients, zero for r >= r_cut).  Basis convention (R3):
 *   t = r/delta, j = min(floor(t), m-1), f = t - j,
 *   U(r) = sum_{a=0..3} coef[s][j+a] B_a(f), uniform cubic B-spline basis.
 * Channel s = 0 same spin, 1 opposite spin.
 * Requirements (else QJ2_EINVAL): L[d] > 0, 0 < r_cut <= min(L)/2 (so the
 * minimum image is exact), 4 <= m <= QJ2_MAX_M, coef[s][m..m+2] == 0 (the
 * functor and its first two derivatives vanish at r_cut), finite values.
 * Passed by pointer to host memory; copied into kernel parameters per call.
 */
typedef struct {
    double  L[3];                      /* orthorhombic periodic cell lengths */
    double  r_cut;                     /* functor cutoff radius */
    int32_t m;                         /* number of B-spline intervals */
    int32_t reserved;                  /* must be 0 */
    double  coef[2][QJ2_MAX_M + 3];    /* [0] same-spin, [1] opposite-spin */
} qj2_functor;

/* ------------------------------------------------------------------------ */
/* Library information                                                       */
/* ------------------------------------------------------------------------ */
int32_t     qj2_version(void);
const char *qj2_status_string(qj2_status s);     /* static string, never NULL */
const char *qj2_last_error(void);                /* thread-local detail, never NULL */

/* QJ2_OK if the current CUDA device is sm_100 (compute capability 10.0),
 * QJ2_ENOTSUP otherwise, QJ2_ECUDA if there is no usable device. */
qj2_status  qj2_device_check(void);

/* ------------------------------------------------------------------------ */
/* padded_size ("Np includes the padding for     */
/* alignment"): *out = smallest multiple of block >= max(n, 1).              */
/* Errors: n < 0 or block < 1 -> QJ2_EINVAL; out == NULL -> QJ2_EINVAL.      */
/* ------------------------------------------------------------------------ */
qj2_status qj2_padded_size(int64_t n, int64_t block, int64_t *out);

/* ------------------------------------------------------------------------ */
/* Scratch needed by qj2_eval for (W, P, N_local, dtype): per-tile fp64      */
/* partial sums plus per-(walker, trial-group) completion counters.          */
/* ------------------------------------------------------------------------ */
qj2_status qj2_eval_workspace_size(int64_t W, int32_t P, int64_t N_local,
                                   qj2_dtype dtype, size_t *bytes);

/* ------------------------------------------------------------------------ */
/* qj2_eval -- THE HOT PATH.             */
/*                                                                           */
/* For every walker w < W and trial p < P, with r = r_trial[w][p]:           */
/*   d_i = minimg(r_i - r)  (1-by-N relations d(k,i),       */
/*         dr(k,i); Fig. 6's temporary row v, computed on   */
/*         the fly)                                         */
/*   V  = sum_{i != k, |d_i| < r_cut} U_s(|d_i|)                             */
/*   G  = -sum U_s'(|d_i|) d_i/|d_i|           (= grad_r V)                  */
/*   L  = sum U_s''(|d_i|) + 2 U_s'(|d_i|)/|d_i|   (= lap_r V)               */
/* over the source slice i in [i_offset, i_offset + N_local).  With the full */
/* range and r = r'_k these are U^2_k(R') of PAPER:1382 (one term of Eq. 5,  */
/* PAPER:885-887) and the J2 shares of grad_k, lap_k at R' (Alg. 1 L8,       */
/* PAPER:849).  Arithmetic: dtype positions and per-term math, fp64          */
/* accumulation and outputs ("quantities per walker ... in double           */
/* precision"); with fp32 positions and a functor finer than  */
/* m = 16 the displacement, r and r/delta are formed in fp64 and only the    */
/* interval fraction is rounded to fp32 (fp32 r/delta would leave ~m*2^-23   */
/* of the functor scale per term).                                           */
/*                                                                           */
/* Arguments                                                                 */
/*   fn        host, functor + cell (see qj2_functor).                       */
/*   dtype     QJ2_FP32 or QJ2_FP64: type of R, r_trial and row_out.         */
/*   W         walkers (>= 0; W == 0 is a no-op).                            */
/*   N_total   electrons per walker (>= 2).  N_up: spin-up electrons are     */
/*             global indices [0, N_up) (0 <= N_up <= N_total).              */
/*   i_offset, N_local: this call's source slice (sharding along the        */
/*             electron axis; 0 <= i_offset, 1 <= N_local,                   */
/*             i_offset + N_local <= N_total else QJ2_ERANGE).  Spin channel */
/*             and self-exclusion use GLOBAL indices, so the slices' partial */
/*             sums add up to the unsplit result.                            */
/*   Np        padded lane length, Np >= N_local, Np % 4 == 0 (fp32) or      */
/*             Np % 2 == 0 (fp64).                                           */
/*   R         device [W][3][Np] dtype, SoA lanes x|y|z (PAPER:1290-1296,    */
/*             Rsoa[3][Np]); coordinates in [0, L_d); 16-byte aligned (fp32  */
/*             rows that start 32-byte aligned -- R so aligned, Np % 8 == 0  */
/*             -- are read with 256-bit loads: same results, faster).        */
/*   k         device [W] int32, active electron, global index < N_total.    */
/*   P         trial positions per walker, 1 <= P <= QJ2_MAX_P.             */
/*   r_trial   device [W][P][3] dtype, coordinates in [0, L_d).              */
/*   out       device [W][P][5] fp64: (V, Gx, Gy, Gz, L) over the slice.     */
/*   row_out   device [W][P][4][Np] dtype (r, dx, dy, dz) or NULL: the       */
/*             candidate distance row v;     */
/*             slot k and padding slots are unspecified.  16-byte aligned.   */
/*   V_cur     device [W] fp64 or NULL: U^2_k(R) from the caller's 5N state  */
/*              for the ratio below.                        */
/*   ratio_out device [W][P][2] fp64 or NULL: (dJ2, exp(dJ2)) with           */
/*             dJ2 = V_p - V_cur[w] (or V_p - V_0 when V_cur == NULL; for    */
/*             P > 1 that is a second, tiny launch after the reduction):     */
/*             the e^{dJ2} factor of Eq. 4.            */
/*             Only for unsharded calls (i_offset == 0, N_local == N_total); */
/*             sharded callers reduce `out` first and call qj2_ratio.        */
/*   workspace device scratch >= qj2_eval_workspace_size() (per-tile fp64   */
/*             partials + completion counters, which the call zeroes itself  */
/*             with one cudaMemsetAsync when the slice spans > 1 tile).  No  */
/*             initialisation needed.  One workspace per concurrent call.    */
/*   stream    cudaStream_t.                                                 */
/* Preconditions not checked on the hot path (see qj2_check_inputs):         */
/* coordinates in range, k < N_total, no coincident source inside the        */
/* cutoff (r = 0 is undefined: the result may be non-finite).                */
/* ------------------------------------------------------------------------ */
qj2_status qj2_eval(const qj2_functor *fn, qj2_dtype dtype,
                    int64_t W, int64_t N_total, int64_t N_up,
                    int64_t i_offset, int64_t N_local, int64_t Np,
                    const void *R, const int32_t *k,
                    int32_t P, const void *r_trial,
                    double *out, void *row_out,
                    const double *V_cur, double *ratio_out,
                    void *workspace, size_t workspace_bytes,
                    void *stream);

/* ------------------------------------------------------------------------ */
/* NEXT-1: one-body Jastrow over the electron-ion (AB) row.                  */
/* PAPER:1376-1381 ("Delta J1 = U^1_k(R') - U^1_k(R), U^1_k = sum_I U_I(     */
/* |r_I - r_k|)"), Eq. (3) first term; per-species functors  */
/* (Fig. 3); ions fixed and shared by every walker            */
/* (PAPER:1306-1308).  Species s: cutoff r_cut[s], m[s] intervals, m[s]+3    */
/* uniform cubic B-spline coefficients (same convention as qj2_functor; tail */
/* coef[s][m[s]..m[s]+2] must be 0).                                         */
/* ------------------------------------------------------------------------ */
typedef struct {
    double  L[3];                                   /* cell */
    int32_t n_species;                              /* 1 <= n_species <= QJ2_MAX_SPECIES */
    int32_t reserved;                               /* must be 0 */
    double  r_cut[QJ2_MAX_SPECIES];                 /* 0 < r_cut[s] <= min(L)/2 */
    int32_t m[QJ2_MAX_SPECIES];                     /* 4 <= m[s] <= QJ2_MAX_M */
    double  coef[QJ2_MAX_SPECIES][QJ2_MAX_M + 3];
} qj2_j1_functor;

/* For every walker w and trial p (r = r_trial[w][p]), over all ions I:        */
/*   V = sum_I U_{s(I)}(|d_I|), G = -sum U' d/|d|, L = sum U'' + 2U'/|d|,      */
/*   d_I = minimg(r_I - r); no self term.  Same output layout, precision,      */
/*   row output ([W][P][4][Np]: the AB row), fused ratio and workspace rules   */
/*   as qj2_eval (workspace size: qj2_eval_workspace_size(W, P, n_ions, dtype)).*/
/*   species_start: host [n_species+1], species_start[0] = 0, nondecreasing;   */
/*   ions are sorted by species: species s owns [species_start[s], [s+1]).     */
/*   ions: device [3][Np] dtype (SoA x|y|z, the ions' Rsoa), coordinates in    */
/*   [0, L_d), padding 0, 16-byte aligned; Np >= n_ions, Np % 4 (fp32) / 2.    */
qj2_status qj2_eval_j1(const qj2_j1_functor *fn, qj2_dtype dtype, int64_t W,
                       const int64_t *species_start, int64_t Np, const void *ions,
                       int32_t P, const void *r_trial, double *out, void *row_out,
                       const double *V_cur, double *ratio_out,
                       void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* qj2_ratio: ratio_out[w][p] = (dJ2, exp(dJ2)), dJ2 = out[w][p][0] - ref,   */
/* ref = V_cur[w] or out[w][0][0] when V_cur == NULL (Eq. 4-5, PAPER:875-887,*/
/* PAPER:1382).  For sharded evaluation after the partial sums are reduced.  */
/* out, V_cur, ratio_out: device fp64.  W >= 0, 1 <= P <= QJ2_MAX_P.         */
/* ------------------------------------------------------------------------ */
qj2_status qj2_ratio(int64_t W, int32_t P, const double *out, const double *V_cur,
                     double *ratio_out, void *stream);

/* ------------------------------------------------------------------------ */
/* NEXT-2: accept-side update (Alg. 1 L9 "Accept r_k <- r'_k or reject",     */
/* PAPER:850) of the positions and the per-electron J2 state.                */
/*                                                                           */
/* The state is the paper's compute-on-the-fly J2 storage, "5N sizeof(T)"    */
/* per walker: for electron e,                             */
/*   V_e = sum_{j != e} U_s(r_ej),  G_e = sum_{j != e} U_s'(r_ej) d_ej/r_ej, */
/*   L_e = sum_{j != e} U_s''(r_ej) + 2 U_s'(r_ej)/r_ej,  d_ej = minimg(r_e - r_j), */
/* i.e. electron e's share of J2 and the gradient/Laplacian of J2 with      */
/* respect to r_e, stored SoA as state[w][5][Np] (rows V, Gx, Gy, Gz, L; the */
/* Rsoa layout), type dtype.                                */
/*                                                                           */
/* For every walker w with accept[w] != 0 (others are not touched), k = k[w]:*/
/*   partners i != k in the slice:                                           */
/*     state_i += T_i(r'_k) - T_i(r_k), T_i(r) = (U, U' d/|d|, U''+2U'/|d|), */
/*     d = minimg(r_i - r), per-term arithmetic in dtype (one rounding of   */
/*     the stored sum per update);                                           */
/*   if k is in the slice: state_k = out_new row w (qj2_eval's V, G, L at    */
/*     r'_k over ALL sources -- after the all-reduce when sharded -- rounded */
/*     to dtype: "reuse the computed values"), and R[:, k] = r'_k */
/*     ("both R and Rsoa (6 floats) are updated").          */
/*                                                                           */
/* Arguments (sizes, slice, N_up, Np, alignment: as qj2_eval)                */
/*   R         device [W][3][Np] dtype, in/out.                              */
/*   state     device [W][5][Np] dtype, in/out, 16-byte aligned; padding     */
/*             slots [N_local, Np) are not modified.                         */
/*   k         device [W] int32, global index of the moved electron.         */
/*   r_new     device dtype, row w at r_new + w*r_stride = r'_k in [0, L_d); */
/*             r_stride >= 3 (3*P for qj2_eval's r_trial[W][P][3]).         */
/*   r_old     device [W][3] dtype, r_k before the move, or NULL: then it is */
/*             gathered from R (every accepted walker's k must lie in the    */
/*             slice; sharded callers whose slice may not hold k pass r_old).*/
/*   accept    device [W] int32, nonzero = accepted.                          */
/*   out_new   device fp64, row w at out_new + w*out_stride = (V, Gx, Gy, Gz,*/
/*             L) at r'_k; out_stride >= 5 (e.g. 5*P for qj2_eval's out).    */
/*   workspace device, >= qj2_accept_workspace_size() (r_old gather; 0 bytes */
/*             needed when r_old != NULL).                                   */
/* Two launches when r_old == NULL (gather, update), else one.  Errors as    */
/* qj2_eval; out-of-range k or coordinates are preconditions.                */
/* ------------------------------------------------------------------------ */
qj2_status qj2_accept_workspace_size(int64_t W, qj2_dtype dtype, size_t *bytes);
qj2_status qj2_accept(const qj2_functor *fn, qj2_dtype dtype,
                      int64_t W, int64_t N_total, int64_t N_up,
                      int64_t i_offset, int64_t N_local, int64_t Np,
                      void *R, void *state, const int32_t *k,
                      const void *r_new, int64_t r_stride, const void *r_old,
                      const int32_t *accept, const double *out_new, int64_t out_stride,
                      void *workspace, size_t workspace_bytes, void *stream);

/* Metropolis decision of Alg. 1 L9 for a J2-only trial function and a       */
/* symmetric proposal: accept[w] = (u[w] < rho_w^2), rho_w = ratio[w*stride  */
/* + 1] = e^{dJ2} (qj2_eval / qj2_ratio's ratio_out; Eq. 4).  */
/* u: device [W] fp64 uniform deviates in [0, 1) drawn by the caller (the    */
/* method's random numbers are inputs).  ratio_stride >= 2 (2*P for          */
/* ratio_out[W][P][2] at trial 0).  accept: device [W] int32 (0/1).          */
qj2_status qj2_metropolis(int64_t W, const double *ratio, int64_t ratio_stride,
                          const double *u, int32_t *accept, void *stream);

/* qj2_metropolis_accept -- qj2_metropolis fused into qj2_accept (one launch */
/* per move instead of three: the paper-sized sweeps are launch-bound).      */
/* Every CTA of walker w takes the same decision                             */
/*   accept[w] = u[w] < rho^2,  rho = exp(V_new - V_ref),                    */
/*   V_new = out_new[w*out_stride], V_ref = v_ref[w*v_ref_stride]            */
/* (v_ref = qj2_eval's out at r_k of the P = 2 drift variant, stride 5P, or  */
/* the caller's V_cur, stride 1), writes it to accept (device [W] int32,     */
/* OUTPUT), and applies the update of qj2_accept to accepted walkers.        */
/* r_old is REQUIRED here (row w at r_old + w*r_stride, e.g. trial 0 of the  */
/* drift variant); r_new likewise with the same stride.  Other arguments and */
/* errors as qj2_accept; no workspace.                                       */
qj2_status qj2_metropolis_accept(const qj2_functor *fn, qj2_dtype dtype,
                                 int64_t W, int64_t N_total, int64_t N_up,
                                 int64_t i_offset, int64_t N_local, int64_t Np,
                                 void *R, void *state, const int32_t *k,
                                 const void *r_new, const void *r_old, int64_t r_stride,
                                 const double *out_new, const double *v_ref, int64_t out_stride,
                                 int64_t v_ref_stride, const double *u, int32_t *accept, void *stream);

/* qj2_sweep -- S particle-by-particle moves of every walker in ONE launch,  */
/* the walker resident in shared memory (the paper's system sizes: Table 1   */
/* N = 256..768).  Alg. 1 L4-L9 for a Jastrow-only trial     */
/* function.  For s = 0..S-1 and walker w, k = ks[s*W + w]:                  */
/*   r_k  = the walker's CURRENT position of electron k (R as updated by the */
/*          earlier accepted moves of this call);                            */
/*   r'_k = wrap(r_k + delta[(s*W + w)*3 ..]): fp32 x = r + d, then x += L_d */
/*          if x < 0, then x -= L_d if x >= L_d (Alg. 1 L5 without the drift */
/*          term, reading R24; precondition |d| < L_d);                      */
/*   dJ2  = U^2_k(R') - U^2_k(R): U^2_k(R') = sum_{i != k} U(|r_i - r'_k|)   */
/*          computed on the fly, U^2_k(R) = state[w][0][k], the stored 5N    */
/*          state (PAPER:1382-1393 -- the caller keeps the state consistent  */
/*          with R: qj2_state_init, qj2_accept, earlier sweeps);             */
/*   accept[s*W + w] = u[s*W + w] < exp(2 dJ) (reading R19), dj[s*W + w] =   */
/*          dJ if dj != NULL;                                                */
/*   on acceptance the update of qj2_accept: state_i += T_i(r'_k) - T_i(r_k) */
/*          for i != k, state_k = (V, G, L) at r'_k, R[:, k] = r'_k.         */
/* Any k sequence is valid (an electron may move any number of times).       */
/* fp32 only: R [W][3][Np], state [W][5][Np] (in/out), delta fp32, u fp64,   */
/* accept int32 (out).  Requirements (else QJ2_EINVAL): 2 <= N <= 1024,      */
/* Np >= N, functor m <= 16 (pair terms are kept in fp32; finer functors use */
/* qj2_eval + qj2_metropolis_accept).  Moves within a call are sequential    */
/* per walker; walkers are independent.  Preconditions (not scanned): a move */
/* whose k is outside [0, N) is never accepted (nothing is written), its     */
/* accept entry is -1 and its dj entry 0.                                    */
/*                                                                           */
/* Optional one-body Jastrow (j1 != NULL; NEXT-1 joined to the move): the   */
/* ratio becomes exp(dJ1 + dJ2) (Eq. 4-5) with dJ1 =         */
/* U^1_k(r'_k) - U^1_k(r_k) over the ions (both computed on the fly), dj     */
/* holds dJ1 + dJ2, and on acceptance electron k's J1 row (U^1_k, grad, lap */
/* at r'_k, as qj2_eval_j1 computes them) is written to j1->state.  Ions    */
/* fixed, <= 256 of them, sorted by species, species m <=  */
/* 16; the J1 functor's cell must equal fn's.                                */
typedef struct {
    const qj2_j1_functor *fn;       /* host: per-species functors and cell   */
    const int64_t *species_start;   /* host [n_species + 1], as qj2_eval_j1  */
    const float *ions;              /* device [3][Np_ion] fp32               */
    int64_t Np_ion;                 /* >= number of ions                     */
    float *state;                   /* device [W][5][Np] fp32 (rows of accepted k written) */
} qj2_sweep_j1;

qj2_status qj2_sweep(const qj2_functor *fn, int64_t W, int64_t N, int64_t N_up, int64_t Np,
                     float *R, float *state, int64_t S, const int32_t *ks, const float *delta,
                     const double *u, int32_t *accept, double *dj, const qj2_sweep_j1 *j1,
                     void *stream);

/* qj2_state_init -- the 5N J2 state of every electron from scratch (the     */
/* "new states are periodically computed from scratch" of PAPER:764-765):    */
/* state[w][:, e] = (V_e, G_e, L_e) as defined for qj2_accept, over all      */
/* partners j != e, fp32 pair terms with fp64 sums of <= 32-term partials.   */
/* With j1 != NULL also every electron's J1 row into j1->state.  Sizes and   */
/* requirements as qj2_sweep (2 <= N <= 1024, m <= 16).  R [W][3][Np] fp32   */
/* (read), state [W][5][Np] fp32 (written; padding untouched).               */
qj2_status qj2_state_init(const qj2_functor *fn, int64_t W, int64_t N, int64_t N_up, int64_t Np,
                          const float *R, float *state, const qj2_sweep_j1 *j1, void *stream);

/* ------------------------------------------------------------------------ */
/* NEXT-4: tricubic B-spline single-particle orbitals (SPOs) and the         */
/* determinant ratio.                                                        */
/*                                                                           */
/* The SPO set is a read-only 3D B-spline table shared by all walkers        */
/* (Table 1 "FFT grid" and "# of unique SPOs", PAPER:936-   */
/* 958), single precision as in the paper ("all the quantities are in double */
/* precision ... except for the Bspline-SPO").  Convention  */
/* (R22): uniform periodic tricubic B-spline on an nx x ny x nz    */
/* grid over the orthorhombic cell; for u = (x mod L_x) / L_x * nx, i =      */
/* floor(u), t = u - i, control points (i - 1 + a) mod nx, a = 0..3, with   */
/* the uniform cubic basis B_a(t) (the same basis as qj2_functor); likewise */
/* y, z:  phi_o(r) = sum_{a,b,c} B_a(t_x) B_b(t_y) B_c(t_z) P[ix][iy][iz][o].*/
/* ------------------------------------------------------------------------ */
typedef struct {
    double  L[3];               /* cell */
    int64_t nx, ny, nz;         /* grid, each >= 4 */
    int64_t n_orb;              /* orbitals, >= 1 */
    int64_t ld;                 /* lane stride of a row, >= n_orb, ld % 4 == 0 */
    const float *coef;          /* device [nx][ny][nz][ld] fp32, 16-byte aligned; */
                                /* nx*ny*nz*ld < 2^31; lanes [n_orb, ld) ignored  */
} qj2_spo_table;

enum { QJ2_SPO_V = 0, QJ2_SPO_VGH = 1, QJ2_SPO_GATHER = 0x10 };

/* qj2_spo_eval -- "Bspline-v" (what = QJ2_SPO_V) or "Bspline-vgh"          */
/* (QJ2_SPO_VGH) at one position per walker, fused with the determinant     */
/* ratio of Eq. 6: with A(i,j) = phi_i(r_j) */
/* and a = row k of A^{-1} (reading R23),                                    */
/*   rho = sum_o a_o phi_o(r'),  G = sum_o a_o grad phi_o(r') / rho,         */
/*   L = sum_o a_o lap phi_o(r') / rho   (the determinant's ratio, grad ln D */
/*   and lap D / D at R'; same lemma).                        */
/* Arguments                                                                 */
/*   tab        host struct (the table itself is device memory).             */
/*   what       QJ2_SPO_V or QJ2_SPO_VGH, optionally | QJ2_SPO_GATHER: use    */
/*              the per-thread-gather kernel (the one taken for rows too long */
/*              for the TMA ring) regardless of the row length -- the same    */
/*              sums in the same order, for validation of that kernel.        */
/*   pos_dtype  QJ2_FP32 / QJ2_FP64 of pos.                                  */
/*   W          evaluations (>= 0).                                          */
/*   pos        device, row w at pos + w*pos_stride elements (x, y, z), any  */
/*              real value (wrapped into the cell); pos_stride >= 3.         */
/*   Ainv       device fp32 or NULL (no ratio): for evaluation w the row of  */
/*              walker a = w / points_per_walker at                          */
/*              Ainv + a*ainv_stride + krow[a]*ainv_ld (krow == NULL: row 0),*/
/*              n_orb entries.                                               */
/*   points_per_walker >= 1: consecutive evaluations sharing one walker's    */
/*              A^{-1} row (12 for the NLPP quadrature).      */
/*   out        device fp64 [W][5] (rho, Gx, Gy, Gz, L) or NULL; with        */
/*              QJ2_SPO_V only rho is computed (G, L written as 0).          */
/*   spo_out    device fp32 [W][10][ld] (v, gx, gy, gz, hxx, hxy, hxz, hyy,  */
/*              hyz, hzz; QJ2_SPO_VGH) or [W][1][ld] (QJ2_SPO_V), or NULL.   */
/* Errors: EINVAL for bad sizes / NULL table / misalignment.                 */
qj2_status qj2_spo_eval(const qj2_spo_table *tab, int32_t what, qj2_dtype pos_dtype, int64_t W,
                        const void *pos, int64_t pos_stride,
                        const float *Ainv, int64_t ainv_stride, int64_t ainv_ld, const int32_t *krow,
                        int64_t points_per_walker, double *out, float *spo_out, void *stream);

/* Synthetic SPO coefficient table (test/bench harness, NOT the method):     */
/* coef[ix][iy][iz][o] = 2u - 1, u = top 24 bits of mix64(key' ^ flat index) */
/* * 2^-24 with key' = mix64(mix64(seed*G + G) ^ 0x5A0C0EFF1C1E17A5), flat   */
/* index = ((ix*ny + iy)*nz + iz)*ld + o; lanes o >= n_orb are 0 (qmcgen).   */
qj2_status qj2gen_spo_table(uint64_t seed, int64_t nx, int64_t ny, int64_t nz, int64_t n_orb,
                            int64_t ld, float *coef, void *stream);

/* ------------------------------------------------------------------------ */
/* Host-buffer variant of qj2_eval (the end-to-end path): R, k, r_trial are  */
/* HOST arrays (pinned for full PCIe rate), out (and ratio_out if non-NULL)  */
/* HOST arrays, same shapes as qj2_eval.  Walkers are streamed in chunks of  */
/* chunk_walkers through two device staging buffers carved from workspace:  */
/* the host->device copy of chunk c+1 overlaps the kernel of chunk c.        */
/* Blocking: returns after out is written (synchronises `stream`).           */
/* workspace: device, >= qj2_eval_host_workspace_size() (no initialisation). */
/* ------------------------------------------------------------------------ */
qj2_status qj2_eval_host_workspace_size(int64_t W, int32_t P, int64_t Np,
                                        qj2_dtype dtype, int64_t chunk_walkers,
                                        size_t *bytes);
qj2_status qj2_eval_host(const qj2_functor *fn, qj2_dtype dtype,
                         int64_t W, int64_t N_total, int64_t N_up,
                         int64_t i_offset, int64_t N_local, int64_t Np,
                         const void *R_host, const int32_t *k_host,
                         int32_t P, const void *r_trial_host,
                         double *out_host, const double *V_cur_host,
                         double *ratio_out_host,
                         int64_t chunk_walkers,
                         void *workspace, size_t workspace_bytes,
                         void *stream);

/* ------------------------------------------------------------------------ */
/* Building blocks, batched on the device (for tests and callers):           */
/* qj2_functor_eval_vgl: out[n][3] fp64 = (U_s, U_s', U_s'')  */
/*   at r[n] (device, dtype), channel s in {0, 1}; zero for r >= r_cut.      */
/* qj2_min_image_disp: out[n][4] dtype =                 */
/*   (|d|, dx, dy, dz), d = minimg(b - a), a/b device [n][3] dtype in        */
/*   [0, L_d); components in (-L_d/2, L_d/2] (+-1 ulp at exact ties).        */
/* ------------------------------------------------------------------------ */
qj2_status qj2_functor_eval_vgl(const qj2_functor *fn, qj2_dtype dtype, int32_t channel,
                                int64_t n, const void *r, double *out, void *stream);
qj2_status qj2_min_image_disp(const double L[3], qj2_dtype dtype, int64_t n,
                              const void *a, const void *b, void *out, void *stream);

/* ------------------------------------------------------------------------ */
/* Optional device-side precondition scan for qj2_eval's data.  ORs into     */
/* *d_flag (device int32, caller zeroes it): 1 = coordinate outside [0,L_d)  */
/* or non-finite in R[:, :, :N_local], 2 = k outside [0, N_total),           */
/* 4 = r_trial coordinate outside [0, L_d) or non-finite.                    */
/* ------------------------------------------------------------------------ */
qj2_status qj2_check_inputs(const qj2_functor *fn, qj2_dtype dtype,
                            int64_t W, int64_t N_total, int64_t N_local, int64_t Np,
                            const void *R, const int32_t *k,
                            int32_t P, const void *r_trial,
                            int32_t *d_flag, void *stream);

/* ------------------------------------------------------------------------ */
/* Synthetic-input generator (test/bench harness, NOT part of the method):   */
/* writes R[w][d][i] for w in [0, W), i in [0, Np) as the counter-based      */
/* hash recipe of qmcgen/ (DESIGN.md "Input recipe"):                        */
/*   key = mix64(seed*G + G), h = mix64(key ^ (((w_offset+w)*3 + d) << 32   */
/*         | (i_offset+i))), u = top 24 (fp32) / 53 (fp64) bits of h,        */
/*   x = fl(L*u) kept below L; padding slots i >= N_local are 0.             */
/* R: device [W][3][Np] dtype.                                               */
/* ------------------------------------------------------------------------ */
qj2_status qj2gen_positions(qj2_dtype dtype, uint64_t seed, int64_t W, int64_t w_offset,
                            int64_t i_offset, int64_t N_local, int64_t Np,
                            double L, void *R, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* QMCJ2_H */
