// sweep.cuh -- NEXT-2 at the paper's system sizes: whole particle-by-particle
// sweeps of the Jastrow factor (J2, optionally with J1) in one persistent
// kernel, the walker resident in shared memory (sm_100a).
//
// One CTA per walker.  For every move s < S (Alg. 1 L4-L9; electron
// k = ks[s][w], proposal displacement delta[s][w]):
//   0. r_k is the walker's CURRENT position of k (shared memory) and
//      r'_k = wrap(r_k + delta) is formed in fp32 (Alg. 1 L5 without drift,
//      reading R24);
//   1. each thread forms, for its partners i != k (i = tid + j*TPB), the pair
//      terms T_i(r'_k) with the eval kernel's fp32 arithmetic (single-rounding
//      minimum image, power-basis Horner), keeps them in registers and sums
//      them: the sums are U^2_k(R') and its gradient / Laplacian (Alg. 1 L7-L8);
//   2. a fixed-order reduce-scatter (fp32 partials of <= 32 terms, then fp64)
//      and ONE barrier;
//   3. dJ2 = U^2_k(R') - U^2_k(R), with U^2_k(R) the electron's entry of the 5N
//      state (the state is kept so the ratio reuses it; the
//      owner of slot k publishes it before the barrier); every thread takes
//      the same Metropolis decision u < exp(2 dJ) (reading R19);
//   4. if accepted: each thread forms T_i(r_k) for its partners and adds
//      T_i(r'_k) - T_i(r_k) to their state; the owner of slot k writes
//      state_k = the sums at r'_k and r_k <- r'_k.
// Rejected moves cost one pass of pair terms, accepted ones two.  R and the
// 5N state stay in shared memory for all S moves (32 B per electron: N <= 1024
// in 32 KB); global memory is touched to load and store them once and to read
// the moves -- no launch per move.
#pragma once

#include "qmcj2.h"
#include "j2_device.cuh"

namespace qj2 {

constexpr int SW_MAXN = 1024;     // electrons per walker (the largest tier: 128 threads x 8 partners)

struct SweepParams {
    int32_t W, N, N_up, m;
    int64_t Np, S;
    float invd;                   // 1/delta in fp32 (the eval kernel's)
    double inv_delta;
    float *R;                     // [W][3][Np] in/out
    float *state;                 // [W][5][Np] in/out
    const int32_t *ks;            // [S][W]
    const float *delta;           // [S][W][3]
    const double *u;              // [S][W]
    int32_t *acc;                 // [S][W] out
    double *dj;                   // [S][W] out (dJ of each move) or NULL
    float L[3];
    double pcoef[2 * (QJ2_MAX_M + 1)][4];
    // optional one-body Jastrow over the electron-ion row (NEXT-1): the move's
    // ratio becomes exp(dJ1 + dJ2); the ions are fixed
    int32_t n_ions, n_species;
    int32_t sp_start[QJ2_MAX_SPECIES + 1];   // ions sorted by species
    int32_t sp_tab[QJ2_MAX_SPECIES];         // first row of species s in pcoef1
    int32_t sp_m[QJ2_MAX_SPECIES];
    int32_t n_rows1;                         // J1 table rows: sum over species of m_s + 1
    float sp_invd[QJ2_MAX_SPECIES];
    const float *ions;                       // [3][Np_ion]
    int64_t Np_ion;
    float *state_j1;                         // [W][5][Np]: electron e's U^1_e, grad, lap (k's row on acceptance)
    double pcoef1[QJ2_MAX_SPECIES * (QJ2_MAX_M + 1)][4];
};

constexpr int SW_MAX_IONS = 256;         // ions of the J1 part of a move (2-4 per thread)

cudaError_t launch_sweep(const SweepParams &p, cudaStream_t s);
// The 5N state (and, with ions, the J1 rows) of every electron from scratch
// (qj2_state_init): same SweepParams (S, ks, delta, u, acc, dj unused).
cudaError_t launch_state_init(const SweepParams &p, cudaStream_t s);

}  // namespace qj2
