// sweep.cuh -- NEXT-2 at the paper's system sizes: a whole particle-by-particle
// sweep of the J2 factor (optionally with J1) in one persistent kernel, the walker
// resident in shared memory (sm_100a).
//
// One CTA per walker.  For every move s < S (Alg. 1 L4-L9; electron
// k = ks[s][w], r_k = trials[s][w][0], r'_k = trials[s][w][1]):
//   1. each thread forms, for its partners i != k (i = tid, tid + TPB, ...), the
//      pair terms T_i at r_k and then at r'_k with the eval kernel's fp32
//      arithmetic (single-rounding minimum image, power-basis Horner) and keeps
//      only the differences T_i(r'_k) - T_i(r_k) in registers;
//   2. a reduce-scatter (fp32 for lanes 16 and 8 apart, then fp64) and ONE barrier
//      give dJ2 = sum_i (U(r'_k) - U(r_k)) and the sums at r'_k (electron k's new
//      state, Eq. 5 / PAPER:1382, Alg. 1 L7-L8); with J1 also dJ1 and k's J1 row;
//   3. every thread takes the same Metropolis decision u < exp(2 dJ) (reading R19);
//   4. if accepted: state_i += the kept differences (no recomputation), state_k =
//      the sums at r'_k, R[:, k] = r'_k.
// R and the 5N state stay in shared memory for all S moves (32 B per electron:
// N <= 1024 in 32 KB); global memory is touched only to load and store them once
// and to read the moves -- no launch per move.
#pragma once

#include "qmcj2.h"
#include "j2_device.cuh"

namespace qj2 {

constexpr int SW_TPB = 256;       // threads per walker (CTA)
constexpr int SW_SPT = 4;         // partners per thread: N <= SW_TPB * SW_SPT
constexpr int SW_MAXN = SW_TPB * SW_SPT;

struct SweepParams {
    int64_t W, N, N_up, Np, S;
    int32_t m;
    float invd;                   // 1/delta in fp32 (the eval kernel's)
    double inv_delta;
    float *R;                     // [W][3][Np] in/out
    float *state;                 // [W][5][Np] in/out
    const int32_t *ks;            // [S][W]
    const float *trials;          // [S][W][2][3]
    const double *u;              // [S][W]
    int32_t *acc;                 // [S][W] out
    double *dj;                   // [S][W] out (dJ2 of each move) or NULL
    float L[3];
    double pcoef[2 * (QJ2_MAX_M + 1)][4];
    // optional one-body Jastrow over the electron-ion row (NEXT-1): the move's
    // ratio becomes exp(dJ1 + dJ2); the ions are fixed (one per thread)
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

constexpr int SW_MAX_IONS = SW_TPB;      // one ion per thread in the J1 part of a move

cudaError_t launch_sweep(const SweepParams &p, cudaStream_t s);

}  // namespace qj2
