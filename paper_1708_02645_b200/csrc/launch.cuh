// launch.cuh -- kernel launch templates (instantiated in launch_*.cu).  One
// kernel variant per argument shape; the A/B alternatives measured against them
// are compile-time builds under tools/ab.
#pragma once

#include "qmcj2.h"
#include "j2_device.cuh"

#include "j2_kernels.cuh"

// fp32 pipeline depths and residency (A/B builds: -DQJ2_EVAL_PF=1 -DQJ2_EVAL_MINB=4 etc.)
#ifndef QJ2_EVAL_PF
#define QJ2_EVAL_PF 2          // CTA kernel: vector groups in flight per thread
#endif
#ifndef QJ2_EVAL_MINB
#define QJ2_EVAL_MINB 3        // CTA kernel: resident CTAs per SM
#endif
#ifndef QJ2_WARP_PF
#define QJ2_WARP_PF 3          // warp kernel
#endif
#ifndef QJ2_WARP_MINB
#define QJ2_WARP_MINB 2
#endif
#ifndef QJ2_EVAL64_PF
#define QJ2_EVAL64_PF 2        // fp64 CTA kernel
#endif
#ifndef QJ2_EVAL64_MINB
#define QJ2_EVAL64_MINB 2
#endif

namespace qj2 {

// Warp kernel, rows of < 4 sub-tiles (C1, C2, C2f64): every vector group of a sub-tile is loaded
// up front (PF = ITERS = 8, ~210 registers, 1 CTA/SM), so a walker's row costs one DRAM round
// trip per sub-tile instead of one per three groups: C1 10.5 -> 9.5 us, C2f64 23.4 -> 20.0 us,
// C2 unchanged (profiles/r02/ab_results.txt).  A/B builds: -DQJ2_WARP_SHORT_PF=n etc.
#ifndef QJ2_WARP_SHORT_PF
#define QJ2_WARP_SHORT_PF 8
#endif
#ifndef QJ2_WARP_SHORT_PF64
#define QJ2_WARP_SHORT_PF64 8
#endif
#ifndef QJ2_WARP_SHORT_MINB
#define QJ2_WARP_SHORT_MINB 1
#endif
// The clean fp32 sub-tiles of the CTA kernel and of the compact warp kernel read with 256-bit
// loads when the rows are 32-byte aligned: C3 1.105 -> 1.083 ms, C5 8.98 -> 8.87, C3P2 1.780 ->
// 1.753, C3P12 9.64 -> 9.55, a C4 wave 12.57 -> 12.17 ms (profiles/r02/ab_results.txt).
#ifndef QJ2_EVAL_V8
#define QJ2_EVAL_V8 1
#endif
#ifndef QJ2_WARP_V8
#define QJ2_WARP_V8 1
#endif
#ifndef QJ2_WARP_SHORT_N
#define QJ2_WARP_SHORT_N 2048  // rows this short take the warp kernel whatever W (A/B builds)
#endif

// Warp-per-walker mapping when a walker's slice is one CTA tile and there
// are enough (walker, trial) units to fill the GPU (or the slice is tiny).
inline bool use_warp_mapping(const EvalParams &p) {
    return p.tiles_per_walker == 1 && (p.W * p.P >= 4096 || p.N_local <= QJ2_WARP_SHORT_N);
}

// fp32 J2 functors finer than this take the fp64 geometry (term_prec): with the fp32 one,
// t = r/delta carries ~m 2^-23 of absolute error into the interval fraction, which U' and U''
// turn into ~m 2^-23 of the functor scale -- above the 1e-5 bar on single-term-dominated sums
// once m passes ~30 (the accept path's ACCEPT_FAST_MAX_M for the same reason).
constexpr int EVAL_FAST_MAX_M = 16;

template <typename T, int MODE, bool PREC>
cudaError_t launch_eval_impl(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s);

template <typename T, int MODE>
cudaError_t launch_eval(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s) {
    if constexpr (sizeof(T) == 4 && MODE == MODE_J2) {
        if (p.m > EVAL_FAST_MAX_M) return launch_eval_impl<T, MODE, true>(p, nblocks, row, s);
    }
    if constexpr (sizeof(T) == 4 && MODE == MODE_J1) {   // the small-ion kernel, a species finer than 16
        int mmax = 0;
        for (int g = 0; g < p.n_src_groups; ++g) mmax = p.grp_m[g] > mmax ? p.grp_m[g] : mmax;
        if (!row && p.N_local <= J1_MAX_IONS && mmax > EVAL_FAST_MAX_M)
            return launch_eval_impl<T, MODE, true>(p, nblocks, row, s);
    }
    return launch_eval_impl<T, MODE, false>(p, nblocks, row, s);
}

template <typename T, int MODE, bool PREC>
cudaError_t launch_eval_impl(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s) {
    if constexpr (MODE == MODE_J1) {
        // small ion sets: one thread per (walker, trial), ions in shared memory
        if (!row && p.N_local <= J1_MAX_IONS) {
            const int64_t units = p.W * p.P;
            const size_t smem = (size_t)p.N_local * 4 * sizeof(T);
            auto kern = j1_thread_kernel<T, PREC>;
            if (smem > 40 * 1024) {   // the static functor table (<= 2.2 KB) comes on top of the 48 KB default
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
            }
            kern<<<(unsigned)((units + TPB - 1) / TPB), TPB, smem, s>>>(p, units);
            return cudaGetLastError();
        }
    }
    if (use_warp_mapping(p)) {
        const int64_t units = p.W * p.P;
        const unsigned nbw = (unsigned)((units + TPB / 32 - 1) / (TPB / 32));
        // fp32: three vector groups in flight per lane at 2 CTAs/SM (128 registers, no spills): on a
        // C4 wave 5.89 TB/s vs 5.31 for two groups at 3 CTAs/SM (80 registers, spilling), 5.51 for
        // four groups, 5.52 for one group at 4 CTAs/SM (profiles/r01_ab_sweep_s3.md)
        if (row) j2_eval_warp_kernel<T, true, 1, 2, MODE, false, PREC><<<nbw, TPB, 0, s>>>(p, units);
        else if constexpr (sizeof(T) == 4) {
            if (p.N_local >= 4 * 32 * Traits<T>::VW * ITERS) {
#if QJ2_WARP_V8
                if (MODE == MODE_J2 && !PREC && p.Np % 8 == 0 && ((uintptr_t)p.R & 31) == 0)
                    j2_eval_warp_kernel<T, false, QJ2_WARP_PF, QJ2_WARP_MINB, MODE, true, false, true>
                        <<<nbw, TPB, 0, s>>>(p, units);
                else
#endif
                    j2_eval_warp_kernel<T, false, QJ2_WARP_PF, QJ2_WARP_MINB, MODE, true, PREC><<<nbw, TPB, 0, s>>>(p, units);
            }
            else
                j2_eval_warp_kernel<T, false, QJ2_WARP_SHORT_PF, QJ2_WARP_SHORT_MINB, MODE, false, PREC>
                    <<<nbw, TPB, 0, s>>>(p, units);
        } else if (p.N_local >= 4 * 32 * Traits<T>::VW * ITERS) {
            j2_eval_warp_kernel<T, false, 2, 2, MODE, true><<<nbw, TPB, 0, s>>>(p, units);
        } else {
            j2_eval_warp_kernel<T, false, QJ2_WARP_SHORT_PF64, QJ2_WARP_SHORT_MINB, MODE><<<nbw, TPB, 0, s>>>(p, units);
        }
        return cudaGetLastError();
    }
    const unsigned nb = (unsigned)nblocks;
    if (row)
        j2_eval_kernel<T, true, 1, sizeof(T) == 4 ? 4 : 2, MODE, PREC><<<nb, TPB, 0, s>>>(p);
    else if constexpr (sizeof(T) == 4)   // two vector groups in flight per thread, 3 CTAs/SM (80 registers):
                                         // measured best on B200 against distance 1 at 4 CTAs/SM and 3 at 2
    {
#if QJ2_EVAL_V8
        // 256-bit loads for the clean sub-tiles when every row starts 32-byte aligned
        if (MODE == MODE_J2 && !PREC && p.Np % 8 == 0 && ((uintptr_t)p.R & 31) == 0)
            j2_eval_kernel<T, false, QJ2_EVAL_PF, QJ2_EVAL_MINB, MODE, false, true><<<nb, TPB, 0, s>>>(p);
        else
#endif
            j2_eval_kernel<T, false, QJ2_EVAL_PF, QJ2_EVAL_MINB, MODE, PREC><<<nb, TPB, 0, s>>>(p);
    }
    else                                 // fp64: two groups in flight, 2 CTAs/SM (256-bit loads: slower, spills)
        j2_eval_kernel<T, false, QJ2_EVAL64_PF, QJ2_EVAL64_MINB, MODE><<<nb, TPB, 0, s>>>(p);
    return cudaGetLastError();
}

// Per translation unit entry points (see launch_*.cu): <dtype>_<mode>.
#define QJ2_DECL(NAME) cudaError_t NAME(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s);
QJ2_DECL(launch_f32_j2) QJ2_DECL(launch_f64_j2) QJ2_DECL(launch_f32_j1) QJ2_DECL(launch_f64_j1)
#undef QJ2_DECL

}  // namespace qj2
