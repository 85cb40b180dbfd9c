// launch.cuh -- kernel launch templates (instantiated in launch_*.cu).
#pragma once

#include "qmcj2.h"
#include "j2_device.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "j2_kernels.cuh"
#include "j2_tma.cuh"

namespace qj2 {

// Kernel choice (A/B measurements only): QJ2_KERNEL=ldg1 (prefetch distance
// 1, 4 CTAs/SM) or tma323 (TMA-pipelined persistent kernel, 3 CTAs/SM, 2
// vectors per lane per stage, 3 stages); default: LDG kernel, prefetch 2.
struct TmaCfg { int minb, vpt, nst; };
constexpr TmaCfg kTmaCfgs[] = {{3, 2, 3}};
inline int kernel_choice() {   // -1 = LDG kernel, else index into kTmaCfgs
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
inline cudaError_t launch_tma(const EvalParams &p, int64_t nblocks, cudaStream_t s) {
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
inline bool use_warp_mapping(const EvalParams &p) {
    return p.tiles_per_walker == 1 && (p.W * p.n_groups >= 4096 || p.N_local <= 2048);
}

template <typename T, int PB, int MODE>
cudaError_t launch_eval(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s) {
    if constexpr (MODE == MODE_J1) {
        // small ion sets: one thread per (walker, trial), ions in shared memory
        if (!row && p.N_local <= J1_MAX_IONS && !getenv("QJ2_J1_WARP")) {
            const int64_t units = p.W * p.P;
            const size_t smem = (size_t)p.N_local * 4 * sizeof(T);
            auto kern = j1_thread_kernel<T>;
            if (smem > 48 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
            }
            kern<<<(unsigned)((units + TPB - 1) / TPB), TPB, smem, s>>>(p, units);
            return cudaGetLastError();
        }
    }
    if (use_warp_mapping(p)) {
        const int64_t units = p.W * p.n_groups;
        const unsigned nbw = (unsigned)((units + TPB / 32 - 1) / (TPB / 32));
        constexpr int MB = (sizeof(T) == 4 && PB == 1) ? 3 : 2;
        // fp32: three vector groups in flight per lane at 2 CTAs/SM (128 registers, no spills): on a
        // C4 wave 5.89 TB/s vs 5.31 for two groups at 3 CTAs/SM (80 registers, spilling), 5.51 for
        // four groups, 5.52 for one group at 4 CTAs/SM (profiles/r01_ab_sweep_s3.md).
        const char *wv = (MODE == MODE_J2 && sizeof(T) == 4) ? getenv("QJ2_WARP") : nullptr;   // A/B variants
        if (row) j2_eval_warp_kernel<T, PB, true, 1, 2, MODE><<<nbw, TPB, 0, s>>>(p, units);
        else if (wv && strcmp(wv, "p2m3") == 0) j2_eval_warp_kernel<T, PB, false, 2, 3, MODE><<<nbw, TPB, 0, s>>>(p, units);
        else if (sizeof(T) == 4) j2_eval_warp_kernel<T, PB, false, 3, 2, MODE><<<nbw, TPB, 0, s>>>(p, units);
        else     j2_eval_warp_kernel<T, PB, false, 2, MB, MODE><<<nbw, TPB, 0, s>>>(p, units);
        return cudaGetLastError();
    }
    const unsigned nb = (unsigned)nblocks;
    if constexpr (MODE == MODE_J2 && PB == 1) {
        if (!row && kernel_choice() == 0) return launch_tma<T, PB, 3, 2, 3>(p, nblocks, s);
    }
    constexpr int MB0 = (sizeof(T) == 4 && PB == 1) ? 4 : 2;
    if (row) {
        j2_eval_kernel<T, PB, true, 1, MB0, MODE><<<nb, TPB, 0, s>>>(p);
    } else if constexpr (PB == 1 && sizeof(T) == 4) {
        const char *e = getenv("QJ2_KERNEL");
        if (MODE == MODE_J2 && e && strcmp(e, "ldg1") == 0)   // A/B: prefetch distance 1, 4 CTAs/SM
            j2_eval_kernel<T, PB, false, 1, 4, MODE><<<nb, TPB, 0, s>>>(p);
        else if (MODE == MODE_J2 && e && strcmp(e, "p3m2") == 0)   // A/B: prefetch distance 3, 2 CTAs/SM
            j2_eval_kernel<T, PB, false, 3, 2, MODE><<<nb, TPB, 0, s>>>(p);
        else    // default: two vector groups in flight per thread, 3 CTAs/SM (80 registers);
                // measured best on B200
            j2_eval_kernel<T, PB, false, 2, 3, MODE><<<nb, TPB, 0, s>>>(p);
    } else if constexpr (PB == 1) {             // fp64: two groups in flight, 2 CTAs/SM
        j2_eval_kernel<T, PB, false, 2, 2, MODE><<<nb, TPB, 0, s>>>(p);
    } else {
        j2_eval_kernel<T, PB, false, 1, MB0, MODE><<<nb, TPB, 0, s>>>(p);
    }
    return cudaGetLastError();
}

// Per translation unit entry points (see launch_*.cu): <dtype>_<trial batch>_<mode>.
#define QJ2_DECL(NAME) \
    cudaError_t NAME(const EvalParams &p, int pb, int64_t nblocks, bool row, cudaStream_t s);
QJ2_DECL(launch_f32_pb1_j2) QJ2_DECL(launch_f64_pb1_j2) QJ2_DECL(launch_f32_pb1_j1) QJ2_DECL(launch_f64_pb1_j1)
#undef QJ2_DECL

}  // namespace qj2
