// spo.cu -- NEXT-4 SPO evaluation launches (own translation unit).
#include "spo.cuh"

#include <algorithm>

#ifndef QJ2_SPO_RING_KB
#define QJ2_SPO_RING_KB 110
#endif

namespace qj2 {

template <bool VGH>
static cudaError_t launch_tma(const SpoParams &p, int nc, cudaStream_t s, bool *done) {
    *done = false;
    const size_t stage = (size_t)16 * p.ld * 4;
    const size_t per_stage = stage + SPO_HDR * 4 + 16;
    const size_t fixed = 2 * SPO_MAXC * 5 * sizeof(double) + 4 * 8 + 128;
    // ring budget per CTA: 110 KB = 2 CTAs/SM (4 plane stages each at 384 orbitals); measured on
    // B200 (S1 vgh): 220 KB / 1 CTA 1.77 ms, 110 KB 1.02 ms, 75 KB / 3 CTAs 1.05, 55 KB / 4 CTAs 1.19
    // (A/B builds: -DQJ2_SPO_RING_KB=n)
    const size_t budget = (size_t)QJ2_SPO_RING_KB * 1024;
    int nst = (int)std::min<size_t>(16, (budget - fixed) / per_stage);
    if (nst < 2) return cudaSuccess;                 // rows too long for a 2-stage ring: LDG kernel
    const size_t smem = (size_t)nst * per_stage + fixed;
    auto kern = spo_tma_kernel<VGH>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = (nc + 1) * 32;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>(p.W, (int64_t)sms * std::max(per_sm, 1));
    kern<<<(unsigned)grid, threads, smem, s>>>(p, nst);
    *done = true;
    return cudaGetLastError();
}

cudaError_t launch_spo(const SpoParams &p, bool vgh, bool force_ldg, cudaStream_t s) {
    const int64_t nc = (p.ld / (vgh ? spo_tma_nv<true>() : spo_tma_nv<false>()) + 31) / 32;
    if (!force_ldg && nc <= SPO_MAXC) {
        bool done = false;
        cudaError_t e = vgh ? launch_tma<true>(p, (int)nc, s, &done) : launch_tma<false>(p, (int)nc, s, &done);
        if (e != cudaSuccess || done) return e;
    }
    const unsigned threads = (unsigned)(p.tpw * p.wpc);
    const unsigned grid = (unsigned)((p.W + p.wpc - 1) / p.wpc);
    if (vgh) spo_kernel<true><<<grid, threads, 0, s>>>(p);
    else     spo_kernel<false><<<grid, threads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace qj2
