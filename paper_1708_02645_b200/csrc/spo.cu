// spo.cu -- NEXT-4 SPO evaluation launches (own translation unit).
#include "spo.cuh"

namespace qj2 {

cudaError_t launch_spo(const SpoParams &p, bool vgh, cudaStream_t s) {
    const unsigned threads = (unsigned)(p.tpw * p.wpc);
    const unsigned grid = (unsigned)((p.W + p.wpc - 1) / p.wpc);
    if (vgh) spo_kernel<true><<<grid, threads, 0, s>>>(p);
    else     spo_kernel<false><<<grid, threads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace qj2
