// launch_accept.cu -- NEXT-2 accept-side update launches (own translation unit).
#include "accept.cuh"

// 256-bit loads / stores in the fp32 accept kernel when the rows are 32-byte aligned: the accept
// kernel of C3S 2.814 -> 2.749 ms (profiles/r02/ab_results.txt).  -DQJ2_ACCEPT_V8=0: 128-bit.
#ifndef QJ2_ACCEPT_V8
#define QJ2_ACCEPT_V8 1
#endif

namespace qj2 {

template <typename T>
static cudaError_t launch_accept(const AcceptParams &p0, void *r_old_ws, cudaStream_t s) {
    AcceptParams p = p0;
    if (!p.r_old) {            // gather r_k before any CTA may overwrite R[:, k]
        gather_rk_kernel<T><<<(unsigned)((p.W + 255) / 256), 256, 0, s>>>(p, static_cast<T *>(r_old_ws));
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        p.r_old = r_old_ws;
        p.r_old_stride = 3;
    }
    const int64_t nb = p.W * p.tiles_per_walker;
    // fp64 geometry when the functor grid is fine enough for fp32's relative
    // error in r to matter per entry (t = r/delta up to m; accept.cuh); fp64
    // positions are exact either way
    if (sizeof(T) == 4 && p.m > ACCEPT_FAST_MAX_M) j2_accept_kernel<T, true><<<(unsigned)nb, ATPB, 0, s>>>(p);
#if QJ2_ACCEPT_V8
    // fp32 rows 32-byte aligned: a thread's two vectors move with 256-bit loads and stores
    else if (sizeof(T) == 4 && p.Np % 8 == 0 && ((uintptr_t)p.R & 31) == 0 && ((uintptr_t)p.state & 31) == 0)
        j2_accept_kernel<T, false, sizeof(T) == 4><<<(unsigned)nb, ATPB, 0, s>>>(p);
#endif
    else                                           j2_accept_kernel<T, false><<<(unsigned)nb, ATPB, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_accept_f32(const AcceptParams &p, void *r_old_ws, cudaStream_t s) {
    return launch_accept<float>(p, r_old_ws, s);
}
cudaError_t launch_accept_f64(const AcceptParams &p, void *r_old_ws, cudaStream_t s) {
    return launch_accept<double>(p, r_old_ws, s);
}

}  // namespace qj2
