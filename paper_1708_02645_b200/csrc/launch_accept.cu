// launch_accept.cu -- NEXT-2 accept-side update launches (own translation unit).
#include "accept.cuh"

namespace qj2 {

template <typename T>
static cudaError_t launch_accept(const AcceptParams &p0, void *r_old_ws, cudaStream_t s) {
    AcceptParams p = p0;
    if (!p.r_old) {            // gather r_k before any CTA may overwrite R[:, k]
        gather_rk_kernel<T><<<(unsigned)((p.W + 255) / 256), 256, 0, s>>>(p, static_cast<T *>(r_old_ws));
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        p.r_old = r_old_ws;
    }
    const int64_t nb = p.W * p.tiles_per_walker;
    j2_accept_kernel<T><<<(unsigned)nb, ATPB, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_accept_f32(const AcceptParams &p, void *r_old_ws, cudaStream_t s) {
    return launch_accept<float>(p, r_old_ws, s);
}
cudaError_t launch_accept_f64(const AcceptParams &p, void *r_old_ws, cudaStream_t s) {
    return launch_accept<double>(p, r_old_ws, s);
}

}  // namespace qj2
