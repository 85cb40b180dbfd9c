// launch_f64_pbn_j2.cu -- kernel instantiations for one dtype / trial-batch size /
// mode (separate translation unit so the build compiles them in parallel).
#include "launch.cuh"

namespace qj2 {

cudaError_t launch_f64_pbn_j2(const EvalParams &p, int pb, int64_t nblocks, bool row, cudaStream_t s) {
    return pb == 2 ? launch_eval<double, 2, MODE_J2>(p, nblocks, row, s)
                   : launch_eval<double, MAXPB, MODE_J2>(p, nblocks, row, s);
}

}  // namespace qj2
