// launch_f64_pb1_j2.cu -- kernel instantiations for one dtype / trial-batch size /
// mode (separate translation unit so the build compiles them in parallel).
#include "launch.cuh"

namespace qj2 {

cudaError_t launch_f64_pb1_j2(const EvalParams &p, int pb, int64_t nblocks, bool row, cudaStream_t s) {
    (void)pb;
    return launch_eval<double, 1, MODE_J2>(p, nblocks, row, s);
}

}  // namespace qj2
