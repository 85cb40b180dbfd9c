// launch_f32_pbn_j1.cu -- kernel instantiations for one dtype / trial-batch size /
// mode (separate translation unit so the build compiles them in parallel).
#include "launch.cuh"

namespace qj2 {

cudaError_t launch_f32_pbn_j1(const EvalParams &p, int pb, int64_t nblocks, bool row, cudaStream_t s) {
    return pb == 2 ? launch_eval<float, 2, MODE_J1>(p, nblocks, row, s)
                   : launch_eval<float, MAXPB, MODE_J1>(p, nblocks, row, s);
}

}  // namespace qj2
