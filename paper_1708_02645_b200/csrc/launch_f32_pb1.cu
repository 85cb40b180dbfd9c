// launch_f32_pb1.cu -- kernel instantiations for one dtype / trial-batch
// size (separate translation unit so the build compiles them in parallel).
#include "launch.cuh"

namespace qj2 {

cudaError_t launch_f32_pb1(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s) {
    return launch_eval<float, 1>(p, nblocks, row, s);
}

}  // namespace qj2
