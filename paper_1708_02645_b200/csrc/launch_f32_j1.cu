// launch_f32_j1.cu -- kernel instantiations for one dtype / mode (separate
// translation unit so the build compiles them in parallel).
#include "launch.cuh"

namespace qj2 {

cudaError_t launch_f32_j1(const EvalParams &p, int64_t nblocks, bool row, cudaStream_t s) {
    return launch_eval<float, MODE_J1>(p, nblocks, row, s);
}

}  // namespace qj2
