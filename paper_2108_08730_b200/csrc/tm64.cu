// complex64 tensor-map apply, 64-column tiles (apply27_tm.cuh)
#include "tm_launch.cuh"

namespace hz {
template cudaError_t launch_apply_tm_tx<64>(const TmLaunch&, const ApplyParams<float, float>&, int, bool, int, cudaStream_t);
}  // namespace hz
