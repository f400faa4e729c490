// complex64 tensor-map apply, 32-column tiles (apply27_tm.cuh)
#include "tm_launch.cuh"

namespace hz {
template cudaError_t launch_apply_tm_tx<32>(const TmLaunch&, const ApplyParams<float, float>&, int, bool, int, cudaStream_t);
}  // namespace hz
