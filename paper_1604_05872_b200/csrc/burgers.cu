// burgers.cu -- Burgers Jacobian element kernel (BASELINE config 5).  Placeholder
// until the tensor-schedule kernel lands.
#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

bool burgers_supported(int, int) { return false; }

cudaError_t launch_burgers(int, long, const double*, const double*, const double*, double, double,
                           double*, int, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace femgpu
