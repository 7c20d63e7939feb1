#include "k2_fused.cuh"

namespace sl {

size_t fused_workspace_bytes(const KernelKey &, const Params &) { return 0; }

cudaError_t launch_fused(const KernelKey &, const Params &, int, double *, size_t, cudaStream_t,
                         int *handled) {
  *handled = 0;
  return cudaSuccess;
}

}  // namespace sl
