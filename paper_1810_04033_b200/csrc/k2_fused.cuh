// k2_fused.cuh — colour-fused, temporally blocked sweep driver (K2) and the
// batched-patch kernel (K3).
#pragma once
#include "dispatch.cuh"

namespace sl {

size_t fused_workspace_bytes(const KernelKey &key, const Params &p);

// Runs `sweeps` sweeps with the fused kernels when they apply; *handled = 0
// leaves the work to the per-colour path.
cudaError_t launch_fused(const KernelKey &key, const Params &p, int sweeps, double *workspace,
                         size_t workspace_bytes, cudaStream_t st, int *handled, bool stream_only);

}  // namespace sl
