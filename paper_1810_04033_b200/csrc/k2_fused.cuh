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

// One fused single-sweep pass src -> dst writing only the slowest-axis planes
// [p.zlo, p.zhi) of dst (the slab runner's boundary / interior split).
// *handled = 0 when no streaming pass kernel covers this stencil and grid.
cudaError_t launch_one_pass(const KernelKey &key, const Params &p, const double *src, double *dst,
                            cudaStream_t st, int *handled);

// launch_one_pass with the peer stores of p.pdn / p.pup compiled in (k2_peer.cu)
cudaError_t launch_one_pass_peer(const KernelKey &key, const Params &p, const double *src, double *dst,
                                 cudaStream_t st);

}  // namespace sl
