// k1_colour.cuh — launchers of the per-colour (K1), indexed-update and
// residual kernels.
#pragma once
#include "dispatch.cuh"

namespace sl {

// Rows (b, z, y) visited by one colour phase; y = y0 + yi*ystep, z likewise.
struct RowMap {
  int64_t rows, cy, cz, y0, z0, ystep, zstep;
};

// colour < 0: every interior point in one racy pass (negative control only).
cudaError_t launch_colour_pass(const KernelKey &key, const Params &p, int colour, cudaStream_t st);
// one lexicographic Gauss-Seidel sweep (hyperplane wavefronts)
cudaError_t launch_lex_sweep(const KernelKey &key, const Params &p, cudaStream_t st);
cudaError_t launch_update_cells(const KernelKey &key, const Params &p, const int64_t *flats,
                                int64_t count, cudaStream_t st);
cudaError_t launch_residual(const KernelKey &key, const Params &p, double *d_out, cudaStream_t st);

}  // namespace sl
