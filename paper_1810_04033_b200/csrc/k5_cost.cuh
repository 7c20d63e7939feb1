// k5_cost.cuh — cost-model updates (k > 0 sine work per stencil entry).
#pragma once
#include "dispatch.cuh"

namespace sl {

struct CostSpec {
  int ramp;      // 0: every cell k; 1: k = min(100*rank/total, 99), rank = lex rank
  int k;
  double *work;  // device accumulator for the consumed sine tally (may be null)
};

// one colour phase (colour >= 0) or one lexicographic sweep (colour < 0)
cudaError_t launch_cost_sweep_phase(const KernelKey &key, const Params &p, const CostSpec &c,
                                    int colour, cudaStream_t st);
// indexed cells (update_cells_batch) of grid 0, constant k
cudaError_t launch_cost_cells(const KernelKey &key, const Params &p, const CostSpec &c,
                              const int64_t *flats, int64_t count, cudaStream_t st);

}  // namespace sl
