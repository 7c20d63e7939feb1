// k3_patch.cuh — K3: batched small patches, every sweep on chip.
//
// BASELINE config 5: B independent 18x18 grids (16x16 interior + a fixed
// halo), 5-point red-black sweeps.  The reference has no batch API (SURVEY
// D3); its semantics are "colouring applied per patch", each patch a Mesh of
// its own (colour parity relative to the patch's (1,1)).
//
// One warp owns one patch for the whole launch and keeps it in registers:
// lane l holds the column pair x = 2p+1, 2p+2 (p = l & 7) of rows
// y = 4g+1 .. 4g+4 (g = l >> 3) — 8 points of u and f — plus copies of the
// rows just above/below its group and of the halo columns it borders.  A
// colour phase updates one point per row per lane; the x-neighbour across
// the pair boundary comes from the adjacent lane (one shuffle per row), the
// y-neighbours from the lane's own rows or the cached boundary rows, which
// are refreshed from the groups above/below (two shuffles) after each phase.
// HBM traffic is one load of u, f and one store of u per launch, so the
// kernel is fp64-issue bound, not HBM bound.
#pragma once
#include "common.cuh"

namespace sl {

template <int FORM, bool UNIT, int DIV>
__device__ __forceinline__ double patch_update(double un, double ul, double ur, double us, double uc,
                                               double fc, const Params &p) {
  // canonical FD5 order: (0,-1), (-1,0), (1,0), (0,1)
  double acc = acc_init<FORM, UNIT>(uc, p);
  acc = acc_add<FORM, UNIT>(acc, un, 0, p);
  acc = acc_add<FORM, UNIT>(acc, ul, 1, p);
  acc = acc_add<FORM, UNIT>(acc, ur, 2, p);
  acc = acc_add<FORM, UNIT>(acc, us, 3, p);
  return acc_finish<FORM, UNIT, DIV>(acc, uc, fc, p);
}

template <int FORM, bool UNIT, int DIV>
__global__ void __launch_bounds__(256)
k3_patch16_fd5(Params p, int sweeps) {
  constexpr int S = 18;  // patch side incl. halo
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= p.batch) return;  // whole warp
  const int pp = lane & 7, g = lane >> 3;
  const int x0 = 2 * pp + 1, y0 = 4 * g + 1;
  double *u = p.u + b * p.bstride;
  const double *f = FORM == 1 ? p.f + b * p.bstride : nullptr;

  double U[4][2], F[4][2], A[2], B[2], HL[4], HR[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      U[r][j] = u[(y0 + r) * S + x0 + j];
      F[r][j] = FORM == 1 ? f[(y0 + r) * S + x0 + j] : 0.0;
    }
    HL[r] = u[(y0 + r) * S + 0];
    HR[r] = u[(y0 + r) * S + S - 1];
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    A[j] = u[(y0 - 1) * S + x0 + j];
    B[j] = u[(y0 + 4) * S + x0 + j];
  }

  for (int sw = 0; sw < sweeps; ++sw) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      // colour of (x, y) = (x + y - 2) & 1; with x0 odd the left column of row
      // r (y = 4g+1+r) has colour r & 1
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int j = ((r & 1) == c) ? 0 : 1;  // compile-time after unrolling
        double ul, ur;
        if (j == 0) {
          const double v = __shfl_up_sync(0xffffffffu, U[r][1], 1, 8);
          ul = pp == 0 ? HL[r] : v;
          ur = U[r][1];
        } else {
          const double v = __shfl_down_sync(0xffffffffu, U[r][0], 1, 8);
          ul = U[r][0];
          ur = pp == 7 ? HR[r] : v;
        }
        const double un = r == 0 ? A[j] : U[r - 1][j];
        const double us = r == 3 ? B[j] : U[r + 1][j];
        U[r][j] = patch_update<FORM, UNIT, DIV>(un, ul, ur, us, U[r][j], F[r][j], p);
      }
      // refresh the rows cached from the neighbouring groups (their colour-c
      // points changed); the outermost groups keep the fixed halo rows
      {
        const int j3 = ((3 & 1) == c) ? 0 : 1;  // changed column of row 3
        const int j0 = ((0 & 1) == c) ? 0 : 1;  // changed column of row 0
        const double up = __shfl_up_sync(0xffffffffu, U[3][j3], 8);
        const double dn = __shfl_down_sync(0xffffffffu, U[0][j0], 8);
        if (g > 0) A[j3] = up;
        if (g < 3) B[j0] = dn;
      }
    }
  }
  unsigned bad = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      bad |= ((unsigned)__double2hiint(U[r][j]) & 0x7ff00000u) == 0x7ff00000u;
      u[(y0 + r) * S + x0 + j] = U[r][j];
    }
  if (bad) atomicOr(p.status, 1);
}

}  // namespace sl
