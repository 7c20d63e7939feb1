// plan.cuh — compile-time schedule of a colour-fused, temporally blocked
// streaming pass (K2).
//
// A pass applies K = m*c colour phases (m sweeps x c colours, phase k has
// colour k % c) while streaming planes along the slowest axis (z in 3D, y in
// 2D).  Phase k processes plane t - lag[k] at step t, phases in order within
// a step.  Exactness argument: a colour-k point at plane p
// reading a colour-b neighbour at plane p+dz must see the value written by
// the latest phase i<k of colour b and not yet the next one; with
// non-decreasing lags this holds iff lag[k] >= lag[i] + dz for that latest
// i (the "next writer" condition follows by symmetry of the stencil).
//
// Tiles are computed redundantly on a ghost margin: need[k][a] is how far
// beyond the owned box along axis a phase k must be correct so that the
// owned box ends bit-exact, obtained backwards from "each colour's last
// phase is correct on the owned box"; load[a] is the input margin that must
// be resident.  Only non-zero-weight offsets count (so Q1, which has no face
// neighbours, needs far less ghost than the full 27-point stencil).
#pragma once
#include "common.cuh"

namespace sl {

constexpr int MAXK = 16;

struct FPlan {
  int dim, K, C, lagmax;
  int colour[MAXK];
  int lag[MAXK];
  int need[MAXK][3];
  int load[3];
};

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cabs(int a) { return a < 0 ? -a : a; }

// colour of (point + o) = colour(point) ^ colour_flip(o)
__host__ __device__ constexpr int colour_flip(int colours, Off o) {
  const int fx = o.x & 1, fy = o.y & 1, fz = o.z & 1;
  return colours == 2 ? ((fx + fy + fz) & 1) : (fx | (fy << 1) | (fz << 2));
}

__host__ __device__ constexpr int off_axis(Off o, int a) { return a == 0 ? o.x : (a == 1 ? o.y : o.z); }

// Is colour a's point adjacent (through a non-zero offset with o.z == dz) to
// a colour-b point?
__host__ __device__ constexpr bool reads_at(int shape, int colours, int a, int b, int dz) {
  const int sa = shape_dim(shape) - 1;  // streaming axis
  for (int q = 0; q < shape_nnz(shape); ++q) {
    const Off o = shape_off(shape, q);
    if (off_axis(o, sa) == dz && (a ^ colour_flip(colours, o)) == b) return true;
  }
  return false;
}

// spread = true: additionally delay a phase until it cannot touch any phase
// processed in the same step — it neither reads a plane an earlier same-step
// phase writes nor writes one it reads — so all phases of a step are
// independent (3D CTA kernels: one block barrier per step; 2D warp strips:
// independent dependency chains the scheduler can interleave).  With 2^d colours a
// colour lives on planes of one parity, so two phases whose lags differ by
// the wrong parity are never active in the same step and cannot conflict.
__host__ __device__ constexpr FPlan make_plan(int shape, int colours, int m, bool spread = false) {
  FPlan P{};
  const int dim = shape_dim(shape);
  const int nnz = shape_nnz(shape);
  const int sa = dim - 1;  // streaming axis
  P.dim = dim;
  P.C = colours;
  P.K = m * colours;
  for (int k = 0; k < P.K; ++k) P.colour[k] = k % colours;
  for (int j = 0; j < P.K; ++j) {
    int L = j ? P.lag[j - 1] : 0;
    for (int q = 0; q < nnz; ++q) {
      const Off o = shape_off(shape, q);
      const int b = P.colour[j] ^ colour_flip(colours, o);
      for (int i = j - 1; i >= 0; --i)
        if (P.colour[i] == b) {
          L = cmax(L, P.lag[i] + off_axis(o, sa));
          break;
        }
    }
    if (spread) {
      for (bool moved = true; moved;) {
        moved = false;
        for (int i = 0; i < j; ++i) {
          const int d = L - P.lag[i];
          if (d < -1 || d > 1) continue;
          // a 2^d colour lives on planes (rows in 2D) of one parity along the streaming axis
          const int qi = (P.colour[i] >> sa) & 1, qj = (P.colour[j] >> sa) & 1;
          const bool coactive = colours == 2 || (((d - (qi - qj)) & 1) == 0);
          if (coactive && reads_at(shape, colours, P.colour[j], P.colour[i], d)) {
            ++L;
            moved = true;
            break;
          }
        }
      }
    }
    P.lag[j] = L;
  }
  P.lagmax = P.lag[P.K - 1];
  for (int k = 0; k < P.K; ++k)
    for (int a = 0; a < 3; ++a) P.need[k][a] = -1;
  for (int c = 0; c < colours; ++c)
    for (int k = P.K - 1; k >= 0; --k)
      if (P.colour[k] == c) {
        for (int a = 0; a < 3; ++a) P.need[k][a] = 0;
        break;
      }
  for (int a = 0; a < 3; ++a) P.load[a] = 0;
  for (int j = P.K - 1; j >= 0; --j) {
    if (P.need[j][0] < 0) continue;
    for (int q = 0; q < nnz; ++q) {
      const Off o = shape_off(shape, q);
      const int b = P.colour[j] ^ colour_flip(colours, o);
      int i = j - 1;
      while (i >= 0 && P.colour[i] != b) --i;
      for (int a = 0; a < 3; ++a) {
        const int req = P.need[j][a] + cabs(off_axis(o, a));
        if (i >= 0)
          P.need[i][a] = cmax(P.need[i][a], req);
        else
          P.load[a] = cmax(P.load[a], req);
      }
    }
  }
  for (int k = 0; k < P.K; ++k)
    for (int a = 0; a < 3; ++a)
      if (P.need[k][a] < 0) P.need[k][a] = 0;
  return P;
}

}  // namespace sl
