// k4_block2d.cuh — K2 variant for small 2D grids: overlapped temporal tiling
// entirely in shared memory.
//
// BASELINE config 1 (FD5, 1026^2, 100 sweeps) is 8.4 MB per array: it lives
// in L2 and a streaming pass is latency-bound.  Here a CTA loads its tile of
// u and f plus the ghost margin of M fused sweeps (plan.cuh: the margin
// shrinks by the dependency radius phase by phase) into shared memory once,
// runs all M*c colour phases there (one block barrier per phase), and writes
// the owned part back — one wave of CTAs per pass, ping-pong between u and
// the workspace like every K2 pass.  Rows are stored de-interleaved by x
// parity so a warp updating one colour and its x+-1 neighbours hits
// consecutive words; warp items reuse update_item() from k2_fused.cu.
#pragma once
#include "plan.cuh"

namespace sl {

template <int S, int M>
struct GeoB2 {
  static constexpr FPlan P = make_plan(S, S == FE9 ? 4 : 2, M);
  static constexpr int K = P.K, C = P.C;
  static constexpr bool RB = (P.C == 2);
  static constexpr int GX = (P.load[0] + 1) & ~1;
  static constexpr int GY = P.load[1];
  static constexpr int NSTRIP = 2;
  static constexpr int PX = 64 * NSTRIP;     // tile width incl. ghost (columns)
  static constexpr int HW = PX / 2 + 2;
  static constexpr int ROWW = 2 * HW;
  static constexpr int PY = 96;              // max tile height incl. ghost (rows)
  static constexpr int TX = PX - 2 * GX;     // max owned width
  static constexpr int TY = PY - 2 * GY;     // max owned height
  static constexpr int RSTEP = RB ? 1 : 2;
  static constexpr int RY = 2;              // point rows per warp item (4: 186 vs 205 GLUP/s on config 1)
  static constexpr int NT = 1024;
  static constexpr int NW = NT / 32;
  static constexpr int PAD_ROWS = (RY - 1) * RSTEP + 2;   // items may read past the last row
  static constexpr int LEAD = 2;                          // ... and one row before the first
  static constexpr int UOFF = LEAD * ROWW;
  static constexpr int FOFF = UOFF + (PY + PAD_ROWS + LEAD) * ROWW;
  static constexpr size_t SMEM = size_t(2 * (PY + PAD_ROWS + LEAD) * ROWW) * sizeof(double);
  static_assert(SMEM <= 227 * 1024, "tile exceeds shared memory");
};

template <int S, int FORM, bool UNIT, int DIV, int M>
__global__ void __launch_bounds__(GeoB2<S, M>::NT, 1)
k4_block2d(Params p, const double *__restrict__ src, double *__restrict__ dst, int ntx, int nty) {
  using G = GeoB2<S, M>;
  constexpr FPlan P = G::P;
  extern __shared__ double sm[];
  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2;
  const int nx = (int)p.nx, ny = (int)p.ny;
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const int x0 = 2 * ((tx * (Sx / 2)) / ntx), x1 = 2 * (((tx + 1) * (Sx / 2)) / ntx);
  const int y0 = (ty * Sy) / nty, y1 = ((ty + 1) * Sy) / nty;
  const int TXo = x1 - x0, TYo = y1 - y0;
  const int gx0 = x0 - G::GX, gy0 = y0 - G::GY;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sy = (int)p.sy;

  // ---- load the tile (u and f) de-interleaved: 16-byte loads, two 8-byte stores ----
  const int rows = TYo + 2 * G::GY;
  for (int k = tid; k < rows * (G::PX / 2); k += G::NT) {
    const int r = k / (G::PX / 2), i = k % (G::PX / 2);
    const int gx = gx0 + 2 * i, gy = gy0 + r;
    double2 u2 = make_double2(0.0, 0.0), f2 = make_double2(0.0, 0.0);
    if (gy >= 0 && gy < Sy && gx >= 0 && gx < Sx) {
      u2 = *reinterpret_cast<const double2 *>(src + (int64_t)gy * sy + gx);
      if (FORM == 1) f2 = __ldg(reinterpret_cast<const double2 *>(p.f + (int64_t)gy * sy + gx));
    }
    sm[G::UOFF + r * G::ROWW + 1 + i] = u2.x;
    sm[G::UOFF + r * G::ROWW + G::HW + 1 + i] = u2.y;
    if (FORM == 1) {
      sm[G::FOFF + r * G::ROWW + 1 + i] = f2.x;
      sm[G::FOFF + r * G::ROWW + G::HW + 1 + i] = f2.y;
    }
  }
  __syncthreads();

  unsigned bad = 0;
  // ---- all M*c phases on the tile ----
  [&]<int... Js>(std::integer_sequence<int, Js...>) {
    (
        [&] {
          constexpr int J = Js;
          constexpr int c = P.colour[J];
          constexpr int nx_ = P.need[J][0], ny_ = P.need[J][1];
          int r_lo = G::GY - ny_, r_hi = G::GY + TYo + ny_;  // tile rows [lo, hi)
          if (gy0 + r_lo < 1) r_lo = 1 - gy0;
          if (gy0 + r_hi > ny + 1) r_hi = ny + 1 - gy0;
          const int r_first = r_lo;
          // item rows start on the parity whose points have local x parity S0
          const int want_qy = G::RB ? ((1 + c) & 1) : ((c >> 1) & 1);
          if (((gy0 + r_lo - 1 + p.py) & 1) != want_qy) --r_lo;
          constexpr int S0 = G::RB ? 0 : (1 ^ (c & 1));
          const int npr = r_hi > r_lo ? (r_hi - r_lo + G::RSTEP - 1) / G::RSTEP : 0;
          const int ngrp = (npr + G::RY - 1) / G::RY;
          const int lx_lo = G::GX - nx_, lx_hi = G::GX + TXo + nx_;
          for (int it = warp; it < ngrp * G::NSTRIP; it += G::NW) {
            const int strip = it % G::NSTRIP;
            const int row0 = r_lo + (it / G::NSTRIP) * G::RY * G::RSTEP;
            const int li = strip * 32 + lane;
            unsigned vmask = 0;
#pragma unroll
            for (int r = 0; r < G::RY; ++r) {
              const int s = G::RB ? (S0 ^ ((r * G::RSTEP) & 1)) : S0;
              const int lx = 2 * li + s, gx = gx0 + lx, row = row0 + r * G::RSTEP;
              const bool v = row >= r_first && row < r_hi && lx >= lx_lo && lx < lx_hi && gx >= 1 && gx <= nx;
              vmask |= (unsigned)v << r;
            }
            const int rb = G::UOFF + (row0 - 1) * G::ROWW + li;
            auto ro = [&](int, int k) -> int { return rb + k * G::ROWW; };
            auto fv = [&](int r, int s) -> double {
              return sm[G::FOFF - G::UOFF + rb + (r * G::RSTEP + 1) * G::ROWW + xoff<G::HW>(s, 0)];
            };
            bad |= update_item<S, FORM, UNIT, DIV, G::RY, G::RSTEP, G::RB, G::HW, S0>(ro, fv, vmask, p);
          }
          __syncthreads();
        }(),
        ...);
  }(std::make_integer_sequence<int, G::K>{});

  // ---- owned part -> dst ----
  for (int k = tid; k < TYo * (TXo / 2); k += G::NT) {
    const int r = G::GY + k / (TXo / 2), i = G::GX / 2 + k % (TXo / 2);
    const double a = sm[G::UOFF + r * G::ROWW + 1 + i], b = sm[G::UOFF + r * G::ROWW + G::HW + 1 + i];
    // (non-finite updates were flagged by update_item as they happened)
    stg2(dst + (int64_t)(gy0 + r) * sy + gx0 + 2 * i, a, b);
  }
  if (bad) atomicOr(p.status, 1);
}

}  // namespace sl
