// k2_strip2d.cuh — K2 for 2D grids: warp-private strip streaming.
//
// One warp owns a strip of 64 columns (lane i holds the column pair
// 2i, 2i+1) and a chunk of rows, and streams the rows through a ring of
// registers: no shared memory, no block barriers, warps fully independent.
// The strip overlaps its neighbours by the ghost margin GX on each side, so
// only TX = 64 - 2*GX columns are owned; x+-1 neighbours of the lane's point
// come from its own pair or, across the pair boundary, from the adjacent
// lane by one warp shuffle.
//
// Phase k processes row t - lag[k] at step t (plan.cuh).  The step loop is
// unrolled by the ring length NR with the row parity of every ring slot
// fixed at compile time, so each phase's colour pattern (which rows hold
// the colour, which x parity its points have) and every ring index are
// compile-time: inactive phases vanish, the hot loop is loads, shuffles and
// fp64 arithmetic.  Rows are prefetched D steps ahead (16-byte LDG per lane).
#pragma once
#include "plan.cuh"

namespace sl {

template <int S, int M>
struct GeoS2 {
  static constexpr FPlan P = make_plan(S, S == FE9 ? 4 : 2, M);
  static constexpr int K = P.K, C = P.C, LAGMAX = P.lagmax;
  static constexpr bool RB = (P.C == 2);
  static constexpr int GX = (P.load[0] + 1) & ~1;
  static constexpr int GY = P.load[1];
  static constexpr int TX = 64 - 2 * GX;
  static constexpr int D = 4;  // prefetch distance (rows)
  static constexpr int NR0 = LAGMAX + 3 + D;
  static constexpr int NR = (NR0 + 1) & ~1;  // even, so slot parity is fixed
  static constexpr int WPB = 4;              // warps per block
  // does the stencil use offset (dx, dy)?
  static constexpr bool uses(int dx, int dy) {
    for (int q = 0; q < shape_nnz(S); ++q) {
      const Off o = shape_off(S, q);
      if (o.x == dx && o.y == dy) return true;
    }
    return false;
  }
};

__device__ __forceinline__ double2 ldg_stream2(const double *p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_pair(double *p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

// Markstein-corrected division for the hot loop: the fallback runs only for
// lanes whose result is used (ghost lanes may hold zeros or garbage).
template <int DIV>
__device__ __forceinline__ double div_wc_lane(double a, bool used, const Params &p) {
  if (DIV == DIV_POW2) return __dmul_rn(a, p.rwc);
  if (DIV == DIV_RCP) {
    const unsigned e = ((unsigned)__double2hiint(a) >> 20) & 0x7ffu;
    const double q0 = __dmul_rn(a, p.rwc);
    const double r = __fma_rn(-p.wc, q0, a);
    double q = __fma_rn(r, p.rwc, q0);
    if (used && (e - 64u) >= 1918u) q = __ddiv_rn(a, p.wc);  // |a| outside [2^-959, 2^959)
    return q;
  }
  return __ddiv_rn(a, p.wc);
}

template <int S, int FORM, bool UNIT, int DIV, int M>
__global__ void __launch_bounds__(32 * GeoS2<S, M>::WPB)
k2_strip2d(Params p, const double *__restrict__ src, double *__restrict__ dst, int64_t nstrip,
           int64_t nchunk) {
  using G = GeoS2<S, M>;
  constexpr FPlan P = G::P;
  constexpr int NR = G::NR;
  constexpr int NNZ = shape_nnz(S);
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * G::WPB + (threadIdx.x >> 5);
  if (wid >= nstrip * nchunk) return;
  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2;
  const int nx = (int)p.nx, ny = (int)p.ny;
  const int strip = (int)(wid % nstrip), chunk = (int)(wid / nstrip);
  const int x0 = (int)(2 * (((int64_t)strip * (Sx / 2)) / nstrip));
  const int x1 = (int)(2 * (((int64_t)(strip + 1) * (Sx / 2)) / nstrip));
  const int y0 = (int)(((int64_t)chunk * Sy) / nchunk), y1 = (int)(((int64_t)(chunk + 1) * Sy) / nchunk);
  const int TXo = x1 - x0;
  const int gx = x0 - G::GX + 2 * lane;  // global x of the lane's even column
  const bool in_x = gx >= 0 && gx < Sx;
  const bool own_x = 2 * lane >= G::GX && 2 * lane < G::GX + TXo;

  // rows of slot 0 have (row - 1 + py) even
  int t_begin = y0 - G::GY - 1;
  if ((t_begin - 1 + p.py) & 1) --t_begin;
  const int t_end = y1 - 1 + G::LAGMAX;
  const int ylim = y1 + G::GY;  // rows >= ylim are never needed

  // per-phase row window and lane validity
  int rlo[G::K], rhi[G::K];
#pragma unroll
  for (int j = 0; j < G::K; ++j) {
    rlo[j] = max(1, y0 - P.need[j][1]);
    rhi[j] = min(ny, y1 - 1 + P.need[j][1]);
  }

  double ulo[NR], uhi[NR], flo[NR], fhi[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) ulo[k] = uhi[k] = flo[k] = fhi[k] = 0.0;

  auto load_row = [&](int row, double &lo, double &hi, double &fl, double &fh) {
    if (row >= 0 && row < Sy && row < ylim && in_x) {
      const int64_t g = (int64_t)row * p.sy + gx;
      const double2 u = ldg_stream2(src + g);
      lo = u.x;
      hi = u.y;
      if (FORM == 1) {
        const double2 f = ldg_stream2(p.f + g);
        fl = f.x;
        fh = f.y;
      }
    }
  };
#pragma unroll
  for (int k = 1; k <= G::D; ++k) load_row(t_begin + k, ulo[k], uhi[k], flo[k], fhi[k]);

  unsigned bad = 0;
  for (int t0 = t_begin; t0 <= t_end; t0 += NR) {
    [&]<int... Ks>(std::integer_sequence<int, Ks...>) {
      (
          [&] {
            constexpr int KS = Ks;  // ring slot of row t
            const int t = t0 + KS;
            {
              constexpr int L = (KS + G::D + 1) % NR;
              load_row(t + G::D + 1, ulo[L], uhi[L], flo[L], fhi[L]);
            }
            // ---- phases in order ----
            [&]<int... Js>(std::integer_sequence<int, Js...>) {
              (
                  [&] {
                    constexpr int J = Js;
                    constexpr int c = P.colour[J];
                    constexpr int R0 = ((KS - P.lag[J]) % NR + NR) % NR;
                    constexpr int RM = (R0 + NR - 1) % NR, RP = (R0 + 1) % NR;
                    constexpr int qy = (KS - P.lag[J]) & 1;  // parity of the row being updated
                    if constexpr (!G::RB && qy != ((c >> 1) & 1)) {
                      return;  // colour absent from this row
                    } else {
                      constexpr int s = 1 ^ (G::RB ? ((c + qy) & 1) : (c & 1));  // x parity
                      const int row = t - P.lag[J];
                      if (row < rlo[J] || row > rhi[J]) return;
                      const int lx = 2 * lane + s;
                      const bool valid = lx >= G::GX - P.need[J][0] && lx < G::GX + TXo + P.need[J][0] &&
                                         gx + s >= 1 && gx + s <= nx;
                      // neighbour values v[dy+1][dx+1]
                      double v[3][3];
                      constexpr int RR[3] = {RM, R0, RP};
#pragma unroll
                      for (int dy = 0; dy < 3; ++dy) {
                        const double lo = ulo[RR[dy]], hi = uhi[RR[dy]];
                        const bool need_l = G::uses(-1, dy - 1), need_r = G::uses(1, dy - 1);
                        if (s == 0) {
                          v[dy][0] = need_l ? __shfl_up_sync(0xffffffffu, hi, 1) : 0.0;
                          v[dy][1] = lo;
                          v[dy][2] = hi;
                        } else {
                          v[dy][0] = lo;
                          v[dy][1] = hi;
                          v[dy][2] = need_r ? __shfl_down_sync(0xffffffffu, lo, 1) : 0.0;
                        }
                      }
                      const double uc = v[1][1];
                      double acc = acc_init<FORM, UNIT>(uc, p);
#pragma unroll
                      for (int q = 0; q < NNZ; ++q) {
                        const Off o = shape_off(S, q);
                        acc = acc_add<FORM, UNIT>(acc, v[o.y + 1][o.x + 1], q, p);
                      }
                      double out;
                      if (FORM == 0) {
                        out = div_wc_lane<DIV>(acc, valid, p);
                      } else {
                        const double fc = s == 0 ? flo[R0] : fhi[R0];
                        const double qd = div_wc_lane<DIV>(__dsub_rn(fc, acc), valid, p);
                        out = __dadd_rn(uc, __dmul_rn(p.omega, qd));
                      }
                      if (valid) {
                        bad |= ((unsigned)__double2hiint(out) & 0x7ff00000u) == 0x7ff00000u;
                        if (s == 0)
                          ulo[R0] = out;
                        else
                          uhi[R0] = out;
                      }
                    }
                  }(),
                  ...);
            }(std::make_integer_sequence<int, G::K>{});
            // ---- row t - LAGMAX is final ----
            {
              constexpr int RO = ((KS - G::LAGMAX) % NR + NR) % NR;
              const int row = t - G::LAGMAX;
              if (row >= y0 && row < y1 && own_x)
                stg_pair(dst + (int64_t)row * p.sy + gx, ulo[RO], uhi[RO]);
            }
          }(),
          ...);
    }(std::make_integer_sequence<int, NR>{});
  }
  if (bad) atomicOr(p.status, 1);
}

}  // namespace sl
