// k2_q1col.cuh — K2 for the trilinear Q1 27-point operator (BASELINE config 4).
//
// Q1 has no face neighbours (their weights are 0), so a point's 20 neighbours
// are the 8 columns around it on planes z+-1 and the 4 diagonal columns on its
// own plane; the 2x2x2 parity colouring gives 8 colours.  Lags are spread
// (plan.cuh: 0,0,1,1,3,3,4,4) so the colour groups active in one step —
// {0,1}@t with {4,5}@t-3 on even steps, {2,3}@t-1 with {6,7}@t-4 on odd
// ones — are mutually independent: one block barrier per step.
//
// A CTA owns a 64 x 48 (x, y) tile (+ the ghost margin 4/4/2 of the plan) and
// a chunk of z; 12 warps.  Thread (warp w, lane i) owns column pair (2i, 2i+1)
// of the RT = 4 tile rows r0 = 4w + delta .. r0 + 3, where delta makes row r0
// a y-parity 0 row: a colour group updates all columns of every other row, so
// each thread updates 2 x 2 points (rows A, A + 2) per group.
//
// Every plane of the tile lives in a shared-memory slot that is always
// current (TMA fills it, each owner publishes its updates).  The "young"
// group of a step (lag 0 or 1) reads the thread's own rows from a register
// ring holding planes t-2 .. t+1 and only the row of the warp above/below from
// shared memory; the "old" group (lag 3 or 4) reads all its rows from shared
// memory.  x+-1 columns come from warp shuffles.  Results are published to the
// slot after both groups of the step have read their inputs.
//
// u planes arrive by TMA (64 x 49 x 1 boxes, zero-filled out of range) into
// 8 smem slots, issued two planes ahead.  The step loop is unrolled by 4 (the
// register ring length), so ring indices are compile-time; slot offsets and
// mbarrier parities are cheap runtime values.  Out-of-range groups and ghost
// points are computed and masked (no branches around the shuffles); the exact
// division fallback runs out of line, per warp, only when a used lane's
// operand leaves the fast range.
#pragma once
#include <cuda.h>

#include "plan.cuh"


namespace sl {

// Exact division out of line: the rare fallback of the Markstein fast path
// must not bloat the unrolled step loop (instruction-cache pressure).
__device__ __noinline__ double q1_div_exact(double a, double b) { return __ddiv_rn(a, b); }

struct Q1Geo {
  static constexpr FPlan P = make_plan(Q1, 8, 1, true);
  static constexpr int LAGMAX = P.lagmax;                 // 4
  static constexpr int GX = 4, GY = 4, GZ = 2;            // plan load margins
  static constexpr int PX = 64, PY = 48;                  // tile incl. ghost
  static constexpr int BOXY = PY + 1;                     // rows loaded (delta shift)
  static constexpr int TX = PX - 2 * GX, TY = PY - 2 * GY;
  static constexpr int S = 8;                             // smem slots
  static constexpr int RR = 4;                            // register ring = unroll
  static constexpr int RT = 4;                            // tile rows per thread
  static constexpr int NT = 32 * PY / RT;                 // 384
  static constexpr int SLOTE = PX * BOXY;
  static constexpr int LEADE = 2 * PX;                    // guard rows before slot 0
  static constexpr size_t SMEM = size_t(LEADE + S * SLOTE + 2 * PX) * sizeof(double) + S * 8;
  static_assert(P.lag[0] == 0 && P.lag[2] == 1 && P.lag[4] == 3 && P.lag[6] == 4, "unexpected plan");
  static_assert(P.lag[1] == P.lag[0] && P.lag[3] == P.lag[2] && P.lag[5] == P.lag[4] &&
                    P.lag[7] == P.lag[6], "colour pairs share a lag");
  static_assert(P.load[0] <= GX && P.load[1] <= GY && P.load[2] <= GZ, "ghost margin");
  // planes t-5 .. t+1 are read at step t and plane t+2 is in flight
  static_assert(S >= LAGMAX + 4, "too few slots");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// group of step parity Q: GI 0 = young (lag 0 / 1), GI 1 = old (lag 3 / 4)
__host__ __device__ constexpr int q1_group(int Q, int GI) { return Q == 0 ? (GI == 0 ? 0 : 4) : (GI == 0 ? 2 : 6); }

template <int FORM, bool UNIT, int DIV>
__global__ void __launch_bounds__(Q1Geo::NT, 1)
k2_q1col(Params p, const __grid_constant__ CUtensorMap tmu, double *__restrict__ dst, int64_t ntx,
         int64_t nty, int64_t nzc) {
  using G = Q1Geo;
  constexpr FPlan P = G::P;
  constexpr int RT = G::RT, H = RT / 2, RR = G::RR;
  extern __shared__ __align__(128) double qsm[];
  double *su = qsm + G::LEADE;  // slot k at su + k*SLOTE
  uint64_t *mb = reinterpret_cast<uint64_t *>(su + G::S * G::SLOTE + 2 * G::PX);
  const uint32_t su_s = (uint32_t)__cvta_generic_to_shared(su);
  const uint32_t mb_s = (uint32_t)__cvta_generic_to_shared(mb);

  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2, Sz = (int)p.nz + 2;
  const int nx = (int)p.nx, ny = (int)p.ny, nz = (int)p.nz;
  const int item = blockIdx.x;
  const int tx = item % (int)ntx, ty = (item / (int)ntx) % (int)nty, zc = item / (int)(ntx * nty);
  const int x0 = (int)(2 * (((int64_t)tx * (Sx / 2)) / ntx)), x1 = (int)(2 * (((int64_t)(tx + 1) * (Sx / 2)) / ntx));
  const int y0 = (int)(((int64_t)ty * Sy) / nty), y1 = (int)(((int64_t)(ty + 1) * Sy) / nty);
  const int z0 = (int)(((int64_t)zc * Sz) / nzc), z1 = (int)(((int64_t)(zc + 1) * Sz) / nzc);
  const int TXo = x1 - x0, TYo = y1 - y0;
  const int gx0 = x0 - G::GX, gy0 = y0 - G::GY;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx = gx0 + 2 * lane;
  const int delta = (1 - p.py - gy0) & 1;        // local row r0 has y parity 0
  const int r0 = RT * warp + delta;              // this thread's rows r0 (qy 0) .. r0 + RT - 1
  const int64_t sz = p.sz;

  int t_begin = z0 - G::GZ - 1;
  if ((t_begin - 1 + p.pz) & 1) --t_begin;       // plane parity of step k is k & 1
  const int t_end = z1 - 1 + G::LAGMAX;
  const int zlim = z1 + G::GZ;
  const int base = t_begin + 1;                  // plane held by slot 0 in use 0

  auto issue = [&](int plane) {
    const int sl = (plane - base) & (G::S - 1);
    const uint32_t bar = mb_s + 8u * sl;
    const bool live = plane >= 0 && plane < Sz && plane < zlim;
    mbar_expect3(bar, live ? (uint32_t)(G::SLOTE * 8) : 0u);
    if (live) tma_load_3d(su_s + sl * G::SLOTE * 8, &tmu, gx0, gy0, plane, bar);
  };

  if (threadIdx.x == 0) {
    for (int k = 0; k < G::S; ++k) mbar_init3(mb_s + 8u * k);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    issue(base);
    issue(base + 1);
  }
  __syncthreads();

  // ---- thread-constant masks ------------------------------------------------
  // ok bit (4*gi + 2*h + s): point s of the h-th row (A + 2h) of group gi
  // (J = 2*gi) is inside the group's need region and the grid interior (x, y)
  unsigned okbits = 0;
#pragma unroll
  for (int gi = 0; gi < 4; ++gi) {
    const int J = 2 * gi;
    const int A = (P.colour[J] >> 1) & 1;
    const int nxj = P.need[J][0], nyj = P.need[J][1];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int r = r0 + A + 2 * h, gy = gy0 + r;
      const bool rok = r >= G::GY - nyj && r < G::GY + TYo + nyj && gy >= 1 && gy <= ny;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int lx = 2 * lane + s;
        const bool cok = lx >= G::GX - nxj && lx < G::GX + TXo + nxj && gx + s >= 1 && gx + s <= nx;
        okbits |= (rok && cok) ? (1u << (4 * gi + 2 * h + s)) : 0u;
      }
    }
  }
  // owned output rows (the tiles partition [0, S) in x and y)
  const bool colown = 2 * lane >= G::GX && 2 * lane < G::GX + TXo;
  unsigned ownbits = 0, fokbits = 0;
  int64_t rowoff[RT];
#pragma unroll
  for (int a = 0; a < RT; ++a) {
    const int r = r0 + a, gy = gy0 + r;
    ownbits |= (colown && r >= G::GY && r < G::GY + TYo) ? (1u << a) : 0u;
    fokbits |= (gy >= 0 && gy < Sy && gx >= 0 && gx + 1 < Sx) ? (1u << a) : 0u;
    rowoff[a] = (int64_t)gy * p.sy + gx;
  }

  double U[RT][RR][2];   // own rows of planes t-2 .. t+1: [row][ring][col]
#pragma unroll
  for (int a = 0; a < RT; ++a)
#pragma unroll
    for (int k = 0; k < RR; ++k) U[a][k][0] = U[a][k][1] = 0.0;
  double2 fcur[2][H], fnext[2][H];
#pragma unroll
  for (int gi = 0; gi < 2; ++gi)
#pragma unroll
    for (int h = 0; h < H; ++h) fcur[gi][h] = fnext[gi][h] = make_double2(0.0, 0.0);

  // f of the two groups processed at step t (plane parity Q of t)
  auto load_f = [&](int t, int Q, double2 (&fv)[2][H]) {
    if (FORM != 1) return;
#pragma unroll
    for (int gi = 0; gi < 2; ++gi) {
      const int J = q1_group(Q, gi);
      const int A = (P.colour[J] >> 1) & 1;
      const int pz = t - P.lag[J];
      const bool zin = pz >= 0 && pz < Sz;
#pragma unroll
      for (int h = 0; h < H; ++h)
        fv[gi][h] = (((fokbits >> (A + 2 * h)) & 1u) && zin)
                        ? __ldg(reinterpret_cast<const double2 *>(p.f + (int64_t)pz * sz + rowoff[A + 2 * h]))
                        : make_double2(0.0, 0.0);
    }
  };
  load_f(t_begin, 0, fcur);

  double *me = su + r0 * G::PX + 2 * lane;  // (slot 0, row r0, col 2*lane)
  // compact Q1 order: index 0 = (-1,-1,-1) corner, 1 = (0,-1,-1) edge
  const double wC = FORM == 0 ? p.aw[0] : p.w[0];
  const double wE = FORM == 0 ? p.aw[1] : p.w[1];
  unsigned emax = 0;   // max exponent field of any used update (0x7ff00000 = non-finite)

  for (int t0 = t_begin, it = 0; t0 <= t_end; t0 += RR, ++it) {
    const int hb = (it & 1) * RR;            // slot of plane t0 + 1 = (4 it) mod 8
    const uint32_t ph = (uint32_t)(it >> 1) & 1u;
    [&]<int... Ks>(std::integer_sequence<int, Ks...>) {
      (
          [&] {
            constexpr int KS = Ks;
            constexpr int Q = KS & 1;  // plane parity of step t
            const int t = t0 + KS;
            // element offset of the slot holding plane t+1-k
            auto slot = [&](int k) -> int { return ((hb + KS - k) & (G::S - 1)) * G::SLOTE; };
            load_f(t + 1, Q ^ 1, fnext);
            // ---- plane t+1 -> ring entry KS ----
            mbar_wait3(mb_s + 8u * (uint32_t)((hb + KS) & (G::S - 1)), ph);
            {
              const double *pl = me + slot(0);
#pragma unroll
              for (int a = 0; a < RT; ++a) {
                const double2 v = *reinterpret_cast<const double2 *>(pl + a * G::PX);
                U[a][KS][0] = v.x;
                U[a][KS][1] = v.y;
              }
            }
            // ---- the two independent colour groups of this step ----
            double out[2][H][2], uc[2][H][2];
            bool ok[2][H][2];
            [&]<int... Gs>(std::integer_sequence<int, Gs...>) {
              (
                  [&] {
                    constexpr int GI = Gs;                       // 0 young (registers), 1 old (smem)
                    constexpr int J = q1_group(Q, GI);
                    constexpr int LAG = P.lag[J];
                    constexpr int A = (P.colour[J] >> 1) & 1;    // rows A, A + 2
                    constexpr int nzj = P.need[J][2];
                    constexpr int KC = LAG + 1;                  // plane pz = t+1-KC
                    static_assert(GI == 1 || KC + 1 < RR, "young group must fit the ring");
                    const int pz = t - LAG;
                    const bool okz = pz >= 1 && pz <= nz && pz >= z0 - nzj && pz < z1 + nzj;
                    // centres
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                      if (GI == 0) {
                        constexpr int RC = (KS - KC + 2 * RR) % RR;
                        uc[GI][h][0] = U[A + 2 * h][RC][0];
                        uc[GI][h][1] = U[A + 2 * h][RC][1];
                      } else {
                        const double2 m = *reinterpret_cast<const double2 *>(me + slot(KC) + (A + 2 * h) * G::PX);
                        uc[GI][h][0] = m.x;
                        uc[GI][h][1] = m.y;
                      }
                    }
                    double acc[H][2];
#pragma unroll
                    for (int h = 0; h < H; ++h)
#pragma unroll
                      for (int s = 0; s < 2; ++s) acc[h][s] = acc_init<FORM, UNIT>(uc[GI][h][s], p);
#pragma unroll
                    for (int dz = -1; dz <= 1; ++dz) {
                      const int kk = KC - dz;                    // plane pz+dz = t+1-kk
                      const int rs = (KS - kk + 2 * RR) % RR;    // its ring entry (young group)
                      const double *pl = me + slot(kk);
                      // rows A-1 .. A+RT-1 (relative to r0) of plane pz+dz, cols -1 .. 2
                      double w[RT + 1][4];
#pragma unroll
                      for (int i = 0; i <= RT; ++i) {
                        const int d = A - 1 + i;
                        if (dz == 0 && ((d - A) & 1) == 0) continue;  // no in-plane face/centre rows
                        double lo, hi;
                        if (GI == 0 && d >= 0 && d < RT) {
                          lo = U[d][rs][0];
                          hi = U[d][rs][1];
                        } else {
                          const double2 m = *reinterpret_cast<const double2 *>(pl + d * G::PX);
                          lo = m.x;
                          hi = m.y;
                        }
                        w[i][0] = __shfl_up_sync(0xffffffffu, hi, 1);
                        w[i][1] = lo;
                        w[i][2] = hi;
                        w[i][3] = __shfl_down_sync(0xffffffffu, lo, 1);
                      }
#pragma unroll
                      for (int q = 0; q < shape_nnz(Q1); ++q) {
                        const Off o = shape_off(Q1, q);
                        if (o.z != dz) continue;
                        // two weight values (edges, corners; checked on the host)
                        const bool corner = o.x != 0 && o.y != 0 && o.z != 0;
                        const double wq = corner ? wC : wE;
#pragma unroll
                        for (int h = 0; h < H; ++h)
#pragma unroll
                          for (int s = 0; s < 2; ++s) {
                            const double v = w[2 * h + 1 + o.y][o.x + 1 + s];
                            if (FORM == 0)
                              acc[h][s] = __dadd_rn(acc[h][s], UNIT ? v : __dmul_rn(wq, v));
                            else if (UNIT)
                              acc[h][s] = __dsub_rn(acc[h][s], v);
                            else
                              acc[h][s] = __dadd_rn(acc[h][s], __dmul_rn(wq, v));
                          }
                      }
                    }
                    // division by w_c; exact fallback per warp, only for used lanes
                    bool slow = false;
                    double a[H][2], q[H][2];
#pragma unroll
                    for (int h = 0; h < H; ++h)
#pragma unroll
                      for (int s = 0; s < 2; ++s) {
                        ok[GI][h][s] = okz && ((okbits >> (2 * J + 2 * h + s)) & 1u);
                        a[h][s] = FORM == 0 ? acc[h][s]
                                            : __dsub_rn(s == 0 ? fcur[GI][h].x : fcur[GI][h].y, acc[h][s]);
                        if (DIV == DIV_RCP) {
                          const double e = __dmul_rn(a[h][s], p.rwc);
                          q[h][s] = __fma_rn(__fma_rn(-p.wc, e, a[h][s]), p.rwc, e);
                          const unsigned xe = ((unsigned)__double2hiint(a[h][s]) >> 20) & 0x7ffu;
                          slow |= ok[GI][h][s] && (xe - 64u) >= 1919u;
                        } else if (DIV == DIV_POW2) {
                          q[h][s] = __dmul_rn(a[h][s], p.rwc);
                        } else {
                          q[h][s] = q1_div_exact(a[h][s], p.wc);
                        }
                      }
                    if (DIV == DIV_RCP && __builtin_expect(__any_sync(0xffffffffu, slow), 0)) {
#pragma unroll
                      for (int h = 0; h < H; ++h)
#pragma unroll
                        for (int s = 0; s < 2; ++s) {
                          const unsigned xe = ((unsigned)__double2hiint(a[h][s]) >> 20) & 0x7ffu;
                          if (ok[GI][h][s] && (xe - 64u) >= 1919u) q[h][s] = q1_div_exact(a[h][s], p.wc);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < H; ++h)
#pragma unroll
                      for (int s = 0; s < 2; ++s)
                        out[GI][h][s] = FORM == 0 ? q[h][s]
                                                  : __dadd_rn(uc[GI][h][s], __dmul_rn(p.omega, q[h][s]));
                  }(),
                  ...);
            }(std::make_integer_sequence<int, 2>{});
            // ---- commit both groups: ring, non-finite tally, publish to smem ----
            [&]<int... Gs>(std::integer_sequence<int, Gs...>) {
              (
                  [&] {
                    constexpr int GI = Gs;
                    constexpr int J = q1_group(Q, GI);
                    constexpr int A = (P.colour[J] >> 1) & 1;
                    constexpr int KC = P.lag[J] + 1;
                    double *pl = me + slot(KC);
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                      double v[2];
#pragma unroll
                      for (int s = 0; s < 2; ++s) {
                        const unsigned ex = (unsigned)__double2hiint(out[GI][h][s]) & 0x7ff00000u;
                        emax = max(emax, ok[GI][h][s] ? ex : 0u);
                        v[s] = ok[GI][h][s] ? out[GI][h][s] : uc[GI][h][s];
                        if (GI == 0) {
                          constexpr int RC = (KS - KC + 2 * RR) % RR;
                          U[A + 2 * h][RC][s] = v[s];
                        }
                      }
                      *reinterpret_cast<double2 *>(pl + (A + 2 * h) * G::PX) = make_double2(v[0], v[1]);
                    }
                  }(),
                  ...);
            }(std::make_integer_sequence<int, 2>{});
            // ---- plane t - LAGMAX is final: owned rows -> dst (from its smem slot) ----
            {
              const int po = t - G::LAGMAX;
              if (po >= z0 && po < z1) {
                const double *pl = me + slot(G::LAGMAX + 1);
#pragma unroll
                for (int a = 0; a < RT; ++a)
                  if ((ownbits >> a) & 1u) {
                    const double2 v = *reinterpret_cast<const double2 *>(pl + a * G::PX);
                    stg_pair(dst + (int64_t)po * sz + rowoff[a], v.x, v.y);
                  }
              }
            }
            __syncthreads();
            // the slot of plane t-5 is free: refill it with plane t+3
            if (threadIdx.x == 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue(t + 3);
            }
#pragma unroll
            for (int gi = 0; gi < 2; ++gi)
#pragma unroll
              for (int h = 0; h < H; ++h) fcur[gi][h] = fnext[gi][h];
          }(),
          ...);
    }(std::make_integer_sequence<int, RR>{});
  }
  if (threadIdx.x == 0) {  // drain the copies still in flight
    const int tl = t_begin + ((t_end - t_begin) / RR + 1) * RR;  // first step not run
    for (int k = 1; k <= 2; ++k) {
      const int pl = tl + k;
      mbar_wait3(mb_s + 8u * (uint32_t)((pl - base) & (G::S - 1)), (uint32_t)(((pl - base) / G::S) & 1));
    }
  }
  __syncthreads();
  if (__any_sync(0xffffffffu, emax == 0x7ff00000u) && lane == 0) atomicOr(p.status, 1);
}

}  // namespace sl
