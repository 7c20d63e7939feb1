// k2_q1col.cuh — K2 for the trilinear Q1 27-point operator (BASELINE config 4).
//
// Q1 has no face neighbours (their weights are 0), so a point's 20 neighbours
// are the 8 columns around it on planes z+-1 and the 4 diagonal columns on its
// own plane; the 2x2x2 parity colouring gives 8 colours.  Lags are spread
// (plan.cuh: 0,0,1,1,3,3,4,4) so the colour groups active in one step —
// {0,1}@t with {4,5}@t-3 on even steps, {2,3}@t-1 with {6,7}@t-4 on odd
// ones — are mutually independent: one block barrier per step.
//
// A CTA owns a 64 x 32 (x, y) tile (+ the ghost margin 4/4/2 of the plan) and
// a chunk of z.  Thread (warp w, lane i) owns column pair (2i, 2i+1) of the
// two tile rows r0 = 2w + delta, r0 + 1, where delta makes row r0 the y-parity
// 0 row: a colour group updates all columns of every other row, so each
// thread updates both points of one of its rows per group.  The thread keeps
// its two rows of the pair for planes t-6 .. t+1 in a register ring (z and
// own-row neighbours), gets the neighbour pair's columns by warp shuffles,
// and reads only the rows owned by the warps above/below from shared memory.
// Updated pairs are written back to the plane's smem slot for those readers.
// u planes arrive by TMA (64 x 33 x 1 boxes, zero-filled out of range) into 9
// smem slots, D = 2 planes ahead; f is prefetched one step ahead per thread.
#pragma once
#include <cuda.h>

#include "plan.cuh"

namespace sl {

struct Q1Geo {
  static constexpr FPlan P = make_plan(Q1, 8, 1, true);
  static constexpr int LAGMAX = P.lagmax;                 // 4
  static constexpr int GX = 4, GY = 4, GZ = 2;            // plan load margins
  static constexpr int PX = 64, PY = 32;                  // tile incl. ghost
  static constexpr int BOXY = PY + 1;                     // rows loaded (delta shift)
  static constexpr int TX = PX - 2 * GX, TY = PY - 2 * GY;
  static constexpr int RR = 8;                            // register ring (planes t-6 .. t+1)
  static constexpr int WS = 9;                            // smem slots (planes t-5 .. t+3)
  static constexpr int D = 2;                             // TMA lookahead beyond plane t+1
  static constexpr int NT = 512;
  static constexpr int SLOTE = PX * BOXY;
  static constexpr int LEADE = 2 * PX;                    // guard rows before slot 0
  static constexpr size_t SMEM = size_t(LEADE + WS * SLOTE + 2 * PX) * sizeof(double) + WS * 8;
  static_assert(P.lag[0] == 0 && P.lag[2] == 1 && P.lag[4] == 3 && P.lag[6] == 4, "unexpected plan");
  static_assert(P.load[0] <= GX && P.load[1] <= GY && P.load[2] <= GZ, "ghost margin");
  static_assert(WS >= LAGMAX + 3 + D && RR >= LAGMAX + 3, "rings too short");
};

template <int FORM, bool UNIT, int DIV>
__global__ void __launch_bounds__(Q1Geo::NT, 1)
k2_q1col(Params p, const __grid_constant__ CUtensorMap tmu, double *__restrict__ dst, int64_t ntx,
         int64_t nty, int64_t nzc) {
  using G = Q1Geo;
  constexpr FPlan P = G::P;
  constexpr int RR = G::RR, WS = G::WS, D = G::D;
  extern __shared__ __align__(128) double qsm[];
  double *su = qsm + G::LEADE;  // slot k at su + k*SLOTE
  uint64_t *mb = reinterpret_cast<uint64_t *>(su + WS * G::SLOTE + 2 * G::PX);
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
  const int r0 = 2 * warp + delta;               // this thread's rows: r0 (qy 0), r0 + 1 (qy 1)
  const int sy = (int)p.sy;
  const int64_t sz = p.sz;

  int t_begin = z0 - G::GZ - 1;
  if ((t_begin - 1 + p.pz) & 1) --t_begin;       // plane parity of step k is k & 1
  const int t_end = z1 - 1 + G::LAGMAX;
  const int zlim = z1 + G::GZ;

  // smem slot offsets (elements), rotated per step: so[k] = slot of plane t+1+D-k
  int so[WS];
#pragma unroll
  for (int k = 0; k < WS; ++k) so[k] = (((t_begin + 1 + D - k) % WS + WS) % WS) * G::SLOTE;

  auto issue = [&](int plane) {
    const int sl = ((plane % WS) + WS) % WS;
    const uint32_t bar = mb_s + 8u * sl;
    const bool live = plane >= 0 && plane < Sz && plane < zlim;
    mbar_expect3(bar, live ? (uint32_t)(G::SLOTE * 8) : 0u);
    if (live) tma_load_3d(su_s + sl * G::SLOTE * 8, &tmu, gx0, gy0, plane, bar);
  };
  // use count of the slot holding `plane` (planes >= t_begin+1 are loaded, in order)
  auto parity_of = [&](int plane) -> uint32_t {
    const int sl = ((plane % WS) + WS) % WS;
    const int first = t_begin + 1 + (((sl - (t_begin + 1)) % WS) + WS) % WS;  // first plane in slot
    return (uint32_t)(((plane - first) / WS) & 1);
  };

  if (threadIdx.x == 0) {
    for (int k = 0; k < WS; ++k) mbar_init3(mb_s + 8u * k);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 1; k <= 1 + D; ++k) issue(t_begin + k);
  }
  __syncthreads();

  // validity per group (need margins are per colour group; both colours of a
  // group share them): group g = J/2 for J = 0,2,4,6
  auto colok = [&](int s, int need) -> bool {
    const int lx = 2 * lane + s;
    return lx >= G::GX - need && lx < G::GX + TXo + need && gx + s >= 1 && gx + s <= nx;
  };
  auto rowok = [&](int r, int need) -> bool {
    const int gy = gy0 + r;
    return r >= G::GY - need && r < G::GY + TYo + need && gy >= 1 && gy <= ny;
  };

  double U[2][RR][2];   // [row][plane ring][col]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < RR; ++k) U[a][k][0] = U[a][k][1] = 0.0;
  double2 fcur[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  double2 fnext[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};

  // f of the two groups processed at step t: (row a, plane pz) for a pair
  auto load_f = [&](int t, double2 (&fv)[2]) {
    if (FORM != 1) return;
    const int q = (t - 1 + p.pz) & 1;                    // plane parity at step t
    const int a = q;                                     // row r0 (q=0) or r0+1 (q=1)
    const int pzs[2] = {q == 0 ? t : t - 1, q == 0 ? t - 3 : t - 4};
    const int gy = gy0 + r0 + a;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int pz = pzs[k];
      const bool ok = pz >= 1 && pz <= nz && gy >= 1 && gy <= ny && gx >= 0 && gx + 1 < Sx;
      fv[k] = ok ? __ldg(reinterpret_cast<const double2 *>(p.f + (int64_t)pz * sz + (int64_t)gy * sy + gx))
                 : make_double2(0.0, 0.0);
    }
  };
  load_f(t_begin, fcur);

  const int lrow0 = r0 * G::PX + 2 * lane;  // element offset of (row r0, col 2*lane) in a slot
  // compact Q1 order: index 0 = (-1,-1,-1) corner, 1 = (0,-1,-1) edge
  const double wC = p.w[0], wE = p.w[1], awC = p.aw[0], awE = p.aw[1];
  unsigned bad = 0;
  for (int t0 = t_begin; t0 <= t_end; t0 += RR) {
    [&]<int... Ks>(std::integer_sequence<int, Ks...>) {
      (
          [&] {
            constexpr int KS = Ks;
            const int t = t0 + KS;
            constexpr int Q = KS & 1;  // plane parity of t
            load_f(t + 1, fnext);
            // ---- plane t+1: wait for its TMA, take this thread's two rows ----
            const int slot_t1 = so[D];  // so[k] = slot of plane t+1+D-k
            mbar_wait3(mb_s + 8u * (uint32_t)(slot_t1 / G::SLOTE), parity_of(t + 1));
            {
              constexpr int R1 = (KS + 1) % RR;
#pragma unroll
              for (int a = 0; a < 2; ++a) {
                const double2 v = *reinterpret_cast<const double2 *>(su + slot_t1 + lrow0 + a * G::PX);
                U[a][R1][0] = v.x;
                U[a][R1][1] = v.y;
              }
            }
            // ---- the two active colour groups of this step ----
            [&]<int... Gs>(std::integer_sequence<int, Gs...>) {
              (
                  [&] {
                    constexpr int GI = Gs;                       // 0: first group, 1: second
                    constexpr int J = Q == 0 ? (GI == 0 ? 0 : 4) : (GI == 0 ? 2 : 6);
                    constexpr int LAG = P.lag[J];
                    constexpr int A = (P.colour[J] >> 1) & 1;     // this group's row (y parity)
                    constexpr int nxj = P.need[J][0], nyj = P.need[J][1], nzj = P.need[J][2];
                    const int pz = t - LAG;
                    if (pz < 1 || pz > nz || pz < z0 - nzj || pz >= z1 + nzj) return;
                    constexpr int RC = ((KS - LAG) % RR + RR) % RR;        // ring slot of plane pz
                    constexpr int RM = (RC + RR - 1) % RR, RP = (RC + 1) % RR;
                    const int sc = so[D + 1 + LAG];                // smem slot of pz
                    const int sm_ = so[D + 2 + LAG], sp = so[D + LAG];
                    // other-warp row: above row r0 (A = 0) or below row r0+1 (A = 1)
                    const int orow = A == 0 ? -1 : 2;              // relative to r0
                    // accumulate plane by plane (dz outer = canonical order), so only one
                    // plane's 3 x 4 window of values is live at a time
                    const double uc0 = U[A][RC][0], uc1 = U[A][RC][1];
                    double acc0 = acc_init<FORM, UNIT>(uc0, p), acc1 = acc_init<FORM, UNIT>(uc1, p);
#pragma unroll
                    for (int dz = -1; dz <= 1; ++dz) {
                      const int ring = dz < 0 ? RM : (dz > 0 ? RP : RC);
                      const int slot = dz < 0 ? sm_ : (dz > 0 ? sp : sc);
                      double w[3][4];  // [dy+1][col+1]
#pragma unroll
                      for (int dy = -1; dy <= 1; ++dy) {
                        if (dz == 0 && dy == 0) continue;  // no in-plane face/centre terms
                        const int d = A + dy;              // row relative to r0
                        if (d == orow) {
                          const double *pr = su + slot + lrow0 + d * G::PX;
                          const double2 m = *reinterpret_cast<const double2 *>(pr);
                          w[dy + 1][0] = pr[-1];
                          w[dy + 1][1] = m.x;
                          w[dy + 1][2] = m.y;
                          w[dy + 1][3] = pr[2];
                        } else {
                          const double lo = U[d][ring][0], hi = U[d][ring][1];
                          w[dy + 1][0] = __shfl_up_sync(0xffffffffu, hi, 1);
                          w[dy + 1][1] = lo;
                          w[dy + 1][2] = hi;
                          w[dy + 1][3] = __shfl_down_sync(0xffffffffu, lo, 1);
                        }
                      }
#pragma unroll
                      for (int q = 0; q < shape_nnz(Q1); ++q) {
                        const Off o = shape_off(Q1, q);
                        if (o.z != dz) continue;
                        // Q1 weights take two values (edges, corners; checked on the
                        // host), held in two registers instead of 20 parameters
                        const bool corner = o.x != 0 && o.y != 0 && o.z != 0;
                        const double wq = FORM == 0 ? (corner ? awC : awE) : (corner ? wC : wE);
                        const double v0 = w[o.y + 1][o.x + 1], v1 = w[o.y + 1][o.x + 2];
                        acc0 = __dadd_rn(acc0, __dmul_rn(wq, v0));
                        acc1 = __dadd_rn(acc1, __dmul_rn(wq, v1));
                      }
                    }
                    const double2 fc = fcur[GI];
                    const bool rok = rowok(r0 + A, nyj);
                    bool ok[2];
                    double out[2];
                    ok[0] = rok && colok(0, nxj);
                    ok[1] = rok && colok(1, nxj);
                    out[0] = acc_finish_used<FORM, UNIT, DIV>(acc0, uc0, fc.x, ok[0], p);
                    out[1] = acc_finish_used<FORM, UNIT, DIV>(acc1, uc1, fc.y, ok[1], p);
#pragma unroll
                    for (int s = 0; s < 2; ++s)
                      if (ok[s]) U[A][RC][s] = out[s];
                    // publish the pair for the warps above/below (same values if not updated)
                    *reinterpret_cast<double2 *>(su + sc + lrow0 + A * G::PX) = make_double2(U[A][RC][0], U[A][RC][1]);
                  }(),
                  ...);
            }(std::make_integer_sequence<int, 2>{});
            // ---- plane t - LAGMAX is final: owned pairs of both rows -> dst ----
            {
              const int pz = t - G::LAGMAX;
              constexpr int RO = ((KS - G::LAGMAX) % RR + RR) % RR;
              if (pz >= z0 && pz < z1 && 2 * lane >= G::GX && 2 * lane < G::GX + TXo) {
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                  const int r = r0 + a, gy = gy0 + r;
                  if (r >= G::GY && r < G::GY + TYo) {
                    const bool in_yz = pz >= 1 && pz <= nz && gy >= 1 && gy <= ny;
                    bad |= (in_yz && gx >= 1 && ((unsigned)__double2hiint(U[a][RO][0]) & 0x7ff00000u) == 0x7ff00000u) |
                           (in_yz && gx + 1 <= nx && ((unsigned)__double2hiint(U[a][RO][1]) & 0x7ff00000u) == 0x7ff00000u);
                    stg_pair(dst + (int64_t)pz * sz + (int64_t)gy * sy + gx, U[a][RO][0], U[a][RO][1]);
                  }
                }
              }
            }
            __syncthreads();
            // rotate the slots; refill the slot of plane t-5 with plane t+2+D
            {
              const int tmp = so[WS - 1];
#pragma unroll
              for (int k = WS - 1; k > 0; --k) so[k] = so[k - 1];
              so[0] = tmp;
            }
            if (threadIdx.x == 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue(t + 2 + D);
            }
            fcur[0] = fnext[0];
            fcur[1] = fnext[1];
          }(),
          ...);
    }(std::make_integer_sequence<int, RR>{});
  }
  if (threadIdx.x == 0) {  // drain the copies still in flight
    const int tl = t_begin + ((t_end - t_begin) / RR + 1) * RR;
    for (int k = 1; k <= 1 + D; ++k) {
      const int pl = tl + k;
      mbar_wait3(mb_s + 8u * (uint32_t)(((pl % WS) + WS) % WS), parity_of(pl));
    }
  }
  __syncthreads();
  if (bad) atomicOr(p.status, 1);
}

}  // namespace sl
