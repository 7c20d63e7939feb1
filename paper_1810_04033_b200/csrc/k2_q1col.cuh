// k2_q1col.cuh — K2 for the trilinear Q1 27-point operator (BASELINE config 4).
//
// Q1 has no face neighbours (their weights are 0), so a point's 20 neighbours
// are the 8 columns around it on planes z+-1 and the 4 diagonal columns on its
// own plane; the 2x2x2 parity colouring gives 8 colours, and a plane holds the
// four colours of its z parity.  Colours pair up by x parity into groups that
// update every column of every other row: G0 = {0,1}, G1 = {2,3} on qz = 0
// planes, G2 = {4,5}, G3 = {6,7} on qz = 1 planes.  The pass follows the
// compact plan (plan.cuh, lags 0,0,0,0,1,1,1,1): the loop advances by plane
// pairs (p, p-1) with p of parity qz = 0 and runs G0@p, G1@p, G2@p-1, G3@p-1
// in colour order with a block barrier between consecutive groups (each group
// reads the previous one's results from the warps above/below).  After the
// pair step both planes are final and are stored.
//
// A CTA owns a 64 x 48 (x, y) tile (+ the ghost margin 4/4/2 of the plan) and
// a chunk of z; 12 warps.  Thread (warp w, lane i) owns column pair (2i, 2i+1)
// of the RT = 4 tile rows r0 = 4w + delta .. r0 + 3, where delta makes row r0
// a y-parity 0 row, so each group updates 2 x 2 points of the thread (rows A,
// A + 2).  The thread keeps its rows of planes p-2 .. p in a register ring
// (plane p+1, read only by G0/G1, comes from its slot); otherwise only the
// row of the warp above/below comes from the plane's shared-memory slot, and
// the x+-1 columns from warp shuffles.  Neighbour values enter the sums as
// weighted products computed once per value and weight and shared (by
// shuffle) with the lanes that need them.  Every update is published to the
// slot for the neighbouring warps.
//
// u planes arrive by TMA (64 x 49 x 1 boxes, zero-filled out of range) into
// 8 smem slots, up to six planes ahead.  The loop is unrolled by two pair
// steps (one ring turn), so ring indices are compile-time; slot offsets and
// mbarrier parities are cheap runtime values.  Out-of-range groups and ghost
// points are computed and masked (no branches around the shuffles: skipping
// the groups a warp has no used point in measured 0.7 % slower, the early exit
// grows the unrolled loop by 60 %); the exact
// division fallback runs out of line, per warp, only when a used lane's
// operand leaves the fast range.
#pragma once
#include <cuda.h>

#include "plan.cuh"

namespace sl {

// Exact division out of line: the rare fallback of the Markstein fast path
// must not bloat the unrolled loop (instruction-cache pressure).
static __device__ __noinline__ double q1_div_exact(double a, double b) { return __ddiv_rn(a, b); }

struct Q1Geo {
  static constexpr FPlan P = make_plan(Q1, 8, 1, false);
  static constexpr int GX = 4, GY = 4, GZ = 2;            // plan load margins
  static constexpr int PX = 64, PY = 48;                  // tile incl. ghost
  static constexpr int BOXY = PY + 1;                     // rows loaded (delta shift)
  static constexpr int TX = PX - 2 * GX, TY = PY - 2 * GY;
  static constexpr int S = 8;                             // smem slots
  static constexpr int RR = 4;                            // ring entries (planes p-2 .. p live)
#ifndef Q1_RT
#define Q1_RT 4
#endif
  static constexpr int RT = Q1_RT;                        // tile rows per thread
  static constexpr int NT = 32 * PY / RT;                 // 384
  static constexpr int LAGMAX = 1;
  static constexpr int SLOTE = PX * BOXY;
  static constexpr int LEADE = 2 * PX;                    // guard rows before slot 0
  static constexpr int FBUFE = 2 * (RT / 2) * 2 * NT;      // f staging: 2 buffers x H rows x 2 cols
  static constexpr size_t SMEM = size_t(LEADE + S * SLOTE + 2 * PX + FBUFE) * sizeof(double) + S * 8;
  static_assert(P.load[0] <= GX && P.load[1] <= GY && P.load[2] <= GZ, "ghost margin");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

constexpr bool q1_plan_ok() {
  for (int k = 0; k < 8; ++k)
    if (Q1Geo::P.colour[k] != k || Q1Geo::P.lag[k] != (k < 4 ? 0 : 1)) return false;
  return true;
}
static_assert(q1_plan_ok(), "unexpected plan");

// EDGE = false: the tile's whole window lies inside the grid interior in x
// and y, so no point needs a mask — every computed point may be updated (points
// outside their phase's need region hold values nobody needed reads, plan.cuh)
// and only owned points are checked for non-finite results, when stored.
// EDGE = true keeps the per-point interior/need masks.
template <int FORM, bool UNIT, int DIV, bool PEER, bool EDGE>
__device__ __forceinline__ void q1col_body(const Params &p, const CUtensorMap &tmu, double *__restrict__ dst,
                                           int64_t ntx, int64_t nty, int64_t nzc) {
  using G = Q1Geo;
  constexpr FPlan P = G::P;
  constexpr int RT = G::RT, H = RT / 2, RR = G::RR;
  extern __shared__ __align__(128) double qsm[];
  double *su = qsm + G::LEADE;  // slot k at su + k*SLOTE
  double *fbuf = su + G::S * G::SLOTE + 2 * G::PX;   // [buffer][h][thread] double2
  uint64_t *mb = reinterpret_cast<uint64_t *>(fbuf + G::FBUFE);
  const uint32_t su_s = (uint32_t)__cvta_generic_to_shared(su);
  const uint32_t mb_s = (uint32_t)__cvta_generic_to_shared(mb);

  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2, Sz = (int)p.nz + 2;
  const int nx = (int)p.nx, ny = (int)p.ny, nz = (int)p.nz;
  const int item = blockIdx.x;
  const int tx = item % (int)ntx, ty = (item / (int)ntx) % (int)nty, zc = item / (int)(ntx * nty);
  const int x0 = (int)(2 * (((int64_t)tx * (Sx / 2)) / ntx)), x1 = (int)(2 * (((int64_t)(tx + 1) * (Sx / 2)) / ntx));
  const int y0 = (int)(((int64_t)ty * Sy) / nty), y1 = (int)(((int64_t)(ty + 1) * Sy) / nty);
  const int zlen = p.zhi - p.zlo;
  const int z0 = p.zlo + (int)(((int64_t)zc * zlen) / nzc), z1 = p.zlo + (int)(((int64_t)(zc + 1) * zlen) / nzc);
  const int TXo = x1 - x0, TYo = y1 - y0;
  const int gx0 = x0 - G::GX, gy0 = y0 - G::GY;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx = gx0 + 2 * lane;
  const int delta = (1 - p.py - gy0) & 1;        // local row r0 has y parity 0
  const int r0 = RT * warp + delta;              // this thread's rows r0 (qy 0) .. r0 + RT - 1
  const int64_t sz = p.sz;

  // pair steps at planes pp = p_begin, p_begin + 2, ... of parity qz = 0;
  // G0/G1 (at pp) and G2/G3 (at pp - 1) must cover [z0 - n, z1 + n)
  constexpr int NZ = [] {
    int m = 0;
    for (int k = 0; k < 8; ++k) m = cmax(m, P.need[k][2]);
    return m;
  }();
  int p_begin = z0 - NZ;
  if ((p_begin - 1 + p.pz) & 1) --p_begin;       // qz(pp) = (pp - 1 + pz) & 1 must be 0
  const int p_end = z1 + NZ;
  const int zlim = z1 + G::GZ;
  const int base = p_begin - 2;                  // plane held by slot 0 / ring 0 in use 0

  auto issue = [&](int plane) {
    const int sl = (plane - base) & (G::S - 1);
    const uint32_t bar = mb_s + 8u * sl;
    const bool live = plane >= 0 && plane < Sz && plane < zlim;
    mbar_expect3(bar, live ? (uint32_t)(G::SLOTE * 8) : 0u);
    if (live) tma_load_3d(su_s + sl * G::SLOTE * 8, &tmu, gx0, gy0, plane, bar);
  };
  auto wait_plane = [&](int plane) {
    mbar_wait3(mb_s + 8u * (uint32_t)((plane - base) & (G::S - 1)), (uint32_t)(((plane - base) >> 3) & 1));
  };
  double *me = su + r0 * G::PX + 2 * lane;  // (slot 0, row r0, col 2*lane)
  auto slot_of = [&](int plane) -> double * { return me + ((plane - base) & (G::S - 1)) * G::SLOTE; };

  if (threadIdx.x == 0) {
    for (int k = 0; k < G::S; ++k) mbar_init3(mb_s + 8u * k);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < 6; ++k) issue(base + k);  // planes p_begin-2 .. p_begin+3
  }
  __syncthreads();

  // ---- thread-constant masks ------------------------------------------------
  // ok bit (4*gi + 2*h + s): point s of the h-th row (A + 2h) of group gi
  // (colours 2gi, 2gi+1) is inside its need region and the grid interior (x, y)
  unsigned okbits = 0;
#pragma unroll
  for (int gi = 0; gi < 4; ++gi) {
    const int A = gi & 1;
    const int nxj = cmax(P.need[2 * gi][0], P.need[2 * gi + 1][0]);
    const int nyj = cmax(P.need[2 * gi][1], P.need[2 * gi + 1][1]);
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
  const int64_t rowoff0 = (int64_t)(gy0 + r0) * p.sy + gx;   // row r0 of this thread
  const int sy32 = (int)p.sy;
  unsigned inbits = 0;   // interior (updated) points: bit 2*a + s
#pragma unroll
  for (int a = 0; a < RT; ++a) {
    const int r = r0 + a, gy = gy0 + r;
    ownbits |= (colown && r >= G::GY && r < G::GY + TYo) ? (1u << a) : 0u;
    fokbits |= (gy >= 0 && gy < Sy && gx >= 0 && gx + 1 < Sx) ? (1u << a) : 0u;
#pragma unroll
    for (int s = 0; s < 2; ++s)
      inbits |= (gy >= 1 && gy <= ny && gx + s >= 1 && gx + s <= nx) ? (1u << (2 * a + s)) : 0u;
  }

  // own rows of planes pp-2 .. pp+1: [row][ring][col]; plane P at (P - base) % RR
  double U[RT][RR][2];
  wait_plane(base);
  wait_plane(base + 1);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double *pl = slot_of(base + k);
#pragma unroll
    for (int a = 0; a < RT; ++a) {
      const double2 v = *reinterpret_cast<const double2 *>(pl + a * G::PX);
      U[a][k][0] = v.x;
      U[a][k][1] = v.y;
    }
  }
#pragma unroll
  for (int a = 0; a < RT; ++a)
#pragma unroll
    for (int k = 2; k < RR; ++k) U[a][k][0] = U[a][k][1] = 0.0;

  // f of group gi at plane pz (rows A + 2h)
  // f rows of group gi at plane pz (rows A + 2h) are staged per thread in
  // shared memory by cp.async, one group ahead of their use, alternating
  // between two buffers (the groups of a pair step use buffers 0, 1, 0, 1).
  // cp.async.wait_group waits for exactly the older copies, so the newest
  // copy in flight never delays a consumer (a register LDG would share its
  // scoreboard with it).  Masked rows are zero-filled (src size 0).
  const double *fthr = p.f + rowoff0;
  const uint32_t fb_s = (uint32_t)__cvta_generic_to_shared(fbuf) + 16u * threadIdx.x;
  auto issue_f = [&](int gi, int pz, int buf) {
    const int A = gi & 1;
    const bool zin = pz >= 0 && pz < Sz;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const bool live = FORM == 1 && ((fokbits >> (A + 2 * h)) & 1u) && zin;
      const double *fp = live ? fthr + (int64_t)pz * sz + (A + 2 * h) * sy32 : p.u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(fb_s + 16u * (buf * H + h) * G::NT),
                   "l"(fp), "r"(live ? 16 : 0));
    }
    asm volatile("cp.async.commit_group;");
  };
  auto read_f = [&](int buf, double2 (&fv)[H]) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
    for (int h = 0; h < H; ++h)
      fv[h] = reinterpret_cast<const double2 *>(fbuf)[(buf * H + h) * G::NT + threadIdx.x];
  };
  if (FORM == 1) issue_f(0, p_begin, 0);

  // compact Q1 order: index 0 = (-1,-1,-1) corner, 1 = (0,-1,-1) edge
  const double wC = FORM == 0 ? p.aw[0] : p.w[0];
  const double wE = FORM == 0 ? p.aw[1] : p.w[1];
  unsigned emax = 0;   // max exponent field of any used update (0x7ff00000 = non-finite)

  // one colour group GI at plane pz = pp - (GI >> 1); RP = ring entry of pp
  auto group = [&]<int GI, int RP>(int pp) {
    // next group's right-hand side in flight, this group's from its buffer
    double2 fv[H];
    if (FORM == 1) {
      constexpr int NGI = (GI + 1) & 3;
      issue_f(NGI, GI == 0 ? pp : GI == 3 ? pp + 2 : pp - 1, NGI & 1);
      read_f(GI & 1, fv);
    }
    constexpr int A = GI & 1;                      // rows A, A + 2
    constexpr int LAGG = GI >> 1;
    constexpr int RC = (RP - LAGG + RR) % RR;      // ring entry of plane pz
    constexpr int NZJ = cmax(P.need[2 * GI][2], P.need[2 * GI + 1][2]);
    const int pz = pp - LAGG;
    // CTA-uniform.  Planes beyond the chunk's need range are computed like
    // ghost points (nobody needed reads them); boundary planes and planes
    // outside the grid are computed too but their results are dropped after
    // the group (a branch around the whole group would wrap every shuffle in
    // convergence code)
    const bool pzin = pz >= 1 && pz <= nz;
    (void)NZJ;
    double acc[H][2];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int s = 0; s < 2; ++s) acc[h][s] = acc_init<FORM, UNIT>(U[A + 2 * h][RC][s], p);
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
      const int rs = (RC + dz + RR) % RR;
      const double *pl = slot_of(pz + dz);
      // rows A-1 .. A+RT-1 (relative to r0) of plane pz+dz, cols -1 .. 2, as
      // weighted products: each value is multiplied once per weight it is
      // used with and the product is shared by the (up to four) points that
      // read it — the same rounded w_j * u_j the canonical sum adds.  Rows of
      // the other y parity on planes z+-1 feed corners and edges (pc, pe),
      // the rest edges only; x+-1 columns arrive by shuffle as products.
      // Rows are visited in order and each row's terms are added as soon as
      // its products exist: per point the terms still arrive in canonical
      // (y, then x ascending) order, and only one row of products is live.
#pragma unroll
      for (int i = 0; i <= RT; ++i) {
        const int d = A - 1 + i;
        const bool odd = ((d - A) & 1) != 0;
        if (dz == 0 && !odd) continue;  // no in-plane face/centre rows
        double lo, hi;
        if (d >= 0 && d < RT && !(LAGG == 0 && dz == 1)) {
          lo = U[d][rs][0];
          hi = U[d][rs][1];
        } else {
          const double2 m = *reinterpret_cast<const double2 *>(pl + d * G::PX);
          lo = m.x;
          hi = m.y;
        }
        double pe[4], pc[4];
        pe[1] = UNIT ? lo : __dmul_rn(wE, lo);
        pe[2] = UNIT ? hi : __dmul_rn(wE, hi);
        if (!UNIT && odd && dz != 0) {
          pc[1] = __dmul_rn(wC, lo);
          pc[2] = __dmul_rn(wC, hi);
          pc[0] = __shfl_up_sync(0xffffffffu, pc[2], 1);
          pc[3] = __shfl_down_sync(0xffffffffu, pc[1], 1);
        } else {
          pe[0] = __shfl_up_sync(0xffffffffu, pe[2], 1);
          pe[3] = __shfl_down_sync(0xffffffffu, pe[1], 1);
          pc[0] = pe[0];
          pc[1] = pe[1];
          pc[2] = pe[2];
          pc[3] = pe[3];
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int oy = i - (2 * h + 1);
          if (oy < -1 || oy > 1) continue;
#pragma unroll
          for (int q = 0; q < shape_nnz(Q1); ++q) {
            const Off o = shape_off(Q1, q);
            if (o.z != dz || o.y != oy) continue;
            const bool corner = o.x != 0 && o.y != 0 && o.z != 0;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const double v = corner ? pc[o.x + 1 + s] : pe[o.x + 1 + s];
              acc[h][s] = (FORM == 1 && UNIT) ? __dsub_rn(acc[h][s], v) : __dadd_rn(acc[h][s], v);
            }
          }
        }
      }
    }
    // division by w_c.  The fast-path range test ignores the lane masks (a
    // zero-filled point outside the grid only sends its warp into the
    // fallback, which applies them), so no mask is kept live across it.
    bool ok[H][2], slow = false;
    double a[H][2], q[H][2];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        ok[h][s] = !EDGE || ((okbits >> (4 * GI + 2 * h + s)) & 1u);
        a[h][s] = FORM == 0 ? acc[h][s] : __dsub_rn(s == 0 ? fv[h].x : fv[h].y, acc[h][s]);
        if (DIV == DIV_RCP) {
          const double e = __dmul_rn(a[h][s], p.rwc);
          q[h][s] = __fma_rn(__fma_rn(-p.wc, e, a[h][s]), p.rwc, e);
          const unsigned xe = (unsigned)__double2hiint(a[h][s]) & 0x7ff00000u;
          slow |= (xe - (64u << 20)) >= (1919u << 20);
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
          const unsigned xe = (unsigned)__double2hiint(a[h][s]) & 0x7ff00000u;
          if (ok[h][s] && (xe - (64u << 20)) >= (1919u << 20)) q[h][s] = q1_div_exact(a[h][s], p.wc);
        }
    }
    // commit: ring, publish to the plane's slot (a dropped plane gets its
    // unchanged values back from the slot)
    double *pc = slot_of(pz);
#pragma unroll
    for (int h = 0; h < H; ++h) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double uc = U[A + 2 * h][RC][s];
        const double out = FORM == 0 ? q[h][s] : __dadd_rn(uc, __dmul_rn(p.omega, q[h][s]));
        U[A + 2 * h][RC][s] = (!EDGE || ok[h][s]) ? out : uc;
      }
    }
    if (pzin) {
#pragma unroll
      for (int h = 0; h < H; ++h)
        *reinterpret_cast<double2 *>(pc + (A + 2 * h) * G::PX) =
            make_double2(U[A + 2 * h][RC][0], U[A + 2 * h][RC][1]);
    } else {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const double2 v = *reinterpret_cast<const double2 *>(pc + (A + 2 * h) * G::PX);
        U[A + 2 * h][RC][0] = v.x;
        U[A + 2 * h][RC][1] = v.y;
      }
    }
  };

  // owned rows of a final plane (ring entry RE) -> dst; the non-finite check
  // covers exactly the updated points of the pass: owned and interior
  double *const dthr = dst + rowoff0;
  auto store_plane = [&](int po, auto RE) {
    constexpr int E = decltype(RE)::value;
    if (po >= z0 && po < z1) {
      double *dp = dthr + (int64_t)po * sz;
      const bool zin = po >= 1 && po <= nz;
#pragma unroll
      for (int a = 0; a < RT; ++a)
        if ((ownbits >> a) & 1u) {
          stg_pair(dp + a * sy32, U[a][E][0], U[a][E][1]);
          stg_pair_peers<PEER>(p, po, (int64_t)po * sz + rowoff0 + a * sy32, U[a][E][0], U[a][E][1]);
          if (zin) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const unsigned ex = (unsigned)__double2hiint(U[a][E][s]) & 0x7ff00000u;
              emax = max(emax, (!EDGE || ((inbits >> (2 * a + s)) & 1u)) ? ex : 0u);
            }
          }
        }
    }
  };

  for (int pp0 = p_begin; pp0 <= p_end; pp0 += 4) {
    [&]<int... Ks>(std::integer_sequence<int, Ks...>) {
      (
          [&] {
            constexpr int KS = Ks;                      // pair step within the ring turn
            constexpr int RP0 = (2 + 2 * KS) % RR;      // ring entry of the pair plane pp
            constexpr int RM1 = (RP0 + RR - 1) % RR;
            const int pp = pp0 + 2 * KS;
            // planes pp-1 and pp -> ring (plane pp+1 is read from its slot:
            // only three planes are ever live in registers)
            wait_plane(pp);
            wait_plane(pp + 1);
            {
              const double *pa = slot_of(pp - 1), *pb = slot_of(pp);
#pragma unroll
              for (int a = 0; a < RT; ++a) {
                const double2 va = *reinterpret_cast<const double2 *>(pa + a * G::PX);
                const double2 vb = *reinterpret_cast<const double2 *>(pb + a * G::PX);
                U[a][RM1][0] = va.x;
                U[a][RM1][1] = va.y;
                U[a][RP0][0] = vb.x;
                U[a][RP0][1] = vb.y;
              }
            }
            group.template operator()<0, RP0>(pp);
            __syncthreads();
            // everybody is past the previous pair step: refill the slots of
            // planes pp-4, pp-3 with planes pp+4, pp+5
            if (threadIdx.x == 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue(pp + 4);
              issue(pp + 5);
            }
            group.template operator()<1, RP0>(pp);
            store_plane(pp, std::integral_constant<int, RP0>{});  // plane pp is final after G1
            __syncthreads();
            group.template operator()<2, RP0>(pp);
            __syncthreads();
            group.template operator()<3, RP0>(pp);
            store_plane(pp - 1, std::integral_constant<int, RM1>{});
          }(),
          ...);
    }(std::make_integer_sequence<int, 2>{});
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // drain the copies issued but never waited for
    const int pl_end = p_begin + ((p_end - p_begin) / 4 + 1) * 4;  // first pair step not run
    for (int pl = pl_end; pl <= pl_end + 3; ++pl) wait_plane(pl);
  }
  __syncthreads();
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (__any_sync(0xffffffffu, emax == 0x7ff00000u) && lane == 0) atomicOr(p.status, 1);
}

template <int FORM, bool UNIT, int DIV, bool PEER = false>
__global__ void __launch_bounds__(Q1Geo::NT, 1)
k2_q1col(Params p, const __grid_constant__ CUtensorMap tmu, double *__restrict__ dst, int64_t ntx,
         int64_t nty, int64_t nzc) {
  using G = Q1Geo;
  // interior tile: its loaded window [x0 - GX, x0 - GX + PX) x [y0 - GY, y0 - GY + BOXY)
  // lies in [1, n] in x and y (same tile arithmetic as the body)
  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2;
  const int item = blockIdx.x;
  const int tx = item % (int)ntx, ty = (item / (int)ntx) % (int)nty;
  const int x0 = (int)(2 * (((int64_t)tx * (Sx / 2)) / ntx));
  const int y0 = (int)(((int64_t)ty * Sy) / nty);
  const bool edge = x0 - G::GX < 1 || x0 - G::GX + G::PX > (int)p.nx + 1 || y0 - G::GY < 1 ||
                    y0 - G::GY + G::BOXY > (int)p.ny + 1;
  if (edge)
    q1col_body<FORM, UNIT, DIV, PEER, true>(p, tmu, dst, ntx, nty, nzc);
  else
    q1col_body<FORM, UNIT, DIV, PEER, false>(p, tmu, dst, ntx, nty, nzc);
}

}  // namespace sl
