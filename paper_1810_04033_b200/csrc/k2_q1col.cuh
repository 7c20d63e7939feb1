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
// A + 2).  (The geometry is a set of build-time constants, Q1Geo below: CPL
// columns per lane, LX lanes along x and 32/LX lane rows per warp.)  The thread keeps its rows of planes p-2 .. p in a register ring
// (plane p+1, read only by G0/G1, comes from its slot); otherwise only the
// row of the warp above/below comes from the plane's shared-memory slot, and
// the x+-1 columns from warp shuffles.  Neighbour values enter the sums as
// weighted products computed once per value and weight and shared (by
// shuffle) with the lanes that need them.  Every update is published to the
// slot for the neighbouring warps.
//
// u planes arrive by TMA (64 x 49 x 1 boxes, zero-filled out of range) into
// 8 smem slots, up to six planes ahead.  One pair step per loop iteration:
// the ring entries have fixed roles (planes pp-2, pp-1, pp) and plane pp moves
// to entry 0 at the end of the step; slot offsets and mbarrier parities are
// cheap runtime values.  Out-of-range groups and ghost
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

// Build-time geometry (A/B switches).  Default: a lane owns a column pair
// (CPL = 2), a warp is 32 lanes along x, 12 warps cover a 64 x 48 tile (384
// threads, 168 registers, 8 plane slots).  Measured alternatives on config 4
// (all bitwise equal, all slower than the default's 140 GLUP/s):
//   -DQ1_CPL=4 -DQ1_LX=16 -DQ1_PY=64 -DQ1_S=6 -DQ1_SHIFT=1   lanes own four
//     columns (half the shuffles per point), warps are 16 x 2 lanes, 8 warps
//     cover 64 x 64 (256 threads, 255 registers): 125 GLUP/s, 127 with
//     -DQ1_NOSWAP (2-way LDS/STS.128 bank conflicts instead of register swaps);
//   the same with -DQ1_RT=2 (16 warps, 128 registers): 118 GLUP/s.
#ifndef Q1_CPL
#define Q1_CPL 2
#endif
#ifndef Q1_LX
#define Q1_LX 32
#endif
#ifndef Q1_PY
#define Q1_PY 48
#endif
#ifndef Q1_S
#define Q1_S 8
#endif
#ifndef Q1_RT
#define Q1_RT 4
#endif
// Q1_SHIFT = 1: the loaded window starts on a y-parity-0 row (its origin moves
// up by the tile's parity offset delta), so PY rows are loaded instead of
// PY + 1 and a tile owns at most PY - 2 GY - 1 rows.
#ifndef Q1_SHIFT
#define Q1_SHIFT 0
#endif
// Q1_CLUSTER = 1 (A/B): CTAs run as thread-block clusters of two along y.  The
// pair shares its facing edge: neither CTA carries ghost rows there; each
// reads the other's boundary row from one extra row of its own plane slots,
// which the owner refreshes with st.shared::cluster after every group that
// updates it, and the three block barriers of a pair step become cluster
// barriers.  A pair owns up to 2 (PY - GY) - 2 rows for 2 PY computed rows.
#ifndef Q1_CLUSTER
#define Q1_CLUSTER 0
#endif
struct Q1Geo {
  static constexpr FPlan P = make_plan(Q1, 8, 1, false);
  static constexpr bool CL = Q1_CLUSTER != 0;
  static constexpr int GX = 4, GY = 4, GZ = 2;            // plan load margins
  static constexpr int CPL = Q1_CPL;                      // columns per lane
  static constexpr int LX = Q1_LX, LY = 32 / LX;          // lanes along x / lane rows per warp
  static constexpr int PX = CPL * LX, PY = Q1_PY;         // tile incl. ghost
  static constexpr bool SHIFT = Q1_SHIFT != 0;
  static constexpr int BOXY = SHIFT ? PY : PY + 1;        // rows loaded
  // rows owned per tile (per pair of tiles with CL)
  static constexpr int TX = PX - 2 * GX, TY = CL ? 2 * (PY - GY) - 2 : PY - 2 * GY - (SHIFT ? 1 : 0);
  static constexpr int S = Q1_S;                          // smem slots (4 live planes + S - 4 ahead)
  static constexpr int RR = 4;                            // ring entries (planes p-2 .. p live)
  static constexpr int RT = Q1_RT;                        // tile rows per thread
  static constexpr int NT = 32 * PY / (RT * LY);
  static constexpr int LAGMAX = 1;
  static constexpr int SLOTE = PX * BOXY;
  static constexpr int LEADE = 2 * PX;                    // guard rows before slot 0
  static constexpr int FBUFE = 2 * (RT / 2) * CPL * NT;   // f staging: 2 buffers x H rows x PX cols per lane row
  static constexpr size_t SMEM = size_t(LEADE + S * SLOTE + 2 * PX + FBUFE) * sizeof(double) + S * 8 + (CL ? 4 * 8 : 0);
  static_assert(P.load[0] <= GX && P.load[1] <= GY && P.load[2] <= GZ, "ghost margin");
  static_assert(CPL % 2 == 0 && LX * LY == 32 && PY % (RT * LY) == 0 && S >= 6 && (S & 1) == 0, "geometry");
  static_assert(4 * (RT / 2) * CPL <= 32 && RT * CPL <= 32, "mask bits");
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(!CL || (CPL == 2 && !SHIFT && LX == 32), "cluster pairs: column-pair geometry only");
};

__device__ __forceinline__ void q1_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store a value pair at the same shared-memory offset in CTA `peer` of the cluster
__device__ __forceinline__ void q1_push_pair(const double *own, unsigned peer, double a, double b) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((uint32_t)__cvta_generic_to_shared(own)), "r"(peer));
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(a), "d"(b) : "memory");
}

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
  constexpr int RT = G::RT, H = RT / 2, C = G::CPL, CP = C / 2;
  constexpr int RR = 3;   // ring entries: planes pp-2, pp-1, pp
  static_assert(CP == 1 || CP == 2, "columns per lane");
  extern __shared__ __align__(128) double qsm[];
  double *su = qsm + G::LEADE;  // slot k at su + k*SLOTE
  double *fbuf = su + G::S * G::SLOTE + 2 * G::PX;   // [lane row][h][PX]
  uint64_t *mb = reinterpret_cast<uint64_t *>(fbuf + G::FBUFE);
  const uint32_t su_s = (uint32_t)__cvta_generic_to_shared(su);
  const uint32_t mb_s = (uint32_t)__cvta_generic_to_shared(mb);

  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2, Sz = (int)p.nz + 2;
  const int nx = (int)p.nx, ny = (int)p.ny, nz = (int)p.nz;
  const int item = G::CL ? blockIdx.x >> 1 : blockIdx.x;
  const int crank = G::CL ? (int)(blockIdx.x & 1) : 0;   // rank in the cluster pair (CL)
  const int tx = item % (int)ntx, ty = (item / (int)ntx) % (int)nty, zc = item / (int)(ntx * nty);
  const int x0 = (int)(2 * (((int64_t)tx * (Sx / 2)) / ntx)), x1 = (int)(2 * (((int64_t)(tx + 1) * (Sx / 2)) / ntx));
  int y0 = (int)(((int64_t)ty * Sy) / nty), y1 = (int)(((int64_t)(ty + 1) * Sy) / nty);
  // CL: [y0, y1) is the pair's range; it is split at ymid, a row of y parity 0,
  // rank 0 computes the PY rows below ymid (global ymid - PY .. ymid - 1), rank 1
  // the PY rows from ymid on
  int ymid = 0;
  if (G::CL) {
    ymid = (y0 + y1) / 2;
    if ((ymid - 1 + p.py) & 1) ++ymid;
    if (crank == 0) y1 = ymid; else y0 = ymid;
  }
  const int zlen = p.zhi - p.zlo;
  const int z0 = p.zlo + (int)(((int64_t)zc * zlen) / nzc), z1 = p.zlo + (int)(((int64_t)(zc + 1) * zlen) / nzc);
  const int TXo = x1 - x0, TYo = y1 - y0;
  const int gx0 = x0 - G::GX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lx = lane % G::LX;                   // lane along x: columns C*lx .. C*lx + C - 1
  const int vrow = warp * G::LY + lane / G::LX;  // band of RT rows
  const int gx = gx0 + C * lx;
  // local row r0 has y parity 0; the tile's first owned row is local row TM
  // CL: rank 0's local rows 0 .. PY-1 end at the shared edge and local row PY
  // is rank 1's first row; rank 1's local row 0 is rank 0's last row and its
  // own rows are 1 .. PY
  const int delta = G::CL ? crank : (1 - p.py - (y0 - G::GY)) & 1;
  const int gy0 = G::CL ? (crank == 0 ? ymid - G::PY : ymid - 1) : G::SHIFT ? y0 - G::GY - delta : y0 - G::GY;
  const int TM = G::CL ? y0 - gy0 : G::SHIFT ? G::GY + delta : G::GY;
  const int r0 = G::SHIFT ? RT * vrow : RT * vrow + delta;   // this thread's rows r0 (qy 0) .. r0 + RT - 1
  // no ghost rows (and no decay of the need region) on the side shared with the cluster peer
  const bool sh_lo = G::CL && crank == 1, sh_hi = G::CL && crank == 0;
  // CL: the warp that owns the row facing the peer — the only one that reads the
  // peer's row and stores into the peer's slots.  It synchronises with the peer's
  // boundary warp only: after a group in which it stores, every lane arrives
  // (release, cluster scope) on the peer's handshake barrier of that group; before
  // a group in which it reads the peer's row it waits for the peer's previous group.
  // rank 0 stores after G1/G3 and reads in G1/G3, rank 1 stores after G0/G2 and reads
  // in G0/G2, so each side's wait also keeps its next store behind the peer's reads
  // of the old value, and neither side can lead by two groups (no phase aliasing).
  const bool bwarp = G::CL && (crank == 0 ? vrow == G::PY / RT - 1 : vrow == 0);
  const uint32_t hb_s = mb_s + 8u * G::S;
  auto pair_arrive = [&](int g) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(hb_s + 8u * g), "r"((unsigned)(crank ^ 1)));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
  };
  auto pair_wait = [&](int g, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nHW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra HW_%=;\n}\n" ::"r"(hb_s + 8u * g),
        "r"(parity)
        : "memory");
    sl_fuzz(320000u);
  };
  uint32_t step = 0;   // pair steps completed (CL handshake phase)
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

  auto slot_idx = [&](int plane) -> int { return (int)((unsigned)(plane - base) % (unsigned)G::S); };
  auto issue = [&](int plane) {
    const int sl = slot_idx(plane);
    const uint32_t bar = mb_s + 8u * sl;
    const bool live = plane >= 0 && plane < Sz && plane < zlim;
    mbar_expect3(bar, live ? (uint32_t)(G::SLOTE * 8) : 0u);
    if (live) tma_load_3d(su_s + sl * G::SLOTE * 8, &tmu, gx0, gy0, plane, bar);
  };
  auto wait_plane = [&](int plane) {
    mbar_wait3(mb_s + 8u * (uint32_t)slot_idx(plane), ((unsigned)(plane - base) / (unsigned)G::S) & 1u);
  };
  // A lane's C = 4 columns are two 16-byte pairs, 32 bytes from the next
  // lane's: eight lanes all accessing "pair 0" would use only every other
  // 16-byte bank group (a 2-way conflict on every LDS/STS.128).  Lanes 4..7 of
  // every eight therefore access their pairs in the opposite order (qsw) and
  // swap in registers: first access at element qa, second at qb.
#ifdef Q1_NOSWAP
  const bool qsw = false;
#else
  const bool qsw = CP == 2 && ((lx >> 2) & 1);
#endif
  const int qa = qsw ? 2 : 0, qb = CP == 2 ? 2 - qa : 0;
  double *me = su + r0 * G::PX + C * lx;  // (slot 0, row r0, first column of the lane)
  auto slot_of = [&](int plane) -> double * { return me + slot_idx(plane) * G::SLOTE; };
  auto ld_row = [&](const double *row, double (&v)[C]) {   // row: the lane's first column
    if constexpr (CP == 1) {
      const double2 m = *reinterpret_cast<const double2 *>(row);
      v[0] = m.x;
      v[1] = m.y;
    } else {
      const double2 a = *reinterpret_cast<const double2 *>(row + qa);
      const double2 b = *reinterpret_cast<const double2 *>(row + qb);
      v[0] = qsw ? b.x : a.x;
      v[1] = qsw ? b.y : a.y;
      v[2] = qsw ? a.x : b.x;
      v[3] = qsw ? a.y : b.y;
    }
  };
  auto st_row = [&](double *row, const double (&v)[C]) {
    if constexpr (CP == 1) {
      *reinterpret_cast<double2 *>(row) = make_double2(v[0], v[1]);
    } else {
      *reinterpret_cast<double2 *>(row + qa) = make_double2(qsw ? v[2] : v[0], qsw ? v[3] : v[1]);
      *reinterpret_cast<double2 *>(row + qb) = make_double2(qsw ? v[0] : v[2], qsw ? v[1] : v[3]);
    }
  };

  if (threadIdx.x == 0) {
    for (int k = 0; k < G::S; ++k) mbar_init3(mb_s + 8u * k);
    if constexpr (G::CL)   // handshake barriers of the cluster pair: one per group, 32 arrivals (a warp)
      for (int k = 0; k < 4; ++k)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(mb_s + 8u * (G::S + k)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < G::S - 2; ++k) issue(base + k);  // planes p_begin-2 .. p_begin+S-5
  }
  __syncthreads();

  // ---- thread-constant masks ------------------------------------------------
  // ok bit ((gi*H + h)*C + s): point s of the h-th row (A + 2h) of group gi
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
      const bool rok = r >= TM - (sh_lo ? 0 : nyj) && r < TM + TYo + (sh_hi ? 0 : nyj) && gy >= 1 && gy <= ny;
#pragma unroll
      for (int s = 0; s < C; ++s) {
        const int lc = C * lx + s;
        const bool cok = lc >= G::GX - nxj && lc < G::GX + TXo + nxj && gx + s >= 1 && gx + s <= nx;
        okbits |= (rok && cok) ? (1u << ((gi * H + h) * C + s)) : 0u;
      }
    }
  }
  // owned output rows and column pairs (the tiles partition [0, S) in x and
  // y; tile starts are even, so a pair is owned as a whole): bit a*CP + pair
  unsigned ownbits = 0, fokbits = 0;
  const int64_t rowoff0 = (int64_t)(gy0 + r0) * p.sy + gx;   // row r0 of this thread
  const int sy32 = (int)p.sy;
  unsigned inbits = 0;   // interior (updated) points: bit C*a + s
#pragma unroll
  for (int a = 0; a < RT; ++a) {
    const int r = r0 + a, gy = gy0 + r;
#pragma unroll
    for (int pr = 0; pr < CP; ++pr) {
      const int lc = C * lx + 2 * pr;
      const bool colown = lc >= G::GX && lc < G::GX + TXo;
      ownbits |= (colown && r >= TM && r < TM + TYo) ? (1u << (a * CP + pr)) : 0u;
      // f is staged by 16-byte chunks of the lane row's PX columns: this lane copies chunks lx + LX*pr
      const int fc = gx0 + 2 * (lx + G::LX * pr);
      fokbits |= (gy >= 0 && gy < Sy && fc >= 0 && fc + 1 < Sx) ? (1u << (a * CP + pr)) : 0u;
    }
#pragma unroll
    for (int s = 0; s < C; ++s)
      inbits |= (gy >= 1 && gy <= ny && gx + s >= 1 && gx + s <= nx) ? (1u << (C * a + s)) : 0u;
  }

  // own rows of planes pp-2, pp-1, pp: [row][ring entry][col] (plane pp+1, read
  // only by G0/G1, comes from its slot).  Entry 0 survives a pair step (it is
  // the previous step's plane pp), entries 1 and 2 are loaded at its start.
  double U[RT][RR][C];
  wait_plane(base);
  wait_plane(base + 1);
  {
    const double *pl = slot_of(base);
#pragma unroll
    for (int a = 0; a < RT; ++a) ld_row(pl + a * G::PX, U[a][0]);
  }

  // f rows of group gi at plane pz (rows A + 2h) are staged per lane row (the
  // LX lanes that share a band of rows) in shared memory by cp.async, one
  // group ahead of their use, alternating between two buffers (the groups of
  // a pair step use buffers 0, 1, 0, 1).  The lanes copy the row's PX columns
  // as consecutive 16-byte chunks (coalesced: chunk lx + LX*j by lane lx) and
  // each lane reads its own columns.  cp.async.wait_group 1 waits for exactly
  // the older copy, so the newest one in flight never delays a consumer, and
  // it does not matter where in the group the scheduler places the wait (a
  // wait for a copy issued in the same group gets hoisted right behind it; a
  // register LDG would share its scoreboard with the plane loads).  Masked
  // chunks are zero-filled (src size 0).  __syncwarp orders the lanes' copies
  // and reads.
  const double *fthr = p.f + (int64_t)(gy0 + r0) * p.sy + gx0 + 2 * lx;
  double *frow = fbuf + vrow * (2 * H * G::PX);
  const uint32_t fb_s = (uint32_t)__cvta_generic_to_shared(frow) + 16u * lx;
  auto issue_f = [&](int gi, int pz, int buf) {
    const int A = gi & 1;
    const bool zin = pz >= 0 && pz < Sz;
    __syncwarp();   // every lane has read this buffer's previous contents
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int pr = 0; pr < CP; ++pr) {
        const bool live = FORM == 1 && ((fokbits >> ((A + 2 * h) * CP + pr)) & 1u) && zin;
        const double *fp = live ? fthr + (int64_t)pz * sz + (A + 2 * h) * sy32 + 2 * G::LX * pr : p.u;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         fb_s + 8u * ((buf * H + h) * G::PX + 2 * G::LX * pr)),
                     "l"(fp), "r"(live ? 16 : 0)
                     : "memory");
      }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto read_f = [&](int buf, double (&fv)[H][C]) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();   // the other lanes' chunks have landed too
#pragma unroll
    for (int h = 0; h < H; ++h) ld_row(frow + (buf * H + h) * G::PX + C * lx, fv[h]);
  };
  if (FORM == 1) issue_f(0, p_begin, 0);

  // compact Q1 order: index 0 = (-1,-1,-1) corner, 1 = (0,-1,-1) edge
  const double wC = FORM == 0 ? p.aw[0] : p.w[0];
  const double wE = FORM == 0 ? p.aw[1] : p.w[1];
  unsigned emax = 0;   // max exponent field of any used update (0x7ff00000 = non-finite)

  // one colour group GI at plane pz = pp - (GI >> 1); RP = ring entry of pp
  auto group = [&]<int GI, int RP>(int pp) {
    constexpr int A = GI & 1;                      // rows A, A + 2
    constexpr int LAGG = GI >> 1;
    if constexpr (G::CL) {
      if (bwarp) {   // the peer's previous group (its stores into this CTA's slots) is complete
        if (crank == 0 && A == 1) pair_wait(GI - 1, step & 1u);
        if (crank == 1 && GI == 2) pair_wait(1, step & 1u);
        if (crank == 1 && GI == 0 && step > 0) pair_wait(3, (step - 1u) & 1u);
      }
    }
    if (FORM == 1) {                               // next group's right-hand side in flight
      constexpr int NGI = (GI + 1) & 3;
      issue_f(NGI, GI == 0 ? pp : GI == 3 ? pp + 2 : pp - 1, NGI & 1);
    }
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
    double acc[H][C];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int s = 0; s < C; ++s) acc[h][s] = acc_init<FORM, UNIT>(U[A + 2 * h][RC][s], p);
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
        double v[C];
        if (d >= 0 && d < RT && !(LAGG == 0 && dz == 1)) {
#pragma unroll
          for (int s = 0; s < C; ++s) v[s] = U[d][rs][s];
        } else {
          ld_row(pl + d * G::PX, v);
        }
        // window columns -1 .. C (index + 1); the two outer ones come from the
        // neighbouring lanes of the same lane row
        double pe[C + 2], pc[C + 2];
#pragma unroll
        for (int s = 0; s < C; ++s) pe[s + 1] = UNIT ? v[s] : __dmul_rn(wE, v[s]);
        if (!UNIT && odd && dz != 0) {
#pragma unroll
          for (int s = 0; s < C; ++s) pc[s + 1] = __dmul_rn(wC, v[s]);
          pc[0] = __shfl_up_sync(0xffffffffu, pc[C], 1, G::LX);
          pc[C + 1] = __shfl_down_sync(0xffffffffu, pc[1], 1, G::LX);
        } else {
          pe[0] = __shfl_up_sync(0xffffffffu, pe[C], 1, G::LX);
          pe[C + 1] = __shfl_down_sync(0xffffffffu, pe[1], 1, G::LX);
#pragma unroll
          for (int s = 0; s < C + 2; ++s) pc[s] = pe[s];
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
            for (int s = 0; s < C; ++s) {
              const double t = corner ? pc[o.x + 1 + s] : pe[o.x + 1 + s];
              acc[h][s] = (FORM == 1 && UNIT) ? __dsub_rn(acc[h][s], t) : __dadd_rn(acc[h][s], t);
            }
          }
        }
      }
    }
    // division by w_c.  The fast-path range test ignores the lane masks (a
    // zero-filled point outside the grid only sends its warp into the
    // fallback, which applies them), so no mask is kept live across it.
    double fv[H][C];
    if (FORM == 1) read_f(GI & 1, fv);
    bool ok[H][C], slow = false;
    double a[H][C], q[H][C];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int s = 0; s < C; ++s) {
        ok[h][s] = !EDGE || ((okbits >> ((GI * H + h) * C + s)) & 1u);
        a[h][s] = FORM == 0 ? acc[h][s] : __dsub_rn(fv[h][s], acc[h][s]);
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
        for (int s = 0; s < C; ++s) {
          const unsigned xe = (unsigned)__double2hiint(a[h][s]) & 0x7ff00000u;
          if (ok[h][s] && (xe - (64u << 20)) >= (1919u << 20)) q[h][s] = q1_div_exact(a[h][s], p.wc);
        }
    }
    // commit: ring, publish to the plane's slot (a dropped plane gets its
    // unchanged values back from the slot)
    double *pcs = slot_of(pz);
#pragma unroll
    for (int h = 0; h < H; ++h) {
#pragma unroll
      for (int s = 0; s < C; ++s) {
        const double uc = U[A + 2 * h][RC][s];
        const double out = FORM == 0 ? q[h][s] : __dadd_rn(uc, __dmul_rn(p.omega, q[h][s]));
        U[A + 2 * h][RC][s] = (!EDGE || ok[h][s]) ? out : uc;
      }
    }
    if (pzin) {
#pragma unroll
      for (int h = 0; h < H; ++h) st_row(pcs + (A + 2 * h) * G::PX, U[A + 2 * h][RC]);
      if constexpr (G::CL) {
        // the row facing the cluster peer also goes into the peer's copy of it:
        // rank 0's last row (local PY - 1, updated by the A = 1 groups) is the
        // peer's local row 0; rank 1's first row (local 1, A = 0 groups) is the
        // peer's local row PY
        constexpr int AR = A == 1 ? RT - 1 : 0;   // this group's candidate row of the thread
        if (A == 1 && crank == 0 && vrow == G::PY / RT - 1)
          q1_push_pair(pcs + (AR - (G::PY - 1)) * G::PX, 1u, U[AR][RC][0], U[AR][RC][1]);
        if (A == 0 && crank == 1 && vrow == 0)
          q1_push_pair(pcs + (G::PY - 1) * G::PX, 0u, U[AR][RC][0], U[AR][RC][1]);
      }
    } else {
#pragma unroll
      for (int h = 0; h < H; ++h) ld_row(pcs + (A + 2 * h) * G::PX, U[A + 2 * h][RC]);
    }
    if constexpr (G::CL) {
      // this group's stores into the peer's slots and reads of the peer's row are done
      if (bwarp && (A == 1) == (crank == 0)) pair_arrive(GI);
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
#pragma unroll
        for (int pr = 0; pr < CP; ++pr)
          if ((ownbits >> (a * CP + pr)) & 1u) {
            stg_pair(dp + a * sy32 + 2 * pr, U[a][E][2 * pr], U[a][E][2 * pr + 1]);
            stg_pair_peers<PEER>(p, po, (int64_t)po * sz + rowoff0 + a * sy32 + 2 * pr, U[a][E][2 * pr],
                                 U[a][E][2 * pr + 1]);
            if (zin) {
#pragma unroll
              for (int s = 2 * pr; s < 2 * pr + 2; ++s) {
                const unsigned ex = (unsigned)__double2hiint(U[a][E][s]) & 0x7ff00000u;
                emax = max(emax, (!EDGE || ((inbits >> (C * a + s)) & 1u)) ? ex : 0u);
              }
            }
          }
    }
  };

  // between colour groups: the block's warps — and with CL the cluster peer, whose
  // boundary row each group may read — must have published the previous group
  auto group_sync = [&] {
    __syncthreads();   // CL: the cluster peer is ordered by the boundary warps' handshake
  };
  // one pair step per iteration (not unrolled: with four columns per lane a
  // second unrolled step made the loop outgrow the instruction cache —
  // no_instructions was the top stall — and the ring turn it saved is 2 % of
  // the step's instructions)
  constexpr int RP0 = 2, RM1 = 1;
  if constexpr (G::CL) {   // both CTAs run, and their first planes have landed, before any peer store
    wait_plane(p_begin);
    wait_plane(p_begin + 1);
    q1_cluster_sync();
  }
#pragma unroll 1
  for (int pp = p_begin; pp <= p_end; pp += 2) {
    // planes pp-1 and pp -> ring
    wait_plane(pp);
    wait_plane(pp + 1);
    {
      const double *pa = slot_of(pp - 1), *pb = slot_of(pp);
#pragma unroll
      for (int a = 0; a < RT; ++a) {
        ld_row(pa + a * G::PX, U[a][RM1]);
        ld_row(pb + a * G::PX, U[a][RP0]);
      }
    }
    group.template operator()<0, RP0>(pp);
    group_sync();
    // everybody is past the previous pair step: refill the slots of
    // planes pp-4, pp-3 with planes pp+S-4, pp+S-3
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(pp + G::S - 4);
      issue(pp + G::S - 3);
    }
    group.template operator()<1, RP0>(pp);
    // plane pp is final after G1
    store_plane(pp, std::integral_constant<int, RP0>{});
#if SL_FUZZ_BREAK != 1
    group_sync();
#endif
    group.template operator()<2, RP0>(pp);
    // CL: the peer stores its boundary row of plane pp+2 into this CTA's slot
    // when its next G0 ends; this CTA's own TMA copy of that plane (which
    // covers the same row) must have landed before, i.e. before the last
    // barrier the peer passes on its way there
    if constexpr (G::CL) {
      wait_plane(pp + 2);
      wait_plane(pp + 3);
    }
    group_sync();
    group.template operator()<3, RP0>(pp);
    store_plane(pp - 1, std::integral_constant<int, RM1>{});
    // plane pp is the next step's plane pp-2
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
      for (int c = 0; c < C; ++c) U[a][0][c] = U[a][RP0][c];
    ++step;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // drain the copies issued but never waited for
    const int pl_end = p_begin + ((p_end - p_begin) / 2 + 1) * 2;  // first pair step not run
    for (int pl = pl_end; pl <= pl_end + G::S - 5; ++pl) wait_plane(pl);
  }
  __syncthreads();
  if constexpr (G::CL) q1_cluster_sync();   // the peer may still be storing into this CTA's slots
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (__any_sync(0xffffffffu, emax == 0x7ff00000u) && lane == 0) atomicOr(p.status, 1);
}

template <int FORM, bool UNIT, int DIV, bool PEER = false>
__global__ void __launch_bounds__(Q1Geo::NT, 1)
k2_q1col(Params p, const __grid_constant__ CUtensorMap tmu, double *__restrict__ dst, int64_t ntx,
         int64_t nty, int64_t nzc) {
  using G = Q1Geo;
  // interior tile: its loaded window [x0 - GX, x0 - GX + PX) x [gy0, gy0 + BOXY)
  // lies in [1, n] in x and y (same tile arithmetic as the body)
  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2;
  const int item = G::CL ? blockIdx.x >> 1 : blockIdx.x;
  const int tx = item % (int)ntx, ty = (item / (int)ntx) % (int)nty;
  const int x0 = (int)(2 * (((int64_t)tx * (Sx / 2)) / ntx));
  const int y0 = (int)(((int64_t)ty * Sy) / nty);
  int gy0 = G::SHIFT ? y0 - G::GY - ((1 - p.py - (y0 - G::GY)) & 1) : y0 - G::GY;
  if (G::CL) {
    const int y1 = (int)(((int64_t)(ty + 1) * Sy) / nty);
    int ymid = (y0 + y1) / 2;
    if ((ymid - 1 + p.py) & 1) ++ymid;
    gy0 = (blockIdx.x & 1) == 0 ? ymid - G::PY : ymid - 1;
  }
  const bool edge = x0 - G::GX < 1 || x0 - G::GX + G::PX > (int)p.nx + 1 || gy0 < 1 ||
                    gy0 + G::BOXY > (int)p.ny + 1;
  if (edge)
    q1col_body<FORM, UNIT, DIV, PEER, true>(p, tmu, dst, ntx, nty, nzc);
  else
    q1col_body<FORM, UNIT, DIV, PEER, false>(p, tmu, dst, ntx, nty, nzc);
}

}  // namespace sl
