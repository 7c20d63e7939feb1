// k2_col3d.cuh — K2 for the 3D 7-point stencil (BASELINE config 3):
// column-owning 2.5D streaming with TMA plane loads.
//
// A CTA owns a 64 x 32 tile of (x, y) columns (plus the ghost margin of the
// plan) and a chunk of z.  Thread (warp w, lane i) owns column pair
// (2i, 2i+1) of tile rows r0 = 2w + delta and r0 + 1, where delta makes row r0
// a y-parity 0 row; so at every plane the red point of each row sits at a
// compile-time column of the pair.  For the face stencil every z-neighbour of
// a point lies in its own column, so each thread keeps its 2 x 2 columns for
// planes t-3 .. t+1 in a register ring; of the in-plane neighbours, the one
// inside the pair and the one in the thread's other row come from registers,
// the rest (row of the warp above/below, column across the pair) from shared
// memory.
//
// Lags are spread (plan.cuh, spread = true): red updates plane t, black
// updates plane t-2, so both colours run between two block barriers:
//   * red at plane t reads black neighbours (old values: the plane as loaded)
//     and writes its result to registers and to the plane's smem slot;
//   * black at plane t-2 reads red neighbours updated two steps earlier; its
//     result is final for this pass and only goes to registers;
//   * plane t-2 is then complete and is stored from registers (STG.128).
// u and f planes arrive by TMA (cp.async.bulk.tensor.3d, 64x33x1 boxes,
// out-of-range parts zero-filled) into a ring of R = 6 smem slots each, issued
// D = 2 planes ahead by one thread, completion tracked by mbarriers.  The step
// loop is unrolled by R with every slot's plane parity fixed at compile time.
// Ghost points are computed and masked; the exact-division fallback runs out
// of line, per warp, only when a used lane's operand leaves the fast range.
#pragma once
#include <cuda.h>

#include "plan.cuh"

namespace sl {

struct Col3Geo {
  static constexpr FPlan P = make_plan(FD7, 2, 1, true);  // lags {0, 2}
  static constexpr int LAGMAX = P.lagmax;
  static constexpr int GX = 2, GY = 2, GZ = 2;             // load margins (plan: 2/2/2)
  static constexpr int PX = 64, PY = 32;
  static constexpr int BOXY = PY + 1;                      // rows loaded (delta shift)
  static constexpr int TX = PX - 2 * GX, TY = PY - 2 * GY;
  static constexpr int R = 6;                              // ring length (registers, smem slots)
  static constexpr int D = 2;                              // TMA lookahead beyond plane t+1
  static constexpr int RT = 2;                             // tile rows per thread (r0, r0 + 1)
  static constexpr int NT = 32 * PY / RT;
  static constexpr int SLOTE = PX * BOXY;                  // doubles per plane slot
  static constexpr int PADE = 2 * PX;                      // guard elements before/after the ring
  static constexpr size_t SMEM = size_t(2 * R * SLOTE + 2 * PADE) * sizeof(double) + 2 * R * 8;
  static_assert(P.lag[0] == 0 && P.lag[1] == 2 && LAGMAX == 2, "unexpected FD7 plan");
  static_assert(P.load[0] <= GX && P.load[1] <= GY && P.load[2] <= GZ, "ghost margin");
  static_assert(R >= LAGMAX + 3 + 1 && R >= D + 4, "ring too short");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// Exact division out of line (rare fallback of the Markstein fast path).
static __device__ __noinline__ double col3_div_exact(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int x, int y, int z,
                                            uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(mbar)
      : "memory");
}

__device__ __forceinline__ void mbar_init3(uint32_t addr) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(addr) : "memory");
}

__device__ __forceinline__ void mbar_expect3(uint32_t addr, uint32_t bytes) {
  sl_fuzz(220000u);   // before a slot is re-armed and refilled
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait3(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW3_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W3_%=;\n}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
  sl_fuzz(210000u);
}

template <int FORM, bool UNIT, int DIV, bool PEER = false>
__global__ void __launch_bounds__(Col3Geo::NT, 1)
k2_col3d_fd7(Params p, const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmf,
             double *__restrict__ dst, int64_t ntx, int64_t nty, int64_t nzc) {
  using G = Col3Geo;
  constexpr int R = G::R, D = G::D;
  extern __shared__ __align__(128) double csm[];
  double *su = csm + G::PADE;            // u slots: su + k*SLOTE
  double *sf = su + R * G::SLOTE;        // f slots
  uint64_t *mb = reinterpret_cast<uint64_t *>(sf + R * G::SLOTE + G::PADE);
  const uint32_t su_s = (uint32_t)__cvta_generic_to_shared(su);
  const uint32_t sf_s = (uint32_t)__cvta_generic_to_shared(sf);
  const uint32_t mb_s = (uint32_t)__cvta_generic_to_shared(mb);  // R u-barriers, then R f-barriers

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
  const int r0 = G::RT * warp + delta;

  // ring slot k holds plane t_begin + k (mod R); plane parity of slot k is k & 1
  int t_begin = z0 - G::GZ - 1;
  if ((t_begin - 1 + p.pz) & 1) --t_begin;
  const int t_end = z1 - 1 + G::LAGMAX;
  const int zlim = z1 + G::GZ;  // planes >= zlim are never needed

  auto issue_u = [&](int plane, int sl) {
    const uint32_t bar = mb_s + 8u * sl;
    const bool live = plane >= 0 && plane < Sz && plane < zlim;
    mbar_expect3(bar, live ? (uint32_t)(G::SLOTE * 8) : 0u);
    if (live) tma_load_3d(su_s + sl * G::SLOTE * 8, &tmu, gx0, gy0, plane, bar);
  };
  auto issue_f = [&](int plane, int sl) {
    const uint32_t bar = mb_s + 8u * (R + sl);
    const bool live = FORM == 1 && plane >= 1 && plane <= nz && plane < zlim;
    mbar_expect3(bar, live ? (uint32_t)(G::SLOTE * 8) : 0u);
    if (live) tma_load_3d(sf_s + sl * G::SLOTE * 8, &tmf, gx0, gy0, plane, bar);
  };

  if (threadIdx.x == 0) {
    for (int k = 0; k < 2 * R; ++k) mbar_init3(mb_s + 8u * k);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // u planes t_begin+1 .. t_begin+1+D, f planes t_begin .. t_begin+D
    for (int k = 1; k <= 1 + D; ++k) issue_u(t_begin + k, k % R);
    for (int k = 0; k <= D; ++k) issue_f(t_begin + k, k % R);
  }
  __syncthreads();

  // masks: bit (2a + s) of redok / blkok = point (row r0+a, column s) is in the
  // colour's need window and the grid interior (x, y); own = row a is stored
  const int n0x = G::P.need[0][0], n0y = G::P.need[0][1], n0z = G::P.need[0][2];
  unsigned redok = 0, blkok = 0, own = 0;
  const bool xown = 2 * lane >= G::GX && 2 * lane < G::GX + TXo;
  int64_t rowoff[G::RT];
#pragma unroll
  for (int a = 0; a < G::RT; ++a) {
    const int ly = r0 + a, gy = gy0 + ly;
    const bool yin = gy >= 1 && gy <= ny;
    const bool row0 = ly >= G::GY - n0y && ly < G::GY + TYo + n0y && yin;
    const bool row1 = ly >= G::GY && ly < G::GY + TYo && yin;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int lx = 2 * lane + s;
      const bool xin = gx + s >= 1 && gx + s <= nx;
      if (row0 && lx >= G::GX - n0x && lx < G::GX + TXo + n0x && xin) redok |= 1u << (2 * a + s);
      if (row1 && lx >= G::GX && lx < G::GX + TXo && xin) blkok |= 1u << (2 * a + s);
    }
    if (xown && ly >= G::GY && ly < G::GY + TYo) own |= 1u << a;
    rowoff[a] = (int64_t)gy * p.sy + gx;
  }
  const int me = r0 * G::PX + 2 * lane;  // element offset of (row r0, col 2*lane) in a slot

  double U[G::RT][R][2];
#pragma unroll
  for (int a = 0; a < G::RT; ++a)
#pragma unroll
    for (int k = 0; k < R; ++k) U[a][k][0] = U[a][k][1] = 0.0;

  unsigned emax = 0;   // max exponent field of any used update (0x7ff00000 = non-finite)
  // the dividend of one update of the point at row a, column s of ring slot
  // SC (neighbour slots SM/SP); the slot's smem copy supplies the other rows
  auto dividend = [&]<int a, int s, int SC, int SM, int SP>(double fc) -> double {
    const double *pl = su + SC * G::SLOTE + me + a * G::PX + s;
    double acc = acc_init<FORM, UNIT>(U[a][SC][s], p);
    acc = acc_add<FORM, UNIT>(acc, U[a][SM][s], 0, p);                             // (0,0,-1)
    acc = acc_add<FORM, UNIT>(acc, a == 1 ? U[0][SC][s] : pl[-G::PX], 1, p);       // (0,-1,0)
    acc = acc_add<FORM, UNIT>(acc, s == 1 ? U[a][SC][0] : pl[-1], 2, p);           // (-1,0,0)
    acc = acc_add<FORM, UNIT>(acc, s == 0 ? U[a][SC][1] : pl[1], 3, p);            // (1,0,0)
    acc = acc_add<FORM, UNIT>(acc, a == 0 ? U[1][SC][s] : pl[G::PX], 4, p);        // (0,1,0)
    acc = acc_add<FORM, UNIT>(acc, U[a][SP][s], 5, p);                             // (0,0,1)
    return FORM == 0 ? acc : __dsub_rn(fc, acc);
  };
  // x / w_c for four updates; the exact fallback is taken per warp, and only
  // for lanes whose result is used
  auto divide4 = [&](const double (&x)[4], const bool (&ok)[4], double (&q)[4]) {
    if (DIV == DIV_RCP) {
      bool slow = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double e = __dmul_rn(x[i], p.rwc);
        q[i] = __fma_rn(__fma_rn(-p.wc, e, x[i]), p.rwc, e);
        const unsigned xe = ((unsigned)__double2hiint(x[i]) >> 20) & 0x7ffu;
        slow |= ok[i] && (xe - 64u) >= 1919u;
      }
      if (__builtin_expect(__any_sync(0xffffffffu, slow), 0)) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const unsigned xe = ((unsigned)__double2hiint(x[i]) >> 20) & 0x7ffu;
          if (ok[i] && (xe - 64u) >= 1919u) q[i] = col3_div_exact(x[i], p.wc);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) q[i] = DIV == DIV_POW2 ? __dmul_rn(x[i], p.rwc) : col3_div_exact(x[i], p.wc);
    }
  };
  // commit: the new value (or the old one where the point is not used)
  auto commit = [&]<int a, int s, int SC>(double q, bool ok) -> double {
    const double uc = U[a][SC][s];
    const double out = FORM == 0 ? q : __dadd_rn(uc, __dmul_rn(p.omega, q));
    emax = max(emax, ok ? ((unsigned)__double2hiint(out) & 0x7ff00000u) : 0u);
    const double v = ok ? out : uc;
    U[a][SC][s] = v;
    return v;
  };

  uint32_t round = 0;
  for (int t0 = t_begin; t0 <= t_end; t0 += R, ++round) {
    [&]<int... Ks>(std::integer_sequence<int, Ks...>) {
      (
          [&] {
            constexpr int KS = Ks;
            const int t = t0 + KS;
            // the unrolled round is left at the chunk's last step (CTA-uniform): a thin
            // slab's chunk is ~28 steps, so rounding up to R = 6 would cost it up to 18 %
            if (t > t_end) return;
            constexpr int S1 = (KS + 1) % R, S0 = KS % R, SM1 = (KS + R - 1) % R;
            constexpr int SM2 = (KS + R - 2) % R, SM3 = (KS + R - 3) % R;
            // ---- plane t+1: smem slot -> register ring (use count of slot S1) ----
            {
              const uint32_t use = round + (uint32_t)((KS + 1) / R);
              mbar_wait3(mb_s + 8u * S1, (use - (S1 == 0 ? 1u : 0u)) & 1u);
#pragma unroll
              for (int a = 0; a < G::RT; ++a) {
                const double2 v = *reinterpret_cast<const double2 *>(su + S1 * G::SLOTE + me + a * G::PX);
                U[a][S1][0] = v.x;
                U[a][S1][1] = v.y;
              }
            }
            if (FORM == 1) {
              const uint32_t use = round + (uint32_t)(KS / R);
              mbar_wait3(mb_s + 8u * (R + S0), use & 1u);
            }
            constexpr int qz = KS & 1;  // (t - 1 + pz) & 1
            // red (colour 0) at plane t: row a holds it at column 1 ^ ((a + qz) & 1);
            // black (colour 1) at plane t-2 at the other column
            constexpr int rs0 = 1 ^ qz, rs1 = qz, bs0 = qz, bs1 = 1 ^ qz;
            const int pz = t - 2;
            const bool rz = t >= 1 && t <= nz && t >= z0 - n0z && t < z1 + n0z;
            const bool bz = pz >= 1 && pz <= nz && pz >= z0 && pz < z1;
            double x[4], q[4];
            bool ok[4];
            {
              const double *fr = sf + S0 * G::SLOTE + me, *fb = sf + SM2 * G::SLOTE + me;
              x[0] = dividend.template operator()<0, rs0, S0, SM1, S1>(FORM == 1 ? fr[rs0] : 0.0);
              x[1] = dividend.template operator()<1, rs1, S0, SM1, S1>(FORM == 1 ? fr[G::PX + rs1] : 0.0);
              x[2] = dividend.template operator()<0, bs0, SM2, SM3, SM1>(FORM == 1 ? fb[bs0] : 0.0);
              x[3] = dividend.template operator()<1, bs1, SM2, SM3, SM1>(FORM == 1 ? fb[G::PX + bs1] : 0.0);
              ok[0] = rz && ((redok >> rs0) & 1u);
              ok[1] = rz && ((redok >> (2 + rs1)) & 1u);
              ok[2] = bz && ((blkok >> bs0) & 1u);
              ok[3] = bz && ((blkok >> (2 + bs1)) & 1u);
            }
            divide4(x, ok, q);
            // red results are published for the warps above/below and the lanes beside
            su[S0 * G::SLOTE + me + rs0] = commit.template operator()<0, rs0, S0>(q[0], ok[0]);
            su[S0 * G::SLOTE + me + G::PX + rs1] = commit.template operator()<1, rs1, S0>(q[1], ok[1]);
            commit.template operator()<0, bs0, SM2>(q[2], ok[2]);
            commit.template operator()<1, bs1, SM2>(q[3], ok[3]);
            // ---- plane t-2 is final: owned rows -> dst ----
            if (pz >= z0 && pz < z1) {
#pragma unroll
              for (int a = 0; a < G::RT; ++a)
                if ((own >> a) & 1u) {
                  const int64_t e = (int64_t)pz * p.sz + rowoff[a];
                  stg_pair(dst + e, U[a][SM2][0], U[a][SM2][1]);
                  stg_pair_peers<PEER>(p, pz, e, U[a][SM2][0], U[a][SM2][1]);
                }
            }
#if SL_FUZZ_BREAK != 3
            __syncthreads();
#endif
            // slots of planes t-3 (u) / t-4 (f) are free: refill them D planes ahead
            if (threadIdx.x == 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue_u(t + 2 + D, (KS + 2 + D) % R);
              issue_f(t + 1 + D, (KS + 1 + D) % R);
            }
          }(),
          ...);
    }(std::make_integer_sequence<int, R>{});
  }
  // drain the copies still in flight before the CTA exits
  if (threadIdx.x == 0) {
    const int tl = t_end + 1;  // first unprocessed step
    for (int k = 0; k <= D; ++k) {
      const int pu = tl + 1 + k, pf = tl + k;
      const int su_i = (pu - t_begin) % R, sf_i = (pf - t_begin) % R;
      mbar_wait3(mb_s + 8u * su_i, (uint32_t)(((pu - t_begin) / R - (su_i == 0 ? 1 : 0)) & 1));
      mbar_wait3(mb_s + 8u * (R + sf_i), (uint32_t)(((pf - t_begin) / R) & 1));
    }
  }
  __syncthreads();
  if (__any_sync(0xffffffffu, emax == 0x7ff00000u) && lane == 0) atomicOr(p.status, 1);
}

}  // namespace sl
