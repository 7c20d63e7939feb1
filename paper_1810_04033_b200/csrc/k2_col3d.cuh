// k2_col3d.cuh — K2 for the 3D 7-point stencil (BASELINE config 3):
// column-owning 2.5D streaming with TMA plane loads.
//
// A CTA owns a 64 x 32 tile of (x, y) columns (plus the ghost margin of the
// plan) and a chunk of z.  Thread (warp w, lane i) owns rows w and w+16 and
// column pair (2i, 2i+1) of the tile for the whole chunk.  For the face stencil every
// z-neighbour of a point lies in the same column, so each thread keeps its
// column's values for planes t-3 .. t+1 in a register ring; only in-plane
// (x+-1, y+-1) neighbours are read from shared memory.
//
// Lags are spread (plan.cuh, spread = true): red updates plane t, black
// updates plane t-2, so both colours run between two block barriers:
//   * red at plane t reads black neighbours (old values: the plane as loaded)
//     and writes its result to registers and to the plane's smem slot;
//   * black at plane t-2 reads red neighbours updated two steps earlier; its
//     result is final for this pass and only goes to registers;
//   * plane t-2 is then complete and is stored from registers (STG.128).
// u and f planes arrive by TMA (cp.async.bulk.tensor.3d, 64x32x1 boxes,
// out-of-range parts zero-filled) into a ring of R = 6 smem slots each, issued
// D = 2 planes ahead by one thread, completion tracked by mbarriers.  The step
// loop is unrolled by R with every slot's plane parity fixed at compile time.
#pragma once
#include <cuda.h>

#include "plan.cuh"

namespace sl {

struct Col3Geo {
  static constexpr FPlan P = make_plan(FD7, 2, 1, true);  // lags {0, 2}
  static constexpr int LAGMAX = P.lagmax;
  static constexpr int GX = 2, GY = 2, GZ = 2;             // load margins (plan: 2/2/2)
  static constexpr int PX = 64, PY = 32;
  static constexpr int TX = PX - 2 * GX, TY = PY - 2 * GY;
  static constexpr int R = 6;                              // ring length (registers, smem slots)
  static constexpr int D = 2;                              // TMA lookahead beyond plane t+1
  static constexpr int RT = 2;                             // tile rows per thread (w, w + PY/RT)
  static constexpr int NT = 32 * PY / RT;
  static constexpr int SLOTE = PX * PY;                    // doubles per plane slot
  static constexpr int PADE = 16;                          // guard elements before/after the ring
  static constexpr size_t SMEM = size_t(2 * R * SLOTE + 2 * PADE) * sizeof(double) + 2 * R * 8;
  static_assert(P.lag[0] == 0 && P.lag[1] == 2 && LAGMAX == 2, "unexpected FD7 plan");
  static_assert(P.load[0] <= GX && P.load[1] <= GY && P.load[2] <= GZ, "ghost margin");
  static_assert(R >= LAGMAX + 3 + 1 && R >= D + 4, "ring too short");
};

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
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait3(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW3_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W3_%=;\n}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

template <int FORM, bool UNIT, int DIV>
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
  const int z0 = (int)(((int64_t)zc * Sz) / nzc), z1 = (int)(((int64_t)(zc + 1) * Sz) / nzc);
  const int TXo = x1 - x0, TYo = y1 - y0;
  const int gx0 = x0 - G::GX, gy0 = y0 - G::GY;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx = gx0 + 2 * lane;

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

  // phase row/col windows (tile-local); red = phase 0 (need 1), black = phase 1 (need 0)
  const int n0x = G::P.need[0][0], n0y = G::P.need[0][1], n0z = G::P.need[0][2];
  auto colok = [&](int s, int need) -> bool {
    const int lx = 2 * lane + s;
    return lx >= G::GX - need && lx < G::GX + TXo + need && gx + s >= 1 && gx + s <= nx;
  };
  const bool xown = 2 * lane >= G::GX && 2 * lane < G::GX + TXo;
  int ly[G::RT], gy[G::RT], qy[G::RT], rowoff[G::RT];
  bool row0[G::RT], row1[G::RT], own_out[G::RT];
#pragma unroll
  for (int r = 0; r < G::RT; ++r) {
    ly[r] = warp + r * (G::PY / G::RT);
    gy[r] = gy0 + ly[r];
    qy[r] = (gy[r] - 1 + p.py) & 1;
    rowoff[r] = ly[r] * G::PX + 2 * lane;  // element offset of the thread's pair in a slot
    row0[r] = ly[r] >= G::GY - n0y && ly[r] < G::GY + TYo + n0y && gy[r] >= 1 && gy[r] <= ny;
    row1[r] = ly[r] >= G::GY && ly[r] < G::GY + TYo && gy[r] >= 1 && gy[r] <= ny;
    own_out[r] = ly[r] >= G::GY && ly[r] < G::GY + TYo && xown;
  }

  double U[G::RT][R][2];
#pragma unroll
  for (int r = 0; r < G::RT; ++r)
#pragma unroll
    for (int k = 0; k < R; ++k) U[r][k][0] = U[r][k][1] = 0.0;

  unsigned bad = 0;
  uint32_t round = 0;
  for (int t0 = t_begin; t0 <= t_end; t0 += R, ++round) {
    [&]<int... Ks>(std::integer_sequence<int, Ks...>) {
      (
          [&] {
            constexpr int KS = Ks;
            const int t = t0 + KS;
            constexpr int S1 = (KS + 1) % R, S0 = KS % R, SM1 = (KS + R - 1) % R;
            constexpr int SM2 = (KS + R - 2) % R, SM3 = (KS + R - 3) % R;
            // ---- plane t+1: smem slot -> register ring (use count of slot S1) ----
            {
              const uint32_t use = round + (uint32_t)((KS + 1) / R);
              mbar_wait3(mb_s + 8u * S1, (use - (S1 == 0 ? 1u : 0u)) & 1u);
#pragma unroll
              for (int r = 0; r < G::RT; ++r) {
                const double2 v = *reinterpret_cast<const double2 *>(su + S1 * G::SLOTE + rowoff[r]);
                U[r][S1][0] = v.x;
                U[r][S1][1] = v.y;
              }
            }
            if (FORM == 1) {
              const uint32_t use = round + (uint32_t)(KS / R);
              mbar_wait3(mb_s + 8u * (R + S0), use & 1u);
            }
            constexpr int qz = KS & 1;  // (t - 1 + pz) & 1
            // ---- red (colour 0) at plane t ----
            if (t >= 1 && t <= nz && t >= z0 - n0z && t < z1 + n0z) {
#pragma unroll
              for (int r = 0; r < G::RT; ++r) {
                const int s = 1 ^ ((qy[r] + qz) & 1);  // x parity of the red point in the pair
                const double *pl = su + S0 * G::SLOTE + rowoff[r] + s;
                const double uc = s ? U[r][S0][1] : U[r][S0][0];
                const double vzm = s ? U[r][SM1][1] : U[r][SM1][0];
                const double vzp = s ? U[r][S1][1] : U[r][S1][0];
                double acc = acc_init<FORM, UNIT>(uc, p);
                acc = acc_add<FORM, UNIT>(acc, vzm, 0, p);            // (0,0,-1)
                acc = acc_add<FORM, UNIT>(acc, pl[-G::PX], 1, p);     // (0,-1,0)
                // x-neighbour inside the pair: the thread's own (black) register;
                // across the pair boundary: the adjacent pair's value in smem
                const double vxm = s ? U[r][S0][0] : pl[-1];
                const double vxp = s ? pl[1] : U[r][S0][1];
                acc = acc_add<FORM, UNIT>(acc, vxm, 2, p);            // (-1,0,0)
                acc = acc_add<FORM, UNIT>(acc, vxp, 3, p);            // (1,0,0)
                acc = acc_add<FORM, UNIT>(acc, pl[G::PX], 4, p);      // (0,1,0)
                acc = acc_add<FORM, UNIT>(acc, vzp, 5, p);            // (0,0,1)
                const bool ok = row0[r] && colok(s, n0x);
                const double fc = FORM == 1 ? sf[S0 * G::SLOTE + rowoff[r] + s] : 0.0;
                const double out = acc_finish_used<FORM, UNIT, DIV>(acc, uc, fc, ok, p);
                if (ok) {
                  if (s) U[r][S0][1] = out; else U[r][S0][0] = out;
                  su[S0 * G::SLOTE + rowoff[r] + s] = out;
                }
              }
            }
            // ---- black (colour 1) at plane t-2 ----
            {
              const int pz = t - 2;
              if (pz >= 1 && pz <= nz && pz >= z0 && pz < z1) {
#pragma unroll
                for (int r = 0; r < G::RT; ++r) {
                  const int s = (qy[r] + qz) & 1;  // the other column of the pair
                  const double *pl = su + SM2 * G::SLOTE + rowoff[r] + s;
                  const double uc = s ? U[r][SM2][1] : U[r][SM2][0];
                  const double vzm = s ? U[r][SM3][1] : U[r][SM3][0];
                  const double vzp = s ? U[r][SM1][1] : U[r][SM1][0];
                  double acc = acc_init<FORM, UNIT>(uc, p);
                  acc = acc_add<FORM, UNIT>(acc, vzm, 0, p);
                  acc = acc_add<FORM, UNIT>(acc, pl[-G::PX], 1, p);
                  const double vxm = s ? U[r][SM2][0] : pl[-1];  // own red register inside the pair
                  const double vxp = s ? pl[1] : U[r][SM2][1];
                  acc = acc_add<FORM, UNIT>(acc, vxm, 2, p);
                  acc = acc_add<FORM, UNIT>(acc, vxp, 3, p);
                  acc = acc_add<FORM, UNIT>(acc, pl[G::PX], 4, p);
                  acc = acc_add<FORM, UNIT>(acc, vzp, 5, p);
                  const bool ok = row1[r] && colok(s, 0);
                  const double fc = FORM == 1 ? sf[SM2 * G::SLOTE + rowoff[r] + s] : 0.0;
                  const double out = acc_finish_used<FORM, UNIT, DIV>(acc, uc, fc, ok, p);
                  if (ok) {
                    if (s) U[r][SM2][1] = out; else U[r][SM2][0] = out;
                  }
                }
              }
              // ---- plane t-2 is final: owned pairs -> dst ----
              if (pz >= z0 && pz < z1) {
#pragma unroll
                for (int r = 0; r < G::RT; ++r)
                  if (own_out[r]) {
                    const bool in_yz = pz >= 1 && pz <= nz && gy[r] >= 1 && gy[r] <= ny;
                    bad |= (in_yz && gx >= 1 &&
                            ((unsigned)__double2hiint(U[r][SM2][0]) & 0x7ff00000u) == 0x7ff00000u) |
                           (in_yz && gx + 1 <= nx &&
                            ((unsigned)__double2hiint(U[r][SM2][1]) & 0x7ff00000u) == 0x7ff00000u);
                    stg_pair(dst + (int64_t)pz * p.sz + (int64_t)gy[r] * p.sy + gx, U[r][SM2][0], U[r][SM2][1]);
                  }
              }
            }
            __syncthreads();
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
    const int tl = t_begin + (int)round * R;  // first unprocessed step
    for (int k = 0; k <= D; ++k) {
      const int pu = tl + 1 + k, pf = tl + k;
      const int su_i = (pu - t_begin) % R, sf_i = (pf - t_begin) % R;
      mbar_wait3(mb_s + 8u * su_i, (uint32_t)(((pu - t_begin) / R - (su_i == 0 ? 1 : 0)) & 1));
      mbar_wait3(mb_s + 8u * (R + sf_i), (uint32_t)(((pf - t_begin) / R) & 1));
    }
  }
  __syncthreads();
  if (bad) atomicOr(p.status, 1);
}

}  // namespace sl
