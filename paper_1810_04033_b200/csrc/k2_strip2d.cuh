// k2_strip2d.cuh — K2 for 2D grids: warp-private strip streaming.
//
// One warp owns a strip of 64*NP columns (lane i holds the NP column pairs
// 2*NP*i .. 2*NP*i + 2*NP - 1) and a chunk of rows, and streams the rows: no block barriers,
// warps fully independent.  The strip overlaps its neighbours by the ghost
// margin GX on each side, so TX = 64 - 2*GX columns are owned; x+-1
// neighbours of the lane's point come from its own pair or, across the pair
// boundary, from the adjacent lane by one warp shuffle.
//
// Memory path: each warp has a private ring of NS row slots in shared
// memory (u row segment + f row segment).  Lane 0 keeps NS rows in
// flight with TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx) —
// one copy per array per row, no registers held while in flight.
// At step t the warp waits on row t+1's mbarrier, moves the lane's pair into
// a small register ring (rows t-LAGMAX-1 .. t+1) and re-arms the slot for
// row t+1+NS.
//
// Phase k processes row t - lag[k] at step t (plan.cuh).  The step loop is
// unrolled by U (a multiple of both ring lengths) with the row parity of
// every slot fixed at compile time, so each phase's colour pattern (which
// rows hold the colour, which x parity its points have) and every ring index
// are compile-time: inactive phases vanish; the hot loop is LDS, shuffles
// and fp64 arithmetic.
#pragma once
#include "plan.cuh"

namespace sl {

template <int S, int M>
struct GeoS2 {
#ifndef STRIP_SPREAD
#define STRIP_SPREAD 0
#endif
  // STRIP_SPREAD = 1 (A/B): spread lags, so the phases active in one step are independent
  static constexpr FPlan P = make_plan(S, S == FE9 ? 4 : 2, M, STRIP_SPREAD != 0 && S == FE9 && M == 1);
  static constexpr int K = P.K, C = P.C, LAGMAX = P.lagmax;
  static constexpr bool RB = (P.C == 2);
  static constexpr int GX = (P.load[0] + 1) & ~1;
  static constexpr int GY = P.load[1];
#ifndef STRIP_NP
#define STRIP_NP 2
#endif
#ifndef STRIP_WPB
#define STRIP_WPB 2
#endif
#ifndef STRIP_NS
#define STRIP_NS 4
#endif
  static constexpr int NP = STRIP_NP;                  // column pairs per lane
  static constexpr int WS = 64 * NP;                   // strip width (columns)
  static constexpr int TX = WS - 2 * GX;
  static constexpr int NRR0 = LAGMAX + 3;             // register ring: rows t-LAGMAX-1 .. t+1
  static constexpr int NRR = NRR0 <= 2 ? 2 : (NRR0 <= 4 ? 4 : 8);
  static constexpr int NS = STRIP_NS;                  // smem ring slots (rows in flight)
  static constexpr int U = NRR > NS ? NRR : NS;        // unroll: multiple of both (powers of 2)
  static constexpr int WPB = STRIP_WPB;                // warps per block
  static constexpr int ROWB = WS * 8;                  // bytes of one array's row segment
  static constexpr int SLOTB = 2 * ROWB;               // u + f
  static constexpr size_t SMEM = size_t(WPB) * NS * SLOTB;
  static_assert(NRR >= NRR0, "register ring too short");
  // ring indices (KS % NS, (KS + 1) % NRR over an unroll of U) wrap correctly only
  // for power-of-two depths that divide U
  static_assert((NS & (NS - 1)) == 0 && U % NS == 0 && U % NRR == 0, "STRIP_NS must be a power of two");
  // does the stencil use offset (dx, dy)?
  static constexpr bool uses(int dx, int dy) {
    for (int q = 0; q < shape_nnz(S); ++q) {
      const Off o = shape_off(S, q);
      if (o.x == dx && o.y == dy) return true;
    }
    return false;
  }
};

__device__ __forceinline__ void stg_pair(double *p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t addr, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint32_t addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
  sl_fuzz(200000u);
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}

// Exact division out of line (rare fallback of the Markstein fast path).
static __device__ __noinline__ double strip_div_exact(double a, double b) { return __ddiv_rn(a, b); }

// EQW: every neighbour weight equal (FE9: -1/3; host-checked).  Then each
// value's product w * u is rounded once per phase and shared by the lane's
// points and, through the shuffle, by the adjacent lane — the same rounded
// terms, added in the same canonical order.
template <int S, int FORM, bool UNIT, int DIV, int M, bool EQW = false, bool PEER = false>
#ifndef STRIP_MINB
#define STRIP_MINB 1
#endif
// STRIP_MINB (A/B): minimum resident blocks per SM asked of ptxas (caps the registers)
__global__ void __launch_bounds__(32 * GeoS2<S, M>::WPB, STRIP_MINB)
k2_strip2d(Params p, const double *__restrict__ src, double *__restrict__ dst, int64_t nstrip,
           int64_t nchunk) {
  using G = GeoS2<S, M>;
  constexpr FPlan P = G::P;
  constexpr int NRR = G::NRR, NS = G::NS;
  constexpr int NNZ = shape_nnz(S);
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t mbar[G::WPB][NS];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wid = (int64_t)blockIdx.x * G::WPB + warp;
  if (wid >= nstrip * nchunk) return;  // whole warp exits together, before any copy
  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2;
  const int nx = (int)p.nx, ny = (int)p.ny;
  const int strip = (int)(wid % nstrip), chunk = (int)(wid / nstrip);
  const int x0 = (int)(2 * (((int64_t)strip * (Sx / 2)) / nstrip));
  const int x1 = (int)(2 * (((int64_t)(strip + 1) * (Sx / 2)) / nstrip));
  const int ylen = p.zhi - p.zlo;  // output rows [zlo, zhi): the slowest axis of a 2D grid
  const int y0 = p.zlo + (int)(((int64_t)chunk * ylen) / nchunk);
  const int y1 = p.zlo + (int)(((int64_t)(chunk + 1) * ylen) / nchunk);
  const int TXo = x1 - x0;
  constexpr int NP = G::NP, NC = 2 * NP;  // pairs / columns per lane
  const int gxs = x0 - G::GX;            // global x of the strip's column 0 (even)
  const int lx0 = NC * lane;             // strip-local x of the lane's first column
  const int gx = gxs + lx0;              // global x of the lane's first column
  // copy window in x, clipped to the array (16-byte granules)
  const int cx0 = gxs < 0 ? 0 : gxs;
  const int cx1 = gxs + G::WS > Sx ? Sx : gxs + G::WS;
  const uint32_t cbytes = (uint32_t)(cx1 - cx0) * 8u;
  const uint32_t cdoff = (uint32_t)(cx0 - gxs) * 8u;

  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smraw) + (uint32_t)(warp * NS * G::SLOTB);
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&mbar[warp][0]);

  // rows of register-ring slot 0 have (row - 1 + py) even
  int t_begin = y0 - G::GY - 1;
  if ((t_begin - 1 + p.py) & 1) --t_begin;
  const int t_end = y1 - 1 + G::LAGMAX;
  const int ylim = y1 + G::GY;  // rows >= ylim are never needed

  // lane 0 streams row `row` into smem slot `sl` (row t_begin+1+k lives in slot k % NS)
  auto issue = [&](int row, int sl) {
    const uint32_t mb = mb0 + 8u * sl;
    const bool live = row >= 0 && row < Sy && row < ylim;
    const uint32_t bytes = live ? (FORM == 1 ? 2u : 1u) * cbytes : 0u;
    mbar_arrive_tx(mb, bytes);
    if (live) {
      const int64_t g = (int64_t)row * p.sy + cx0;
      const uint32_t d = ring + (uint32_t)sl * G::SLOTB + cdoff;
      bulk_g2s(d, src + g, cbytes, mb);
      if (FORM == 1) bulk_g2s(d + G::ROWB, p.f + g, cbytes, mb);
    }
  };

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(mb0 + 8u * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int k = 0; k < NS; ++k) issue(t_begin + 1 + k, k);
  }
  __syncwarp();

  int rlo[G::K], rhi[G::K];
  unsigned colok = 0;  // bit (J * NC + cc): lane column cc is in phase J's need window and the interior
#pragma unroll
  for (int j = 0; j < G::K; ++j) {
    rlo[j] = max(1, y0 - P.need[j][1]);
    rhi[j] = min(ny, y1 - 1 + P.need[j][1]);
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      const int lx = lx0 + cc;
      if (lx >= G::GX - P.need[j][0] && lx < G::GX + TXo + P.need[j][0] && gx + cc >= 1 && gx + cc <= nx)
        colok |= 1u << (j * NC + cc);
    }
  }
  static_assert(G::K * NC <= 32, "validity bits");

  double uu[NRR][NC], ff[NRR][NC];
#pragma unroll
  for (int k = 0; k < NRR; ++k)
#pragma unroll
    for (int j = 0; j < NC; ++j) uu[k][j] = ff[k][j] = 0.0;

  // per-kernel constants in registers: without the opaque moves the compiler
  // re-reads them from the constant bank (LDCU + R2UR) in every phase
  double c_rwc, c_wc, c_om, c_w0;
  asm("mov.b64 %0, %1;" : "=d"(c_rwc) : "d"(p.rwc));
  asm("mov.b64 %0, %1;" : "=d"(c_wc) : "d"(p.wc));
  asm("mov.b64 %0, %1;" : "=d"(c_om) : "d"(p.omega));
  asm("mov.b64 %0, %1;" : "=d"(c_w0) : "d"(FORM == 0 ? p.aw[0] : p.w[0]));

  unsigned bad = 0;
  uint32_t round = 0;  // completed passes over the smem ring
  for (int t0 = t_begin; t0 <= t_end; t0 += G::U, round += G::U / NS) {
    [&]<int... Ks>(std::integer_sequence<int, Ks...>) {
      (
          [&] {
            constexpr int KS = Ks;  // t - t_begin (mod U)
            const int t = t0 + KS;
            // ---- row t+1: smem slot -> register ring, re-arm the slot ----
            {
              constexpr int SL = KS % NS;
              constexpr int RR = (KS + 1) % NRR;
#if SL_FUZZ_BREAK != 2   // negative control: read the row slot without waiting for its TMA copy
              mbar_wait(mb0 + 8u * SL, (round + (uint32_t)(KS / NS)) & 1u);
#endif
              const uint32_t a = ring + SL * G::SLOTB + lane * (NC * 8u);
#pragma unroll
              for (int k = 0; k < NP; ++k) {
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                             : "=d"(uu[RR][2 * k]), "=d"(uu[RR][2 * k + 1]) : "r"(a + 16u * k) : "memory");
                if (FORM == 1)
                  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                               : "=d"(ff[RR][2 * k]), "=d"(ff[RR][2 * k + 1]) : "r"(a + G::ROWB + 16u * k) : "memory");
              }
              __syncwarp();
              if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(t + 1 + NS, SL);
              }
            }
            // ---- phases in order ----
            [&]<int... Js>(std::integer_sequence<int, Js...>) {
              (
                  [&] {
                    constexpr int J = Js;
                    constexpr int c = P.colour[J];
                    constexpr int R0 = ((KS - P.lag[J]) % NRR + NRR) % NRR;
                    constexpr int RM = (R0 + NRR - 1) % NRR, RP = (R0 + 1) % NRR;
                    constexpr int qy = (KS - P.lag[J]) & 1;  // parity of the row being updated
                    if constexpr (!G::RB && qy != ((c >> 1) & 1)) {
                      return;  // colour absent from this row
                    } else {
                      constexpr int s = 1 ^ (G::RB ? ((c + qy) & 1) : (c & 1));  // x parity
                      const int row = t - P.lag[J];
                      const bool rok = row >= rlo[J] && row <= rhi[J];   // warp-uniform
                      // the lane's NP points of this colour: local columns 2k + s
                      double vl[3], vr[3];  // left / right ghost column from the adjacent lanes
                      constexpr int RRW[3] = {RM, R0, RP};
                      // EQW: products of the lane's columns (unused ones are dead code)
                      double pw[3][NC];
                      const double w0 = c_w0;
                      if constexpr (EQW) {
#pragma unroll
                        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                          for (int c2 = 0; c2 < NC; ++c2) pw[dy][c2] = __dmul_rn(w0, uu[RRW[dy]][c2]);
                      }
#pragma unroll
                      for (int dy = 0; dy < 3; ++dy) {
                        if (s == 0 && G::uses(-1, dy - 1))
                          vl[dy] = __shfl_up_sync(0xffffffffu, EQW ? pw[dy][NC - 1] : uu[RRW[dy]][NC - 1], 1);
                        if (s == 1 && G::uses(1, dy - 1))
                          vr[dy] = __shfl_down_sync(0xffffffffu, EQW ? pw[dy][0] : uu[RRW[dy]][0], 1);
                      }
                      double xv[NP], qv[NP];
                      bool valid[NP], slow = false;
#pragma unroll
                      for (int k = 0; k < NP; ++k) {
                        const int cc = 2 * k + s;  // lane-local column of the point
                        valid[k] = rok && ((colok >> (J * NC + cc)) & 1u);
                        auto val = [&](int dy, int dx) -> double {
                          const int col = cc + dx;
                          if (col < 0) return vl[dy];
                          if (col >= NC) return vr[dy];
                          return EQW ? pw[dy][col] : uu[RRW[dy]][col];
                        };
                        double acc = acc_init<FORM, UNIT>(uu[R0][cc], p);
#pragma unroll
                        for (int q = 0; q < NNZ; ++q) {
                          const Off o = shape_off(S, q);
                          const double v = val(o.y + 1, o.x);
                          if (EQW)
                            acc = __dadd_rn(acc, v);  // v is already w * u, rounded
                          else if (FORM == 0)
                            acc = __dadd_rn(acc, UNIT ? v : __dmul_rn(p.aw[q], v));
                          else
                            acc = UNIT ? __dsub_rn(acc, v) : __dadd_rn(acc, __dmul_rn(p.w[q], v));
                        }
                        xv[k] = FORM == 0 ? acc : __dsub_rn(ff[R0][cc], acc);
                        if (DIV == DIV_RCP) {
                          const double e = __dmul_rn(xv[k], c_rwc);
                          qv[k] = __fma_rn(__fma_rn(-c_wc, e, xv[k]), c_rwc, e);
                          const unsigned xe = ((unsigned)__double2hiint(xv[k]) >> 20) & 0x7ffu;
                          slow |= valid[k] && (xe - 64u) >= 1919u;
                        } else if (DIV == DIV_POW2) {
                          qv[k] = __dmul_rn(xv[k], c_rwc);
                        } else {
                          qv[k] = strip_div_exact(xv[k], p.wc);
                        }
                      }
                      // exact fallback, per warp, only for used lanes
                      if (DIV == DIV_RCP && __builtin_expect(__any_sync(0xffffffffu, slow), 0)) {
#pragma unroll
                        for (int k = 0; k < NP; ++k) {
                          const unsigned xe = ((unsigned)__double2hiint(xv[k]) >> 20) & 0x7ffu;
                          if (valid[k] && (xe - 64u) >= 1919u) qv[k] = strip_div_exact(xv[k], p.wc);
                        }
                      }
#pragma unroll
                      for (int k = 0; k < NP; ++k) {
                        const int cc = 2 * k + s;
                        const double uc = uu[R0][cc];
                        const double out = FORM == 0 ? qv[k] : __dadd_rn(uc, __dmul_rn(c_om, qv[k]));
                        uu[R0][cc] = valid[k] ? out : uc;
                      }
                    }
                  }(),
                  ...);
            }(std::make_integer_sequence<int, G::K>{});
            // ---- row t - LAGMAX is final: owned pairs -> dst; non-finite check ----
            {
              constexpr int RO = ((KS - G::LAGMAX) % NRR + NRR) % NRR;
              const int row = t - G::LAGMAX;
              if (row >= y0 && row < y1) {
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                  const int lx = lx0 + 2 * k;
                  if (lx >= G::GX && lx < G::GX + TXo) {
                    const double a = uu[RO][2 * k], b = uu[RO][2 * k + 1];
                    // non-finite results are sticky through later updates, so
                    // checking each owned value once, when final, catches them
                    const bool in_y = row >= 1 && row <= ny;
                    bad |= (in_y && gx + 2 * k >= 1 &&
                            ((unsigned)__double2hiint(a) & 0x7ff00000u) == 0x7ff00000u) |
                           (in_y && gx + 2 * k + 1 <= nx &&
                            ((unsigned)__double2hiint(b) & 0x7ff00000u) == 0x7ff00000u);
                    stg_pair(dst + (int64_t)row * p.sy + gx + 2 * k, a, b);
                    stg_pair_peers<PEER>(p, row, (int64_t)row * p.sy + gx + 2 * k, a, b);
                  }
                }
              }
            }
          }(),
          ...);
    }(std::make_integer_sequence<int, G::U>{});
  }
  // drain: the NS rows still in flight (one per slot) must land before exit
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_wait(mb0 + 8u * s, round & 1u);
  }
  __syncwarp();
  if (bad) atomicOr(p.status, 1);
}

}  // namespace sl
