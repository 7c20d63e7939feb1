// k2_fused.cu — K2: colour-fused, temporally blocked streaming sweep.
//
// Replaces the per-colour pass loop of sweep_colouring (reference
// strategies.py:374-393) times the multi-sweep loop of run_sweeps
// (bench.py:186-188): one HBM pass applies all c colour phases of M sweeps.
//
// Data movement per pass (ping-pong: read `src`, write `dst`, so no tile
// ever reads a value another tile already overwrote):
//   * a CTA owns a tile of the non-streaming axes (3D: TX x TY columns,
//     2D: TX columns) and a chunk of the streaming axis (z / y);
//   * it streams planes (3D) / row blocks (2D) of the tile plus a ghost
//     margin through a circular shared-memory window.  Global loads are
//     16-byte coalesced (LDG.128) one step ahead into registers, then
//     stored DE-INTERLEAVED by x parity (even x | odd x halves), so that
//     the 32 lanes of a warp updating one colour — every other x — hit 32
//     consecutive 8-byte words (conflict-free), and so do their x+-1
//     neighbours;
//   * each phase k updates its colour's points on plane t - lag[k] in
//     place in shared memory, redundantly on the ghost margin need[k]
//     (plan.cuh), f is read straight from global (L1-cached, used once);
//   * finished planes of the owned box are written to `dst` with STG.128.
// The per-point arithmetic is common.cuh's, in canonical neighbour order,
// so the result is bitwise identical to the per-colour path and the oracle.
#include "k2_fused.cuh"
#include "plan.cuh"

#include <utility>

namespace sl {

__host__ __device__ constexpr int natural_colours(int s) {
  return (s == FD5 || s == FD7) ? 2 : (s == FE9 ? 4 : 8);
}

__host__ __device__ constexpr int even_up(int v) { return (v + 1) & ~1; }

// start of tile k of n over [0, len) — even, non-decreasing, last = len
__host__ __device__ inline int64_t tile_start(int64_t k, int64_t len, int64_t n) {
  return 2 * ((k * (len / 2)) / n);  // len is even (checked on the host)
}

__host__ __device__ inline int64_t chunk_start(int64_t k, int64_t len, int64_t n) {
  return (k * len) / n;
}

__device__ __forceinline__ double2 ldg_nc2(const double *p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ double ldg_nc(const double *p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void stg2(double *p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

// ---------------------------------------------------------------------------
// geometry

template <int S, int M>
struct Geo3 {
  static constexpr FPlan P = make_plan(S, natural_colours(S), M);
  static constexpr int K = P.K, C = P.C, LAGMAX = P.lagmax;
  static constexpr int GX = even_up(P.load[0]);
  static constexpr int GY = P.load[1];
  static constexpr int GZ = P.load[2];
  static constexpr int PX = 64;             // one warp: 32 lanes x 2 columns
  static constexpr int HW = PX / 2 + 2;      // half-row incl. one pad each side
  static constexpr int ROWW = 2 * HW;
  static constexpr int PY = 32;
  static constexpr int TX = PX - 2 * GX;
  static constexpr int TY = PY - 2 * GY;
  static constexpr int W = LAGMAX + 4;       // plane slots in the window
  static constexpr int SLOT = PY * ROWW;
  static constexpr int NT = 256;
  static constexpr int NW = NT / 32;
  static constexpr int PAIRS = PY * PX / 2;
  static constexpr int LPT = PAIRS / NT;
  static constexpr size_t SMEM = size_t(W) * SLOT * sizeof(double);
  static_assert(PAIRS % NT == 0, "plane load split");
  static_assert(TX >= 8 && TY >= 4, "ghost margin too wide for the tile");
};

template <int S, int M>
struct Geo2 {
  static constexpr FPlan P = make_plan(S, natural_colours(S), M);
  static constexpr int K = P.K, C = P.C, LAGMAX = P.lagmax;
  static constexpr int GX = even_up(P.load[0]);
  static constexpr int GY = P.load[1];       // streaming-axis margin
  static constexpr int NSTRIP = 4;
  static constexpr int PX = 64 * NSTRIP;
  static constexpr int HW = PX / 2 + 2;
  static constexpr int ROWW = 2 * HW;
  static constexpr int R = 8;                // rows per macro-step
  static constexpr int NB = 4;               // row blocks in the window
  static constexpr int WR = NB * R;
  static constexpr int TX = PX - 2 * GX;
  static constexpr int NT = 256;
  static constexpr int NW = NT / 32;
  static constexpr int PAIRS = R * PX / 2;
  static constexpr int LPT = PAIRS / NT;
  static constexpr size_t SMEM = size_t(WR) * ROWW * sizeof(double);
  static_assert(LAGMAX + 1 <= R, "row block shorter than the phase lag");
  static_assert(PAIRS % NT == 0, "block load split");
};

struct Tiles {
  int64_t ntx, nty, nzc;  // tiles along x, y (3D) and chunks along the streaming axis
};

// offsets, relative to (row base + lane i), of the x-1 / x / x+1 neighbours
// of a point at local x = 2i + s in the de-interleaved row layout
template <int HW>
struct XOff {
  int m, c, p;
  __device__ __forceinline__ XOff(int s)
      : m((1 - s) * HW + s), c(s * HW + 1), p((1 - s) * HW + 1 + s) {}
  __device__ __forceinline__ int at(int dx) const { return dx < 0 ? m : (dx == 0 ? c : p); }
};

// ---------------------------------------------------------------------------
// 3D: z-streaming over (TX x TY) tiles

template <int S, int FORM, bool UNIT, int DIV, int M>
__global__ void __launch_bounds__(256, 2)
k2_stream3d(Params p, const double *__restrict__ src, double *__restrict__ dst, Tiles tl) {
  using G = Geo3<S, M>;
  constexpr FPlan P = G::P;
  constexpr int NNZ = shape_nnz(S);
  extern __shared__ double sm[];

  const int64_t Sx = p.nx + 2, Sy = p.ny + 2, Sz = p.nz + 2;
  const int64_t item = blockIdx.x;
  const int64_t tx = item % tl.ntx;
  const int64_t ty = (item / tl.ntx) % tl.nty;
  const int64_t zc = item / (tl.ntx * tl.nty);
  const int64_t x0 = tile_start(tx, Sx, tl.ntx), x1 = tile_start(tx + 1, Sx, tl.ntx);
  const int64_t y0 = chunk_start(ty, Sy, tl.nty), y1 = chunk_start(ty + 1, Sy, tl.nty);
  const int64_t z0 = chunk_start(zc, Sz, tl.nzc), z1 = chunk_start(zc + 1, Sz, tl.nzc);
  const int TXo = (int)(x1 - x0), TYo = (int)(y1 - y0);
  const int64_t gx0 = x0 - G::GX, gy0 = y0 - G::GY;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int base_par = (int)((gx0 - 1 + p.px) & 1);

  auto slot_of = [](int64_t gz) -> int { return (int)((gz % G::W + G::W) % G::W); };

  // register-staged plane load (16-byte coalesced), then de-interleaved STS
  auto load_regs = [&](int64_t gz, double2 (&r)[G::LPT]) {
#pragma unroll
    for (int k = 0; k < G::LPT; ++k) {
      const int pair = tid + k * G::NT;
      const int row = pair / (G::PX / 2), i = pair % (G::PX / 2);
      const int64_t gx = gx0 + 2 * i, gy = gy0 + row;
      const bool ok = gz >= 0 && gz < Sz && gy >= 0 && gy < Sy && gx >= 0 && gx < Sx;
      r[k] = ok ? ldg_nc2(src + gz * p.sz + gy * p.sy + gx) : make_double2(0.0, 0.0);
    }
  };
  auto store_regs = [&](int64_t gz, const double2 (&r)[G::LPT]) {
    double *slot = sm + slot_of(gz) * G::SLOT;
#pragma unroll
    for (int k = 0; k < G::LPT; ++k) {
      const int pair = tid + k * G::NT;
      const int row = pair / (G::PX / 2), i = pair % (G::PX / 2);
      slot[row * G::ROWW + 1 + i] = r[k].x;
      slot[row * G::ROWW + G::HW + 1 + i] = r[k].y;
    }
  };

  const int64_t t_begin = z0 - G::GZ - 1;
  const int64_t t_end = z1 - 1 + G::LAGMAX;
  {
    double2 r[G::LPT];
    load_regs(t_begin + 1, r);
    store_regs(t_begin + 1, r);
    load_regs(t_begin + 2, r);
    store_regs(t_begin + 2, r);
  }
  __syncthreads();

  int bad = 0;
  for (int64_t t = t_begin; t <= t_end; ++t) {
    double2 pf[G::LPT];
    const int64_t gz_pf = t + 2;
    const bool do_pf = gz_pf < z1 + G::GZ;
    if (do_pf) load_regs(gz_pf, pf);

    // ---- colour phases, in order ----
    [&]<int... Js>(std::integer_sequence<int, Js...>) {
      (
          [&] {
            constexpr int J = Js;
            constexpr int c = P.colour[J];
            constexpr int nx_ = P.need[J][0], ny_ = P.need[J][1], nz_ = P.need[J][2];
            const int64_t pz = t - P.lag[J];
            bool active = pz >= 1 && pz <= p.nz && pz >= z0 - nz_ && pz < z1 + nz_;
            const int qz = (int)((pz - 1 + p.pz) & 1);
            if (G::C == 8 && qz != ((c >> 2) & 1)) active = false;
            if (!active) return;
            const double *sl_m = sm + slot_of(pz - 1) * G::SLOT;
            double *sl_c = sm + slot_of(pz) * G::SLOT;
            const double *sl_p = sm + slot_of(pz + 1) * G::SLOT;
            // point rows of this phase (local slot rows)
            int ly_lo = G::GY - ny_, ly_hi = G::GY + TYo + ny_;  // [lo, hi)
            if (gy0 + ly_lo < 1) ly_lo = (int)(1 - gy0);
            if (gy0 + ly_hi > p.ny + 1) ly_hi = (int)(p.ny + 1 - gy0);
            int rstep = 1;
            if (G::C != 2) {
              rstep = 2;
              const int want = (c >> 1) & 1;
              if ((int)((gy0 + ly_lo - 1 + p.py) & 1) != want) ++ly_lo;
            }
            const int lx_lo = G::GX - nx_, lx_hi = G::GX + TXo + nx_;
            for (int ly = ly_lo + warp * rstep; ly < ly_hi; ly += G::NW * rstep) {
              const int64_t gy = gy0 + ly;
              const int qy = (int)((gy - 1 + p.py) & 1);
              const int qxt = G::C == 2 ? ((c + qy + qz) & 1) : (c & 1);
              const int s = (qxt ^ base_par) & 1;
              const int lx = 2 * lane + s;
              const int64_t gx = gx0 + lx;
              const bool valid = lx >= lx_lo && lx < lx_hi && gx >= 1 && gx <= p.nx;
              double fc = 0.0;
              if (FORM == 1 && valid) fc = ldg_nc(p.f + pz * p.sz + gy * p.sy + gx);
              const XOff<G::HW> xo(s);
              const int rb = ly * G::ROWW + lane;
              const double uc = sl_c[rb + xo.c];
              double acc = acc_init<FORM, UNIT>(uc, p);
#pragma unroll
              for (int q = 0; q < NNZ; ++q) {
                const Off o = shape_off(S, q);
                const double *pl = o.z < 0 ? sl_m : (o.z > 0 ? sl_p : sl_c);
                acc = acc_add<FORM, UNIT>(acc, pl[rb + o.y * G::ROWW + xo.at(o.x)], q, p);
              }
              const double out = acc_finish<FORM, UNIT, DIV>(acc, uc, fc, p);
              if (valid) {
                bad |= !finite64(out);
                sl_c[rb + xo.c] = out;
              }
            }
            __syncthreads();
          }(),
          ...);
    }(std::make_integer_sequence<int, G::K>{});

    // ---- finished plane of the owned box -> dst ----
    const int64_t gz_out = t - G::LAGMAX;
    if (gz_out >= z0 && gz_out < z1) {
      const double *slot = sm + slot_of(gz_out) * G::SLOT;
#pragma unroll
      for (int k = 0; k < G::LPT; ++k) {
        const int pair = tid + k * G::NT;
        const int row = pair / (G::PX / 2), i = pair % (G::PX / 2);
        const int lx = 2 * i;
        if (row >= G::GY && row < G::GY + TYo && lx >= G::GX && lx < G::GX + TXo) {
          const int64_t g = gz_out * p.sz + (gy0 + row) * p.sy + gx0 + lx;
          stg2(dst + g, slot[row * G::ROWW + 1 + i], slot[row * G::ROWW + G::HW + 1 + i]);
        }
      }
    }
    if (do_pf) store_regs(gz_pf, pf);
    __syncthreads();
  }
  if (bad) atomicOr(p.status, 1);
}

// ---------------------------------------------------------------------------
// 2D: y-streaming in row blocks of R over TX-column tiles

template <int S, int FORM, bool UNIT, int DIV, int M>
__global__ void __launch_bounds__(256, 2)
k2_stream2d(Params p, const double *__restrict__ src, double *__restrict__ dst, Tiles tl) {
  using G = Geo2<S, M>;
  constexpr FPlan P = G::P;
  constexpr int NNZ = shape_nnz(S);
  extern __shared__ double sm[];

  const int64_t Sx = p.nx + 2, Sy = p.ny + 2;
  const int64_t item = blockIdx.x;
  const int64_t tx = item % tl.ntx;
  const int64_t yc = item / tl.ntx;
  const int64_t x0 = tile_start(tx, Sx, tl.ntx), x1 = tile_start(tx + 1, Sx, tl.ntx);
  const int64_t y0 = chunk_start(yc, Sy, tl.nty), y1 = chunk_start(yc + 1, Sy, tl.nty);
  const int TXo = (int)(x1 - x0);
  const int64_t gx0 = x0 - G::GX;
  const int64_t yb = y0 - G::GY;  // first row of block 0
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int base_par = (int)((gx0 - 1 + p.px) & 1);

  auto srow = [](int64_t gy, int64_t yb_) -> int { return (int)((gy - yb_) % G::WR); };

  auto load_regs = [&](int64_t blk, double2 (&r)[G::LPT]) {
#pragma unroll
    for (int k = 0; k < G::LPT; ++k) {
      const int pair = tid + k * G::NT;
      const int row = pair / (G::PX / 2), i = pair % (G::PX / 2);
      const int64_t gx = gx0 + 2 * i, gy = yb + blk * G::R + row;
      const bool ok = gy >= 0 && gy < Sy && gy < y1 + G::GY && gx >= 0 && gx < Sx;
      r[k] = ok ? ldg_nc2(src + gy * p.sy + gx) : make_double2(0.0, 0.0);
    }
  };
  auto store_regs = [&](int64_t blk, const double2 (&r)[G::LPT]) {
#pragma unroll
    for (int k = 0; k < G::LPT; ++k) {
      const int pair = tid + k * G::NT;
      const int row = pair / (G::PX / 2), i = pair % (G::PX / 2);
      double *rp = sm + srow(yb + blk * G::R + row, yb) * G::ROWW;
      rp[1 + i] = r[k].x;
      rp[G::HW + 1 + i] = r[k].y;
    }
  };

  // last step: the block whose output window contains row y1-1
  const int64_t T_end = (y1 - 1 + G::LAGMAX - yb) / G::R;
  {
    double2 r[G::LPT];
    load_regs(0, r);
    store_regs(0, r);
    load_regs(1, r);
    store_regs(1, r);
  }
  __syncthreads();

  int bad = 0;
  for (int64_t T = 0; T <= T_end; ++T) {
    double2 pf[G::LPT];
    const int64_t blk_pf = T + 2;
    const bool do_pf = yb + blk_pf * G::R < y1 + G::GY;
    if (do_pf) load_regs(blk_pf, pf);
    const int64_t front = yb + T * G::R;

    [&]<int... Js>(std::integer_sequence<int, Js...>) {
      (
          [&] {
            constexpr int J = Js;
            constexpr int c = P.colour[J];
            constexpr int nx_ = P.need[J][0], ny_ = P.need[J][1];
            int64_t r_lo = front - P.lag[J], r_hi = r_lo + G::R;  // [lo, hi)
            if (r_lo < 1) r_lo = 1;
            if (r_lo < y0 - ny_) r_lo = y0 - ny_;
            if (r_hi > p.ny + 1) r_hi = p.ny + 1;
            if (r_hi > y1 + ny_) r_hi = y1 + ny_;
            if (r_lo >= r_hi) return;
            int rstep = 1;
            if (G::C != 2) {
              rstep = 2;
              if ((int)((r_lo - 1 + p.py) & 1) != ((c >> 1) & 1)) ++r_lo;
            }
            const int nrows = r_lo < r_hi ? (int)((r_hi - r_lo + rstep - 1) / rstep) : 0;
            const int lx_lo = G::GX - nx_, lx_hi = G::GX + TXo + nx_;
            for (int it = warp; it < nrows * G::NSTRIP; it += G::NW) {
              const int strip = it % G::NSTRIP;
              const int64_t gy = r_lo + (int64_t)(it / G::NSTRIP) * rstep;
              const int qy = (int)((gy - 1 + p.py) & 1);
              const int qxt = G::C == 2 ? ((c + qy) & 1) : (c & 1);
              const int s = (qxt ^ base_par) & 1;
              const int li = strip * 32 + lane;  // pair index in the row
              const int lx = 2 * li + s;
              const int64_t gx = gx0 + lx;
              const bool valid = lx >= lx_lo && lx < lx_hi && gx >= 1 && gx <= p.nx;
              double fc = 0.0;
              if (FORM == 1 && valid) fc = ldg_nc(p.f + gy * p.sy + gx);
              const XOff<G::HW> xo(s);
              double *rc = sm + srow(gy, yb) * G::ROWW + li;
              const double *rm = sm + srow(gy - 1, yb) * G::ROWW + li;
              const double *rp = sm + srow(gy + 1, yb) * G::ROWW + li;
              const double uc = rc[xo.c];
              double acc = acc_init<FORM, UNIT>(uc, p);
#pragma unroll
              for (int q = 0; q < NNZ; ++q) {
                const Off o = shape_off(S, q);
                const double *rr = o.y < 0 ? rm : (o.y > 0 ? rp : rc);
                acc = acc_add<FORM, UNIT>(acc, rr[xo.at(o.x)], q, p);
              }
              const double out = acc_finish<FORM, UNIT, DIV>(acc, uc, fc, p);
              if (valid) {
                bad |= !finite64(out);
                rc[xo.c] = out;
              }
            }
            __syncthreads();
          }(),
          ...);
    }(std::make_integer_sequence<int, G::K>{});

    // finished rows [front - LAGMAX, front + R - LAGMAX) of the owned box -> dst
#pragma unroll
    for (int k = 0; k < G::LPT; ++k) {
      const int pair = tid + k * G::NT;
      const int row = pair / (G::PX / 2), i = pair % (G::PX / 2);
      const int64_t gy = front - G::LAGMAX + row;
      const int lx = 2 * i;
      if (gy >= y0 && gy < y1 && lx >= G::GX && lx < G::GX + TXo) {
        const double *rp = sm + srow(gy, yb) * G::ROWW;
        stg2(dst + gy * p.sy + gx0 + lx, rp[1 + i], rp[G::HW + 1 + i]);
      }
    }
    if (do_pf) store_regs(blk_pf, pf);
    __syncthreads();
  }
  if (bad) atomicOr(p.status, 1);
}

// ---------------------------------------------------------------------------
// host side

static bool fused_supported(const KernelKey &key, const Params &p) {
  if (p.batch != 1) return false;
  if (p.colours != natural_colours(key.shape)) return false;
  const int64_t Sx = p.nx + 2;
  if (Sx & 1) return false;  // 16-byte row alignment
  if (((uintptr_t)p.u & 15) || (p.f && ((uintptr_t)p.f & 15))) return false;
  return true;
}

size_t fused_workspace_bytes(const KernelKey &key, const Params &p) {
  if (!fused_supported(key, p)) return 0;
  const int64_t elems = (p.nx + 2) * (p.ny + 2) * (shape_dim(key.shape) == 3 ? (p.nz + 2) : 1);
  return (size_t)elems * sizeof(double);
}

// Chunks along the streaming axis: balance wave quantisation against the
// per-chunk warm-up/drain cost (`extra` steps per chunk).
static int64_t pick_chunks(int64_t cols, int64_t len, int64_t slots, int64_t extra, int64_t min_len) {
  int64_t best = 1;
  double best_cost = 1e300;
  const int64_t maxc = len / min_len > 0 ? len / min_len : 1;
  for (int64_t c = 1; c <= maxc; ++c) {
    const int64_t items = cols * c;
    const int64_t waves = (items + slots - 1) / slots;
    const double cost = (double)waves * ((double)len / c + extra);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = c;
    }
  }
  return best;
}

template <typename Kern>
static cudaError_t prepare(Kern kern, size_t smem, int threads, int64_t *slots) {
  static thread_local int cached_dev = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0, sms = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  cached_dev = dev;
  *slots = (int64_t)(occ > 0 ? occ : 1) * sms;
  return cudaSuccess;
}

template <int S, int FORM, bool UNIT, int DIV, int M>
static cudaError_t launch_pass(const Params &p, const double *src, double *dst, cudaStream_t st) {
  if constexpr (shape_dim(S) == 3) {
    using G = Geo3<S, M>;
    auto kern = k2_stream3d<S, FORM, UNIT, DIV, M>;
    static thread_local int64_t slots = 0;
    if (!slots) {
      cudaError_t e = prepare(kern, G::SMEM, G::NT, &slots);
      if (e != cudaSuccess) return e;
    }
    Tiles tl;
    const int64_t Sx = p.nx + 2, Sy = p.ny + 2, Sz = p.nz + 2;
    tl.ntx = (Sx + G::TX - 1) / G::TX;
    tl.nty = (Sy + G::TY - 1) / G::TY;
    tl.nzc = pick_chunks(tl.ntx * tl.nty, Sz, slots, G::GZ + G::LAGMAX + 1, 16);
    const int64_t items = tl.ntx * tl.nty * tl.nzc;
    kern<<<(unsigned)items, G::NT, G::SMEM, st>>>(p, src, dst, tl);
    note_launch();
    return cudaGetLastError();
  } else {
    using G = Geo2<S, M>;
    auto kern = k2_stream2d<S, FORM, UNIT, DIV, M>;
    static thread_local int64_t slots = 0;
    if (!slots) {
      cudaError_t e = prepare(kern, G::SMEM, G::NT, &slots);
      if (e != cudaSuccess) return e;
    }
    Tiles tl;
    const int64_t Sx = p.nx + 2, Sy = p.ny + 2;
    tl.ntx = (Sx + G::TX - 1) / G::TX;
    tl.nty = pick_chunks(tl.ntx, Sy, slots, G::GY + G::LAGMAX + G::R, 2 * G::R);
    tl.nzc = 1;
    const int64_t items = tl.ntx * tl.nty;
    kern<<<(unsigned)items, G::NT, G::SMEM, st>>>(p, src, dst, tl);
    note_launch();
    return cudaGetLastError();
  }
}

cudaError_t launch_fused(const KernelKey &key, const Params &p, int sweeps, double *workspace,
                         size_t workspace_bytes, cudaStream_t st, int *handled) {
  *handled = 0;
  if (!fused_supported(key, p)) return cudaSuccess;
  const size_t need = fused_workspace_bytes(key, p);
  if (!workspace || workspace_bytes < need || ((uintptr_t)workspace & 15)) return cudaSuccess;
  *handled = 1;
  // passes alternate u -> ws -> u ...; an odd count ends with one copy back
  double *bufs[2] = {p.u, workspace};
  int cur = 0;
  cudaError_t e = cudaSuccess;
  for (int s = 0; s < sweeps && e == cudaSuccess; ++s) {
    e = dispatch(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
      return launch_pass<S, F, U, D, 1>(p, bufs[cur], bufs[cur ^ 1], st);
    });
    cur ^= 1;
  }
  if (e == cudaSuccess && cur == 1) {
    e = cudaMemcpyAsync(p.u, workspace, need, cudaMemcpyDeviceToDevice, st);
  }
  return e;
}

}  // namespace sl
