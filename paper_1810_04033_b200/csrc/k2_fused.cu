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
//   * it streams planes (3D) / row blocks (2D) of u and f for the tile plus
//     a ghost margin through circular shared-memory windows.  Global loads
//     are 16-byte coalesced (LDG.128), issued one step ahead into registers
//     and stored DE-INTERLEAVED by x parity (even-x half | odd-x half) at
//     the start of the next step, so the 32 lanes of a warp updating one
//     colour (every other x) and their x+-1 neighbours each hit 32
//     consecutive 8-byte words: conflict-free;
//   * phase k updates its colour's points on plane t - lag[k] in place in
//     shared memory, redundantly on the ghost margin need[k] (plan.cuh).  A
//     warp item is a 32-lane strip x RY point rows whose neighbour rows are
//     loaded once and shared (register blocking), all loads before any store;
//   * finished planes of the owned box are written to `dst` with STG.128.
// The per-point arithmetic is common.cuh's, in canonical neighbour order,
// so the result is bitwise identical to the per-colour path and the oracle.
#include "k2_fused.cuh"
#include "plan.cuh"
#include "k2_strip2d.cuh"
#include "k3_patch.cuh"
#include "k2_col3d.cuh"
#include "k2_q1col.cuh"
#include "k6_resident2d.cuh"

#include <cudaTypedefs.h>

#include <mutex>
#include <utility>
#include <vector>

namespace sl {

__host__ __device__ constexpr int natural_colours(int s) {
  return (s == FD5 || s == FD7) ? 2 : (s == FE9 ? 4 : 8);
}

__host__ __device__ constexpr int even_up(int v) { return (v + 1) & ~1; }

// start of tile k of n over [0, len) — even, non-decreasing, last = len (len even)
__host__ __device__ inline int64_t tile_start(int64_t k, int64_t len, int64_t n) {
  return 2 * ((k * (len / 2)) / n);
}

__host__ __device__ inline int64_t chunk_start(int64_t k, int64_t len, int64_t n) {
  return (k * len) / n;
}

__device__ __forceinline__ double2 ldg_nc2(const double *p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void stg2(double *p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

// ---------------------------------------------------------------------------
// geometry

template <int S, int M>
struct Geo3 {
  // lags spread so that all phases of a step are independent (plan.cuh):
  // one block barrier per step.  FE27 (26 neighbours) would need a window of
  // 8 lags, so it keeps per-phase barriers.
  static constexpr bool SPREAD = (S != FE27);
  static constexpr FPlan P = make_plan(S, natural_colours(S), M, SPREAD);
  static constexpr int K = P.K, C = P.C, LAGMAX = P.lagmax;
  static constexpr bool RB = (P.C == 2);
  static constexpr int GX = even_up(P.load[0]);
  static constexpr int GY = P.load[1];
  static constexpr int GZ = P.load[2];
  static constexpr int PX = 64;             // one warp: 32 lanes x 2 columns
  static constexpr int HW = PX / 2 + 2;      // half-row incl. one pad each side
  static constexpr int ROWW = 2 * HW;
  static constexpr int PY = 32;
  static constexpr int TX = PX - 2 * GX;
  static constexpr int TY = PY - 2 * GY;
  static constexpr int W = LAGMAX + 3;       // u plane slots: t-LAGMAX-1 .. t+1
  static constexpr int SLOT = PY * ROWW;
  static constexpr int RSTEP = RB ? 1 : 2;   // point rows of one colour
  static constexpr int RY = RB ? 4 : (S == Q1 || S == FE27 ? 1 : 2);  // point rows per warp item
  static constexpr int NT = 256;
  static constexpr int MINB = (S == Q1 || S == FE27) ? 1 : 2;  // Q1/FE27: 255-register budget
  static constexpr int PAD_ROWS = (RY - 1) * RSTEP + 2;
  static constexpr int NW = NT / 32;
  static constexpr int PAIRS = PY * PX / 2;
  static constexpr int LPT = PAIRS / NT;
  static constexpr int LEAD = 2;             // item reads may start one row before a slot
  static constexpr size_t SMEM = size_t(W * SLOT + (PAD_ROWS + LEAD) * ROWW) * sizeof(double);
  static_assert(PAIRS % NT == 0, "plane load split");
  static_assert(TX >= 8 && TY >= 4, "ghost margin too wide for the tile");
  static_assert(SMEM <= 227 * 1024, "window exceeds shared memory");
};

struct Tiles {
  int64_t ntx, nty, nzc;  // tiles along x, y (3D) and chunks along the streaming axis
};

// Offset (relative to row base + lane) of the x+dx neighbour of a point at
// local x = 2*lane + s in a de-interleaved row [pad, even.., pad | pad, odd.., pad].
template <int HW>
__host__ __device__ constexpr int xoff(int s, int dx) {
  return (((s + dx) & 1) ? HW : 0) + 1 + ((s + dx) >> 1);
}

// Non-finite detector: exponent field all ones.
__device__ __forceinline__ unsigned nonfinite_bits(double v) {
  return ((unsigned)__double2hiint(v) & 0x7ff00000u) == 0x7ff00000u;
}

// ---------------------------------------------------------------------------
// one warp item: RY point rows of a 32-lane strip, x parity pattern fixed at
// compile time (S0 = parity of row 0; red-black rows alternate).
//   ro(dz, k): smem element offset of source row k of plane dz (point row r
//   uses k = r*RSTEP + dy + 1), lane included;  fv(r, s): f of point row r.
// All loads precede all stores, so repeated (row, x) loads are CSE'd.

template <int S, int FORM, bool UNIT, int DIV, int RY, int RSTEP, bool RB, int HW, int S0,
          typename RowOff, typename FOff>
__device__ __forceinline__ unsigned update_item(const RowOff &ro, const FOff &fv, unsigned vmask,
                                                const Params &p) {
  extern __shared__ double sm[];
  constexpr int NNZ = shape_nnz(S);
  double out[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int s = RB ? (S0 ^ ((r * RSTEP) & 1)) : S0;
    const int kc = r * RSTEP + 1;
    const double uc = sm[ro(1, kc) + xoff<HW>(s, 0)];
    double acc = acc_init<FORM, UNIT>(uc, p);
#pragma unroll
    for (int q = 0; q < NNZ; ++q) {
      const Off o = shape_off(S, q);
      acc = acc_add<FORM, UNIT>(acc, sm[ro(o.z + 1, kc + o.y) + xoff<HW>(s, o.x)], q, p);
    }
    double fc = 0.0;
    if (FORM == 1) fc = fv(r, s);
    out[r] = acc_finish_warp<FORM, UNIT, DIV>(acc, uc, fc, (vmask >> r) & 1, p);  // warp-uniform callers
  }
  unsigned bad = 0;
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int s = RB ? (S0 ^ ((r * RSTEP) & 1)) : S0;
    if (vmask & (1u << r)) {
      bad |= nonfinite_bits(out[r]);
      sm[ro(1, r * RSTEP + 1) + xoff<HW>(s, 0)] = out[r];
    }
  }
  return bad;
}

// x parity (0 = even local x) of colour c's points in a row/plane with y/z
// parities qy, qz.  Tiles start at an even global x (origin x parity 0), so
// local and global x parity agree and q_x = 1 - (x & 1).
__host__ __device__ constexpr int x_parity(int colours, int c, int qy, int qz) {
  return 1 ^ (colours == 2 ? ((c + qy + qz) & 1) : (c & 1));
}

// ---------------------------------------------------------------------------
// 3D: z-streaming over (TX x TY) tiles

template <int S, int FORM, bool UNIT, int DIV, int M, bool PEER = false>
__global__ void __launch_bounds__(Geo3<S, M>::NT, Geo3<S, M>::MINB)
k2_stream3d(Params p, const double *__restrict__ src, double *__restrict__ dst, Tiles tl) {
  using G = Geo3<S, M>;
  constexpr FPlan P = G::P;
  extern __shared__ double sm[];

  const int Sx = (int)p.nx + 2, Sy = (int)p.ny + 2, Sz = (int)p.nz + 2;
  const int nx = (int)p.nx, ny = (int)p.ny, nz = (int)p.nz;
  const int item = blockIdx.x;
  const int tx = item % (int)tl.ntx;
  const int ty = (item / (int)tl.ntx) % (int)tl.nty;
  const int zc = item / (int)(tl.ntx * tl.nty);
  const int x0 = (int)tile_start(tx, Sx, tl.ntx), x1 = (int)tile_start(tx + 1, Sx, tl.ntx);
  const int y0 = (int)chunk_start(ty, Sy, tl.nty), y1 = (int)chunk_start(ty + 1, Sy, tl.nty);
  const int z0 = p.zlo + (int)chunk_start(zc, p.zhi - p.zlo, tl.nzc);
  const int z1 = p.zlo + (int)chunk_start(zc + 1, p.zhi - p.zlo, tl.nzc);
  const int TXo = x1 - x0, TYo = y1 - y0;
  const int gx0 = x0 - G::GX, gy0 = y0 - G::GY;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // lane validity in x for both parities: local x = 2*lane + s, global gx0 + x
  auto xok = [&](int s, int need) -> bool {
    const int lx = 2 * lane + s, gx = gx0 + lx;
    return lx >= G::GX - need && lx < G::GX + TXo + need && gx >= 1 && gx <= nx;
  };

  // per-thread plane coordinates are the same for every plane: precompute
  // the in-plane global offset, bounds flag, smem offset and ownership once
  int goff[G::LPT], soff[G::LPT];
  unsigned inxy = 0, ownm = 0;
#pragma unroll
  for (int k = 0; k < G::LPT; ++k) {
    const int pair = tid + k * G::NT;
    const int row = pair / (G::PX / 2), i = pair % (G::PX / 2);
    const int gx = gx0 + 2 * i, gy = gy0 + row;
    goff[k] = gy * (int)p.sy + gx;
    soff[k] = row * G::ROWW + 1 + i;
    inxy |= (unsigned)(gy >= 0 && gy < Sy && gx >= 0 && gx < Sx) << k;
    ownm |= (unsigned)(row >= G::GY && row < G::GY + TYo && 2 * i >= G::GX && 2 * i < G::GX + TXo) << k;
  }
  auto load_regs = [&](const double *base, int gz, double2 (&r)[G::LPT]) {
    const bool zok = gz >= 0 && gz < Sz;
    const double *pb = base + (int64_t)gz * p.sz;
#pragma unroll
    for (int k = 0; k < G::LPT; ++k)
      r[k] = (zok && ((inxy >> k) & 1)) ? ldg_nc2(pb + goff[k]) : make_double2(0.0, 0.0);
  };
  auto store_regs = [&](int off, const double2 (&r)[G::LPT]) {
#pragma unroll
    for (int k = 0; k < G::LPT; ++k) {
      sm[off + soff[k]] = r[k].x;
      sm[off + soff[k] + G::HW] = r[k].y;
    }
  };
  const int t_begin = z0 - G::GZ - 1;
  const int t_end = z1 - 1 + G::LAGMAX;
  const int zlim = z1 + G::GZ;
  int so[G::W];  // so[k] = smem offset of the slot holding plane t+1-k (rotated per step)
#pragma unroll
  for (int k = 0; k < G::W; ++k) so[k] = (((t_begin + 1 - k) % G::W + G::W) % G::W) * G::SLOT + G::LEAD * G::ROWW;
  double2 pu[G::LPT];
  load_regs(src, t_begin + 1, pu);

  unsigned bad = 0;
  for (int t = t_begin; t <= t_end; ++t) {
    // the plane loaded during the previous step goes into its (free) slot
    if (t + 1 < zlim) store_regs(so[0], pu);
    __syncthreads();
    if (t + 2 < zlim) load_regs(src, t + 2, pu);

    // ---- colour phases, in order; with spread lags they are independent and
    // their warp items are pooled (phase J starts where J-1's items ended) ----
    int ibase = 0;
    [&]<int... Js>(std::integer_sequence<int, Js...>) {
      (
          [&] {
            constexpr int J = Js;
            constexpr int c = P.colour[J];
            constexpr int nx_ = P.need[J][0], ny_ = P.need[J][1], nz_ = P.need[J][2];
            const int pz = t - P.lag[J];
            if (pz < 1 || pz > nz || pz < z0 - nz_ || pz >= z1 + nz_) return;
            const int qz = (pz - 1 + p.pz) & 1;
            if (!G::RB && ((c >> 2) & 1) != qz) return;
            int ly_lo = G::GY - ny_, ly_hi = G::GY + TYo + ny_;  // [lo, hi) slot rows
            if (gy0 + ly_lo < 1) ly_lo = 1 - gy0;
            if (gy0 + ly_hi > ny + 1) ly_hi = ny + 1 - gy0;
            // align row 0 of every item to the parity with x parity 0
            const int want_qy = G::RB ? ((1 + c + qz) & 1) : ((c >> 1) & 1);
            const int ly_first = ly_lo;
            if (((gy0 + ly_lo - 1 + p.py) & 1) != want_qy) --ly_lo;
            constexpr int S0 = G::RB ? 0 : x_parity(G::C, c, (c >> 1) & 1, 0);
            const int npr = ly_hi > ly_lo ? (ly_hi - ly_lo + G::RSTEP - 1) / G::RSTEP : 0;
            const int nitems = (npr + G::RY - 1) / G::RY;
            const bool ok0 = xok(S0, nx_), ok1 = xok(S0 ^ 1, nx_);
            const int um = so[P.lag[J] + 2] + lane, uc = so[P.lag[J] + 1] + lane, up = so[P.lag[J]] + lane;
            const int sy = (int)p.sy;
            const double *fpl = FORM == 1 ? p.f + (int64_t)pz * p.sz + gy0 * sy + gx0 + 2 * lane : nullptr;
            int first = G::SPREAD ? (warp - ibase) % G::NW : warp;
            if (first < 0) first += G::NW;
            for (int it = first; it < nitems; it += G::NW) {
              const int ly0 = ly_lo + it * G::RY * G::RSTEP;
              unsigned vmask = 0;
#pragma unroll
              for (int r = 0; r < G::RY; ++r) {
                const int ly = ly0 + r * G::RSTEP;
                const bool xo = (G::RB && (r & 1)) ? ok1 : ok0;
                vmask |= (unsigned)(xo && ly >= ly_first && ly < ly_hi) << r;
              }
              const int rb = (ly0 - 1) * G::ROWW;
              auto ro = [&](int d, int k) -> int { return (d == 0 ? um : (d == 1 ? uc : up)) + rb + k * G::ROWW; };
              const double *frow0 = fpl + ly0 * sy;
              auto fv = [&](int r, int s) -> double {
                return ((vmask >> r) & 1) ? __ldg(frow0 + r * G::RSTEP * sy + s) : 0.0;
              };
              bad |= update_item<S, FORM, UNIT, DIV, G::RY, G::RSTEP, G::RB, G::HW, S0>(ro, fv, vmask, p);
            }
            ibase += nitems;
            if (!G::SPREAD)
              __syncthreads();
            else
              asm volatile("" ::: "memory");  // keep phases' register live ranges apart
          }(),
          ...);
    }(std::make_integer_sequence<int, G::K>{});
    if (G::SPREAD) __syncthreads();

    // ---- finished plane of the owned box -> dst ----
    const int gz_out = t - G::LAGMAX;
    if (gz_out >= z0 && gz_out < z1) {
      const int sout = so[G::LAGMAX + 1];
      double *pb = dst + (int64_t)gz_out * p.sz;
#pragma unroll
      for (int k = 0; k < G::LPT; ++k)
        if ((ownm >> k) & 1) {
          stg2(pb + goff[k], sm[sout + soff[k]], sm[sout + soff[k] + G::HW]);
          stg_pair_peers<PEER>(p, gz_out, (int64_t)gz_out * p.sz + goff[k], sm[sout + soff[k]],
                         sm[sout + soff[k] + G::HW]);
        }
    }
    {  // rotate: the slot of plane t-LAGMAX-1 becomes the slot of plane t+2
      const int tmp = so[G::W - 1];
#pragma unroll
      for (int k = G::W - 1; k > 0; --k) so[k] = so[k - 1];
      so[0] = tmp;
    }
  }
  if (bad) atomicOr(p.status, 1);
}

}  // namespace sl

// K4 (small 2D grids) reuses update_item / xoff / stg2 above
#include "k4_block2d.cuh"

namespace sl {

// ---------------------------------------------------------------------------
// host side

// K2 is instantiated only for the natural (shape, colours, weights) combos
// of the reference kinds and Q1; anything else runs the per-colour path.
static bool natural_key(const KernelKey &k) {
  switch (k.shape) {
    case FD5: return k.unit && k.div == DIV_POW2;
    case FD7: return k.unit && k.div == DIV_RCP;
    case FE9: return !k.unit && k.div == DIV_RCP;
    case FE27: return k.unit && k.div == DIV_RCP;
    case Q1: return !k.unit && k.div == DIV_RCP;
  }
  return false;
}

template <typename Fn>
static cudaError_t dispatch_fused(const KernelKey &k, Fn &&fn) {
  const bool d = k.form == 1;
  switch (k.shape) {
    case FD5: return d ? fn.template operator()<FD5, 1, true, DIV_POW2>() : fn.template operator()<FD5, 0, true, DIV_POW2>();
    case FD7: return d ? fn.template operator()<FD7, 1, true, DIV_RCP>() : fn.template operator()<FD7, 0, true, DIV_RCP>();
    case FE9: return d ? fn.template operator()<FE9, 1, false, DIV_RCP>() : fn.template operator()<FE9, 0, false, DIV_RCP>();
    case FE27: return d ? fn.template operator()<FE27, 1, true, DIV_RCP>() : fn.template operator()<FE27, 0, true, DIV_RCP>();
    case Q1: return d ? fn.template operator()<Q1, 1, false, DIV_RCP>() : fn.template operator()<Q1, 0, false, DIV_RCP>();
  }
  return cudaErrorInvalidValue;
}

static bool fused_supported(const KernelKey &key, const Params &p) {
  if (p.batch != 1 || !natural_key(key)) return false;
  if (p.px != 0) return false;  // tiles assume even global x at local x = 0
  if (p.colours != natural_colours(key.shape)) return false;
  const int64_t Sx = p.nx + 2, Sy = p.ny + 2, Sz = p.nz + 2;
  if (Sx & 1) return false;  // 16-byte row alignment
  if (Sx * Sy * (shape_dim(key.shape) == 3 ? Sz : 1) >= (int64_t(1) << 40)) return false;
  if (Sx > (1 << 20) || Sy > (1 << 20) || Sz > (1 << 20)) return false;  // 32-bit tile maths
  if (((uintptr_t)p.u & 15) || (p.f && ((uintptr_t)p.f & 15))) return false;
  return true;
}

// K6 (resident red-black 2D) needs two exchange grids and the tile flags
constexpr size_t K6_FLAG_BYTES = 4096;

static bool resident_candidate(const KernelKey &key, const Params &p) {
  return key.shape == FD5 && key.unit && key.div == DIV_POW2 && p.colours == 2 && p.px == 0 &&
         p.py == 0 && (p.nx + 2) * (p.ny + 2) <= (int64_t)4 * 1024 * 1024;
}

#ifndef SL_PEER_TU
size_t fused_workspace_bytes(const KernelKey &key, const Params &p) {
  if (!fused_supported(key, p)) return 0;
  const int64_t elems = (p.nx + 2) * (p.ny + 2) * (shape_dim(key.shape) == 3 ? (p.nz + 2) : 1);
  if (resident_candidate(key, p)) return (size_t)(2 * elems) * sizeof(double) + K6_FLAG_BYTES;
  return (size_t)elems * sizeof(double);
}
#endif

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

// Resident-block count of a kernel variant on the current device, cached per
// (thread, device): cudaFuncSetAttribute and the occupancy query are
// per-device, so a second GPU used from the same thread gets its own entry.
constexpr int MAX_DEVICES = 64;

template <typename Kern>
static cudaError_t prepare(Kern kern, size_t smem, int threads, int64_t (&cache)[MAX_DEVICES],
                           int64_t *slots) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < MAX_DEVICES && cache[dev]) {
    *slots = cache[dev];
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  int occ = 0, sms = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  *slots = (int64_t)(occ > 0 ? occ : 1) * sms;
  if (dev >= 0 && dev < MAX_DEVICES) cache[dev] = *slots;
  return cudaSuccess;
}

// 3D fp64 tensor map over a dense (n+2)^3 grid with a 64 x 32 x 1 box.
// Encoded maps are cached per (base, extents, strides, box): a sweep's passes
// alternate between two buffers, so after the first two passes no pass
// re-encodes (the cache is small and cleared when full).
struct TmapKey {
  const double *base;
  int64_t nx, ny, nz, sy, sz;
  int boxx, boxy;
  bool operator==(const TmapKey &o) const {
    return base == o.base && nx == o.nx && ny == o.ny && nz == o.nz && sy == o.sy && sz == o.sz &&
           boxx == o.boxx && boxy == o.boxy;
  }
};

static cudaError_t encode_tmap3(CUtensorMap *map, const double *base, const Params &p, int boxx,
                                int boxy);

static cudaError_t make_tmap3(CUtensorMap *map, const double *base, const Params &p,
                              int boxx = Col3Geo::PX, int boxy = Col3Geo::PY) {
  static std::mutex mu;
  static std::vector<std::pair<TmapKey, CUtensorMap>> cache;
  const TmapKey key{base, p.nx, p.ny, p.nz, p.sy, p.sz, boxx, boxy};
  std::lock_guard<std::mutex> lock(mu);
  for (const auto &e : cache)
    if (e.first == key) {
      *map = e.second;
      return cudaSuccess;
    }
  const cudaError_t e = encode_tmap3(map, base, p, boxx, boxy);
  if (e != cudaSuccess) return e;
  if (cache.size() >= 32) cache.clear();
  cache.emplace_back(key, *map);
  return cudaSuccess;
}

// L2 promotion of the plane loads (A/B: -DSL_TMAP_PROMO=CU_TENSOR_MAP_L2_PROMOTION_L2_128B / _NONE)
#ifndef SL_TMAP_PROMO
#define SL_TMAP_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
static cudaError_t encode_tmap3(CUtensorMap *map, const double *base, const Params &p, int boxx,
                                int boxy) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)(p.nx + 2), (cuuint64_t)(p.ny + 2), (cuuint64_t)(p.nz + 2)};
  const cuuint64_t strides[2] = {(cuuint64_t)p.sy * 8, (cuuint64_t)p.sz * 8};
  const cuuint32_t box[3] = {(cuuint32_t)boxx, (cuuint32_t)boxy, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides,
                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      SL_TMAP_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int S, int FORM, bool UNIT, int DIV, int M, bool PEER = false>
static cudaError_t launch_stream3d(const Params &p, const double *src, double *dst, cudaStream_t st) {
    using G = Geo3<S, M>;
    auto kern = k2_stream3d<S, FORM, UNIT, DIV, M, PEER>;
    static thread_local int64_t cache[MAX_DEVICES] = {};  // resident blocks (per kernel variant)
    int64_t slots = 0;
    {
      cudaError_t e = prepare(kern, G::SMEM, G::NT, cache, &slots);
      if (e != cudaSuccess) return e;
    }
    Tiles tl;
    const int64_t Sx = p.nx + 2, Sy = p.ny + 2, Sz = p.nz + 2;
    tl.ntx = (Sx + G::TX - 1) / G::TX;
    tl.nty = (Sy + G::TY - 1) / G::TY;
    tl.nzc = pick_chunks(tl.ntx * tl.nty, p.zhi - p.zlo, slots, G::GZ + G::LAGMAX + 1, 16);
    const int64_t items = tl.ntx * tl.nty * tl.nzc;
    kern<<<(unsigned)items, G::NT, G::SMEM, st>>>(p, src, dst, tl);
    note_launch();
    return cudaGetLastError();
}

// all neighbour weights of the shape equal (signed; |w| then equal too)
static bool equal_weights(const Params &p, int shape) {
  for (int j = 1; j < shape_nnz(shape); ++j)
    if (p.w[j] != p.w[0]) return false;
  return true;
}

// k2_q1col holds the Q1 weights as two values: all edges equal, all corners equal
static bool q1_two_weights(const Params &p) {
  for (int j = 0; j < shape_nnz(Q1); ++j) {
    const Off o = shape_off(Q1, j);
    const bool corner = o.x != 0 && o.y != 0 && o.z != 0;
    if (p.w[j] != (corner ? p.w[0] : p.w[1])) return false;
  }
  return true;
}

template <int S, int FORM, bool UNIT, int DIV, int M, bool PEER = false>
static cudaError_t launch_pass(const Params &p, const double *src, double *dst, cudaStream_t st) {
  if constexpr (S == FD7 && M == 1) {
    using G = Col3Geo;
    auto kern = k2_col3d_fd7<FORM, UNIT, DIV, PEER>;
    static thread_local int64_t cache[MAX_DEVICES] = {};  // resident blocks (per kernel variant)
    int64_t slots = 0;
    {
      cudaError_t e = prepare(kern, G::SMEM, G::NT, cache, &slots);
      if (e != cudaSuccess) return e;
    }
    CUtensorMap tmu, tmf;
    cudaError_t e = make_tmap3(&tmu, src, p, G::PX, G::BOXY);
    if (e == cudaSuccess) e = make_tmap3(&tmf, FORM == 1 ? p.f : src, p, G::PX, G::BOXY);
    if (e != cudaSuccess) return e;
    const int64_t Sx = p.nx + 2, Sy = p.ny + 2, Sz = p.nz + 2;
    const int64_t ntx = (Sx + G::TX - 1) / G::TX, nty = (Sy + G::TY - 1) / G::TY;
    // per chunk: GZ + 1 (+1 parity) ghost planes, LAGMAX drain steps and the ring fill
    const int64_t nzc = pick_chunks(ntx * nty, p.zhi - p.zlo, slots, G::GZ + G::LAGMAX + 4, 16);
    kern<<<(unsigned)(ntx * nty * nzc), G::NT, G::SMEM, st>>>(p, tmu, tmf, dst, ntx, nty, nzc);
    note_launch();
    return cudaGetLastError();
  } else if constexpr (S == Q1 && M == 1) {
    if (!q1_two_weights(p)) return launch_stream3d<S, FORM, UNIT, DIV, M, PEER>(p, src, dst, st);
    using G = Q1Geo;
    auto kern = k2_q1col<FORM, UNIT, DIV, PEER>;
    static thread_local int64_t cache[MAX_DEVICES] = {};  // resident blocks (per kernel variant)
    int64_t slots = 0;
    {
      cudaError_t e = prepare(kern, G::SMEM, G::NT, cache, &slots);
      if (e != cudaSuccess) return e;
    }
    CUtensorMap tmu;
    cudaError_t e = make_tmap3(&tmu, src, p, G::PX, G::BOXY);
    if (e != cudaSuccess) return e;
    const int64_t Sx = p.nx + 2, Sy = p.ny + 2, Sz = p.nz + 2;
    const int64_t ntx = (Sx + G::TX - 1) / G::TX, nty = (Sy + G::TY - 1) / G::TY;
    if constexpr (G::CL) {
      // nty counts pairs of tiles: each is one thread-block cluster of two CTAs along y
      const int64_t nzc = pick_chunks(2 * ntx * nty, p.zhi - p.zlo, slots, G::GZ + G::LAGMAX + G::RR, 16);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(2 * ntx * nty * nzc));
      cfg.blockDim = dim3(G::NT);
      cfg.dynamicSmemBytes = G::SMEM;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      double *dstp = dst;
      int64_t a_ntx = ntx, a_nty = nty, a_nzc = nzc;
      cudaError_t el = cudaLaunchKernelEx(&cfg, kern, p, tmu, dstp, a_ntx, a_nty, a_nzc);
      note_launch();
      return el != cudaSuccess ? el : cudaGetLastError();
    }
    const int64_t nzc = pick_chunks(ntx * nty, p.zhi - p.zlo, slots, G::GZ + G::LAGMAX + G::RR, 16);
    kern<<<(unsigned)(ntx * nty * nzc), G::NT, G::SMEM, st>>>(p, tmu, dst, ntx, nty, nzc);
    note_launch();
    return cudaGetLastError();
  } else if constexpr (shape_dim(S) == 3) {
    return launch_stream3d<S, FORM, UNIT, DIV, M, PEER>(p, src, dst, st);
  } else {
    using G = GeoS2<S, M>;
    auto run = [&](auto kern) -> cudaError_t {
      static thread_local int64_t cache[MAX_DEVICES] = {};  // resident blocks (per kernel variant)
      int64_t slots = 0;
      {
        cudaError_t e = prepare(kern, G::SMEM, 32 * G::WPB, cache, &slots);
        if (e != cudaSuccess) return e;
      }
      const int64_t Sx = p.nx + 2;
      const int64_t nstrip = (Sx + G::TX - 1) / G::TX;
      const int64_t nchunk = pick_chunks(nstrip, p.zhi - p.zlo, slots * G::WPB, G::GY + G::LAGMAX + G::U, 16);
      const int64_t warps = nstrip * nchunk;
      const int64_t blocks = (warps + G::WPB - 1) / G::WPB;
      kern<<<(unsigned)blocks, 32 * G::WPB, G::SMEM, st>>>(p, src, dst, nstrip, nchunk);
      note_launch();
      return cudaSuccess;
    };
    cudaError_t e;
    if constexpr (S == FE9 && !UNIT)
      e = equal_weights(p, S) ? run(k2_strip2d<S, FORM, UNIT, DIV, M, true, PEER>)
                              : run(k2_strip2d<S, FORM, UNIT, DIV, M, false, PEER>);
    else
      e = run(k2_strip2d<S, FORM, UNIT, DIV, M, false, PEER>);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
}

// K3: batches of 16x16 FD5 patches, every sweep in one launch, in place
static bool patch_supported(const KernelKey &key, const Params &p) {
  return p.batch >= 1 && key.shape == FD5 && key.unit && key.div == DIV_POW2 && p.colours == 2 &&
         p.nx == 16 && p.ny == 16 && p.px == 0 && p.py == 0;
}

static cudaError_t launch_patches(const KernelKey &key, const Params &p, int sweeps, cudaStream_t st) {
  const int64_t threads = p.batch * 32;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  cudaError_t e = cudaSuccess;
  if (key.form == 1)
    k3_patch16_fd5<1, true, DIV_POW2><<<blocks, 256, 0, st>>>(p, sweeps);
  else
    k3_patch16_fd5<0, true, DIV_POW2><<<blocks, 256, 0, st>>>(p, sweeps);
  note_launch();
  e = cudaGetLastError();
  return e;
}

// K6: the whole red-black 2D grid resident on chip (one tile per SM, cooperative
// launch), rounds of M sweeps between exchanges; the largest M whose tiling fits
// the co-resident CTAs (fewest exchanges: a tile's compute per sweep does not
// depend on M).  Returns cudaErrorNotSupported when no tiling fits.
template <int FORM, bool UNIT, int DIV, int M>
static cudaError_t launch_resident_m(const Params &p, double *ws, int sweeps, cudaStream_t st) {
  using R = ResGeo;
  auto kern = k6_resident2d<FORM, UNIT, DIV, M>;
  static thread_local int64_t cache[MAX_DEVICES] = {};
  int64_t slots = 0;
  {
    cudaError_t e = prepare(kern, R::SMEM, R::NT, cache, &slots);
    if (e != cudaSuccess) return e;
  }
  const int64_t Sx = p.nx + 2, Sy = p.ny + 2;
  int ntx = (int)((Sx + R::own_w(M) - 1) / R::own_w(M));
  while (2 * ((Sx / 2 + ntx - 1) / ntx) > R::own_w(M)) ++ntx;   // even tile starts
  const int nty = (int)((Sy + R::own_h(M) - 1) / R::own_h(M));
  if ((int64_t)ntx * nty > slots || (int64_t)ntx * nty * 4 > (int64_t)K6_FLAG_BYTES) return cudaErrorNotSupported;
  // every tile must own at least its ghost width, so only the 8 neighbours read it
  if (Sx / ntx < 2 * M + 2 || Sy / nty < 2 * M + 2) return cudaErrorNotSupported;
  const int64_t elems = Sx * Sy;
  double *ex0 = ws, *ex1 = ws + elems;
  int *flags = reinterpret_cast<int *>(ws + 2 * elems);
  cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)ntx * nty * sizeof(int), st);
  if (e != cudaSuccess) return e;
  Params pp = p;
  int a_ntx = ntx, a_nty = nty, a_sw = sweeps;
  void *args[] = {&pp, &ex0, &ex1, &flags, &a_ntx, &a_nty, &a_sw};
  e = cudaLaunchCooperativeKernel((const void *)kern, dim3((unsigned)(ntx * nty)), dim3(R::NT), args, R::SMEM, st);
  note_launch();
  return e;
}

template <int FORM, bool UNIT, int DIV>
static cudaError_t launch_resident(const Params &p, double *ws, int sweeps, cudaStream_t st) {
  int coop = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess || !coop)
    return cudaErrorNotSupported;
  cudaError_t e = cudaErrorNotSupported;
  [&]<int... Ms>(std::integer_sequence<int, Ms...>) {
    // M = MAXM, MAXM-1, ..., 1: first that fits
    ((e == cudaErrorNotSupported ? (e = launch_resident_m<FORM, UNIT, DIV, ResGeo::MAXM - Ms>(p, ws, sweeps, st))
                                 : e),
     ...);
  }(std::make_integer_sequence<int, ResGeo::MAXM>{});
  return e;
}

// K4: 2D grids small enough to be L2-resident run M sweeps per pass in
// shared-memory tiles (one wave of 1024-thread CTAs).
static bool block2d_preferred(const KernelKey &key, const Params &p) {
  return shape_dim(key.shape) == 2 && (p.nx + 2) * (p.ny + 2) <= (int64_t)4 * 1024 * 1024;
}

template <int S, int FORM, bool UNIT, int DIV, int M>
static cudaError_t launch_block2d(const Params &p, const double *src, double *dst, cudaStream_t st) {
  using G = GeoB2<S, M>;
  auto kern = k4_block2d<S, FORM, UNIT, DIV, M>;
  static thread_local int64_t cache[MAX_DEVICES] = {};  // resident blocks (per kernel variant)
  int64_t slots = 0;
  {
    cudaError_t e = prepare(kern, G::SMEM, G::NT, cache, &slots);
    if (e != cudaSuccess) return e;
  }
  const int64_t Sx = p.nx + 2, Sy = p.ny + 2;
  // Tile count: at least what the maximal tile needs; more (smaller) tiles
  // when that fills idle SMs of the wave — cost = waves x work per tile incl. ghost.
  const int ntx0 = (int)((Sx + G::TX - 1) / G::TX), nty0 = (int)((Sy + G::TY - 1) / G::TY);
  int ntx = ntx0, nty = nty0;
  double best = 1e300;
  for (int a = ntx0; a <= ntx0 + 8; ++a)
    for (int b = nty0; b <= nty0 + 32; ++b) {
      const int64_t waves = ((int64_t)a * b + slots - 1) / slots;
      const double w = 2.0 * (double)((Sx / 2 + a - 1) / a) + 2 * G::GX;
      const double h = (double)((Sy + b - 1) / b) + 2 * G::GY;
      const double cost = (double)waves * w * h;
      if (cost < best * 0.999) {
        best = cost;
        ntx = a;
        nty = b;
      }
    }
  kern<<<(unsigned)(ntx * nty), G::NT, G::SMEM, st>>>(p, src, dst, ntx, nty);
  note_launch();
  return cudaGetLastError();
}

#ifdef SL_PEER_TU
// the peer-exchange instantiations (own translation unit: k2_peer.cu)
cudaError_t launch_one_pass_peer(const KernelKey &key, const Params &p, const double *src, double *dst,
                                 cudaStream_t st) {
  return dispatch_fused(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
    return launch_pass<S, F, U, D, 1, true>(p, src, dst, st);
  });
}
#else
cudaError_t launch_one_pass(const KernelKey &key, const Params &p, const double *src, double *dst,
                            cudaStream_t st, int *handled) {
  *handled = 0;
  if (p.batch > 1 || !fused_supported(key, p)) return cudaSuccess;
  if (((uintptr_t)src & 15) || ((uintptr_t)dst & 15)) return cudaSuccess;
  *handled = 1;
  if (p.zhi <= p.zlo) return cudaSuccess;
  if (p.pdn || p.pup) return launch_one_pass_peer(key, p, src, dst, st);
  return dispatch_fused(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
    return launch_pass<S, F, U, D, 1>(p, src, const_cast<double *>(dst), st);
  });
}

cudaError_t launch_fused(const KernelKey &key, const Params &p, int sweeps, double *workspace,
                         size_t workspace_bytes, cudaStream_t st, int *handled, bool stream_only) {
  *handled = 0;
  if (p.batch > 1 || (!stream_only && p.nx == 16 && p.ny == 16 && shape_dim(key.shape) == 2)) {
    if (!patch_supported(key, p)) return cudaSuccess;
    *handled = 1;
    return launch_patches(key, p, sweeps, st);
  }
  if (!fused_supported(key, p)) return cudaSuccess;
  const size_t need = fused_workspace_bytes(key, p);
  if (!workspace || workspace_bytes < need || ((uintptr_t)workspace & 15)) return cudaSuccess;
  // the grid itself (the workspace may be larger: K6 keeps its exchange grids there)
  const size_t grid_bytes = (size_t)((p.nx + 2) * (p.ny + 2) * (shape_dim(key.shape) == 3 ? (p.nz + 2) : 1)) * sizeof(double);
  *handled = 1;
  // passes alternate u -> ws -> u ...; an odd count ends with one copy back
  double *bufs[2] = {p.u, workspace};
  int cur = 0;
  cudaError_t e = cudaSuccess;
  if (!stream_only && resident_candidate(key, p) && workspace_bytes >= need) {
    cudaError_t er = dispatch_fused(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
      if constexpr (S == FD5 && U && D == DIV_POW2)
        return launch_resident<F, U, D>(p, workspace, sweeps, st);
      else
        return cudaErrorNotSupported;
    });
    if (er != cudaErrorNotSupported) return er;
    cudaGetLastError();   // clear the (non-sticky) not-supported status
  }
  if (!stream_only && block2d_preferred(key, p)) {
    // FD5: 4 sweeps per pass, FE9: 2 (ghost 8 columns); remainder 1 at a time
    // (8 FD5 sweeps per pass measured slower: ghost and phase count outgrow the saved passes)
    for (int s = 0; s < sweeps && e == cudaSuccess;) {
      const int left = sweeps - s;
      const int m = key.shape == FD5 ? (left >= 4 ? 4 : 1) : (left >= 2 ? 2 : 1);
      e = dispatch_fused(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
        if constexpr (S == FD5)
          return m == 4 ? launch_block2d<S, F, U, D, 4>(p, bufs[cur], bufs[cur ^ 1], st)
                        : launch_block2d<S, F, U, D, 1>(p, bufs[cur], bufs[cur ^ 1], st);
        else if constexpr (S == FE9)
          return m == 2 ? launch_block2d<S, F, U, D, 2>(p, bufs[cur], bufs[cur ^ 1], st)
                        : launch_block2d<S, F, U, D, 1>(p, bufs[cur], bufs[cur ^ 1], st);
        else
          return cudaErrorInvalidValue;
      });
      s += m;
      cur ^= 1;
    }
    if (e == cudaSuccess && cur == 1) {
      e = cudaMemcpyAsync(p.u, workspace, grid_bytes, cudaMemcpyDeviceToDevice, st);
      note_launch();
    }
    return e;
  }
  // FD5 (red-black 2D) fuses two sweeps per pass: half the passes, and the
  // 2-sweep ghost (4 columns/rows) still fits a 64-column strip
  // FD5 and FE9 fuse two sweeps per pass (FE9: 241 vs 230 GLUP/s on config 2,
  // DESIGN.md §8); -DSL_NO_FE9_M2 restores one FE9 sweep per pass, -DSL_FD7_M2 runs
  // FD7 two sweeps per pass through the generic stream kernel (A/B only)
#ifndef SL_NO_FE9_M2
#define SL_FE9_M2
#endif
#ifdef SL_FD7_M2
  const bool two = (key.shape == FD5 || key.shape == FE9 || key.shape == FD7) && sweeps >= 2;
#elif defined(SL_FE9_M2)
  const bool two = (key.shape == FD5 || key.shape == FE9) && sweeps >= 2;
#else
  const bool two = key.shape == FD5 && sweeps >= 2;
#endif
  for (int s = 0; s < sweeps && e == cudaSuccess;) {
    const int m = (two && sweeps - s >= 2) ? 2 : 1;
    e = dispatch_fused(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
      if constexpr (S == FD5)
        return m == 2 ? launch_pass<S, F, U, D, 2>(p, bufs[cur], bufs[cur ^ 1], st)
                      : launch_pass<S, F, U, D, 1>(p, bufs[cur], bufs[cur ^ 1], st);
#ifdef SL_FE9_M2
      else if constexpr (S == FE9)
        return m == 2 ? launch_pass<S, F, U, D, 2>(p, bufs[cur], bufs[cur ^ 1], st)
                      : launch_pass<S, F, U, D, 1>(p, bufs[cur], bufs[cur ^ 1], st);
#endif
#ifdef SL_FD7_M2
      else if constexpr (S == FD7)
        return m == 2 ? launch_stream3d<S, F, U, D, 2>(p, bufs[cur], bufs[cur ^ 1], st)
                      : launch_pass<S, F, U, D, 1>(p, bufs[cur], bufs[cur ^ 1], st);
#endif
      else
        return launch_pass<S, F, U, D, 1>(p, bufs[cur], bufs[cur ^ 1], st);
    });
    s += m;
    cur ^= 1;
  }
  if (e == cudaSuccess && cur == 1) {
    e = cudaMemcpyAsync(p.u, workspace, grid_bytes, cudaMemcpyDeviceToDevice, st);
    note_launch();
  }
  return e;
}

#endif  // SL_PEER_TU

}  // namespace sl
