// k5_cost.cu — the reference cost model on the device (kernels.py:113-145,
// :168-200, :234-244).  With k > 0 every stencil entry and the centre get
// k sine evaluations d = sum_i sin(x + i); the entry's weight is perturbed by
// 0.0*d and the centre divisor by 0.0*d_centre, which leaves every value
// bit-identical to the k = 0 update while the sines still execute.  Their
// sum goes into a device work tally so the compiler cannot drop them.
//
// This is compute-bound (k*(nnz+1) double sines per cell) and therefore a
// plain one-thread-per-cell kernel: colour phases (colouring / hyb-*) or the
// lexicographic hyperplane wavefront (serial / taskgraph).  All the exact
// division rewrites of the fast paths produce the correctly rounded quotient,
// so IEEE division here gives the same bits.
#include "k5_cost.cuh"

namespace sl {

namespace {

__device__ __forceinline__ double sine_work(double x, int k) {
  double d = 0.0;
  for (int i = 0; i < k; ++i) d = __dadd_rn(d, sin(__dadd_rn(x, (double)i)));
  return d;
}

template <int S, int FORM>
__device__ __forceinline__ double cost_update(const Params &p, double *ub, const double *fb,
                                              int64_t c, int k, double &work) {
  constexpr int NNZ = shape_nnz(S);
  const double uc = ub[c];
  const double dc = sine_work(uc, k);
  double dummy = dc;
  const double wc = __dadd_rn(p.wc, __dmul_rn(0.0, dc));
  double acc = FORM == 0 ? 0.0 : __dmul_rn(wc, uc);
#pragma unroll
  for (int j = 0; j < NNZ; ++j) {
    const Off o = shape_off(S, j);
    const double x = ub[c + o.x + o.y * p.sy + o.z * p.sz];
    const double d = sine_work(x, k);
    dummy = __dadd_rn(dummy, d);
    const double wj = __dadd_rn(FORM == 0 ? p.aw[j] : p.w[j], __dmul_rn(0.0, d));
    acc = __dadd_rn(acc, __dmul_rn(wj, x));
  }
  work = __dadd_rn(work, dummy);
  if (FORM == 0) return __ddiv_rn(acc, wc);
  return __dadd_rn(uc, __dmul_rn(p.omega, __ddiv_rn(__dsub_rn(fb[c], acc), wc)));
}

__device__ __forceinline__ int cell_k(const Params &p, const CostSpec &c, int64_t x, int64_t y,
                                      int64_t z) {
  if (!c.ramp) return c.k;
  const int64_t total = p.nx * p.ny * p.nz;
  const int64_t rank = ((z > 0 ? z - 1 : 0) * p.ny + (y - 1)) * p.nx + (x - 1);
  const int64_t k = (100 * rank) / total;
  return (int)(k < 99 ? k : 99);
}

__device__ __forceinline__ void flush_work(double work, double *out) {
  for (int o = 16; o > 0; o >>= 1) work += __shfl_xor_sync(0xffffffffu, work, o);
  if ((threadIdx.x & 31) == 0 && out) atomicAdd(out, work);
}

// items: per (b, z, y) row, `xw` candidate points; phase >= 0 colour, < 0 lex
// hyperplane h (one candidate per row)
template <int S, int FORM>
__global__ void __launch_bounds__(128)
k5_cost_phase(Params p, CostSpec cs, int colour, int64_t h, int64_t xw, int64_t items) {
  constexpr int DIM = shape_dim(S);
  constexpr bool FACE = (S == FD5 || S == FD7);
  double work = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < items;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / xw, t = i - r * xw;
    const int64_t per_b = p.ny * p.nz;
    const int64_t b = r / per_b;
    const int64_t rem = r - b * per_b;
    const int64_t z = DIM == 3 ? 1 + rem / p.ny : 0;
    const int64_t y = 1 + rem % p.ny;
    int64_t x;
    if (colour >= 0) {
      const int qy = (int)((y - 1 + p.py) & 1);
      const int qz = DIM == 3 ? (int)((z - 1 + p.pz) & 1) : 0;
      const int qx = p.colours == 2 ? ((colour + qy + qz) & 1) : (colour & 1);
      if (p.colours != 2 && (qy != ((colour >> 1) & 1) || (DIM == 3 && qz != ((colour >> 2) & 1))))
        continue;
      x = 1 + ((qx ^ p.px) & 1) + 2 * t;
    } else {
      x = h - (FACE ? 1 : 2) * y - (DIM == 3 ? (FACE ? 1 : 4) * z : 0);
      if (x < 1) continue;
    }
    if (x > p.nx) continue;
    double *ub = p.u + b * p.bstride;
    const double *fb = FORM == 1 ? p.f + b * p.bstride : nullptr;
    const int64_t c = z * p.sz + y * p.sy + x;
    const double out = cost_update<S, FORM>(p, ub, fb, c, cell_k(p, cs, x, y, z), work);
    if (!finite64(out)) atomicOr(p.status, 1);
    ub[c] = out;
  }
  flush_work(work, cs.work);
}

// Two launches like k1_update_cells: COMMIT = false flags and tallies the
// sine work, COMMIT = true stores iff nothing was flagged (values are
// bitwise independent of k, so the commit pass runs with k = 0).
template <int S, int FORM, bool COMMIT>
__global__ void __launch_bounds__(128)
k5_cost_cells(Params p, CostSpec cs, const int64_t *__restrict__ flats, int64_t count) {
  if (COMMIT && *(volatile int32_t *)p.status != 0) return;
  double work = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = flats[i];
    const double out = cost_update<S, FORM>(p, p.u, p.f, c, COMMIT ? 0 : cs.k, work);
    if (COMMIT)
      p.u[c] = out;
    else if (!finite64(out))
      atomicOr(p.status, 1);
  }
  if (!COMMIT) flush_work(work, cs.work);
}

KernelKey generic(KernelKey k) {
  k.unit = false;
  k.div = DIV_IEEE;
  return k;
}

unsigned blocks_for(int64_t items, int threads) {
  int64_t b = (items + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b > 0 ? b : 1);
}

}  // namespace

cudaError_t launch_cost_sweep_phase(const KernelKey &key, const Params &p, const CostSpec &c,
                                    int colour, cudaStream_t st) {
  const int dim = shape_dim(key.shape);
  const int64_t rows = p.batch * p.ny * p.nz;
  const int threads = 128;
  if (colour >= 0) {
    const int64_t xw = (p.nx + 1) / 2;
    const int64_t items = rows * xw;
    return dispatch(generic(key), [&]<int S, int F, bool U, int D>() -> cudaError_t {
      if constexpr (U || D) {
        return cudaErrorNotSupported;
      } else {
        k5_cost_phase<S, F><<<blocks_for(items, threads), threads, 0, st>>>(p, c, colour, 0, xw,
                                                                           items);
        note_launch();
        return cudaGetLastError();
      }
    });
  }
  const bool face = key.shape == FD5 || key.shape == FD7;
  const int64_t ay = face ? 1 : 2, az = face ? 1 : 4;
  const int64_t hmin = 1 + ay + (dim == 3 ? az : 0);
  const int64_t hmax = p.nx + ay * p.ny + (dim == 3 ? az * p.nz : 0);
  cudaError_t e = cudaSuccess;
  for (int64_t h = hmin; h <= hmax && e == cudaSuccess; ++h) {
    e = dispatch(generic(key), [&]<int S, int F, bool U, int D>() -> cudaError_t {
      if constexpr (U || D) {
        return cudaErrorNotSupported;
      } else {
        k5_cost_phase<S, F><<<blocks_for(rows, threads), threads, 0, st>>>(p, c, -1, h, 1, rows);
        note_launch();
        return cudaGetLastError();
      }
    });
  }
  return e;
}

cudaError_t launch_cost_cells(const KernelKey &key, const Params &p, const CostSpec &c,
                              const int64_t *flats, int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int threads = 128;
  return dispatch(generic(key), [&]<int S, int F, bool U, int D>() -> cudaError_t {
    if constexpr (U || D) {
      return cudaErrorNotSupported;
    } else {
      k5_cost_cells<S, F, false><<<blocks_for(count, threads), threads, 0, st>>>(p, c, flats, count);
      k5_cost_cells<S, F, true><<<blocks_for(count, threads), threads, 0, st>>>(p, c, flats, count);
      note_launch(2);
      return cudaGetLastError();
    }
  });
}

}  // namespace sl
