// k1_colour.cu — K1: one colour phase in place over a dense grid, plus the
// indexed update (update_cells_batch) and the residual reduction.
//
// K1 replaces one `pool.parallel_for(rows, body)` pass of sweep_colouring
// (reference strategies.py:374-393 -> kernels.update_cells_batch,
// kernels.py:212-251): the colour's rows become grid.y, the colour's points
// of a row (every other x) become threads.  Same-colour points are never
// adjacent (reference tests/test_strategies.py:41-51), so the pass is
// race-free and its result independent of thread order.  It reads the whole
// grid and writes 1/c of it per phase: the simple, always-available path
// (and the independent GPU oracle behind sweep_colouring_reference).
#include "k1_colour.cuh"

namespace sl {

template <int S, int FORM, bool UNIT, int DIV>
__global__ void __launch_bounds__(256)
k1_colour_pass(Params p, int colour, RowMap rm) {
  constexpr int DIM = shape_dim(S);
  constexpr int NNZ = shape_nnz(S);
  const bool merged = colour < 0;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t r = blockIdx.y; r < rm.rows; r += gridDim.y) {
    const int64_t per_b = rm.cy * rm.cz;
    const int64_t b = r / per_b;
    const int64_t rem = r - b * per_b;
    const int64_t zi = rem / rm.cy;
    const int64_t yi = rem - zi * rm.cy;
    const int64_t y = rm.y0 + yi * rm.ystep;
    const int64_t z = DIM == 3 ? rm.z0 + zi * rm.zstep : 0;
    int64_t x;
    if (merged) {
      x = 1 + t;
    } else {
      const int qy = (int)((y - 1 + p.py) & 1);
      const int qz = DIM == 3 ? (int)((z - 1 + p.pz) & 1) : 0;
      const int qx = p.colours == 2 ? ((colour + qy + qz) & 1) : (colour & 1);
      x = 1 + ((qx ^ p.px) & 1) + 2 * t;
    }
    if (x > p.nx) continue;
    double *ub = p.u + b * p.bstride;
    const double *fb = FORM == 1 ? p.f + b * p.bstride : nullptr;
    const int64_t c = z * p.sz + y * p.sy + x;
    const double uc = ub[c];
    double acc = acc_init<FORM, UNIT>(uc, p);
#pragma unroll
    for (int j = 0; j < NNZ; ++j) {
      const Off o = shape_off(S, j);
      acc = acc_add<FORM, UNIT>(acc, ub[c + o.x + o.y * p.sy + o.z * p.sz], j, p);
    }
    const double out = acc_finish<FORM, UNIT, DIV>(acc, uc, FORM == 1 ? fb[c] : 0.0, p);
    if (!finite64(out)) atomicOr(p.status, 1);
    ub[c] = out;
  }
}

// Indexed update in two stream-ordered launches, so that a batch with a
// non-finite result leaves the mesh untouched like the reference
// (kernels.py:243-251: the check precedes `u[F] = out`): COMMIT = false only
// flags, COMMIT = true recomputes (the cells are mutually non-adjacent, so the
// inputs are unchanged and the values identical) and stores iff no flag is set.
template <int S, int FORM, bool UNIT, int DIV, bool COMMIT>
__global__ void __launch_bounds__(256)
k1_update_cells(Params p, const int64_t *__restrict__ flats, int64_t count) {
  constexpr int NNZ = shape_nnz(S);
  if (COMMIT && *(volatile int32_t *)p.status != 0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = flats[i];
    const double uc = p.u[c];
    double acc = acc_init<FORM, UNIT>(uc, p);
#pragma unroll
    for (int j = 0; j < NNZ; ++j) acc = acc_add<FORM, UNIT>(acc, p.u[c + p.delta[j]], j, p);
    const double out = acc_finish<FORM, UNIT, DIV>(acc, uc, FORM == 1 ? p.f[c] : 0.0, p);
    if (COMMIT)
      p.u[c] = out;
    else if (!finite64(out))
      atomicOr(p.status, 1);
  }
}

// residual: max |Au| (Form R) or |f - Au| (Form D), Au accumulated exactly
// like reference residual_max (kernels.py:260-264): acc = w_c*u; acc += w_j*u_j.
template <int S, int FORM>
__global__ void __launch_bounds__(256)
k1_residual(Params p, RowMap rm, unsigned long long *out) {
  constexpr int DIM = shape_dim(S);
  constexpr int NNZ = shape_nnz(S);
  unsigned long long best = 0;  // bit pattern of a non-negative double (monotone)
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t r = blockIdx.y; r < rm.rows; r += gridDim.y) {
    const int64_t per_b = rm.cy * rm.cz;
    const int64_t b = r / per_b;
    const int64_t rem = r - b * per_b;
    const int64_t z = DIM == 3 ? 1 + rem / rm.cy : 0;
    const int64_t y = 1 + (rem % rm.cy);
    const int64_t x = 1 + t;
    if (x > p.nx) continue;
    const double *ub = p.u + b * p.bstride;
    const int64_t c = z * p.sz + y * p.sy + x;
    double acc = __dmul_rn(p.wc, ub[c]);
#pragma unroll
    for (int j = 0; j < NNZ; ++j) {
      const Off o = shape_off(S, j);
      acc = __dadd_rn(acc, __dmul_rn(p.w[j], ub[c + o.x + o.y * p.sy + o.z * p.sz]));
    }
    if (FORM == 1) acc = __dsub_rn(p.f[b * p.bstride + c], acc);
    const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(acc));
    best = bits > best ? bits : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
    best = v > best ? v : best;
  }
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

// Lexicographic Gauss-Seidel (reference serial sweep, strategies.py:341-345):
// a point's earlier-in-lex neighbours all lie on smaller hyperplanes
// t = x + y (+ z) (face stencils) or t = x + 2y (+ 4z) (box stencils) and its
// later ones on larger hyperplanes, so sweeping the hyperplanes in order with
// all points of one hyperplane in parallel reproduces the lex order exactly.
template <int S, int FORM, bool UNIT, int DIV>
__global__ void __launch_bounds__(256)
k1_hyperplane(Params p, int64_t h, int64_t rows) {
  constexpr int DIM = shape_dim(S);
  constexpr int NNZ = shape_nnz(S);
  constexpr bool FACE = (S == FD5 || S == FD7);
  const int64_t ay = FACE ? 1 : 2, az = FACE ? 1 : 4;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t per_b = p.ny * p.nz;
    const int64_t b = r / per_b;
    const int64_t rem = r - b * per_b;
    const int64_t z = DIM == 3 ? 1 + rem / p.ny : 0;
    const int64_t y = 1 + rem % p.ny;
    const int64_t x = h - ay * y - (DIM == 3 ? az * z : 0);
    if (x < 1 || x > p.nx) continue;
    double *ub = p.u + b * p.bstride;
    const double *fb = FORM == 1 ? p.f + b * p.bstride : nullptr;
    const int64_t c = z * p.sz + y * p.sy + x;
    const double uc = ub[c];
    double acc = acc_init<FORM, UNIT>(uc, p);
#pragma unroll
    for (int j = 0; j < NNZ; ++j) {
      const Off o = shape_off(S, j);
      acc = acc_add<FORM, UNIT>(acc, ub[c + o.x + o.y * p.sy + o.z * p.sz], j, p);
    }
    const double out = acc_finish<FORM, UNIT, DIV>(acc, uc, FORM == 1 ? fb[c] : 0.0, p);
    if (!finite64(out)) atomicOr(p.status, 1);
    ub[c] = out;
  }
}

// ---------------------------------------------------------------------------
// launchers

static RowMap colour_rows(const Params &p, int dim, int colour) {
  RowMap rm{};
  rm.ystep = rm.zstep = 1;
  rm.y0 = rm.z0 = 1;
  rm.cy = p.ny;
  rm.cz = dim == 3 ? p.nz : 1;
  if (colour >= 0 && p.colours != 2) {
    // per-axis parity colours: only rows whose (y, z) parities match
    const int qy = (colour >> 1) & 1, qz = (colour >> 2) & 1;
    rm.ystep = 2;
    rm.y0 = 1 + ((qy ^ p.py) & 1);
    rm.cy = rm.y0 <= p.ny ? (p.ny - rm.y0) / 2 + 1 : 0;
    if (dim == 3) {
      rm.zstep = 2;
      rm.z0 = 1 + ((qz ^ p.pz) & 1);
      rm.cz = rm.z0 <= p.nz ? (p.nz - rm.z0) / 2 + 1 : 0;
    }
  }
  rm.rows = p.batch * rm.cy * rm.cz;
  return rm;
}

cudaError_t launch_colour_pass(const KernelKey &key, const Params &p, int colour, cudaStream_t st) {
  const int dim = shape_dim(key.shape);
  const RowMap rm = colour_rows(p, dim, colour);
  if (rm.rows == 0 || p.nx == 0) return cudaSuccess;
  const int64_t pts = colour < 0 ? p.nx : (p.nx + 1) / 2;
  const int threads = pts >= 256 ? 256 : (pts >= 128 ? 128 : 64);
  dim3 grid((unsigned)((pts + threads - 1) / threads), (unsigned)(rm.rows < 65535 ? rm.rows : 65535));
  return dispatch(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
    k1_colour_pass<S, F, U, D><<<grid, threads, 0, st>>>(p, colour, rm);
    note_launch();
    return cudaGetLastError();
  });
}

cudaError_t launch_lex_sweep(const KernelKey &key, const Params &p, cudaStream_t st) {
  const int dim = shape_dim(key.shape);
  const bool face = key.shape == FD5 || key.shape == FD7;
  const int64_t ay = face ? 1 : 2, az = face ? 1 : 4;
  const int64_t hmin = 1 + ay + (dim == 3 ? az : 0);
  const int64_t hmax = p.nx + ay * p.ny + (dim == 3 ? az * p.nz : 0);
  const int64_t rows = p.batch * p.ny * p.nz;
  const int threads = 256;
  int64_t blocks = (rows + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaError_t e = cudaSuccess;
  for (int64_t h = hmin; h <= hmax && e == cudaSuccess; ++h) {
    e = dispatch(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
      k1_hyperplane<S, F, U, D><<<(unsigned)blocks, threads, 0, st>>>(p, h, rows);
      note_launch();
      return cudaGetLastError();
    });
  }
  return e;
}

cudaError_t launch_update_cells(const KernelKey &key, const Params &p, const int64_t *flats,
                                int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (count + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  return dispatch(key, [&]<int S, int F, bool U, int D>() -> cudaError_t {
    k1_update_cells<S, F, U, D, false><<<(unsigned)blocks, threads, 0, st>>>(p, flats, count);
    k1_update_cells<S, F, U, D, true><<<(unsigned)blocks, threads, 0, st>>>(p, flats, count);
    note_launch(2);
    return cudaGetLastError();
  });
}

cudaError_t launch_residual(const KernelKey &key, const Params &p, double *d_out, cudaStream_t st) {
  const int dim = shape_dim(key.shape);
  RowMap rm = colour_rows(p, dim, -1);
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(double), st);
  if (e != cudaSuccess || rm.rows == 0 || p.nx == 0) return e;
  const int threads = p.nx >= 256 ? 256 : 64;
  dim3 grid((unsigned)((p.nx + threads - 1) / threads), (unsigned)(rm.rows < 65535 ? rm.rows : 65535));
  auto *out = reinterpret_cast<unsigned long long *>(d_out);
  KernelKey k = key;
  k.unit = false;
  k.div = DIV_IEEE;
  return dispatch(k, [&]<int S, int F, bool U, int D>() -> cudaError_t {
    if constexpr (U || D) {  // residual depends on shape and form only
      return cudaErrorNotSupported;
    } else {
      k1_residual<S, F><<<grid, threads, 0, st>>>(p, rm, out);
      note_launch();
      return cudaGetLastError();
    }
  });
}

}  // namespace sl
