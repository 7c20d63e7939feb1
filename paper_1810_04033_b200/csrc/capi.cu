// capi.cu — the extern "C" boundary (include/stencil_sweep.h): argument
// validation (reference error conventions), shape/weight
// resolution to a kernel template key, and the sweep driver that picks the
// fused (K2/K3) or per-colour (K1) kernels.
#include <atomic>
#include <cmath>
#include <cstring>

#include "../../include/stencil_sweep.h"
#include "k1_colour.cuh"
#include "k5_cost.cuh"
#include "k2_fused.cuh"
#include "plan.cuh"

#include <vector>

namespace sl {

static thread_local int g_last_cuda = 0;
static std::atomic<uint64_t> g_launches{0};

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return SL_OK;
  g_last_cuda = (int)e;
  return SL_E_CUDA;
}

// Canonical offsets of the public sl_shape (FE27 = all 26).
static int public_shape_internal(int shape) {
  switch (shape) {
    case SL_FD5: return FD5;
    case SL_FE9: return FE9;
    case SL_FD7: return FD7;
    case SL_FE27: return FE27;
  }
  return -1;
}

static bool is_pow2(double v) {
  if (!(v > 0.0) || !std::isfinite(v)) return false;
  int e;
  double m = std::frexp(v, &e);
  return m == 0.5 && e > -1000 && e < 1000;
}

// Resolve shape + weights into a kernel key and fill the weight tables.
static int resolve(const sl_stencil *s, int dim, KernelKey *key, Params *p) {
  const int base = public_shape_internal(s->shape);
  if (base < 0 || shape_dim(base) != dim) return SL_E_INVAL;
  if (s->form != SL_FORM_R && s->form != SL_FORM_D) return SL_E_INVAL;
  if (!(s->colours == 2 || s->colours == (1 << dim))) return SL_E_INVAL;
  // red-black needs a face-only neighbour set, else same-colour cells touch
  if (s->colours == 2 && !(base == FD5 || base == FD7)) return SL_E_INVAL;
  if (!std::isfinite(s->wc) || s->wc == 0.0) return SL_E_INVAL;
  const int nb = shape_nnz(base);
  int shape = base;
  bool has_zero = false;
  for (int j = 0; j < nb; ++j) has_zero |= (s->w[j] == 0.0);
  if (has_zero) {
    if (base != FE27) return SL_E_UNSUPPORTED;
    // only the Q1 pattern (all faces zero, edges/corners non-zero) has a kernel
    for (int j = 0; j < nb; ++j) {
      const Off o = shape_off(FE27, j);
      const int nzc = (o.x != 0) + (o.y != 0) + (o.z != 0);
      if ((nzc == 1) != (s->w[j] == 0.0)) return SL_E_UNSUPPORTED;
    }
    shape = Q1;
  }
  // compact weights in the kernel shape's canonical order
  int k = 0;
  bool unit = true;
  for (int j = 0; j < nb; ++j) {
    if (s->w[j] == 0.0) continue;
    if (!std::isfinite(s->w[j])) return SL_E_INVAL;
    p->w[k] = s->w[j];
    p->aw[k] = std::fabs(s->w[j]);
    unit &= (s->w[j] == -1.0);
    ++k;
  }
  if (k != shape_nnz(shape)) return SL_E_UNSUPPORTED;
  p->wc = s->wc;
  p->omega = s->omega;
  p->colours = s->colours;
  key->shape = shape;
  key->form = s->form;
  key->unit = unit;
  // rwc = RN(1/w_c): exact for a power of two, the Markstein seed otherwise
  key->div = is_pow2(std::fabs(s->wc)) ? DIV_POW2
             : (s->wc > 0.0 && std::isnormal(s->wc) && std::isnormal(1.0 / s->wc)) ? DIV_RCP
                                                                                  : DIV_IEEE;
  p->rwc = 1.0 / s->wc;
  return SL_OK;
}

static int make_params(const sl_grid *g, const sl_stencil *s, int32_t *d_status, KernelKey *key,
                       Params *p) {
  if (!g || !s) return SL_E_INVAL;
  std::memset(p, 0, sizeof(*p));
  if (g->dim != 2 && g->dim != 3) return SL_E_INVAL;
  for (int a = 0; a < g->dim; ++a)
    if (g->n[a] < 0) return SL_E_INVAL;
  if (g->batch < 1 || !g->u) return SL_E_INVAL;
  const int64_t sx = g->n[0] + 2, sy = g->n[1] + 2, sz = g->dim == 3 ? g->n[2] + 2 : 1;
  if (g->batch > 1 && g->batch_stride < sx * sy * sz) return SL_E_INVAL;
  int rc = resolve(s, g->dim, key, p);
  if (rc != SL_OK) return rc;
  if (s->form == SL_FORM_D && !g->f) return SL_E_INVAL;
  p->u = g->u;
  p->f = g->f;
  p->status = d_status;
  p->nx = g->n[0];
  p->ny = g->n[1];
  p->nz = g->dim == 3 ? g->n[2] : 1;
  p->sy = sx;
  p->sz = g->dim == 3 ? sx * sy : 0;
  p->batch = g->batch;
  p->bstride = g->batch_stride;
  p->px = (int)(g->origin[0] & 1);
  p->py = (int)(g->origin[1] & 1);
  p->pz = g->dim == 3 ? (int)(g->origin[2] & 1) : 0;
  p->zlo = 0;
  p->zhi = (int32_t)(g->dim == 3 ? sz : sy);
  for (int j = 0; j < shape_nnz(key->shape); ++j) {
    const Off o = shape_off(key->shape, j);
    p->delta[j] = o.x + o.y * p->sy + o.z * p->sz;
  }
  return SL_OK;
}

static bool empty_grid(const Params &p) { return p.nx == 0 || p.ny == 0 || p.nz == 0; }

// Launches go to the device that owns the caller's stream (a tensor on a
// non-current GPU comes with that GPU's stream): make it current for the call
// and restore the caller's device afterwards.  The legacy/per-thread default
// streams (0, 1, 2) belong to the current device.
class StreamDevice {
 public:
  explicit StreamDevice(void *stream) {
    if ((uintptr_t)stream <= 2 || cudaGetDevice(&prev_) != cudaSuccess) return;
    int dev = prev_;
    if (cudaStreamGetDevice((cudaStream_t)stream, &dev) == cudaSuccess && dev != prev_ &&
        cudaSetDevice(dev) == cudaSuccess)
      switched_ = true;
  }
  ~StreamDevice() {
    if (switched_) cudaSetDevice(prev_);
  }
  StreamDevice(const StreamDevice &) = delete;
  StreamDevice &operator=(const StreamDevice &) = delete;

 private:
  int prev_ = 0;
  bool switched_ = false;
};

// Host version of plan.cuh's margin DP for any number of sweeps: the input
// margin along axis `axis` that `sweeps` fused sweeps of `shape` consume.
static int load_margin(int shape, int colours, int sweeps, int axis) {
  const int K = sweeps * colours;
  const int nnz = shape_nnz(shape);
  std::vector<int> need(K, -1);
  for (int c = 0; c < colours; ++c)
    for (int k = K - 1; k >= 0; --k)
      if (k % colours == c) {
        need[k] = 0;
        break;
      }
  int load = 0;
  for (int j = K - 1; j >= 0; --j) {
    if (need[j] < 0) continue;
    for (int q = 0; q < nnz; ++q) {
      const Off o = shape_off(shape, q);
      const int b = (j % colours) ^ colour_flip(colours, o);
      int i = j - 1;
      while (i >= 0 && i % colours != b) --i;
      const int req = need[j] + cabs(off_axis(o, axis));
      if (i >= 0)
        need[i] = cmax(need[i], req);
      else
        load = cmax(load, req);
    }
  }
  return load;
}

}  // namespace sl

using namespace sl;

extern "C" {

int sl_abi_version(void) { return SL_ABI_VERSION; }

const char *sl_strerror(int code) {
  switch (code) {
    case SL_OK: return "ok";
    case SL_E_NONFINITE: return "non-finite cell update";
    case SL_E_INVAL: return "invalid argument";
    case SL_E_CUDA: return "CUDA error";
    case SL_E_UNSUPPORTED: return "unsupported stencil shape or weight pattern";
  }
  return "unknown status";
}

int sl_last_cuda_error(void) { return g_last_cuda; }

uint64_t sl_launch_count(void) { return g_launches.load(); }

size_t sl_workspace_bytes(const sl_grid *g, const sl_stencil *s) {
  KernelKey key;
  Params p;
  if (make_params(g, s, nullptr, &key, &p) != SL_OK) return 0;
  return fused_workspace_bytes(key, p);
}

int sl_colour_pass(const sl_grid *g, const sl_stencil *s, int32_t colour, int32_t *d_status,
                   void *stream) {
  StreamDevice guard(stream);
  KernelKey key;
  Params p;
  int rc = make_params(g, s, d_status, &key, &p);
  if (rc != SL_OK) return rc;
  if (!d_status || colour < 0 || colour >= p.colours) return SL_E_INVAL;
  if (empty_grid(p)) return SL_OK;
  return cuda_status(launch_colour_pass(key, p, colour, (cudaStream_t)stream));
}

int sl_sweep(const sl_grid *g, const sl_stencil *s, int32_t sweeps, uint32_t flags,
             double *workspace, size_t workspace_bytes, int32_t *d_status, void *stream) {
  StreamDevice guard(stream);
  KernelKey key;
  Params p;
  int rc = make_params(g, s, d_status, &key, &p);
  if (rc != SL_OK) return rc;
  if (!d_status || sweeps < 0) return SL_E_INVAL;
  if (sweeps == 0 || empty_grid(p)) return SL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (flags & SL_FLAG_LEX) {
    // lexicographic order is global: slabs (non-zero origin) are not supported
    if (g->origin[0] || g->origin[1] || (g->dim == 3 && g->origin[2])) return SL_E_UNSUPPORTED;
    for (int i = 0; i < sweeps; ++i) {
      rc = cuda_status(launch_lex_sweep(key, p, st));
      if (rc != SL_OK) return rc;
    }
    return SL_OK;
  }
  if (flags & SL_FLAG_MERGE_COLOURS) {
    for (int i = 0; i < sweeps; ++i) {
      rc = cuda_status(launch_colour_pass(key, p, -1, st));
      if (rc != SL_OK) return rc;
    }
    return SL_OK;
  }
  if (!(flags & SL_FLAG_PER_COLOUR)) {
    int handled = 0;
    rc = cuda_status(launch_fused(key, p, sweeps, workspace, workspace_bytes, st, &handled,
                                  (flags & SL_FLAG_STREAM) != 0));
    if (rc != SL_OK || handled) return rc;
  }
  for (int i = 0; i < sweeps; ++i)
    for (int c = 0; c < p.colours; ++c) {
      rc = cuda_status(launch_colour_pass(key, p, c, st));
      if (rc != SL_OK) return rc;
    }
  return SL_OK;
}

static int sweep_pass_impl(const sl_grid *g, const sl_stencil *s, const double *src, double *dst,
                           int64_t zbegin, int64_t zend, double *pdn, int64_t dn_last, double *pup,
                           int64_t up_first, int32_t *d_status, void *stream) {
  StreamDevice guard(stream);
  if (!g || !src || !dst || src == dst) return SL_E_INVAL;
  sl_grid gs = *g;
  gs.u = const_cast<double *>(src);
  KernelKey key;
  Params p;
  int rc = make_params(&gs, s, d_status, &key, &p);
  if (rc != SL_OK) return rc;
  if (!d_status || zbegin < 0 || zend < zbegin || zend > p.zhi) return SL_E_INVAL;
  if (empty_grid(p)) return SL_OK;
  p.zlo = (int32_t)zbegin;
  p.zhi = (int32_t)zend;
  if ((pdn && ((uintptr_t)pdn & 15)) || (pup && ((uintptr_t)pup & 15))) return SL_E_INVAL;
  p.pdn = pdn;
  p.pup = pup;
  p.dn_last = (int32_t)(dn_last < -1 ? -1 : (dn_last > p.zhi ? p.zhi : dn_last));
  p.up_first = (int32_t)(up_first < 0 ? 0 : (up_first > (int64_t)1 << 30 ? (int64_t)1 << 30 : up_first));
  int handled = 0;
  rc = cuda_status(launch_one_pass(key, p, src, dst, (cudaStream_t)stream, &handled));
  if (rc != SL_OK) return rc;
  return handled ? SL_OK : SL_E_UNSUPPORTED;
}

int sl_sweep_pass(const sl_grid *g, const sl_stencil *s, const double *src, double *dst, int64_t zbegin,
                  int64_t zend, int32_t *d_status, void *stream) {
  return sweep_pass_impl(g, s, src, dst, zbegin, zend, nullptr, -1, nullptr, 0, d_status, stream);
}

int sl_sweep_pass_peer(const sl_grid *g, const sl_stencil *s, const double *src, double *dst,
                       int64_t zbegin, int64_t zend, double *peer_dn, int64_t dn_last, double *peer_up,
                       int64_t up_first, int32_t *d_status, void *stream) {
  return sweep_pass_impl(g, s, src, dst, zbegin, zend, peer_dn, dn_last, peer_up, up_first, d_status,
                         stream);
}

int sl_update_cells(const sl_grid *g, const sl_stencil *s, const int64_t *d_flats, int64_t count,
                    int32_t *d_status, void *stream) {
  StreamDevice guard(stream);
  KernelKey key;
  Params p;
  int rc = make_params(g, s, d_status, &key, &p);
  if (rc != SL_OK) return rc;
  if (!d_status || count < 0 || (count > 0 && !d_flats)) return SL_E_INVAL;
  return cuda_status(launch_update_cells(key, p, d_flats, count, (cudaStream_t)stream));
}

int sl_sweep_cost(const sl_grid *g, const sl_stencil *s, const sl_cost *cost, int32_t sweeps,
                  uint32_t flags, int32_t *d_status, void *stream) {
  StreamDevice guard(stream);
  KernelKey key;
  Params p;
  int rc = make_params(g, s, d_status, &key, &p);
  if (rc != SL_OK) return rc;
  if (!d_status || !cost || sweeps < 0 || (flags & ~SL_FLAG_LEX)) return SL_E_INVAL;
  if (cost->mode != SL_COST_CONST && cost->mode != SL_COST_RAMP) return SL_E_INVAL;
  if (cost->mode == SL_COST_CONST && cost->k < 0) return SL_E_INVAL;
  const bool origin = g->origin[0] || g->origin[1] || (g->dim == 3 && g->origin[2]);
  if (origin && (cost->mode == SL_COST_RAMP || (flags & SL_FLAG_LEX))) return SL_E_UNSUPPORTED;
  if (sweeps == 0 || empty_grid(p)) return SL_OK;
  CostSpec cs{cost->mode == SL_COST_RAMP, cost->k, cost->d_work};
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < sweeps; ++i) {
    if (flags & SL_FLAG_LEX) {
      rc = cuda_status(launch_cost_sweep_phase(key, p, cs, -1, st));
      if (rc != SL_OK) return rc;
      continue;
    }
    for (int c = 0; c < p.colours; ++c) {
      rc = cuda_status(launch_cost_sweep_phase(key, p, cs, c, st));
      if (rc != SL_OK) return rc;
    }
  }
  return SL_OK;
}

int sl_update_cells_cost(const sl_grid *g, const sl_stencil *s, const int64_t *d_flats,
                         int64_t count, const sl_cost *cost, int32_t *d_status, void *stream) {
  StreamDevice guard(stream);
  KernelKey key;
  Params p;
  int rc = make_params(g, s, d_status, &key, &p);
  if (rc != SL_OK) return rc;
  if (!d_status || !cost || count < 0 || (count > 0 && !d_flats)) return SL_E_INVAL;
  if (cost->mode != SL_COST_CONST || cost->k < 0) return SL_E_INVAL;
  CostSpec cs{0, cost->k, cost->d_work};
  return cuda_status(launch_cost_cells(key, p, cs, d_flats, count, (cudaStream_t)stream));
}

int sl_ghost_depth(const sl_stencil *s, int32_t dim, int32_t sweeps) {
  if (!s || (dim != 2 && dim != 3) || sweeps < 0) return -SL_E_INVAL;
  KernelKey key;
  Params p;
  std::memset(&p, 0, sizeof(p));
  if (resolve(s, dim, &key, &p) != SL_OK) return -SL_E_INVAL;
  if (sweeps == 0) return 0;
  return load_margin(key.shape, s->colours, sweeps, dim - 1);
}

int sl_residual_max(const sl_grid *g, const sl_stencil *s, double *d_out, void *stream) {
  StreamDevice guard(stream);
  KernelKey key;
  Params p;
  int rc = make_params(g, s, nullptr, &key, &p);
  if (rc != SL_OK) return rc;
  if (!d_out) return SL_E_INVAL;
  return cuda_status(launch_residual(key, p, d_out, (cudaStream_t)stream));
}

}  // extern "C"
