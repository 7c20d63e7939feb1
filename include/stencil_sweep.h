/*
 * stencil_sweep.h — C ABI of the B200 colour-scheduled smoother sweep.
 *
 * Drop-in boundary for the hot path of the reference `stencil_lab`
 * (/root/reference/pkg/src/stencil_lab).  The reference boundary is
 * Python-level (it has no FFI); each entry point below replaces
 * one reference function, cited next to it.  The Python mirror of the
 * reference API (paper_1810_04033_b200/) binds these through ctypes; the
 * binding a maintainer would add to the reference itself is in INTEGRATION.md.
 *
 * Conventions
 *  - All pointers in sl_grid are DEVICE pointers owned by the caller; the
 *    library never allocates on a call path.  `stream` is a cudaStream_t
 *    passed as void* (NULL = legacy default stream); every call is
 *    stream-ordered and asynchronous.
 *  - Non-finite updates (reference NumericsError, kernels.py:38-39,
 *    :247-249) are reported by OR-ing SL_E_NONFINITE into *d_status
 *    (device int32, caller zeroes it); the caller reads it back after the
 *    stream has drained.  Grid contents after such an error are unspecified.
 *    Bit 1 (value 2) of *d_status is set when the on-chip 2D sweep (one
 *    cooperative launch for all sweeps, red-black grids that fit the chip)
 *    gave up waiting for a neighbouring tile's exchange flag (a bounded
 *    spin, so a broken co-residency assumption cannot hang the device); the
 *    grid contents are then invalid too.
 *  - Return value: SL_OK, SL_E_INVAL (bad argument; reference ValueError),
 *    SL_E_UNSUPPORTED (stencil shape/weight pattern without a kernel) or
 *    SL_E_CUDA (launch error; see sl_last_cuda_error()).
 */
#ifndef STENCIL_SWEEP_H
#define STENCIL_SWEEP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SL_ABI_VERSION 1

#if defined(__GNUC__)
#define SL_API __attribute__((visibility("default")))
#else
#define SL_API
#endif

enum sl_status {
    SL_OK = 0,
    SL_E_NONFINITE = 1,
    SL_E_INVAL = 2,
    SL_E_CUDA = 3,
    SL_E_UNSUPPORTED = 4
};

/* Neighbour set, offsets in canonical order (ascending flat delta,
 * kernels.py:78-80).  FE27 with all six face weights zero is the trilinear
 * Q1 operator of BASELINE config 4 and gets its own 20-neighbour kernel. */
enum sl_shape { SL_FD5 = 0, SL_FE9 = 1, SL_FD7 = 2, SL_FE27 = 3 };

/* Update form.  R: u_c = (sum_j |w_j| u_j) / w_c, the reference arithmetic
 * (kernels.py:224-232).  D: u_c += omega * ((f_c - A u)/w_c) with
 * A u = w_c u_c + sum_j w_j u_j (BASELINE.json configs). */
enum sl_form { SL_FORM_R = 0, SL_FORM_D = 1 };

/* sl_sweep flags */
#define SL_FLAG_PER_COLOUR 0x1u   /* one in-place launch per colour phase (K1), no fusion */
#define SL_FLAG_MERGE_COLOURS 0x2u /* negative control: all colours in ONE racy pass
                                      (reference _fault_merge_colours, strategies.py:364-369) */
#define SL_FLAG_STREAM 0x4u        /* fused path: always the streaming kernels (no small-grid
                                      tile kernel, no on-chip patch kernel) — for testing */
#define SL_FLAG_LEX 0x8u           /* lexicographic Gauss-Seidel order instead of colours: the
                                      reference serial / taskgraph sweeps (strategies.py:341-345,
                                      :477-487), run as hyperplane wavefronts */

typedef struct sl_grid {
    int32_t dim;              /* 2 or 3 */
    int32_t reserved0;
    int64_t n[3];             /* interior extent along x, y, z (n[2] ignored for dim 2) */
    int64_t batch;            /* independent grids back to back (patches); >= 1 */
    int64_t batch_stride;     /* elements between grid b and b+1 (>= (n+2) product) */
    int64_t origin[3];        /* global coordinate offset of this grid (colour parity of
                                 slabs); 0 for a whole mesh */
    double *u;                /* dense (n[0]+2)(n[1]+2)[(n[2]+2)] fp64, x fastest (mesh.py:20-51) */
    const double *f;          /* same layout, read only; required for SL_FORM_D, else ignored */
} sl_grid;

typedef struct sl_stencil {
    int32_t shape;            /* enum sl_shape */
    int32_t colours;          /* 2 (red-black) or 2^dim (per-axis parity) */
    int32_t form;             /* enum sl_form */
    int32_t reserved0;
    double w[26];             /* signed weight per canonical offset of `shape` (0 = skipped) */
    double wc;                /* centre weight */
    double omega;             /* damping, SL_FORM_D only */
} sl_stencil;

SL_API int sl_abi_version(void);
SL_API const char *sl_strerror(int code);
SL_API int sl_last_cuda_error(void);
/* Process-wide count of kernels this library has launched (bench evidence). */
SL_API uint64_t sl_launch_count(void);

/* Bytes of device scratch sl_sweep uses to fuse colour phases and sweeps into
 * one HBM pass (0 = fusion not available for this grid; sl_sweep then runs
 * per-colour in place). */
SL_API size_t sl_workspace_bytes(const sl_grid *g, const sl_stencil *s);

/* `sweeps` full colour-ordered sweeps, in place.  Replaces
 * strategies.sweep_colouring (strategies.py:348-393; one sweep) and
 * bench.StrategyRunner.run_sweeps (bench.py:186-188; many).  The result is
 * bitwise identical for every flag/workspace choice (except MERGE_COLOURS). */
SL_API int sl_sweep(const sl_grid *g, const sl_stencil *s, int32_t sweeps, uint32_t flags,
             double *workspace, size_t workspace_bytes, int32_t *d_status, void *stream);

/* One fused sweep from `src` to `dst` (two distinct buffers of g's layout;
 * g->u is ignored) that writes only the planes [zbegin, zend) of the slowest
 * axis (z in 3D, y in 2D) of dst and reads src around them.  The multi-GPU
 * slab runner computes its boundary planes first and exchanges them while the
 * interior pass runs (there is no reference counterpart: the reference is
 * single-process).  SL_E_UNSUPPORTED when no streaming kernel covers the
 * stencil/grid (odd row length, batch > 1, odd x origin). */
SL_API int sl_sweep_pass(const sl_grid *g, const sl_stencil *s, const double *src, double *dst,
                         int64_t zbegin, int64_t zend, int32_t *d_status, void *stream);

/* sl_sweep_pass that also stores every owned value of slow-axis plane
 * q <= dn_last at peer_dn + e and of plane q >= up_first at peer_up + e, where
 * e is the value's element index in g's layout.  The slab runner passes the
 * neighbouring ranks' slab buffers (peer memory over NVLink), offset so that
 * e lands in their ghost planes: the halo exchange is fused into the pass and
 * overlaps it store by store.  NULL peers = sl_sweep_pass.  16-byte aligned. */
SL_API int sl_sweep_pass_peer(const sl_grid *g, const sl_stencil *s, const double *src, double *dst,
                              int64_t zbegin, int64_t zend, double *peer_dn, int64_t dn_last,
                              double *peer_up, int64_t up_first, int32_t *d_status, void *stream);

/* One colour phase in place: one parallel_for pass of sweep_colouring
 * (strategies.py:374-393) / one colour of sweep_colouring_reference (:420-433). */
SL_API int sl_colour_pass(const sl_grid *g, const sl_stencil *s, int32_t colour,
                   int32_t *d_status, void *stream);

/* In-place update of `count` mutually non-adjacent cells of grid 0 given as
 * device int64 flat indices — kernels.update_cells_batch (kernels.py:212-251).
 * Like the reference, a batch with a non-finite result is not written at all:
 * *d_status must be 0 on entry; it becomes non-zero and the grid is unchanged. */
SL_API int sl_update_cells(const sl_grid *g, const sl_stencil *s, const int64_t *d_flats,
                    int64_t count, int32_t *d_status, void *stream);

/* Cost model (reference kernels.py:113-145): k sine evaluations per stencil
 * entry and centre, folded into the weights as 0.0*d so the values stay
 * bit-identical to k = 0; the consumed sine sum is added to *d_work. */
#define SL_COST_CONST 0
#define SL_COST_RAMP 1 /* k = min(100*rank/total, 99), rank = lex rank of the cell in its grid */
typedef struct sl_cost {
    int32_t mode;   /* SL_COST_CONST / SL_COST_RAMP */
    int32_t k;      /* SL_COST_CONST: k >= 0 */
    double *d_work; /* device double accumulator for the sine tally, or NULL */
} sl_cost;

/* `sweeps` sweeps with the cost model: colour order by default, lexicographic
 * with SL_FLAG_LEX (the only flag honoured).  One launch per colour phase /
 * hyperplane; replaces the k > 0 paths of strategies.py:341-393.  Ramp cost
 * needs origin 0 (the rank is lexicographic over the whole grid). */
SL_API int sl_sweep_cost(const sl_grid *g, const sl_stencil *s, const sl_cost *cost,
                         int32_t sweeps, uint32_t flags, int32_t *d_status, void *stream);

/* update_cells_batch with k > 0 (kernels.py:234-244); mode must be CONST. */
SL_API int sl_update_cells_cost(const sl_grid *g, const sl_stencil *s, const int64_t *d_flats,
                                int64_t count, const sl_cost *cost, int32_t *d_status,
                                void *stream);

/* Ghost depth along the slowest axis (z in 3D, y in 2D) needed to run
 * `sweeps` colour-ordered sweeps on a slab without exchanging: the input must
 * be valid this many planes beyond the slab for its own planes to come out
 * exact (the dependency DP of the fused schedule).  < 0 on bad arguments. */
SL_API int sl_ghost_depth(const sl_stencil *s, int32_t dim, int32_t sweeps);

/* max over interior cells of |A u| (Form R) or |f - A u| (Form D), written to
 * *d_out (device double) — kernels.residual_max (kernels.py:254-265).  With
 * batch > 1 the max runs over all grids. */
SL_API int sl_residual_max(const sl_grid *g, const sl_stencil *s, double *d_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* STENCIL_SWEEP_H */
