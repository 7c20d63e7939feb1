/*
 * Plain-C restatement of the reference colour sweep — TEST INFRASTRUCTURE.
 *
 * Used only by tests/ (large-size checker), __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs (the "port" CPU baseline).
 * Never linked into the product library.
 *
 * Follows (paths under /root/reference/pkg/src/stencil_lab):
 *   layout, flat index ............ mesh.py:20-51  (x fastest, halo width 1)
 *   canonical offset order ........ kernels.py:78-80 (caller passes offsets sorted)
 *   colour id / pass order ........ strategies.py:62-69, :201-214, :371-393
 *   Form R arithmetic ............. kernels.py:224-232 (acc=+0.0; acc+=|w|*u_j; /w_c)
 *   non-finite check .............. kernels.py:247-249 (returns 1 instead of raising)
 * Form D (damped, with rhs f) is the repo's own definition (oracle/restate.py
 * docstring):  Au = w_c*u_c; Au = Au + w_j*u_j ...; u_c = u_c + omega*((f_c-Au)/w_c).
 *
 * Must be compiled with -ffp-contract=off and without -ffast-math: every
 * operation is a separately rounded binary64 op, like NumPy's ufuncs.
 * Within one colour all cells are mutually non-adjacent, so the rows of a
 * colour may be split across pthreads without changing any bit (the image has
 * no libgomp, so the row split is done by hand).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <unistd.h>

#define MAXNB 26

int oracle_max_threads(void);

typedef struct {
    int dim, nnz, colours, form, colour;
    int64_t n, batch, bstride, r0, r1;
    double *u;
    const double *f;
    const int64_t *delta;
    const double *w, *aw;
    double wc, omega;
    int bad;
} pass_args;

/* one cell update in place; returns 1 when the new value is non-finite */
static inline int update_point(double *ub, const double *fb, int64_t c, int form, int nnz,
                               const int64_t *delta, const double *w, const double *aw,
                               double wc, double omega)
{
    double out;
    if (form == 0) {
        double acc = 0.0;
        for (int j = 0; j < nnz; ++j) {
            double t = aw[j] * ub[c + delta[j]];
            acc = acc + t;
        }
        out = acc / wc;
    } else {
        const double uc = ub[c];
        double au = wc * uc;
        for (int j = 0; j < nnz; ++j) {
            double t = w[j] * ub[c + delta[j]];
            au = au + t;
        }
        double q = (fb[c] - au) / wc;
        double t = omega * q;
        out = uc + t;
    }
    ub[c] = out;
    return !isfinite(out);
}

/* Lexicographic Gauss-Seidel sweep (reference strategies.py:341-345 serial,
 * cells in increasing flat index, strategies.py:226-234 / mesh.py:79-88). */
static int lex_sweep(int dim, int64_t n, int64_t batch, int64_t bstride, double *u,
                     const double *f, int nnz, const int64_t *delta, const double *w,
                     const double *aw, double wc, int form, double omega)
{
    const int64_t S = n + 2;
    int bad = 0;
    for (int64_t b = 0; b < batch; ++b) {
        double *ub = u + b * bstride;
        const double *fb = f ? f + b * bstride : 0;
        for (int64_t z = (dim == 3 ? 1 : 0); z < (dim == 3 ? n + 1 : 1); ++z)
            for (int64_t y = 1; y <= n; ++y)
                for (int64_t x = 1; x <= n; ++x)
                    bad |= update_point(ub, fb, (z * S + y) * S + x, form, nnz, delta, w, aw,
                                        wc, omega);
    }
    return bad;
}

static void *pass_rows(void *vp)
{
    pass_args *a = (pass_args *)vp;
    const int dim = a->dim, nnz = a->nnz, colour = a->colour;
    const int64_t n = a->n, S = n + 2;
    const int64_t nz = (dim == 3) ? n : 1;
    int bad = 0;
    for (int64_t r = a->r0; r < a->r1; ++r) {
        const int64_t b = r / (nz * n);
        const int64_t rem = r % (nz * n);
        const int64_t z = (dim == 3) ? rem / n + 1 : 0;
        const int64_t y = rem % n + 1;
        const int64_t qy = (y - 1) & 1, qz = (dim == 3) ? ((z - 1) & 1) : 0;
        int64_t qx;
        if (a->colours == 2) {
            qx = ((colour - qy - qz) % 2 + 2) % 2;
        } else {
            if (qy != ((colour >> 1) & 1)) continue;
            if (dim == 3 && qz != ((colour >> 2) & 1)) continue;
            qx = colour & 1;
        }
        double *ub = a->u + b * a->bstride;
        const double *fb = a->f ? a->f + b * a->bstride : 0;
        const int64_t rowbase = (dim == 3) ? (z * S + y) * S : y * S;
        for (int64_t x = 1 + qx; x <= n; x += 2)
            bad |= update_point(ub, fb, rowbase + x, a->form, nnz, a->delta, a->w, a->aw,
                                a->wc, a->omega);
    }
    a->bad = bad;
    return 0;
}

#define MAXT 256

static int colour_pass(int dim, int64_t n, int64_t batch, int64_t bstride,
                       double *u, const double *f, int nnz, const int64_t *delta,
                       const double *w, const double *aw, double wc, int colours,
                       int form, double omega, int colour, int threads)
{
    const int64_t nz = (dim == 3) ? n : 1;
    const int64_t rows = batch * nz * n; /* (b, z, y) rows */
    if (threads > rows) threads = (int)rows;
    if (threads < 1) threads = 1;
    pass_args args[MAXT];
    pthread_t tid[MAXT];
    for (int t = 0; t < threads; ++t) {
        pass_args *a = &args[t];
        a->dim = dim; a->nnz = nnz; a->colours = colours; a->form = form; a->colour = colour;
        a->n = n; a->batch = batch; a->bstride = bstride;
        a->r0 = rows * t / threads; a->r1 = rows * (t + 1) / threads;
        a->u = u; a->f = f; a->delta = delta; a->w = w; a->aw = aw;
        a->wc = wc; a->omega = omega; a->bad = 0;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], 0, pass_rows, &args[t]);
    pass_rows(&args[0]);
    int bad = args[0].bad;
    for (int t = 1; t < threads; ++t) {
        pthread_join(tid[t], 0);
        bad |= args[t].bad;
    }
    return bad;
}

/*
 * sweeps full colour-ordered sweeps in place.
 * off: nnz x 3 int32 displacements (x, y, z), canonical order, zero weights
 * already removed by the caller.  batch grids of (n+2)^dim, bstride apart.
 * form 0 = R (f ignored), 1 = D.  threads <= 0: all online cores.
 * colours 0: lexicographic (serial) sweeps instead of colour passes.
 * Returns 0 ok, 1 non-finite update seen, 2 bad arguments.
 */
int oracle_sweep(int dim, int64_t n, int64_t batch, int64_t bstride,
                 double *u, const double *f, int nnz, const int32_t *off,
                 const double *w, double wc, int colours, int form,
                 double omega, int sweeps, int threads)
{
    if ((dim != 2 && dim != 3) || n < 1 || nnz < 0 || nnz > MAXNB) return 2;
    if (colours != 0 && colours != 2 && colours != (1 << dim)) return 2;
    if (form == 1 && !f) return 2;
    if (threads <= 0) threads = oracle_max_threads();
    if (threads > MAXT) threads = MAXT;
    const int64_t S = n + 2;
    int64_t delta[MAXNB];
    for (int j = 0; j < nnz; ++j)
        delta[j] = off[3 * j] + off[3 * j + 1] * S + (dim == 3 ? off[3 * j + 2] * S * S : 0);
    double aw[MAXNB];
    for (int j = 0; j < nnz; ++j) aw[j] = fabs(w[j]);
    int bad = 0;
    if (colours == 0) {
        for (int s = 0; s < sweeps; ++s)
            bad |= lex_sweep(dim, n, batch, bstride, u, f, nnz, delta, w, aw, wc, form, omega);
        return bad;
    }
    for (int s = 0; s < sweeps; ++s)
        for (int c = 0; c < colours; ++c)
            bad |= colour_pass(dim, n, batch, bstride, u, f, nnz, delta, w, aw, wc,
                               colours, form, omega, c, threads);
    return bad;
}

int oracle_max_threads(void)
{
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c < 1 ? 1 : (int)c;
}
