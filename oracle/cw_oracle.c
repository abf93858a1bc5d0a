/*
 * cw_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A float64 CPU restatement of the reference `clutterwhiten` per-pixel
 * pipeline (arXiv 1408.3526 package, /root/reference/pkg/src/clutterwhiten).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.
 *
 * Every stage follows the reference loop structure and accumulation order
 * so that, fed the same numpy-built phase tables, the arithmetic is the
 * same IEEE-754 double sequence as the reference's numba kernels
 * (compile with -ffp-contract=off; no -ffast-math).  Row (or column)
 * blocks are distributed over OpenMP threads exactly like the reference's
 * BlockExecutor fork-join (parallel.py:62-73): every output index has one
 * writer, so results do not depend on the thread count.
 *
 * Layouts (C-contiguous, complex = interleaved re,im doubles), as in
 * _kernels.py:1-26:
 *   frame  (H,W) f32          xf   (H,W,Mx) c128
 *   ring   (Mz,H,W,My,Mx) c128 bins (H,W,Mz,My,Mx) c128
 *   pw     (H,W,Mz*My*Mx) f64  r/rhat (H,W,Ly,Lx) f64
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double re, im;
} cplx;

static inline cplx cmul(cplx a, cplx b)
{
    cplx r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}

static inline cplx cadd(cplx a, cplx b)
{
    cplx r = {a.re + b.re, a.im + b.im};
    return r;
}

static inline cplx csub(cplx a, cplx b)
{
    cplx r = {a.re - b.re, a.im - b.im};
    return r;
}

/* complex * real, as numba promotes the real operand to (x + 0j). */
static inline cplx cmulr(cplx a, double x)
{
    cplx r;
    r.re = a.re * x - a.im * 0.0;
    r.im = a.re * 0.0 + a.im * x;
    return r;
}

typedef struct cwo_pipe {
    int kx, ky, kz, bx, by, mhx, mhy, mhz;
    int mx, my, mz, nb, nc, lx, ly;
    int W, H;
    double alpha;
    int nthreads;
    /* tables (numpy-built by the caller, spectrum.py:65-74, flow.py:87-97,147-163) */
    cplx *ex, *ey, *ez; /* (M,M) e[ik,m] = exp(+j2pi k m / M) */
    cplx *twx, *twy;    /* e[:,1] */
    cplx *az, *axl, *ayl;
    double *lag_x, *lag_y, *gx, *gy;
    double norm;
    /* bank (Ly,Lx,NC) complex64 promoted at use, retained (NC,) */
    float *bank;
    int64_t *retained;
    /* stream state */
    cplx *xf, *ring, *sbins, *cond;
    double *pw, *r, *rhat;
    int have_rhat;
    int32_t *idx;
    double *vel;
    float *pred, *res, *imag;
    float *delay; /* (mhz+1, H, W) ring of raw frames */
    long long frames_seen;
} cwo_pipe;

/* ---- kernels ------------------------------------------------------------ */

/* _kernels.py:31-45 (sdft_rows): direct sum at x = Mx-1, then comb + resonator. */
static void k_sdft_rows(const cwo_pipe *p, const float *frame, int lo, int hi)
{
    const int W = p->W, Mx = p->mx;
    for (int y = lo; y < hi; y++) {
        cplx *row = p->xf + (size_t)y * W * Mx;
        for (int ik = 0; ik < Mx; ik++) {
            cplx acc = {0.0, 0.0};
            for (int m = 0; m < Mx; m++)
                acc = cadd(acc, cmulr(p->ex[ik * Mx + m], (double)frame[(size_t)y * W + (Mx - 1 - m)]));
            row[(size_t)(Mx - 1) * Mx + ik] = acc;
        }
        for (int x = Mx; x < W; x++) {
            double comb = (double)frame[(size_t)y * W + x] - (double)frame[(size_t)y * W + x - Mx];
            for (int ik = 0; ik < Mx; ik++) {
                cplx t = cmul(p->twx[ik], row[(size_t)(x - 1) * Mx + ik]);
                cplx c = {comb, 0.0};
                row[(size_t)x * Mx + ik] = cadd(t, c);
            }
        }
    }
}

/* _kernels.py:48-68 (sdft_cols): y-slide of the x-stage into one ring slot. */
static void k_sdft_cols(const cwo_pipe *p, cplx *sp, int lo, int hi)
{
    const int W = p->W, H = p->H, Mx = p->mx, My = p->my;
    const int x_min = Mx - 1;
    for (int x = lo; x < hi; x++) {
        if (x < x_min)
            continue;
        for (int iy = 0; iy < My; iy++)
            for (int ix = 0; ix < Mx; ix++) {
                cplx acc = {0.0, 0.0};
                for (int m = 0; m < My; m++)
                    acc = cadd(acc, cmul(p->ey[iy * My + m], p->xf[((size_t)(My - 1 - m) * W + x) * Mx + ix]));
                sp[(((size_t)(My - 1) * W + x) * My + iy) * Mx + ix] = acc;
            }
        for (int y = My; y < H; y++)
            for (int iy = 0; iy < My; iy++) {
                cplx t = p->twy[iy];
                for (int ix = 0; ix < Mx; ix++) {
                    cplx comb = csub(p->xf[((size_t)y * W + x) * Mx + ix], p->xf[((size_t)(y - My) * W + x) * Mx + ix]);
                    cplx prev = sp[(((size_t)(y - 1) * W + x) * My + iy) * Mx + ix];
                    sp[(((size_t)y * W + x) * My + iy) * Mx + ix] = cadd(cmul(t, prev), comb);
                }
            }
    }
}

/* _kernels.py:71-90 (temporal_dft): exact ring-buffer DFT over Mz slots. */
static void k_temporal_dft(const cwo_pipe *p, const int64_t *slots, int lo, int hi)
{
    const int W = p->W, Mx = p->mx, My = p->my, Mz = p->mz, H = p->H;
    const int x_min = Mx - 1, y_min = My - 1;
    const size_t slot_stride = (size_t)H * W * My * Mx;
    cplx taps[64];
    for (int y = lo; y < hi; y++) {
        if (y < y_min)
            continue;
        for (int x = x_min; x < W; x++)
            for (int iy = 0; iy < My; iy++)
                for (int ix = 0; ix < Mx; ix++) {
                    size_t off = (((size_t)y * W + x) * My + iy) * Mx + ix;
                    for (int m = 0; m < Mz; m++)
                        taps[m] = p->ring[(size_t)slots[m] * slot_stride + off];
                    for (int iz = 0; iz < Mz; iz++) {
                        cplx acc = {0.0, 0.0};
                        for (int m = 0; m < Mz; m++)
                            acc = cadd(acc, cmul(p->ez[iz * Mz + m], taps[m]));
                        /* numba: norm (float) * acc (complex) -> complex(norm,0)*acc */
                        cplx o;
                        o.re = p->norm * acc.re - 0.0 * acc.im;
                        o.im = p->norm * acc.im + 0.0 * acc.re;
                        p->sbins[((((size_t)y * W + x) * Mz + iz) * My + iy) * Mx + ix] = o;
                    }
                }
    }
}

/* _kernels.py:156-174: copy_field then zero_spatial_dc. */
static void k_copy_zero_dc(const cwo_pipe *p, int lo, int hi)
{
    const size_t per = (size_t)p->nb;
    for (int y = lo; y < hi; y++) {
        size_t base = (size_t)y * p->W * per;
        memcpy(p->cond + base, p->sbins + base, sizeof(cplx) * p->W * per);
        for (int x = 0; x < p->W; x++)
            for (int iz = 0; iz < p->mz; iz++) {
                cplx *c = p->cond + base + (size_t)x * per + ((size_t)iz * p->my + p->ky) * p->mx + p->kx;
                c->re = 0.0;
                c->im = 0.0;
            }
    }
}

/* _kernels.py:177-217 (hann3): circular (-1/4, 1/2, -1/4) along kx, ky, kz. */
static void k_hann3(const cwo_pipe *p, int lo, int hi)
{
    const int Mx = p->mx, My = p->my, Mz = p->mz, nb = p->nb;
    cplx *b1 = (cplx *)malloc(sizeof(cplx) * nb);
    cplx *b2 = (cplx *)malloc(sizeof(cplx) * nb);
#define I3(z, y, x) (((z) * My + (y)) * Mx + (x))
    for (int y = lo; y < hi; y++)
        for (int x = 0; x < p->W; x++) {
            cplx *s = p->cond + ((size_t)y * p->W + x) * nb;
            memcpy(b1, s, sizeof(cplx) * nb);
            for (int iz = 0; iz < Mz; iz++)
                for (int iy = 0; iy < My; iy++)
                    for (int ix = 0; ix < Mx; ix++) {
                        int l = ix > 0 ? ix - 1 : Mx - 1, h = ix < Mx - 1 ? ix + 1 : 0;
                        cplx a = b1[I3(iz, iy, l)], b = b1[I3(iz, iy, h)], c = b1[I3(iz, iy, ix)];
                        b2[I3(iz, iy, ix)].re = 0.5 * c.re - 0.25 * (a.re + b.re);
                        b2[I3(iz, iy, ix)].im = 0.5 * c.im - 0.25 * (a.im + b.im);
                    }
            for (int iz = 0; iz < Mz; iz++)
                for (int iy = 0; iy < My; iy++) {
                    int l = iy > 0 ? iy - 1 : My - 1, h = iy < My - 1 ? iy + 1 : 0;
                    for (int ix = 0; ix < Mx; ix++) {
                        cplx a = b2[I3(iz, l, ix)], b = b2[I3(iz, h, ix)], c = b2[I3(iz, iy, ix)];
                        b1[I3(iz, iy, ix)].re = 0.5 * c.re - 0.25 * (a.re + b.re);
                        b1[I3(iz, iy, ix)].im = 0.5 * c.im - 0.25 * (a.im + b.im);
                    }
                }
            for (int iz = 0; iz < Mz; iz++) {
                int l = iz > 0 ? iz - 1 : Mz - 1, h = iz < Mz - 1 ? iz + 1 : 0;
                for (int iy = 0; iy < My; iy++)
                    for (int ix = 0; ix < Mx; ix++) {
                        cplx a = b1[I3(l, iy, ix)], b = b1[I3(h, iy, ix)], c = b1[I3(iz, iy, ix)];
                        s[I3(iz, iy, ix)].re = 0.5 * c.re - 0.25 * (a.re + b.re);
                        s[I3(iz, iy, ix)].im = 0.5 * c.im - 0.25 * (a.im + b.im);
                    }
            }
        }
#undef I3
    free(b1);
    free(b2);
}

/* _kernels.py:220-227 (power). */
static void k_power(const cwo_pipe *p, int lo, int hi)
{
    for (int y = lo; y < hi; y++)
        for (size_t i = (size_t)y * p->W * p->nb; i < (size_t)(y + 1) * p->W * p->nb; i++) {
            cplx v = p->cond[i];
            p->pw[i] = v.re * v.re + v.im * v.im;
        }
}

/* _kernels.py:230-258 (autocorr): kz collapse -> per-lx -> per-ly. */
static void k_autocorr(const cwo_pipe *p, int lo, int hi)
{
    const int Mx = p->mx, My = p->my, Mz = p->mz, Lx = p->lx, Ly = p->ly;
    cplx tz[32 * 32], by[32];
    for (int y = lo; y < hi; y++)
        for (int x = 0; x < p->W; x++) {
            const double *pp = p->pw + ((size_t)y * p->W + x) * p->nb;
            double *out = p->r + ((size_t)y * p->W + x) * Ly * Lx;
            for (int iy = 0; iy < My; iy++)
                for (int ix = 0; ix < Mx; ix++) {
                    cplx acc = {0.0, 0.0};
                    for (int iz = 0; iz < Mz; iz++)
                        acc = cadd(acc, cmulr(p->az[iz], pp[(iz * My + iy) * Mx + ix]));
                    tz[iy * Mx + ix] = acc;
                }
            for (int il = 0; il < Lx; il++) {
                for (int iy = 0; iy < My; iy++) {
                    cplx acc = {0.0, 0.0};
                    for (int ix = 0; ix < Mx; ix++)
                        acc = cadd(acc, cmul(p->axl[il * Mx + ix], tz[iy * Mx + ix]));
                    by[iy] = acc;
                }
                for (int jl = 0; jl < Ly; jl++) {
                    cplx acc = {0.0, 0.0};
                    for (int iy = 0; iy < My; iy++)
                        acc = cadd(acc, cmul(p->ayl[jl * My + iy], by[iy]));
                    out[jl * Lx + il] = acc.re;
                }
            }
        }
}

/* _kernels.py:261-271 (smooth). */
static void k_smooth(const cwo_pipe *p, int lo, int hi)
{
    const double beta = 1.0 - p->alpha;
    const size_t per = (size_t)p->lx * p->ly;
    for (size_t i = (size_t)lo * p->W * per; i < (size_t)hi * p->W * per; i++)
        p->rhat[i] = beta * p->r[i] + p->alpha * p->rhat[i];
}

/* _kernels.py:274-302 (pick): envelope-compensated argmax, total-order ties. */
static void k_pick(const cwo_pipe *p, int lo, int hi)
{
    const int Lx = p->lx, Ly = p->ly;
    for (int y = lo; y < hi; y++)
        for (int x = 0; x < p->W; x++) {
            const double *rh = p->rhat + ((size_t)y * p->W + x) * Ly * Lx;
            double best = rh[0] * p->gy[0] * p->gx[0];
            int bix = 0, biy = 0;
            double bnorm = p->lag_x[0] * p->lag_x[0] + p->lag_y[0] * p->lag_y[0];
            for (int jy = 0; jy < Ly; jy++)
                for (int jx = 0; jx < Lx; jx++) {
                    double v = rh[jy * Lx + jx] * p->gy[jy] * p->gx[jx];
                    if (v < best)
                        continue;
                    double n2 = p->lag_x[jx] * p->lag_x[jx] + p->lag_y[jy] * p->lag_y[jy];
                    if (v > best || (n2 < bnorm || (n2 == bnorm && (jx < bix || (jx == bix && jy < biy))))) {
                        best = v;
                        bix = jx;
                        biy = jy;
                        bnorm = n2;
                    }
                }
            size_t o = ((size_t)y * p->W + x) * 2;
            p->idx[o] = bix;
            p->idx[o + 1] = biy;
            p->vel[o] = p->lag_x[bix];
            p->vel[o + 1] = p->lag_y[biy];
        }
}

/* _kernels.py:305-342 (pef): retained-bin inner product at the anchor. */
static void k_pef(const cwo_pipe *p, const float *delayed, int lo, int hi)
{
    const int ox_lo = p->mx - 1 - p->mhx, ox_hi = p->W - 1 - p->mhx;
    const int oy_lo = p->my - 1 - p->mhy, oy_hi = p->H - 1 - p->mhy;
    const int NC = p->nc;
    for (int oy = lo; oy < hi; oy++) {
        if (oy < oy_lo || oy > oy_hi)
            continue;
        for (int ox = ox_lo; ox <= ox_hi; ox++) {
            int ny = oy + p->mhy, nx = ox + p->mhx;
            size_t a = (size_t)ny * p->W + nx;
            int bix = p->idx[a * 2], biy = p->idx[a * 2 + 1];
            const float *bk = p->bank + (((size_t)biy * p->lx + bix) * NC) * 2;
            const cplx *s = p->sbins + a * p->nb;
            cplx acc = {0.0, 0.0};
            for (int j = 0; j < NC; j++) {
                cplx c = {(double)bk[2 * j], (double)bk[2 * j + 1]};
                acc = cadd(acc, cmul(c, s[p->retained[j]]));
            }
            double pr = acc.re;
            size_t o = (size_t)oy * p->W + ox;
            p->pred[o] = (float)pr;
            p->res[o] = (float)((double)delayed[o] - pr);
            p->imag[o] = (float)fabs(acc.im);
        }
    }
}

/* ---- fork-join over a partition axis (parallel.py:62-73) ----------------- */



#define FORK(p, n, CALL)                                                         \
    do {                                                                         \
        int _n = (n), _w = (p)->nthreads < 1 ? 1 : (p)->nthreads;                \
        int _step = (_n + _w - 1) / _w;                                          \
        _Pragma("omp parallel for schedule(static, 1) num_threads(_w)")          \
        for (int _b = 0; _b < _w; _b++) {                                        \
            int lo = _b * _step, hi = lo + _step < _n ? lo + _step : _n;         \
            if (lo < hi) {                                                       \
                CALL;                                                            \
            }                                                                    \
        }                                                                        \
    } while (0)

/* ---- public C ABI (ctypes, oracle/oracle.py) ---------------------------- */

static void *xcalloc(size_t n, size_t sz)
{
    void *q = calloc(n ? n : 1, sz);
    return q;
}

cwo_pipe *cwo_create(const int *geom, /* kx ky kz bx by mhx mhy mhz W H nthreads */
                     double alpha, int nlx, const double *lag_x, int nly, const double *lag_y,
                     const double *ex, const double *ey, const double *ez, const double *az,
                     const double *axl, const double *ayl, const double *gx, const double *gy,
                     const float *bank, const int64_t *retained, int nc)
{
    cwo_pipe *p = (cwo_pipe *)xcalloc(1, sizeof(cwo_pipe));
    if (!p)
        return NULL;
    p->kx = geom[0];
    p->ky = geom[1];
    p->kz = geom[2];
    p->bx = geom[3];
    p->by = geom[4];
    p->mhx = geom[5];
    p->mhy = geom[6];
    p->mhz = geom[7];
    p->W = geom[8];
    p->H = geom[9];
    p->nthreads = geom[10];
    p->mx = 2 * p->kx + 1;
    p->my = 2 * p->ky + 1;
    p->mz = 2 * p->kz + 1;
    p->nb = p->mx * p->my * p->mz;
    p->nc = nc;
    p->lx = nlx;
    p->ly = nly;
    p->alpha = alpha;
    p->norm = 1.0 / sqrt((double)p->nb);
    const int Mx = p->mx, My = p->my, Mz = p->mz;
    const size_t HW = (size_t)p->W * p->H;
    p->ex = (cplx *)xcalloc(Mx * Mx, sizeof(cplx));
    p->ey = (cplx *)xcalloc(My * My, sizeof(cplx));
    p->ez = (cplx *)xcalloc(Mz * Mz, sizeof(cplx));
    p->twx = (cplx *)xcalloc(Mx, sizeof(cplx));
    p->twy = (cplx *)xcalloc(My, sizeof(cplx));
    p->az = (cplx *)xcalloc(Mz, sizeof(cplx));
    p->axl = (cplx *)xcalloc((size_t)nlx * Mx, sizeof(cplx));
    p->ayl = (cplx *)xcalloc((size_t)nly * My, sizeof(cplx));
    memcpy(p->ex, ex, sizeof(cplx) * Mx * Mx);
    memcpy(p->ey, ey, sizeof(cplx) * My * My);
    memcpy(p->ez, ez, sizeof(cplx) * Mz * Mz);
    for (int i = 0; i < Mx; i++)
        p->twx[i] = p->ex[i * Mx + 1];
    for (int i = 0; i < My; i++)
        p->twy[i] = p->ey[i * My + 1];
    memcpy(p->az, az, sizeof(cplx) * Mz);
    memcpy(p->axl, axl, sizeof(cplx) * nlx * Mx);
    memcpy(p->ayl, ayl, sizeof(cplx) * nly * My);
    p->lag_x = (double *)xcalloc(nlx, sizeof(double));
    p->lag_y = (double *)xcalloc(nly, sizeof(double));
    p->gx = (double *)xcalloc(nlx, sizeof(double));
    p->gy = (double *)xcalloc(nly, sizeof(double));
    memcpy(p->lag_x, lag_x, sizeof(double) * nlx);
    memcpy(p->lag_y, lag_y, sizeof(double) * nly);
    memcpy(p->gx, gx, sizeof(double) * nlx);
    memcpy(p->gy, gy, sizeof(double) * nly);
    p->bank = (float *)xcalloc((size_t)nly * nlx * nc * 2, sizeof(float));
    memcpy(p->bank, bank, sizeof(float) * nly * nlx * nc * 2);
    p->retained = (int64_t *)xcalloc(nc, sizeof(int64_t));
    memcpy(p->retained, retained, sizeof(int64_t) * nc);
    p->xf = (cplx *)xcalloc(HW * Mx, sizeof(cplx));
    p->ring = (cplx *)xcalloc(HW * Mz * My * Mx, sizeof(cplx));
    p->sbins = (cplx *)xcalloc(HW * p->nb, sizeof(cplx));
    p->cond = (cplx *)xcalloc(HW * p->nb, sizeof(cplx));
    p->pw = (double *)xcalloc(HW * p->nb, sizeof(double));
    p->r = (double *)xcalloc(HW * nlx * nly, sizeof(double));
    p->rhat = (double *)xcalloc(HW * nlx * nly, sizeof(double));
    p->idx = (int32_t *)xcalloc(HW * 2, sizeof(int32_t));
    p->vel = (double *)xcalloc(HW * 2, sizeof(double));
    p->pred = (float *)xcalloc(HW, sizeof(float));
    p->res = (float *)xcalloc(HW, sizeof(float));
    p->imag = (float *)xcalloc(HW, sizeof(float));
    p->delay = (float *)xcalloc(HW * (p->mhz + 1), sizeof(float));
    if (!p->xf || !p->ring || !p->sbins || !p->cond || !p->pw || !p->r || !p->rhat || !p->delay)
        return NULL;
    return p;
}

void cwo_destroy(cwo_pipe *p)
{
    if (!p)
        return;
    void *ptrs[] = {p->ex, p->ey, p->ez, p->twx, p->twy, p->az, p->axl, p->ayl, p->lag_x, p->lag_y, p->gx,
                    p->gy, p->bank, p->retained, p->xf, p->ring, p->sbins, p->cond, p->pw, p->r, p->rhat,
                    p->idx, p->vel, p->pred, p->res, p->imag, p->delay};
    for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); i++)
        free(ptrs[i]);
    free(p);
}

void cwo_set_threads(cwo_pipe *p, int n) { p->nthreads = n < 1 ? 1 : n; }

/*
 * One Pipeline.process_frame (pipeline.py:201-294).  Returns 1 when an
 * output is ready (written to res/pred/idx/vel, *imag_peak, *frame_index),
 * 0 during warm-up.  forced_ix < 0 disables the forced velocity override
 * (pipeline.py:260-265).  timings (may be NULL): [spectrum, conditioning,
 * autocorr, filtering] seconds, as last_timings.
 */
static double now_s(void)
{
#ifdef _OPENMP
    return omp_get_wtime();
#else
    return 0.0;
#endif
}

int cwo_push(cwo_pipe *p, const float *frame, float *res, float *pred, int32_t *idx, double *vel,
             double *imag_peak, long long *frame_index, int forced_ix, int forced_iy, double *timings)
{
    const int H = p->H, W = p->W;
    const size_t HW = (size_t)H * W;
    double t0 = now_s();
    /* delay deque(maxlen=mhz+1) (pipeline.py:168,209): slot = n % (mhz+1) */
    long long n = p->frames_seen;
    memcpy(p->delay + (size_t)(n % (p->mhz + 1)) * HW, frame, sizeof(float) * HW);

    /* SpectrumStream.push (spectrum.py:192-243) */
    cplx *sp = p->ring + (size_t)(n % p->mz) * HW * p->my * p->mx;
    FORK(p, H, k_sdft_rows(p, frame, lo, hi));
    FORK(p, W, k_sdft_cols(p, sp, lo, hi));
    p->frames_seen++;
    if (p->frames_seen < p->mz) {
        if (timings)
            timings[0] = now_s() - t0;
        return 0;
    }
    int64_t slots[64];
    for (int m = 0; m < p->mz; m++)
        slots[m] = ((n - m) % p->mz + p->mz) % p->mz;
    FORK(p, H, k_temporal_dft(p, slots, lo, hi));
    double t1 = now_s();
    /* conditioning (pipeline.py:228-235) */
    FORK(p, H, k_copy_zero_dc(p, lo, hi));
    FORK(p, H, k_hann3(p, lo, hi));
    FORK(p, H, k_power(p, lo, hi));
    double t2 = now_s();
    /* flow (pipeline.py:239-265) */
    FORK(p, H, k_autocorr(p, lo, hi));
    if (!p->have_rhat) {
        memcpy(p->rhat, p->r, sizeof(double) * HW * p->lx * p->ly);
        p->have_rhat = 1;
    } else {
        FORK(p, H, k_smooth(p, lo, hi));
    }
    FORK(p, H, k_pick(p, lo, hi));
    if (forced_ix >= 0) {
        for (size_t i = 0; i < HW; i++) {
            p->idx[2 * i] = forced_ix;
            p->idx[2 * i + 1] = forced_iy;
            p->vel[2 * i] = p->lag_x[forced_ix];
            p->vel[2 * i + 1] = p->lag_y[forced_iy];
        }
    }
    double t3 = now_s();
    /* PEF (pipeline.py:269-282); delayed = frame n - mhz */
    const float *delayed = p->delay + (size_t)((n - p->mhz) % (p->mhz + 1)) * HW;
    FORK(p, H, k_pef(p, delayed, lo, hi));
    double t4 = now_s();
    if (res)
        memcpy(res, p->res, sizeof(float) * HW);
    if (pred)
        memcpy(pred, p->pred, sizeof(float) * HW);
    if (idx)
        memcpy(idx, p->idx, sizeof(int32_t) * HW * 2);
    if (vel)
        memcpy(vel, p->vel, sizeof(double) * HW * 2);
    if (imag_peak) {
        float mx = p->imag[0];
        for (size_t i = 1; i < HW; i++)
            if (p->imag[i] > mx)
                mx = p->imag[i];
        *imag_peak = (double)mx;
    }
    if (frame_index)
        *frame_index = n - p->mhz;
    if (timings) {
        timings[0] = t1 - t0;
        timings[1] = t2 - t1;
        timings[2] = t3 - t2;
        timings[3] = t4 - t3;
    }
    return 1;
}

/* Debug views for the parity tests: (H,W,Mz,My,Mx) c128 and (H,W,Ly,Lx) f64. */
const double *cwo_sbins(const cwo_pipe *p) { return (const double *)p->sbins; }
const double *cwo_rhat(const cwo_pipe *p) { return p->rhat; }
long long cwo_frames_seen(const cwo_pipe *p) { return p->frames_seen; }
