/*
 * escape_oracle.c -- CPU ORACLE for the escape-time hot path of arXiv 1611.03079.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_1611_03079_b200/csrc).
 *
 * Plain, slow, obviously-correct scalar C.  Citations: P:n = /root/reference/PAPER.md
 * line n, S:n = SPEC.md line n.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread
 * (FP contraction OFF, no FTZ/DAZ: every +, -, * below is one IEEE-754
 * round-to-nearest-even operation in the declared type.)
 *
 * Two operation sequences of the same count definition: the strict one
 * (oracle_escape_f32/f64, DESIGN.md §2 / reading c-9) and the FAST one
 * (oracle_escape_fma_f32/f64: explicit C99 fmaf/fma calls, each one correctly
 * rounded fused operation, on the doubled state; reading c-10 and its
 * supplement).
 */
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#if defined(__x86_64__) || defined(__i386__)
#include <xmmintrin.h>
#endif

#if !defined(FLT_EVAL_METHOD) || FLT_EVAL_METHOD != 0
#error "oracle requires FLT_EVAL_METHOD == 0 (each float op rounded in its own type)"
#endif
#if defined(__FAST_MATH__)
#error "oracle must not be built with -ffast-math"
#endif

/* ------------------------------------------------------------------------- */
/* Floating-point environment checks (reading c-9: no FTZ/DAZ,     */
/* no contraction).                                                          */
/* ------------------------------------------------------------------------- */

/* 1 iff MXCSR has FTZ (bit 15) and DAZ (bit 6) clear, i.e. denormals kept. */
int oracle_fp_env_ok(void) {
#if defined(__x86_64__) || defined(__i386__)
    unsigned int csr = _mm_getcsr();
    return ((csr & (1u << 15)) == 0) && ((csr & (1u << 6)) == 0);
#else
    return 1;
#endif
}

/* Contraction canaries: a*b+c written as two operations.  With contraction
 * off these return fl(fl(a*b)+c); a fused build would return fma(a,b,c). */
double oracle_mul_add_f64(double a, double b, double c) { return a * b + c; }
float oracle_mul_add_f32(float a, float b, float c) { return a * b + c; }

/* ------------------------------------------------------------------------- */
/* Region-covering routine ("pixels are scaled to the complex plane";   */
/* term from ref [8]).  DESIGN.md reading c-3: pixel centres, row 0 =  */
/* top, evaluated in binary64 with separately rounded ops:       */
/*   hx = half_w / W,  re(px) = center_re + (2px + 1 - W) * hx               */
/*   hy = half_h / H,  im(py) = center_im + (H - 1 - 2py) * hy               */
/* ------------------------------------------------------------------------- */

double oracle_pixel_re(double center_re, double half_w, int64_t width, int64_t px) {
    double hx = half_w / (double)width;
    double k = (double)(2 * px + 1 - width); /* exact: |k| < 2^53 */
    double off = k * hx;
    return center_re + off;
}

double oracle_pixel_im(double center_im, double half_h, int64_t height, int64_t py) {
    double hy = half_h / (double)height;
    double k = (double)(height - 1 - 2 * py);
    double off = k * hy;
    return center_im + off;
}

/* ------------------------------------------------------------------------- */
/* Escape time ("the number of iterations that initial value takes to   */
/* either diverge or not", limit 100; count definition, bailout S:73-75).*/
/* count = smallest n in [0, max_iter-1] with |Z_n|^2 > 4, else max_iter.     */
/* Operation sequence, exactly (reading c-9):        */
/*   xx = x*x; yy = y*y; m = xx + yy; if (m > 4) return n;                    */
/*   xy = x*y; x = (xx - yy) + cr; y = (xy + xy) + ci;                        */
/* ------------------------------------------------------------------------- */

int oracle_escape_f32(float zre, float zim, float cre, float cim, int max_iter) {
    float x = zre, y = zim;
    for (int n = 0; n < max_iter; ++n) {
        float xx = x * x;
        float yy = y * y;
        float m = xx + yy;
        if (m > 4.0f) return n;
        float xy = x * y;
        float t = xx - yy;
        float s = xy + xy;
        x = t + cre;
        y = s + cim;
    }
    return max_iter;
}

int oracle_escape_f64(double zre, double zim, double cre, double cim, int max_iter) {
    double x = zre, y = zim;
    for (int n = 0; n < max_iter; ++n) {
        double xx = x * x;
        double yy = y * y;
        double m = xx + yy;
        if (m > 4.0) return n;
        double xy = x * y;
        double t = xx - yy;
        double s = xy + xy;
        x = t + cre;
        y = s + cim;
    }
    return max_iter;
}

/* ------------------------------------------------------------------------- */
/* FAST-mode escape time: the same count definition with the FMA-contracted  */
/* operation sequence that DEFINES the *_FAST modes (reading c-10, */
/* §5 "State representation"; the paper fixes no contraction, so FAST is the */
/* project's own definition).  The state is kept doubled, X = 2x, Y = 2y,    */
/* CR = 2cr, CI = 2ci (each doubling exact: no overflow below 2^127), and    */
/* one iteration is, with C99's correctly rounded fmaf/fma:                   */
/*   YY = Y*Y; M = fma(X, X, YY); if (M > 16) return n;                       */
/*   T = fma(X, X, -YY); Y' = fma(X, Y, CI); X' = fma(T, 0.5, CR);             */
/* This is the FMA contraction of reading c-9's iteration scaled by 2 -- it   */
/* equals the unscaled contraction below (oracle_escape_fma_unscaled_*)       */
/* step by step whenever no unscaled product (x*x, y*y, 2x*y) is subnormal,   */
/* because then every rounding commutes with the power-of-two scaling; where */
/* one is subnormal the doubled product keeps bits the unscaled one loses     */
/* (reading c-10, "doubled state").                                 */
/* ------------------------------------------------------------------------- */

int oracle_escape_fma_f32(float zre, float zim, float cre, float cim, int max_iter) {
    float X = zre + zre, Y = zim + zim, CR = cre + cre, CI = cim + cim;
    for (int n = 0; n < max_iter; ++n) {
        float YY = Y * Y;
        float M = fmaf(X, X, YY);
        if (M > 16.0f) return n;
        float T = fmaf(X, X, -YY);
        float Yn = fmaf(X, Y, CI);
        X = fmaf(T, 0.5f, CR);
        Y = Yn;
    }
    return max_iter;
}

int oracle_escape_fma_f64(double zre, double zim, double cre, double cim, int max_iter) {
    double X = zre + zre, Y = zim + zim, CR = cre + cre, CI = cim + cim;
    for (int n = 0; n < max_iter; ++n) {
        double YY = Y * Y;
        double M = fma(X, X, YY);
        if (M > 16.0) return n;
        double T = fma(X, X, -YY);
        double Yn = fma(X, Y, CI);
        X = fma(T, 0.5, CR);
        Y = Yn;
    }
    return max_iter;
}

/* The unscaled FMA contraction of reading c-9's iteration (for the          */
/* equivalence pin in tests/test_oracle_fast.py only):                       */
/*   yy = y*y; m = fma(x, x, yy); if (m > 4) return n;                        */
/*   t = fma(x, x, -yy); y = fma(x + x, y, ci); x = t + cr;   (x + x exact)   */
int oracle_escape_fma_unscaled_f32(float zre, float zim, float cre, float cim, int max_iter) {
    float x = zre, y = zim;
    for (int n = 0; n < max_iter; ++n) {
        float yy = y * y;
        float m = fmaf(x, x, yy);
        if (m > 4.0f) return n;
        float t = fmaf(x, x, -yy);
        float yn = fmaf(x + x, y, cim);
        x = t + cre;
        y = yn;
    }
    return max_iter;
}

int oracle_escape_fma_unscaled_f64(double zre, double zim, double cre, double cim,
                                   int max_iter) {
    double x = zre, y = zim;
    for (int n = 0; n < max_iter; ++n) {
        double yy = y * y;
        double m = fma(x, x, yy);
        if (m > 4.0) return n;
        double t = fma(x, x, -yy);
        double yn = fma(x + x, y, cim);
        x = t + cre;
        y = yn;
    }
    return max_iter;
}

/* One pixel of a Julia frame (Z_0 from the pixel, fixed C) or of a
 * Mandelbrot parameter map (C from the pixel, Z_0 = 0).  precision is
 * 32 or 64; for 32 the double inputs are rounded to binary32 once (c-8). */
static int pixel_count_n(int mandel, int precision, double c_re, double c_im,
                         double center_re, double center_im, double half_w, double half_h,
                         int64_t width, int64_t height, int64_t px, int64_t py, int max_iter,
                         int nudge, int fast) {
    double re = oracle_pixel_re(center_re, half_w, width, px);
    double im = oracle_pixel_im(center_im, half_h, height, py);
    if (precision == 32) {
        int (*esc)(float, float, float, float, int) =
            fast ? oracle_escape_fma_f32 : oracle_escape_f32;
        float r = (float)re;
        for (int k = 0; k < nudge; ++k) r = nextafterf(r, INFINITY);
        if (mandel) return esc(0.0f, 0.0f, r, (float)im, max_iter);
        return esc(r, (float)im, (float)c_re, (float)c_im, max_iter);
    }
    int (*esc64)(double, double, double, double, int) =
        fast ? oracle_escape_fma_f64 : oracle_escape_f64;
    for (int k = 0; k < nudge; ++k) re = nextafter(re, INFINITY);
    if (mandel) return esc64(0.0, 0.0, re, im, max_iter);
    return esc64(re, im, c_re, c_im, max_iter);
}

static int pixel_count(int mandel, int precision, double c_re, double c_im, double center_re,
                       double center_im, double half_w, double half_h, int64_t width,
                       int64_t height, int64_t px, int64_t py, int max_iter, int fast) {
    return pixel_count_n(mandel, precision, c_re, c_im, center_re, center_im, half_w, half_h,
                         width, height, px, py, max_iter, 0, fast);
}

/* ------------------------------------------------------------------------- */
/* Whole-grid renderer: "a main loop to cover the pixel region", rows */
/* handed to threads dynamically (rows are independent).              */
/* out[py * width + px], row-major, uint16 counts (max_iter <= 65535).       */
/* ------------------------------------------------------------------------- */

typedef struct {
    int mandel, precision, max_iter;
    double c_re, c_im, center_re, center_im, half_w, half_h;
    int64_t width, height;
    uint16_t* out;
    /* pixel-list mode (n_pix > 0): px[i], py[i] -> out[i] */
    const int64_t* px;
    const int64_t* py;
    int64_t n_pix;
    int64_t next; /* shared work counter */
    int nudge;    /* ulps added to the start value's real part (0 = none) */
    int fast;     /* 1: the FAST (FMA-contracted) sequence, 0: strict */
} job_t;

static void* grid_worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (;;) {
        int64_t row = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (row >= j->height) break;
        for (int64_t px = 0; px < j->width; ++px)
            j->out[row * j->width + px] = (uint16_t)pixel_count(
                j->mandel, j->precision, j->c_re, j->c_im, j->center_re, j->center_im,
                j->half_w, j->half_h, j->width, j->height, px, row, j->max_iter, j->fast);
    }
    return NULL;
}

static void* list_worker(void* arg) {
    job_t* j = (job_t*)arg;
    const int64_t chunk = 64;
    for (;;) {
        int64_t i0 = __atomic_fetch_add(&j->next, chunk, __ATOMIC_RELAXED);
        if (i0 >= j->n_pix) break;
        int64_t i1 = i0 + chunk < j->n_pix ? i0 + chunk : j->n_pix;
        for (int64_t i = i0; i < i1; ++i)
            j->out[i] = (uint16_t)pixel_count_n(j->mandel, j->precision, j->c_re, j->c_im,
                                                j->center_re, j->center_im, j->half_w,
                                                j->half_h, j->width, j->height, j->px[i],
                                                j->py[i], j->max_iter, j->nudge, j->fast);
    }
    return NULL;
}

static int run_threads(job_t* j, int threads, void* (*fn)(void*)) {
    if (threads < 1) threads = 1;
    if (threads > 1024) threads = 1024;
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    if (!tids) return -1;
    int started = 0;
    for (int t = 1; t < threads; ++t) {
        if (pthread_create(&tids[t], NULL, fn, j) != 0) break;
        ++started;
    }
    fn(j);
    for (int t = 1; t <= started; ++t) pthread_join(tids[t], NULL);
    free(tids);
    return 0;
}

static int args_ok(int precision, int64_t width, int64_t height, int max_iter) {
    return (precision == 32 || precision == 64) && width >= 1 && height >= 1 && max_iter >= 1 &&
           max_iter <= 65535;
}

/* Julia frame.  Returns 0 on success, -1 on bad arguments. */
int oracle_julia(double c_re, double c_im, double center_re, double center_im, double half_w,
                 double half_h, int64_t width, int64_t height, int max_iter, int precision,
                 uint16_t* out, int threads) {
    if (!args_ok(precision, width, height, max_iter) || !out) return -1;
    job_t j = {0, precision, max_iter, c_re, c_im, center_re, center_im, half_w, half_h,
               width, height, out, NULL, NULL, 0, 0, 0};
    return run_threads(&j, threads, grid_worker);
}

/* Mandelbrot parameter map ("choosing values for C from the complex
 * plane (corresponding to pixels) ... Z_0 is given the value 0"). */
int oracle_mandel(double center_re, double center_im, double half_w, double half_h,
                  int64_t width, int64_t height, int max_iter, int precision, uint16_t* out,
                  int threads) {
    if (!args_ok(precision, width, height, max_iter) || !out) return -1;
    job_t j = {1, precision, max_iter, 0.0, 0.0, center_re, center_im, half_w, half_h,
               width, height, out, NULL, NULL, 0, 0, 0};
    return run_threads(&j, threads, grid_worker);
}

/* Sampled pixels of a Julia (mandel = 0) or Mandelbrot (mandel = 1) grid of
 * width x height: out[i] = count at (px[i], py[i]).  Used for parity at full
 * BASELINE sizes the oracle cannot finish whole. */
int oracle_pixels(int mandel, double c_re, double c_im, double center_re, double center_im,
                  double half_w, double half_h, int64_t width, int64_t height, int max_iter,
                  int precision, const int64_t* px, const int64_t* py, int64_t n_pix,
                  uint16_t* out, int threads) {
    if (!args_ok(precision, width, height, max_iter) || n_pix < 0) return -1;
    if (n_pix == 0) return 0;
    if (!px || !py || !out) return -1;
    for (int64_t i = 0; i < n_pix; ++i)
        if (px[i] < 0 || px[i] >= width || py[i] < 0 || py[i] >= height) return -1;
    job_t j = {mandel ? 1 : 0, precision, max_iter, c_re, c_im, center_re, center_im, half_w,
               half_h, width, height, out, px, py, n_pix, 0, 0};
    return run_threads(&j, threads, list_worker);
}

/* As oracle_pixels, with the start value's real part (Julia Z_0, Mandelbrot C) moved by
 * `nudge` ulps of the working precision toward +inf: the problem's own 1-ulp
 * sensitivity, against which fast-mode differences are judged (reading c-10). */
int oracle_pixels_nudged(int mandel, double c_re, double c_im, double center_re,
                         double center_im, double half_w, double half_h, int64_t width,
                         int64_t height, int max_iter, int precision, const int64_t* px,
                         const int64_t* py, int64_t n_pix, int nudge, uint16_t* out,
                         int threads) {
    if (!args_ok(precision, width, height, max_iter) || n_pix < 0 || nudge < 0) return -1;
    if (n_pix == 0) return 0;
    if (!px || !py || !out) return -1;
    for (int64_t i = 0; i < n_pix; ++i)
        if (px[i] < 0 || px[i] >= width || py[i] < 0 || py[i] >= height) return -1;
    job_t j = {mandel ? 1 : 0, precision, max_iter, c_re, c_im, center_re, center_im, half_w,
               half_h, width, height, out, px, py, n_pix, 0, nudge};
    return run_threads(&j, threads, list_worker);
}

/* FAST-mode frames and sampled pixels (oracle_escape_fma_*): the same grids and
 * start values as oracle_julia / oracle_mandel / oracle_pixels, iterated with the
 * FMA-contracted sequence that defines the *_FAST modes.  mandel selects the map. */
int oracle_frame_fma(int mandel, double c_re, double c_im, double center_re,
                     double center_im, double half_w, double half_h, int64_t width,
                     int64_t height, int max_iter, int precision, uint16_t* out, int threads) {
    if (!args_ok(precision, width, height, max_iter) || !out) return -1;
    job_t j = {mandel ? 1 : 0, precision, max_iter, c_re, c_im, center_re, center_im, half_w,
               half_h, width, height, out, NULL, NULL, 0, 0, 0, 1};
    return run_threads(&j, threads, grid_worker);
}

int oracle_pixels_fma(int mandel, double c_re, double c_im, double center_re,
                      double center_im, double half_w, double half_h, int64_t width,
                      int64_t height, int max_iter, int precision, const int64_t* px,
                      const int64_t* py, int64_t n_pix, uint16_t* out, int threads) {
    if (!args_ok(precision, width, height, max_iter) || n_pix < 0) return -1;
    if (n_pix == 0) return 0;
    if (!px || !py || !out) return -1;
    for (int64_t i = 0; i < n_pix; ++i)
        if (px[i] < 0 || px[i] >= width || py[i] < 0 || py[i] >= height) return -1;
    job_t j = {mandel ? 1 : 0, precision, max_iter, c_re, c_im, center_re, center_im, half_w,
               half_h, width, height, out, px, py, n_pix, 0, 0, 1};
    return run_threads(&j, threads, list_worker);
}

/* ------------------------------------------------------------------------- */
/* Colour levels ("assigned color levels according to the number of     */
/* iterations"; rule S:245): count == max_iter -> interior colour, else      */
/* palette[count mod n].  palette: n RGBA quadruples; out: RGBA per pixel.   */
/* ------------------------------------------------------------------------- */

int oracle_colorize(const uint16_t* counts, int64_t n_pixels, int max_iter,
                    const uint8_t* palette, int n, const uint8_t* interior, uint8_t* out) {
    if (n_pixels < 0 || n < 1 || max_iter < 1) return -1;
    for (int64_t i = 0; i < n_pixels; ++i) {
        const uint8_t* src;
        if ((int)counts[i] == max_iter)
            src = interior;
        else
            src = palette + 4 * ((int)counts[i] % n);
        out[4 * i + 0] = src[0];
        out[4 * i + 1] = src[1];
        out[4 * i + 2] = src[2];
        out[4 * i + 3] = src[3];
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* The paper's cardioid path: f(t) = ([2cos t - cos 2t]/a,            */
/* [2 sin t - sin 2t]/a), a = 3.9; "the border of the main cardioid of the   */
/* Mandelbrot set is this function when a = 4".                              */
/* ------------------------------------------------------------------------- */

void oracle_cardioid_point(double t, double a, double* re, double* im) {
    *re = (2.0 * cos(t) - cos(2.0 * t)) / a;
    *im = (2.0 * sin(t) - sin(2.0 * t)) / a;
}

/* ------------------------------------------------------------------------- */
/* Fast-mode tolerance tools (reading c-10).                        */
/* ------------------------------------------------------------------------- */

/* Distance estimate DE = |Z_n| ln|Z_n| / |Z'_n| in binary64 (standard exterior
 * distance estimator; Koebe-type bound: distance to the set boundary >= DE/2).
 * Julia: Z_0 = z0, Z'_0 = 1, Z'_{k+1} = 2 Z_k Z'_k.  Mandelbrot: Z_0 = 0, Z'_0 = 0,
 * Z'_{k+1} = 2 Z_k Z'_k + 1 (derivative in c).  Bailout |Z|^2 > 1e20; returns 0 if
 * the orbit has not escaped after max_iter iterations (treated as "in the set"). */
double oracle_distance_estimate(int mandel, double zre, double zim, double cre, double cim,
                                long max_iter) {
    double x = mandel ? 0.0 : zre, y = mandel ? 0.0 : zim;
    double dx = mandel ? 0.0 : 1.0, dy = 0.0;
    for (long n = 0; n < max_iter; ++n) {
        double m = x * x + y * y;
        if (m > 1e20) {
            double r = sqrt(m);
            double dr = sqrt(dx * dx + dy * dy);
            return r * log(r) / dr;
        }
        /* Z' <- 2 Z Z' (+1 for Mandelbrot), using the old Z */
        double ndx = 2.0 * (x * dx - y * dy) + (mandel ? 1.0 : 0.0);
        double ndy = 2.0 * (x * dy + y * dx);
        dx = ndx;
        dy = ndy;
        double nx = x * x - y * y + cre;
        double ny = 2.0 * x * y + cim;
        x = nx;
        y = ny;
    }
    return 0.0;
}

/* DE at selected pixel centres (exact binary64 pixel centres, reading c-3). */
int oracle_distance_pixels(int mandel, double c_re, double c_im, double center_re,
                           double center_im, double half_w, double half_h, int64_t width,
                           int64_t height, const int64_t* px, const int64_t* py, int64_t n_pix,
                           long max_iter, double* out) {
    if (width < 1 || height < 1 || n_pix < 0) return -1;
    for (int64_t i = 0; i < n_pix; ++i) {
        if (px[i] < 0 || px[i] >= width || py[i] < 0 || py[i] >= height) return -1;
        double re = oracle_pixel_re(center_re, half_w, width, px[i]);
        double im = oracle_pixel_im(center_im, half_h, height, py[i]);
        out[i] = mandel ? oracle_distance_estimate(1, 0.0, 0.0, re, im, max_iter)
                        : oracle_distance_estimate(0, re, im, c_re, c_im, max_iter);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* NEXT-3: other iteration maps ("many other functions yield fruitful    */
/* explorations"; Figure 4, garbled as z^4 + (z^2+1)/(z^2+1) + c and   */
/* read per SPEC S:35 as z^4 + (z^2+1)/(z^2-1) + c; reading c-14). */
/* fn 0: z^2 + c;  fn 1: z^4 + c;  fn 2: z^4 + (z^2+1)/(z^2-1) + c.           */
/* Same count definition and bailout |Z_n|^2 > 4.  Operation sequence:        */
/*   w = z^2 = (xx - yy, xy + xy);  z^4 = w^2 = (wx*wx - wy*wy, p + p),       */
/*   p = wx*wy;  rational: q = (w + 1)/(w - 1) by the textbook formula        */
/*   ((a c + b d) + i (b c - a d)) / (c^2 + d^2); pole (c^2 + d^2 == 0):      */
/*   Z_{n+1} = +inf (escapes at the next test).                     */
/* ------------------------------------------------------------------------- */

#define DEF_FN_ESCAPE(NAME, T, LIM)                                                   \
    int NAME(int fn, T zre, T zim, T cre, T cim, int max_iter) {                     \
        T x = zre, y = zim;                                                           \
        for (int n = 0; n < max_iter; ++n) {                                          \
            T xx = x * x;                                                             \
            T yy = y * y;                                                             \
            T m = xx + yy;                                                            \
            if (m > LIM) return n;                                                    \
            T xy = x * y;                                                             \
            T wx = xx - yy;                                                           \
            T wy = xy + xy;                                                           \
            if (fn == 0) {                                                            \
                x = wx + cre;                                                         \
                y = wy + cim;                                                         \
                continue;                                                             \
            }                                                                         \
            T u = wx * wx;                                                            \
            T v = wy * wy;                                                            \
            T p = wx * wy;                                                            \
            T fx = u - v;                                                             \
            T fy = p + p;                                                             \
            if (fn == 2) {                                                            \
                T a = wx + (T)1;                                                      \
                T c = wx - (T)1;                                                      \
                T b = wy;                                                             \
                T d = wy;                                                             \
                T den = c * c + d * d;                                                \
                if (den == (T)0) {                                                    \
                    x = (T)INFINITY;                                                  \
                    y = (T)0;                                                         \
                    continue;                                                         \
                }                                                                     \
                T qx = (a * c + b * d) / den;                                         \
                T qy = (b * c - a * d) / den;                                         \
                fx = fx + qx;                                                         \
                fy = fy + qy;                                                         \
            }                                                                         \
            x = fx + cre;                                                             \
            y = fy + cim;                                                             \
        }                                                                             \
        return max_iter;                                                              \
    }

DEF_FN_ESCAPE(oracle_escape_fn_f32, float, 4.0f)
DEF_FN_ESCAPE(oracle_escape_fn_f64, double, 4.0)

/* Julia frame of map fn (single-threaded rows are fine for test sizes). */
int oracle_julia_fn(int fn, double c_re, double c_im, double center_re, double center_im,
                    double half_w, double half_h, int64_t width, int64_t height, int max_iter,
                    int precision, uint16_t* out) {
    if (!args_ok(precision, width, height, max_iter) || !out || fn < 0 || fn > 2) return -1;
    for (int64_t py = 0; py < height; ++py)
        for (int64_t px = 0; px < width; ++px) {
            double re = oracle_pixel_re(center_re, half_w, width, px);
            double im = oracle_pixel_im(center_im, half_h, height, py);
            out[py * width + px] =
                (uint16_t)(precision == 32
                               ? oracle_escape_fn_f32(fn, (float)re, (float)im, (float)c_re,
                                                      (float)c_im, max_iter)
                               : oracle_escape_fn_f64(fn, re, im, c_re, c_im, max_iter));
        }
    return 0;
}
